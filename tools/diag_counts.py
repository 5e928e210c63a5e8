import sys; sys.path.insert(0, "/root/repo")
from paper_1510_03560_b200 import capi
from tests import scenarios
for name in sorted(scenarios.ALL):
    make, steps = scenarios.ALL[name]
    sc = make()
    e = capi.gpu_engine(sc)
    e.step(steps)
    c = e.counters()
    print(name, c["negative_populations"], c["psi_clamps"], c["zero_rho_forcings"])
    e.close()
