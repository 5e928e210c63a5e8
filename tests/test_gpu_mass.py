"""Mass conservation per component (north star: "total mass per component
must be conserved to a stated bound").

Stated bound: relative drift |m(k) - m(0)| / m(0) < 1e-10 per component, the
reference's own acceptance bound (proj/tests/acceptance.cpp:206-237, criterion
2, measured there at 6.1e-12).  m = sum over fluid cells of sum_i f (the
reference's interior_mass, acceptance.cpp:130-143), here the exactly rounded
sum (math.fsum) of the gathered density field (rho = sum_i f, 0 on solids).

Only closed systems conserve mass: solid walls with bounce-back, or periodic
boundaries, and a static mesh (a progressive mesh exchanges populations with
the ambient region by construction: absent neighbours supply feq_amb).

* acceptance criterion 2 on the B200 engine: 32^3 closed box, one 32^3 tile,
  tau 0.9, 1000 steps, drift checked every 100 steps; the final density field
  must also equal the reference engine's bit for bit;
* the bench workload's physics at full size: 256^3, 32^3 tiles, two-component
  Peng-Robinson MPMC, fully periodic, static, 100 steps.
"""
import math

import numpy as np
import pytest

from paper_1510_03560_b200 import capi
from paper_1510_03560_b200 import scenario as S
from tests.conftest import have_ref

BOUND = 1e-10


def _mass(eng, c):
    return math.fsum(eng.gather_field("rho", c).ravel().tolist())


def _closed_box_32():
    n = 32
    sc = S.Scenario(domain=(n, n, n), tile_extent=32, mode=S.MODE_STATIC,
                    components=[S.Component(tau=0.9)],
                    seeds=[S.Seed(box_min=(8, 8, 8), box_max=(24, 24, 24), rho=1.2,
                                  velocity=(0.04, 0.02, 0.01))])
    g = np.zeros((n, n, n), np.uint8)
    g[0, :, :] = g[-1, :, :] = g[:, 0, :] = g[:, -1, :] = g[:, :, 0] = g[:, :, -1] = 1
    sc.geometry = g
    return sc


@pytest.mark.gpu
def test_acceptance_c2_closed_box_mass(built, tmp_path):
    sc = _closed_box_32()
    eng = capi.gpu_engine(sc)
    m0 = _mass(eng, 0)
    worst = 0.0
    for _ in range(10):
        eng.step(100)
        worst = max(worst, abs(_mass(eng, 0) - m0) / m0)
    print(f"closed box 32^3, 1000 steps: max relative mass drift {worst:.3e}")
    assert worst < BOUND
    if have_ref():
        ref = capi.ref_engine(sc)
        ref.step(1000)
        a, b = str(tmp_path / "gpu"), str(tmp_path / "ref")
        eng.dump_field("rho", 0, 1000, a, False)
        ref.dump_field("rho", 0, 1000, b, False)
        assert open(a + ".raw", "rb").read() == open(b + ".raw", "rb").read()
        ref.close()
    eng.close()


@pytest.mark.gpu
def test_bench_physics_periodic_mass_full_size(built):
    sc = S.mpmc_release(n=256, extent=32, mode=S.MODE_STATIC)
    sc.periodic = (1, 1, 1)
    eng = capi.gpu_engine(sc)
    m0 = [_mass(eng, c) for c in range(sc.n_components)]
    eng.step(100)
    c = eng.counters()
    assert c["iteration"] == 100 and c["tiles"] == 512
    for k in range(sc.n_components):
        drift = abs(_mass(eng, k) - m0[k]) / m0[k]
        print(f"256^3 periodic MPMC, component {k}: relative mass drift after 100 steps {drift:.3e}")
        assert drift < BOUND
    eng.close()
