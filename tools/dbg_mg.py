"""Debug helper: several ranks in one process (device protocol) vs one engine,
field by field after every step."""
import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
from paper_1510_03560_b200 import capi, dist, scenario as S
from tests import scenarios
from tests.test_multigpu import _attach
from tests.compare import FIELDS

def make_named(name):
    if name == "static_e32":
        return S.mpmc_release(n=64, extent=32, mode=S.MODE_STATIC, r_core=8, devices=2), 6
    make, steps = scenarios.ALL[name]
    return make(), steps

for name in sys.argv[1:]:
    for protocol in ("device",):
        sc, steps = make_named(name)
        sc.devices = max(sc.devices, 2)
        single = capi.gpu_engine(sc, capture=True)
        engs = _attach(sc, 2)
        for k in range(1, 4):
            single.step(1)
            t0 = time.time()
            try:
                if protocol == "device":
                    dist.step_ranks_threaded(engs, 1)
                else:
                    dist.step_same_process(engs, 1)
            except Exception as ex:
                print(name, protocol, "step", k, "EXC", ex, round(time.time() - t0, 2), flush=True)
                break
            bad = []
            for coords, _, _ in single.tiles():
                r = engs[0].tile_rank(coords)
                for comp in range(sc.n_components):
                    for f in FIELDS:
                        a = single.read_tile(coords, comp, f); b = engs[r].read_tile(coords, comp, f)
                        if not np.array_equal(a.view(np.uint64), b.view(np.uint64)):
                            d = np.abs(a - b); idx = np.unravel_index(np.argmax(d), d.shape)
                            bad.append((coords, r, comp, f, float(d.max()), idx, int((d > 0).sum())))
            print(name, protocol, "step", k, round(time.time() - t0, 3), "bad", len(bad), bad[:3], flush=True)
            if bad:
                break
        for e in engs:
            e.close()
        single.close()
