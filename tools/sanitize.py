"""Small runs of every kernel path for compute-sanitizer (memcheck):
A-B and A-A storage, E = 8 / 16 / 32 / 64, progressive with births, solids,
periodic axes, and 2 in-process ranks with the device protocol.

    compute-sanitizer --tool memcheck python tools/sanitize.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_03560_b200 import capi, dist  # noqa: E402
from tests import scenarios  # noqa: E402

CASES = ["c1_progressive", "mpmc_progressive_e16", "mpmc_e32", "mpmc_e32_solid_periodic", "mpmc_e64",
         "mpmc3_e64_solid", "mpmc_channel_e16", "mpmc3_static"]
for name in CASES:
    make, steps = scenarios.ALL[name]
    for storage in ("ab", "aa"):
        sc = make()
        if storage == "aa" and sc.tile_extent == 64 and sc.n_components > 2:
            continue
        e = capi.gpu_engine(sc, capture=True, storage=storage)
        e.step(min(steps, 6))
        e.read_tile(e.tiles()[0][0], 0, 0)
        e.close()
        print("ok", name, storage, flush=True)
# two ranks, device protocol
sc = scenarios.ALL["mpmc_progressive_e16"][0]()
sc.devices = 2
engs = [capi.gpu_engine(sc, rank=r, world=2) for r in range(2)]
pools = [e.pool_pointers() for e in engs]
engs[0].set_peer_pools(1, pools[1])
engs[1].set_peer_pools(0, pools[0])
for e in engs:
    e.prepare()
dist.step_ranks_threaded(engs, 5)
print("ok ranks", engs[0].counters()["tiles"], flush=True)
