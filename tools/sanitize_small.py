"""A few fused-kernel steps for compute-sanitizer racecheck / synccheck."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_03560_b200 import capi  # noqa: E402
from tests import scenarios  # noqa: E402

for name in sys.argv[1:] or ["mpmc_progressive_e16", "mpmc_e32"]:
    for storage in ("ab", "aa"):
        e = capi.gpu_engine(scenarios.ALL[name][0](), storage=storage)
        e.step(3)
        e.close()
        print("ok", name, storage, flush=True)
