"""Device time per step of plbm_gpu_step(h, n) (queued steps) against
plbm_gpu_step(h, 1) per call, for the speculation depths (PLBM_SPEC_DEPTH)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_03560_b200 import capi, scenario as S  # noqa: E402

depth = os.environ.get("PLBM_SPEC_DEPTH", "default")
eng = capi.gpu_engine(S.bench_c2())
eng.step(110)
eng.sync()
stream = torch.cuda.ExternalStream(eng.stream())
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
n = 40
torch.cuda.synchronize()
ev[0].record(stream)
eng.step(n)
ev[1].record(stream)
torch.cuda.synchronize()
ev[2].record(stream)
for _ in range(n):
    eng.step(1)
ev[3].record(stream)
torch.cuda.synchronize()
print(json.dumps({"depth": depth, "queued_ms": round(ev[0].elapsed_time(ev[1]) / n, 4),
                  "single_ms": round(ev[2].elapsed_time(ev[3]) / n, 4)}))
