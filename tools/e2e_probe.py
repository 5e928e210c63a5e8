"""Host-side cost of the reference driver's loop (one plbm_gpu_step + one
plbm_gpu_counters per iteration) on the C2 bench workload: per-call host
times against the device time of the same steps."""
import json
import sys
import time

import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_1510_03560_b200 import capi, scenario as S  # noqa: E402

eng = capi.gpu_engine(S.bench_c2())
eng.step(100)
eng.sync()
stream = torch.cuda.ExternalStream(eng.stream())
for _ in range(5):
    eng.step(1)
    eng.counters()
n = 30
t_step = t_cnt = 0.0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(stream)
T0 = time.perf_counter()
for _ in range(n):
    a = time.perf_counter()
    eng.step(1)
    b = time.perf_counter()
    eng.counters()
    c = time.perf_counter()
    t_step += b - a
    t_cnt += c - b
T1 = time.perf_counter()
e1.record(stream)
torch.cuda.synchronize()
eng.step(n)  # the same number of steps queued back to back
e2 = torch.cuda.Event(enable_timing=True)
e3 = torch.cuda.Event(enable_timing=True)
e2.record(stream)
eng.step(n)
e3.record(stream)
torch.cuda.synchronize()
print(json.dumps({"loop_ms_per_step": round((T1 - T0) * 1e3 / n, 4),
                  "step_call_ms": round(t_step * 1e3 / n, 4), "counters_call_ms": round(t_cnt * 1e3 / n, 4),
                  "loop_device_ms_per_step": round(e0.elapsed_time(e1) / n, 4),
                  "queued_device_ms_per_step": round(e2.elapsed_time(e3) / n, 4)}))
