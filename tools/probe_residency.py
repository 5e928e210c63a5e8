"""Measures how many fused-kernel CTAs are co-resident per SM (PLBM_PROBE)."""
import ctypes as C
import os
import sys
import numpy as np

os.environ["PLBM_PROBE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_03560_b200 import capi, scenario as S  # noqa: E402

sc = S.mpmc_release(n=256, extent=32, threshold=1e-9)
eng = capi.gpu_engine(sc)
eng.step(int(sys.argv[1]) if len(sys.argv) > 1 else 100)
eng.sync()
lib = eng.lib
lib.plbm_gpu_probe.restype = C.c_int
lib.plbm_gpu_probe.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
buf = np.zeros(3 * 513 * 16, np.uint64)
n = lib.plbm_gpu_probe(eng._h, buf.ctypes.data_as(C.c_void_p), buf.size)
rec = buf[:3 * n].reshape(n, 3)
rec = rec[rec[:, 1] > 0]
sm, t0, t1 = rec[:, 0].astype(int), rec[:, 1].astype(np.int64), rec[:, 2].astype(np.int64)
base = t0.min()
t0 -= base
t1 -= base
print("CTAs", len(rec), "SMs used", len(set(sm)), "kernel span us", (t1.max()) / 1e3)
events = sorted([(a, 1) for a in t0] + [(b, -1) for b in t1])
cur = mx = 0
for _, d in events:
    cur += d
    mx = max(mx, cur)
print("max concurrent CTAs (GPU)", mx)
per = {}
for s in set(sm):
    ev = sorted([(a, 1) for a, ss in zip(t0, sm) if ss == s] + [(b, -1) for b, ss in zip(t1, sm) if ss == s])
    c = m = 0
    for _, d in ev:
        c += d
        m = max(m, c)
    per[s] = m
vals = np.array(list(per.values()))
print("max concurrent CTAs per SM: histogram", {int(k): int((vals == k).sum()) for k in np.unique(vals)})
print("mean CTA duration us", float((t1 - t0).mean()) / 1e3)
