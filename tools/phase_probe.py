"""Per-warp cycle accounting of k_main_pc's plane loop (measurement build
with -DPLBM_PHASES; see build.py --exp).  Prints, per warp of the CTA, the
share of cycles in each phase of the plane loop, averaged over the timed
steps of the bench workload.

    PLBM_GPU_LIB=build/exp/libphases.so python tools/phase_probe.py [variant]
"""
import ctypes as C
import os
import sys

import numpy as np

os.environ["PLBM_PROBE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_03560_b200 import capi, scenario as S  # noqa: E402

PH = ["land_wait", "psi_pass", "issue_pulls", "coll_head", "poll_wait", "barrier", "flush_ring", "collide"]
sc = S.bench_c2()
eng = capi.gpu_engine(sc)
if len(sys.argv) > 1:
    eng.set_kernel_variant(int(sys.argv[1]))
lib = eng.lib
lib.plbm_gpu_probe.restype = C.c_int
lib.plbm_gpu_probe.argtypes = [C.c_void_p, C.c_void_p, C.c_int]


def snap():
    buf = np.zeros(3 * 16 * 600, np.uint64)
    lib.plbm_gpu_probe(eng._h, buf.ctypes.data_as(C.c_void_p), buf.size)
    return buf[:64].astype(np.float64).reshape(8, 8)


eng.step(105)
a = snap()
eng.step(10)
b = snap()
d = b - a
tot = d.sum(axis=1, keepdims=True)
print("warp " + " ".join(f"{p:>11s}" for p in PH) + "   Mcycles")
for w in range(8):
    print(f"{w:4d} " + " ".join(f"{100 * d[w, k] / tot[w, 0]:10.1f}%" for k in range(8)) + f"  {tot[w, 0] / 1e6:8.1f}")
s = d.sum(axis=0)
print(" all " + " ".join(f"{100 * s[k] / s.sum():10.1f}%" for k in range(8)))
