"""Cluster placement of the fused kernel (PLBM_PROBE build): for every
8-CTA cluster of k_main_pc<32, 2>, which cluster ranks share an SM, and the
CTA durations by rank (component c = rank / NB, or rank % C with
-DPLBM_RANK_IL).

    PLBM_GPU_LIB=... python tools/probe_cluster.py [steps]
"""
import ctypes as C
import os
import sys
from collections import Counter, defaultdict

import numpy as np

os.environ["PLBM_PROBE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1510_03560_b200 import capi, scenario as S  # noqa: E402

CL = 8
sc = S.bench_c2()
eng = capi.gpu_engine(sc)
eng.step(int(sys.argv[1]) if len(sys.argv) > 1 else 105)
eng.sync()
lib = eng.lib
lib.plbm_gpu_probe.restype = C.c_int
lib.plbm_gpu_probe.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
buf = np.zeros(3 * 513 * 16, np.uint64)
n = lib.plbm_gpu_probe(eng._h, buf.ctypes.data_as(C.c_void_p), buf.size)
rec = buf[:3 * n].reshape(n, 3).astype(np.int64)
ok = rec[:, 1] > 0
idx = np.nonzero(ok)[0]
pairs = Counter()
dur = defaultdict(list)
skew = []
for cl in range(int(idx.max()) // CL + 1):
    ranks = [b for b in range(cl * CL, cl * CL + CL) if b < len(rec) and rec[b, 1] > 0]
    if len(ranks) < CL:
        continue
    sm = {b - cl * CL: int(rec[b, 0]) for b in ranks}
    by_sm = defaultdict(list)
    for r, s_ in sm.items():
        by_sm[s_].append(r)
    for s_, rs in by_sm.items():
        if len(rs) == 2:
            pairs[tuple(sorted(rs))] += 1
    for b in ranks:
        dur[b - cl * CL].append(rec[b, 2] - rec[b, 1])
    ends = [rec[b, 2] for b in ranks]
    skew.append(max(ends) - min(ends))
print("rank pairs sharing an SM (count over clusters):", dict(pairs.most_common(12)))
print("mean CTA duration us by rank:", {r: round(float(np.mean(v)) / 1e3, 1) for r, v in sorted(dur.items())})
print("mean end skew within a cluster us:", round(float(np.mean(skew)) / 1e3, 2))
