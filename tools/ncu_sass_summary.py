"""Summarise an ncu --page source --csv --print-source sass export:
dynamic instruction mix and stall samples by opcode and by code region."""
import csv
import re
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
ops = Counter()
stall = Counter()
stall_by_reason = Counter()
seq = []
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
for r in rows[2:]:
    if len(r) < len(h):
        continue
    src = r[idx["Source"]].strip()
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", src)
    if not m:
        continue
    op = m.group(2)
    n = int(r[idx["Thread Instructions Executed"]] or 0)
    s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    ops[op] += n
    stall[op] += s
    for k in reasons:
        v = r[idx[k]]
        if v and v != "0":
            stall_by_reason[k] += int(v)
    seq.append((r[idx["Address"]], src, n, s))
tot = sum(ops.values())
den = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
print(f"total thread instructions {tot:.4g}  per unit {tot/den:.1f}")
for op, n in ops.most_common(30):
    print(f"{op:10s} {n/den:9.1f}  stall samples {stall[op]}")
print("stall reasons:")
ts = sum(stall_by_reason.values())
for k, v in stall_by_reason.most_common(12):
    print(f"  {k:28s} {v:8d} {100*v/ts:5.1f}%")
if len(sys.argv) > 3:
    top = sorted(seq, key=lambda t: -t[3])[: int(sys.argv[3])]
    for a, src, n, s in top:
        print(f"{s:7d} {n/den:7.2f} {src}")
