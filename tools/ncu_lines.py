"""Attribute ncu per-SASS stall samples to CUDA source lines.
usage: ncu_lines.py <sass.csv from ncu --page source --print-source sass> <nvdisasm -g -c dump>
                    <mangled kernel> <units> [csrc dir]"""
import csv
import os
import re
import sys
from collections import Counter, defaultdict

csvf, dis, kern, units = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
srcdir = sys.argv[5] if len(sys.argv) > 5 else os.path.join(os.path.dirname(__file__), "..",
                                                             "paper_1510_03560_b200", "csrc")
txt = open(dis).read().splitlines()
start = next(i for i, l in enumerate(txt) if l.startswith(f".text.{kern}:"))
offs, line = {}, None
for l in txt[start + 1:]:
    if l.startswith(".text.") or l.strip().startswith(".section"):
        break
    m = re.search(r'## File "([^"]+)", line (\d+)', l)
    if m:
        line = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        offs[int(m.group(1), 16)] = line
rows = list(csv.reader(open(csvf)))
h = rows[1]
ix = {k: i for i, k in enumerate(h)}
body = [r for r in rows[2:] if len(r) >= len(h)]
base = int(body[0][0], 16)
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
by, byn, byr = Counter(), Counter(), defaultdict(Counter)
for r in body:
    key = offs.get(int(r[0], 16) - base)
    by[key] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    byn[key] += int(r[ix["Thread Instructions Executed"]] or 0)
    for k in reasons:
        v = r[ix[k]]
        if v and v != "0":
            byr[key][k] += int(v)
tot = sum(by.values())
cache = {}


def src(f, n):
    if f not in cache:
        p = os.path.join(srcdir, f)
        cache[f] = open(p).read().splitlines() if os.path.exists(p) else []
    L = cache[f]
    return L[n - 1].strip()[:64] if 0 < n <= len(L) else "?"


print(f"samples {tot}, instructions/unit {sum(byn.values())/units:.1f}")
for k, v in by.most_common(int(sys.argv[6]) if len(sys.argv) > 6 else 40):
    t = src(*k) if k else ""
    top = ", ".join(f"{a[6:]}:{b}" for a, b in byr[k].most_common(3))
    print(f"{v:6d} {100*v/tot:5.1f}% {byn[k]/units:6.1f} {k[0][:10] if k else ''}:{k[1] if k else ''} {t} | {top}")
