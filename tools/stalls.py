"""Stall summary of one kernel from `ncu -i REP --page source --csv --kernel-name regex:K`
(SASS view): stall reasons over all samples and the hottest instructions.
python tools/stalls.py CSV [top]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
h = rows[1]
ia, isrc, ismp = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
st = [i for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
tot = Counter()
ins = []
for r in rows[2:]:
    if len(r) < len(h) or r[ia] == "Address":
        continue
    s = float(r[ismp] or 0)
    c = Counter()
    for i in st:
        v = float(r[i] or 0)
        tot[h[i]] += v
        c[h[i]] = v
    ins.append((s, r[ia], r[isrc], c.most_common(2)))
T = sum(tot.values())
print("stall reasons:", ", ".join(f"{k[6:]} {100 * v / T:.1f}%" for k, v in tot.most_common(8)))
S = sum(x[0] for x in ins)
for s, a, src, c in sorted(ins, reverse=True)[:top]:
    print(f"{100 * s / S:5.1f}% {a} {src[:60]:60s} {' '.join(f'{k[6:]}:{int(v)}' for k, v in c)}")
