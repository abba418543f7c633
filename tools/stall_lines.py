"""Warp-stall samples per CUDA source line from
`ncu -i REP --page source --csv --kernel-name regex:K --print-source cuda,sass`.
python tools/stall_lines.py CSV [top]"""
import csv
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
ism = h.index("Warp Stall Sampling (All Samples)")
st = [i for i, k in enumerate(h) if k.startswith("stall_") and "Not Issued" not in k]
samp = Counter()
why = defaultdict(Counter)
src = {}
for r in rows[hi + 1:]:
    if len(r) < len(h) or not r[0].isdigit():
        continue
    ln = int(r[0])
    src[ln] = r[1]
    try:
        samp[ln] += float(r[ism] or 0)
    except ValueError:
        continue
    for i in st:
        why[ln][h[i][6:]] += float(r[i] or 0)
T = sum(samp.values()) or 1
for ln, v in samp.most_common(top):
    w = " ".join(f"{k}:{int(x)}" for k, x in why[ln].most_common(2))
    print(f"{100 * v / T:5.1f}% L{ln:4d} {src[ln].strip()[:70]:70s} {w}")
