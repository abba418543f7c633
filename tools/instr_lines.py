"""Executed warp instructions and lane utilisation per CUDA source line from
`ncu -i REP --page source --csv --kernel-name regex:K --print-source cuda,sass`.
python tools/instr_lines.py CSV [top]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hi]
ie, ite = h.index("Instructions Executed"), h.index("Thread Instructions Executed")
cnt, tcnt, src = Counter(), Counter(), {}
for r in rows[hi + 1:]:
    if len(r) < len(h) or not r[0].isdigit():
        continue
    ln = int(r[0])
    src[ln] = r[1]
    try:
        cnt[ln] += float(r[ie] or 0)
        tcnt[ln] += float(r[ite] or 0)
    except ValueError:
        pass
T = sum(cnt.values()) or 1
print(f"warp instr {T:.3g}, lane utilisation {sum(tcnt.values()) / T / 32:.2f}")
for ln, v in cnt.most_common(top):
    print(f"{100 * v / T:5.1f}% util {tcnt[ln] / v / 32 if v else 0:4.2f} L{ln:4d} {src[ln].strip()[:72]}")
