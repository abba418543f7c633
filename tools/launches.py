"""Summarise an ncu launch list (gpu__time_duration.sum [, dram bytes]) of the
last frame: per kernel name, count and total ms.  python tools/launches.py CSV"""
import csv
import sys
from collections import OrderedDict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, im, iv, iid, iu = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Metric Unit"))
SC = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}
L = OrderedDict()
for r in rows[1:]:
    if r[im] == "gpu__time_duration.sum":
        L[int(r[iid])] = (r[ik], float(r[iv].replace(",", "")) * SC.get(r[iu], 1.0))
ids = sorted(L)
units = [i for i in ids if "units" in L[i][0]]
start = units[-1] if units else ids[0]
agg = OrderedDict()
for i in ids:
    if i < start:
        continue
    name = L[i][0].split("(")[0][:70]
    c, t = agg.get(name, (0, 0.0))
    agg[name] = (c + 1, t + L[i][1])
tot = 0.0
for k, (c, t) in agg.items():
    print(f"{t:8.2f} ms  x{c:<3d} {k}")
    tot += t
print(f"{tot:8.2f} ms  total (last frame, serialised)")
