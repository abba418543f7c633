"""Per-frame DRAM traffic of the query path from an ncu launch list:

  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none --csv --log-file gpurun_out/traffic.csv \
      python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-comparator
  python tools/traffic.py gpurun_out/traffic.csv > profiles/query_path_traffic.json

Takes the launches of the last frame (from its units kernel through the next
frame's units kernel / the end) and sums the query-path kernels (everything
but the units kernel and the temporal-change tree)."""
import csv
import json
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
iu = h.index("Metric Unit")
SCALE = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
by = defaultdict(dict)
names = {}
for r in rows[1:]:
    i = int(r[iid])
    names[i] = r[ik]
    by[i][r[im]] = float(r[iv].replace(",", "")) * SCALE.get(r[iu], 1.0)
ids = sorted(by)
units = [i for i in ids if "units" in names[i]]
start = units[-2] if len(units) > 1 else ids[0]
end = units[-1]
frame = [i for i in ids if start <= i < end]
launches, rd, wr, ms = [], 0.0, 0.0, 0.0
for i in frame:
    m = by[i]
    t = m.get("gpu__time_duration.sum", 0.0)  # ms
    r_, w_ = m.get("dram__bytes_read.sum", 0.0), m.get("dram__bytes_write.sum", 0.0)
    launches.append({"kernel": names[i], "ms": t, "dram_read_GB": r_ / 1e9, "dram_write_GB": w_ / 1e9})
    if "units" in names[i] or "pw_tree" in names[i]:
        continue
    rd += r_
    wr += w_
    ms += t
json.dump({"config": "cfg3_1080p_rgb",
           "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum over the "
                     "last frame of `python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-comparator` "
                     "(serialised, cold-cache launches); tools/traffic.py",
           "dram_bytes_per_frame": rd + wr, "query_path_ms_serialised": ms,
           "frame_dram_read_bytes": rd, "frame_dram_write_bytes": wr, "launches": launches},
          sys.stdout, indent=1)
