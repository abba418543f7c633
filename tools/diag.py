"""Step-by-step GPU diagnostic (development)."""
import sys
import time

sys.path.insert(0, ".")
T0 = time.time()


def log(*a):
    print(f"[{time.time() - T0:7.2f}s]", *a, flush=True)


import numpy as np

log("numpy")
import paper_1508_07953_b200 as R

log("import pkg")
u, nr = R.normalize_rows(np.ones((2, 4), np.float32))
log("normalize_rows", u[0], nr)
s = np.float32(np.sqrt(2) / 2)
tri = R.ReferenceModel.from_refs(np.array([[1, 0], [0, 1], [s, s]], np.float32), (2, 1))
log("tri tables", tri.sorted_idx.tolist())
log("ring", R.ring_candidates(tri, 0, 0.765367, 0.191342))
r = R.riann_query(tri, tri.refs[2], 0)
log("query generic", r)
from paper_1508_07953_b200 import workloads as W

cfg = W.CONFIGS[0]
frames = W.clip(cfg, 2)
refs = W.reference_set(cfg)
log("data")
m = R.ReferenceModel.from_refs(refs, cfg.patch)
m.table_rows(0, 1)
log("cfg0 tables")
r = R.riann_query(m, refs[5], 7)
log("query D64", r.match_index, r.rings_drawn, r.distance_evals)
f0 = R.init_field(57, 57, m.n)
f1, st = R.process_frame(frames[0], f0, m)
log("process_frame", st)
