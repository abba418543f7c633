"""Quick per-frame timing of the GPU path on a config (development probe)."""
import argparse
import sys
import time

sys.path.insert(0, ".")
import numpy as np

import paper_1508_07953_b200 as R
from paper_1508_07953_b200 import workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=1)
ap.add_argument("--frames", type=int, default=8)
a = ap.parse_args()
cfg = W.CONFIGS[a.cfg]
t0 = time.time()
frames = W.clip(cfg, a.frames)
refs = W.reference_set(cfg)
print(f"cfg{a.cfg}: data {time.time() - t0:.1f}s", flush=True)
model = R.ReferenceModel.from_refs(refs, cfg.patch, channels=cfg.channels)
t0 = time.time()
model.table_rows(0, 1)
print(f"table build+upload {time.time() - t0:.2f}s", flush=True)
for t, (_, fld, st) in enumerate(R.stream_fields(model, frames)):
    pass
t0 = time.time()
it = R.stream_fields(model, frames)
last = time.time()
for t, (_, fld, st) in enumerate(it):
    now = time.time()
    Q = st.queries
    print(f"frame {t+1}: {1e3*(now-last):.1f} ms  {Q/(now-last)/1e6:.2f} Mq/s  evals/q {st.total_distance_evals/Q:.1f} "
          f"rings/q {st.total_rings/Q:.2f} W1/q {st.first_ring_total/Q:.1f} candF {st.mean_candidates:.1f} "
          f"tests/q {st.ring_tests_total/Q:.0f} exact/q {st.exact_evals_total/Q:.2f} heavy {st.fallback_queries/Q*100:.1f}%", flush=True)
    last = now
