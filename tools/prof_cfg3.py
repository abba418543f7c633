"""Profiling driver: config-3 statistics (RGB, D=192, n=65,536) on a row crop."""
import argparse
import sys
import time
from dataclasses import replace

sys.path.insert(0, ".")
import paper_1508_07953_b200 as R
from paper_1508_07953_b200 import workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=270)
ap.add_argument("--frames", type=int, default=3)
ap.add_argument("--cfg", type=int, default=3)
a = ap.parse_args()
base = W.CONFIGS[a.cfg]
cfg = replace(base, height=a.rows)
frames = W.clip(cfg, a.frames)
refs = W.reference_set(base)
model = R.ReferenceModel.from_refs(refs, cfg.patch, channels=cfg.channels)
model.table_rows(0, 1)
last = time.time()
for t, (_, fld, st) in enumerate(R.stream_fields(model, frames)):
    now = time.time()
    print(f"frame {t+1}: {1e3*(now-last):.1f} ms evals/q {st.total_distance_evals/st.queries:.1f}", flush=True)
    last = now
