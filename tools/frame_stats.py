"""Per-frame RIANN statistics of the bench workload (config 3 by default):
rings, first-ring sizes, ring membership tests, exact evaluations, final
candidate counts, per query.  python tools/frame_stats.py [--cfg 3] [--frames 6]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_07953_b200 as R  # noqa: E402
from paper_1508_07953_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=3)
ap.add_argument("--frames", type=int, default=6)
a = ap.parse_args()
cfg = W.CONFIGS[a.cfg]
refs = W.reference_set(cfg)
model = R.ReferenceModel.from_refs(refs, cfg.patch, channels=cfg.channels)
for t, (_, fld, st) in enumerate(R.stream_fields(model, W.iter_clip(cfg, a.frames))):
    q = st.queries
    print(f"frame {t + 1}: rings/q {st.total_rings / q:.2f} evals/q {st.total_distance_evals / q:.1f} "
          f"first_ring/q {st.first_ring_total / q:.1f} ring_tests/q {st.ring_tests_total / q:.1f} "
          f"exact/q {st.exact_evals_total / q:.1f} cand_final/q {st.mean_candidates:.1f} "
          f"fallback {st.fallback_queries}", flush=True)
