"""Per-frame phase split (CUDA events, riann_timing_phases) and fallback
counts of the config-3 stream, frames 1..T:

    python tools/frame_phases.py [T]
"""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_07953_b200 as R  # noqa: E402
from paper_1508_07953_b200 import _native as N  # noqa: E402
from paper_1508_07953_b200 import workloads as W  # noqa: E402
from paper_1508_07953_b200.bands import BandStream  # noqa: E402

NPH = 10  # RIANN_NPHASES
T = int(sys.argv[1]) if len(sys.argv) > 1 else 25
cfg = W.CONFIGS[int(os.environ.get("CFG", "3"))]
frames = list(W.iter_clip(cfg, T))
refs = W.reference_set(cfg)
model = R.ReferenceModel.from_refs(refs, cfg.patch, channels=cfg.channels)
gw, gh = cfg.grid
nb = int(os.environ.get("BANDS", "1"))  # time band 0 of nb (the per-GPU share of an nb-GPU run)
y1 = gh // nb
if nb > 1:
    from paper_1508_07953_b200.bands import frame_band

    frames = [frame_band(f, 0, y1, cfg.patch[1]) for f in frames]
bs = BandStream(model, gw, gh, 0, y1)
ctx = bs.ctx
lib = N.lib()
names = [lib.riann_phase_name(k).decode().split(":")[1] for k in range(NPH)]
for t in range(T):
    with ctx.lock:
        N.check(lib.riann_timing_enable(ctx.h, 1))
    idx, dist, st = bs.step(frames[t])
    ph = (C.c_double * NPH)()
    with ctx.lock:
        N.check(lib.riann_timing_phases(ctx.h, ph, NPH))
        N.check(lib.riann_timing_enable(ctx.h, 0))
    row = {"t": t + 1, "total": round(sum(ph), 2), "fallback": st.fallback_queries,
           "evals/q": round(st.total_distance_evals / st.queries, 1),
           "first/q": round(st.first_ring_total / st.queries, 1),
           "tests/q": round(st.ring_tests_total / st.queries, 1),
           "exact/q": round(st.exact_evals_total / st.queries, 2)}
    row.update({names[k]: round(ph[k], 2) for k in range(NPH) if ph[k] > 0})
    print(json.dumps(row), flush=True)
