"""Experiment: two half-frame bands of one config-3 stream on TWO contexts of
one GPU, running concurrently half a frame apart (the HBM-bound filter of one
band against the issue-bound P0b / final scan of the other), vs one context.

    python tools/dual_ctx.py [T] [offset_ms]
"""
import os
import sys
import threading
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_07953_b200 as R  # noqa: E402
from paper_1508_07953_b200 import _native as N  # noqa: E402
from paper_1508_07953_b200 import workloads as W  # noqa: E402
from paper_1508_07953_b200 import bands as B  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 16
OFF = float(sys.argv[2]) if len(sys.argv) > 2 else 20.0
mode = os.environ.get("MODE", "dual")
cfg = W.CONFIGS[3]
frames = list(W.iter_clip(cfg, T))
refs = W.reference_set(cfg)
model = R.ReferenceModel.from_refs(refs, cfg.patch, channels=cfg.channels)
gw, gh = cfg.grid
ph = cfg.patch[1]

if mode == "single":
    bs = B.BandStream(model, gw, gh, 0, gh)
    t0 = None
    for t in range(T):
        if t == 6:
            t0 = time.perf_counter()
        bs.step(frames[t])
    dt = (time.perf_counter() - t0) / (T - 6) * 1e3
    print(f"single: {dt:.2f} ms/frame (frames 7..{T}, wall, public API)")
    sys.exit(0)

ctxs = [N.context(0), N.Context(0)]
mid = gh // 2
spans = [(0, mid), (mid, gh)]
streams = []
for (y0, y1), ctx in zip(spans, ctxs):
    real = N.context
    N.context = lambda device=None, _c=ctx: _c
    B.N.context = N.context
    try:
        streams.append(B.BandStream(model, gw, gh, y0, y1))
    finally:
        N.context = real
        B.N.context = real
bframes = [[B.frame_band(f, y0, y1, ph) for f in frames] for (y0, y1) in spans]
# frame 1 (heavy) and table builds outside the timed window, one band after the other
for k in range(2):
    streams[k].step(bframes[k][0])
out = [[None] * T for _ in range(2)]
marks = [[0.0] * (T + 1) for _ in range(2)]


def run(k):
    if k == 1:
        time.sleep(OFF * 1e-3)
    for t in range(1, T):
        marks[k][t] = time.perf_counter()
        out[k][t] = streams[k].step(bframes[k][t])[0].copy()
    marks[k][T] = time.perf_counter()


ths = [threading.Thread(target=run, args=(k,)) for k in range(2)]
for th in ths:
    th.start()
for th in ths:
    th.join()
start = min(marks[0][6], marks[1][6])
end = max(marks[0][T], marks[1][T])
print(f"dual (offset {OFF} ms, share {os.environ.get('RIANN_SM_SHARE', '1')}): {(end - start) / (T - 6) * 1e3:.2f} ms/frame; "
      f"band times {[(marks[k][T] - marks[k][6]) / (T - 6) * 1e3 for k in range(2)]}")
# the assembled field equals the one-context field
bs = B.BandStream(model, gw, gh, 0, gh)
ok = True
for t in range(T):
    idx = bs.step(frames[t])[0]
    if t >= 1:
        ok &= bool(np.array_equal(idx[:mid], out[0][t]) and np.array_equal(idx[mid:], out[1][t]))
print("fields identical to one band:", ok)
