"""Output-side rows on the GPU, kernel time by CUDA events on
the library stream (device-resident inputs) plus the public-API time:

  * ANNF frame payload pack from the device field (riann_field_pack): 12 bytes
    read + 8 written per position;
  * reconstruct_frame / apply_effect (riann_apply_effect) at VGA and 4K
    grayscale (configs 1 and 4 geometry): algorithmic bytes per frame =
    frame read 4·H·W + matches 4·Q + payload rows 4·pw·ph·Q (each row read
    once) + output write 4·H·W (+ norms pass: frame again).

  python tools/bench_effects.py [--reps 5]
"""

import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1508_07953_b200 as R  # noqa: E402
from paper_1508_07953_b200 import _native as N  # noqa: E402
from paper_1508_07953_b200 import transforms as T  # noqa: E402
from paper_1508_07953_b200 import workloads as W  # noqa: E402


def peak_gbs():
    p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return float(json.load(f).get("hbm_gbs", 6537.6))
    return 6537.6


def timed(ctx, fn, reps):
    s = torch.cuda.ExternalStream(N.lib().riann_ctx_stream(ctx.h))
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    N.check(N.lib().riann_sync(ctx.h))
    t0 = time.perf_counter()
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    N.check(N.lib().riann_sync(ctx.h))
    return e0.elapsed_time(e1) / reps, (time.perf_counter() - t0) * 1e3 / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    out = {"peak_gbs": peak_gbs()}
    ctx = N.context()
    for ci, H, Wd in ((1, 480, 640), (4, 2160, 3840)):
        cfg = W.CONFIGS[ci]
        refs = W.reference_set(W.CONFIGS[1])  # 8,192 references (the effect cost does not depend on n)
        model = R.ReferenceModel.from_refs(refs, (8, 8))
        frame = W.clip(cfg, 1)[0][:H, :Wd].copy()
        gw, gh = Wd - 7, H - 7
        Q = gw * gh
        rng = np.random.default_rng(0)
        idx = rng.integers(0, model.n, size=(gh, gw), dtype=np.int32)
        field = R.AnnField(width=gw, height=gh, indices=idx, distances=np.zeros((gh, gw)))
        table = T.reconstruction_table(model)
        res = {}
        # public API (host frame + field in, raster out)
        T.reconstruct_frame(frame, field, model)
        t0 = time.perf_counter()
        for _ in range(a.reps):
            T.reconstruct_frame(frame, field, model)
        res["api_ms"] = (time.perf_counter() - t0) * 1e3 / a.reps
        # kernel-only: device field (run one frame so the field is resident) and timed effect calls
        f32 = np.ascontiguousarray(frame, dtype=np.float32)
        outp = np.empty((1, H, Wd), np.float32)
        with ctx.lock:
            R.model.resident(ctx, model)
        for _ in R.stream_fields(model, [frame]):
            pass
        with ctx.lock:
            dev_ms, host_ms = timed(ctx, lambda: N.check(N.lib().riann_apply_effect(
                ctx.h, N.ptr(f32), H, Wd, None, None, model.n, model.dim, 0, N.ptr(outp), None)), a.reps)
            payload = np.empty(2 * Q, np.uint32)
            pk_ms, pk_host = timed(ctx, lambda: N.check(N.lib().riann_field_pack(ctx.h, N.ptr(payload), Q)),
                                   a.reps)
        alg = 4 * H * Wd * 2 + 4 * Q + 4 * 64 * Q + 4 * H * Wd
        res.update(geometry=f"{Wd}x{H} gray, 8x8 patches, Q={Q}", effect_call_ms=dev_ms,
                   effect_call_host_ms=host_ms, effect_alg_bytes=alg,
                   note="effect_call_ms includes the frame H2D and raster D2H of the C call",
                   pack_call_ms=pk_ms, pack_bytes=20 * Q)
        out[cfg.name] = res
    print(json.dumps(out))


if __name__ == "__main__":
    main()
