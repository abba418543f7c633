"""K4 exact comparator throughput: tensor-core screen + float64 re-check vs
the SIMT full scan, on config-3 shapes (D=192, n=65,536 references, frame
units of a 1080p RGB frame).  Device-resident queries, CUDA events on the
context stream.

  python tools/bench_exact.py [--m 65536] [--n 65536] [--simt-m 4096] [--cfg 3]
"""

import argparse
import ctypes
import json
import os
import sys
from dataclasses import replace

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_1508_07953_b200 as R  # noqa: E402
from paper_1508_07953_b200 import _native as N  # noqa: E402
from paper_1508_07953_b200 import workloads as W  # noqa: E402
from paper_1508_07953_b200.evaluation import _upload_refs  # noqa: E402


def run(ctx, q, idx, dist, reps):
    st = (ctypes.c_uint64 * 2)()
    s = torch.cuda.ExternalStream(N.lib().riann_ctx_stream(ctx.h))
    N.check(N.lib().riann_exact_nn_device(ctx.h, q.data_ptr(), q.shape[0], idx.data_ptr(), dist.data_ptr(), st))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    N.check(N.lib().riann_sync(ctx.h))
    e0.record(s)
    for _ in range(reps):
        N.check(N.lib().riann_exact_nn_device(ctx.h, q.data_ptr(), q.shape[0], idx.data_ptr(), dist.data_ptr(), None))
    e1.record(s)
    N.check(N.lib().riann_sync(ctx.h))
    return e0.elapsed_time(e1) / reps, int(st[0]), int(st[1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", type=int, default=3)
    ap.add_argument("--m", type=int, default=65536)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--simt-m", type=int, default=2048)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    cfg = W.CONFIGS[a.cfg]
    if a.n:
        cfg = replace(cfg, n_refs=a.n)
    frame = W.clip(cfg, 1)[0]
    refs = W.reference_set(cfg)
    model = R.ReferenceModel.from_refs(refs, cfg.patch, channels=cfg.channels)
    units = R.frame_units(frame, model)
    rng = np.random.default_rng(0)
    sel = np.sort(rng.choice(units.shape[0], size=min(a.m, units.shape[0]), replace=False))
    q = torch.from_numpy(np.ascontiguousarray(units[sel])).cuda()
    m, D = q.shape
    n = model.n
    idx = torch.empty(m, dtype=torch.int32, device="cuda")
    dist = torch.empty(m, dtype=torch.float64, device="cuda")
    ctx = N.context()
    out = {"config": cfg.name, "m": m, "n": n, "dim": D}
    with ctx.lock:
        _upload_refs(ctx, model)
        torch.cuda.synchronize()
        ms, checked, fb = run(ctx, q, idx, dist, a.reps)
        flop = 2.0 * m * n * D  # algorithmic: one D-term dot product per (query, reference)
        out.update(tc_ms=ms, tc_queries_per_s=m / ms * 1e3, tc_tflops=flop / ms / 1e9,
                   rechecks_per_query=checked / m, fallback_queries=fb)
        tc_idx = idx.cpu().numpy().copy()
        tc_dist = dist.cpu().numpy().copy()
        N.check(N.lib().riann_ctx_set_path(ctx.h, 2))
        try:
            ms2 = ms_simt = None
            ms_m = min(a.simt_m, m)
            ms2, _, _ = run(ctx, q[:ms_m], idx[:ms_m], dist[:ms_m], 1)
            out.update(simt_m=ms_m, simt_ms=ms2, simt_queries_per_s=ms_m / ms2 * 1e3)
            si = idx[:ms_m].cpu().numpy()
            sd = dist[:ms_m].cpu().numpy()
            out["identical_to_simt"] = bool(np.array_equal(si, tc_idx[:ms_m]) and
                                            np.array_equal(sd.view(np.uint64), tc_dist[:ms_m].view(np.uint64)))
        finally:
            N.check(N.lib().riann_ctx_set_path(ctx.h, 0))
    out["speedup_vs_simt"] = out["tc_queries_per_s"] / out["simt_queries_per_s"]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
