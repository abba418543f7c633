"""Parity campaign: whole clips on the GPU vs the CPU oracle on stratified
position samples through every frame (bit-exact idx, f64 dist, rings, evals,
final candidates; whole-frame FrameStats are not comparable on a sample).

    python tools/parity_campaign.py [out.json]

config 3: 60 frames (1080p RGB, n = 65,536), 2,048 positions;
configs 1 and 2: 30 frames (VGA, n = 8,192), 16,384 positions.
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1508_07953_b200 as R  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_1508_07953_b200 import workloads as W  # noqa: E402


def stratified(gw, gh, count, seed):
    rng = np.random.default_rng(seed)
    rows = np.linspace(0, gh - 1, num=min(count, gh)).astype(np.int64)
    per = -(-count // len(rows))
    pos = np.concatenate([y * gw + rng.choice(gw, size=min(per, gw), replace=False) for y in rows])
    return np.unique(pos)[:count]


def campaign(cid, npos):
    cfg = W.CONFIGS[cid]
    frames = list(W.iter_clip(cfg))
    refs = W.reference_set(cfg)
    model = R.ReferenceModel.from_refs(refs, cfg.patch, channels=cfg.channels)
    gw, gh = cfg.grid
    pos = stratified(gw, gh, npos, 100 + cid)
    t0 = time.time()
    gpu = [(f.indices.ravel()[pos].copy(), f.distances.ravel()[pos].copy())
           for _, f, _ in R.stream_fields(model, frames)]
    t_gpu = time.time() - t0
    om = O.LazyOracleModel(refs) if cfg.n_refs > 8192 else O.OracleModel.build(refs)
    prev = O.init_field_indices(gw, gh, cfg.n_refs, 0).ravel()[pos]
    bad_idx = bad_dist = 0
    t0 = time.time()
    evals = []
    for t, f in enumerate(frames):
        unit = O.normalize_rows(W.patch_rows(f, cfg.patch, pos // gw, pos % gw))[0]
        r = O.query_positions(om, unit, prev, pos, gw, 0, t + 1)
        bad_idx += int(np.sum(r["idx"] != gpu[t][0]))
        bad_dist += int(np.sum(r["dist"].view(np.uint64) != gpu[t][1].view(np.uint64)))
        evals.append(float(r["evals"].mean()))
        prev = r["idx"]
    return {"config": cfg.name, "frames": len(frames), "positions": int(len(pos)),
            "queries_compared": int(len(pos) * len(frames)), "idx_mismatches": bad_idx,
            "dist_bit_mismatches": bad_dist, "gpu_stream_s": t_gpu, "oracle_s": time.time() - t0,
            "oracle_evals_per_query_by_frame": evals}


if __name__ == "__main__":
    out = sys.argv[1] if len(sys.argv) > 1 else "parity_campaign.json"
    res = [campaign(3, 2048), campaign(1, 16384), campaign(2, 16384)]
    json.dump({"method": __doc__.strip(), "results": res}, open(out, "w"), indent=1)
    for r in res:
        print(r["config"], r["queries_compared"], r["idx_mismatches"], r["dist_bit_mismatches"])
