"""Multi-rank band partitioning on CPU (gloo, world size 2).

Each rank takes its grid-row band (bands.band_rows), slices the frame with the
(ph-1)-row halo (bands.frame_band), runs the band's positions with global RNG
keys (the oracle stands in for the GPU runner here), and rank 0 assembles the
gathered bands: the field must equal the single-process full-frame result,
the analogue of the reference's thread-count invariance (test_engine.py:101-109).
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle import oracle as O
        from paper_1508_07953_b200 import workloads as W
        from paper_1508_07953_b200.bands import band_rows, frame_band

        cfg = W.CONFIGS[0]
        frames = W.clip(cfg, 3)
        refs = W.reference_set(cfg)
        model = O.OracleModel.build(refs, nthreads=1)
        gw, gh = cfg.grid
        y0, y1 = band_rows(gh, world, rank)
        prev = O.init_field_indices(gw, gh, model.n, 0)[y0:y1].ravel()
        pos = (np.arange(y0, y1)[:, None] * gw + np.arange(gw)[None, :]).ravel().astype(np.int64)
        fields = []
        for t in range(3):
            band = frame_band(frames[t], y0, y1, cfg.patch[1])
            assert band.shape[0] == (y1 - y0) + cfg.patch[1] - 1
            units, _ = O.frame_units(band, cfg.patch)
            r = O.query_positions(model, units, prev, pos, gw, 0, t + 1, nthreads=1)
            prev = r["idx"]
            gathered = [None] * world
            dist.all_gather_object(gathered, (y0, y1, r["idx"], r["dist"], int(r["evals"].sum())))
            fields.append(gathered)
        if rank == 0:
            out.put(fields)
    finally:
        dist.destroy_process_group()


def test_two_band_field_equals_full_frame(oracle_mod):
    from paper_1508_07953_b200 import workloads as W

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    fields = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cfg = W.CONFIGS[0]
    frames = W.clip(cfg, 3)
    model = oracle_mod.OracleModel.build(W.reference_set(cfg))
    gw, gh = cfg.grid
    prev = oracle_mod.init_field_indices(gw, gh, model.n, 0)
    for t in range(3):
        idx, dist_, st, _ = oracle_mod.process_frame(model, frames[t], prev, cfg.patch, t + 1)
        parts = sorted(fields[t], key=lambda x: x[0])
        assert parts[0][0] == 0 and parts[-1][1] == gh
        got_i = np.concatenate([p[2] for p in parts]).reshape(gh, gw)
        got_d = np.concatenate([p[3] for p in parts]).reshape(gh, gw)
        assert np.array_equal(got_i, idx)
        assert np.array_equal(got_d.view(np.uint64), dist_.view(np.uint64))
        assert sum(p[4] for p in parts) == st["total_distance_evals"]
        prev = idx


def test_band_rows_partition():
    from paper_1508_07953_b200.bands import band_rows

    for gh in (1, 7, 57, 473, 1073):
        for world in (1, 2, 3, 4, 8):
            if world > gh:
                continue
            rows = [band_rows(gh, world, r) for r in range(world)]
            assert rows[0][0] == 0 and rows[-1][1] == gh
            assert all(rows[i][1] == rows[i + 1][0] for i in range(world - 1))
            assert max(b - a for a, b in rows) - min(b - a for a, b in rows) <= 1
    with pytest.raises(ValueError):
        band_rows(10, 2, 2)
