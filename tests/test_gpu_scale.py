"""GPU parity at the benchmarked shapes, row-band invariance on the CUDA path,
and stream isolation on one device.

* config 3's D=192 path against the live-reference golden (golden_cfg3.npz)
  and, at full scale (1080p RGB, n=65,536), against the CPU oracle on 4,096
  stratified positions through 3 frames (search.py:83-151, engine.py:137-143);
* K4 exact comparator at config 4's shape (n=262,144, D=64) against the
  golden and the oracle's exact_nn (evaluation.py:24-33);
* 1 / 2 / 3 / 5 row bands (bands.py) on one GPU: fields and every FrameStats
  field byte-identical to the single stream (the analogue of the reference's
  thread invariance, test_engine.py:101-109);
* interleaved streams on one context never share device state (each stream
  owns a slot).
"""

import os
import socket

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    import paper_1508_07953_b200 as R

    return R


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def _same_stats(a, b):
    assert a.total_rings == b.total_rings
    assert a.total_distance_evals == b.total_distance_evals
    assert a.queries == b.queries
    assert a.first_ring_total == b.first_ring_total and a.cand_total == b.cand_total
    assert _bits(np.float64(a.mean_candidates)) == _bits(np.float64(b.mean_candidates))
    assert _bits(np.float64(a.temporal_change)) == _bits(np.float64(b.temporal_change))


def _stratified(gw, gh, count, seed):
    rng = np.random.default_rng(seed)
    rows = np.linspace(0, gh - 1, num=min(count, gh)).astype(np.int64)
    per = -(-count // len(rows))
    pos = np.concatenate([y * gw + rng.choice(gw, size=per, replace=False) for y in rows])
    return np.unique(pos)[:count]


# ---------------------------------------------------------------------------
def test_cfg3_d192_golden(R):
    """Live-reference golden on config 3's 1080p RGB clip (n=8,192): every GPU
    position of 10 full frames computed, 256 compared bit for bit."""
    from dataclasses import replace

    from paper_1508_07953_b200 import workloads as W

    g = load_golden("golden_cfg3.npz")
    cfg = replace(W.CONFIGS[3], n_refs=int(g["n_refs"]))
    refs = W.reference_set(cfg)
    assert W.digest(refs) == str(g["refs_digest"])
    model = R.ReferenceModel.from_refs(refs, cfg.patch, channels=3)
    sd, si = model.table_rows(0, model.n)
    assert W.digest(sd, si) == str(g["table_digest"])
    pos = g["positions"]
    T = g["idx"].shape[0]
    frames = W.iter_clip(cfg, T)
    for t, (frame, fld, st) in enumerate(R.stream_fields(model, frames, R.SearchParams())):
        assert W.digest(frame) == str(g["frame_digests"][t])
        assert np.array_equal(fld.indices.ravel()[pos], g["idx"][t]), t
        assert np.array_equal(_bits(fld.distances.ravel()[pos]), _bits(g["dist"][t])), t
    units = R.frame_units(frame, model)
    assert np.array_equal(units[pos], g["units"][-1])


def test_cfg3_full_scale_vs_oracle(R, oracle_mod):
    """The benchmarked configuration itself: 1080p RGB, n=65,536.  4,096
    stratified positions through frames 1-3 (frame 1 starts from init_field,
    the heaviest frame) vs the oracle with lazily built table rows: idx, f64
    dist, rings, evals and final candidates bit-exact."""
    from paper_1508_07953_b200 import workloads as W

    cfg = W.CONFIGS[3]
    T = 3
    frames = list(W.iter_clip(cfg, T))
    refs = W.reference_set(cfg)
    model = R.ReferenceModel.from_refs(refs, cfg.patch, channels=3)
    gw, gh = cfg.grid
    pos = _stratified(gw, gh, 4096, 33)
    gpu = [(fld.indices.ravel()[pos].copy(), fld.distances.ravel()[pos].copy())
           for _, fld, _ in R.stream_fields(model, frames, R.SearchParams())]
    om = oracle_mod.LazyOracleModel(refs)
    prev = oracle_mod.init_field_indices(gw, gh, cfg.n_refs, 0).ravel()[pos]
    for t in range(T):
        unit = oracle_mod.normalize_rows(W.patch_rows(frames[t], cfg.patch, pos // gw, pos % gw))[0]
        r = oracle_mod.query_positions(om, unit, prev, pos, gw, 0, t + 1)
        assert np.array_equal(gpu[t][0], r["idx"]), t
        assert np.array_equal(_bits(gpu[t][1]), _bits(r["dist"])), t
        prev = r["idx"]


@pytest.mark.parametrize("L,alpha,max_rings", [(20, 0.25, 8), (2, 0.4, 14), (40, 0.15, 20)])
def test_dense_lists_compaction_vs_oracle(R, oracle_mod, L, alpha, max_rings):
    """Dense first rings (config 2: high motion, first rings ~60 % of n; frame 1
    from init_field: ~70 %): the lists are rewritten between ring phases
    (bulk_compact_kernel), several times with long ring caps.  8,192
    stratified positions through 4 frames, bit-exact vs the oracle."""
    from paper_1508_07953_b200 import workloads as W

    cfg = W.CONFIGS[2]
    T = 4
    frames = list(W.iter_clip(cfg, T))
    refs = W.reference_set(cfg)
    model = R.ReferenceModel.from_refs(refs, cfg.patch, channels=cfg.channels)
    gw, gh = cfg.grid
    pos = _stratified(gw, gh, 8192, 35)
    params = R.SearchParams(L=L, alpha=alpha, max_rings=max_rings)
    gpu = [(fld.indices.ravel()[pos].copy(), fld.distances.ravel()[pos].copy())
           for _, fld, _ in R.stream_fields(model, frames, params)]
    om = oracle_mod.LazyOracleModel(refs)
    prev = oracle_mod.init_field_indices(gw, gh, cfg.n_refs, 0).ravel()[pos]
    for t in range(T):
        unit = oracle_mod.normalize_rows(W.patch_rows(frames[t], cfg.patch, pos // gw, pos % gw))[0]
        r = oracle_mod.query_positions(om, unit, prev, pos, gw, 0, t + 1, L=L, alpha=alpha, max_rings=max_rings)
        assert np.array_equal(gpu[t][0], r["idx"]), t
        assert np.array_equal(_bits(gpu[t][1]), _bits(r["dist"])), t
        prev = r["idx"]


def test_cfg3_full_scale_rings_evals(R, oracle_mod):
    """Same workload through riann_query_batch (the per-query kernel on the
    same model): rings, evals and |S| per position equal the oracle's."""
    from paper_1508_07953_b200 import workloads as W

    cfg = W.CONFIGS[3]
    frame = next(W.iter_clip(cfg, 1))
    refs = W.reference_set(cfg)
    model = R.ReferenceModel.from_refs(refs, cfg.patch, channels=3)
    gw, gh = cfg.grid
    pos = _stratified(gw, gh, 1024, 34)
    unit = oracle_mod.normalize_rows(W.patch_rows(frame, cfg.patch, pos // gw, pos % gw))[0]
    prev = oracle_mod.init_field_indices(gw, gh, cfg.n_refs, 0).ravel()[pos]
    keys = [R.query_rng_key(0, int(g % gw), int(g // gw), 1) for g in pos]
    res = R.riann_query_batch(model, unit, prev, R.SearchParams(), keys=keys)
    om = oracle_mod.LazyOracleModel(refs)
    r = oracle_mod.query_positions(om, unit, prev, pos, gw, 0, 1)
    for k in ("idx", "rings", "evals", "cand", "first"):
        assert np.array_equal(res[k], r[k]), k
    assert np.array_equal(_bits(res["dist"]), _bits(r["dist"]))


# ---------------------------------------------------------------------------
def test_exact_tc_cfg4_scale(R, oracle_mod):
    """K4 at config 4's shape (n=262,144, D=64): the live-reference golden
    (256 positions) and 1,024 further positions of the first 4K frame vs the
    oracle's exact_nn, through field_exact_oracle (all 8.25 M positions)."""
    from paper_1508_07953_b200 import workloads as W

    g = load_golden("golden_cfg4x.npz")
    cfg = W.CONFIGS[4]
    refs = W.reference_set(cfg)
    assert W.digest(refs) == str(g["refs_digest"])
    frame = next(W.iter_clip(cfg, 1))
    model = R.ReferenceModel.from_refs(refs, cfg.patch)
    fld = R.field_exact_oracle(frame, model)
    gpos = g["positions"]
    assert np.array_equal(fld.indices.ravel()[gpos], g["idx"])
    assert np.array_equal(_bits(fld.distances.ravel()[gpos]), _bits(g["dist"]))
    gw, gh = cfg.grid
    pos = _stratified(gw, gh, 1024, 44)
    unit = oracle_mod.normalize_rows(W.patch_rows(frame, cfg.patch, pos // gw, pos % gw))[0]
    wi, wd = oracle_mod.exact_nn_batch(refs, unit)
    assert np.array_equal(fld.indices.ravel()[pos], wi)
    assert np.array_equal(_bits(fld.distances.ravel()[pos]), _bits(wd))


# ---------------------------------------------------------------------------
def _clip_and_model(R, cfg_id, frames, **kw):
    from dataclasses import replace

    from paper_1508_07953_b200 import workloads as W

    cfg = replace(W.CONFIGS[cfg_id], **kw) if kw else W.CONFIGS[cfg_id]
    clip = W.clip(cfg, frames)
    refs = W.reference_set(cfg)
    return clip, R.ReferenceModel.from_refs(refs, cfg.patch, channels=cfg.channels)


@pytest.mark.parametrize("cfg_id,frames,kw", [(1, 6, {}), (3, 4, dict(height=60, width=90, n_refs=2048)),
                                              (2, 12, {})])
def test_band_invariance_on_gpu(R, cfg_id, frames, kw):
    """The CUDA band path (bands.py): 2, 3 and 5 bands of each frame, run one
    after another on one GPU in their own stream slots, assemble fields and
    FrameStats (temporal_change included) byte-identical to one stream."""
    clip, model = _clip_and_model(R, cfg_id, frames, **kw)
    base = [(f.indices.copy(), f.distances.copy(), s) for _, f, s in R.stream_fields(model, clip)]
    for nb in (2, 3, 5):
        got = list(R.stream_fields(model, clip, devices=[0], bands=nb))
        assert len(got) == len(base)
        for t, ((_, f, s), (bi, bd, bs)) in enumerate(zip(got, base)):
            assert np.array_equal(f.indices, bi), (nb, t)
            assert np.array_equal(_bits(f.distances), _bits(bd)), (nb, t)
            _same_stats(s, bs)


def test_band_streams_interleaved_with_reuploads(R):
    """BandStreams sharing one GPU, stepped in an interleaved order with a
    different model made resident between frames: each band re-uploads its
    own state, the assembled field still equals the single stream's."""
    from paper_1508_07953_b200.bands import BandStream, band_rows, frame_band

    clip, model = _clip_and_model(R, 1, 4)
    _, other = _clip_and_model(R, 0, 1)
    base = [f.indices.copy() for _, f, _ in R.stream_fields(model, clip)]
    gw, gh = R.grid_shape(clip.shape[1:3], model.patch_size)
    cuts = [band_rows(gh, 3, k) for k in range(3)]
    bands = [BandStream(model, gw, gh, a, b) for a, b in cuts]
    for t in range(clip.shape[0]):
        order = [2, 0, 1] if t % 2 else [1, 2, 0]
        parts = {}
        for k in order:
            parts[k] = bands[k].step(frame_band(clip[t], *cuts[k], model.patch_size[1]))[0]
        if t == 1:
            R.field_exact_oracle(np.ascontiguousarray(clip[0][:64, :64]), other)  # another model's refs
            list(R.stream_fields(other, [clip[0][:64, :64]]))                     # and its tables
        assert np.array_equal(np.concatenate([parts[k] for k in range(3)]), base[t]), t
    for b in bands:
        b.close()


def test_interleaved_streams_isolated(R):
    """zip(stream_fields(m, A), stream_fields(m, B)) with process_frame calls
    in between: each stream's fields and temporal_change equal its solo run
    (the reference's stream_fields is a pure generator)."""
    clip, model = _clip_and_model(R, 0, 8)
    A, B = clip, clip[::-1].copy()
    solo_a = [(f.indices.copy(), s) for _, f, s in R.stream_fields(model, A)]
    solo_b = [(f.indices.copy(), s) for _, f, s in R.stream_fields(model, B)]
    init = R.init_field(*R.grid_shape(A.shape[1:3], model.patch_size), model.n)
    units = R.frame_units(A[3], model)
    for t, ((_, fa, sa), (_, fb, sb)) in enumerate(zip(R.stream_fields(model, A), R.stream_fields(model, B))):
        R.process_frame(A[1], init, model, prev_unit=units)  # writes slot 0's units and field
        assert np.array_equal(fa.indices, solo_a[t][0]) and np.array_equal(fb.indices, solo_b[t][0]), t
        _same_stats(sa, solo_a[t][1])
        _same_stats(sb, solo_b[t][1])


def test_replaced_field_not_taken_from_device(R):
    """dataclasses.replace(fld, indices=new) must not reuse the stale device
    field (AnnField._dev is not an init field)."""
    from dataclasses import replace

    clip, model = _clip_and_model(R, 0, 3)
    f1, _ = R.process_frame(clip[0], R.init_field(57, 57, model.n), model)
    other = R.init_field(57, 57, model.n, seed=5)
    f_rep = replace(f1, indices=other.indices.copy())
    a, _ = R.process_frame(clip[1], f_rep, model)
    b, _ = R.process_frame(clip[1], replace(other, frame_t=f1.frame_t), model)
    assert np.array_equal(a.indices, b.indices)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_distributed_stream_single_rank(R):
    """DistributedStream (NCCL gather path) with one rank equals stream_fields."""
    import torch.distributed as dist

    from paper_1508_07953_b200.bands import DistributedStream

    clip, model = _clip_and_model(R, 1, 4)
    base = [(f.indices.copy(), f.distances.copy(), s) for _, f, s in R.stream_fields(model, clip)]
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        gw, gh = R.grid_shape(clip.shape[1:3], model.patch_size)
        ds = DistributedStream(model, gw, gh)
        for t in range(clip.shape[0]):
            f, s = ds.step(clip[t])
            assert np.array_equal(f.indices, base[t][0]), t
            assert np.array_equal(_bits(f.distances), _bits(base[t][1])), t
            _same_stats(s, base[t][2])
        ds.close()
    finally:
        dist.destroy_process_group()
