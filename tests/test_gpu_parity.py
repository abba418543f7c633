"""GPU parity: the CUDA path through the C ABI vs the live-reference goldens
and the CPU oracle.  Bar: bit-exact indices, float64 distances and integer
FrameStats (the design target; BASELINE's tolerance is >= 99.9% / 1e-4 rel).
"""

import numpy as np
import pytest

from conftest import load_golden, ragged

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    import paper_1508_07953_b200 as R

    return R


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


# ---------------------------------------------------------------------------
def test_one_to_many_and_normalize_golden(R):
    g = load_golden("golden_arith.npz")
    for i, d in enumerate(g["dims"]):
        d = int(d)
        q = ragged(g["q"], g["q_off"], i)
        r = ragged(g["r"], g["r_off"], i).reshape(-1, d)
        got = R.EUCLIDEAN.one_to_many(q, r)
        assert np.array_equal(_bits(got), _bits(ragged(g["d"], g["d_off"], i))), d
        v = ragged(g["norm_in"], g["norm_in_off"], i).reshape(-1, d)
        u, nr = R.normalize_rows(v)
        assert np.array_equal(_bits(u), _bits(ragged(g["norm_unit"], g["norm_in_off"], i).reshape(-1, d))), d
        assert np.array_equal(nr, ragged(g["norm_norms"], g["norm_off"], i)), d


def test_one_to_many_float64_inputs(R, oracle_mod):
    rng = np.random.default_rng(3)
    q = rng.uniform(-1, 1, size=16)
    refs = rng.uniform(-1, 1, size=(50, 16))
    want = np.sqrt(np.sum((refs - q) ** 2, axis=1))
    assert np.array_equal(R.EUCLIDEAN.one_to_many(q, refs), want)


def test_sorted_tables_golden(R):
    g = load_golden("golden_tables.npz")
    for i, (n, d) in enumerate(g["shapes"]):
        refs = ragged(g["refs"], g["refs_off"], i).reshape(int(n), int(d))
        sd, si = R.compute_sorted_lists(refs)
        assert sd.dtype == np.float64 and si.dtype == np.int32
        assert np.array_equal(sd.ravel(), ragged(g["sdist"], g["tab_off"], i).astype(np.float64))
        assert np.array_equal(si.ravel(), ragged(g["sidx"], g["tab_off"], i))


def _golden_models(R, g):
    models = []
    for i, (n, d) in enumerate(g["model_shapes"]):
        refs = ragged(g["models"], g["model_off"], i).reshape(int(n), int(d))
        models.append(R.ReferenceModel.from_refs(refs, (int(d), 1)))
    return models


def test_riann_query_golden(R):
    g = load_golden("golden_queries.npz")
    models = _golden_models(R, g)
    for c in range(len(g["mid"])):
        m = models[int(g["mid"][c])]
        key = tuple(int(v) for v in ragged(g["key"], g["key_off"], c))
        p = R.SearchParams(L=int(g["L"][c]), alpha=float(g["alpha"][c]), max_rings=int(g["mr"][c]))
        r = R.riann_query(m, ragged(g["q"], g["q_off"], c), int(g["prev"][c]), p, rng_state=key)
        assert r.match_index == g["idx"][c], c
        assert r.match_distance == g["dist"][c], c
        assert r.rings_drawn == g["rings"][c], c
        assert r.distance_evals == g["evals"][c], c
        assert r.candidates_final == g["cand"][c], c
        assert np.array_equal(r.scanned, ragged(g["scanned"], g["scanned_off"], c)), c


def test_riann_query_batch_matches_single(R):
    g = load_golden("golden_queries.npz")
    models = _golden_models(R, g)
    sel = [c for c in range(len(g["mid"])) if int(g["mid"][c]) == 9]
    m = models[9]
    qs = np.stack([ragged(g["q"], g["q_off"], c) for c in sel])
    keys = [tuple(int(v) for v in ragged(g["key"], g["key_off"], c)) for c in sel]
    same = [c for c in sel if g["L"][c] == 20 and g["mr"][c] == 8 and g["alpha"][c] == 0.25]
    idx = [sel.index(c) for c in same]
    r = R.riann_query_batch(m, qs[idx], g["prev"][same], R.SearchParams(), keys=[keys[i] for i in idx])
    assert np.array_equal(r["idx"], g["idx"][same])
    assert np.array_equal(_bits(r["dist"]), _bits(g["dist"][same]))
    assert np.array_equal(r["evals"], g["evals"][same])


# ---------------------------------------------------------------------------
# ports of the reference's known-answer tests (test_search.py:31-114)
@pytest.fixture()
def tri(R):
    s = np.float32(np.sqrt(2.0) / 2.0)
    return R.ReferenceModel.from_refs(np.array([[1, 0], [0, 1], [s, s]], np.float32), (2, 1))


def test_ring_windows_known_answers(R, tri):
    assert R.ring_candidates(tri, 0, 0.765367, 0.191342).tolist() == [2]
    assert R.ring_candidates(tri, 1, 0.0, 0.0).tolist() == [1]
    top = float(tri.sorted_dist[0, -1])
    assert sorted(R.ring_candidates(tri, 0, top, top).tolist()) == [0, 1, 2]
    d = float(tri.sorted_dist[0, 1])
    assert R.ring_candidates(tri, 0, d, 0.0).tolist() == [2]
    with pytest.raises(IndexError):
        R.ring_candidates(tri, 3, 0.5, 0.1)
    with pytest.raises(ValueError):
        R.ring_candidates(tri, 0, -0.1, 0.1)


def test_ring_windows_brute_force(R):
    rng = np.random.default_rng(12345)
    rows = rng.normal(size=(80, 12))
    rows = (rows / np.linalg.norm(rows, axis=1, keepdims=True)).astype(np.float32)
    m = R.ReferenceModel.from_refs(rows, (12, 1))
    for _ in range(200):
        a = int(rng.integers(80))
        d = float(rng.uniform(0, 1.6))
        eps = float(rng.uniform(0, 0.4))
        row = m.metric.one_to_many(rows[a], rows).astype(np.float32).astype(np.float64)
        want = set(np.flatnonzero((row >= d - eps) & (row <= d + eps)).tolist())
        assert set(R.ring_candidates(m, a, d, eps).tolist()) == want


def test_query_known_answers(R, tri):
    r = R.riann_query(tri, tri.refs[1], 1)
    assert (r.match_index, r.match_distance, r.rings_drawn) == (1, 0.0, 1)
    r = R.riann_query(tri, tri.refs[2], 0)
    assert (r.match_index, r.match_distance, r.rings_drawn, r.candidates_final) == (2, 0.0, 1, 1)
    assert r.scanned.tolist() == [0, 2]
    r = R.riann_query(tri, np.zeros(2, np.float32), 0)
    assert r.match_distance == pytest.approx(1.0, abs=1e-6)
    tie = R.ReferenceModel.from_refs(np.array([[1, 0], [0, 1], [1, 0]], np.float32), (2, 1))
    r = R.riann_query(tie, tie.refs[0], 2)
    assert (r.match_index, r.match_distance) == (0, 0.0)
    with pytest.raises(IndexError):
        R.riann_query(tri, tri.refs[0], 3)
    with pytest.raises(R.DimensionError):
        R.riann_query(tri, np.ones(3, np.float32), 0)


def test_query_accounting_and_scope(R, oracle_mod):
    rng = np.random.default_rng(7)
    rows = rng.normal(size=(150, 16))
    rows = (rows / np.linalg.norm(rows, axis=1, keepdims=True)).astype(np.float32)
    m = R.ReferenceModel.from_refs(rows, (16, 1))
    qs, _ = R.normalize_rows(rows[rng.integers(0, 150, 300)] + rng.normal(scale=0.08, size=(300, 16)).astype(np.float32))
    prev = rng.integers(0, 150, 300)
    keys = [(7, k) for k in range(300)]
    r = R.riann_query_batch(m, qs, prev, R.SearchParams(), keys=keys, scanned=True)
    for k in range(300):
        sc = r["scanned"][k]
        assert r["evals"][k] == 1 + (r["rings"][k] - 1) + sc.size
        rescan = m.metric.one_to_many(qs[k], rows[sc])
        assert r["dist"][k] == rescan.min()
        assert r["idx"][k] == sc[int(np.argmin(rescan))]
        assert 1 <= r["rings"][k] <= 8


# ---------------------------------------------------------------------------
def test_cfg0_stream_golden(R):
    """Config 0 end to end: every position of all 8 frames, FrameStats exact."""
    from paper_1508_07953_b200 import workloads as W

    g = load_golden("golden_cfg0.npz")
    model = R.ReferenceModel.from_refs(g["refs"], (8, 8))
    out = list(R.stream_fields(model, list(g["frames"]), R.SearchParams()))
    assert len(out) == 8
    for t, (_, fld, st) in enumerate(out):
        assert fld.frame_t == t + 1
        assert np.array_equal(fld.indices, g["idx"][t]), t
        assert np.array_equal(_bits(fld.distances), _bits(g["dist"][t])), t
        assert [st.total_rings, st.total_distance_evals, st.queries] == list(g["stats_int"][t]), t
        assert st.mean_candidates == g["stats_f"][t][0], t
        assert st.temporal_change == g["stats_f"][t][1], t
    assert W.digest(model.sorted_dist.astype(np.float32), model.sorted_idx) == str(g["table_digest"])


def test_cfg0_process_frame_host_prev_matches_stream(R):
    g = load_golden("golden_cfg0.npz")
    model = R.ReferenceModel.from_refs(g["refs"], (8, 8))
    f0 = R.init_field(57, 57, model.n, seed=0)
    a, sa = R.process_frame(g["frames"][0], f0, model, threads=1)
    b, sb = R.process_frame(g["frames"][0], f0, model, threads=4)
    assert np.array_equal(a.indices, g["idx"][0]) and np.array_equal(b.indices, a.indices)
    assert np.array_equal(a.distances, b.distances) and sa == sb
    u0 = R.frame_units(g["frames"][0], model)
    c, sc = R.process_frame(g["frames"][1], a, model, prev_unit=u0)
    assert np.array_equal(c.indices, g["idx"][1])
    assert sc.temporal_change == g["stats_f"][1][1]


def test_cfg0_exact_field_golden(R):
    g = load_golden("golden_cfg0.npz")
    model = R.ReferenceModel.from_refs(g["refs"], (8, 8))
    fld = R.field_exact_oracle(g["frames"][-1], model)
    s = int(g["exact_stride"])
    assert np.array_equal(fld.indices.ravel()[::s], g["exact_idx"])
    assert np.array_equal(_bits(fld.distances.ravel()[::s]), _bits(g["exact_dist"]))


@pytest.mark.parametrize("cfg_id", [1, 2])
def test_vga_full_frames_match_golden_positions(R, cfg_id):
    """Configs 1-2: all 299,409 positions per frame on the GPU; the golden
    positions (live reference, engine.py:137-143) must match bit for bit."""
    from paper_1508_07953_b200 import workloads as W

    g = load_golden(f"golden_cfg{cfg_id}.npz")
    cfg = W.CONFIGS[cfg_id]
    frames = W.clip(cfg)
    assert W.digest(frames) == str(g["frames_digest"])
    refs = W.reference_set(cfg)
    model = R.ReferenceModel.from_refs(refs, cfg.patch)
    rows = g["table_rows"]
    sd, si = model.table_rows(0, model.n)
    assert np.array_equal(sd[rows], g["table_rows_dist"])
    assert np.array_equal(si[rows], g["table_rows_idx"])
    assert W.digest(sd, si) == str(g["table_digest"])
    pos = g["positions"]
    for t, (_, fld, st) in enumerate(R.stream_fields(model, frames, R.SearchParams())):
        assert np.array_equal(fld.indices.ravel()[pos], g["idx"][t]), t
        assert np.array_equal(_bits(fld.distances.ravel()[pos]), _bits(g["dist"][t])), t


def test_rgb_small_clip_vs_oracle(R, oracle_mod):
    """D=192 (plane-major RGB) path on a small config-3-like clip, all positions."""
    from dataclasses import replace

    from paper_1508_07953_b200 import workloads as W

    cfg = replace(W.CONFIGS[3], height=48, width=72, frames=4, n_refs=2048)
    frames = W.clip(cfg)
    refs = W.reference_set(cfg)
    model = R.ReferenceModel.from_refs(refs, cfg.patch, channels=3)
    om = oracle_mod.OracleModel.build(refs)
    sd, si = model.table_rows(0, model.n)
    assert np.array_equal(sd, om.sorted_dist) and np.array_equal(si, om.sorted_idx)
    gw, gh = cfg.grid
    prev = oracle_mod.init_field_indices(gw, gh, model.n, 0)
    prev_unit = None
    for t, (_, fld, st) in enumerate(R.stream_fields(model, frames, R.SearchParams())):
        idx, dist, ost, unit = oracle_mod.process_frame(om, frames[t], prev, cfg.patch, t + 1, prev_unit=prev_unit)
        assert np.array_equal(fld.indices, idx), t
        assert np.array_equal(_bits(fld.distances), _bits(dist)), t
        assert st.total_rings == ost["total_rings"] and st.total_distance_evals == ost["total_distance_evals"]
        assert st.mean_candidates == ost["mean_candidates"]
        assert st.temporal_change == ost["temporal_change"]
        assert st.first_ring_total == ost["sum_first_ring"]
        prev, prev_unit = idx, unit


def test_engine_properties(R):
    """test_engine.py:79-169 ports: never worse, monotone on a static frame,
    frame counter, stats counting, error paths."""
    from paper_1508_07953_b200 import workloads as W

    rng = np.random.default_rng(2)
    frame = W.clip(W.CONFIGS[0], 1)[0][:32, :32].copy()
    refs, _ = R.normalize_rows(R.extract_patches(frame, (4, 4)).values[rng.choice(29 * 29, 40, replace=False)])
    model = R.ReferenceModel.from_refs(refs, (4, 4))
    gw, gh = R.grid_shape(frame.shape, model.patch_size)
    f0 = R.init_field(gw, gh, model.n, seed=0)
    f1, st = R.process_frame(frame, f0, model)
    unit = R.frame_units(frame, model)
    dprev = np.array([model.metric(unit[g], model.refs[int(p)]) for g, p in enumerate(f0.indices.ravel())])
    assert np.all(f1.distances.ravel() <= dprev + 1e-12)
    assert st.queries == gw * gh and st.total_distance_evals >= 2 * st.queries
    assert st.total_rings >= st.queries and st.temporal_change == 0.0
    fld, prevd = R.init_field(gw, gh, model.n, seed=1), np.full((gh, gw), np.inf)
    for k in range(5):
        fld, _ = R.process_frame(frame, fld, model)
        assert fld.frame_t == k + 1
        assert np.all(fld.distances <= prevd)
        prevd = fld.distances
    with pytest.raises(R.DimensionError):
        R.process_frame(frame, R.init_field(5, 5, model.n), model)
    with pytest.raises(R.DimensionError):
        R.process_frame(frame, f0, model, prev_unit=np.zeros((3, 16), np.float32))
    with pytest.raises(ValueError):
        R.process_frame(frame, f0, model, threads=0)
    moved = np.roll(frame, 2, axis=1)
    _, s2 = R.process_frame(moved, f1, model, prev_unit=unit)
    u2 = R.frame_units(moved, model)
    diff = u2.astype(np.float64) - unit.astype(np.float64)
    assert s2.temporal_change == float(np.sum(np.sqrt(np.sum(diff * diff, axis=1))))


@pytest.mark.parametrize("path", [0, 1])
def test_frame_paths_identical(R, oracle_mod, path):
    """The anchor-grouped (bulk) frame path and the per-query kernel give the
    same bits as the oracle (D=64 config 0 and D=192 RGB clip)."""
    from dataclasses import replace

    from paper_1508_07953_b200 import _native as N
    from paper_1508_07953_b200 import workloads as W

    N.set_frame_path(path)
    try:
        for cfg in (W.CONFIGS[0], replace(W.CONFIGS[3], height=40, width=96, frames=3, n_refs=4096)):
            frames = W.clip(cfg, 3)
            refs = W.reference_set(cfg)
            model = R.ReferenceModel.from_refs(refs, cfg.patch, channels=cfg.channels)
            sd, si = model.table_rows(0, model.n)
            om = oracle_mod.OracleModel(refs, sd, si)
            gw, gh = cfg.grid
            prev = oracle_mod.init_field_indices(gw, gh, model.n, 0)
            for t, (_, fld, st) in enumerate(R.stream_fields(model, frames)):
                idx, dist, ost, _ = oracle_mod.process_frame(om, frames[t], prev, cfg.patch, t + 1)
                assert np.array_equal(fld.indices, idx), (cfg.name, t)
                assert np.array_equal(_bits(fld.distances), _bits(dist)), (cfg.name, t)
                assert st.total_distance_evals == ost["total_distance_evals"]
                assert st.total_rings == ost["total_rings"]
                prev = idx
    finally:
        N.set_frame_path(0)


# ---------------------------------------------------------------------------
# K4 exact comparator: tensor-core screen (tcgen05) + float64 re-check vs the
# oracle's exact_nn (evaluation.py:24-33) and vs the SIMT full scan.
def _exact_both_paths(R, queries, model):
    from paper_1508_07953_b200 import _native as N

    a = R.exact_nn_batch(queries, model)
    N.set_frame_path(2)
    try:
        b = R.exact_nn_batch(queries, model)
    finally:
        N.set_frame_path(0)
    return a, b


def _exact_stats(model, queries):
    import ctypes

    from paper_1508_07953_b200 import _native as N
    from paper_1508_07953_b200.evaluation import _upload_refs

    import torch

    q = torch.from_numpy(np.ascontiguousarray(queries, np.float32)).cuda()
    idx = torch.empty(q.shape[0], dtype=torch.int32, device="cuda")
    dist = torch.empty(q.shape[0], dtype=torch.float64, device="cuda")
    st = (ctypes.c_uint64 * 2)()
    ctx = N.context()
    with ctx.lock:
        _upload_refs(ctx, model)
        torch.cuda.synchronize()
        N.check(N.lib().riann_exact_nn_device(ctx.h, q.data_ptr(), q.shape[0], idx.data_ptr(), dist.data_ptr(), st))
        N.check(N.lib().riann_sync(ctx.h))
    return idx.cpu().numpy(), dist.cpu().numpy(), int(st[0]), int(st[1])


@pytest.mark.parametrize("dim,patch,ch", [(64, (8, 8), 1), (192, (8, 8), 3)])
@pytest.mark.parametrize("n,m", [(1, 5), (7, 130), (1000, 1001), (4096, 3000)])
def test_exact_tc_vs_oracle(R, oracle_mod, dim, patch, ch, n, m):
    rng = np.random.default_rng(dim * 7 + n)
    refs, _ = R.normalize_rows(rng.standard_normal((n, dim)).astype(np.float32))
    q, _ = R.normalize_rows(rng.standard_normal((m, dim)).astype(np.float32))
    q[: min(m, n) // 2] = refs[: min(m, n) // 2]           # exact hits (distance 0)
    model = R.ReferenceModel.from_refs(refs, patch, channels=ch)
    want_i, want_d = oracle_mod.exact_nn_batch(refs, q)
    (ai, ad), (bi, bd) = _exact_both_paths(R, q, model)
    assert np.array_equal(ai, want_i) and np.array_equal(_bits(ad), _bits(want_d))
    assert np.array_equal(bi, want_i) and np.array_equal(_bits(bd), _bits(want_d))


@pytest.mark.parametrize("dim,patch,ch", [(64, (8, 8), 1), (192, (8, 8), 3)])
def test_exact_tc_ties_and_overflow(R, oracle_mod, dim, patch, ch):
    """Duplicate references (ties -> lowest index, numpy argmin) and clusters of
    near-identical references that overflow the screen's candidate list (those
    queries take the exact full scan)."""
    rng = np.random.default_rng(11)
    base, _ = R.normalize_rows(rng.standard_normal((8, dim)).astype(np.float32))
    near = np.repeat(base, 40, axis=0) + rng.standard_normal((320, dim)).astype(np.float32) * 1e-6
    dup = np.repeat(base[:4], 3, axis=0)
    refs = np.concatenate([near, dup, rng.standard_normal((200, dim)).astype(np.float32)])
    refs, _ = R.normalize_rows(refs)
    q = np.concatenate([base, refs[::7], rng.standard_normal((300, dim)).astype(np.float32) * 0.1])
    q = np.ascontiguousarray(q, np.float32)
    model = R.ReferenceModel.from_refs(refs, patch, channels=ch)
    want_i, want_d = oracle_mod.exact_nn_batch(refs, q)
    gi, gd, checked, fb = _exact_stats(model, q)
    assert np.array_equal(gi, want_i) and np.array_equal(_bits(gd), _bits(want_d))
    assert fb >= 8, "near-identical clusters should overflow the candidate list"
    (ai, ad), (bi, bd) = _exact_both_paths(R, q, model)
    assert np.array_equal(ai, want_i) and np.array_equal(bi, want_i)


def test_exact_tc_field_cfg3_sample(R):
    """Config-3 shape (D=192, n=8192 here): the tensor-core path and the SIMT
    scan agree bit for bit on 20,000 frame units; the screen re-checks only a
    few candidates per query."""
    from dataclasses import replace

    from paper_1508_07953_b200 import workloads as W

    cfg = replace(W.CONFIGS[3], height=120, width=200, frames=1, n_refs=8192)
    frame = W.clip(cfg, 1)[0]
    refs = W.reference_set(cfg)
    model = R.ReferenceModel.from_refs(refs, cfg.patch, channels=cfg.channels)
    units = R.frame_units(frame, model)[:20000]
    (ai, ad), (bi, bd) = _exact_both_paths(R, units, model)
    assert np.array_equal(ai, bi) and np.array_equal(_bits(ad), _bits(bd))
    _, _, checked, fb = _exact_stats(model, units)
    assert checked < 8 * len(units) and fb < len(units) // 100


def test_model_switch_smaller_n(R, oracle_mod):
    """A context reused for a model with fewer references: stale pool entries
    from the larger model must never be used as indices (regression)."""
    from dataclasses import replace

    from paper_1508_07953_b200 import workloads as W

    big = replace(W.CONFIGS[1], height=48, width=72, frames=2)
    mb = R.ReferenceModel.from_refs(W.reference_set(W.CONFIGS[1]), big.patch)
    for _ in R.stream_fields(mb, W.clip(big)):
        pass
    cfg = replace(W.CONFIGS[3], height=40, width=64, frames=3, n_refs=2048)
    frames = W.clip(cfg)
    refs = W.reference_set(cfg)
    model = R.ReferenceModel.from_refs(refs, cfg.patch, channels=3)
    sd, si = model.table_rows(0, model.n)
    om = oracle_mod.OracleModel(refs, sd, si)
    gw, gh = cfg.grid
    prev = oracle_mod.init_field_indices(gw, gh, model.n, 0)
    for t, (_, fld, st) in enumerate(R.stream_fields(model, frames)):
        idx, dist, ost, _ = oracle_mod.process_frame(om, frames[t], prev, cfg.patch, t + 1)
        assert np.array_equal(fld.indices, idx), t
        assert np.array_equal(_bits(fld.distances), _bits(dist)), t
        prev = idx


@pytest.mark.parametrize("L,alpha,max_rings", [(4, 0.3, 12), (1, 0.25, 2), (50, 0.1, 8), (1, 0.9, 80)])
def test_frame_path_search_params(R, oracle_mod, L, alpha, max_rings):
    """Non-default SearchParams through the bulk path: long ring caps (more
    used anchors than the draw kernel tracks: those queries are finished by K2
    from scratch), a single ring phase, a large L.  Bit-identical to the oracle."""
    from paper_1508_07953_b200 import workloads as W

    cfg = W.CONFIGS[0]
    frames = W.clip(cfg, 3)
    refs = W.reference_set(cfg)
    model = R.ReferenceModel.from_refs(refs, cfg.patch)
    sd, si = model.table_rows(0, model.n)
    om = oracle_mod.OracleModel(refs, sd, si)
    gw, gh = cfg.grid
    prev = oracle_mod.init_field_indices(gw, gh, model.n, 0)
    params = R.SearchParams(L=L, alpha=alpha, max_rings=max_rings)
    for t, (_, fld, st) in enumerate(R.stream_fields(model, frames, params)):
        idx, dist, ost, _ = oracle_mod.process_frame(om, frames[t], prev, cfg.patch, t + 1, L=L, alpha=alpha,
                                                     max_rings=max_rings)
        assert np.array_equal(fld.indices, idx), t
        assert np.array_equal(_bits(fld.distances), _bits(dist)), t
        assert st.total_rings == ost["total_rings"] and st.total_distance_evals == ost["total_distance_evals"]
        prev = idx


def test_frame_path_k2_only_model(R, oracle_mod):
    """n % 16 != 0: the bulk path declines the model and every query runs K2;
    still bit-identical to the oracle."""
    from paper_1508_07953_b200 import workloads as W

    cfg = W.CONFIGS[0]
    frames = W.clip(cfg, 3)
    refs = W.reference_set(cfg)[:1000]
    model = R.ReferenceModel.from_refs(refs, cfg.patch)
    sd, si = model.table_rows(0, model.n)
    om = oracle_mod.OracleModel(refs, sd, si)
    gw, gh = cfg.grid
    prev = oracle_mod.init_field_indices(gw, gh, model.n, 0)
    for t, (_, fld, st) in enumerate(R.stream_fields(model, frames)):
        idx, dist, ost, _ = oracle_mod.process_frame(om, frames[t], prev, cfg.patch, t + 1)
        assert np.array_equal(fld.indices, idx), t
        assert np.array_equal(_bits(fld.distances), _bits(dist)), t
        assert st.total_rings == ost["total_rings"] and st.total_distance_evals == ost["total_distance_evals"]
        prev = idx


def test_many_used_anchors_inside_s(R, oracle_mod):
    """A drawn anchor stays inside S only if its own ring contains it, i.e. at
    distance 0 (search.py:131-135): 50 exact copies of the query among the
    references, L = 1, max_rings = 80.  Every draw picks a copy and keeps S, so
    the used anchors inside S (prev included) grow to 50 until avail is empty
    (search.py:122-124).  K2 tracks up to 128 of them (was 32:
    NotImplementedError).  All outputs equal the oracle's."""
    rng = np.random.default_rng(8)
    other, _ = R.normalize_rows(rng.normal(size=(250, 64)).astype(np.float32))
    v = other[:1]
    refs = np.concatenate([other[1:100], np.repeat(v, 50, axis=0), other[100:]])
    model = R.ReferenceModel.from_refs(refs, (64, 1))
    dup = np.arange(99, 149)
    q = np.repeat(v, 8, axis=0)
    prev = dup[rng.integers(0, 50, 8)]
    params = R.SearchParams(L=1, alpha=0.25, max_rings=80)
    keys = [(3, int(i), 1, 2) for i in range(8)]
    res = R.riann_query_batch(model, q, prev, params, keys=keys, scanned=True)
    sd, si = model.table_rows(0, model.n)
    om = oracle_mod.OracleModel(refs, sd, si)
    for i in range(8):
        r = oracle_mod.query(om, q[i], int(prev[i]), L=1, alpha=0.25, max_rings=80, key=keys[i])
        assert r["match_index"] == res["idx"][i] and r["rings_drawn"] == res["rings"][i], i
        assert r["distance_evals"] == res["evals"][i] and r["candidates_final"] == res["cand"][i], i
        assert np.array_equal(r["scanned"], res["scanned"][i]), i
    assert (res["rings"] == 50).all()  # first ring + 49 draws: prev is a used copy too


@pytest.mark.parametrize("n", [4112, 8208])
def test_bulk_path_unaligned_half(R, oracle_mod, n):
    """n % 16 == 0 but n/2 not a multiple of the P0b bucket width nor of 32
    (n = 4,112: n/2 = 2,056): the part-A/B split falls inside a bucket of the
    radix path and inside a bitmap word of the bitmap path.  Whole frames vs
    the oracle, bit for bit."""
    from dataclasses import replace

    from paper_1508_07953_b200 import workloads as W

    cfg = replace(W.CONFIGS[1], height=72, width=96, frames=3, n_refs=n)
    clip = W.clip(cfg)
    refs = W.reference_set(cfg)
    model = R.ReferenceModel.from_refs(refs, cfg.patch)
    om = oracle_mod.OracleModel.build(refs)
    gw, gh = cfg.grid
    prev = oracle_mod.init_field_indices(gw, gh, n, 0)
    prev_unit = None
    for t, (_, fld, st) in enumerate(R.stream_fields(model, clip)):
        idx, dist, ost, unit = oracle_mod.process_frame(om, clip[t], prev, cfg.patch, t + 1, prev_unit=prev_unit)
        assert np.array_equal(fld.indices, idx), t
        assert np.array_equal(_bits(fld.distances), _bits(dist)), t
        assert st.total_rings == ost["total_rings"] and st.total_distance_evals == ost["total_distance_evals"]
        prev, prev_unit = idx, unit
