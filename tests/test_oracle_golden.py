"""Pin the CPU oracle (oracle/) against golden vectors from the live reference.

The fixtures come from tests/golden/make_golden.py, which imports the
reference package (/root/reference/pkg/src/riann) in the build container.
"""

import numpy as np
import pytest

from conftest import load_golden, ragged


def test_fixture_numpy_version_matches():
    g = load_golden("golden_rng.npz")
    assert str(g["numpy_version"]) == np.__version__


def test_rng_draw_sequences(oracle_mod):
    g = load_golden("golden_rng.npz")
    koff = g["key_off"]
    for i in range(len(koff) - 1):
        key = [int(v) for v in ragged(g["key_flat"], koff, i)]
        p = oracle_mod.Pcg64(tuple(key))
        got = [p.integers(int(k)) for k in g["k"][i]]
        assert got == [int(v) for v in g["draws"][i]], (i, key)


def test_init_field_matches_numpy_stream(oracle_mod):
    g = load_golden("golden_rng.npz")
    for i, (gw, gh, n, seed) in enumerate(g["init_args"]):
        want = ragged(g["init_flat"], g["init_off"], i).reshape(int(gh), int(gw))
        got = oracle_mod.init_field_indices(int(gw), int(gh), int(n), int(seed))
        assert np.array_equal(got, want)


def test_one_to_many_bit_exact(oracle_mod):
    g = load_golden("golden_arith.npz")
    for i, d in enumerate(g["dims"]):
        q = ragged(g["q"], g["q_off"], i)
        r = ragged(g["r"], g["r_off"], i).reshape(-1, int(d))
        want = ragged(g["d"], g["d_off"], i)
        got = oracle_mod.one_to_many(q, r)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), int(d)


def test_normalize_rows_bit_exact(oracle_mod):
    g = load_golden("golden_arith.npz")
    for i, d in enumerate(g["dims"]):
        v = ragged(g["norm_in"], g["norm_in_off"], i).reshape(-1, int(d))
        want_u = ragged(g["norm_unit"], g["norm_in_off"], i).reshape(-1, int(d))
        want_n = ragged(g["norm_norms"], g["norm_off"], i)
        u, nr = oracle_mod.normalize_rows(v)
        assert np.array_equal(u.view(np.uint32), want_u.view(np.uint32)), int(d)
        assert np.array_equal(nr, want_n), int(d)


def test_sorted_lists_bit_exact(oracle_mod):
    g = load_golden("golden_tables.npz")
    for i, (n, d) in enumerate(g["shapes"]):
        refs = ragged(g["refs"], g["refs_off"], i).reshape(int(n), int(d))
        sd, si = oracle_mod.sorted_lists(refs, nthreads=2)
        assert np.array_equal(sd.ravel().view(np.uint32),
                              ragged(g["sdist"], g["tab_off"], i).view(np.uint32))
        assert np.array_equal(si.ravel(), ragged(g["sidx"], g["tab_off"], i))


def _query_models(oracle_mod, g):
    models = []
    for i, (n, d) in enumerate(g["model_shapes"]):
        refs = ragged(g["models"], g["model_off"], i).reshape(int(n), int(d))
        models.append(oracle_mod.OracleModel.build(refs, nthreads=2))
    return models


def test_riann_query_all_outputs(oracle_mod):
    g = load_golden("golden_queries.npz")
    models = _query_models(oracle_mod, g)
    for c in range(len(g["mid"])):
        m = models[int(g["mid"][c])]
        key = tuple(int(v) for v in ragged(g["key"], g["key_off"], c))
        r = oracle_mod.query(m, ragged(g["q"], g["q_off"], c), int(g["prev"][c]),
                             int(g["L"][c]), float(g["alpha"][c]), int(g["mr"][c]), key)
        assert r["match_index"] == g["idx"][c], c
        assert r["match_distance"] == g["dist"][c], c
        assert r["rings_drawn"] == g["rings"][c], c
        assert r["distance_evals"] == g["evals"][c], c
        assert r["candidates_final"] == g["cand"][c], c
        assert np.array_equal(r["scanned"], ragged(g["scanned"], g["scanned_off"], c)), c


def test_cfg0_stream_bit_exact(oracle_mod):
    """Config 0 end to end (engine.py:205-227): every position, all frames."""
    from paper_1508_07953_b200 import workloads as W

    g = load_golden("golden_cfg0.npz")
    cfg = W.CONFIGS[0]
    frames, refs = g["frames"], g["refs"]
    assert W.digest(frames) == W.digest(W.clip(cfg))
    assert W.digest(refs) == W.digest(W.reference_set(cfg))
    model = oracle_mod.OracleModel.build(refs)
    assert W.digest(model.sorted_dist, model.sorted_idx) == str(g["table_digest"])
    gw, gh = cfg.grid
    prev = oracle_mod.init_field_indices(gw, gh, model.n, 0)
    prev_unit = None
    for t in range(frames.shape[0]):
        idx, dist, st, unit = oracle_mod.process_frame(model, frames[t], prev, cfg.patch, t + 1,
                                                       prev_unit=prev_unit)
        assert np.array_equal(idx, g["idx"][t])
        assert np.array_equal(dist.view(np.uint64), g["dist"][t].view(np.uint64))
        assert [st["total_rings"], st["total_distance_evals"], st["queries"]] == list(g["stats_int"][t])
        assert st["mean_candidates"] == g["stats_f"][t][0]
        assert st["temporal_change"] == g["stats_f"][t][1]
        prev, prev_unit = idx, unit


def test_cfg0_exact_nn(oracle_mod):
    from paper_1508_07953_b200 import workloads as W

    g = load_golden("golden_cfg0.npz")
    cfg = W.CONFIGS[0]
    unit, _ = oracle_mod.frame_units(g["frames"][-1], cfg.patch)
    s = int(g["exact_stride"])
    idx, dist = oracle_mod.exact_nn_batch(g["refs"], unit[::s])
    assert np.array_equal(idx, g["exact_idx"])
    assert np.array_equal(dist, g["exact_dist"])


@pytest.mark.parametrize("cfg_id", [1, 2])
def test_vga_sampled_positions(oracle_mod, cfg_id):
    """Configs 1-2: seeded positions through all 30 frames (engine.py:137-143)."""
    from paper_1508_07953_b200 import workloads as W

    g = load_golden(f"golden_cfg{cfg_id}.npz")
    cfg = W.CONFIGS[cfg_id]
    frames = W.clip(cfg)
    assert W.digest(frames) == str(g["frames_digest"])
    refs = W.reference_set(cfg)
    assert W.digest(refs) == str(g["refs_digest"])
    sd, si = oracle_mod.sorted_lists(refs, rows=None)
    assert W.digest(sd, si) == str(g["table_digest"])
    model = oracle_mod.OracleModel(refs, sd, si)
    gw, gh = cfg.grid
    pos = g["positions"]
    prev = g["init_prev"].copy()
    for t in range(frames.shape[0]):
        ys = pos // gw
        unit, _ = oracle_mod.frame_units(frames[t], cfg.patch)
        r = oracle_mod.query_positions(model, unit[pos], prev, pos, gw, 0, t + 1)
        assert np.array_equal(r["idx"], g["idx"][t]), t
        assert np.array_equal(r["dist"], g["dist"][t]), t
        assert np.array_equal(r["rings"], g["rings"][t]), t
        assert np.array_equal(r["evals"], g["evals"][t]), t
        assert np.array_equal(r["cand"], g["cand"][t]), t
        prev = r["idx"]
        del ys


def _cfg3_golden_setup(g):
    from dataclasses import replace

    from paper_1508_07953_b200 import workloads as W

    cfg = replace(W.CONFIGS[3], n_refs=int(g["n_refs"]))
    refs = W.reference_set(cfg)
    assert W.digest(refs) == str(g["refs_digest"])
    return W, cfg, refs


def test_cfg3_d192_units_and_queries(oracle_mod):
    """D=192 (config 3's 1080p RGB clip, n=8,192 config-3-shaped reference set):
    plane-major unit rows and riann_query through 10 frames vs the live
    reference (search.py:83-151 on transforms.py:152-157-style rows)."""
    g = load_golden("golden_cfg3.npz")
    W, cfg, refs = _cfg3_golden_setup(g)
    sd, si = oracle_mod.sorted_lists(refs)
    rows = g["table_rows"]
    assert np.array_equal(sd[rows], g["table_rows_dist"])
    assert np.array_equal(si[rows], g["table_rows_idx"])
    assert W.digest(sd, si) == str(g["table_digest"])
    model = oracle_mod.OracleModel(refs, sd, si)
    gw, gh = cfg.grid
    pos = g["positions"]
    prev = g["init_prev"].copy()
    for t, frame in enumerate(W.iter_clip(cfg, g["idx"].shape[0])):
        assert W.digest(frame) == str(g["frame_digests"][t])
        unit = oracle_mod.normalize_rows(W.patch_rows(frame, cfg.patch, pos // gw, pos % gw))[0]
        assert np.array_equal(unit, g["units"][t]), t
        r = oracle_mod.query_positions(model, unit, prev, pos, gw, 0, t + 1)
        for k in ("idx", "dist", "rings", "evals", "cand"):
            assert np.array_equal(r[k], g[k][t]), (k, t)
        prev = r["idx"]


def test_cfg4_exact_nn_golden(oracle_mod):
    """exact_nn (evaluation.py:24-33) at config 4's shape, n=262,144, D=64."""
    from paper_1508_07953_b200 import workloads as W

    g = load_golden("golden_cfg4x.npz")
    cfg = W.CONFIGS[4]
    refs = W.reference_set(cfg)
    assert W.digest(refs) == str(g["refs_digest"])
    frame = next(W.iter_clip(cfg, 1))
    assert W.digest(frame) == str(g["frame_digest"])
    gw, gh = cfg.grid
    pos = g["positions"]
    unit = oracle_mod.normalize_rows(W.patch_rows(frame, cfg.patch, pos // gw, pos % gw))[0]
    assert np.array_equal(unit, g["units"])
    idx, dist = oracle_mod.exact_nn_batch(refs, unit)
    assert np.array_equal(idx, g["idx"])
    assert np.array_equal(dist, g["dist"])
