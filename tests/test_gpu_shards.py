"""Row-sharded tables (shards.py): shards built by K3 on
row ranges, attached to a querying context, read by the per-query kernel
through the shard table.  On one GPU the shards are separate allocations
owned by separate contexts; on a multi-GPU node the same pointers are NVLink
peer pointers.  Bar: tables, query outputs and fields identical to the
unsharded model and to the CPU oracle (model.py:162-189, search.py:83-151)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def R():
    import paper_1508_07953_b200 as R

    return R


def _bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def _setup(R, n, shards, height=96, width=128, frames=3):
    from dataclasses import replace

    from paper_1508_07953_b200 import workloads as W

    cfg = replace(W.CONFIGS[1], height=height, width=width, frames=frames, n_refs=n)
    clip = W.clip(cfg)
    refs = W.reference_set(cfg)
    full = R.ReferenceModel.from_refs(refs, cfg.patch)
    sharded = R.ReferenceModel.from_refs(refs, cfg.patch)
    st = R.shard_model(sharded, devices=[0] * shards, shards=shards)
    return cfg, clip, refs, full, sharded, st


@pytest.mark.parametrize("n,shards", [(4096, 4), (2048, 3), (1000, 7)])
def test_shard_tables_match_oracle(R, oracle_mod, n, shards):
    cfg, clip, refs, full, sharded, st = _setup(R, n, shards)
    for r0, rows in st.rows:
        probe = [r0, r0 + rows // 2, r0 + rows - 1]
        want_d, want_i = oracle_mod.sorted_lists(refs, rows=(r0, r0 + rows))
        for r in probe:
            sd, si = st.table_rows(r, 1)
            assert np.array_equal(sd[0], want_d[r - r0]) and np.array_equal(si[0], want_i[r - r0])
    st.close()


@pytest.mark.parametrize("n,shards", [(4096, 4), (2048, 3)])
def test_sharded_stream_equals_unsharded_and_oracle(R, oracle_mod, n, shards):
    cfg, clip, refs, full, sharded, st = _setup(R, n, shards)
    base = [(f.indices.copy(), f.distances.copy(), s) for _, f, s in R.stream_fields(full, clip)]
    got = [(f.indices.copy(), f.distances.copy(), s) for _, f, s in R.stream_fields(sharded, clip)]
    om = oracle_mod.OracleModel.build(refs)
    gw, gh = cfg.grid
    prev = oracle_mod.init_field_indices(gw, gh, n, 0)
    prev_unit = None
    for t in range(clip.shape[0]):
        assert np.array_equal(got[t][0], base[t][0]), t
        assert np.array_equal(_bits(got[t][1]), _bits(base[t][1])), t
        assert got[t][2] == base[t][2]
        idx, dist, ost, unit = oracle_mod.process_frame(om, clip[t], prev, cfg.patch, t + 1, prev_unit=prev_unit)
        assert np.array_equal(got[t][0], idx) and np.array_equal(_bits(got[t][1]), _bits(dist)), t
        assert got[t][2].total_rings == ost["total_rings"]
        assert got[t][2].total_distance_evals == ost["total_distance_evals"]
        prev, prev_unit = idx, unit
    st.close()


def test_sharded_query_batch(R, oracle_mod):
    cfg, clip, refs, full, sharded, st = _setup(R, 4096, 4)
    rng = np.random.default_rng(5)
    q, _ = R.normalize_rows(refs[rng.integers(0, 4096, 600)] + rng.normal(0, 0.02, (600, 64)).astype(np.float32))
    prev = rng.integers(0, 4096, 600)
    keys = [(0, int(i), 7, 3) for i in range(600)]
    a = R.riann_query_batch(sharded, q, prev, R.SearchParams(), keys=keys, scanned=True)
    b = R.riann_query_batch(full, q, prev, R.SearchParams(), keys=keys, scanned=True)
    for k in ("idx", "rings", "evals", "cand", "first"):
        assert np.array_equal(a[k], b[k]), k
    assert np.array_equal(_bits(a["dist"]), _bits(b["dist"]))
    assert all(np.array_equal(x, y) for x, y in zip(a["scanned"], b["scanned"]))
    om = oracle_mod.OracleModel.build(refs)
    for i in range(0, 600, 37):
        r = oracle_mod.query(om, q[i], int(prev[i]), key=keys[i])
        assert r["match_index"] == a["idx"][i] and r["rings_drawn"] == a["rings"][i]
    st.close()


def test_closed_shards_fail_loudly(R):
    """After ShardedTables.close() the querying context has no tables: a
    later call re-attaches (model.resident) or fails, never reads freed rows."""
    cfg, clip, refs, full, sharded, st = _setup(R, 1024, 2)
    list(R.stream_fields(sharded, clip[:1]))
    st.close()
    object.__setattr__(sharded, "_sharded", None)
    from paper_1508_07953_b200 import _native as N

    ctx = N.context()
    with ctx.lock:
        assert ctx.model_token is None
    # the model is simply re-made resident with its own tables
    a = [f.indices.copy() for _, f, _ in R.stream_fields(sharded, clip)]
    b = [f.indices.copy() for _, f, _ in R.stream_fields(full, clip)]
    assert all(np.array_equal(x, y) for x, y in zip(a, b))
