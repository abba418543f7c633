"""Generate golden fixtures from the LIVE reference (run in the build container).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--skip-vga]

Imports riann from /root/reference/pkg/src (read-only; it does not exist on
the GPU box, so only this script touches it) and writes small .npz fixtures
next to this file.  Each fixture records the numpy version, because numpy's
Generator streams are not guaranteed stable across versions.

Fixtures:
  golden_rng.npz      SeedSequence/PCG64/Generator.integers draw sequences for
                      keys of 1, 2, 4 and 5+ words; init_field outputs.
  golden_arith.npz    one_to_many (patches.py:151-159) and normalize_rows
                      (patches.py:100-115) on random rows of many widths,
                      including zero and sub-threshold rows.
  golden_tables.npz   compute_sorted_lists (model.py:162-189) on models with
                      exact duplicates and ties.
  golden_queries.npz  riann_query (search.py:83-151) on seeded small models,
                      all outputs incl. scanned sets, many param settings.
  golden_cfg0.npz     config 0 end to end: stream_fields (engine.py:205-227)
                      over all 8 frames, every position, FrameStats.
  golden_annf.npz     ANNF containers written by the reference AnnfWriter
                      (engine.py:228-279) from the config-0 golden fields, and
                      an empty stream.
  golden_effects.npz  apply_effect (transforms.py:192-246) for the three
                      payload kinds on the config-0 field and on a small
                      non-square-patch model.
  golden_coherency.npz coherency_stats (evaluation.py:86-138) on the first 4
                      config-0 frames (exact fields, shift/residual samples).
  golden_rian.npz     RIAN containers from the reference serialize_model
                      (model.py:398-411) for two small models (one 3-channel).
  golden_cfg1.npz /   configs 1-2: riann_query at a seeded sample of positions
  golden_cfg2.npz     through all 30 frames, exactly as engine.py:137-143
                      calls it (positions are independent).
  golden_cfg3.npz     the D=192 path (config 3's 1080p RGB clip, first 10
                      frames): a config-3-shaped reference set cut to n=8,192
                      (reference compute_sorted_lists), plane-major 192-D unit
                      rows built with the reference's own extract_patches per
                      plane + normalize_rows (transforms.py:152-157
                      precedent), riann_query at 256 seeded
                      positions through the 10 frames.
  golden_cfg4x.npz    exact_nn (evaluation.py:24-33) at config 4's shape
                      (n=262,144, D=64) on 256 positions of the first frame.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

from riann.engine import stream_fields  # noqa: E402
from riann.evaluation import exact_nn  # noqa: E402
from riann.model import ReferenceModel, compute_sorted_lists  # noqa: E402
from riann.patches import EUCLIDEAN, extract_patches, normalize_rows  # noqa: E402
from riann.search import SearchParams, query_rng_key, riann_query  # noqa: E402

from paper_1508_07953_b200 import workloads as W  # noqa: E402

NPV = np.__version__


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, numpy_version=np.array(NPV), **arrays)
    print(f"wrote {name} ({os.path.getsize(path) / 1024:.0f} KiB)")


def ragged(seqs, dtype):
    off = np.zeros(len(seqs) + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(s) for s in seqs])
    flat = np.concatenate([np.asarray(s, dtype=dtype) for s in seqs]) if seqs else np.zeros(0, dtype)
    return flat, off


def make_model(refs, patch_size=None):
    refs = np.asarray(refs, dtype=np.float32)
    sd, si = compute_sorted_lists(refs)
    if patch_size is None:
        patch_size = (refs.shape[1], 1)
    return ReferenceModel(refs=refs, sorted_dist=sd, sorted_idx=si, patch_size=patch_size)


def gen_rng():
    rng = np.random.default_rng(2024)
    keys, draws, ks = [], [], []
    key_shapes = [1, 2, 4, 4, 4, 5, 7]
    for i in range(400):
        nk = key_shapes[i % len(key_shapes)]
        key = [int(v) for v in rng.integers(0, 2**32, size=nk)]
        if i % 11 == 0:
            key = [0] * nk
        if i % 13 == 0:
            key[0] = int(rng.integers(2**32, 2**63))  # multi-word component
        kseq = [int(v) for v in rng.choice([1, 2, 3, 7, 20, 21, 999, 1024, 8191, 65536,
                                             2**31 - 1, 3 * 2**30, 2**32], size=12)]
        g = np.random.default_rng(tuple(key))
        d = [int(g.integers(k)) for k in kseq]
        keys.append(key)
        ks.append(kseq)
        draws.append(d)
    key_flat = [w for k in keys for w in k]
    kflat, koff = ragged(keys, np.uint64)
    inits = []
    for gw, gh, n, seed in [(3, 2, 10, 7), (50, 40, 7, 0), (57, 57, 1024, 0),
                            (233, 101, 8192, 0), (17, 5, 1, 3), (9, 9, 65536, 2**40 + 5)]:
        g = np.random.default_rng(seed)
        inits.append((gw, gh, n, seed, g.integers(0, n, size=(gh, gw), dtype=np.int32).ravel()))
    iflat, ioff = ragged([x[4] for x in inits], np.int32)
    save("golden_rng.npz", key_flat=kflat, key_off=koff,
         k=np.array(ks, dtype=np.uint64), draws=np.array(draws, dtype=np.uint64),
         init_args=np.array([x[:4] for x in inits], dtype=np.uint64),
         init_flat=iflat, init_off=ioff)
    del key_flat


def gen_arith():
    rng = np.random.default_rng(99)
    dims = [1, 2, 3, 5, 7, 8, 12, 16, 17, 64, 100, 128, 129, 192, 200, 256, 300]
    qs, rs, outs, nin, nunit, nnorm = [], [], [], [], [], []
    for d in dims:
        q = rng.uniform(-1, 1, size=d).astype(np.float32)
        r = rng.uniform(-1, 1, size=(9, d)).astype(np.float32)
        r[0] = q  # identical row -> exact zero
        qs.append(q)
        rs.append(r.ravel())
        outs.append(EUCLIDEAN.one_to_many(q, r))
        v = (rng.uniform(size=(6, d)) * rng.choice([1.0, 1e-3, 1e3], size=(6, 1))).astype(np.float32)
        v[1] = 0.0
        v[2] = 1e-14  # below the zero-norm threshold
        v[3, :] = 0.0
        v[3, 0] = 3.0
        if d > 1:
            v[3, 1] = 4.0
        u, nr = normalize_rows(v)
        nin.append(v.ravel())
        nunit.append(u.ravel())
        nnorm.append(nr)
    q_flat, q_off = ragged(qs, np.float32)
    r_flat, r_off = ragged(rs, np.float32)
    o_flat, o_off = ragged(outs, np.float64)
    ni, ni_off = ragged(nin, np.float32)
    nu, _ = ragged(nunit, np.float32)
    nn, nn_off = ragged(nnorm, np.float64)
    save("golden_arith.npz", dims=np.array(dims), q=q_flat, q_off=q_off, r=r_flat, r_off=r_off,
         d=o_flat, d_off=o_off, norm_in=ni, norm_in_off=ni_off, norm_unit=nu,
         norm_norms=nn, norm_off=nn_off)


def gen_tables():
    rng = np.random.default_rng(5)
    models = []
    s = np.sqrt(2.0) / 2.0
    models.append(np.array([[1.0, 0.0], [0.0, 1.0], [s, s]], dtype=np.float32))
    models.append(np.array([[1, 0], [0, 1], [1, 0], [1, 0], [0, 1]], dtype=np.float32))
    base = rng.normal(size=(40, 16))
    base /= np.linalg.norm(base, axis=1, keepdims=True)
    base = base.astype(np.float32)
    base[7] = base[3]
    base[30] = base[3]
    base[12] = base[29]
    models.append(base)
    blur = W.reference_set(W.CONFIGS[0], 300)
    models.append(blur)
    refs, sd, si = [], [], []
    for m in models:
        d, i = compute_sorted_lists(m)
        refs.append(m.ravel())
        sd.append(d.astype(np.float32).ravel())
        si.append(i.ravel())
        assert np.array_equal(d.astype(np.float32).astype(np.float64), d)
    rf, roff = ragged(refs, np.float32)
    df, _ = ragged(sd, np.float32)
    xf, xoff = ragged(si, np.int32)
    save("golden_tables.npz", shapes=np.array([m.shape for m in models]), refs=rf, refs_off=roff,
         sdist=df, sidx=xf, tab_off=xoff)


def gen_queries():
    rng = np.random.default_rng(77)
    cases = []  # (model_id, q, prev, L, alpha, max_rings, key)
    models = []
    s = np.sqrt(2.0) / 2.0
    models.append(np.array([[1.0, 0.0], [0.0, 1.0], [s, s]], dtype=np.float32))
    models.append(np.array([[1, 0], [0, 1], [1, 0]], dtype=np.float32))
    for n, d in [(120, 16), (150, 16), (200, 16), (5, 8), (80, 12), (500, 64)]:
        r = rng.normal(size=(n, d))
        r /= np.linalg.norm(r, axis=1, keepdims=True)
        models.append(r.astype(np.float32))
    models.append(W.reference_set(W.CONFIGS[0], 1024))
    dup = W.reference_set(W.CONFIGS[0], 256).copy()
    dup[100:140] = dup[0:40]  # exact duplicates exercise ties and self-first rows
    models.append(dup)
    built = [make_model(m) for m in models]
    # tri-model known answers
    cases.append((0, models[0][1], 1, 20, 0.25, 8, 0))
    cases.append((0, models[0][2], 0, 20, 0.25, 8, 0))
    cases.append((0, np.zeros(2, np.float32), 0, 20, 0.25, 8, 0))
    cases.append((1, models[1][0], 2, 20, 0.25, 8, 0))
    for mid in range(2, len(models)):
        n, d = models[mid].shape
        for k in range(60):
            base = models[mid][rng.integers(n)]
            q, _ = normalize_rows((base + rng.normal(scale=rng.choice([0.02, 0.08, 0.3]), size=d))[None])
            if k % 17 == 0:
                q[:] = 0.0
            prev = int(rng.integers(n))
            L = int(rng.choice([1, 2, 5, 20, 20, 20, 50]))
            alpha = float(rng.choice([0.1, 0.25, 0.25, 0.5, 0.9]))
            mr = int(rng.choice([1, 2, 8, 8, 8, 20]))
            kl = int(rng.choice([1, 2, 4, 4]))
            key = tuple(int(v) for v in rng.integers(0, 2**32, size=kl))
            cases.append((mid, q[0], prev, L, alpha, mr, key))
    out = {k: [] for k in ["mid", "prev", "L", "alpha", "mr", "idx", "dist", "rings", "evals", "cand"]}
    qs, keys, scanned = [], [], []
    for (mid, q, prev, L, alpha, mr, key) in cases:
        res = riann_query(built[mid], q, prev, SearchParams(L=L, alpha=alpha, max_rings=mr), rng_state=key)
        out["mid"].append(mid)
        out["prev"].append(prev)
        out["L"].append(L)
        out["alpha"].append(alpha)
        out["mr"].append(mr)
        out["idx"].append(res.match_index)
        out["dist"].append(res.match_distance)
        out["rings"].append(res.rings_drawn)
        out["evals"].append(res.distance_evals)
        out["cand"].append(res.candidates_final)
        qs.append(np.asarray(q, np.float32))
        keys.append(list(key) if isinstance(key, tuple) else [key])
        scanned.append(res.scanned)
    mf, moff = ragged([m.ravel() for m in models], np.float32)
    qf, qoff = ragged(qs, np.float32)
    kf, koff = ragged(keys, np.uint64)
    sf, soff = ragged(scanned, np.int32)
    save("golden_queries.npz", model_shapes=np.array([m.shape for m in models]), models=mf,
         model_off=moff, q=qf, q_off=qoff, key=kf, key_off=koff, scanned=sf, scanned_off=soff,
         **{k: np.array(v) for k, v in out.items()})


def gen_cfg0():
    cfg = W.CONFIGS[0]
    frames = W.clip(cfg)
    refs = W.reference_set(cfg)
    t0 = time.time()
    model = make_model(refs, cfg.patch)
    tb = time.time() - t0
    idx, dist, st, stats_f = [], [], [], []
    t0 = time.time()
    for _, field, stats in stream_fields(model, list(frames), SearchParams(), threads=1):
        idx.append(field.indices.copy())
        dist.append(field.distances.copy())
        st.append([stats.total_rings, stats.total_distance_evals, stats.queries])
        stats_f.append([stats.mean_candidates, stats.temporal_change])
    tq = time.time() - t0
    exact_i, exact_d = [], []
    unit, _ = normalize_rows(extract_patches(frames[-1], cfg.patch).values)
    for g in range(0, unit.shape[0], 7):
        i, d = exact_nn(unit[g], model)
        exact_i.append(i)
        exact_d.append(d)
    print(f"cfg0: table {tb:.2f}s, stream {tq:.2f}s")
    save("golden_cfg0.npz", frames=frames, refs=refs, idx=np.array(idx), dist=np.array(dist),
         stats_int=np.array(st, dtype=np.int64), stats_f=np.array(stats_f),
         table_digest=np.array(W.digest(model.sorted_dist.astype(np.float32), model.sorted_idx)),
         exact_stride=np.array(7), exact_idx=np.array(exact_i, np.int32),
         exact_dist=np.array(exact_d), ref_seconds_stream=np.array(tq))


def gen_vga(cfg_id, model=None, refs=None, npos=256):
    cfg = W.CONFIGS[cfg_id]
    frames = W.clip(cfg)
    if model is None:
        refs = W.reference_set(cfg)
        t0 = time.time()
        model = make_model(refs, cfg.patch)
        print(f"cfg{cfg_id}: table build {time.time() - t0:.1f}s")
    gw, gh = cfg.grid
    rng = np.random.default_rng(1000 + cfg_id)
    pos = np.sort(rng.choice(gw * gh, size=npos, replace=False))
    init = np.random.default_rng(0).integers(0, model.n, size=(gh, gw), dtype=np.int32).ravel()
    prev = init[pos].copy()
    params = SearchParams()
    T = len(frames)
    res = {k: np.empty((T, npos), dt) for k, dt in
           [("idx", np.int32), ("dist", np.float64), ("rings", np.int32),
            ("evals", np.int64), ("cand", np.int64)]}
    t0 = time.time()
    nq = 0
    for t in range(T):
        unit, _ = normalize_rows(extract_patches(frames[t], cfg.patch).values)
        for j, g in enumerate(pos):
            y, x = divmod(int(g), gw)
            r = riann_query(model, unit[g], int(prev[j]), params,
                            rng_state=query_rng_key(params.seed, x, y, t + 1))
            res["idx"][t, j] = r.match_index
            res["dist"][t, j] = r.match_distance
            res["rings"][t, j] = r.rings_drawn
            res["evals"][t, j] = r.distance_evals
            res["cand"][t, j] = r.candidates_final
            nq += 1
        prev = res["idx"][t].copy()
    dt = time.time() - t0
    print(f"cfg{cfg_id}: {nq} queries in {dt:.1f}s ({nq / dt:.0f} q/s single thread)")
    save(f"golden_cfg{cfg_id}.npz", positions=pos, init_prev=init[pos], frames_digest=np.array(W.digest(frames)),
         refs_digest=np.array(W.digest(refs)),
         table_digest=np.array(W.digest(model.sorted_dist.astype(np.float32), model.sorted_idx)),
         table_rows=np.arange(0, model.n, 997),
         table_rows_dist=model.sorted_dist[::997].astype(np.float32),
         table_rows_idx=model.sorted_idx[::997], ref_qps=np.array(nq / dt), **res)
    return model, refs


def rgb_units(frame, patch, pos):
    """Plane-major 192-D unit rows of a (H, W, 3) frame at grid positions,
    built from the reference's extract_patches (one plane at a time, the
    reference has no colour path) and normalize_rows."""
    planes = [extract_patches(np.ascontiguousarray(frame[..., c]), patch).values[pos]
              for c in range(frame.shape[2])]
    unit, _ = normalize_rows(np.concatenate(planes, axis=1))
    return unit


def gen_cfg3(npos=256, nframes=10, n=8192):
    from dataclasses import replace

    cfg = replace(W.CONFIGS[3], n_refs=n)
    refs = W.reference_set(cfg)
    t0 = time.time()
    sd, si = compute_sorted_lists(refs)
    model = ReferenceModel(refs=refs, sorted_dist=sd, sorted_idx=si, patch_size=cfg.patch, channels=3)
    print(f"cfg3 (n={n}, D=192): table build {time.time() - t0:.1f}s")
    gw, gh = cfg.grid
    rng = np.random.default_rng(1003)
    pos = np.sort(rng.choice(gw * gh, size=npos, replace=False))
    init = np.random.default_rng(0).integers(0, model.n, size=(gh, gw), dtype=np.int32).ravel()
    prev = init[pos].copy()
    params = SearchParams()
    res = {k: np.empty((nframes, npos), dt) for k, dt in
           [("idx", np.int32), ("dist", np.float64), ("rings", np.int32),
            ("evals", np.int64), ("cand", np.int64)]}
    units = []
    digests = []
    t0 = time.time()
    for t, frame in enumerate(W.iter_clip(cfg, nframes)):
        digests.append(W.digest(frame))
        unit = rgb_units(frame, cfg.patch, pos)
        units.append(unit)
        for j, g in enumerate(pos):
            y, x = divmod(int(g), gw)
            r = riann_query(model, unit[j], int(prev[j]), params,
                            rng_state=query_rng_key(params.seed, x, y, t + 1))
            res["idx"][t, j] = r.match_index
            res["dist"][t, j] = r.match_distance
            res["rings"][t, j] = r.rings_drawn
            res["evals"][t, j] = r.distance_evals
            res["cand"][t, j] = r.candidates_final
        prev = res["idx"][t].copy()
    print(f"cfg3: {nframes * npos} queries in {time.time() - t0:.1f}s")
    save("golden_cfg3.npz", n_refs=np.array(n), positions=pos, init_prev=init[pos],
         frame_digests=np.array(digests), refs_digest=np.array(W.digest(refs)),
         table_digest=np.array(W.digest(sd.astype(np.float32), si)),
         table_rows=np.arange(0, n, 997), table_rows_dist=sd[::997].astype(np.float32),
         table_rows_idx=si[::997], units=np.array(units), **res)


def gen_cfg4x(npos=256):
    cfg = W.CONFIGS[4]
    refs = W.reference_set(cfg)
    frame = next(W.iter_clip(cfg, 1))
    gw, gh = cfg.grid
    rng = np.random.default_rng(1004)
    pos = np.sort(rng.choice(gw * gh, size=npos, replace=False))
    unit, _ = normalize_rows(extract_patches(frame, cfg.patch).values[pos])
    # refs-only model: exact_nn reads refs and the metric only
    model = ReferenceModel(refs=refs, sorted_dist=np.zeros((0, 0)), sorted_idx=np.zeros((0, 0), np.int32),
                           patch_size=cfg.patch)
    t0 = time.time()
    idx, dist = [], []
    for j in range(npos):
        i, d = exact_nn(unit[j], model)
        idx.append(i)
        dist.append(d)
    print(f"cfg4 exact_nn: {npos} queries over n={model.n} in {time.time() - t0:.1f}s")
    save("golden_cfg4x.npz", positions=pos, refs_digest=np.array(W.digest(refs)),
         frame_digest=np.array(W.digest(frame)), units=unit, idx=np.array(idx, np.int32),
         dist=np.array(dist))


def gen_annf():
    import tempfile

    from riann.engine import AnnField, AnnfWriter

    g = np.load(os.path.join(HERE, "golden_cfg0.npz"))
    idx, dist = g["idx"], g["dist"]
    gh, gw = idx.shape[1:]
    out = {}
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "cfg0.annf")
        with AnnfWriter(path, gw, gh, (8, 8)) as w:
            for t in range(idx.shape[0]):
                w.append(AnnField(width=gw, height=gh, indices=idx[t], distances=dist[t], frame_t=t + 1))
        out["cfg0_bytes"] = np.frombuffer(open(path, "rb").read(), np.uint8)
        path = os.path.join(d, "empty.annf")
        AnnfWriter(path, 7, 5, (8, 8)).close()
        out["empty_bytes"] = np.frombuffer(open(path, "rb").read(), np.uint8)
    save("golden_annf.npz", **out)


def gen_effects():
    from riann.engine import AnnField
    from riann.transforms import (KIND_CHROMA, KIND_FULL, EffectTable, apply_effect,
                                  reconstruct_frame)

    out = {}
    # config 0: the golden field of the last frame
    g = np.load(os.path.join(HERE, "golden_cfg0.npz"))
    frame = g["frames"][-1]
    model = make_model(g["refs"], (8, 8))
    gh, gw = g["idx"].shape[1:]
    field = AnnField(width=gw, height=gh, indices=g["idx"][-1], distances=g["dist"][-1], frame_t=8)
    rng = np.random.default_rng(77)
    full = rng.uniform(0, 1, size=(model.n, 64)).astype(np.float32)
    chroma = rng.uniform(-60, 60, size=(model.n, 128)).astype(np.float32)
    out["c0_recon"] = reconstruct_frame(frame, field, model)
    out["c0_full_pay"] = full
    out["c0_full"] = apply_effect(frame, field, EffectTable(full, KIND_FULL, (8, 8)), model)
    out["c0_chroma_pay"] = chroma
    out["c0_chroma"] = apply_effect(frame, field, EffectTable(chroma, KIND_CHROMA, (8, 8)), model)
    # small model, non-square patch (pw=4, ph=3), random field
    refs, _ = normalize_rows(rng.standard_normal((30, 12)).astype(np.float32))
    sm = make_model(refs, (4, 3))
    fr = rng.uniform(0, 1, size=(9, 11)).astype(np.float32)
    fr[0:3, 0:4] = 0.0  # a zero patch: norm 0
    sidx = rng.integers(0, 30, size=(9 - 3 + 1, 11 - 4 + 1), dtype=np.int32)
    sf = AnnField(width=8, height=7, indices=sidx, distances=np.zeros((7, 8)), frame_t=1)
    sfull = rng.uniform(-2, 2, size=(30, 12)).astype(np.float32)
    schroma = rng.uniform(-300, 300, size=(30, 24)).astype(np.float32)
    out.update(s_refs=refs, s_frame=fr, s_idx=sidx, s_full_pay=sfull, s_chroma_pay=schroma,
               s_recon=reconstruct_frame(fr, sf, sm),
               s_full=apply_effect(fr, sf, EffectTable(sfull, KIND_FULL, (4, 3)), sm),
               s_chroma=apply_effect(fr, sf, EffectTable(schroma, KIND_CHROMA, (4, 3)), sm))
    save("golden_effects.npz", **out)


def gen_rian():
    from riann.model import serialize_model

    rng = np.random.default_rng(91)
    out = {}
    for tag, n, patch, ch in (("a", 40, (4, 4), 1), ("b", 30, (2, 2), 3)):
        dim = patch[0] * patch[1] * ch
        raw = rng.standard_normal((n, dim)).astype(np.float32)
        raw[5] = raw[3]  # an exact duplicate: ties in the sorted rows
        refs, _ = normalize_rows(raw)
        sd, si = compute_sorted_lists(refs)
        m = ReferenceModel(refs=refs, sorted_dist=sd, sorted_idx=si, patch_size=patch, channels=ch)
        out[f"{tag}_refs"] = refs
        out[f"{tag}_bytes"] = np.frombuffer(serialize_model(m), np.uint8)
        out[f"{tag}_patch"] = np.array(patch)
        out[f"{tag}_channels"] = np.array(ch)
    save("golden_rian.npz", **out)


def gen_coherency():
    from riann.evaluation import coherency_stats

    cfg = W.CONFIGS[0]
    frames = W.clip(cfg)[:4]
    model = make_model(W.reference_set(cfg), cfg.patch)
    st = coherency_stats(frames, model)
    save("golden_coherency.npz", shift_samples=st.shift_samples, residual_samples=st.residual_samples,
         shift_hist=st.shift_hist, shift_edges=st.shift_edges, residual_hist=st.residual_hist,
         residual_edges=st.residual_edges, excluded=np.array(st.excluded))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-vga", action="store_true")
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    only = set(a.only.split(",")) if a.only else None
    steps = [("rng", gen_rng), ("arith", gen_arith), ("tables", gen_tables),
             ("queries", gen_queries), ("cfg0", gen_cfg0), ("annf", gen_annf), ("effects", gen_effects),
             ("rian", gen_rian), ("coherency", gen_coherency)]
    for name, fn in steps:
        if only is None or name in only:
            fn()
    if only is not None and "cfg3" in only:
        gen_cfg3()
    if only is not None and "cfg4x" in only:
        gen_cfg4x()
    if not a.skip_vga and (only is None or "vga" in only):
        model, refs = gen_vga(1)
        gen_vga(2, model, refs)


if __name__ == "__main__":
    main()
