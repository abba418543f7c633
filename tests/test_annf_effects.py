"""ANNF container (engine.py:228-332) and effect transfer (transforms.py:175-265),
SURVEY §8f rows 1-2: byte-identical files and bit-identical rasters vs fixtures
written by the live reference (tests/golden/make_golden.py)."""

import struct

import numpy as np
import pytest

from conftest import load_golden


@pytest.fixture(scope="module")
def R():
    import paper_1508_07953_b200 as R

    return R


def _cfg0_fields(R):
    g = load_golden("golden_cfg0.npz")
    gh, gw = g["idx"].shape[1:]
    return [R.AnnField(width=gw, height=gh, indices=g["idx"][t], distances=g["dist"][t], frame_t=t + 1)
            for t in range(g["idx"].shape[0])]


# ---- CPU: host writer / reader ---------------------------------------------
def test_writer_host_fields_byte_identical(R, tmp_path):
    fields = _cfg0_fields(R)
    path = tmp_path / "c0.annf"
    with R.AnnfWriter(path, fields[0].width, fields[0].height, (8, 8)) as w:
        for f in fields:
            w.append(f)
    assert path.read_bytes() == load_golden("golden_annf.npz")["cfg0_bytes"].tobytes()


def test_reader_round_trip_and_empty(R, tmp_path):
    path = tmp_path / "c0.annf"
    path.write_bytes(load_golden("golden_annf.npz")["cfg0_bytes"].tobytes())
    s = R.read_annf(path)
    g = load_golden("golden_cfg0.npz")
    assert s.frame_count == g["idx"].shape[0] and s.patch_size == (8, 8)
    assert np.array_equal(s.indices, g["idx"])
    assert np.array_equal(s.distances, g["dist"].astype(np.float32))
    e = tmp_path / "e.annf"
    R.AnnfWriter(e, 7, 5, (8, 8)).close()
    assert e.read_bytes() == load_golden("golden_annf.npz")["empty_bytes"].tobytes()
    s = R.read_annf(e)
    assert s.frame_count == 0 and (s.grid_w, s.grid_h) == (7, 5)


def test_annf_errors(R, tmp_path):
    bad = R.AnnField(width=3, height=2, indices=np.zeros((2, 3), np.int32), distances=np.zeros((2, 3)))
    with R.AnnfWriter(tmp_path / "b.annf", 4, 4, (3, 3)) as w:
        with pytest.raises(R.DimensionError):
            w.append(bad)
    p = tmp_path / "junk.annf"
    p.write_bytes(b"JUNK" + bytes(struct.calcsize("<HIIHHI")))
    with pytest.raises(R.FormatError):
        R.read_annf(p)
    p.write_bytes(b"ANNF\x01\x00")
    with pytest.raises(R.FormatError):
        R.read_annf(p)
    R.AnnfWriter(p, 2, 2, (3, 3)).close()
    raw = bytearray(p.read_bytes())
    raw[4 + struct.calcsize("<HIIHH"):][:4] = struct.pack("<I", 5)
    off = 4 + struct.calcsize("<HIIHH")
    raw[off:off + 4] = struct.pack("<I", 5)
    p.write_bytes(bytes(raw))
    with pytest.raises(R.FormatError):
        R.read_annf(p)
    p.write_bytes(b"ANNF" + struct.pack("<HIIHHI", 9, 1, 1, 3, 3, 0))
    with pytest.raises(R.FormatError):
        R.read_annf(p)
    f2 = R.AnnField(width=2, height=2, indices=np.zeros((2, 2), np.int32), distances=np.zeros((2, 2)))
    w = R.AnnfWriter(tmp_path / "count.annf", 2, 2, (3, 3))
    w.append(f2)
    w.append(f2)
    w.close()
    raw = (tmp_path / "count.annf").read_bytes()
    assert struct.unpack("<I", raw[off:off + 4])[0] == 2


# ---- CPU: host helpers and validation of the effect API ----------------------
def test_ycocg_round_trip_and_rounding():
    from paper_1508_07953_b200 import transforms as T

    rng = np.random.default_rng(5)
    rgb = rng.integers(0, 256, size=(13, 17, 3))
    assert np.array_equal(T.ycocg_to_rgb(T.rgb_to_ycocg(rgb)), rgb)
    assert list(T.round_half_away(np.array([0.5, -0.5, 1.49, -2.5, 0.0]))) == [1, -1, 1, -3, 0]
    assert list(T.quantize_u8(np.array([-3.0, 255.6, 7.5]))) == [0, 255, 8]
    with pytest.raises(T.DimensionError):
        T.rgb_to_ycocg(np.zeros((4, 4)))


def test_effect_table_and_apply_validation(R):
    from paper_1508_07953_b200 import transforms as T

    with pytest.raises(ValueError):
        T.EffectTable(np.zeros((3, 16), np.float32), "bogus", (4, 4))
    with pytest.raises(R.DimensionError):
        T.EffectTable(np.zeros((3, 15), np.float32), T.KIND_FULL, (4, 4))
    with pytest.raises(R.DimensionError):
        T.EffectTable(np.zeros((3, 16), np.float32), T.KIND_CHROMA, (4, 4))
    refs = np.eye(16, dtype=np.float32)[:5]
    model = R.ReferenceModel(refs, np.zeros((5, 5)), np.zeros((5, 5), np.int32), (4, 4))
    field = R.AnnField(width=5, height=5, indices=np.zeros((5, 5), np.int32), distances=np.zeros((5, 5)))
    with pytest.raises(R.DimensionError):
        T.apply_effect(np.zeros((8, 8, 3), np.float32), field, T.reconstruction_table(model), model)
    with pytest.raises(R.DimensionError):  # grid mismatch
        T.apply_effect(np.zeros((9, 9), np.float32), field, T.reconstruction_table(model), model)
    with pytest.raises(R.DimensionError):  # payload count
        T.apply_effect(np.zeros((8, 8), np.float32), field,
                       T.EffectTable(np.zeros((4, 16), np.float32), T.KIND_FULL, (4, 4)), model)
    with pytest.raises(NotImplementedError):
        T.build_effect_table(model, None, None, None)
    with pytest.raises(ValueError):
        T.reconstruction_error(np.zeros((2, 2)), np.zeros((2, 2)))


# ---- GPU: device pack, full pipeline, effects ---------------------------------
def _bits(a):
    return np.ascontiguousarray(a).view(np.uint32)


@pytest.mark.gpu
def test_writer_device_fields_and_stream_to_annf(R, tmp_path):
    from paper_1508_07953_b200 import workloads as W

    cfg = W.CONFIGS[0]
    frames = W.clip(cfg)
    model = R.ReferenceModel.from_refs(W.reference_set(cfg), cfg.patch)
    gw, gh = cfg.grid
    golden = load_golden("golden_annf.npz")["cfg0_bytes"].tobytes()
    a = tmp_path / "dev.annf"
    with R.AnnfWriter(a, gw, gh, cfg.patch) as w:
        for _, fld, _ in R.stream_fields(model, frames):
            w.append(fld)  # resident field: packed on the device
    assert a.read_bytes() == golden
    b = tmp_path / "pipe.annf"
    stats = R.stream_to_annf(model, frames, b)
    assert b.read_bytes() == golden and len(stats) == len(frames)
    g = load_golden("golden_cfg0.npz")
    assert [s.total_rings for s in stats] == [int(x) for x in g["stats_int"][:, 0]]


@pytest.mark.gpu
def test_apply_effect_golden(R):
    from paper_1508_07953_b200 import transforms as T

    g = load_golden("golden_effects.npz")
    c0 = load_golden("golden_cfg0.npz")
    model = R.ReferenceModel.from_refs(c0["refs"], (8, 8))
    gh, gw = c0["idx"].shape[1:]
    field = R.AnnField(width=gw, height=gh, indices=c0["idx"][-1], distances=c0["dist"][-1], frame_t=8)
    frame = c0["frames"][-1]
    out = T.reconstruct_frame(frame, field, model)
    assert out.dtype == np.float32 and np.array_equal(_bits(out), _bits(g["c0_recon"]))
    out = T.apply_effect(frame, field, T.EffectTable(g["c0_full_pay"], T.KIND_FULL, (8, 8)), model)
    assert np.array_equal(_bits(out), _bits(g["c0_full"]))
    out = T.apply_effect(frame, field, T.EffectTable(g["c0_chroma_pay"], T.KIND_CHROMA, (8, 8)), model)
    assert out.dtype == np.uint8 and np.array_equal(out, g["c0_chroma"])
    sm = R.ReferenceModel.from_refs(g["s_refs"], (4, 3))
    sf = R.AnnField(width=8, height=7, indices=g["s_idx"], distances=np.zeros((7, 8)), frame_t=1)
    out = T.reconstruct_frame(g["s_frame"], sf, sm)
    assert np.array_equal(_bits(out), _bits(g["s_recon"]))
    out = T.apply_effect(g["s_frame"], sf, T.EffectTable(g["s_full_pay"], T.KIND_FULL, (4, 3)), sm)
    assert np.array_equal(_bits(out), _bits(g["s_full"]))
    out = T.apply_effect(g["s_frame"], sf, T.EffectTable(g["s_chroma_pay"], T.KIND_CHROMA, (4, 3)), sm)
    assert np.array_equal(out, g["s_chroma"])
    err = T.reconstruction_error(frame, T.reconstruct_frame(frame, field, model))
    assert 0.0 < err < 1.0


# ---- RIAN model container (model.py:398-461) -----------------------------------
def test_rian_host_round_trip(R, tmp_path):
    g = load_golden("golden_rian.npz")
    for tag in ("a", "b"):
        blob = g[f"{tag}_bytes"].tobytes()
        m = R.deserialize_model(blob)
        assert np.array_equal(m.refs, g[f"{tag}_refs"]) and m.channels == int(g[f"{tag}_channels"])
        assert m.sorted_dist.dtype == np.float64 and m.sorted_idx.dtype == np.int32
        assert R.serialize_model(m) == blob
        p = tmp_path / f"{tag}.rian"
        R.save_model(p, m)
        assert p.read_bytes() == blob
        lm = R.load_model(p)
        assert np.array_equal(lm.refs, m.refs) and np.array_equal(np.asarray(lm.sorted_idx), m.sorted_idx)
        assert np.array_equal(np.asarray(lm.sorted_dist, np.float64), m.sorted_dist)
        assert R.model_memory_bytes(m.n, m.dim) == len(blob) - 16


def test_rian_errors(R, tmp_path):
    blob = load_golden("golden_rian.npz")["a_bytes"].tobytes()
    with pytest.raises(R.FormatError):
        R.deserialize_model(blob[:10])
    with pytest.raises(R.FormatError):
        R.deserialize_model(b"JUNK" + blob[4:])
    with pytest.raises(R.FormatError):
        R.deserialize_model(blob[:4] + struct.pack("<H", 7) + blob[6:])
    with pytest.raises(R.FormatError):
        R.deserialize_model(blob[:-4])
    p = tmp_path / "cut.rian"
    p.write_bytes(blob[:-4])
    with pytest.raises(R.FormatError):
        R.load_model(p)


@pytest.mark.gpu
def test_rian_gpu_tables_byte_identical(R, tmp_path):
    """Tables built on the GPU (K3) stream into a file byte-identical to the
    reference's serialize_model; a mapped model uploads without a rebuild."""
    g = load_golden("golden_rian.npz")
    for tag in ("a", "b"):
        m = R.ReferenceModel.from_refs(g[f"{tag}_refs"], tuple(int(v) for v in g[f"{tag}_patch"]),
                                       channels=int(g[f"{tag}_channels"]))
        p = tmp_path / f"{tag}.rian"
        R.save_model(p, m)
        assert p.read_bytes() == g[f"{tag}_bytes"].tobytes()
        lm = R.load_model(p)
        sd, si = lm.table_rows(0, lm.n)
        ref = R.deserialize_model(g[f"{tag}_bytes"].tobytes())
        assert np.array_equal(sd.astype(np.float64), ref.sorted_dist) and np.array_equal(si, ref.sorted_idx)


# ---- exact-field statistics (evaluation.py:86-138) ------------------------------
def test_coherency_validation(R):
    with pytest.raises(ValueError):
        R.coherency_stats([np.zeros((16, 16), np.float32)], None)
    with pytest.raises(ValueError):
        R.coherency_stats([np.zeros((16, 16), np.float32)] * 2, None, bin_width=0)


@pytest.mark.gpu
def test_coherency_stats_golden(R):
    from paper_1508_07953_b200 import workloads as W

    g = load_golden("golden_coherency.npz")
    cfg = W.CONFIGS[0]
    model = R.ReferenceModel.from_refs(W.reference_set(cfg), cfg.patch)
    st = R.coherency_stats(W.clip(cfg)[:4], model)
    assert st.excluded == int(g["excluded"]) and st.samples == g["shift_samples"].size
    assert np.array_equal(st.shift_samples.view(np.uint64), g["shift_samples"].view(np.uint64))
    assert np.array_equal(st.residual_samples.view(np.uint64), g["residual_samples"].view(np.uint64))
    for k in ("shift_hist", "shift_edges", "residual_hist", "residual_edges"):
        assert np.array_equal(getattr(st, k), g[k]), k
