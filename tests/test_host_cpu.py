"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares; host-side logic (init_field's numpy stream, seed coercion,
parameter validation, error mapping) matches the reference."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO, load_golden, ragged


@pytest.fixture(scope="session")
def built():
    from paper_1508_07953_b200 import build

    return build.build()


def header_symbols():
    src = open(os.path.join(REPO, "include", "riann_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(riann_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol(built):
    lib = ctypes.CDLL(built)
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_covers_header(built):
    from paper_1508_07953_b200 import _native as N

    assert set(header_symbols()) == set(N.SIGNATURES)


def test_library_is_sm100a(built):
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", built], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_init_field_matches_numpy_golden(built):
    import paper_1508_07953_b200 as R

    g = load_golden("golden_rng.npz")
    for i, (gw, gh, n, seed) in enumerate(g["init_args"]):
        f = R.init_field(int(gw), int(gh), int(n), seed=int(seed))
        assert np.array_equal(f.indices, ragged(g["init_flat"], g["init_off"], i).reshape(int(gh), int(gw)))
        assert np.all(np.isinf(f.distances)) and f.frame_t == 0


def test_init_field_reference_examples(built):
    import paper_1508_07953_b200 as R

    f = R.init_field(3, 2, 10, seed=7)
    assert np.array_equal(f.indices, np.random.default_rng(7).integers(0, 10, size=(2, 3), dtype=np.int32))
    f = R.init_field(50, 40, 7, seed=0)
    assert f.indices.min() >= 0 and f.indices.max() < 7
    with pytest.raises(ValueError):
        R.init_field(3, 2, 0)
    with pytest.raises(ValueError):
        R.init_field(0, 2, 5)


def test_seed_words_match_numpy_entropy():
    from paper_1508_07953_b200._native import seed_words

    for e in [0, 7, 2**32, 2**40 + 5, (1, 2, 3, 4), (0, 5), (2**33, 1, 0, 9)]:
        words = [int(w) for w in seed_words(e)]
        assert (np.random.SeedSequence(e).generate_state(8).tolist()
                == np.random.SeedSequence(words).generate_state(8).tolist())
    with pytest.raises(ValueError):
        seed_words(-1)
    with pytest.raises(TypeError):
        seed_words(1.5)


def test_search_params_validation():
    import paper_1508_07953_b200 as R

    p = R.SearchParams()
    assert (p.L, p.alpha, p.max_rings, p.seed) == (20, 0.25, 8, 0)
    for kw in [{"L": 0}, {"alpha": 0.0}, {"alpha": 1.0}, {"alpha": -0.1}, {"max_rings": 0}]:
        with pytest.raises(ValueError):
            R.SearchParams(**kw)


def test_annfield_and_grid_validation():
    import paper_1508_07953_b200 as R

    with pytest.raises(R.DimensionError):
        R.AnnField(width=3, height=2, indices=np.zeros((3, 3), np.int32), distances=np.zeros((2, 3)))
    with pytest.raises(R.DimensionError):
        R.AnnField(width=3, height=2, indices=np.zeros((2, 3), np.int32), distances=np.zeros((3, 2)))
    assert R.grid_shape((32, 48), (8, 8)) == (41, 25)
    assert R.grid_shape((8, 8), (8, 8)) == (1, 1)
    with pytest.raises(R.DimensionError):
        R.grid_shape((4, 4), (8, 8))


def test_error_hierarchy():
    import paper_1508_07953_b200 as R

    for e in (R.DimensionError, R.FormatError, R.ModelCapacityError):
        assert issubclass(e, R.RiannError)


def test_compute_calls_fail_loudly_without_gpu(built):
    """No CPU fallback: on a GPU-less host every compute entry point raises."""
    import torch

    import paper_1508_07953_b200 as R

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(R.RiannError):
        R.normalize_rows(np.ones((2, 4), np.float32))


def test_pairwise_sum_native_matches_numpy(built):
    from paper_1508_07953_b200 import _native as N

    rng = np.random.default_rng(0)
    for n in [0, 1, 7, 8, 100, 129, 1000, 3249, 299409]:
        a = rng.uniform(size=n)
        assert N.lib().riann_pairwise_sum(N.ptr(a), n) == np.sum(a)
