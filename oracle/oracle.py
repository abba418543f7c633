"""ctypes front end of the CPU oracle (oracle/riann_oracle.c).

TEST INFRASTRUCTURE ONLY: the checker the CUDA path is compared against.  It
may be imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, never by paper_1508_07953_b200/.

Each wrapper names the reference function (file:line under
/root/reference/pkg/src/riann/) whose behaviour it restates.  The C library is
pinned against golden vectors produced by the live reference
(tests/golden/make_golden.py, tests/test_oracle_golden.py).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libriann_oracle.so")
_lib = None


def build() -> str:
    """Compile the oracle library (make in oracle/)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _L():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = C.CDLL(_LIB_PATH)
        P = C.c_void_p
        i64, i32, u32, u64, dbl = C.c_int64, C.c_int, C.c_uint32, C.c_uint64, C.c_double
        lib.rno_pairwise_sum.argtypes = [P, i64]
        lib.rno_pairwise_sum.restype = dbl
        lib.rno_one_to_many.argtypes = [P, P, P, i64, i32, P]
        lib.rno_normalize_rows.argtypes = [P, i64, i32, P, P]
        lib.rno_frame_units.argtypes = [P, i32, i32, i32, i32, i32, i32, i32, P, P]
        lib.rno_sorted_lists.argtypes = [P, i64, i32, i64, i64, P, P, i32]
        lib.rno_init_field.argtypes = [i32, i32, i64, P, i32, P]
        lib.rno_pcg64_seed.argtypes = [P, P, i32]
        lib.rno_integers.argtypes = [P, u64]
        lib.rno_integers.restype = u64
        lib.rno_pcg64_next64.argtypes = [P]
        lib.rno_pcg64_next64.restype = u64
        lib.rno_query.argtypes = [P, P, i32, i32, dbl, i32, P, i32, P, P, P]
        lib.rno_query_positions.argtypes = [
            P, P, P, P, i64, i32, u64, u32, i32, dbl, i32, i32, P, P, P, P, P, P]
        lib.rno_temporal_change.argtypes = [P, P, i64, i32]
        lib.rno_temporal_change.restype = dbl
        lib.rno_exact_nn_batch.argtypes = [P, i64, i32, P, i64, i32, P, P]
        lib.rno_lazy_tables_create.argtypes = [i64, C.POINTER(P), C.POINTER(P), C.POINTER(P)]
        lib.rno_lazy_tables_free.argtypes = [i64, P, P, P]
        lib.rno_lazy_rows_ready.argtypes = [P, i64]
        lib.rno_lazy_rows_ready.restype = i64
        _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class _Model(C.Structure):
    _fields_ = [
        ("refs", C.c_void_p),
        ("sorted_dist", C.c_void_p),
        ("sorted_idx", C.c_void_p),
        ("n", C.c_int64),
        ("dim", C.c_int),
        ("row_state", C.c_void_p),
    ]


class _Result(C.Structure):
    _fields_ = [
        ("match_index", C.c_int32),
        ("rings", C.c_int32),
        ("match_distance", C.c_double),
        ("evals", C.c_int64),
        ("cand_final", C.c_int64),
        ("first_ring", C.c_int64),
    ]


class _Pcg(C.Structure):
    _fields_ = [
        ("state_hi", C.c_uint64),
        ("state_lo", C.c_uint64),
        ("inc_hi", C.c_uint64),
        ("inc_lo", C.c_uint64),
        ("has_uint32", C.c_int),
        ("uinteger", C.c_uint32),
    ]


# --------------------------------------------------------------------------
def seed_words(seed) -> np.ndarray:
    """numpy's _coerce_to_uint32_array for ints and (nested) int sequences:
    each non-negative int becomes its little-endian 32-bit words ([0] for 0)."""
    if isinstance(seed, (int, np.integer)):
        v = int(seed)
        if v < 0:
            raise ValueError("seed words must be non-negative")
        if v == 0:
            return np.zeros(1, dtype=np.uint32)
        out = []
        while v > 0:
            out.append(v & 0xFFFFFFFF)
            v >>= 32
        return np.array(out, dtype=np.uint32)
    parts = [seed_words(v) for v in seed]
    if not parts:
        return np.zeros(0, dtype=np.uint32)
    return np.concatenate(parts).astype(np.uint32)


class Pcg64:
    """SeedSequence -> PCG64 -> Generator.integers restatement (numpy)."""

    def __init__(self, seed):
        self._g = _Pcg()
        w = seed_words(seed)
        _L().rno_pcg64_seed(C.byref(self._g), _p(w), len(w))

    def integers(self, k: int) -> int:
        return int(_L().rno_integers(C.byref(self._g), int(k)))

    def next64(self) -> int:
        return int(_L().rno_pcg64_next64(C.byref(self._g)))


def pairwise_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(_L().rno_pairwise_sum(_p(a), a.size))


def one_to_many(q, refs) -> np.ndarray:
    """patches.py:151-159."""
    q = np.ascontiguousarray(q, dtype=np.float32)
    refs = np.ascontiguousarray(refs, dtype=np.float32)
    out = np.empty(refs.shape[0], dtype=np.float64)
    _L().rno_one_to_many(_p(q), _p(refs), None, refs.shape[0], refs.shape[1], _p(out))
    return out


def normalize_rows(values):
    """patches.py:100-115 (f32 input rows)."""
    v = np.ascontiguousarray(values, dtype=np.float32)
    unit = np.empty(v.shape, dtype=np.float32)
    norms = np.empty(v.shape[0], dtype=np.float64)
    _L().rno_normalize_rows(_p(v), v.shape[0], v.shape[1], _p(unit), _p(norms))
    return unit, norms


def frame_units(frame, patch_size, y0=0, y1=None):
    """extract_patches + normalize_rows (patches.py:65-115); (H,W,3) frames use
    plane-major patches.  Returns (unit rows, norms) for grid rows [y0, y1)."""
    f = np.ascontiguousarray(frame, dtype=np.float32)
    H, W = f.shape[:2]
    Cn = 1 if f.ndim == 2 else f.shape[2]
    pw, ph = patch_size
    gw, gh = W - pw + 1, H - ph + 1
    y1 = gh if y1 is None else y1
    dim = pw * ph * Cn
    unit = np.empty(((y1 - y0) * gw, dim), dtype=np.float32)
    norms = np.empty((y1 - y0) * gw, dtype=np.float64)
    rc = _L().rno_frame_units(_p(f), H, W, Cn, pw, ph, y0, y1, _p(unit), _p(norms))
    if rc:
        raise ValueError("bad frame/patch geometry")
    return unit, norms


def sorted_lists(refs, rows=None, nthreads=None):
    """model.py:162-189 compute_sorted_lists (f32 values, i32 order)."""
    refs = np.ascontiguousarray(refs, dtype=np.float32)
    n, dim = refs.shape
    r0, r1 = (0, n) if rows is None else rows
    sd = np.empty((r1 - r0, n), dtype=np.float32)
    si = np.empty((r1 - r0, n), dtype=np.int32)
    _L().rno_sorted_lists(_p(refs), n, dim, r0, r1 - r0, _p(sd), _p(si),
                          nthreads or os.cpu_count() or 1)
    return sd, si


def init_field_indices(gw, gh, n, seed=0) -> np.ndarray:
    """engine.py:72-82 indices."""
    w = seed_words(seed)
    out = np.empty((gh, gw), dtype=np.int32)
    if _L().rno_init_field(gw, gh, n, _p(w), len(w), _p(out)):
        raise ValueError("bad init_field arguments")
    return out


@dataclass
class OracleModel:
    refs: np.ndarray          # (n, dim) f32
    sorted_dist: np.ndarray   # (n, n) f32 (the reference's f64 values, exactly)
    sorted_idx: np.ndarray    # (n, n) i32

    def __post_init__(self):
        self.refs = np.ascontiguousarray(self.refs, dtype=np.float32)
        self.sorted_dist = np.ascontiguousarray(self.sorted_dist, dtype=np.float32)
        self.sorted_idx = np.ascontiguousarray(self.sorted_idx, dtype=np.int32)
        self._s = _Model(self.refs.ctypes.data, self.sorted_dist.ctypes.data,
                         self.sorted_idx.ctypes.data, self.refs.shape[0], self.refs.shape[1], None)

    @property
    def n(self):
        return self.refs.shape[0]

    @property
    def dim(self):
        return self.refs.shape[1]

    @classmethod
    def build(cls, refs, nthreads=None):
        sd, si = sorted_lists(refs, nthreads=nthreads)
        return cls(refs, sd, si)

    @classmethod
    def lazy(cls, refs):
        """Tables built row by row on first use (for n where the full
        (n, n) build is impractical on the CPU, e.g. config 3)."""
        return LazyOracleModel(refs)


class LazyOracleModel:
    """OracleModel whose sorted-table rows are computed on demand."""

    def __init__(self, refs):
        self.refs = np.ascontiguousarray(refs, dtype=np.float32)
        n, dim = self.refs.shape
        sd, si, st = C.c_void_p(), C.c_void_p(), C.c_void_p()
        if _L().rno_lazy_tables_create(n, C.byref(sd), C.byref(si), C.byref(st)):
            raise MemoryError("cannot map lazy tables")
        self._ptrs = (sd.value, si.value, st.value)
        self._s = _Model(self.refs.ctypes.data, sd.value, si.value, n, dim, st.value)

    @property
    def n(self):
        return self.refs.shape[0]

    @property
    def dim(self):
        return self.refs.shape[1]

    def rows_ready(self) -> int:
        return int(_L().rno_lazy_rows_ready(self._ptrs[2], self.n))

    def __del__(self):
        try:
            _L().rno_lazy_tables_free(self.n, *self._ptrs)
        except Exception:
            pass


def ring_window(model: OracleModel, anchor: int, d: float, eps: float):
    """search.py:63-80: the [lo, hi) window and its index slice."""
    row = model.sorted_dist[anchor].astype(np.float64)
    lo = int(np.searchsorted(row, d - eps, side="left"))
    hi = int(np.searchsorted(row, d + eps, side="right"))
    return lo, hi, model.sorted_idx[anchor, lo:hi]


def query(model: OracleModel, q, prev: int, L=20, alpha=0.25, max_rings=8, key=0):
    """search.py:83-151 with rng_state=key.  Returns a dict."""
    q = np.ascontiguousarray(q, dtype=np.float32)
    w = seed_words(key)
    res = _Result()
    scanned = np.empty(model.n + 1, dtype=np.int32)
    ns = C.c_int64(0)
    rc = _L().rno_query(C.byref(model._s), _p(q), int(prev), int(L), float(alpha),
                        int(max_rings), _p(w), len(w), C.byref(res), _p(scanned), C.byref(ns))
    if rc:
        raise IndexError("prev index out of range")
    return dict(match_index=res.match_index, match_distance=res.match_distance,
                rings_drawn=res.rings, distance_evals=res.evals,
                candidates_final=res.cand_final, first_ring=res.first_ring,
                scanned=scanned[: ns.value].copy())


def query_positions(model: OracleModel, units, prev, positions, gw, seed, t,
                    L=20, alpha=0.25, max_rings=8, nthreads=None):
    """engine.py:134-148 for the listed grid positions (units/prev aligned
    with positions)."""
    units = np.ascontiguousarray(units, dtype=np.float32)
    prev = np.ascontiguousarray(prev, dtype=np.int32)
    pos = np.ascontiguousarray(positions, dtype=np.int64)
    k = pos.size
    oi = np.empty(k, np.int32)
    od = np.empty(k, np.float64)
    orr = np.empty(k, np.int32)
    oe = np.empty(k, np.int64)
    oc = np.empty(k, np.int64)
    of = np.empty(k, np.int64)
    rc = _L().rno_query_positions(C.byref(model._s), _p(units), _p(prev), _p(pos), k,
                                  int(gw), int(seed), int(t), int(L), float(alpha),
                                  int(max_rings), nthreads or os.cpu_count() or 1,
                                  _p(oi), _p(od), _p(orr), _p(oe), _p(oc), _p(of))
    if rc:
        raise IndexError("prev index out of range")
    return dict(idx=oi, dist=od, rings=orr, evals=oe, cand=oc, first=of)


def temporal_change(unit, prev_unit) -> float:
    """engine.py:163-171."""
    u = np.ascontiguousarray(unit, dtype=np.float32)
    p = np.ascontiguousarray(prev_unit, dtype=np.float32)
    return float(_L().rno_temporal_change(_p(u), _p(p), u.shape[0], u.shape[1]))


def exact_nn_batch(refs, queries, nthreads=None):
    """evaluation.py:24-33 for many queries."""
    refs = np.ascontiguousarray(refs, dtype=np.float32)
    qs = np.ascontiguousarray(queries, dtype=np.float32)
    idx = np.empty(qs.shape[0], np.int32)
    dist = np.empty(qs.shape[0], np.float64)
    _L().rno_exact_nn_batch(_p(refs), refs.shape[0], refs.shape[1], _p(qs), qs.shape[0],
                            nthreads or os.cpu_count() or 1, _p(idx), _p(dist))
    return idx, dist


def process_frame(model: OracleModel, frame, prev_idx, patch_size, t, L=20,
                  alpha=0.25, max_rings=8, seed=0, prev_unit=None, nthreads=None):
    """engine.py:93-187 for a whole frame: returns (idx, dist, stats dict, unit)."""
    unit, _ = frame_units(frame, patch_size)
    H, W = frame.shape[:2]
    gw, gh = W - patch_size[0] + 1, H - patch_size[1] + 1
    Q = gw * gh
    r = query_positions(model, unit, np.asarray(prev_idx).reshape(-1),
                        np.arange(Q, dtype=np.int64), gw, seed, t, L, alpha,
                        max_rings, nthreads)
    tc = temporal_change(unit, prev_unit) if prev_unit is not None else 0.0
    stats = dict(total_rings=int(r["rings"].sum()), total_distance_evals=int(r["evals"].sum()),
                 mean_candidates=float(np.sum(r["cand"])) / Q, temporal_change=tc,
                 queries=Q, sum_first_ring=int(r["first"].sum()))
    return r["idx"].reshape(gh, gw), r["dist"].reshape(gh, gw), stats, unit
