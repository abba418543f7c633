"""Ring-intersection search (reference search.py) on the GPU.

SearchParams / QueryResult / query_rng_key keep the reference's definitions
(search.py:21-60, :154-157).  ring_candidates and riann_query run the K2
kernel through the C ABI; results (index, float64 distance, rings, evals,
final candidates, scanned set) are bit-identical to the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import DimensionError
from .model import resident

DEFAULT_L = 20
DEFAULT_ALPHA = 0.25
DEFAULT_MAX_RINGS = 8


@dataclass(frozen=True)
class SearchParams:
    """Query-loop knobs (search.py:26-48)."""

    L: int = DEFAULT_L
    alpha: float = DEFAULT_ALPHA
    max_rings: int = DEFAULT_MAX_RINGS
    seed: int = 0

    def __post_init__(self):
        if self.L < 1:
            raise ValueError(f"L must be >= 1, got {self.L}")
        if not 0.0 < self.alpha < 1.0:
            raise ValueError(f"alpha must lie in (0, 1), got {self.alpha}")
        if self.max_rings < 1:
            raise ValueError(f"max_rings must be >= 1, got {self.max_rings}")


@dataclass(frozen=True)
class QueryResult:
    match_index: int
    match_distance: float
    rings_drawn: int
    distance_evals: int
    candidates_final: int
    scanned: np.ndarray = None  # type: ignore[assignment]


def query_rng_key(seed: int, x: int, y: int, t: int) -> tuple[int, int, int, int]:
    """Per-position RNG key (search.py:154-157)."""
    return (seed, x, y, t)


def _clamp_i32(v) -> int:
    # L / max_rings beyond 2^31-1 behave exactly like 2^31-1: neither a
    # candidate set nor a ring count can exceed n <= 2^31-1
    return int(min(int(v), 2**31 - 1))


def _as_f32_rows(a) -> np.ndarray:
    a = np.asarray(a)
    q = np.ascontiguousarray(a, dtype=np.float32)
    if a.dtype != np.float32 and not np.array_equal(q.astype(a.dtype), a):
        # the device keeps query rows in float32 (what the engine feeds,
        # engine.py:120); silently rounding a wider query would change results
        raise NotImplementedError("query values must be exactly representable in float32")
    return q


def ring_candidates(model, anchor: int, d: float, eps: float) -> np.ndarray:
    """References whose distance to ``anchor`` lies in [d - eps, d + eps]
    (search.py:63-80): two binary searches on the anchor's sorted row, done by
    one warp on the GPU; returns the index slice in distance order."""
    n = model.n
    if not 0 <= anchor < n:
        raise IndexError(f"anchor {anchor} out of range for {n} references")
    if d < 0 or eps < 0:
        raise ValueError("ring radius and width must be nonnegative")
    ctx = N.context()
    with ctx.lock:
        resident(ctx, model)
        lo, hi = N.i64(), N.i64()
        out = np.empty(n, dtype=np.int32)
        N.check(N.lib().riann_ring_candidates(ctx.h, int(anchor), float(d), float(eps), lo, hi, N.ptr(out)))
    return out[: hi.value - lo.value].copy()


def riann_query_batch(model, queries, prev_index, params: SearchParams = SearchParams(), keys=None,
                      scanned: bool = False) -> dict:
    """Many independent riann_query calls in one launch (one warp each).

    ``keys``: per-query rng_state seeds (ints or int tuples, numpy
    SeedSequence semantics); None -> params.seed for every query.
    Returns arrays idx, dist, rings, evals, cand, first and, with
    scanned=True, a list of scanned index arrays.
    """
    q = _as_f32_rows(queries)
    if q.ndim != 2 or q.shape[1] != model.dim:
        raise DimensionError(f"queries shape {q.shape} does not match model dim {model.dim}")
    m = q.shape[0]
    prev = np.ascontiguousarray(prev_index, dtype=np.int64).reshape(-1)
    if prev.size != m:
        raise DimensionError("one prev_index per query")
    if m and (prev.min() < 0 or prev.max() >= model.n):
        bad = int(prev[(prev < 0) | (prev >= model.n)][0])
        raise IndexError(f"prev_index {bad} out of range for {model.n} references")
    prev = prev.astype(np.int32)
    if keys is None:
        keys = [params.seed] * m
    words = [N.seed_words(k) for k in keys]
    off = np.zeros(m + 1, dtype=np.int64)
    off[1:] = np.cumsum([len(w) for w in words])
    kw = np.concatenate(words).astype(np.uint32) if m else np.zeros(1, np.uint32)
    L = _clamp_i32(params.L)
    mr = _clamp_i32(params.max_rings)
    out = {k: np.empty(m, dt) for k, dt in [("idx", np.int32), ("dist", np.float64), ("rings", np.int32),
                                            ("evals", np.int64), ("cand", np.int64), ("first", np.int64)]}
    sc = np.empty((m, model.n + 1), dtype=np.int32) if scanned else None
    sl = np.empty(m, dtype=np.int64)
    if m:
        ctx = N.context()
        with ctx.lock:
            resident(ctx, model)
            N.check(N.lib().riann_query_batch(
                ctx.h, N.ptr(q), N.ptr(prev), N.ptr(kw), N.ptr(off), m, L,
                float(params.alpha), mr, N.ptr(out["idx"]), N.ptr(out["dist"]), N.ptr(out["rings"]),
                N.ptr(out["evals"]), N.ptr(out["cand"]), N.ptr(out["first"]), N.ptr(sc), N.ptr(sl)))
    if scanned:
        out["scanned"] = [sc[i, : sl[i]].copy() for i in range(m)]
    return out


def riann_query(model, query, prev_index: int, params: SearchParams = SearchParams(),
                rng_state=None) -> QueryResult:
    """Approximate nearest reference for one unit-norm (or zero) query
    (search.py:83-151), evaluated by the GPU query kernel.

    ``rng_state``: anything numpy's default_rng accepts as a seed (int or
    sequence of ints; the engine passes (seed, x, y, t)); None -> params.seed.
    A live numpy Generator cannot be continued on the device and raises.
    """
    query = np.asarray(query)
    if query.shape != (model.dim,):
        raise DimensionError(f"query shape {query.shape} does not match model dim {model.dim}")
    if not 0 <= prev_index < model.n:
        raise IndexError(f"prev_index {prev_index} out of range for {model.n} references")
    if isinstance(rng_state, np.random.Generator):
        raise TypeError("riann_b200: a numpy Generator rng_state cannot run on the GPU; pass a seed key")
    key = params.seed if rng_state is None else rng_state
    r = riann_query_batch(model, query[None, :], [prev_index], params, keys=[key], scanned=True)
    return QueryResult(
        match_index=int(r["idx"][0]),
        match_distance=float(r["dist"][0]),
        rings_drawn=int(r["rings"][0]),
        distance_evals=int(r["evals"][0]),
        candidates_final=int(r["cand"][0]),
        scanned=r["scanned"][0],
    )
