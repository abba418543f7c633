"""Exact brute-force comparator on the GPU (reference evaluation.py:24-50).

exact_nn / field_exact_oracle scan every reference with the reference's
float64 distance (bit-identical) and keep the first minimum (lowest index on
ties).  Only model.refs is used, so a refs-only model works for n where the
sorted tables would not fit.  The statistics half of the
reference module (coherency / efficiency reports) is out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .engine import AnnField, _frame_for
from .errors import DimensionError
from .model import resident_refs


def _upload_refs(ctx, model):
    resident_refs(ctx, model)


def exact_nn(query, model) -> tuple[int, float]:
    """Exact nearest reference by full scan; ties take the lowest index."""
    query = np.asarray(query)
    if query.shape != (model.dim,):
        raise DimensionError(f"query shape {query.shape} does not match model dim {model.dim}")
    q = np.ascontiguousarray(query, dtype=np.float32)[None, :]
    idx = np.empty(1, np.int32)
    dist = np.empty(1, np.float64)
    ctx = N.context()
    with ctx.lock:
        _upload_refs(ctx, model)
        N.check(N.lib().riann_exact_nn_batch(ctx.h, N.ptr(q), 1, N.ptr(idx), N.ptr(dist)))
    return int(idx[0]), float(dist[0])


def exact_nn_batch(queries, model):
    """exact_nn for many query rows: (idx int32, dist float64)."""
    q = np.ascontiguousarray(queries, dtype=np.float32)
    if q.ndim != 2 or q.shape[1] != model.dim:
        raise DimensionError(f"queries shape {q.shape} does not match model dim {model.dim}")
    m = q.shape[0]
    idx = np.empty(m, np.int32)
    dist = np.empty(m, np.float64)
    if m:
        ctx = N.context()
        with ctx.lock:
            _upload_refs(ctx, model)
            N.check(N.lib().riann_exact_nn_batch(ctx.h, N.ptr(q), m, N.ptr(idx), N.ptr(dist)))
    return idx, dist


def field_exact_oracle(frame, model) -> AnnField:
    """Ground-truth field: exact_nn at every grid position (evaluation.py:36-50)."""
    f = _frame_for(model, frame)
    pw, ph = model.patch_size
    H, W = f.shape[0], f.shape[1]
    Cn = 1 if f.ndim == 2 else f.shape[2]
    if W < pw or H < ph:
        raise DimensionError(f"frame {W}x{H} smaller than patch {pw}x{ph}")
    gw, gh = W - pw + 1, H - ph + 1
    idx = np.empty((gh, gw), np.int32)
    dist = np.empty((gh, gw), np.float64)
    ctx = N.context()
    with ctx.lock:
        _upload_refs(ctx, model)
        N.check(N.lib().riann_exact_field(ctx.h, N.ptr(f), H, W, Cn, N.ptr(idx), N.ptr(dist)))
    return AnnField(width=gw, height=gh, indices=idx, distances=dist)


# ---------------------------------------------------------------------------
# Exact-field statistics (evaluation.py:53-138) on K4.
DEFAULT_BIN_WIDTH = 0.1


@dataclass(frozen=True)
class CoherencyStats:
    """How far exact matches move between consecutive frames (evaluation.py:53-76)."""

    shift_hist: np.ndarray
    shift_edges: np.ndarray
    residual_hist: np.ndarray
    residual_edges: np.ndarray
    excluded: int
    shift_samples: np.ndarray
    residual_samples: np.ndarray

    @property
    def samples(self) -> int:
        return int(self.shift_samples.size)


def _histogram(samples: np.ndarray, bin_width: float):
    top = float(samples.max()) if samples.size else bin_width
    edges = np.arange(0.0, top + bin_width, bin_width)
    if len(edges) < 2:
        edges = np.array([0.0, bin_width])
    return np.histogram(samples, bins=edges)


def coherency_stats(video, model, bin_width: float = DEFAULT_BIN_WIDTH) -> CoherencyStats:
    """Match drift across a clip from exact fields (evaluation.py:86-138): the
    exact fields come from K4 (tensor-core screen + FP64 re-check), and for every
    position whose exact match changes, shift = dist(r_prev, r_cur) and
    residual = |shift - dist(r_prev, q)| are float64 numpy-order distances from
    riann_pair_dist.  Sample order, exclusions and histograms as the reference."""
    from .engine import frame_units

    frames = [np.asarray(f) for f in video]
    if len(frames) < 2:
        raise ValueError(f"coherency needs at least 2 frames, got {len(frames)}")
    if bin_width <= 0:
        raise ValueError(f"bin_width must be positive, got {bin_width}")
    shifts, residuals = [], []
    excluded = 0
    prev_idx = field_exact_oracle(frames[0], model).indices.reshape(-1)
    for t in range(1, len(frames)):
        cur_idx = field_exact_oracle(frames[t], model).indices.reshape(-1)
        moved = np.flatnonzero(prev_idx != cur_idx)
        excluded += int(prev_idx.size - moved.size)
        if moved.size:
            unit = frame_units(frames[t], model)
            ia = np.ascontiguousarray(prev_idx[moved], dtype=np.int32)
            ib = np.ascontiguousarray(cur_idx[moved], dtype=np.int32)
            u = np.ascontiguousarray(unit[moved], dtype=np.float32)
            sh = np.empty(moved.size, np.float64)
            pr = np.empty(moved.size, np.float64)
            ctx = N.context()
            with ctx.lock:
                _upload_refs(ctx, model)
                N.check(N.lib().riann_pair_dist(ctx.h, N.ptr(ia), N.ptr(ib), N.ptr(u), moved.size, N.ptr(sh),
                                                N.ptr(pr)))
            shifts.append(sh)
            residuals.append(np.abs(sh - pr))
        prev_idx = cur_idx
    shift_samples = np.concatenate(shifts) if shifts else np.zeros(0, np.float64)
    residual_samples = np.concatenate(residuals) if residuals else np.zeros(0, np.float64)
    shift_hist, shift_edges = _histogram(shift_samples, bin_width)
    residual_hist, residual_edges = _histogram(residual_samples, bin_width)
    return CoherencyStats(shift_hist=shift_hist, shift_edges=shift_edges, residual_hist=residual_hist,
                          residual_edges=residual_edges, excluded=excluded, shift_samples=shift_samples,
                          residual_samples=residual_samples)
