"""Exact brute-force comparator on the GPU (reference evaluation.py:24-50).

exact_nn / field_exact_oracle scan every reference with the reference's
float64 distance (bit-identical) and keep the first minimum (lowest index on
ties).  Only model.refs is used, so a refs-only model works for n where the
sorted tables would not fit.  The statistics half of the
reference module (coherency / efficiency reports) is out of scope.
"""

from __future__ import annotations

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
