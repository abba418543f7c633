"""The reference model (refs + sorted distance tables), resident on the GPU.

Mirrors ReferenceModel (reference model.py:56-83) and compute_sorted_lists
(:162-189).  Tables live in HBM as float32 distances (the reference's float64
values are float32-quantised, :178-179, so this is lossless) and int32
indices; the GPU builds them bit-identically to compute_sorted_lists (K3).
The clustering builders (:86-160, :192-395) are out of scope;
the RIAN file format (:398-456) is in ``modelio.py``.
"""

from __future__ import annotations

import weakref

import numpy as np

from . import _native as N
from .errors import DimensionError
from .patches import EUCLIDEAN, Metric, get_metric

DEFAULT_REF_CAP = 20_000  # the reference's builder cap (model.py:23); the GPU path is bounded by HBM


class ReferenceModel:
    """Unit references plus sorted distance rows (model.py:56-83).

    Same constructor as the reference (refs, sorted_dist, sorted_idx,
    patch_size, channels, metric_id).  ``sorted_dist`` / ``sorted_idx`` may be
    None: the tables are then built on the GPU (K3) and only copied to the host
    if those attributes are read.
    """

    def __init__(self, refs, sorted_dist=None, sorted_idx=None, patch_size=None, channels: int = 1,
                 metric_id: int = 0):
        self._refs = np.ascontiguousarray(refs, dtype=np.float32)
        if self._refs.ndim != 2:
            raise DimensionError(f"refs must be (n, dim), got shape {self._refs.shape}")
        if (sorted_dist is None) != (sorted_idx is None):
            raise ValueError("sorted_dist and sorted_idx must be given together")
        self._sd = None if sorted_dist is None else np.asarray(sorted_dist)
        self._si = None if sorted_idx is None else np.asarray(sorted_idx)
        if patch_size is None:
            patch_size = (self._refs.shape[1], 1)
        self._patch = (int(patch_size[0]), int(patch_size[1]))
        self._channels = int(channels)
        self._metric_id = int(metric_id)

    @classmethod
    def from_refs(cls, refs, patch_size, channels: int = 1, metric_id: int = 0) -> "ReferenceModel":
        """Model whose sorted tables are built on the GPU (bit-identical to
        compute_sorted_lists)."""
        return cls(refs, None, None, patch_size, channels, metric_id)

    # -- reference attributes ------------------------------------------------
    @property
    def refs(self) -> np.ndarray:
        return self._refs

    @property
    def patch_size(self):
        return self._patch

    @property
    def channels(self) -> int:
        return self._channels

    @property
    def metric_id(self) -> int:
        return self._metric_id

    @property
    def n(self) -> int:
        return int(self._refs.shape[0])

    @property
    def dim(self) -> int:
        return int(self._refs.shape[1])

    @property
    def metric(self) -> Metric:
        return get_metric(self._metric_id)

    @property
    def has_host_tables(self) -> bool:
        return self._sd is not None

    @property
    def sorted_dist(self) -> np.ndarray:
        """(n, n) float64 (values exactly float32), fetched from the GPU on demand."""
        if self._sd is None:
            self._fetch_tables()
        return self._sd

    @property
    def sorted_idx(self) -> np.ndarray:
        if self._si is None:
            self._fetch_tables()
        return self._si

    def table_rows(self, row0: int, rows: int):
        """Rows [row0, row0+rows) of the tables as (float32, int32), from the GPU."""
        ctx = N.context()
        with ctx.lock:
            resident(ctx, self)
            sd = np.empty((rows, self.n), dtype=np.float32)
            si = np.empty((rows, self.n), dtype=np.int32)
            N.check(N.lib().riann_model_get_tables(ctx.h, int(row0), int(rows), N.ptr(sd), N.ptr(si)))
        return sd, si

    def _fetch_tables(self):
        sd, si = self.table_rows(0, self.n)
        self._sd = sd.astype(np.float64)
        self._si = si


def _upload_refs_only(ctx: N.Context, model) -> None:
    refs = np.ascontiguousarray(model.refs, dtype=np.float32)
    n, dim = refs.shape
    pw, ph = int(model.patch_size[0]), int(model.patch_size[1])
    channels = int(getattr(model, "channels", 1))
    if pw * ph * channels != dim:
        pw, ph, channels = dim, 1, 1
    ctx.model_token = None
    ctx.refs_token = None
    N.check(N.lib().riann_model_set_refs(ctx.h, N.ptr(refs), n, dim, pw, ph, channels,
                                         int(getattr(model, "metric_id", 0))))
    ctx.refs_token = weakref.ref(model)
    ctx.model_epoch += 1


def resident_refs(ctx: N.Context, model) -> None:
    """Make ``model``'s reference rows resident on ``ctx`` without the sorted
    tables (enough for frame units and the exact comparator; n x n tables do
    not fit at config 4's n = 262,144)."""
    for tok in (ctx.model_token, ctx.refs_token):
        if tok is not None and tok() is model:
            return
    _upload_refs_only(ctx, model)


def resident(ctx: N.Context, model) -> None:
    """Make ``model`` (this package's or the reference's ReferenceModel) the
    model resident on ``ctx``; no-op when it already is."""
    tok = ctx.model_token
    if tok is not None and tok() is model:
        return
    sharded = getattr(model, "_sharded", None)
    if sharded is not None:  # row-sharded tables (shards.py)
        sharded.attach(ctx, model)
        return
    refs = np.ascontiguousarray(model.refs, dtype=np.float32)
    n, dim = refs.shape
    pw, ph = int(model.patch_size[0]), int(model.patch_size[1])
    channels = int(getattr(model, "channels", 1))
    metric_id = int(getattr(model, "metric_id", 0))
    if pw * ph * channels != dim:
        # reference test models use patch_size=(dim, 1); other layouts are
        # still valid for query-only use, so keep dim and derive a flat patch
        pw, ph, channels = dim, 1, 1
    ctx.model_token = None
    ctx.refs_token = None
    N.check(N.lib().riann_model_set_refs(ctx.h, N.ptr(refs), n, dim, pw, ph, channels, metric_id))
    own = isinstance(model, ReferenceModel)
    if own and model._sd is None:
        N.check(N.lib().riann_model_build_tables(ctx.h))
    else:
        sd = np.asarray(model._sd if own else model.sorted_dist)
        si = np.ascontiguousarray(model._si if own else model.sorted_idx, dtype=np.int32)
        if sd.shape != (n, n) or si.shape != (n, n):
            raise DimensionError(f"sorted tables must be ({n}, {n})")
        sd32 = np.ascontiguousarray(sd, dtype=np.float32)
        if sd.dtype != np.float32 and not np.array_equal(sd32, sd):
            raise ValueError("sorted_dist values must be exactly representable in float32 (model.py:178-179)")
        N.check(N.lib().riann_model_set_tables(ctx.h, N.ptr(sd32), N.ptr(si)))
    ctx.model_token = weakref.ref(model)
    ctx.refs_token = ctx.model_token
    ctx.model_epoch += 1


def compute_sorted_lists(refs, metric: Metric = EUCLIDEAN):
    """Per-reference ascending distance rows with aligned index permutations
    (model.py:162-189), built on the GPU: float64 (float32-exact) distances,
    stable ascending order with the self entry first."""
    if metric is not EUCLIDEAN:
        raise NotImplementedError("only the Euclidean metric has a GPU table builder")
    refs = np.ascontiguousarray(refs, dtype=np.float32)
    if refs.ndim != 2 or refs.shape[0] == 0:
        raise ValueError("cannot build sorted lists over an empty reference set")
    m = ReferenceModel.from_refs(refs, (refs.shape[1], 1))
    sd, si = m.table_rows(0, m.n)
    return sd.astype(np.float64), si
