"""Row-sharded sorted tables (config 4: SURVEY §7.5).

The reference holds the whole (n, n) table pair in memory (model.py:162-189).
At config 4 (n = 262,144) the GPU form of that pair plus the index-ordered
distance rows the per-query kernel reads is 768 GiB -- more than one B200's
180 GB, but 96 GiB per GPU over eight.  Here each shard (a contiguous row
range) is built by K3 on its own GPU (``riann_model_build_table_rows``) and
every querying context gets the shards' device pointers
(``riann_model_attach_shards``): rows on another GPU are read with NVLink
peer loads.  The query path over attached shards is the per-query kernel K2,
whose only table reads are the prev's sorted row (first ring) and the
anchors' index-ordered rows (ring membership), so results are identical to
the unsharded model.

Shards are owned by private contexts, so several shards may share one GPU
(that is how the single-GPU tests exercise the shard addressing).
"""

from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _native as N


class ShardedTables:
    """The sorted tables of ``model`` split into ``shards`` row ranges, shard
    s built on ``devices[s % len(devices)]``."""

    def __init__(self, model, devices=(0,), shards: int | None = None):
        devices = [int(d) for d in devices]
        if not devices:
            raise ValueError("need at least one device")
        n = int(model.n)
        S = len(devices) if shards is None else int(shards)
        if not 1 <= S <= min(n, 64):
            raise ValueError(f"shards must be in [1, {min(n, 64)}], got {S}")
        self.n, self.shards = n, S
        self.shard_rows = -(-n // S)
        if (S - 1) * self.shard_rows >= n:
            raise ValueError(f"{S} shards of {self.shard_rows} rows leave an empty shard for n={n}")
        refs = np.ascontiguousarray(model.refs, dtype=np.float32)
        dim = refs.shape[1]
        pw, ph = int(model.patch_size[0]), int(model.patch_size[1])
        ch = int(getattr(model, "channels", 1))
        if pw * ph * ch != dim:
            pw, ph, ch = dim, 1, 1
        self.owners, self.rows = [], []
        sd, si, dm = [], [], []
        for s in range(S):
            r0 = s * self.shard_rows
            rows = min(self.shard_rows, n - r0)
            ctx = N.Context(devices[s % len(devices)])  # private: owns this shard only
            N.check(N.lib().riann_model_set_refs(ctx.h, N.ptr(refs), n, dim, pw, ph, ch,
                                                 int(getattr(model, "metric_id", 0))))
            N.check(N.lib().riann_model_build_table_rows(ctx.h, r0, rows))
            a, b, c = C.c_void_p(), C.c_void_p(), C.c_void_p()
            g0, gr = C.c_int64(), C.c_int64()
            N.check(N.lib().riann_model_table_ptrs(ctx.h, C.byref(a), C.byref(b), C.byref(c), C.byref(g0),
                                                   C.byref(gr)))
            self.owners.append(ctx)
            self.rows.append((r0, rows))
            sd.append(a.value)
            si.append(b.value)
            dm.append(c.value)
        self._ptrs = tuple((C.c_void_p * S)(*v) for v in (sd, si, dm))
        self._attached = []  # contexts holding these shards' pointers

    def table_rows(self, row0: int, rows: int):
        """Rows [row0, row0+rows) of one shard as (float32, int32), from its GPU."""
        for ctx, (r0, nr) in zip(self.owners, self.rows):
            if r0 <= row0 and row0 + rows <= r0 + nr:
                sd = np.empty((rows, self.n), np.float32)
                si = np.empty((rows, self.n), np.int32)
                with ctx.lock:
                    N.check(N.lib().riann_model_get_tables(ctx.h, int(row0), int(rows), N.ptr(sd), N.ptr(si)))
                return sd, si
        raise IndexError(f"rows [{row0}, {row0 + rows}) span shards")

    def attach(self, ctx: N.Context, model) -> None:
        """Make ``model`` resident on ``ctx`` with these shards as its tables."""
        refs = np.ascontiguousarray(model.refs, dtype=np.float32)
        n, dim = refs.shape
        pw, ph = int(model.patch_size[0]), int(model.patch_size[1])
        ch = int(getattr(model, "channels", 1))
        if pw * ph * ch != dim:
            pw, ph, ch = dim, 1, 1
        with ctx.lock:
            ctx.model_token = None
            ctx.refs_token = None
            N.check(N.lib().riann_model_set_refs(ctx.h, N.ptr(refs), n, dim, pw, ph, ch,
                                                 int(getattr(model, "metric_id", 0))))
            N.check(N.lib().riann_model_attach_shards(ctx.h, self.shards, self.shard_rows, *self._ptrs))
            ctx.model_token = weakref.ref(model)
            ctx.refs_token = ctx.model_token
            ctx.model_epoch += 1
            ctx.shards = self  # keep the owners alive while attached
            if ctx not in self._attached:
                self._attached.append(ctx)

    def close(self):
        """Detach from every context still using the shards, then free them."""
        for ctx in self._attached:
            if getattr(ctx, "shards", None) is self and ctx.h:
                with ctx.lock:
                    N.check(N.lib().riann_model_detach_shards(ctx.h))
                    ctx.model_token = None
                    ctx.refs_token = None
                    ctx.model_epoch += 1
                    ctx.shards = None
        self._attached = []
        for ctx in self.owners:
            ctx.close()
        self.owners = []


def shard_model(model, devices=(0,), shards: int | None = None, query_devices=None) -> ShardedTables:
    """Build ``model``'s tables as row shards over ``devices`` and make the
    model resident with them on every device in ``query_devices`` (default:
    ``devices``), so process_frame / stream_fields / riann_query run over the
    shards there."""
    st = ShardedTables(model, devices, shards)
    object.__setattr__(model, "_sharded", st)  # model.resident attaches instead of building tables
    for d in sorted({int(x) for x in (devices if query_devices is None else query_devices)}):
        st.attach(N.context(d), model)
    return st
