"""Row-band partitioning of a frame across GPUs (reference engine.py:150-161).

Positions are independent (engine.py:1-7): a band owns grid rows
[y0, y1), receives frame rows [y0, y1 + ph - 1) (a ph-1 halo) and keeps its
previous indices and unit rows resident on its GPU across frames.  RNG keys
use global (x, y), so the assembled field is identical for any number of
bands (the analogue of the reference's thread-count invariance,
test_engine.py:101-109).  The only exchange is the field gather (idx i32 +
dist f64 per position, plus the per-position temporal-change term so that
FrameStats.temporal_change is summed in numpy's pairwise order over the whole
frame and stays bit-identical to the single-GPU value).

Three entry points:

* ``BandStream`` -- one band on one GPU (its own stream slot on the device's
  context, so several bands or clips may share a GPU);
* ``stream_fields_bands`` / ``stream_fields(..., devices=[...])`` -- one
  process driving several GPUs (a host thread per device; ctypes releases the
  GIL), each band written into a disjoint slice of one host ``AnnField``;
* ``DistributedStream`` -- one process per GPU (torchrun): each rank runs its
  band with device pointers and the band fields are gathered to rank 0 with
  NCCL, device to device.
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _native as N
from .engine import AnnField, FrameStats, _frame_for, _restore_units, _seed_u64, grid_shape, init_field
from .model import resident
from .search import SearchParams


def band_rows(grid_h: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced grid-row band [y0, y1) of ``rank`` out of ``world``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return (rank * grid_h) // world, ((rank + 1) * grid_h) // world


def frame_band(frame: np.ndarray, y0: int, y1: int, ph: int) -> np.ndarray:
    """Frame rows a band needs: [y0, y1 + ph - 1)."""
    return np.ascontiguousarray(frame[y0:y1 + ph - 1])


def _stats(st, q, temporal, tc=None) -> FrameStats:
    return FrameStats(int(st.total_rings), int(st.total_distance_evals),
                      float(int(st.sum_cand_final)) / max(q, 1),
                      (float(st.temporal_change) if tc is None else tc) if temporal else 0.0, q,
                      first_ring_total=int(st.sum_first_ring), cand_total=int(st.sum_cand_final),
                      ring_tests_total=int(st.sum_ring_tests), exact_evals_total=int(st.sum_exact_evals),
                      fallback_queries=int(st.queries_fallback))


class BandStream:
    """stream_fields for one row band on one GPU, in a stream slot of its own.

    step(frame_band) advances the band by one frame and returns
    (indices (y1-y0, gw) int32, distances float64, FrameStats of the band).
    With ``out_tc`` (float64, (y1-y0)*gw) the per-position temporal-change
    terms are returned too, for an exact whole-frame sum.
    """

    def __init__(self, model, grid_w: int, grid_h: int, y0: int, y1: int,
                 params: SearchParams = SearchParams(), device: int | None = None):
        if not 0 <= y0 < y1 <= grid_h:
            raise ValueError(f"bad band [{y0}, {y1}) of {grid_h} rows")
        self.model, self.params = model, params
        self.gw, self.gh, self.y0, self.y1 = grid_w, grid_h, y0, y1
        self.ctx = N.context(device)
        self.slot = self.ctx.new_slot()
        full = init_field(grid_w, grid_h, model.n, seed=params.seed)
        self._last_idx = np.ascontiguousarray(full.indices[y0:y1]).reshape(-1)
        self._last_frame = None
        self._token = None
        self.t = 0

    def close(self):
        if self.slot is not None:
            self.ctx.free_slot(self.slot)
            self.slot = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, band_frame, out_idx=None, out_dist=None, out_tc=None):
        f = _frame_for(self.model, band_frame)
        pw, ph = int(self.model.patch_size[0]), int(self.model.patch_size[1])
        rows = self.y1 - self.y0
        if f.shape[0] != rows + ph - 1 or f.shape[1] != self.gw + pw - 1:
            raise ValueError(f"band frame shape {f.shape[:2]} != {(rows + ph - 1, self.gw + pw - 1)}")
        Cn = 1 if f.ndim == 2 else f.shape[2]
        q = rows * self.gw
        idx = np.empty((rows, self.gw), np.int32) if out_idx is None else out_idx
        dist = np.empty((rows, self.gw), np.float64) if out_dist is None else out_dist
        st = N.FrameStatsC()
        temporal = self.t > 0
        flags = N.F_KEEP_UNITS | (N.F_TEMPORAL if temporal else 0)
        with self.ctx.lock:
            resident(self.ctx, self.model)
            self.ctx.select(self.slot)
            prev = None
            if self._token is None or self._token != self.ctx.token(self.slot):
                # first frame, or a model upload invalidated the slot: host state in
                prev = self._last_idx
                if temporal:
                    _restore_units(self.ctx, self.slot, self.model, self._last_frame)
            N.check(N.lib().riann_process_frame(
                self.ctx.h, N.ptr(f), f.shape[0], f.shape[1], Cn, self.y0, N.ptr(prev),
                _seed_u64(self.params.seed), self.t + 1, int(min(self.params.L, 2**31 - 1)),
                float(self.params.alpha), int(min(self.params.max_rings, 2**31 - 1)), flags,
                N.ptr(idx), N.ptr(dist), C.byref(st)))
            if out_tc is not None and temporal:
                N.check(N.lib().riann_tc_get(self.ctx.h, N.ptr(out_tc), q, 0))
            self._token = self.ctx.advance(self.slot)
        # host copy of the last band field, only read if the slot is invalidated
        self._last_idx, self._last_frame = idx.reshape(-1), f
        self.t += 1
        return idx, dist, _stats(st, q, temporal)


def assemble(parts):
    """Concatenate per-band (idx, dist) in rank order into a full field."""
    return (np.concatenate([p[0] for p in parts], axis=0),
            np.concatenate([p[1] for p in parts], axis=0))


def combine_stats(stats, tc_terms=None) -> FrameStats:
    """Whole-frame FrameStats from band stats.  With the per-position
    temporal-change terms of every band (in row order), temporal_change is
    numpy's pairwise sum over the frame, as engine.py:163-171 computes it;
    otherwise the band partial sums are added."""
    q = sum(s.queries for s in stats)
    cand = sum(s.cand_total for s in stats)
    if tc_terms is not None:
        tc = float(np.sum(np.concatenate(tc_terms))) if q else 0.0
    else:
        tc = float(sum(s.temporal_change for s in stats))
    return FrameStats(sum(s.total_rings for s in stats), sum(s.total_distance_evals for s in stats),
                      float(cand) / q, tc, q,
                      first_ring_total=sum(s.first_ring_total for s in stats), cand_total=cand,
                      ring_tests_total=sum(s.ring_tests_total for s in stats),
                      exact_evals_total=sum(s.exact_evals_total for s in stats),
                      fallback_queries=sum(s.fallback_queries for s in stats))


def grid_of(model, frame_shape):
    return grid_shape(frame_shape, model.patch_size)


def stream_fields_bands(model, frames, params: SearchParams = SearchParams(), devices=(0,),
                        bands: int | None = None):
    """stream_fields (engine.py:205-227) with each frame split into row bands
    over ``devices`` (band k runs on devices[k % len(devices)]).  Yields
    (frame, AnnField, FrameStats), field and FrameStats identical to the
    single-GPU stream.  Bands on different GPUs run concurrently (one host
    thread per GPU); bands sharing a GPU run one after another in their own
    stream slots."""
    devices = [int(d) for d in devices]
    if not devices:
        raise ValueError("need at least one device")
    nb = len(devices) if bands is None else int(bands)
    streams = None
    try:
        for t, frame in enumerate(frames):
            frame = np.asarray(frame)
            gw, gh = grid_shape(frame.shape[:2], model.patch_size)
            ph = int(model.patch_size[1])
            if streams is None:
                if not 1 <= nb <= gh:
                    raise ValueError(f"bands must be in [1, {gh}], got {nb}")
                cuts = [band_rows(gh, nb, k) for k in range(nb)]
                streams = [BandStream(model, gw, gh, y0, y1, params, device=devices[k % len(devices)])
                           for k, (y0, y1) in enumerate(cuts)]
                grid = (gw, gh)
            elif (gw, gh) != grid:
                from .errors import DimensionError

                raise DimensionError(f"frame yields grid {gw}x{gh}, field is {grid[0]}x{grid[1]}")
            idx = np.empty((gh, gw), np.int32)
            dist = np.empty((gh, gw), np.float64)
            tcs = [np.empty((s.y1 - s.y0) * gw, np.float64) for s in streams]
            stats = [None] * len(streams)
            errors = []

            def run(ks):
                try:
                    for k in ks:
                        s = streams[k]
                        _, _, stats[k] = s.step(frame_band(frame, s.y0, s.y1, ph), out_idx=idx[s.y0:s.y1],
                                                out_dist=dist[s.y0:s.y1], out_tc=tcs[k])
                except BaseException as e:  # re-raised on the caller's thread
                    errors.append(e)

            by_dev = {}
            for k, s in enumerate(streams):
                by_dev.setdefault(s.ctx.device, []).append(k)
            if len(by_dev) == 1:
                run(list(range(len(streams))))
            else:
                ths = [threading.Thread(target=run, args=(ks,)) for ks in by_dev.values()]
                for th in ths:
                    th.start()
                for th in ths:
                    th.join()
            if errors:
                raise errors[0]
            fs = combine_stats(stats, tcs if t > 0 else None)
            yield frame, AnnField(width=gw, height=gh, indices=idx, distances=dist, frame_t=t + 1), fs
    finally:
        for s in streams or []:
            s.close()


class DistributedStream:
    """One row band per rank (one process per GPU, torchrun), band fields
    gathered to rank 0 device-to-device with NCCL.

    step(band_frame) runs this rank's band (frame rows [y0, y1 + ph - 1) as a
    host array; uploaded on the library stream) and returns, on rank 0, the
    whole frame's (AnnField, FrameStats) read back to the host, and None on the
    other ranks.  The band's field never leaves the device between frames.
    Gather payload per position: idx i32, dist f64, temporal-change term f64
    (20 B), bands padded to the largest band.
    """

    def __init__(self, model, grid_w: int, grid_h: int, params: SearchParams = SearchParams(),
                 group=None, device: int | None = None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.model, self.params = model, params
        self.gw, self.gh = grid_w, grid_h
        self.y0, self.y1 = band_rows(grid_h, self.world, self.rank)
        self.cuts = [band_rows(grid_h, self.world, r) for r in range(self.world)]
        self.ctx = N.context(device)
        self.slot = self.ctx.new_slot()
        self.dev = torch.device("cuda", self.ctx.device)
        self.stream = torch.cuda.ExternalStream(self.ctx.stream, device=self.dev)
        rows_max = max(b - a for a, b in self.cuts)
        self.m = rows_max * grid_w + (rows_max * grid_w) % 2  # even: the f64 regions stay 8-byte aligned
        q = (self.y1 - self.y0) * grid_w
        self.q = q
        full = init_field(grid_w, grid_h, model.n, seed=params.seed)
        # two send buffers (this frame's idx is the next frame's prev): [idx | dist | tc] as int32 words
        self.send = [torch.zeros(5 * self.m, dtype=torch.int32, device=self.dev) for _ in range(2)]
        self.send[1][:q].copy_(torch.from_numpy(np.ascontiguousarray(full.indices[self.y0:self.y1]).ravel()))
        self.recv = (torch.empty((self.world, 5 * self.m), dtype=torch.int32, device=self.dev)
                     if self.rank == 0 else None)
        self.host = (torch.empty((self.world, 5 * self.m), dtype=torch.int32, pin_memory=True)
                     if self.rank == 0 else None)
        self.counters = torch.zeros(6, dtype=torch.int64, device=self.dev)
        # the buffers were filled on torch's stream; the library stream is non-blocking
        torch.cuda.synchronize(self.dev)
        self.t = 0
        self.cur = 0

    def close(self):
        if self.slot is not None:
            self.ctx.free_slot(self.slot)
            self.slot = None

    def _regions(self, buf):
        m = self.m
        return buf[:m], buf[m:3 * m].view(self.torch.float64), buf[3 * m:5 * m].view(self.torch.float64)

    def step(self, band_frame):
        torch, dist = self.torch, self.dist
        f = _frame_for(self.model, band_frame)
        pw, ph = int(self.model.patch_size[0]), int(self.model.patch_size[1])
        rows = self.y1 - self.y0
        if f.shape[0] != rows + ph - 1 or f.shape[1] != self.gw + pw - 1:
            raise ValueError(f"band frame shape {f.shape[:2]} != {(rows + ph - 1, self.gw + pw - 1)}")
        Cn = 1 if f.ndim == 2 else f.shape[2]
        temporal = self.t > 0
        out, prev = self.send[self.cur], self.send[self.cur ^ 1]
        oi, od, otc = self._regions(out)
        st = N.FrameStatsC()
        flags = N.F_DEVICE_PTRS | N.F_KEEP_UNITS | (N.F_TEMPORAL if temporal else 0)
        with self.ctx.lock, torch.cuda.stream(self.stream):
            resident(self.ctx, self.model)
            self.ctx.select(self.slot)
            if temporal and self._token != self.ctx.token(self.slot):
                _restore_units(self.ctx, self.slot, self.model, self._last_frame)
            src = torch.from_numpy(f)
            fd = src.pin_memory().to(self.dev, non_blocking=True) if not src.is_pinned() else \
                src.to(self.dev, non_blocking=True)
            N.check(N.lib().riann_process_frame(
                self.ctx.h, C.c_void_p(fd.data_ptr()), f.shape[0], f.shape[1], Cn, self.y0,
                C.c_void_p(prev.data_ptr()), _seed_u64(self.params.seed), self.t + 1,
                int(min(self.params.L, 2**31 - 1)), float(self.params.alpha),
                int(min(self.params.max_rings, 2**31 - 1)), flags,
                C.c_void_p(oi.data_ptr()), C.c_void_p(od.data_ptr()), C.byref(st)))
            if temporal:
                N.check(N.lib().riann_tc_get(self.ctx.h, C.c_void_p(otc.data_ptr()), self.q, N.F_DEVICE_PTRS))
            self._token = self.ctx.advance(self.slot)
            self._last_frame = f
            c = torch.tensor([st.total_rings, st.total_distance_evals, st.sum_cand_final, st.sum_first_ring,
                              st.sum_ring_tests, st.sum_exact_evals], dtype=torch.int64)
            self.counters.copy_(c, non_blocking=False)
            dist.gather(out, list(self.recv.unbind(0)) if self.rank == 0 else None, dst=0, group=self.group)
            dist.reduce(self.counters, dst=0, group=self.group)
            if self.rank == 0:
                self.host.copy_(self.recv, non_blocking=True)
                cnt = self.counters.cpu().numpy()
            self.stream.synchronize()
        self.cur ^= 1
        self.t += 1
        if self.rank != 0:
            return None
        h = self.host.numpy()
        idx = np.empty((self.gh, self.gw), np.int32)
        dst = np.empty((self.gh, self.gw), np.float64)
        tcs = []
        for r, (a, b) in enumerate(self.cuts):
            qr = (b - a) * self.gw
            idx[a:b] = h[r, :qr].reshape(b - a, self.gw)
            dst[a:b] = h[r, self.m:3 * self.m].view(np.float64)[:qr].reshape(b - a, self.gw)
            tcs.append(h[r, 3 * self.m:5 * self.m].view(np.float64)[:qr])
        Q = self.gw * self.gh
        fs = FrameStats(int(cnt[0]), int(cnt[1]), float(int(cnt[2])) / Q,
                        float(np.sum(np.concatenate(tcs))) if temporal else 0.0, Q,
                        first_ring_total=int(cnt[3]), cand_total=int(cnt[2]), ring_tests_total=int(cnt[4]),
                        exact_evals_total=int(cnt[5]))
        return AnnField(width=self.gw, height=self.gh, indices=idx, distances=dst, frame_t=self.t), fs
