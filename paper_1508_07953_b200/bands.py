"""Row-band partitioning of one frame across ranks (one process per GPU).

Positions are independent (engine.py:1-7): a rank owns grid rows
[y0, y1), receives frame rows [y0, y1 + ph - 1) (a ph-1 halo) and keeps its
band's previous indices resident across frames.  RNG keys use global (x, y),
so the assembled field is identical for any number of bands (the analogue of
the reference's thread-count invariance, test_engine.py:101-109).  The only
exchange is the field gather to rank 0 (12 B per position).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .engine import FrameStats, _frame_for, _seed_u64, grid_shape, init_field
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


class BandStream:
    """stream_fields for one row band on this process's GPU.

    step(frame_band) advances the band by one frame and returns
    (indices (y1-y0, gw) int32, distances float64, FrameStats of the band).
    Integer stats sum across bands; temporal_change partial sums are combined
    in float64 (equal to the single-GPU value up to summation order).
    """

    def __init__(self, model, grid_w: int, grid_h: int, y0: int, y1: int,
                 params: SearchParams = SearchParams(), device: int | None = None):
        self.model, self.params = model, params
        self.gw, self.gh, self.y0, self.y1 = grid_w, grid_h, y0, y1
        self.ctx = N.context(device)
        full = init_field(grid_w, grid_h, model.n, seed=params.seed)
        self._prev = np.ascontiguousarray(full.indices[y0:y1]).reshape(-1)
        self.t = 0

    def step(self, band_frame, out_idx=None, out_dist=None):
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
        flags = N.F_KEEP_UNITS | (N.F_TEMPORAL if self.t > 0 else 0)
        with self.ctx.lock:
            resident(self.ctx, self.model)
            prev = self._prev
            N.check(N.lib().riann_process_frame(
                self.ctx.h, N.ptr(f), f.shape[0], f.shape[1], Cn, self.y0, N.ptr(prev),
                _seed_u64(self.params.seed), self.t + 1, int(min(self.params.L, 2**31 - 1)),
                float(self.params.alpha), int(min(self.params.max_rings, 2**31 - 1)), flags,
                N.ptr(idx), N.ptr(dist), C.byref(st)))
            self.ctx.field_gen += 1
        self._prev = None  # the band's field is device-resident from now on
        self.t += 1
        stats = FrameStats(int(st.total_rings), int(st.total_distance_evals),
                           float(int(st.sum_cand_final)) / max(q, 1),
                           float(st.temporal_change) if self.t > 1 else 0.0, q,
                           first_ring_total=int(st.sum_first_ring), cand_total=int(st.sum_cand_final),
                           ring_tests_total=int(st.sum_ring_tests), exact_evals_total=int(st.sum_exact_evals))
        return idx, dist, stats


def assemble(parts):
    """Concatenate per-band (idx, dist) in rank order into a full field."""
    return (np.concatenate([p[0] for p in parts], axis=0),
            np.concatenate([p[1] for p in parts], axis=0))


def combine_stats(stats) -> FrameStats:
    q = sum(s.queries for s in stats)
    cand = sum(s.cand_total for s in stats)
    return FrameStats(sum(s.total_rings for s in stats), sum(s.total_distance_evals for s in stats),
                      float(cand) / q, float(sum(s.temporal_change for s in stats)), q,
                      first_ring_total=sum(s.first_ring_total for s in stats), cand_total=cand)


def grid_of(model, frame_shape):
    return grid_shape(frame_shape, model.patch_size)
