"""ANNF field-stream container (engine.py:228-332; format SPEC.md:284).

    "ANNF" | <HIIHHI version, grid_w, grid_h, patch_w, patch_h, frame_count
    then per frame: grid_h*grid_w little-endian u32 indices, then as many
    little-endian f32 distances (the float64 field distances rounded to
    nearest).  frame_count is back-patched when the writer closes.

Files are byte-identical to the reference writer's (tests/golden).  A field
that is still resident on the GPU (the latest output of process_frame /
stream_fields on this context) is packed on the device (riann_field_pack:
8 bytes per position leave the GPU); other fields are converted on the host.
``stream_to_annf`` runs a whole clip on the GPU and writes only the packed
payloads (the `riann run` pipeline, cli.py:178).
"""

from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .engine import (AnnField, FrameStats, _device_prev, _frame_for, _restore_units, _seed_u64, grid_shape,
                     init_field)
from .errors import DimensionError, FormatError
from .model import resident
from .search import SearchParams

ANNF_MAGIC = b"ANNF"
ANNF_VERSION = 1
_ANNF_HEADER = "<HIIHHI"  # version, grid_w, grid_h, patch_w, patch_h, frame_count


class AnnfWriter:
    """Streaming writer (engine.py:228-279): header with a zero frame count
    goes out immediately and the count is patched on close."""

    def __init__(self, path, grid_w: int, grid_h: int, patch_size: tuple[int, int]):
        self.grid_w = int(grid_w)
        self.grid_h = int(grid_h)
        self.patch_size = (int(patch_size[0]), int(patch_size[1]))
        self.frame_count = 0
        self._f = open(path, "wb")
        self._f.write(ANNF_MAGIC)
        self._f.write(struct.pack(_ANNF_HEADER, ANNF_VERSION, self.grid_w, self.grid_h,
                                  self.patch_size[0], self.patch_size[1], 0))

    def _check(self, width, height):
        if (width, height) != (self.grid_w, self.grid_h):
            raise DimensionError(f"field grid {width}x{height} does not match stream "
                                 f"{self.grid_w}x{self.grid_h}")

    def append(self, field: AnnField) -> None:
        self._check(field.width, field.height)
        dev = getattr(field, "_dev", None)
        ctx = N.context() if dev is not None else None
        packed = False
        if ctx is not None:
            with ctx.lock:
                if _device_prev(ctx, dev[0][1], field):
                    payload = np.empty(2 * self.grid_w * self.grid_h, dtype=np.uint32)
                    ctx.select(dev[0][1])
                    N.check(N.lib().riann_field_pack(ctx.h, N.ptr(payload), self.grid_w * self.grid_h))
                    self._f.write(payload.tobytes())
                    packed = True
        if not packed:
            self._f.write(np.ascontiguousarray(field.indices, dtype="<u4").tobytes())
            self._f.write(np.ascontiguousarray(field.distances, dtype="<f4").tobytes())
        self.frame_count += 1

    def append_payload(self, payload: np.ndarray) -> None:
        """One frame's packed payload (u32 indices then f32 distance bits)."""
        if payload.size != 2 * self.grid_w * self.grid_h:
            raise DimensionError(f"payload of {payload.size} words for a {self.grid_w}x{self.grid_h} grid")
        self._f.write(np.ascontiguousarray(payload, dtype="<u4").tobytes())
        self.frame_count += 1

    def close(self) -> None:
        if self._f.closed:
            return
        self._f.seek(4 + struct.calcsize("<HIIHH"))
        self._f.write(struct.pack("<I", self.frame_count))
        self._f.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


@dataclass(frozen=True)
class AnnfStream:
    grid_w: int
    grid_h: int
    patch_size: tuple[int, int]
    indices: np.ndarray  # (frames, grid_h, grid_w) int32
    distances: np.ndarray  # (frames, grid_h, grid_w) float32

    @property
    def frame_count(self) -> int:
        return int(self.indices.shape[0])


def read_annf(path) -> AnnfStream:
    """Load a container written by AnnfWriter (engine.py:292-332), with the
    same validation and FormatError messages."""
    with open(path, "rb") as f:
        data = f.read()
    header_len = 4 + struct.calcsize(_ANNF_HEADER)
    if len(data) < header_len:
        raise FormatError("field stream truncated inside the header")
    if data[:4] != ANNF_MAGIC:
        raise FormatError(f"bad magic {data[:4]!r}, expected {ANNF_MAGIC!r}")
    version, gw, gh, pw, ph, frames = struct.unpack(_ANNF_HEADER, data[4:header_len])
    if version != ANNF_VERSION:
        raise FormatError(f"unsupported field stream version {version}")
    per_frame = 8 * gw * gh
    expected = header_len + frames * per_frame
    if len(data) != expected:
        raise FormatError(f"field stream length {len(data)} does not match header "
                          f"({frames} frames of {gw}x{gh} require {expected} bytes)")
    cells = gw * gh
    body = np.frombuffer(data, dtype="<u4", offset=header_len).reshape(frames, 2, cells)
    idx = body[:, 0].astype(np.int32).reshape(frames, gh, gw)
    dist = body[:, 1].copy().view("<f4").astype(np.float32).reshape(frames, gh, gw)
    return AnnfStream(grid_w=gw, grid_h=gh, patch_size=(pw, ph), indices=idx, distances=dist)


def stream_to_annf(model, frames, path, params: SearchParams = SearchParams()):
    """Run a clip on the GPU and write its ANNF stream: the field stays on the
    device, each frame leaves it as one packed payload.  Same fields as
    stream_fields + AnnfWriter (engine.py:205-227, 257-267).  Returns the
    per-frame FrameStats."""
    ctx = N.context()
    slot = ctx.new_slot()
    stats = []
    writer = None
    last_token = last_idx = last_frame = None
    try:
        t = 0
        for frame in frames:
            f = _frame_for(model, frame)
            pw, ph = int(model.patch_size[0]), int(model.patch_size[1])
            H, W = f.shape[0], f.shape[1]
            Cn = 1 if f.ndim == 2 else f.shape[2]
            gw, gh = grid_shape(f.shape[:2], model.patch_size)
            if writer is None:
                writer = AnnfWriter(path, gw, gh, model.patch_size)
                prev = np.ascontiguousarray(init_field(gw, gh, model.n, seed=params.seed).indices).reshape(-1)
            elif (gw, gh) != (writer.grid_w, writer.grid_h):
                raise DimensionError(f"frame yields grid {gw}x{gh}, stream is {writer.grid_w}x{writer.grid_h}")
            if pw * ph * Cn != model.dim:
                raise DimensionError(f"patch dim {pw * ph * Cn} does not match model dim {model.dim}")
            Q = gw * gh
            st = N.FrameStatsC()
            flags = N.F_KEEP_UNITS | (N.F_TEMPORAL if t > 0 else 0)
            payload = np.empty(2 * Q, dtype=np.uint32)
            with ctx.lock:
                resident(ctx, model)
                ctx.select(slot)
                if prev is None and last_token != ctx.token(slot):
                    # another model was uploaded meanwhile: rebuild this stream's state
                    prev = np.ascontiguousarray(last_idx).reshape(-1)
                    _restore_units(ctx, slot, model, last_frame)
                N.check(N.lib().riann_process_frame(
                    ctx.h, N.ptr(f), H, W, Cn, 0, N.ptr(prev), _seed_u64(params.seed), t + 1,
                    int(min(params.L, 2**31 - 1)), float(params.alpha), int(min(params.max_rings, 2**31 - 1)),
                    flags, None, None, C.byref(st)))
                last_token = ctx.advance(slot)
                N.check(N.lib().riann_field_pack(ctx.h, N.ptr(payload), Q))
            prev = None
            last_idx, last_frame = payload[:Q].view(np.int32), f
            writer.append_payload(payload)
            stats.append(FrameStats(int(st.total_rings), int(st.total_distance_evals),
                                    float(int(st.sum_cand_final)) / Q,
                                    float(st.temporal_change) if t > 0 else 0.0, Q,
                                    first_ring_total=int(st.sum_first_ring), cand_total=int(st.sum_cand_final),
                                    ring_tests_total=int(st.sum_ring_tests),
                                    exact_evals_total=int(st.sum_exact_evals),
                                    fallback_queries=int(st.queries_fallback)))
            t += 1
    finally:
        ctx.free_slot(slot)
        if writer is not None:
            writer.close()
    return stats
