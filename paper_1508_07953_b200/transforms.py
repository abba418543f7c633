"""Patch replacement, overlap blending and effect transfer on the GPU
(transforms.py:1-265 of the reference).

``apply_effect`` / ``reconstruct_frame`` run ``riann_apply_effect``: payload
rows gathered by match index (rescaled by each query patch's norm for the
reconstruction kind), the uniform average of the overlapping windows in the
reference's float32 addition order, and for the chroma kind the integer
luminance/chroma finish -- bit-identical to the reference.  The integer
colour-space helpers are small host functions (numpy), as in the reference.
``build_effect_table`` needs the clustering builder's tree assignments, which
are out of scope: it raises NotImplementedError.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .engine import AnnField
from .errors import DimensionError
from .model import resident_refs
from .patches import extract_patches

KIND_RECONSTRUCTION = "reconstruction"
KIND_CHROMA = "chroma-pair"
KIND_FULL = "full-patch"
_KINDS = (KIND_RECONSTRUCTION, KIND_CHROMA, KIND_FULL)
_KIND_ID = {KIND_RECONSTRUCTION: 0, KIND_FULL: 1, KIND_CHROMA: 2}


@dataclass(frozen=True)
class EffectTable:
    """Per-reference payload patches aligned with model indices (transforms.py:27-55)."""

    payloads: np.ndarray  # (n, payload_dim) float32
    payload_kind: str
    patch_size: tuple[int, int]

    def __post_init__(self):
        if self.payload_kind not in _KINDS:
            raise ValueError(f"unknown payload kind {self.payload_kind!r}")
        pw, ph = self.patch_size
        per_kind = pw * ph * (2 if self.payload_kind == KIND_CHROMA else 1)
        if self.payloads.ndim != 2 or self.payloads.shape[1] != per_kind:
            raise DimensionError(f"{self.payload_kind} payloads must be (n, {per_kind}), got "
                                 f"{self.payloads.shape}")

    @property
    def n(self) -> int:
        return int(self.payloads.shape[0])


def round_half_away(x: np.ndarray) -> np.ndarray:
    """Round to nearest integer, halves away from zero (transforms.py:58-61)."""
    x = np.asarray(x)
    return (np.sign(x) * np.floor(np.abs(x) + 0.5)).astype(np.int64)


def quantize_u8(x: np.ndarray) -> np.ndarray:
    return np.clip(round_half_away(x), 0, 255).astype(np.uint8)


def rgb_to_ycocg(rgb: np.ndarray) -> np.ndarray:
    """Reversible integer luminance/chroma split (transforms.py:68-88)."""
    rgb = np.asarray(rgb)
    if rgb.ndim != 3 or rgb.shape[2] != 3:
        raise DimensionError(f"expected (h, w, 3) raster, got {rgb.shape}")
    r, g, b = (rgb[..., k].astype(np.int64) for k in range(3))
    co = r - b
    t = b + (co >> 1)
    cg = g - t
    return np.stack([t + (cg >> 1), co, cg], axis=-1)


def ycocg_to_rgb(ycocg: np.ndarray) -> np.ndarray:
    """Exact integer inverse of rgb_to_ycocg (transforms.py:91-101)."""
    ycocg = np.asarray(ycocg)
    if ycocg.ndim != 3 or ycocg.shape[2] != 3:
        raise DimensionError(f"expected (h, w, 3) raster, got {ycocg.shape}")
    y, co, cg = (ycocg[..., k].astype(np.int64) for k in range(3))
    t = y - (cg >> 1)
    g = cg + t
    b = t - (co >> 1)
    return np.stack([b + co, g, b], axis=-1)


def luminance(rgb: np.ndarray) -> np.ndarray:
    return rgb_to_ycocg(rgb)[..., 0]


def reconstruction_table(model) -> EffectTable:
    """Identity payloads: the model's own unit references (transforms.py:109-115)."""
    return EffectTable(payloads=np.array(model.refs, dtype=np.float32), payload_kind=KIND_RECONSTRUCTION,
                       patch_size=tuple(model.patch_size))


def build_effect_table(model, source_frame_raw, source_frame_transformed, tree_assignments):
    raise NotImplementedError("effect tables from keyframe pairs need the clustering model builder "
                              "(model.py:86-160), which is outside this package's scope")


def apply_effect(frame: np.ndarray, field: AnnField, table: EffectTable, model) -> np.ndarray:
    """Replace every patch with its match's payload and blend overlaps
    (transforms.py:192-246), on the GPU.  Grayscale kinds return float32 (H, W);
    the chroma kind returns uint8 (H, W, 3)."""
    frame = np.asarray(frame)
    if frame.ndim != 2:
        raise DimensionError(f"expected a single-plane frame, got shape {frame.shape}")
    if table.n != model.n:
        raise DimensionError(f"table holds {table.n} payloads for a model of {model.n} references")
    if tuple(table.patch_size) != tuple(model.patch_size):
        raise DimensionError(f"table patch size {table.patch_size} does not match model {model.patch_size}")
    pw, ph = int(model.patch_size[0]), int(model.patch_size[1])
    h, w = frame.shape
    if w < pw or h < ph:
        grid = extract_patches(frame, model.patch_size)  # raises the reference's DimensionError
    gw, gh = w - pw + 1, h - ph + 1
    if (gw, gh) != (field.width, field.height):
        raise DimensionError(f"frame yields grid {gw}x{gh}, field is {field.width}x{field.height}")
    kind = _KIND_ID[table.payload_kind]
    f32 = np.ascontiguousarray(frame, dtype=np.float32)
    idx = np.ascontiguousarray(field.indices, dtype=np.int32).reshape(-1)
    if idx.size and (idx.min() < 0 or idx.max() >= model.n):
        raise IndexError("field indices out of range for the model")
    pay = None if (kind == 0 and table.payloads is model.refs) else np.ascontiguousarray(table.payloads, np.float32)
    planes = 2 if kind == 2 else 1
    out = np.empty((planes, h, w), dtype=np.float32)
    rgb = np.empty((h, w, 3), dtype=np.uint8) if kind == 2 else None
    ctx = N.context()
    with ctx.lock:
        resident_refs(ctx, model)
        N.check(N.lib().riann_apply_effect(ctx.h, N.ptr(f32), h, w, N.ptr(idx), N.ptr(pay),
                                           table.n, table.payloads.shape[1], kind,
                                           None if kind == 2 else N.ptr(out), N.ptr(rgb)))
    return rgb if kind == 2 else out[0]


def reconstruct_frame(frame: np.ndarray, field: AnnField, model) -> np.ndarray:
    """Rebuild a frame from its matches alone (transforms.py:249-253)."""
    return apply_effect(frame, field, reconstruction_table(model), model)


def reconstruction_error(gt: np.ndarray, rec: np.ndarray) -> float:
    """Relative error between rasters (transforms.py:256-265)."""
    gt = np.asarray(gt, dtype=np.float64)
    rec = np.asarray(rec, dtype=np.float64)
    if gt.shape != rec.shape:
        raise DimensionError(f"raster shapes differ: {gt.shape} vs {rec.shape}")
    denom = float(np.linalg.norm(gt))
    if denom == 0.0:
        raise ValueError("reconstruction error undefined for all-zero ground truth")
    return float(np.linalg.norm(gt - rec) / denom)
