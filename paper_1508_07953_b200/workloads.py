"""Seeded synthetic clips and reference sets with BASELINE.json's config shapes.

The reference publishes no benchmark data for this path,
so every config is synthetic.  Choices (fixed here, documented in DESIGN.md):

* content: uniform noise blurred by ``scipy.ndimage.gaussian_filter`` (sigma
  per config, mode 'reflect', truncate 4.0) on a canvas with a 48 px margin;
* motion: each frame shows the scene canvas translated by the cumulative sum
  of seeded per-frame subpixel shifts (uniform in [-s, s] per axis), sampled
  once with bilinear weights, so motion does not accumulate interpolation
  blur;
* noise: fresh N(0, sigma_n) per frame, then clip to [0, 1], float32;
* scene cuts (config 2): a fresh canvas every ``cut_every`` frames;
* RGB (config 3): three independently blurred planes sharing the shift;
* reference sets: crops at positions drawn without replacement from separate
  frames generated the same way, normalised exactly like the reference's
  ``normalize_rows`` (patches.py:100-115: float64, numpy pairwise sum, cast to
  float32), plane-major for RGB (transforms.py:152-157 precedent).

Parity never depends on these choices: CPU oracle and GPU consume the same
arrays.
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np

MARGIN = 48


@dataclass(frozen=True)
class ClipConfig:
    name: str
    height: int
    width: int
    channels: int
    frames: int
    sigma_blur: float
    max_shift: float
    noise: float
    cut_every: int
    n_refs: int
    ref_frames: int
    clip_seed: int
    ref_seed: int
    patch: tuple = (8, 8)
    ref_config: int = -1  # >= 0: share that config's reference set

    @property
    def grid(self):
        return (self.width - self.patch[0] + 1, self.height - self.patch[1] + 1)

    @property
    def queries(self):
        gw, gh = self.grid
        return gw * gh

    @property
    def dim(self):
        return self.patch[0] * self.patch[1] * self.channels


# BASELINE.json configs[0..4]
CONFIGS = {
    0: ClipConfig("cfg0_tiny_64x64", 64, 64, 1, 8, 1.5, 0.5, 0.01, 0, 1024, 1, 0, 1),
    1: ClipConfig("cfg1_vga_slow", 480, 640, 1, 30, 1.5, 0.5, 0.01, 0, 8192, 4, 10, 11),
    2: ClipConfig("cfg2_vga_high_motion", 480, 640, 1, 30, 1.5, 4.0, 0.03, 10, 8192, 4, 20, 11, ref_config=1),
    3: ClipConfig("cfg3_1080p_rgb", 1080, 1920, 3, 60, 2.0, 1.0, 0.01, 0, 65536, 8, 30, 31),
    4: ClipConfig("cfg4_4k_large_dict", 2160, 3840, 1, 16, 1.5, 1.0, 0.02, 0, 262144, 16, 40, 41),
}


def _canvas(rng, cfg: ClipConfig) -> np.ndarray:
    from scipy.ndimage import gaussian_filter

    h, w = cfg.height + 2 * MARGIN, cfg.width + 2 * MARGIN
    planes = []
    for _ in range(cfg.channels):
        planes.append(gaussian_filter(rng.uniform(size=(h, w)), cfg.sigma_blur,
                                      mode="reflect", truncate=4.0))
    return np.stack(planes, axis=-1)  # (h, w, C) float64


def _sample(canvas: np.ndarray, cfg: ClipConfig, oy: float, ox: float) -> np.ndarray:
    """Bilinear sample of the canvas at a (fractional) offset from the margin."""
    fy, fx = np.floor(oy), np.floor(ox)
    wy, wx = oy - fy, ox - fx
    y0, x0 = MARGIN + int(fy), MARGIN + int(fx)
    H, W = cfg.height, cfg.width
    a = canvas[y0:y0 + H, x0:x0 + W]
    b = canvas[y0:y0 + H, x0 + 1:x0 + 1 + W]
    c = canvas[y0 + 1:y0 + 1 + H, x0:x0 + W]
    d = canvas[y0 + 1:y0 + 1 + H, x0 + 1:x0 + 1 + W]
    return (1 - wy) * ((1 - wx) * a + wx * b) + wy * ((1 - wx) * c + wx * d)


def _observe(rng, content: np.ndarray, cfg: ClipConfig) -> np.ndarray:
    noisy = content + rng.normal(0.0, cfg.noise, size=content.shape)
    out = np.clip(noisy, 0.0, 1.0).astype(np.float32)
    return out[..., 0] if cfg.channels == 1 else np.ascontiguousarray(out)


def iter_clip(cfg: ClipConfig, frames: int | None = None):
    """Yield the clip's frames ((H, W) or (H, W, 3) float32) in order."""
    rng = np.random.default_rng(cfg.clip_seed)
    total = cfg.frames if frames is None else frames
    lim = MARGIN - 2
    canvas, oy, ox = None, 0.0, 0.0
    for t in range(total):
        if canvas is None or (cfg.cut_every and t % cfg.cut_every == 0):
            canvas, oy, ox = _canvas(rng, cfg), 0.0, 0.0
        else:
            dy, dx = rng.uniform(-cfg.max_shift, cfg.max_shift, size=2)
            oy = float(np.clip(oy + dy, -lim, lim))
            ox = float(np.clip(ox + dx, -lim, lim))
        yield _observe(rng, _sample(canvas, cfg, oy, ox), cfg)


def clip(cfg: ClipConfig, frames: int | None = None) -> np.ndarray:
    return np.stack(list(iter_clip(cfg, frames)))


def patch_rows(frame: np.ndarray, patch, ys, xs) -> np.ndarray:
    """Raw (unnormalised) patch rows at top-left (x, y), plane-major."""
    pw, ph = patch
    f = frame if frame.ndim == 3 else frame[..., None]
    Cn = f.shape[2]
    out = np.empty((len(ys), pw * ph * Cn), dtype=np.float32)
    for c in range(Cn):
        plane = f[..., c]
        for dy in range(ph):
            for dx in range(pw):
                out[:, c * pw * ph + dy * pw + dx] = plane[ys + dy, xs + dx]
    return out


def normalize_rows_numpy(values: np.ndarray):
    """The reference's normalize_rows arithmetic (patches.py:100-115), used to
    build reference sets; numpy here IS the reference's arithmetic."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    norms = np.sqrt(np.sum(v * v, axis=1))
    ok = norms >= 1e-12
    unit = np.zeros(v.shape, dtype=np.float32)
    if np.any(ok):
        unit[ok] = (v[ok] / norms[ok, None]).astype(np.float32)
    return unit, np.where(ok, norms, 0.0)


def reference_set(cfg: ClipConfig, n: int | None = None) -> np.ndarray:
    """(n, dim) float32 unit reference rows: crops without replacement from
    ``cfg.ref_frames`` separately generated frames."""
    if cfg.ref_config >= 0:
        return reference_set(CONFIGS[cfg.ref_config], n)
    n = cfg.n_refs if n is None else n
    rng = np.random.default_rng(cfg.ref_seed)
    gw, gh = cfg.grid
    per = [n // cfg.ref_frames + (1 if k < n % cfg.ref_frames else 0) for k in range(cfg.ref_frames)]
    rows = []
    for k in range(cfg.ref_frames):
        canvas = _canvas(rng, cfg)
        frame = _observe(rng, _sample(canvas, cfg, 0.0, 0.0), cfg)
        pos = rng.choice(gw * gh, size=per[k], replace=False)
        rows.append(patch_rows(frame, cfg.patch, pos // gw, pos % gw))
    unit, _ = normalize_rows_numpy(np.concatenate(rows))
    return unit


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()
