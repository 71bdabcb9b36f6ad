"""Seeded synthetic inputs for the five BASELINE configurations.

BASELINE.json names no public dataset: every frame is generated from a fixed
seed.  Frame i of config k uses ``default_rng((k, i))`` so any
shard can regenerate its own frames; model weights use ``default_rng((k, 10**6))``.
"Blurred" frames are ``gaussian_filter(uniform[0,1) noise, sigma)`` min-max
rescaled to 0..255 and rounded (``rint``) to uint8.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Config:
    key: str
    index: int          # k in the seed tuple
    frames: int
    channels: int
    height: int
    width: int
    bins: int
    stride: int
    sigma: float | None  # None: i.i.d. uniform noise
    rects: int = 0
    normalization: str = "none"
    scored: bool = True
    pyramid_step: float | None = None
    cell: int = 8
    window_w: int = 64
    window_h: int = 128

    @property
    def pixels_per_frame(self) -> int:
        return self.height * self.width

    @property
    def descriptor_length(self) -> int:
        return (self.window_w // self.cell) * (self.window_h // self.cell) * self.bins


CONFIGS = {
    "c1": Config("c1", 1, 1, 1, 600, 800, 8, 8, None),
    "c2": Config("c2", 2, 512, 1, 480, 640, 8, 4, 2.0, scored=False),
    "c3": Config("c3", 3, 64, 1, 1080, 1920, 9, 8, 1.5, rects=20, normalization="l2",
                 scored=False),
    "c4": Config("c4", 4, 256, 3, 720, 1280, 8, 8, 2.0),
    "c5": Config("c5", 5, 32, 1, 4320, 7680, 18, 8, 3.0, pyramid_step=1.2),
}


def _blur_to_u8(rng, shape, sigma):
    from scipy.ndimage import gaussian_filter

    u = rng.random(shape)
    g = gaussian_filter(u, sigma)
    lo, hi = float(g.min()), float(g.max())
    scaled = (g - lo) * (255.0 / (hi - lo)) if hi > lo else np.zeros_like(g)
    return np.clip(np.rint(scaled), 0, 255).astype(np.uint8)


def make_frame(cfg: Config, i: int) -> np.ndarray:
    """(C, H, W) uint8 frame i of config cfg."""
    rng = np.random.default_rng((cfg.index, i))
    C, H, W = cfg.channels, cfg.height, cfg.width
    if cfg.sigma is None:
        return rng.integers(0, 256, size=(C, H, W), dtype=np.uint8)
    planes = np.stack([_blur_to_u8(rng, (H, W), cfg.sigma) for _ in range(C)])
    if cfg.rects:
        rr = np.random.default_rng((cfg.index, i, 1))
        for _ in range(cfg.rects):
            rw = int(rr.integers(W // 32, W // 4 + 1))
            rh = int(rr.integers(H // 32, H // 4 + 1))
            x0 = int(rr.integers(0, W - rw + 1))
            y0 = int(rr.integers(0, H - rh + 1))
            val = rr.integers(0, 256, size=C, dtype=np.uint8)
            planes[:, y0:y0 + rh, x0:x0 + rw] = val[:, None, None]
    return planes


def make_batch(cfg: Config, first: int = 0, count: int | None = None) -> np.ndarray:
    """(N, C, H, W) uint8 frames first..first+count-1."""
    count = cfg.frames if count is None else count
    out = np.empty((count, cfg.channels, cfg.height, cfg.width), dtype=np.uint8)
    for j in range(count):
        out[j] = make_frame(cfg, first + j)
    return out


def make_weights(cfg: Config) -> tuple[np.ndarray, float]:
    """float32 N(0, 0.01) weights promoted to float64, bias 0 (BASELINE configs)."""
    rng = np.random.default_rng((cfg.index, 10**6))
    w = rng.normal(0.0, 0.01, cfg.descriptor_length).astype(np.float32).astype(np.float64)
    return w, 0.0


def batch_sha256(frames: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(frames).tobytes()).hexdigest()
