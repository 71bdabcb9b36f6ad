"""The input type of the hot path: an 8-bit channel-planar image
(reference image_io.py:20-46).  PNM decoding/encoding: image_io.py here."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Image:
    """8-bit image, planes (channels, height, width) uint8; channels 1 or 3."""

    planes: np.ndarray

    def __post_init__(self):
        if self.planes.ndim != 3 or self.planes.dtype != np.uint8:
            raise ValueError("planes must be a (channels, height, width) uint8 array")
        if self.planes.shape[0] not in (1, 3):
            raise ValueError(f"channels must be 1 or 3, got {self.planes.shape[0]}")

    @property
    def channels(self) -> int:
        return self.planes.shape[0]

    @property
    def height(self) -> int:
        return self.planes.shape[1]

    @property
    def width(self) -> int:
        return self.planes.shape[2]
