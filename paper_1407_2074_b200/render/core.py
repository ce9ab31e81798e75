"""Render counters and image helpers (render/core.py:20-31, 158-159).  The
march/composite loop itself is the device kernel (csrc/render.cu)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class RenderCounters:
    samples: int = 0
    tf_lookups: int = 0
    avg_fallbacks: int = 0
    coarse_fallbacks: int = 0
    bricks_requested: int = 0
    bricks_used_marks: int = 0

    def merged(self, other: "RenderCounters") -> "RenderCounters":
        return RenderCounters(*(getattr(self, f) + getattr(other, f)
                                for f in self.__dataclass_fields__))

    @classmethod
    def from_vt(cls, c) -> "RenderCounters":
        return cls(int(c.samples), int(c.tf_lookups), int(c.avg_fallbacks),
                   int(c.coarse_fallbacks), int(c.bricks_requested), int(c.bricks_used_marks))


def image_to_rgba8(image: np.ndarray) -> np.ndarray:
    """RGBA float [0,1] -> uint8 with half-even rounding (core.py:158-159)."""
    return np.clip(np.round(image * 255.0), 0, 255).astype(np.uint8)
