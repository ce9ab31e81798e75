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

    # not a reference counter (kept out of the dataclass fields, so equality
    # and field lists match voxtree's): of ``samples``, how many the exact
    # empty-space skip accounted without computing them
    samples_skipped = 0

    def merged(self, other: "RenderCounters") -> "RenderCounters":
        out = RenderCounters(*(getattr(self, f) + getattr(other, f)
                               for f in self.__dataclass_fields__))
        out.samples_skipped = self.samples_skipped + other.samples_skipped
        return out

    @classmethod
    def from_vt(cls, c) -> "RenderCounters":
        out = cls(int(c.samples), int(c.tf_lookups), int(c.avg_fallbacks),
                  int(c.coarse_fallbacks), int(c.bricks_requested), int(c.bricks_used_marks))
        out.samples_skipped = int(c.samples_skipped)
        return out


def image_to_rgba8(image: np.ndarray) -> np.ndarray:
    """RGBA float [0,1] -> uint8 with half-even rounding (core.py:158-159)."""
    return np.clip(np.round(image * 255.0), 0, 255).astype(np.uint8)
