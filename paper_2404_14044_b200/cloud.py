"""Point cloud container (reference ``cloud.py:18-53``).

Positions are float64 (n, 3) C-contiguous; colours optional float64 (n, 3) in
[0, 1].  PLY/CSV file IO is out of scope for the hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

__all__ = ["PointCloud"]


@dataclass(frozen=True)
class PointCloud:
    positions: np.ndarray
    colors: np.ndarray | None = None

    def __post_init__(self):
        xyz = np.array(self.positions, dtype=np.float64)
        if xyz.size == 0:
            xyz = xyz.reshape(0, 3)
        if xyz.ndim != 2 or xyz.shape[1] != 3:
            raise ValueError("positions must have shape (n, 3)")
        if not np.isfinite(xyz).all():
            raise ValueError("positions must be finite")
        xyz = np.ascontiguousarray(xyz)
        xyz.flags.writeable = False
        object.__setattr__(self, "positions", xyz)
        if self.colors is None:
            return
        rgb = np.array(self.colors, dtype=np.float64)
        if rgb.size == 0:
            rgb = rgb.reshape(0, 3)
        if rgb.shape != (xyz.shape[0], 3):
            raise ValueError("colors must have shape (n, 3)")
        if (not np.isfinite(rgb).all() or rgb.min(initial=0.0) < 0.0
                or rgb.max(initial=0.0) > 1.0):
            raise ValueError("colors must be finite and within [0, 1]")
        rgb = np.ascontiguousarray(rgb)
        rgb.flags.writeable = False
        object.__setattr__(self, "colors", rgb)

    @property
    def count(self) -> int:
        return self.positions.shape[0]

    def __len__(self) -> int:
        return self.count

    @property
    def has_colors(self) -> bool:
        return self.colors is not None
