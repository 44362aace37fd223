"""Support types of the reconstruction boundary: voxel grid, coordinates, result image.

Mirrors the parts of the reference's `nfs/core.py` that the engine API exposes
(`Grid` nfs/core.py:54-99, `grid_coordinates` :102-113, `ReconImage` :182-188).
Linear voxel order is x fastest, then y, then z (l = ix + nx*(iy + ny*iz)).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Grid:
    """Integer extents and field of view in metres (nfs/core.py:54-99)."""

    dims: tuple
    fov_m: tuple

    def __post_init__(self):
        if len(self.dims) != 3 or any(int(n) < 1 for n in self.dims):
            raise ValueError(f"grid extents must be >= 1, got {self.dims}")
        if any(f <= 0 for f in self.fov_m):
            raise ValueError(f"FOV extents must be > 0, got {self.fov_m}")
        object.__setattr__(self, "dims", tuple(int(n) for n in self.dims))
        object.__setattr__(self, "fov_m", tuple(float(f) for f in self.fov_m))

    @property
    def nvox(self) -> int:
        return int(np.prod(self.dims))

    @property
    def ndim(self) -> int:
        return 2 if self.dims[2] == 1 else 3

    @property
    def pitch_m(self):
        return tuple(f / n for f, n in zip(self.fov_m, self.dims))

    def to_array(self, vec):
        return np.asarray(vec).reshape(self.dims, order="F")

    def to_vec(self, arr):
        return np.asarray(arr).reshape(-1, order="F")

    def linear_index(self, ix, iy, iz):
        nx, ny, _ = self.dims
        return np.asarray(ix) + nx * (np.asarray(iy) + ny * np.asarray(iz))

    def multi_index(self, l):
        nx, ny, _ = self.dims
        l = np.asarray(l)
        return l % nx, (l // nx) % ny, l // (nx * ny)


def grid_coordinates(grid: Grid) -> np.ndarray:
    """Centred voxel coordinates (L, 3) in metres: pitch * (m - (n-1)/2) per axis."""
    axes = [(fov / n) * (np.arange(n) - (n - 1) / 2.0) for n, fov in zip(grid.dims, grid.fov_m)]
    mesh = np.meshgrid(*axes, indexing="ij")
    return np.column_stack([grid.to_vec(m) for m in mesh])


@dataclass
class ReconImage:
    """Reconstructed image on the full grid plus CG metadata (nfs/core.py:182-188)."""

    values: np.ndarray
    iterations: int = 0
    final_residual: float = 0.0
