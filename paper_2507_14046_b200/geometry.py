"""Voxel-order contract and the synthetic-workload geometry.

Only what the DIP step needs: the grid record the drivers validate against
(`pkg/src/d2ip/geometry.py:76-118`), the canonical vectorisation order
q = ((p*R) + r)*C + c (`geometry.py:294-315`, mirrored by `_vectorize_t` at
`pkg/src/d2ip/pipeline.py:252-254`), and the measurement enumeration of
`generate_protocol` (`geometry.py:250-291`) used to order the rows of the
synthetic Jacobians. Reference geometry objects are accepted by duck typing
(``rows``/``cols``/``planes``/``shape``/``voxel_count``/``ref_id``).
"""

from __future__ import annotations

import hashlib
import json
import math
from dataclasses import dataclass

import numpy as np


def _short_hash(payload: str) -> str:
    return hashlib.sha256(payload.encode()).hexdigest()[:12]


@dataclass(frozen=True)
class GridGeometry:
    """Regular R x C x P voxel grid. ``extent`` is the unit cylinder box
    x, y in [-1, 1], z in [0, 1] unless given."""

    rows: int
    cols: int
    planes: int
    extent: tuple = ((-1.0, 1.0), (-1.0, 1.0), (0.0, 1.0))

    def __post_init__(self):
        for name, n in (("rows", self.rows), ("cols", self.cols), ("planes", self.planes)):
            if n < 1:
                raise ValueError(f"{name} must be positive, got {n}")

    @property
    def shape(self) -> tuple[int, int, int]:
        return (self.rows, self.cols, self.planes)

    @property
    def voxel_count(self) -> int:
        return self.rows * self.cols * self.planes

    @property
    def ref_id(self) -> str:
        payload = json.dumps(
            {"R": self.rows, "C": self.cols, "P": self.planes, "extent": [list(e) for e in self.extent]},
            sort_keys=True,
        )
        return _short_hash(payload)

    def axis_centers(self):
        """(y of rows, x of cols, z of planes) voxel-centre coordinates."""
        (x0, x1), (y0, y1), (z0, z1) = self.extent
        ys = y0 + (np.arange(self.rows) + 0.5) * (y1 - y0) / self.rows
        xs = x0 + (np.arange(self.cols) + 0.5) * (x1 - x0) / self.cols
        zs = z0 + (np.arange(self.planes) + 0.5) * (z1 - z0) / self.planes
        return ys, xs, zs


def vectorize(volume: np.ndarray, grid=None) -> np.ndarray:
    """(R, C, P) -> length-Q vector, element q = ((p*R)+r)*C+c
    (`pkg/src/d2ip/geometry.py:294-304`)."""
    vol = np.asarray(volume)
    if vol.ndim != 3:
        raise ValueError(f"expected a 3D volume, got shape {vol.shape}")
    if grid is not None and vol.shape != tuple(grid.shape):
        raise ValueError(f"volume shape {vol.shape} does not match grid {grid.shape}")
    return np.transpose(vol, (2, 0, 1)).reshape(-1)


def devectorize(vector: np.ndarray, shape) -> np.ndarray:
    """Exact inverse of :func:`vectorize` (`geometry.py:307-315`)."""
    if hasattr(shape, "shape") and not isinstance(shape, tuple):
        shape = tuple(shape.shape)
    rows, cols, planes = shape
    vec = np.asarray(vector)
    if vec.ndim != 1 or vec.size != rows * cols * planes:
        raise ValueError(f"vector of size {vec.size} does not match shape {shape}")
    return np.transpose(vec.reshape(planes, rows, cols), (1, 2, 0))


def cylinder_mask(grid: GridGeometry) -> np.ndarray:
    """(R, C, P) bool: voxel centre inside the inscribed cylinder x^2+y^2 <= 1
    (BASELINE.json shared convention (a))."""
    ys, xs, _ = grid.axis_centers()
    inside = (xs[None, :] ** 2 + ys[:, None] ** 2) <= 1.0
    return np.broadcast_to(inside[:, :, None], grid.shape).copy()


def ring_electrodes(n_per_ring: int, heights) -> np.ndarray:
    """(E, 3) electrode xyz on the unit cylinder, layer-major, angle 2*pi*k/n
    from +x counter-clockwise (`geometry.py:185-205`)."""
    pos = []
    for h in heights:
        for k in range(n_per_ring):
            th = 2 * math.pi * k / n_per_ring
            pos.append((math.cos(th), math.sin(th), float(h)))
    return np.asarray(pos, dtype=np.float64)


def adjacent_protocol(n_electrodes: int) -> np.ndarray:
    """(M, 4) quadruples of `generate_protocol(..., "adjacent_in_layer")` on an
    array whose electrodes all share layer 0 (`geometry.py:265-277`):
    drive pairs (k, k+1 mod n); measure pairs touching neither drive electrode,
    in electrode-index order. M = n (n - 3)."""
    ring = list(range(n_electrodes))
    adjacent = [(ring[k], ring[(k + 1) % n_electrodes]) for k in range(n_electrodes)]
    quads = []
    for d_pos, d_neg in adjacent:
        for m_pos, m_neg in adjacent:
            if {m_pos, m_neg} & {d_pos, d_neg}:
                continue
            quads.append((d_pos, d_neg, m_pos, m_neg))
    return np.asarray(quads, dtype=np.int64)
