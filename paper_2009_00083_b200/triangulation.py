"""Implicit Freudenthal-triangulated regular grids (reference
triangulation.py:1-169, grid part only; explicit meshes are out of scope).

The B200 path never materialises a CSR adjacency: every kernel evaluates the
stencil implicitly.  ``neighbors`` / ``link_adjacency`` are host-side metadata
helpers for single vertices (tests, debugging), not part of the hot path.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .errors import MeshError

# reference triangulation.py:32-45 (same order: CSR rows follow it, F8)
_OFFSETS_2D = np.array([(1, 0), (0, 1), (1, 1), (-1, 0), (0, -1), (-1, -1)], dtype=np.int64)
_OFFSETS_3D = np.array(
    [(1, 0, 0), (0, 1, 0), (0, 0, 1), (1, 1, 0), (1, 0, 1), (0, 1, 1), (1, 1, 1),
     (-1, 0, 0), (0, -1, 0), (0, 0, -1), (-1, -1, 0), (-1, 0, -1), (0, -1, -1), (-1, -1, -1)],
    dtype=np.int64)


def _binary(d) -> bool:
    return bool(np.all((d == 0) | (d == 1)))


def _face_triple(a, b) -> bool:
    """triangulation.py:52-66: {0, a, b} accepted when some ordering x<=y<=z has
    consecutive differences in {0,1}^d (z-x unchecked: over-connected, F3)."""
    z = np.zeros_like(a)
    for x, y, w in ((z, a, b), (z, b, a), (a, z, b), (b, z, a), (a, b, z), (b, a, z)):
        if _binary(y - x) and _binary(w - y):
            return True
    return False


def _pairs(offsets):
    out = [(i, j) for i in range(len(offsets)) for j in range(i + 1, len(offsets))
           if _face_triple(offsets[i], offsets[j])]
    return np.array(out, dtype=np.int64)


_LINK_PAIRS_2D = _pairs(_OFFSETS_2D)
_LINK_PAIRS_3D = _pairs(_OFFSETS_3D)


def grid_link_tables(dim: int):
    """Stencil offsets and link-edge index pairs (triangulation.py:273-277)."""
    if dim == 2:
        return _OFFSETS_2D, _LINK_PAIRS_2D
    if dim == 3:
        return _OFFSETS_3D, _LINK_PAIRS_3D
    raise MeshError(f"grid must be 2D or 3D, got {dim}")


@dataclass
class Triangulation:
    """Grid connectivity (reference Triangulation, triangulation.py:81-125)."""

    dim: int
    n: int
    grid_dims: Optional[tuple] = None
    spacing: float = 1.0

    @property
    def is_grid(self) -> bool:
        return self.grid_dims is not None

    @property
    def shape(self) -> tuple:
        """numpy/torch array shape (slowest axis first)."""
        return tuple(self.grid_dims[::-1])

    def grid_coords(self, v: int) -> tuple:
        nx = self.grid_dims[0]
        if self.dim == 2:
            return (v % nx, v // nx)
        ny = self.grid_dims[1]
        return (v % nx, (v // nx) % ny, v // (nx * ny))

    def grid_index(self, coords) -> int:
        nx = self.grid_dims[0]
        if self.dim == 2:
            return int(coords[0] + nx * coords[1])
        return int(coords[0] + nx * (coords[1] + self.grid_dims[1] * coords[2]))

    def neighbors(self, v: int) -> np.ndarray:
        if not 0 <= v < self.n:
            raise MeshError(f"vertex {v} out of range (n={self.n})")
        offs, _ = grid_link_tables(self.dim)
        c = np.array(self.grid_coords(v))
        out = []
        for o in offs:
            q = c + o
            if np.all((q >= 0) & (q < np.array(self.grid_dims))):
                out.append(self.grid_index(q))
        return np.array(out, dtype=np.int64)

    def degree(self, v: int) -> int:
        return int(self.neighbors(v).size)


MAX_GRID_VERTICES = 1 << 27  # liblts_sm100.so's limit (512^3), same check as lts_sm100.cu setup()


def build_grid_triangulation(dims, spacing: float = 1.0) -> Triangulation:
    """reference triangulation.py:128-169 (without the CSR arrays)."""
    dims = tuple(int(d) for d in dims)
    if len(dims) not in (2, 3):
        raise MeshError(f"grid must be 2D or 3D, got {len(dims)} axes")
    if any(d < 2 for d in dims):
        raise MeshError(f"every grid axis needs at least 2 vertices, got {dims}")
    n = int(np.prod(dims))
    if n > MAX_GRID_VERTICES:
        raise MeshError(f"grid too large for the device path (n={n} > 2^27): the classification "
                        "kernel packs rank << 4 | stencil index into 32 bits")
    return Triangulation(dim=len(dims), n=n, grid_dims=dims, spacing=spacing)


def link_adjacency(mesh: Triangulation, v: int) -> list:
    """Link edges of v as vertex pairs (triangulation.py:238-264, grid part)."""
    if not 0 <= v < mesh.n:
        raise MeshError(f"vertex {v} out of range (n={mesh.n})")
    offs, pairs = grid_link_tables(mesh.dim)
    c = np.array(mesh.grid_coords(v))
    dims = np.array(mesh.grid_dims)
    valid = np.all((c + offs >= 0) & (c + offs < dims), axis=1)
    out = []
    for i, j in pairs:
        if valid[i] and valid[j]:
            out.append((mesh.grid_index(c + offs[i]), mesh.grid_index(c + offs[j])))
    return out
