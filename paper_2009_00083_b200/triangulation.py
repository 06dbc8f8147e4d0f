"""Triangulations (reference triangulation.py): implicit Freudenthal grids and
explicit 2-manifold triangle meshes.

Grids: the B200 path never materialises a CSR adjacency; every kernel
evaluates the stencil implicitly.  Explicit meshes are built on
the host like the reference's (CSR adjacency, per-vertex link edges, link
validation, OFF files, canonical test surfaces) and uploaded once as int32
device arrays that the CSR kernels of liblts_sm100.so read.  ``neighbors`` /
``link_adjacency`` are host-side metadata helpers for single vertices.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .errors import MeshError, NonManifoldEdge, NonTriangleFace

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
    """Mesh connectivity (reference Triangulation, triangulation.py:81-125):
    a grid (grid_dims) or an explicit triangle mesh (points / triangles with
    the CSR adjacency indptr / indices, link edges link_ptr / link_a / link_b
    and the boundary mask, host int64 arrays)."""

    dim: int
    n: int
    grid_dims: Optional[tuple] = None
    spacing: float = 1.0
    points: Optional[np.ndarray] = None
    triangles: Optional[np.ndarray] = None
    indptr: Optional[np.ndarray] = field(default=None, repr=False)
    indices: Optional[np.ndarray] = field(default=None, repr=False)
    link_ptr: Optional[np.ndarray] = field(default=None, repr=False)
    link_a: Optional[np.ndarray] = field(default=None, repr=False)
    link_b: Optional[np.ndarray] = field(default=None, repr=False)
    boundary: Optional[np.ndarray] = field(default=None, repr=False)
    _dev: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def is_grid(self) -> bool:
        return self.grid_dims is not None

    def device_arrays(self, device) -> dict:
        """int32 device copies of the explicit mesh's CSR and link arrays
        (uploaded once per device)."""
        import torch
        key = str(device)
        d = self._dev.get(key)
        if d is None:
            d = {name: torch.from_numpy(np.ascontiguousarray(getattr(self, name), np.int32)).to(device)
                 for name in ("indptr", "indices", "link_ptr", "link_a", "link_b")}
            self._dev[key] = d
        return d

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
        if not self.is_grid:
            return self.indices[self.indptr[v]:self.indptr[v + 1]]
        offs, _ = grid_link_tables(self.dim)
        c = np.array(self.grid_coords(v))
        out = []
        for o in offs:
            q = c + o
            if np.all((q >= 0) & (q < np.array(self.grid_dims))):
                out.append(self.grid_index(q))
        return np.array(out, dtype=np.int64)

    def degree(self, v: int) -> int:
        if not self.is_grid:
            return int(self.indptr[v + 1] - self.indptr[v])
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
    """Link edges of v as vertex pairs (triangulation.py:238-264)."""
    if not 0 <= v < mesh.n:
        raise MeshError(f"vertex {v} out of range (n={mesh.n})")
    if not mesh.is_grid:
        lo, hi = int(mesh.link_ptr[v]), int(mesh.link_ptr[v + 1])
        return list(zip(mesh.link_a[lo:hi].tolist(), mesh.link_b[lo:hi].tolist()))
    offs, pairs = grid_link_tables(mesh.dim)
    c = np.array(mesh.grid_coords(v))
    dims = np.array(mesh.grid_dims)
    valid = np.all((c + offs >= 0) & (c + offs < dims), axis=1)
    out = []
    for i, j in pairs:
        if valid[i] and valid[j]:
            out.append((mesh.grid_index(c + offs[i]), mesh.grid_index(c + offs[j])))
    return out


# ---------------------------------------------------------------------------
# explicit 2-manifold triangle meshes (reference triangulation.py:172-250)
# ---------------------------------------------------------------------------

def build_explicit_triangulation(points, triangles) -> Triangulation:
    """Explicit 2-manifold triangle mesh with or without boundary: symmetric
    CSR adjacency (rows ascending), the link edges of every vertex (for each
    incident triangle, its two other vertices), the boundary vertices (on an
    edge of a single triangle), then link validation.  Raises NonTriangleFace,
    NonManifoldEdge or MeshError like the reference."""
    pts = np.asarray(points, dtype=np.float64)
    tris = np.asarray(triangles, dtype=np.int64)
    if tris.size == 0:
        tris = tris.reshape(0, 3)
    if tris.ndim != 2 or tris.shape[1] != 3:
        raise NonTriangleFace("faces must be triangles")
    n = len(pts)
    if tris.size and (tris.min() < 0 or tris.max() >= n):
        raise MeshError("triangle references an unknown vertex")
    # every triangle side as (lo, hi); a side in > 2 triangles is non-manifold
    sides = np.concatenate([tris[:, [0, 1]], tris[:, [1, 2]], tris[:, [0, 2]]])
    lo, hi = sides.min(axis=1), sides.max(axis=1)
    key, count = np.unique(lo * max(n, 1) + hi, return_counts=True)
    if np.any(count > 2):
        bad = int(key[np.argmax(count > 2)])
        raise NonManifoldEdge(f"edge ({bad // n},{bad % n}) lies in {int(count.max())} triangles")
    eu, ev = key // max(n, 1), key % max(n, 1)
    src = np.concatenate([eu, ev])
    dst = np.concatenate([ev, eu])
    order = np.lexsort((dst, src))
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=indptr[1:])
    indices = dst[order].astype(np.int64)
    # link edges, grouped by owner vertex (triangle order within a vertex)
    owner = tris.T.reshape(-1)                                   # a..., b..., c...
    la = np.concatenate([tris[:, 1], tris[:, 0], tris[:, 0]])
    lb = np.concatenate([tris[:, 2], tris[:, 2], tris[:, 1]])
    tri_id = np.tile(np.arange(len(tris)), 3)
    lorder = np.lexsort((tri_id, owner))
    link_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(owner, minlength=n), out=link_ptr[1:])
    boundary = np.zeros(n, dtype=bool)
    boundary[eu[count == 1]] = True
    boundary[ev[count == 1]] = True
    mesh = Triangulation(dim=2, n=n, points=pts, triangles=tris, indptr=indptr, indices=indices,
                         link_ptr=link_ptr, link_a=la[lorder].astype(np.int64),
                         link_b=lb[lorder].astype(np.int64), boundary=boundary)
    _validate_vertex_links(mesh)
    return mesh


def _validate_vertex_links(mesh: Triangulation) -> None:
    """Each vertex link must be one cycle (interior) or one path (boundary)
    (triangulation.py:216-250)."""
    for v in range(mesh.n):
        lo, hi = int(mesh.link_ptr[v]), int(mesh.link_ptr[v + 1])
        if lo == hi:
            if mesh.indptr[v + 1] > mesh.indptr[v]:
                raise MeshError(f"vertex {v} has neighbors but no link edges")
            continue
        a, b = mesh.link_a[lo:hi], mesh.link_b[lo:hi]
        nodes, deg = np.unique(np.concatenate([a, b]), return_counts=True)
        if np.any(deg > 2) or int(np.sum(deg == 1)) not in (0, 2):
            raise MeshError(f"link of vertex {v} is not a single cycle or path")
        # a cycle or path is connected iff it has |nodes| - 1 (path) or |nodes|
        # (cycle) edges and one union-find component
        parent = {int(x): int(x) for x in nodes}

        def find(x):
            while parent[x] != x:
                parent[x] = parent[parent[x]]
                x = parent[x]
            return x

        for x, y in zip(a.tolist(), b.tolist()):
            rx, ry = find(x), find(y)
            if rx != ry:
                parent[ry] = rx
        if len({find(int(x)) for x in nodes}) != 1:
            raise MeshError(f"link of vertex {v} is disconnected")


def load_off(text: str) -> Triangulation:
    """OFF text (triangle faces only) -> explicit triangulation
    (triangulation.py:284-309)."""
    tokens = []
    for line in text.splitlines():
        line = line.split("#", 1)[0].strip()
        if line:
            tokens.extend(line.split())
    if not tokens or tokens[0] != "OFF":
        raise MeshError("missing OFF header")
    try:
        nv, nf = int(tokens[1]), int(tokens[2])
        pts = np.array(tokens[4:4 + 3 * nv], dtype=np.float64).reshape(nv, 3)
        pos = 4 + 3 * nv
        tris = np.empty((nf, 3), dtype=np.int64)
        for f in range(nf):
            k = int(tokens[pos])
            if k != 3:
                raise NonTriangleFace(f"face with {k} vertices; triangles only")
            tris[f] = [int(t) for t in tokens[pos + 1:pos + 4]]
            pos += 4
    except (IndexError, ValueError) as exc:
        raise MeshError(f"malformed OFF data: {exc}") from exc
    return build_explicit_triangulation(pts, tris)


def write_off(mesh: Triangulation) -> str:
    if mesh.is_grid:
        raise MeshError("OFF output requires an explicit mesh")
    out = ["OFF", f"{mesh.n} {len(mesh.triangles)} 0"]
    out += [" ".join(repr(float(x)) for x in p) for p in mesh.points]
    out += ["3 " + " ".join(str(int(v)) for v in t) for t in mesh.triangles]
    return "\n".join(out) + "\n"


def make_octahedron() -> Triangulation:
    """Closed octahedron (triangulation.py:316-320): 6 vertices on the axes."""
    pts = np.array([(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)], float)
    # upper cap around +z, lower cap around -z (same orientation as the reference)
    tris = [(0, 2, 4), (2, 1, 4), (1, 3, 4), (3, 0, 4), (2, 0, 5), (1, 2, 5), (3, 1, 5), (0, 3, 5)]
    return build_explicit_triangulation(pts, np.array(tris, dtype=np.int64))


def make_icosahedron() -> Triangulation:
    """Closed icosahedron (triangulation.py:323-340): the 12 cyclic
    permutations of (0, +-1, +-phi); faces are the vertex triples at mutual
    edge distance 2, listed in lexicographic order."""
    phi = (1 + np.sqrt(5)) / 2
    pts = np.array([p for a, b in ((1, phi), (-1, phi), (1, -phi), (-1, -phi))
                    for p in ((0, a, b), (a, b, 0), (b, 0, a))], dtype=np.float64)
    adj = np.isclose(((pts[:, None] - pts[None]) ** 2).sum(-1), 4.0)
    tris = [(i, j, k) for i in range(12) for j in range(i + 1, 12) if adj[i, j]
            for k in range(j + 1, 12) if adj[i, k] and adj[j, k]]
    return build_explicit_triangulation(pts, np.array(tris, dtype=np.int64))


def make_torus(p: int = 8, q: int = 8) -> Triangulation:
    """Flat torus (triangulation.py:343-361): a p x q vertex grid with
    wraparound, each cell split along its (x, y) -> (x+1, y+1) diagonal."""
    if p < 3 or q < 3:
        raise MeshError("torus grid needs at least 3 vertices per axis")
    y, x = np.mgrid[0:q, 0:p]
    u, v = 2 * np.pi * x.ravel() / p, 2 * np.pi * y.ravel() / q
    r = 2 + np.cos(v)
    pts = np.stack([r * np.cos(u), r * np.sin(u), np.sin(v)], axis=1)
    a = (x % p + p * (y % q)).ravel()
    b = ((x + 1) % p + p * (y % q)).ravel()
    c = (x % p + p * ((y + 1) % q)).ravel()
    d = ((x + 1) % p + p * ((y + 1) % q)).ravel()
    tris = np.stack([np.stack([a, b, d], 1), np.stack([a, d, c], 1)], axis=1).reshape(-1, 3)
    return build_explicit_triangulation(pts, tris.astype(np.int64))
