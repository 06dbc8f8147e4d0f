"""Vertex classification (reference critical.py) on the device stencil kernel."""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import torch

from . import _native as N
from .errors import MeshError
from .order import OrderField
from .triangulation import Triangulation


class Kind(Enum):
    REGULAR = "regular"
    MINIMUM = "minimum"
    MAXIMUM = "maximum"
    SADDLE = "saddle"


@dataclass(frozen=True)
class Criticality:
    kind: Kind
    lower_components: int
    upper_components: int

    @property
    def degenerate(self) -> bool:
        return self.lower_components > 2 or self.upper_components > 2


@dataclass
class CriticalSet:
    minima: torch.Tensor
    maxima: torch.Tensor
    saddles: torch.Tensor
    lower_components: torch.Tensor
    upper_components: torch.Tensor

    def kinds(self) -> torch.Tensor:
        k = torch.zeros(self.lower_components.numel(), dtype=torch.int8,
                        device=self.lower_components.device)
        k[self.minima] = 1
        k[self.maxima] = 2
        k[self.saddles] = 3
        return k


def _kind_from_counts(lower: int, upper: int) -> Kind:
    """critical.py:56-65."""
    if lower == 0 and upper == 0:
        raise MeshError("isolated vertex cannot be classified")
    if lower == 0:
        return Kind.MINIMUM
    if upper == 0:
        return Kind.MAXIMUM
    if lower == 1 and upper == 1:
        return Kind.REGULAR
    return Kind.SADDLE


def _classify(mesh: Triangulation, order: OrderField, flags, lower, upper):
    """lts_classify on grids (classify_grid, _kernels.py:128-156) or
    lts_classify_csr on explicit meshes (classify_explicit, :159-187)."""
    dev = order.rank32.device
    L = N.load()
    with torch.cuda.device(dev):
        if mesh.is_grid:
            N.check(L.lts_classify(N.ptr(order.rank32), mesh.dim, N.dims_arg(mesh.grid_dims),
                                   N.ptr(flags), N.ptr(lower), N.ptr(upper), N.stream_ptr(dev)))
        else:
            d = mesh.device_arrays(dev)
            N.check(L.lts_classify_csr(N.ptr(order.rank32), mesh.n, N.ptr(d["indptr"]), N.ptr(d["indices"]),
                                       N.ptr(d["link_ptr"]), N.ptr(d["link_a"]), N.ptr(d["link_b"]),
                                       N.ptr(flags), N.ptr(lower), N.ptr(upper), N.stream_ptr(dev)))


def classify_flags(mesh: Triangulation, order: OrderField) -> torch.Tensor:
    """uint8 per vertex: bit0 minimum, bit1 maximum (device stencil)."""
    dev = order.rank32.device
    flags = torch.empty(mesh.n, dtype=torch.uint8, device=dev)
    _classify(mesh, order, flags, None, None)
    return flags


def classify_all(mesh: Triangulation, order: OrderField):
    """Lower/upper link component counts for every vertex (critical.py:95-112)."""
    dev = order.rank32.device
    lower = torch.empty(mesh.n, dtype=torch.int16, device=dev)
    upper = torch.empty(mesh.n, dtype=torch.int16, device=dev)
    _classify(mesh, order, None, lower, upper)
    return lower, upper


def classify_vertex(mesh: Triangulation, order: OrderField, v: int) -> Criticality:
    """critical.py:68-92 (single vertex, read from the device classification)."""
    if not 0 <= v < mesh.n:
        raise MeshError(f"vertex {v} out of range (n={mesh.n})")
    lower, upper = classify_all(mesh, order)
    lo, up = int(lower[v]), int(upper[v])
    return Criticality(_kind_from_counts(lo, up), lo, up)


def extract_critical_points(mesh: Triangulation, order: OrderField) -> CriticalSet:
    """critical.py:115-121."""
    lower, upper = classify_all(mesh, order)
    minima = torch.nonzero(lower == 0).flatten()
    maxima = torch.nonzero(upper == 0).flatten()
    saddles = torch.nonzero((lower > 0) & (upper > 0) & ((lower > 1) | (upper > 1))).flatten()
    return CriticalSet(minima=minima, maxima=maxima, saddles=saddles,
                       lower_components=lower, upper_components=upper)


def extrema(mesh: Triangulation, order: OrderField):
    """(minima, maxima) vertex ids, ascending (flag-only stencil)."""
    fl = classify_flags(mesh, order)
    return torch.nonzero(fl & 1).flatten(), torch.nonzero(fl & 2).flatten()
