"""Order fields (reference order.py): the injective re-indexing of vertices by
(value, id).  ``compute_order_field`` runs the onesweep radix sort of
liblts_sm100.so on the device; ranks stay int32 on the device and are exposed
as int64 like the reference's arrays.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from enum import Enum

import numpy as np
import torch

from . import _native as N
from .errors import FieldError
from .triangulation import Triangulation


def _as_cuda(x, dtype) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        t = x
    else:
        t = torch.from_numpy(np.ascontiguousarray(x))
    if t.device.type != "cuda":
        N.require_cuda()
        t = t.pin_memory().to("cuda", non_blocking=True) if t.dtype == dtype else t.to("cuda")
    return t.to(dtype).contiguous().reshape(-1)


@dataclass
class ScalarField:
    """Real values on the vertices (order.py:23-40); float32 on the device."""

    mesh: Triangulation
    values: torch.Tensor

    def __post_init__(self):
        N.require_cuda()
        v = _as_cuda(self.values, torch.float32)
        if v.numel() != self.mesh.n:
            raise FieldError(f"expected {self.mesh.n} values, got {tuple(v.shape)}")
        self.values = v

    @property
    def value_range(self) -> float:
        return float(self.values.max() - self.values.min())


@dataclass(eq=False)
class OrderField:
    """Bijection vertices -> {0..n-1} (order.py:43-59).  ``rank32``/``inverse32``
    are the device arrays; ``rank``/``inverse`` are int64 views."""

    rank32: torch.Tensor
    inverse32: torch.Tensor = None
    _r64: torch.Tensor = field(default=None, repr=False)
    _i64: torch.Tensor = field(default=None, repr=False)

    @property
    def n(self) -> int:
        return int(self.rank32.numel())

    @property
    def rank(self) -> torch.Tensor:
        if self._r64 is None:
            self._r64 = self.rank32.to(torch.int64)
        return self._r64

    @property
    def inverse(self) -> torch.Tensor:
        if self.inverse32 is None:
            inv = torch.empty_like(self.rank32)
            inv[self.rank32.long()] = torch.arange(self.n, dtype=torch.int32, device=self.rank32.device)
            self.inverse32 = inv
        if self._i64 is None:
            self._i64 = self.inverse32.to(torch.int64)
        return self._i64

    def reversed(self) -> "OrderField":
        rev = (self.n - 1) - self.rank32
        inv = None if self.inverse32 is None else torch.flip(self.inverse32, dims=[0]).contiguous()
        return OrderField(rank32=rev.contiguous(), inverse32=inv)

    def __eq__(self, other) -> bool:
        return isinstance(other, OrderField) and torch.equal(self.rank32, other.rank32)


class ZetaMode(Enum):
    RELATIVE_EPSILON = "relative-epsilon"
    ULP_DECREMENT = "ulp-decrement"


@dataclass
class ZetaPolicy:
    """order.py:62-83.  The device path realises with ULP_DECREMENT / step 0
    (contract D1: every output value is a copy of an input value)."""

    mode: ZetaMode = ZetaMode.ULP_DECREMENT
    factor: float = 1e-12

    def step(self, value_range: float) -> float:
        if self.mode is ZetaMode.ULP_DECREMENT:
            return 0.0
        return self.factor * value_range


def compute_order_field(f: ScalarField) -> OrderField:
    """Sort vertices by (value, id) on the device (order.py:86-91)."""
    mesh = f.mesh
    dims = N.dims_arg(mesh.grid_dims)
    rank = torch.empty(mesh.n, dtype=torch.int32, device=f.values.device)
    inv = torch.empty(mesh.n, dtype=torch.int32, device=f.values.device)
    ws = N.workspace(mesh.grid_dims, f.values.device)
    N.check(N.load().lts_order_field(N.ptr(f.values), mesh.dim, dims, N.ptr(rank), N.ptr(inv),
                                     N.ptr(ws), ws.numel(), N.stream_ptr()))
    return OrderField(rank32=rank, inverse32=inv)


def order_from_ranks(rank) -> OrderField:
    """order.py:94-99."""
    r = _as_cuda(rank, torch.int32)
    return OrderField(rank32=r.clone())
