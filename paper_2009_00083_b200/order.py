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


def _to_f32_exact(x):
    """float32 view of the caller's values.  The reference keeps float64
    (order.py:31); the device path sorts and realises float32, so float64
    input is accepted only when every value is exactly a float32 (else two
    values that differ below float32 precision would silently become a tie)."""
    if isinstance(x, torch.Tensor):
        if x.dtype == torch.float64:
            x32 = x.to(torch.float32)
            bad = ~((x32.to(torch.float64) == x) | torch.isnan(x))
            if bool(bad.any()):
                raise FieldError("float64 values that float32 cannot represent exactly: the device path "
                                 "orders and realises float32 (round the field to float32 first)")
            return x32
        return x
    a = np.asarray(x)
    if a.dtype == np.float64:
        a32 = a.astype(np.float32)
        with np.errstate(invalid="ignore"):
            bad = ~((a32.astype(np.float64) == a) | np.isnan(a))
        if bad.any():
            raise FieldError("float64 values that float32 cannot represent exactly: the device path "
                             "orders and realises float32 (round the field to float32 first)")
        return a32
    return a


@dataclass
class ScalarField:
    """Real values on the vertices (order.py:23-40); float32 on the device.
    Construction checks the size and finiteness like the reference
    (order.py:32-36, FieldError) -- the finiteness check runs on the device."""

    mesh: Triangulation
    values: torch.Tensor

    def __post_init__(self):
        N.require_cuda()
        v = _as_cuda(_to_f32_exact(self.values), torch.float32)
        if v.numel() != self.mesh.n:
            raise FieldError(f"expected {self.mesh.n} values, got {tuple(v.shape)}")
        with torch.cuda.device(v.device):
            N.check(N.load().lts_check_field(N.ptr(v), v.numel(), N.stream_ptr(v.device)))
        self.values = v

    @classmethod
    def _wrap(cls, mesh: Triangulation, values: torch.Tensor) -> "ScalarField":
        """A field computed on the device (already checked; float32 or float64)."""
        obj = cls.__new__(cls)
        obj.mesh = mesh
        obj.values = values
        return obj

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
    """order.py:62-83 (same default: relative 1e-12 of the value range).
    simplify_field's default realisation is contract D1 (per-pass, step 0:
    every output value is a copy of an input value); realize_numeric and
    simplify_field(options.zeta=...) apply this policy literally."""

    mode: ZetaMode = ZetaMode.RELATIVE_EPSILON
    factor: float = 1e-12

    def step(self, value_range: float) -> float:
        if self.mode is ZetaMode.ULP_DECREMENT:
            return 0.0
        return self.factor * value_range


def compute_order_field(f: ScalarField) -> OrderField:
    """Sort vertices by (value, id) on the device (order.py:86-91)."""
    mesh = f.mesh
    rank = torch.empty(mesh.n, dtype=torch.int32, device=f.values.device)
    inv = torch.empty(mesh.n, dtype=torch.int32, device=f.values.device)
    dev = f.values.device
    if mesh.is_grid:
        ndim, dims, ws = mesh.dim, N.dims_arg(mesh.grid_dims), N.workspace(mesh.grid_dims, dev)
    else:  # an explicit mesh: the order field only sees its n vertices
        ndim, dims, ws = 1, N.dims_arg((mesh.n,)), N.workspace(None, dev, explicit_n=mesh.n)
    with torch.cuda.device(dev):
        N.check(N.load().lts_order_field(N.ptr(f.values), ndim, dims, N.ptr(rank), N.ptr(inv),
                                         N.ptr(ws), ws.numel(), N.stream_ptr(dev)))
    return OrderField(rank32=rank, inverse32=inv)


def order_from_ranks(rank) -> OrderField:
    """order.py:94-99."""
    r = _as_cuda(rank, torch.int32)
    return OrderField(rank32=r.clone())


def realize_numeric(f: ScalarField, order: OrderField, zeta: ZetaPolicy | None = None) -> ScalarField:
    """order.py:102-116: the literal descending realisation sweep
    (_kernels.py:84-99) in float64 on the device (lts_realize_numeric).
    Returns a float64 ScalarField."""
    if order.n != f.mesh.n:
        raise FieldError("order field size does not match the scalar field")
    zeta = zeta or ZetaPolicy()
    dev = f.values.device
    g = f.values.to(torch.float64).clone()
    step = zeta.step(float(g.max() - g.min()) if g.numel() else 0.0)
    inv = order.inverse32 if order.inverse32 is not None else order.inverse.to(torch.int32)
    inv = inv.to(dev).contiguous()
    with torch.cuda.device(dev):
        N.check(N.load().lts_realize_numeric(N.ptr(g), N.ptr(inv), g.numel(), float(step), N.stream_ptr(dev)))
    return ScalarField._wrap(f.mesh, g)
