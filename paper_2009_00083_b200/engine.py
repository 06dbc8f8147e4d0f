"""LTS engine surface (module lts-engine) on the B200 path.

The reference package ships no engine; this module keeps SPEC's
names and argument meaning.  Every operation is one call into
liblts_sm100.so (device-resident; no CPU fallback):

  simplify_field(mesh, f, constraints, options) -> (g, G, report)
  remove_extrema(mesh, F, discardMaxima, discardMinima, options) -> (G, report)
  discover_regions / remove_pass: one maxima (or minima) pass with its regions
  verify_constraints(mesh, G, constraints) -> VerifyReport
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import _native as N
from .critical import classify_flags, extrema
from .errors import ConstraintNotExtremum, FieldError, MeshError
from .order import OrderField, ScalarField, ZetaPolicy, ZetaMode, compute_order_field, realize_numeric, _as_cuda
from .triangulation import Triangulation


@dataclass
class ConstraintSet:
    """Preserve sets (SPEC ConstraintSet).  Empty sets get the global extremum."""

    preserveMinima: object = ()
    preserveMaxima: object = ()


@dataclass
class SimplifyOptions:
    """SPEC SimplifyOptions.

    zeta: None (default) realises g by contract D1: per pass, every
    flattened vertex takes its region saddle's value, so g only holds copies of
    input values.  A ZetaPolicy instead applies SPEC's literal
    ``g = realize_numeric(f, G, zeta)`` (float64 output, order.py:102-116).
    threadCount: the reference's CPU thread count; the device path's result
    does not depend on it, values < 0 are rejected."""

    zeta: Optional[ZetaPolicy] = None
    restoreInteriorExtrema: bool = True
    maxIterations: int = 100
    threadCount: int = 0
    collectTiming: bool = False

    def __post_init__(self):
        if int(self.maxIterations) < 1:
            raise ValueError("maxIterations must be >= 1 (SPEC.md:304)")
        if int(self.threadCount) < 0:
            raise ValueError("threadCount must be >= 0")
        if self.zeta is not None and not isinstance(self.zeta, ZetaPolicy):
            raise TypeError("zeta must be a ZetaPolicy or None")


@dataclass
class PassReport:
    kind: str
    seeds: int
    regions: int
    claimed: int
    largest: int
    n_iter_max: int
    capped: int
    shared_saddles: int
    maxima_edges: int = 0
    boruvka_rounds: int = 0
    big_regions: int = 0


@dataclass
class SimplifyReport:
    """SPEC SimplifyReport."""

    ok: bool
    outerIterations: int
    restored: int
    passes: list
    regionCount: int
    largestRegion: int
    maxNI: int
    capped: int
    regionNI: list = field(default_factory=list)  # per pass: int32 tensor of each region's N_I
    linf: Optional[float] = None
    phase_ms: dict = field(default_factory=dict)
    extra_max: int = 0
    lost_max: int = 0
    extra_min: int = 0
    lost_min: int = 0


@dataclass
class VerifyReport:
    ok: bool
    extra_maxima: torch.Tensor
    lost_maxima: torch.Tensor
    extra_minima: torch.Tensor
    lost_minima: torch.Tensor


def _workspace(mesh: Triangulation, dev):
    if mesh.is_grid:
        return N.workspace(mesh.grid_dims, dev)
    return N.workspace(None, dev, explicit_n=mesh.n)


def _ids(x, device) -> torch.Tensor:
    if x is None:
        return torch.empty(0, dtype=torch.int64, device=device)
    if isinstance(x, torch.Tensor):
        t = x.to(device=device, dtype=torch.int64)
    else:
        t = torch.as_tensor(np.asarray(list(x) if isinstance(x, (set, frozenset)) else x,
                                       dtype=np.int64), device=device)
    return t.reshape(-1).contiguous()


def _report(rep: "N.lts_report_t", ni: Optional[torch.Tensor] = None) -> SimplifyReport:
    passes = []
    for i in range(rep.n_passes):
        p = rep.passes[i]
        passes.append(PassReport("max" if p.kind == 0 else "min", p.seeds, p.regions, p.claimed,
                                 p.largest, p.n_iter_max, p.capped, p.shared_saddles,
                                 p.maxima_edges, p.boruvka_rounds, p.big_regions))
    ph = {name: float(rep.phase_ms[i]) for i, name in enumerate(N.PHASES)}
    return SimplifyReport(
        ok=bool(rep.ok), outerIterations=int(rep.outer_iterations), restored=int(rep.restored),
        passes=passes, regionCount=sum(p.regions for p in passes),
        largestRegion=max([p.largest for p in passes] + [0]),
        maxNI=max([p.n_iter_max for p in passes] + [0]), capped=sum(p.capped for p in passes),
        regionNI=_split_ni(ni, passes, int(rep.region_ni_count)),
        phase_ms=ph, extra_max=int(rep.extra_max), lost_max=int(rep.lost_max),
        extra_min=int(rep.extra_min), lost_min=int(rep.lost_min))


def _split_ni(ni, passes, count):
    if ni is None:
        return []
    out, off = [], 0
    for p in passes:
        out.append(ni[off:off + p.regions] if off + p.regions <= ni.numel() else None)
        off += p.regions
    return out


def simplify_raw(mesh: Triangulation, values: Optional[torch.Tensor], pres_max: torch.Tensor,
                 pres_min: torch.Tensor, order: Optional[torch.Tensor] = None,
                 options: Optional[SimplifyOptions] = None, g_out=None, G_out=None, ni_out=None):
    """Device-tensor entry point: values float32 (cuda; None = orders only,
    then `order` is required), pres_* int64 (cuda).  ni_out (optional int32
    device tensor) receives the per-region N_I of every pass.
    Returns (g float32 or None, G int32 ranks, lts_report_t).  No host copies."""
    options = options or SimplifyOptions()
    dev = values.device if values is not None else order.device
    g = None
    if values is not None:
        g = g_out if g_out is not None else torch.empty(mesh.n, dtype=torch.float32, device=dev)
    G = G_out if G_out is not None else torch.empty(mesh.n, dtype=torch.int32, device=dev)
    ws = _workspace(mesh, dev)
    opt = N.lts_options_t()
    opt.max_iterations = int(options.maxIterations)
    opt.restore_interior_extrema = 1 if options.restoreInteriorExtrema else 0
    opt.collect_timing = 1 if options.collectTiming else 0
    if ni_out is not None:
        opt.region_ni_out = ni_out.data_ptr()
        opt.region_ni_capacity = ni_out.numel()
    rep = N.lts_report_t()
    with torch.cuda.device(dev):
        tail = (N.ptr(pres_max), pres_max.numel(), N.ptr(pres_min), pres_min.numel(),
                N.ptr(order) if order is not None else None, N.ptr(g), N.ptr(G),
                ctypes.byref(rep), ctypes.byref(opt), N.ptr(ws), ws.numel(), N.stream_ptr(dev))
        if mesh.is_grid:
            rc = N.load().lts_simplify(N.ptr(values), mesh.dim, N.dims_arg(mesh.grid_dims), *tail)
        else:
            d = mesh.device_arrays(dev)
            rc = N.load().lts_simplify_csr(N.ptr(values), mesh.n, N.ptr(d["indptr"]), N.ptr(d["indices"]), *tail)
    N.check(rc)
    return g, G, rep


_host_scratch: dict = {}


def simplify_field_host(mesh: Triangulation, f_host: torch.Tensor, constraints: ConstraintSet,
                        options: Optional[SimplifyOptions] = None, g_out: Optional[torch.Tensor] = None,
                        G_out: Optional[torch.Tensor] = None, device=None):
    """simplify_field over HOST buffers (the reference's numpy-facing call,
    SPEC.md:348-356): f_host float32 (n) in host memory, ideally page-locked;
    the preserve lists are host id arrays.  Returns (g float32, G int32 ranks,
    SimplifyReport) as page-locked host tensors (g_out / G_out when given).
    One C call (lts_simplify_host): the upload, the pass, and the downloads,
    g leaving for the host while the last pass still floods.  Grids only."""
    if not mesh.is_grid:
        raise MeshError("simplify_field_host covers grids; use simplify_field for explicit meshes")
    N.require_cuda()
    options = options or SimplifyOptions()
    if options.zeta is not None:
        raise ValueError("simplify_field_host realises by contract D1 (zeta=None)")
    dev = torch.device(device or "cuda")
    f_host = f_host.reshape(-1)
    if f_host.device.type != "cpu" or f_host.dtype != torch.float32 or f_host.numel() != mesh.n:
        raise FieldError("f_host: a host float32 tensor of n values")
    pm = torch.as_tensor(np.asarray(constraints.preserveMaxima, dtype=np.int64).reshape(-1))
    pn = torch.as_tensor(np.asarray(constraints.preserveMinima, dtype=np.int64).reshape(-1))
    g = g_out if g_out is not None else torch.empty(mesh.n, dtype=torch.float32).pin_memory()
    G = G_out if G_out is not None else torch.empty(mesh.n, dtype=torch.int32).pin_memory()
    nb = ctypes.c_size_t(0)
    N.check(N.load().lts_host_scratch_size(mesh.dim, N.dims_arg(mesh.grid_dims), pm.numel(), pn.numel(),
                                           ctypes.byref(nb)))
    key = (str(dev), int(nb.value))
    scratch = _host_scratch.get(key)
    if scratch is None:
        _host_scratch.clear()
        scratch = _host_scratch[key] = torch.empty(int(nb.value), dtype=torch.uint8, device=dev)
    ws = _workspace(mesh, dev)
    opt = N.lts_options_t()
    opt.max_iterations = int(options.maxIterations)
    opt.restore_interior_extrema = 1 if options.restoreInteriorExtrema else 0
    opt.collect_timing = 1 if options.collectTiming else 0
    rep = N.lts_report_t()
    with torch.cuda.device(dev):
        rc = N.load().lts_simplify_host(N.ptr(f_host), mesh.dim, N.dims_arg(mesh.grid_dims), N.ptr(pm), pm.numel(),
                                        N.ptr(pn), pn.numel(), N.ptr(g), N.ptr(G), ctypes.byref(rep),
                                        ctypes.byref(opt), N.ptr(scratch), scratch.numel(), N.ptr(ws), ws.numel(),
                                        N.stream_ptr(dev))
    N.check(rc)
    return g, G, _report(rep)


def simplify_field(mesh: Triangulation, f, constraints: ConstraintSet,
                   options: Optional[SimplifyOptions] = None, order: Optional[OrderField] = None):
    """SPEC.md:348-356.  f: ScalarField (or array-like of n float32 values).
    Returns (g: ScalarField, G: OrderField, SimplifyReport)."""
    if not isinstance(f, ScalarField):
        f = ScalarField(mesh, f)
    options = options or SimplifyOptions()
    dev = f.values.device
    pmax = _ids(constraints.preserveMaxima, dev)
    pmin = _ids(constraints.preserveMinima, dev)
    ni = torch.empty(mesh.n, dtype=torch.int32, device=dev)
    g, G, rep = simplify_raw(mesh, f.values, pmax, pmin,
                             order.rank32 if order is not None else None, options, ni_out=ni)
    report = _report(rep, ni)
    Gf = OrderField(rank32=G)
    if options.zeta is not None:
        # SPEC.md:351 literal post-condition g = realize_numeric(f, G, zeta)
        gf = realize_numeric(f, Gf, options.zeta)
        report.linf = float((gf.values - f.values.to(torch.float64)).abs().max()) if mesh.n else 0.0
        return gf, Gf, report
    report.linf = float((g.to(torch.float64) - f.values.to(torch.float64)).abs().max()) if mesh.n else 0.0
    return ScalarField._wrap(mesh, g), Gf, report


def remove_extrema(mesh: Triangulation, F: OrderField, discardMaxima, discardMinima,
                   options: Optional[SimplifyOptions] = None):
    """SPEC.md:339-347 (black-list form).  Discards must be extrema of F."""
    dev = F.rank32.device
    mn, mx = extrema(mesh, F)
    dmax = _ids(discardMaxima, dev)
    dmin = _ids(discardMinima, dev)
    if dmax.numel() and not torch.isin(dmax, mx).all():
        raise ConstraintNotExtremum("a discard vertex is not a maximum of F")
    if dmin.numel() and not torch.isin(dmin, mn).all():
        raise ConstraintNotExtremum("a discard vertex is not a minimum of F")
    pmax = mx[~torch.isin(mx, dmax)]
    pmin = mn[~torch.isin(mn, dmin)]
    ni = torch.empty(mesh.n, dtype=torch.int32, device=dev)
    _, G, rep = simplify_raw(mesh, None, pmax.contiguous(), pmin.contiguous(), F.rank32.contiguous(), options,
                             ni_out=ni)
    return OrderField(rank32=G), _report(rep, ni)


@dataclass
class PassRegions:
    """Regions of one pass (SPEC Region list): region_ptr/verts are device
    arrays in the reference's localize_regions layout ([saddle] + vertices by
    ascending rank), plus the per-region local orders and N_I."""

    kind: str
    region_ptr: torch.Tensor
    region_verts: torch.Tensor
    local_rank: torch.Tensor
    n_iters: torch.Tensor
    status: torch.Tensor
    topseed: torch.Tensor
    report: PassReport
    new_order: OrderField


def _view_tensor(ws: torch.Tensor, addr, count, dtype):
    """Copy `count` elements at device address `addr` (inside the workspace
    tensor `ws`) into a fresh tensor; the view is only valid until the next call."""
    if count == 0 or not addr:
        return torch.empty(0, dtype=dtype, device=ws.device)
    off = int(addr) - ws.data_ptr()
    nbytes = count * torch.empty(0, dtype=dtype).element_size()
    assert 0 <= off and off + nbytes <= ws.numel()
    return ws[off:off + nbytes].view(dtype).clone()


def remove_pass(mesh: Triangulation, F: OrderField, preserve: ConstraintSet, kind: str = "max",
                max_iterations: int = 100) -> PassRegions:
    """One maxima pass (discover -> localize -> integrate) or one minima pass
    (on the reversed order) with its region artefacts."""
    dev = F.rank32.device
    pmark = torch.zeros(mesh.n, dtype=torch.uint8, device=dev)
    pm = _ids(preserve.preserveMaxima, dev)
    pn = _ids(preserve.preserveMinima, dev)
    if pm.numel():
        pmark[pm] |= 2
    if pn.numel():
        pmark[pn] |= 1
    inv = F.inverse32 if F.inverse32 is not None else F.inverse.to(torch.int32)
    nr = torch.empty_like(F.rank32)
    ni = torch.empty_like(F.rank32)
    ws = _workspace(mesh, dev)
    rep = N.lts_pass_report_t()
    view = N.lts_regions_view_t()
    with torch.cuda.device(dev):
        head = (0 if kind == "max" else 1, N.ptr(F.rank32), N.ptr(inv), N.ptr(pmark))
        tail = (int(max_iterations), N.ptr(nr), N.ptr(ni), None, ctypes.byref(rep), ctypes.byref(view),
                N.ptr(ws), ws.numel(), N.stream_ptr(dev))
        if mesh.is_grid:
            N.check(N.load().lts_remove_pass(*head, mesh.dim, N.dims_arg(mesh.grid_dims), *tail))
        else:
            d = mesh.device_arrays(dev)
            N.check(N.load().lts_remove_pass_csr(*head, mesh.n, N.ptr(d["indptr"]), N.ptr(d["indices"]), *tail))
        torch.cuda.current_stream(dev).synchronize()
    R, S = int(view.regions), int(view.slots)
    pr = PassReport(kind, rep.seeds, rep.regions, rep.claimed, rep.largest, rep.n_iter_max,
                    rep.capped, rep.shared_saddles, rep.maxima_edges, rep.boruvka_rounds,
                    rep.big_regions)
    return PassRegions(
        kind=kind,
        region_ptr=_view_tensor(ws, view.region_ptr, R + 1 if R else 0, torch.int64),
        region_verts=_view_tensor(ws, view.region_verts, S, torch.int32),
        local_rank=_view_tensor(ws, view.local_rank, S, torch.int32),
        n_iters=_view_tensor(ws, view.n_iters, R, torch.int32),
        status=_view_tensor(ws, view.status, R, torch.int32),
        topseed=_view_tensor(ws, view.topseed, R, torch.int32),
        report=pr, new_order=OrderField(rank32=nr, inverse32=ni))


def discover_regions(mesh: Triangulation, F: OrderField, discardMaxima) -> PassRegions:
    """regions of the maxima pass that discards discardMaxima."""
    mn, mx = extrema(mesh, F)
    d = _ids(discardMaxima, F.rank32.device)
    if d.numel() and not torch.isin(d, mx).all():
        raise ConstraintNotExtremum("a discard vertex is not a maximum of F")
    keep = mx[~torch.isin(mx, d)]
    return remove_pass(mesh, F, ConstraintSet(preserveMinima=mn, preserveMaxima=keep), "max")


def verify_constraints(mesh: Triangulation, G: OrderField, constraints: ConstraintSet) -> VerifyReport:
    """recompute extrema of G and compare with the preserve sets."""
    dev = G.rank32.device
    mn, mx = extrema(mesh, G)
    pm = _ids(constraints.preserveMaxima, dev)
    pn = _ids(constraints.preserveMinima, dev)
    extra_max = mx[~torch.isin(mx, pm)]
    lost_max = pm[~torch.isin(pm, mx)]
    extra_min = mn[~torch.isin(mn, pn)]
    lost_min = pn[~torch.isin(pn, mn)]
    ok = not (extra_max.numel() or lost_max.numel() or extra_min.numel() or lost_min.numel())
    return VerifyReport(ok, extra_max, lost_max, extra_min, lost_min)
