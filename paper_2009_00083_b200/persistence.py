"""Persistence-driven mode (persistence module; reference
pairs_sweep, _kernels.py:309-421).

``compute_extremum_saddle_pairs`` runs on the GPU (``lts_extremum_pairs``,
csrc/persistence.cuh): the maxima graph of the discover kernels, its maximum
spanning forest, and an Elder-rule sweep over the forest edges, which equals
the reference's truncated propagation sweep for every epsilon (DESIGN.md,
tests/test_pairs.py).  ``persistence_simplify`` is the persistence-driven
specialisation of LTS (§4.5): the non-surviving extrema of both polarities are
discarded and the LTS pass removes them; ||f - g||_inf <= epsilon.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _native as N
from .engine import ConstraintSet, SimplifyOptions, simplify_field
from .order import OrderField, ScalarField
from .triangulation import Triangulation


@dataclass
class PersistencePairs:
    """Pairs of one polarity: ``extrema`` (vertex ids, ascending) and
    ``saddles`` (the junction vertex each one dies at, -1 for survivors);
    ``persistence`` = |f(extremum) - f(saddle)| (inf for survivors)."""

    polarity: str
    epsilon: float
    extrema: torch.Tensor
    saddles: torch.Tensor
    persistence: torch.Tensor

    @property
    def survivors(self) -> torch.Tensor:
        return self.extrema[self.saddles < 0]

    def pairs(self):
        """(extremum, saddle, persistence) of the pairs below epsilon."""
        m = self.saddles >= 0
        return self.extrema[m], self.saddles[m], self.persistence[m]


def compute_extremum_saddle_pairs(mesh: Triangulation, f, F: Optional[OrderField] = None,
                                  polarity: str = "max", epsilon: float = float("inf")) -> PersistencePairs:
    """SPEC compute_extremum_saddle_pairs."""
    if polarity not in ("max", "min"):
        raise ValueError("polarity must be 'max' or 'min' (use both calls for 'both')")
    if not mesh.is_grid:
        from .errors import MeshError
        raise MeshError("the persistence-driven mode runs on grids (explicit meshes: simplify_field)")
    if not isinstance(f, ScalarField):
        f = ScalarField(mesh, f)
    N.require_cuda()
    vals = f.values
    n = mesh.n
    dev = vals.device
    ext = torch.empty(n, dtype=torch.int32, device=dev)
    sad = torch.empty(n, dtype=torch.int32, device=dev)
    cnt = ctypes.c_int64(0)
    ws = N.workspace(mesh.grid_dims, dev)
    order = F.rank32 if F is not None else None
    with torch.cuda.device(dev):
        N.check(N.load().lts_extremum_pairs(N.ptr(vals), N.ptr(order), mesh.dim, N.dims_arg(mesh.grid_dims),
                                            0 if polarity == "max" else 1, float(epsilon), N.ptr(ext), N.ptr(sad),
                                            ctypes.byref(cnt), N.ptr(ws), ws.numel(), N.stream_ptr(dev)))
    k = int(cnt.value)
    e = ext[:k].to(torch.int64)
    s = sad[:k].to(torch.int64)
    v64 = vals.to(torch.float64)
    p = torch.full((k,), float("inf"), dtype=torch.float64, device=dev)
    m = s >= 0
    p[m] = (v64[e[m]] - v64[s[m]]).abs()
    return PersistencePairs(polarity, float(epsilon), e, s, p)


def persistence_curve(pairs, value_range: Optional[float] = None):
    """SPEC persistence_curve: for each distinct persistence
    t, the number of pairs with persistence >= t.  ``pairs``: PersistencePairs
    (or a list of them); survivors count with persistence = value_range when
    given (the global pair convention), else they are left out."""
    if isinstance(pairs, PersistencePairs):
        pairs = [pairs]
    ps = []
    for pp in pairs:
        p = pp.persistence.cpu().numpy()
        fin = p[np.isfinite(p)]
        ps.append(fin)
        if value_range is not None:
            ps.append(np.full(int((~np.isfinite(p)).sum()), float(value_range)))
    allp = np.sort(np.concatenate(ps)) if ps else np.zeros(0)
    thr = np.unique(allp)
    counts = allp.size - np.searchsorted(allp, thr, side="left")
    return thr, counts


def persistence_simplify(mesh: Triangulation, f, epsilon: float, options: Optional[SimplifyOptions] = None):
    """SPEC persistence_simplify: discard every extremum less
    persistent than epsilon (both polarities) and run LTS.  Returns
    (g, G, (max pairs, min pairs), report)."""
    if not isinstance(f, ScalarField):
        f = ScalarField(mesh, f)
    from .order import compute_order_field
    F = compute_order_field(f)
    pmax = compute_extremum_saddle_pairs(mesh, f, F, "max", epsilon)
    pmin = compute_extremum_saddle_pairs(mesh, f, F, "min", epsilon)
    cs = ConstraintSet(preserveMinima=pmin.survivors, preserveMaxima=pmax.survivors)
    g, G, rep = simplify_field(mesh, f, cs, options, order=F)
    return g, G, (pmax, pmin), rep
