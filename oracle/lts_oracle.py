"""CPU oracle for the LTS hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.  It is the checker, never the
thing measured as the product and never a fallback of the product path.

It restates the reference (``/root/reference``) in two layers:

* ``liblts_oracle.so`` (lts_oracle.c): the reference's numba kernels
  (_kernels.py: classify_grid, discover_sweep, localize_regions, realize_sweep),
  the order field (order.py:86-91) and SPEC's integration key sort.
* this file: the missing engine glue, restated from SPEC.md:281-404 with the
  frozen decisions D1-D11 of SURVEY.md section 8c.

Parity pin: tests/test_oracle_golden.py checks this oracle against fixtures
made by tests/golden/make_golden.py, which runs the reference's own numba
kernels (imported read-only from /root/reference) in this container.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import time
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblts_oracle.so")
SRC_PATH = os.path.join(HERE, "lts_oracle.c")

CLAIMED = 2  # _kernels.py:20


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC_PATH):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", SRC_PATH, "-o", LIB_PATH, "-lm"])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i64, i32 = ctypes.c_int64, ctypes.c_int
        L.orc_grid_tables.argtypes = [i32, P, P]
        L.orc_order_field.argtypes = [P, i64, P, P]
        L.orc_order_field.restype = i64
        L.orc_classify_grid.argtypes = [P, i32, P, P, P, i32]
        L.orc_discover_sweep.argtypes = [P, i32, P, P, i64, P, P, P, P, P]
        L.orc_localize_regions.argtypes = [P, i64, P, P, i32, P, i32, P, P, P, i32]
        L.orc_integrate.argtypes = [P, i64, P, i64, P, P, P, P]
        L.orc_integrate.restype = i64
        L.orc_realize_sweep_f32.argtypes = [P, P, i64]
        L.orc_pairs_sweep.argtypes = [P, P, i32, P, P, i64, ctypes.c_double, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _dims(dims):
    return np.ascontiguousarray(np.asarray(dims, dtype=np.int64))


class OracleError(ValueError):
    pass


# --------------------------------------------------------------------------
# kernels (thin wrappers)
# --------------------------------------------------------------------------

def grid_tables(ndim: int):
    """Offsets and link pairs (triangulation.py:30-78)."""
    K = 6 if ndim == 2 else 14
    offs = np.zeros(K * ndim, np.int32)
    pairs = np.zeros(2 * 96, np.int32)
    npairs = lib().orc_grid_tables(ndim, _p(offs), _p(pairs))
    return offs.reshape(K, ndim), pairs[:2 * npairs].reshape(npairs, 2)


def order_field(f32: np.ndarray):
    """order.py:86-91: stable argsort by value, ties by id -> (rank, inverse) int32."""
    f = np.ascontiguousarray(f32.ravel(), dtype=np.float32)
    n = f.size
    rank = np.empty(n, np.int32)
    inv = np.empty(n, np.int32)
    bad = lib().orc_order_field(_p(f), n, _p(rank), _p(inv))
    if bad:
        raise OracleError("scalar field contains NaN or infinite values")
    return rank, inv


def classify(dims, rank: np.ndarray, nthreads: int = 0):
    """classify_grid (_kernels.py:128-156): (lower, upper) int16 counts."""
    rank = np.ascontiguousarray(rank, dtype=np.int32)
    d = _dims(dims)
    lo = np.empty(rank.size, np.int16)
    up = np.empty(rank.size, np.int16)
    lib().orc_classify_grid(_p(rank), d.size, _p(d), _p(lo), _p(up), nthreads)
    return lo, up


def extrema(dims, rank, nthreads: int = 0):
    lo, up = classify(dims, rank, nthreads)
    return np.flatnonzero(lo == 0), np.flatnonzero(up == 0)  # minima, maxima


def discover(dims, rank, seeds):
    """discover_sweep (_kernels.py:194-303)."""
    rank = np.ascontiguousarray(rank, dtype=np.int32)
    seeds = np.ascontiguousarray(seeds, dtype=np.int32)
    d = _dims(dims)
    n = rank.size
    m = seeds.size
    state = np.empty(n, np.int8)
    owner = np.empty(n, np.int32)
    saddle = np.empty(max(m, 1), np.int32)
    parked = np.empty(max(m, 1), np.uint8)
    topseed = np.empty(max(m, 1), np.int32)
    err = lib().orc_discover_sweep(_p(rank), d.size, _p(d), _p(seeds), m, _p(state), _p(owner),
                                   _p(saddle), _p(parked), _p(topseed))
    return state, owner, saddle[:m], parked[:m].astype(bool), topseed[:m], err


def localize(dims, region_ptr, region_verts, rank, max_iter=100, nthreads: int = 0):
    """localize_regions (_kernels.py:578-591)."""
    d = _dims(dims)
    region_ptr = np.ascontiguousarray(region_ptr, dtype=np.int64)
    region_verts = np.ascontiguousarray(region_verts, dtype=np.int32)
    rank = np.ascontiguousarray(rank, dtype=np.int32)
    R = region_ptr.size - 1
    local = np.empty(region_verts.size, np.int32)
    nit = np.empty(max(R, 1), np.int32)
    st = np.empty(max(R, 1), np.int32)
    lib().orc_localize_regions(_p(region_ptr), R, _p(region_verts), _p(rank), d.size, _p(d),
                               int(max_iter), _p(local), _p(nit), _p(st), nthreads)
    return local, nit[:R], st[:R]


def integrate(rank, region_ptr, region_verts, local, topseed_rank):
    """G = position in (primary, secondary, tertiary) key order."""
    rank = np.ascontiguousarray(rank, dtype=np.int32)
    region_ptr = np.ascontiguousarray(region_ptr, dtype=np.int64)
    region_verts = np.ascontiguousarray(region_verts, dtype=np.int32)
    local = np.ascontiguousarray(local, dtype=np.int32)
    topseed_rank = np.ascontiguousarray(topseed_rank, dtype=np.int32)
    out = np.empty(rank.size, np.int32)
    coll = lib().orc_integrate(_p(rank), rank.size, _p(region_ptr), region_ptr.size - 1,
                               _p(region_verts), _p(local), _p(topseed_rank), _p(out))
    if coll:
        raise OracleError(f"integration key collision ({coll})")
    return out


def pairs(dims, rank: np.ndarray, values: np.ndarray, kind: str = "max", eps: float = float("inf")):
    """Truncated extremum-saddle pairs (reference pairs_sweep, _kernels.py:309-421)
    from every maximum (kind "max") or every minimum (kind "min": the same sweep
    on the reversed order n-1-rank and negated values, SPEC persistence).
    Returns (extrema ids ascending, pair saddle per extremum or -1 = survivor, err)."""
    rank = np.ascontiguousarray(rank, np.int32)
    values = np.ascontiguousarray(values, np.float64)
    n = rank.size
    mn, mx = extrema(dims, rank)
    if kind == "max":
        seeds, r, v = mx, rank, values
    else:
        seeds, r, v = mn, np.ascontiguousarray(n - 1 - rank, np.int32), np.ascontiguousarray(-values)
    seeds = np.ascontiguousarray(np.sort(seeds), np.int32)
    out = np.full(seeds.size, -1, np.int32)
    err = lib().orc_pairs_sweep(_p(r), _p(v), len(dims), _p(_dims(dims)), _p(seeds), seeds.size,
                                float(eps), _p(out))
    if err < 0:
        raise OracleError("bad grid")
    return seeds.astype(np.int64), out.astype(np.int64), int(err)


def realize_sweep_f32(g: np.ndarray, inverse: np.ndarray) -> None:
    """realize_sweep (_kernels.py:84-99) in place on float32 with zeta = 0."""
    assert g.dtype == np.float32 and g.flags.c_contiguous
    inverse = np.ascontiguousarray(inverse, dtype=np.int32)
    lib().orc_realize_sweep_f32(_p(g), _p(inverse), g.size)


def inverse_of(rank: np.ndarray) -> np.ndarray:
    """order_from_ranks (order.py:94-99)."""
    inv = np.empty(rank.size, np.int32)
    inv[rank] = np.arange(rank.size, dtype=np.int32)
    return inv


# --------------------------------------------------------------------------
# engine glue (decisions D1-D11)
# --------------------------------------------------------------------------

@dataclass
class PassInfo:
    kind: str                 # "max" or "min"
    seeds: int = 0
    regions: int = 0
    claimed: int = 0
    largest: int = 0          # largest region size, saddle included
    n_iter_max: int = 0
    capped: int = 0
    region_ptr: np.ndarray = field(default=None, repr=False)
    region_verts: np.ndarray = field(default=None, repr=False)
    local: np.ndarray = field(default=None, repr=False)
    n_iters: np.ndarray = field(default=None, repr=False)
    topseed: np.ndarray = field(default=None, repr=False)
    seconds: dict = field(default_factory=dict)


def assemble_regions(rank, state, owner, saddle, topseed):
    """D7: region = [saddle] + claimed vertices of one root by ascending rank."""
    claimed = np.flatnonzero(state == CLAIMED)
    own = owner[claimed]
    roots = np.unique(own)
    order = np.lexsort((rank[claimed], own))
    cl = claimed[order]
    sizes = np.bincount(np.searchsorted(roots, own[order]), minlength=roots.size) + 1
    ptr = np.zeros(roots.size + 1, np.int64)
    np.cumsum(sizes, out=ptr[1:])
    verts = np.empty(int(ptr[-1]), np.int32)
    head = np.zeros(verts.size, bool)
    head[ptr[:-1]] = True
    verts[ptr[:-1]] = saddle[roots]
    verts[~head] = cl
    return ptr, verts, topseed[roots], roots


def remove_pass(dims, rank, seeds, max_iter=100, kind="max", nthreads=0):
    """One maxima pass (discover -> localize -> integrate) on ``rank``."""
    info = PassInfo(kind=kind, seeds=int(seeds.size))
    if seeds.size == 0:
        return rank.copy(), info
    t0 = time.perf_counter()
    state, owner, saddle, parked, topseed, err = discover(dims, rank, seeds)
    if err:
        raise OracleError("discover_sweep reported err=1")
    t1 = time.perf_counter()
    ptr, verts, tops, roots = assemble_regions(rank, state, owner, saddle, topseed)
    if np.any(saddle[roots] < 0):
        raise OracleError("region without a saddle (every maximum discarded?)")
    t2 = time.perf_counter()
    local, nit, st = localize(dims, ptr, verts, rank, max_iter, nthreads)
    if np.any(st == 1):
        raise OracleError("region without an admissible boundary minimum (status 1)")
    t3 = time.perf_counter()
    newrank = integrate(rank, ptr, verts, local, tops)
    t4 = time.perf_counter()
    sizes = np.diff(ptr)
    info.regions = int(roots.size)
    info.claimed = int(sizes.sum() - roots.size)
    info.largest = int(sizes.max())
    info.n_iter_max = int(nit.max())
    info.capped = int(np.sum(st == 2))
    info.region_ptr, info.region_verts, info.local = ptr, verts, local
    info.n_iters, info.topseed = nit, tops
    info.seconds = dict(discover=t1 - t0, assemble=t2 - t1, localize=t3 - t2, integrate=t4 - t3)
    return newrank, info


def neighbor_ranks(dims, rank, v):
    offs, _ = grid_tables(len(dims))
    c = []
    rest = int(v)
    for a in range(len(dims)):
        c.append(rest % dims[a])
        rest //= dims[a]
    out = []
    for o in offs:
        q = [c[a] + int(o[a]) for a in range(len(dims))]
        if all(0 <= q[a] < dims[a] for a in range(len(dims))):
            u = q[0] + dims[0] * (q[1] + (dims[1] * q[2] if len(dims) == 3 else 0))
            out.append(int(rank[u]))
    return out


def restore_extrema(dims, rank, lost_min, lost_max):
    """D6: re-rank each lost preserved minimum just below its
    lowest neighbour and each lost maximum just above its highest neighbour,
    in ascending vertex-id order, minima first."""
    rank = rank.copy()
    for x in sorted(int(v) for v in lost_min):
        rx = int(rank[x])
        ry = min(neighbor_ranks(dims, rank, x))
        if ry < rx:
            sel = (rank >= ry) & (rank < rx)
            rank[sel] += 1
            rank[x] = ry
    for x in sorted(int(v) for v in lost_max):
        rx = int(rank[x])
        ry = max(neighbor_ranks(dims, rank, x))
        if ry > rx:
            sel = (rank > rx) & (rank <= ry)
            rank[sel] -= 1
            rank[x] = ry
    return rank


@dataclass
class OracleResult:
    F_rank: np.ndarray
    G_rank: np.ndarray
    g: np.ndarray
    ok: bool
    outer_iterations: int
    passes: list
    pres_max: np.ndarray
    pres_min: np.ndarray
    restored: int
    seconds: dict


def simplify(dims, f32, pres_max, pres_min, max_iterations=100, restore=True, nthreads=0,
             F=None):
    """simplify_field with D1-D11.  Returns OracleResult."""
    tt = {}
    t0 = time.perf_counter()
    f = np.ascontiguousarray(np.asarray(f32, np.float32).ravel())
    n = f.size
    if F is None:
        rank0, _ = order_field(f)
    else:
        rank0 = np.ascontiguousarray(F, np.int32)
    tt["order"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    mn0, mx0 = extrema(dims, rank0, nthreads)
    tt["classify"] = time.perf_counter() - t0
    pmax = np.unique(np.asarray(pres_max, np.int64))
    pmin = np.unique(np.asarray(pres_min, np.int64))
    if pmax.size == 0:
        pmax = np.array([int(np.argmax(rank0))])
    if pmin.size == 0:
        pmin = np.array([int(np.argmin(rank0))])
    if not np.all(np.isin(pmax, mx0)) or not np.all(np.isin(pmin, mn0)):
        raise OracleError("ConstraintNotExtremum")
    G = rank0.copy()
    g = f.copy()
    passes = []
    ok = False
    restored = 0
    it = 0
    for it in range(1, max_iterations + 1):
        # maxima pass
        _, mx = extrema(dims, G, nthreads)
        G1, info = remove_pass(dims, G, np.setdiff1d(mx, pmax), max_iterations, "max", nthreads)
        passes.append(info)
        if info.regions:
            realize_sweep_f32(g, inverse_of(G1))
        # minima pass on the reversed order (D3)
        mn1, _ = extrema(dims, G1, nthreads)
        G2r, info = remove_pass(dims, (n - 1) - G1, np.setdiff1d(mn1, pmin), max_iterations, "min",
                                nthreads)
        passes.append(info)
        G2 = (n - 1) - G2r
        if info.regions:
            h = -g
            realize_sweep_f32(h, inverse_of(G2)[::-1].copy())
            g = -h
        # restoration (D6) and verification
        mn2, mx2 = extrema(dims, G2, nthreads)
        lost_min = np.setdiff1d(pmin, mn2)
        lost_max = np.setdiff1d(pmax, mx2)
        if restore and (lost_min.size or lost_max.size):
            restored += int(lost_min.size + lost_max.size)
            G2 = restore_extrema(dims, G2, lost_min, lost_max)
            mn2, mx2 = extrema(dims, G2, nthreads)
        G = G2.astype(np.int32)
        if np.array_equal(mx2, pmax) and np.array_equal(mn2, pmin):
            ok = True
            break
    g[g == 0] = 0.0  # D10: canonical +0.0
    return OracleResult(F_rank=rank0, G_rank=G, g=g, ok=ok, outer_iterations=it, passes=passes,
                        pres_max=pmax, pres_min=pmin, restored=restored, seconds=tt)
