"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container only (needs /root/reference and numba):

    python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src and
runs its own numba kernels -- compute_order_field (order.py:86-91),
classify_grid (_kernels.py:128-156, re-jitted serially because its
parallel=True build fails under numba 0.65), discover_sweep
(_kernels.py:194-303), localize_regions (_kernels.py:578-591) and
realize_sweep (_kernels.py:84-99) -- glued together by SPEC.md:281-404 with the
SURVEY section 8c decisions D1-D11 (the engine glue is missing from the
reference).  The outputs pin the C/numpy oracle in oracle/ and the
GPU path; the fixtures are small .npz files committed under tests/golden/.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import numba  # noqa: E402
from topoflat import _kernels as K  # noqa: E402  (reference, read-only)
from topoflat import order as O  # noqa: E402
from topoflat import triangulation as T  # noqa: E402

from paper_2009_00083_b200 import synthetic as S  # noqa: E402

classify_grid_serial = numba.njit(cache=False)(K.classify_grid.py_func)


def ref_classify(mesh, rank):
    lo = np.empty(mesh.n, np.int16)
    up = np.empty(mesh.n, np.int16)
    if not mesh.is_grid:  # explicit mesh: the reference's classify_explicit
        K.classify_explicit(np.asarray(rank, np.int64), mesh.indptr, mesh.indices, mesh.link_ptr,
                            mesh.link_a, mesh.link_b, lo, up)
        return lo, up
    offs, pairs = T.grid_link_tables(mesh.dim)
    dims = np.asarray(mesh.grid_dims, np.int64)
    strides = np.array([1, dims[0]] + ([dims[0] * dims[1]] if mesh.dim == 3 else []), np.int64)
    classify_grid_serial(np.asarray(rank, np.int64), dims, strides, offs,
                         pairs[:, 0].copy(), pairs[:, 1].copy(), lo, up)
    return lo, up


def ref_pass(mesh, rank, seeds, max_iter):
    """maxima pass with the reference kernels + SPEC integration key sort."""
    n = mesh.n
    rank = np.asarray(rank, np.int64)
    if seeds.size == 0:
        return rank.copy(), None
    state, owner, saddle, parked, topseed, parent, err = K.discover_sweep(
        rank, mesh.indptr, mesh.indices, seeds.astype(np.int64))
    assert err == 0
    claimed = np.flatnonzero(state == K.CLAIMED)
    own = owner[claimed]
    roots = np.unique(own)
    order = np.lexsort((rank[claimed], own))
    cl = claimed[order]
    ow = own[order]
    starts = np.searchsorted(ow, roots, "left")
    ends = np.searchsorted(ow, roots, "right")
    sizes = ends - starts + 1
    rp = np.zeros(roots.size + 1, np.int64)
    np.cumsum(sizes, out=rp[1:])
    rv = np.empty(rp[-1], np.int64)
    for i, r in enumerate(roots):
        rv[rp[i]] = saddle[r]
        rv[rp[i] + 1:rp[i + 1]] = cl[starts[i]:ends[i]]
    loc = np.empty(rp[-1], np.int64)
    nit = np.empty(roots.size, np.int64)
    st = np.empty(roots.size, np.int64)
    K.localize_regions(rp, rv, rank, mesh.indptr, mesh.indices, max_iter, loc, nit, st)
    assert not np.any(st == 1)
    big = np.int64(2 ** 62)
    p1 = rank.copy()
    p2 = np.zeros(n, np.int64)
    p3 = np.zeros(n, np.int64)
    for i, r in enumerate(roots):
        lo, hi = rp[i], rp[i + 1]
        s = rv[lo]
        vs = rv[lo + 1:hi]
        p1[vs] = rank[s]
        p2[vs] = loc[lo + 1:hi]
        p3[vs] = topseed[r]
        p2[s] = big
        p3[s] = big
    inv = np.lexsort((p3, p2, p1))
    newrank = np.empty(n, np.int64)
    newrank[inv] = np.arange(n)
    art = dict(region_ptr=rp, region_verts=rv, local=loc, n_iters=nit, status=st,
               topseed=topseed[roots], state=state)
    return newrank, art


def nbr_ranks(mesh, rank, v):
    return [int(rank[u]) for u in mesh.neighbors(int(v))]


def ref_simplify(mesh, f32, pmax, pmin, max_iter=100):
    n = mesh.n
    F = O.compute_order_field(O.ScalarField(mesh, f32.astype(np.float64)))
    G = F.rank.copy()
    g = f32.copy()
    first = {}
    it = 0
    ok = False
    for it in range(1, max_iter + 1):
        lo, up = ref_classify(mesh, G)
        G1, a1 = ref_pass(mesh, G, np.setdiff1d(np.flatnonzero(up == 0), pmax), max_iter)
        if a1 is not None:
            K.realize_sweep(g, O.order_from_ranks(G1).inverse, 0.0)
        lo1, up1 = ref_classify(mesh, G1)
        G2r, a2 = ref_pass(mesh, (n - 1) - G1, np.setdiff1d(np.flatnonzero(lo1 == 0), pmin),
                           max_iter)
        G2 = (n - 1) - G2r
        if a2 is not None:
            h = -g
            K.realize_sweep(h, O.order_from_ranks(G2).inverse[::-1].copy(), 0.0)
            g = -h
        if it == 1:
            first = dict(G1=G1, G2=G2, max=a1, min=a2)
        lo2, up2 = ref_classify(mesh, G2)
        mn2 = np.flatnonzero(lo2 == 0)
        mx2 = np.flatnonzero(up2 == 0)
        lost_min = np.setdiff1d(pmin, mn2)
        lost_max = np.setdiff1d(pmax, mx2)
        if lost_min.size or lost_max.size:  # D6
            for x in sorted(lost_min.tolist()):
                rx = G2[x]
                ry = min(nbr_ranks(mesh, G2, x))
                if ry < rx:
                    G2[(G2 >= ry) & (G2 < rx)] += 1
                    G2[x] = ry
            for x in sorted(lost_max.tolist()):
                rx = G2[x]
                ry = max(nbr_ranks(mesh, G2, x))
                if ry > rx:
                    G2[(G2 > rx) & (G2 <= ry)] -= 1
                    G2[x] = ry
            lo2, up2 = ref_classify(mesh, G2)
            mn2 = np.flatnonzero(lo2 == 0)
            mx2 = np.flatnonzero(up2 == 0)
        G = G2
        if np.array_equal(mx2, pmax) and np.array_equal(mn2, pmin):
            ok = True
            break
    g[g == 0] = 0.0
    return F, G, g, ok, it, first


def cases():
    """(name, f32 array (numpy shape), n_keep_max, n_keep_min)."""
    out = []
    for s in (0, 1):
        r = np.random.default_rng(100 + s)
        f = np.round(r.random((29, 33)) * 16) / 16  # many exact ties
        out.append((f"rand2d_33x29_s{s}", f.astype(np.float32), 3, 2))
        r = np.random.default_rng(200 + s)
        f = np.round(r.random((7, 8, 9)) * 20) / 20
        out.append((f"rand3d_9x8x7_s{s}", f.astype(np.float32), 3, 3))
    r = np.random.default_rng(300)
    f = r.standard_normal((24, 24)).astype(np.float32)
    f[r.random((24, 24)) < 0.15] = 0.0
    f[r.random((24, 24)) < 0.15] = -0.0
    out.append(("zeros2d_24x24", f, 1, 1))  # stress: only global extrema kept
    r = np.random.default_rng(301)
    out.append(("stress3d_12x10x11", r.random((11, 10, 12)).astype(np.float32), 1, 1))
    out.append(("const2d_8x8", np.full((8, 8), 0.5, np.float32), 1, 1))
    out.append(("cfg1_64", S.cfg1(0, N=64), 4, 1))
    out.append(("cfg2_16", S.cfg2(0, N=16), 8, 1))
    out.append(("cfg3_32", S.cfg3(0, N=32), 10, 10))
    # scaled cfg3 whose maxima pass is non-empty (cfg3_32 has one maximum)
    out.append(("cfg3_48_s5", S.cfg3(5, N=48), 1, 3))
    out.append(("cfg4_192", S.cfg4(0, N=192, ndisk=20), 20, 1))
    out.append(("cfg5_24", S.cfg5(0, N=24), 12, 12))
    # outer loop > 1 and capped (status 2) regions (SURVEY F5 at small scale)
    out.append(("cfg4_160_s1", S.cfg4(1, N=160, ndisk=12), 12, 1))
    for s in (0, 2):
        r = np.random.default_rng(s)
        out.append((f"quant2d_40_s{s}", (np.round(r.random((40, 40)) * 6) / 6).astype(np.float32), 1, 1))
    # restoration (D6): preserved minimum in a crater on a discarded hill
    y, x = np.mgrid[0:11, 0:21].astype(np.float64)
    f = (2 * np.exp(-((x - 5) ** 2 + (y - 5) ** 2) / 8) + 1.5 * np.exp(-((x - 15) ** 2 + (y - 5) ** 2) / 8)
         - 0.8 * np.exp(-((x - 15) ** 2 + (y - 5) ** 2) / 1.0) + 0.001 * x + 0.0007 * y)
    out.append(("crater2d_21x11", f.astype(np.float32), 1, (0, 15 + 21 * 5)))
    r = np.random.default_rng(7)
    z, yy, xx = np.mgrid[0:20, 0:18, 0:22].astype(np.float64)
    f = sum(r.uniform(0.5, 1) * np.exp(-((xx - r.uniform(0, 22)) ** 2 + (yy - r.uniform(0, 18)) ** 2
                                        + (z - r.uniform(0, 20)) ** 2) / (2 * r.uniform(2, 5) ** 2))
            for _ in range(6)) + 0.05 * r.random((20, 18, 22))
    out.append(("gauss3d_22x18x20", f.astype(np.float32), 4, 4))
    return out


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main(only=()):
    for name, f, kmax, kmin in cases():
        if only and name not in only:
            continue
        dims = tuple(f.shape[::-1])
        mesh = T.build_grid_triangulation(dims)
        f32 = np.ascontiguousarray(f.ravel(), np.float32)
        F = O.compute_order_field(O.ScalarField(mesh, f32.astype(np.float64)))
        lo, up = ref_classify(mesh, F.rank)
        mx = np.flatnonzero(up == 0)
        mn = np.flatnonzero(lo == 0)
        if isinstance(kmin, tuple):  # explicit minima: (0 -> global min, ids...)
            pmax, _ = S.select_preserved(F.rank, mx, mn, kmax, 0)
            pmin = np.array(sorted({int(F.inverse[0])} | set(kmin[1:])), np.int64)
        else:
            pmax, pmin = S.select_preserved(F.rank, mx, mn, kmax, kmin)
        Fr, G, g, ok, it, first = ref_simplify(mesh, f32, pmax, pmin)
        rec = dict(dims=np.array(dims, np.int64), f=f32, pres_max=pmax, pres_min=pmin,
                   F_rank=F.rank.astype(np.int32), lower=lo, upper=up,
                   G_rank=G.astype(np.int32), g=g, ok=np.array(ok), outer=np.array(it),
                   G1=first["G1"].astype(np.int32), G2_first=first["G2"].astype(np.int32))
        for kind in ("max", "min"):
            a = first[kind]
            if a is None:
                continue
            for key in ("region_ptr", "region_verts", "local", "n_iters", "status", "topseed"):
                rec[f"{kind}_{key}"] = np.asarray(a[key])
            rec[f"{kind}_claimed"] = np.flatnonzero(a["state"] == K.CLAIMED).astype(np.int32)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **rec)
        print(f"{name}: n={f32.size} maxima={mx.size} minima={mn.size} ok={ok} outer={it} "
              f"G={sha(G.astype(np.int32))[:12]} g={sha(g)[:12]}", flush=True)


if __name__ == "__main__":
    main(tuple(sys.argv[1:]))
