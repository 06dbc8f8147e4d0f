"""Golden fixtures for explicit triangle meshes, made by the
REFERENCE implementation: its own mesh builders (triangulation.py:172-361),
classify_explicit (_kernels.py:159-187), discover_sweep / localize_regions
over the mesh CSR (_kernels.py:194-303, 578-591) and realize_sweep, glued by
the same SPEC engine restatement as make_golden.py.  Run in the build
container only:

    python tests/golden/make_explicit_golden.py

Output: tests/golden/explicit/*.npz (mesh points / triangles, field, preserve
lists, F, lower / upper counts, G, g, first-pass regions).
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as MG  # noqa: E402  (imports the reference read-only)
from make_golden import K, O, T  # noqa: E402

OUT = os.path.join(HERE, "explicit")


def fig5_mesh():
    """The paper's running example: a hexagon
    of the triangular lattice, rows y = 2..-2, vertices A..X in reading order."""
    rows = [(2, [1, 2, 3, 4]), (1, [0.5, 1.5, 2.5, 3.5, 4.5]), (0, [0, 1, 2, 3, 4, 5]),
            (-1, [0.5, 1.5, 2.5, 3.5, 4.5]), (-2, [1, 2, 3, 4])]
    pts = np.array([(x, y, 0.0) for y, xs in rows for x in xs], np.float64)
    d = pts[:, None, :2] - pts[None, :, :2]
    adj = np.isclose((d[..., 0] ** 2) + (d[..., 1] / 2) ** 2 * 4 * 0.25 * 4, 1.0)  # lattice unit steps
    adj = np.isclose(np.abs(d[..., 0]) + 0.5 * np.abs(d[..., 1]), 1.0) & (np.abs(d[..., 1]) <= 1)
    n = len(pts)
    tris = [(i, j, k) for i in range(n) for j in range(i + 1, n) if adj[i, j]
            for k in range(j + 1, n) if adj[i, k] and adj[j, k]]
    return T.build_explicit_triangulation(pts, np.array(tris, np.int64))


# Fig. 5a orders, A..X
FIG5_F = [3, 2, 1, 0, 4, 17, 16, 15, 14, 23, 10, 18, 12, 19, 13, 9, 11, 20, 21, 22, 8, 7, 6, 5]


def icosphere(level):
    m = T.make_icosahedron()
    pts = m.points / np.linalg.norm(m.points, axis=1, keepdims=True)
    tris = m.triangles
    for _ in range(level):
        cache = {}
        pts = list(pts)

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in cache:
                p = (pts[a] + pts[b]) / 2
                pts.append(p / np.linalg.norm(p))
                cache[key] = len(pts) - 1
            return cache[key]

        nt = []
        for a, b, c in tris:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nt += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        pts, tris = np.array(pts), np.array(nt, np.int64)
    return T.build_explicit_triangulation(pts, tris)


def cases():
    r = np.random.default_rng(11)
    out = []
    m = T.make_octahedron()
    out.append(("octahedron", m, (m.points @ np.array([0.3, -0.2, 1.0])).astype(np.float32), 1, 1))
    m = T.make_icosahedron()
    out.append(("icosahedron", m, r.random(m.n).astype(np.float32), 1, 1))
    m = T.make_torus(8, 8)
    out.append(("torus_8x8", m, np.round(r.random(m.n) * 20).astype(np.float32) / 20, 2, 2))
    m = T.make_torus(24, 18)
    f = (np.sin(m.points[:, 0]) + np.cos(2 * m.points[:, 1]) + 0.3 * r.random(m.n)).astype(np.float32)
    out.append(("torus_24x18", m, f, 3, 3))
    m = fig5_mesh()
    out.append(("fig5", m, np.array(FIG5_F, np.float32), None, None))
    m = icosphere(4)  # 2562 vertices: regions above the CTA-flood threshold
    p = m.points
    f = (np.sin(3 * p[:, 0]) * np.cos(2 * p[:, 1]) + p[:, 2] + 0.15 * r.random(m.n)).astype(np.float32)
    out.append(("icosphere4", m, f, 1, 1))  # stress: only the global extrema kept
    # two smooth hills, the lower one discarded: a region above the
    # CTA-flood threshold (256 vertices), then its minima pass
    a, b = np.array([0.0, 0.0, 1.0]), np.array([0.0, 0.0, -1.0])
    f = (np.exp(-((p - a) ** 2).sum(1) / 0.6) + 0.8 * np.exp(-((p - b) ** 2).sum(1) / 0.6)
         + 0.02 * r.random(m.n)).astype(np.float32)
    out.append(("icosphere4_hills", m, f, 1, 1))
    return out


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, mesh, f, kmax, kmin in cases():
        f32 = np.ascontiguousarray(f, np.float32)
        F = O.compute_order_field(O.ScalarField(mesh, f32.astype(np.float64)))
        lo, up = MG.ref_classify(mesh, F.rank)
        mx, mn = np.flatnonzero(up == 0), np.flatnonzero(lo == 0)
        if name == "fig5":  # the paper's example: discard only the maximum of order 22 (vertex T)
            pmax = np.setdiff1d(mx, [19]).astype(np.int64)
            pmin = mn.astype(np.int64)
        else:
            pmax, pmin = MG.S.select_preserved(F.rank, mx, mn, kmax, kmin)
        Fr, G, g, ok, it, first = MG.ref_simplify(mesh, f32, pmax, pmin)
        rec = dict(points=mesh.points, triangles=mesh.triangles, f=f32, pres_max=pmax, pres_min=pmin,
                   F_rank=F.rank.astype(np.int32), lower=lo, upper=up, G_rank=G.astype(np.int32), g=g,
                   ok=np.array(ok), outer=np.array(it), G1=first["G1"].astype(np.int32))
        a = first.get("max")
        if a is not None:
            for key in ("region_ptr", "region_verts", "local", "n_iters", "status", "topseed"):
                rec[f"max_{key}"] = np.asarray(a[key])
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **rec)
        sizes = np.diff(a["region_ptr"]) if a is not None else []
        print(f"{name}: n={mesh.n} maxima={mx.size} minima={mn.size} ok={ok} outer={it} "
              f"largest max-pass region={max(sizes) if len(sizes) else 0}", flush=True)


if __name__ == "__main__":
    main()
