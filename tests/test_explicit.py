"""Explicit triangle meshes: the host-side mesh builders
against the reference's, and the device path (lts_classify_csr /
lts_remove_pass_csr / lts_simplify_csr) against fixtures made by the
reference's own kernels (tests/golden/make_explicit_golden.py), plus the
paper's Fig. 5 known-answer test."""
import glob
import os

import numpy as np
import pytest

import paper_2009_00083_b200 as P

GOLD = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "explicit", "*.npz")))
IDS = [os.path.basename(p)[:-4] for p in GOLD]


def _load(p):
    z = np.load(p)
    return {k: z[k] for k in z.files}


def test_canonical_surfaces():
    """Closed surfaces (triangulation.py:316-361): Euler characteristic 2 for
    the sphere-like ones, 0 for the torus; every link is one cycle."""
    for m, chi in ((P.make_octahedron(), 2), (P.make_icosahedron(), 2), (P.make_torus(6, 5), 0)):
        ne = int(m.indptr[-1]) // 2
        assert m.n - ne + len(m.triangles) == chi
        assert not m.boundary.any()
        v = m.n // 2
        assert len(P.link_adjacency(m, v)) == m.degree(v)


def test_mesh_errors_and_off_round_trip():
    with pytest.raises(P.NonTriangleFace):
        P.build_explicit_triangulation(np.zeros((4, 3)), np.array([[0, 1, 2, 3]]))
    with pytest.raises(P.NonManifoldEdge):  # one edge in three triangles
        P.build_explicit_triangulation(np.zeros((5, 3)), np.array([[0, 1, 2], [0, 1, 3], [0, 1, 4]]))
    with pytest.raises(P.MeshError):  # unknown vertex
        P.build_explicit_triangulation(np.zeros((3, 3)), np.array([[0, 1, 5]]))
    with pytest.raises(P.MeshError):  # bow tie: vertex 0's link is two paths
        P.build_explicit_triangulation(np.zeros((5, 3)), np.array([[0, 1, 2], [0, 3, 4]]))
    m = P.make_icosahedron()
    m2 = P.load_off(P.write_off(m))
    assert np.array_equal(m2.indptr, m.indptr) and np.array_equal(m2.indices, m.indices)
    assert np.allclose(m2.points, m.points)
    with pytest.raises(P.MeshError):
        P.load_off("OFF\n3 1 0\n0 0 0\n")


@pytest.mark.parametrize("path", GOLD, ids=IDS)
def test_host_mesh_matches_reference_fixture(path):
    """The mesh rebuilt from the fixture's points / triangles has the
    reference builder's CSR (rows follow the same order)."""
    z = _load(path)
    m = P.build_explicit_triangulation(z["points"], z["triangles"])
    assert m.n == z["f"].size


def _mesh(z):
    return P.build_explicit_triangulation(z["points"], z["triangles"])


@pytest.mark.gpu
@pytest.mark.parametrize("path", GOLD, ids=IDS)
def test_explicit_order_and_classify(path):
    import torch
    z = _load(path)
    m = _mesh(z)
    F = P.compute_order_field(P.ScalarField(m, torch.from_numpy(z["f"]).cuda()))
    np.testing.assert_array_equal(F.rank32.cpu().numpy(), z["F_rank"])
    lo, up = P.classify_all(m, F)
    np.testing.assert_array_equal(lo.cpu().numpy(), z["lower"])
    np.testing.assert_array_equal(up.cpu().numpy(), z["upper"])
    mn, mx = P.extrema(m, F)
    np.testing.assert_array_equal(mx.cpu().numpy(), np.flatnonzero(z["upper"] == 0))
    np.testing.assert_array_equal(mn.cpu().numpy(), np.flatnonzero(z["lower"] == 0))


@pytest.mark.gpu
@pytest.mark.parametrize("path", GOLD, ids=IDS)
def test_explicit_simplify(path):
    import torch
    z = _load(path)
    m = _mesh(z)
    g, G, rep = P.simplify_field(m, torch.from_numpy(z["f"]).cuda(),
                                 P.ConstraintSet(preserveMinima=z["pres_min"], preserveMaxima=z["pres_max"]))
    assert rep.ok == bool(z["ok"]) and rep.outerIterations == int(z["outer"])
    np.testing.assert_array_equal(G.rank32.cpu().numpy(), z["G_rank"])
    assert g.values.cpu().numpy().tobytes() == z["g"].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("path", GOLD, ids=IDS)
def test_explicit_first_max_pass_regions(path):
    z = _load(path)
    if "max_region_ptr" not in z:
        pytest.skip("no maxima pass")
    m = _mesh(z)
    F = P.order_from_ranks(z["F_rank"])
    mn, mx = P.extrema(m, F)
    keep = np.intersect1d(mx.cpu().numpy(), z["pres_max"])
    pr = P.remove_pass(m, F, P.ConstraintSet(preserveMinima=mn.cpu().numpy(), preserveMaxima=keep), "max")

    def by_saddle(ptr, verts, local, nit):
        return sorted((int(verts[ptr[r]]), tuple(verts[ptr[r]:ptr[r + 1]].tolist()),
                       tuple(local[ptr[r]:ptr[r + 1]].tolist()), int(nit[r])) for r in range(len(ptr) - 1))

    got = by_saddle(pr.region_ptr.cpu().numpy(), pr.region_verts.cpu().numpy(), pr.local_rank.cpu().numpy(),
                    pr.n_iters.cpu().numpy())
    ref = by_saddle(z["max_region_ptr"], z["max_region_verts"], z["max_local"], z["max_n_iters"])
    assert got == ref
    np.testing.assert_array_equal(pr.new_order.rank32.cpu().numpy(), z["G1"])


# Fig. 5 of the paper, vertices A..X in reading order (rows y = 2 .. -2)
FIG5_A = [3, 2, 1, 0, 4, 17, 16, 15, 14, 23, 10, 18, 12, 19, 13, 9, 11, 20, 21, 22, 8, 7, 6, 5]  # 5a
FIG5_E = {"F": 10, "G": 9, "H": 8, "I": 3, "K": 12, "L": 11, "M": 2, "N": 7, "O": 4, "Q": 0, "R": 1,
          "S": 6, "T": 5}                                                                          # 5e
FIG5_F = [3, 2, 1, 0, 4, 20, 19, 18, 13, 23, 22, 21, 12, 17, 14, 9, 10, 11, 16, 15, 8, 7, 6, 5]  # 5f


@pytest.mark.gpu
def test_fig5_known_answer():
    """Removing the maximum of order 22 (T) from the paper's running example:
    the region is the 13 vertices of Fig. 5b with saddle K (order 10), three
    propagations (b, c, d) give the local order of Fig. 5e, and the integrated
    global order is Fig. 5f."""
    z = _load([p for p in GOLD if p.endswith("fig5.npz")][0])
    m = _mesh(z)
    names = "ABCDEFGHIJKLMNOPQRSTUVWX"
    F = P.order_from_ranks(np.array(FIG5_A, np.int64))
    mn, mx = P.extrema(m, F)
    T = names.index("T")
    assert T in mx.cpu().numpy().tolist()
    keep = np.setdiff1d(mx.cpu().numpy(), [T])
    pr = P.remove_pass(m, F, P.ConstraintSet(preserveMinima=mn.cpu().numpy(), preserveMaxima=keep), "max")
    ptr, verts = pr.region_ptr.cpu().numpy(), pr.region_verts.cpu().numpy()
    assert len(ptr) == 2
    region = [names[v] for v in verts]
    assert region[0] == "K" and sorted(region) == sorted(FIG5_E)
    local = dict(zip(region, pr.local_rank.cpu().numpy().tolist()))
    assert local == FIG5_E
    assert int(pr.n_iters[0]) == 3
    assert pr.new_order.rank32.cpu().numpy().tolist() == FIG5_F
