"""GPU tests of the public entry points and the boundary semantics of the
drop-in (reference order.py / critical.py, SPEC.md lts-engine): every call
goes through liblts_sm100.so and is checked against the pinned oracle or the
reference-made fixtures."""
import glob
import os

import numpy as np
import pytest
import torch

import paper_2009_00083_b200 as P
from oracle import lts_oracle as O
from paper_2009_00083_b200 import synthetic as S

pytestmark = pytest.mark.gpu
GOLD = {os.path.basename(p)[:-4]: p for p in sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))}


def _load(name):
    z = np.load(GOLD[name])
    return {k: z[k] for k in z.files}


def _cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _mesh(dims):
    return P.build_grid_triangulation(tuple(int(d) for d in dims))


@pytest.mark.parametrize("name", ["cfg1_64", "gauss3d_22x18x20", "stress3d_12x10x11", "zeros2d_24x24"])
def test_extract_critical_points_and_classify_vertex(name):
    """critical.py:115-121 on the device counts vs the reference's
    classify_grid counts (fixtures made by the reference's own kernels)."""
    z = _load(name)
    mesh = _mesh(z["dims"])
    F = P.order_from_ranks(z["F_rank"])
    cs = P.extract_critical_points(mesh, F)
    lo, up = z["lower"], z["upper"]
    np.testing.assert_array_equal(cs.minima.cpu().numpy(), np.flatnonzero(lo == 0))
    np.testing.assert_array_equal(cs.maxima.cpu().numpy(), np.flatnonzero(up == 0))
    sad = np.flatnonzero((lo > 0) & (up > 0) & ((lo > 1) | (up > 1)))
    np.testing.assert_array_equal(cs.saddles.cpu().numpy(), sad)
    kinds = cs.kinds().cpu().numpy()
    rng = np.random.default_rng(0)
    for v in rng.choice(mesh.n, 12, replace=False).tolist() + [int(sad[0])] if sad.size else []:
        c = P.classify_vertex(mesh, F, int(v))
        assert (c.lower_components, c.upper_components) == (int(lo[v]), int(up[v]))
        expect = {1: P.Kind.MINIMUM, 2: P.Kind.MAXIMUM, 3: P.Kind.SADDLE, 0: P.Kind.REGULAR}[int(kinds[v])]
        assert c.kind is expect
    with pytest.raises(P.MeshError):
        P.classify_vertex(mesh, F, mesh.n)


@pytest.mark.parametrize("name", ["cfg1_64", "stress3d_12x10x11", "rand2d_33x29_s0"])
def test_discover_regions_matches_reference_first_pass(name):
    """SPEC.md:311-320 black-list form: discard = maxima of F minus the
    preserved ones -> the reference sweep's regions (fixture)."""
    z = _load(name)
    if "max_region_ptr" not in z:
        pytest.skip("no maxima pass in this fixture")
    mesh = _mesh(z["dims"])
    F = P.order_from_ranks(z["F_rank"])
    mn, mx = O.extrema(tuple(z["dims"]), z["F_rank"])
    discard = np.setdiff1d(mx, z["pres_max"])
    pr = P.discover_regions(mesh, F, discard)
    ptr, verts = pr.region_ptr.cpu().numpy(), pr.region_verts.cpu().numpy()
    got = sorted((int(verts[ptr[r]]), tuple(sorted(verts[ptr[r] + 1:ptr[r + 1]].tolist())))
                 for r in range(len(ptr) - 1))
    rp, rv = z["max_region_ptr"], z["max_region_verts"]
    ref = sorted((int(rv[rp[r]]), tuple(sorted(rv[rp[r] + 1:rp[r + 1]].tolist()))) for r in range(len(rp) - 1))
    assert got == ref
    with pytest.raises(P.ConstraintNotExtremum):
        P.discover_regions(mesh, F, [int(mn[0])] if not np.isin(mn[0], mx) else [])


@pytest.mark.parametrize("name", ["cfg1_64", "stress3d_12x10x11", "quant2d_40_s0"])
def test_remove_extrema_matches_simplify_order(name):
    """remove_extrema(F, discard) with discard = extrema
    minus the preserve sets gives simplify_field's G (orders only, no g)."""
    z = _load(name)
    mesh = _mesh(z["dims"])
    F = P.order_from_ranks(z["F_rank"])
    mn, mx = O.extrema(tuple(z["dims"]), z["F_rank"])
    G, rep = P.remove_extrema(mesh, F, np.setdiff1d(mx, z["pres_max"]), np.setdiff1d(mn, z["pres_min"]))
    assert rep.ok == bool(z["ok"])
    np.testing.assert_array_equal(G.rank32.cpu().numpy(), z["G_rank"])
    # discard nothing -> G = F, no regions (SPEC example)
    G0, rep0 = P.remove_extrema(mesh, F, [], [])
    assert torch.equal(G0.rank32, F.rank32) and rep0.regionCount == 0


def test_remove_extrema_discard_everything_but_global():
    """The paper's stress case: discard every non-global extremum."""
    f = np.random.default_rng(3).random((40, 50)).astype(np.float32)
    dims = (50, 40)
    mesh = _mesh(dims)
    rank, _ = O.order_field(f.ravel())
    mn, mx = O.extrema(dims, rank)
    gmax, gmin = int(np.argmax(rank)), int(np.argmin(rank))
    G, rep = P.remove_extrema(mesh, P.order_from_ranks(rank), np.setdiff1d(mx, [gmax]), np.setdiff1d(mn, [gmin]))
    ref = O.simplify(dims, f.ravel(), [gmax], [gmin])
    np.testing.assert_array_equal(G.rank32.cpu().numpy(), ref.G_rank)
    mn2, mx2 = P.extrema(mesh, G)
    assert mn2.tolist() == [gmin] and mx2.tolist() == [gmax]


def test_field_errors_at_construction_and_with_order():
    """ScalarField rejects NaN/inf at construction (order.py:35-36), and so does
    simplify_field(order=F) (the finiteness check runs even when the caller
    brings the order field)."""
    mesh = _mesh((8, 6))
    f = np.random.default_rng(1).random(48).astype(np.float32)
    F = P.compute_order_field(P.ScalarField(mesh, _cu(f)))
    for bad in (np.nan, np.inf, -np.inf):
        fb = f.copy()
        fb[17] = bad
        with pytest.raises(P.FieldError):
            P.ScalarField(mesh, _cu(fb))
        with pytest.raises(P.FieldError):
            P.simplify_raw(mesh, _cu(fb), torch.empty(0, dtype=torch.int64, device="cuda"),
                           torch.empty(0, dtype=torch.int64, device="cuda"), F.rank32)
    # an order that is not a permutation is refused
    bad_order = F.rank32.clone()
    bad_order[3] = bad_order[4]
    with pytest.raises(P.LTSNativeError):
        P.simplify_raw(mesh, _cu(f), torch.empty(0, dtype=torch.int64, device="cuda"),
                       torch.empty(0, dtype=torch.int64, device="cuda"), bad_order)


def test_float64_input():
    """The reference keeps float64 (order.py:31); float64 input that is exactly
    float32 is accepted and gives the float32 result, anything else raises."""
    mesh = _mesh((9, 7))
    f32 = np.random.default_rng(2).random(63).astype(np.float32)
    a = P.ScalarField(mesh, f32.astype(np.float64))
    b = P.ScalarField(mesh, f32)
    assert torch.equal(a.values, b.values)
    assert torch.equal(P.ScalarField(mesh, _cu(f32.astype(np.float64))).values, b.values)
    with pytest.raises(P.FieldError):
        P.ScalarField(mesh, f32.astype(np.float64) + 1e-12)


def test_misaligned_view_input():
    """A view with a storage offset (not 16-byte aligned) goes through the
    vectorised sort histogram correctly."""
    rng = np.random.default_rng(4)
    base = torch.from_numpy(rng.random(4097 * 1 + 64 * 64).astype(np.float32)).cuda()
    for off in (1, 2, 3, 5):
        x = base[off:off + 64 * 64]
        assert x.data_ptr() % 16 != 0
        mesh = _mesh((64, 64))
        F = P.compute_order_field(P.ScalarField(mesh, x))
        rank, _ = O.order_field(x.cpu().numpy())
        np.testing.assert_array_equal(F.rank32.cpu().numpy(), rank)
        _, Gf, _ = P.simplify_field(mesh, x, P.ConstraintSet())
        ref = O.simplify((64, 64), x.cpu().numpy(), [], [])
        np.testing.assert_array_equal(Gf.rank32.cpu().numpy(), ref.G_rank)


def _realize_sweep64(g, inverse, zeta):
    """_kernels.py:84-99, literal, in float64 (test restatement)."""
    g = g.copy()
    n = inverse.size
    prev = inverse[n - 1]
    for i in range(n - 2, -1, -1):
        v = inverse[i]
        if g[v] > g[prev] or (g[v] == g[prev] and v > prev):
            nv = g[prev] - zeta
            if nv >= g[prev]:
                nv = np.nextafter(g[prev], -np.inf)
            g[v] = nv
        prev = v
    return g


@pytest.mark.parametrize("mode", ["relative", "ulp"])
def test_realize_numeric_literal(mode):
    """realize_numeric (order.py:102-116) on the device equals the literal
    float64 sweep; simplify_field(options.zeta=...) returns it."""
    rng = np.random.default_rng(9)
    f = (np.round(rng.random((30, 40)) * 50) / 50).astype(np.float32)
    dims = (40, 30)
    mesh = _mesh(dims)
    zeta = P.ZetaPolicy() if mode == "relative" else P.ZetaPolicy(P.ZetaMode.ULP_DECREMENT)
    rank, _ = O.order_field(f.ravel())
    mn, mx = O.extrema(dims, rank)
    pm, pn = S.select_preserved(rank, mx, mn, 3, 2)
    g, G, rep = P.simplify_field(mesh, f.ravel(), P.ConstraintSet(preserveMinima=pn, preserveMaxima=pm),
                                 P.SimplifyOptions(zeta=zeta))
    assert g.values.dtype == torch.float64
    Gn = G.rank32.cpu().numpy()
    inv = np.empty_like(Gn)
    inv[Gn] = np.arange(Gn.size, dtype=Gn.dtype)
    step = zeta.step(float(f.max() - f.min()))
    ref = _realize_sweep64(f.ravel().astype(np.float64), inv, step)
    assert g.values.cpu().numpy().tobytes() == ref.tobytes()
    # realize(f, order(f)) == f exactly (order.py:108-110)
    F = P.compute_order_field(P.ScalarField(mesh, f.ravel()))
    same = P.realize_numeric(P.ScalarField(mesh, f.ravel()), F, zeta)
    assert np.array_equal(same.values.cpu().numpy(), f.ravel().astype(np.float64))


@pytest.mark.parametrize("name", ["cfg1_512", "cfg3_96"])
def test_report_per_region_ni_and_distance_bound(name):
    """SimplifyReport carries every region's N_I, equal to
    the oracle's; ||f-g||_inf stays within the largest region height
    (f(m_top) - f(s) over the maxima-pass regions, and the mirrored
    depth over the minima-pass regions)."""
    f = S.cfg1(0) if name == "cfg1_512" else S.cfg3(0, N=96)
    kmax, kmin = (16, 1) if name == "cfg1_512" else (30, 30)
    dims = tuple(f.shape[::-1])
    f32 = np.ascontiguousarray(f.ravel(), np.float32)
    rank, _ = O.order_field(f32)
    mn, mx = O.extrema(dims, rank)
    pm, pn = S.select_preserved(rank, mx, mn, kmax, kmin)
    ref = O.simplify(dims, f32, pm, pn)
    mesh = _mesh(dims)
    g, G, rep = P.simplify_field(mesh, _cu(f32), P.ConstraintSet(preserveMinima=pn, preserveMaxima=pm))
    assert len(rep.regionNI) == len(ref.passes)
    assert ref.outer_iterations == 1
    # hill heights in f (maxima pass), pit depths in g1 = f flattened by the
    # maxima pass (contract D1): a vertex in both moves by at most the larger
    bound = 0.0
    gcur = f32.astype(np.float64)
    for got, p in zip(rep.regionNI, ref.passes):
        if p.regions == 0:
            continue
        # region order differs (device: region index; oracle: root order):
        # compare the multisets and the maximum
        assert sorted(got.cpu().numpy().tolist()) == sorted(p.n_iters.tolist())
        assert int(got.max()) == p.n_iter_max
        nxt = gcur.copy()
        for r in range(len(p.region_ptr) - 1):
            seg = p.region_verts[p.region_ptr[r]:p.region_ptr[r + 1]]
            if p.kind == "max":
                bound = max(bound, float(gcur[seg].max() - gcur[seg[0]]))
            else:
                bound = max(bound, float(gcur[seg[0]] - gcur[seg].min()))
            nxt[seg[1:]] = gcur[seg[0]]
        gcur = nxt
    assert rep.maxNI == max(p.n_iter_max for p in ref.passes)
    assert rep.linf <= bound
    assert rep.linf == float(np.abs(g.values.cpu().numpy().astype(np.float64) - f32.astype(np.float64)).max())


def test_simplify_field_host_matches_device_call_and_oracle():
    """lts_simplify_host: host buffers in, host buffers out (g copied out beside
    the last pass's floods), same bits as the device-tensor call and the oracle;
    covers an outer loop > 1 (g copied again) and a pass without regions."""
    import glob
    import os
    gold = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))
    picks = [p for p in gold if any(t in p for t in ("quant2d_40", "cfg3_48", "const2d", "crater", "rand3d"))][:6]
    assert picks
    for path in picks:
        z = np.load(path)
        dims = tuple(int(d) for d in z["dims"])
        mesh = P.build_grid_triangulation(dims)
        f_host = torch.from_numpy(np.ascontiguousarray(z["f"], np.float32)).pin_memory()
        g, G, rep = P.simplify_field_host(mesh, f_host, P.ConstraintSet(preserveMinima=z["pres_min"],
                                                                        preserveMaxima=z["pres_max"]))
        assert g.device.type == "cpu" and G.device.type == "cpu"
        assert rep.ok == bool(z["ok"]) and rep.outerIterations == int(z["outer"])
        np.testing.assert_array_equal(G.numpy(), z["G_rank"])
        assert g.numpy().tobytes() == z["g"].tobytes()


def test_simplify_field_host_errors():
    mesh = P.build_grid_triangulation((16, 12))
    f = torch.rand(16 * 12, dtype=torch.float32)
    f[5] = float("nan")
    with pytest.raises(P.FieldError):
        P.simplify_field_host(mesh, f.pin_memory(), P.ConstraintSet(preserveMinima=[], preserveMaxima=[]))
    with pytest.raises(P.FieldError):
        P.simplify_field_host(mesh, torch.rand(7), P.ConstraintSet(preserveMinima=[], preserveMaxima=[]))
