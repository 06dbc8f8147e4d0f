"""Persistence-driven mode (reference pairs_sweep, _kernels.py:309-421; SPEC
persistence module).  The C oracle's restatement is pinned to fixtures made by
running the reference's own numba pairs_sweep (tests/golden/make_pairs_golden.py);
the GPU pairing (maxima graph -> maximum spanning forest -> Elder-rule sweep)
must reproduce the oracle exactly, extremum by extremum, for every epsilon."""
import glob
import os

import numpy as np
import pytest

from oracle import lts_oracle as O

GOLD = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "pairs", "*.npz")))
IDS = [os.path.basename(p)[:-4] for p in GOLD]


def _load(p):
    z = np.load(p)
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("path", GOLD, ids=IDS)
def test_oracle_pairs_match_reference(path):
    z = _load(path)
    dims = tuple(int(d) for d in z["dims"])
    rank, _ = O.order_field(z["f"])
    vals = z["f"].astype(np.float64)
    for kind in ("max", "min"):
        for i, e in enumerate(z["eps"]):
            seeds, sad, err = O.pairs(dims, rank, vals, kind, e)
            assert err == 0
            np.testing.assert_array_equal(seeds, z[f"{kind}_seeds"])
            np.testing.assert_array_equal(sad, z[f"{kind}_saddle_{i}"])


def _case(path):
    z = _load(path)
    return tuple(int(d) for d in z["dims"]), z["f"], z["eps"]


@pytest.mark.gpu
@pytest.mark.parametrize("path", GOLD, ids=IDS)
def test_gpu_pairs_golden(path):
    import torch

    import paper_2009_00083_b200 as P
    dims, f, eps = _case(path)
    z = _load(path)
    mesh = P.build_grid_triangulation(dims)
    fd = torch.from_numpy(f).cuda()
    for kind in ("max", "min"):
        for i, e in enumerate(eps):
            pr = P.compute_extremum_saddle_pairs(mesh, fd, polarity=kind, epsilon=float(e))
            ext = pr.extrema.cpu().numpy()
            sad = pr.saddles.cpu().numpy()
            np.testing.assert_array_equal(ext, z[f"{kind}_seeds"])
            np.testing.assert_array_equal(sad, z[f"{kind}_saddle_{i}"])


GPU_CASES = {
    "rand2d_300x200": lambda: np.random.default_rng(21).random((200, 300)).astype(np.float32),
    "quant3d_40": lambda: (np.round(np.random.default_rng(22).random((40, 40, 40)) * 30) / 30).astype(np.float32),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(GPU_CASES))
def test_gpu_pairs_vs_oracle(name):
    import torch

    import paper_2009_00083_b200 as P
    f = GPU_CASES[name]()
    dims = f.shape[::-1]
    rank, _ = O.order_field(f.ravel())
    mesh = P.build_grid_triangulation(dims)
    fd = torch.from_numpy(f.ravel()).cuda()
    fr = float(f.max() - f.min())
    for kind in ("max", "min"):
        for e in (float("inf"), 0.05 * fr, 0.25 * fr):
            seeds, sad, err = O.pairs(dims, rank, f.ravel().astype(np.float64), kind, e)
            pr = P.compute_extremum_saddle_pairs(mesh, fd, polarity=kind, epsilon=e)
            np.testing.assert_array_equal(pr.extrema.cpu().numpy(), seeds)
            np.testing.assert_array_equal(pr.saddles.cpu().numpy(), sad)


@pytest.mark.gpu
@pytest.mark.parametrize("frac", [0.0, 0.05, 0.3, 2.0])
def test_gpu_persistence_simplify(frac):
    """discard sets = non-surviving extrema of both
    polarities; the result equals the oracle LTS pass with the oracle's
    survivors preserved, ||f - g||_inf <= epsilon, and epsilon beyond the value
    range leaves exactly one minimum and one maximum."""
    import torch

    import paper_2009_00083_b200 as P
    f = (np.round(np.random.default_rng(31).random((48, 56)) * 64) / 64).astype(np.float32)
    dims = f.shape[::-1]
    fv = f.ravel()
    eps = frac * float(fv.max() - fv.min())
    rank, _ = O.order_field(fv)
    smax, pmax, _ = O.pairs(dims, rank, fv.astype(np.float64), "max", eps)
    smin, pmin, _ = O.pairs(dims, rank, fv.astype(np.float64), "min", eps)
    keep_max, keep_min = smax[pmax < 0], smin[pmin < 0]
    ref = O.simplify(dims, fv, keep_max, keep_min)
    mesh = P.build_grid_triangulation(dims)
    g, G, (qmax, qmin), rep = P.persistence_simplify(mesh, torch.from_numpy(fv).cuda(), eps)
    np.testing.assert_array_equal(qmax.survivors.cpu().numpy(), keep_max)
    np.testing.assert_array_equal(qmin.survivors.cpu().numpy(), keep_min)
    assert rep.ok == ref.ok
    np.testing.assert_array_equal(G.rank32.cpu().numpy(), ref.G_rank)
    assert g.values.cpu().numpy().tobytes() == ref.g.tobytes()
    assert float(np.abs(g.values.cpu().numpy().astype(np.float64) - fv).max()) <= eps
    if frac == 0.0:
        assert np.array_equal(g.values.cpu().numpy(), fv)
    if frac > 1.0:
        mn, mx = P.extrema(mesh, G)
        assert mn.numel() == 1 and mx.numel() == 1


def test_persistence_curve_monotone():
    import types
    import torch

    from paper_2009_00083_b200.persistence import PersistencePairs, persistence_curve
    p = PersistencePairs("max", float("inf"), torch.tensor([1, 2, 3]), torch.tensor([5, 6, -1]),
                         torch.tensor([2.0, 0.5, float("inf")], dtype=torch.float64))
    thr, cnt = persistence_curve(p, value_range=9.0)
    assert thr.tolist() == [0.5, 2.0, 9.0] and cnt.tolist() == [3, 2, 1]
    assert np.all(np.diff(cnt) <= 0)
    thr, cnt = persistence_curve([], None)
    assert thr.size == 0 and cnt.size == 0


@pytest.mark.gpu
@pytest.mark.parametrize("path", GOLD, ids=IDS)
def test_gpu_pairs_global_memory_sweep(path, monkeypatch):
    """The Elder-rule sweep's global-memory branch (taken by fields with more
    than ~56 K forest nodes left after peeling, e.g. cfg2 and cfg4) forced on
    the reference fixtures: same pairs."""
    import torch

    import paper_2009_00083_b200 as P
    monkeypatch.setenv("LTS_PAIRS_FORCE_GLOBAL", "1")
    dims, f, eps = _case(path)
    z = _load(path)
    mesh = P.build_grid_triangulation(dims)
    fd = torch.from_numpy(f).cuda()
    for kind in ("max", "min"):
        for i, e in enumerate(eps):
            pr = P.compute_extremum_saddle_pairs(mesh, fd, polarity=kind, epsilon=float(e))
            np.testing.assert_array_equal(pr.saddles.cpu().numpy(), z[f"{kind}_saddle_{i}"])


FULL_PAIRS = os.path.join(os.path.dirname(__file__), "golden", "full_pairs.json")


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(__import__("json").load(open(FULL_PAIRS))) if os.path.exists(FULL_PAIRS) else [])
def test_gpu_pairs_full_size(key):
    """Full-size cfg1-3 pairings (both polarities, eps = inf and 1 % of the
    range) against the oracle's digests (tools/make_full_pairs.py); cfg2 runs
    the global-memory sweep branch (> 56 K forest nodes)."""
    import hashlib
    import json

    import torch

    import paper_2009_00083_b200 as P
    from paper_2009_00083_b200 import synthetic as S
    rec = json.load(open(FULL_PAIRS))[key]
    f = S.make_field(rec["cfg"], rec["seed"]).ravel()
    mesh = P.build_grid_triangulation(S.CONFIGS[rec["cfg"]].dims)
    fd = torch.from_numpy(f).cuda()
    pr = P.compute_extremum_saddle_pairs(mesh, fd, polarity=rec["kind"], epsilon=float(rec["eps"]))
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a, np.int64).tobytes()).hexdigest()
    assert int(pr.extrema.numel()) == rec["count"]
    assert sha(pr.extrema.cpu().numpy()) == rec["extrema_sha"]
    assert sha(pr.saddles.cpu().numpy()) == rec["saddles_sha"]
