"""Full-size parity on the five BASELINE configs (seed 0).

The CPU oracle (oracle/, pinned to the reference kernels by
test_oracle_golden.py) was run once on each full-size field by
tools/make_full_hashes.py; its SHA-256 digests of the inputs, the preserve
lists and the outputs (G int32 ranks, g float32) are committed in
tests/golden/full_hashes.json.  Here the GPU path regenerates each field with
the same seeded generator (seed 0 for all configs, seeds 1 and 2 for cfg1-3),
selects the preserve lists with its own
classification + order field, and must reproduce every digest bit for bit.
Size-independent properties are checked as well: G is a permutation, the
extremum set of G equals the requested set, g takes only input values."""
import hashlib
import json
import os

import numpy as np
import pytest
import torch

import paper_2009_00083_b200 as P
from paper_2009_00083_b200 import synthetic as S

pytestmark = pytest.mark.gpu
HASHES = os.path.join(os.path.dirname(__file__), "golden", "full_hashes.json")
DATA = json.load(open(HASHES)) if os.path.exists(HASHES) else {}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _key_cfg_seed(key):
    c, _, s = key.partition("_s")
    return int(c), int(s or 0)


@pytest.mark.parametrize("key", sorted(DATA, key=lambda k: _key_cfg_seed(k)[::-1]))
def test_full_config_bit_exact(key):
    """Seed 0 of all five configs and seeds 1, 2 of cfg1-3."""
    ref = DATA[key]
    cfg, seed = _key_cfg_seed(key)
    C = S.CONFIGS[cfg]
    f = S.make_field(cfg, seed).ravel()
    assert sha(f) == ref["f_sha"], "generator drifted"
    mesh = P.build_grid_triangulation(C.dims)
    fd = torch.from_numpy(f).cuda()
    F = P.compute_order_field(P.ScalarField(mesh, fd))
    assert sha(F.rank32.cpu().numpy()) == ref["F_sha"]
    mn, mx = P.extrema(mesh, F)
    assert (mx.numel(), mn.numel()) == (ref["maxima"], ref["minima"])
    pm, pn = S.select_preserved(F.rank32.cpu().numpy(), mx.cpu().numpy(), mn.cpu().numpy(),
                                C.n_keep_max, C.n_keep_min)
    assert sha(pm) == ref["pres_max_sha"] and sha(pn) == ref["pres_min_sha"]
    g, G, rep = P.simplify_field(mesh, fd, P.ConstraintSet(preserveMinima=pn, preserveMaxima=pm),
                                 order=F)
    assert rep.ok == ref["ok"]
    assert rep.outerIterations == ref["outer"]
    for a, b in zip(rep.passes, ref["passes"]):
        assert (a.regions, a.claimed, a.largest, a.n_iter_max, a.capped) == \
            (b["regions"], b["claimed"], b["largest"], b["n_iter_max"], b["capped"])
    Gn = G.rank32.cpu().numpy()
    gn = g.values.cpu().numpy()
    assert sha(Gn) == ref["G_sha"]
    assert sha(gn) == ref["g_sha"]
    # size-independent properties
    assert np.array_equal(np.sort(Gn), np.arange(mesh.n, dtype=np.int32))
    v = P.verify_constraints(mesh, G, P.ConstraintSet(preserveMinima=pn, preserveMaxima=pm))
    assert v.ok
    fz = np.where(f == 0, np.float32(0), f)
    assert np.all(np.isin(gn, fz))
    # g realises G (non-decreasing along G's order) and never moves a value
    # past the range of f
    inv = np.empty_like(Gn)
    inv[Gn] = np.arange(mesh.n, dtype=np.int32)
    assert np.all(np.diff(gn[inv]) >= 0)
    assert gn.min() >= fz.min() and gn.max() <= fz.max()


@pytest.mark.parametrize("cfg", [c for c in (1, 3) if str(c) in DATA])
def test_full_config_determinism_and_idempotence(cfg):
    """Two runs are bit-identical (parallel schedule independence);
    simplifying g again with the same constraints and order G changes nothing
    (idempotence); vertices whose rank did not move keep f."""
    C = S.CONFIGS[cfg]
    f = S.make_field(cfg, 0).ravel()
    mesh = P.build_grid_triangulation(C.dims)
    fd = torch.from_numpy(f).cuda()
    F = P.compute_order_field(P.ScalarField(mesh, fd))
    mn, mx = P.extrema(mesh, F)
    pm, pn = S.select_preserved(F.rank32.cpu().numpy(), mx.cpu().numpy(), mn.cpu().numpy(),
                                C.n_keep_max, C.n_keep_min)
    cs = P.ConstraintSet(preserveMinima=pn, preserveMaxima=pm)
    g1, G1, _ = P.simplify_field(mesh, fd, cs, order=F)
    g2, G2, _ = P.simplify_field(mesh, fd, cs, order=F)
    assert torch.equal(G1.rank32, G2.rank32) and torch.equal(g1.values, g2.values)
    g3, G3, rep3 = P.simplify_field(mesh, g1.values.clone(), cs, order=G1)
    assert rep3.ok and rep3.regionCount == 0
    assert torch.equal(G3.rank32, G1.rank32) and torch.equal(g3.values, g1.values)
    # locality: vertices outside every region keep f and their
    # relative order.  A vertex whose float32 value is unique in f and unchanged
    # in g is outside every region or a region's saddle (region vertices take
    # another vertex's value), and saddles keep their place too.  (cfg3 has
    # many exact float32 ties, so "unchanged" alone would admit region
    # vertices tied with their saddle.)
    fz = torch.where(fd == 0, torch.zeros_like(fd), fd)
    _, inv_u, cnt = torch.unique(fz, return_inverse=True, return_counts=True)
    same = (g1.values == fz) & (cnt[inv_u] == 1)
    Fr, Gr = F.rank32[same], G1.rank32[same]
    assert torch.equal(torch.argsort(Fr), torch.argsort(Gr))
