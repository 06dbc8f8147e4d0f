"""Randomised parity sweep of the level-parallel floods (csrc/localize_level.cuh).

Every large region is forced onto the level path and the full pass is compared
bit for bit with the CPU oracle over many small random fields: white noise
(rough regions, shallow level trees), quantised noise (ties broken by vertex
id), noise on a hill (climbing floods with long prefixes), 2-D and 3-D, with
few preserved extrema so regions are large and floods repeat (N_I > 1)."""
import numpy as np
import pytest
import torch

import paper_2009_00083_b200 as P
from oracle import lts_oracle as O
from paper_2009_00083_b200 import synthetic as S

pytestmark = pytest.mark.gpu


def _field(kind, shape, rng):
    if kind == "noise":
        return rng.random(shape)
    if kind == "quant":
        return np.round(rng.random(shape) * 9) / 9
    if kind == "hill":
        ax = np.indices(shape).astype(np.float64)
        r2 = sum(((a - (s - 1) / 2) / (0.35 * s)) ** 2 for a, s in zip(ax, shape))
        return np.exp(-r2) + 0.12 * rng.random(shape)
    raise ValueError(kind)


CASES = [(kind, shape, seed)
         for kind in ("noise", "quant", "hill")
         for shape in ((48, 56), (72, 40), (14, 18, 16), (10, 24, 20))
         for seed in (11, 12)]


@pytest.mark.parametrize("kind,shape,seed", CASES, ids=lambda v: "x".join(map(str, v)) if isinstance(v, tuple) else str(v))
def test_level_floods_random_fields(kind, shape, seed, monkeypatch):
    monkeypatch.setenv("LTS_LEVEL_MIN", "0")
    monkeypatch.setenv("LTS_LEVEL_RATIO", "1000000")
    rng = np.random.default_rng(seed)
    f32 = np.ascontiguousarray(_field(kind, shape, rng).ravel(), np.float32)
    dims = tuple(shape[::-1])
    rank, _ = O.order_field(f32)
    mn, mx = O.extrema(dims, rank)
    pm, pn = S.select_preserved(rank, mx, mn, 1 + seed % 3, 1 + seed % 2)
    ref = O.simplify(dims, f32, pm, pn)
    mesh = P.build_grid_triangulation(dims)
    g, G, rep = P.simplify_field(mesh, torch.from_numpy(f32).cuda(),
                                 P.ConstraintSet(preserveMinima=pn, preserveMaxima=pm))
    assert rep.ok == ref.ok and rep.outerIterations == ref.outer_iterations
    np.testing.assert_array_equal(G.rank32.cpu().numpy(), ref.G_rank)
    assert g.values.cpu().numpy().tobytes() == ref.g.tobytes()
    for a, b in zip(rep.passes, ref.passes):
        assert (a.regions, a.claimed, a.n_iter_max, a.capped) == (b.regions, b.claimed, b.n_iter_max, b.capped)
