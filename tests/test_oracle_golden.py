"""Pin the CPU oracle (oracle/) against fixtures produced by running the
reference's own numba kernels (tests/golden/make_golden.py)."""
import glob
import os

import numpy as np
import pytest

from oracle import lts_oracle as O

GOLD = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def _load(p):
    z = np.load(p)
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("path", GOLD, ids=[os.path.basename(p)[:-4] for p in GOLD])
def test_oracle_matches_reference(path):
    z = _load(path)
    dims = tuple(int(d) for d in z["dims"])
    rank, inv = O.order_field(z["f"])
    np.testing.assert_array_equal(rank, z["F_rank"])
    np.testing.assert_array_equal(inv, O.inverse_of(rank))
    lo, up = O.classify(dims, rank)
    np.testing.assert_array_equal(lo, z["lower"])
    np.testing.assert_array_equal(up, z["upper"])
    res = O.simplify(dims, z["f"], z["pres_max"], z["pres_min"])
    assert res.ok == bool(z["ok"])
    assert res.outer_iterations == int(z["outer"])
    np.testing.assert_array_equal(res.G_rank, z["G_rank"])
    assert res.g.tobytes() == z["g"].tobytes()
    # first max pass artefacts (discover -> assemble -> localize)
    if "max_region_ptr" in z:
        p = res.passes[0]
        np.testing.assert_array_equal(p.region_ptr, z["max_region_ptr"])
        np.testing.assert_array_equal(p.region_verts, z["max_region_verts"])
        np.testing.assert_array_equal(p.local, z["max_local"])
        np.testing.assert_array_equal(p.n_iters, z["max_n_iters"])
        np.testing.assert_array_equal(p.topseed, z["max_topseed"])


def test_link_tables_match_reference_counts():
    offs2, pairs2 = O.grid_tables(2)
    offs3, pairs3 = O.grid_tables(3)
    assert offs2.shape == (6, 2) and offs3.shape == (14, 3)
    assert len(pairs2) == 13 and len(pairs3) == 73  # SURVEY F3 (over-connected)
