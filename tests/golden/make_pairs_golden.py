"""Golden fixtures for the persistence-driven mode, made by running the
REFERENCE's own numba ``pairs_sweep`` (_kernels.py:309-421) on small seeded
fields.  Build container only (needs /root/reference and numba):

    python tests/golden/make_pairs_golden.py

Seeds = every maximum of the order field (kind "max"), or every minimum with
the sweep run on the reversed order and negated values (kind "min", SPEC
persistence: "identical machinery on the negated comparison order").  Values
are the float32 field widened to float64, as ScalarField does (order.py:30-36).
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from topoflat import _kernels as K  # noqa: E402  (reference, read-only)
from topoflat import order as RO  # noqa: E402
from topoflat import triangulation as T  # noqa: E402

from paper_2009_00083_b200 import synthetic as S  # noqa: E402

OUT = os.path.join(HERE, "pairs")
FRACS = (0.02, 0.1, 0.3)  # epsilon as a fraction of the value range (plus infinity)


def reference_pairs(dims, f32, kind, eps):
    f64 = f32.astype(np.float64)
    tri = T.build_grid_triangulation(tuple(int(d) for d in dims))
    F = RO.compute_order_field(RO.ScalarField(tri, f64))
    rank = np.asarray(F.rank, np.int64)
    n = rank.size
    upper = np.zeros(n, bool)
    lower = np.zeros(n, bool)
    for v in range(n):
        nb = tri.indices[tri.indptr[v]:tri.indptr[v + 1]]
        upper[v] = np.any(rank[nb] > rank[v])
        lower[v] = np.any(rank[nb] < rank[v])
    if kind == "max":
        seeds, r, vals = np.flatnonzero(~upper), rank, f64
    else:
        seeds, r, vals = np.flatnonzero(~lower), n - 1 - rank, -f64
    seeds = np.sort(seeds).astype(np.int64)
    ps, err = K.pairs_sweep(np.ascontiguousarray(r, np.int64), np.ascontiguousarray(vals), tri.indptr,
                            tri.indices, seeds, float(eps))
    return seeds, np.asarray(ps, np.int64), int(err)


CASES = {
    "rand2d_31x23": lambda: np.random.default_rng(1).random((23, 31)).astype(np.float32),
    "quant2d_40": lambda: (np.round(np.random.default_rng(2).random((40, 40)) * 12) / 12).astype(np.float32),
    "rand3d_9x10x11": lambda: np.random.default_rng(3).random((11, 10, 9)).astype(np.float32),
    "cfg1_64": lambda: S.cfg1(0, N=64).astype(np.float32),
    "cfg3_24": lambda: S.cfg3(0, N=24).astype(np.float32),
    "cfg4_96": lambda: S.cfg4(0, N=96, ndisk=12).astype(np.float32),
}


def main():
    os.makedirs(OUT, exist_ok=True)
    for name, make in CASES.items():
        f = make()
        dims = np.asarray(f.shape[::-1], np.int64)
        fr = float(f.max()) - float(f.min())
        eps = np.asarray([np.inf] + [a * fr for a in FRACS], np.float64)
        out = {"dims": dims, "f": f.ravel(), "eps": eps}
        for kind in ("max", "min"):
            for i, e in enumerate(eps):
                seeds, ps, err = reference_pairs(dims, f.ravel(), kind, e)
                assert err == 0
                out[f"{kind}_seeds"] = seeds
                out[f"{kind}_saddle_{i}"] = ps
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
        print(name, dims.tolist(), {k: int((v >= 0).sum()) for k, v in out.items() if "saddle" in k})


if __name__ == "__main__":
    main()
