"""One-off randomised sweep of the flood paths against the CPU oracle.

    python tools/stress_level.py [first_seed] [n_seeds]

For every seed: 2-D and 3-D fields of three kinds (white noise, quantised
noise with ties, noise on a hill), random shapes and preserve counts, with every
large region forced level-parallel, then with the default policy.  Prints one
line per mismatch and a summary; exit code 1 on any mismatch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_00083_b200 as P  # noqa: E402
from oracle import lts_oracle as O  # noqa: E402
from paper_2009_00083_b200 import synthetic as S  # noqa: E402

first = int(sys.argv[1]) if len(sys.argv) > 1 else 100
count = int(sys.argv[2]) if len(sys.argv) > 2 else 40


def field(kind, shape, rng):
    if kind == "noise":
        return rng.random(shape)
    if kind == "quant":
        return np.round(rng.random(shape) * rng.integers(4, 30)) / 7
    ax = np.indices(shape).astype(np.float64)
    r2 = sum(((a - (s - 1) / 2) / (0.35 * s)) ** 2 for a, s in zip(ax, shape))
    return np.exp(-r2) + rng.uniform(0.02, 0.3) * rng.random(shape)


bad = total = big = 0
for seed in range(first, first + count):
    rng = np.random.default_rng(seed)
    for kind in ("noise", "quant", "hill"):
        nd = int(rng.integers(2, 4))
        shape = tuple(int(x) for x in (rng.integers(20, 90, 2) if nd == 2 else rng.integers(8, 28, 3)))
        f32 = np.ascontiguousarray(field(kind, shape, rng).ravel(), np.float32)
        dims = tuple(shape[::-1])
        rank, _ = O.order_field(f32)
        mn, mx = O.extrema(dims, rank)
        pm, pn = S.select_preserved(rank, mx, mn, int(rng.integers(1, 6)), int(rng.integers(1, 4)))
        ref = O.simplify(dims, f32, pm, pn)
        mesh = P.build_grid_triangulation(dims)
        for mode in ("level", "default"):
            if mode == "level":
                os.environ["LTS_LEVEL_MIN"] = "0"
                os.environ["LTS_LEVEL_RATIO"] = "1000000"
            else:
                os.environ.pop("LTS_LEVEL_MIN", None)
                os.environ.pop("LTS_LEVEL_RATIO", None)
            g, G, rep = P.simplify_field(mesh, torch.from_numpy(f32).cuda(),
                                         P.ConstraintSet(preserveMinima=pn, preserveMaxima=pm))
            ok = (rep.ok == ref.ok and np.array_equal(G.rank32.cpu().numpy(), ref.G_rank)
                  and g.values.cpu().numpy().tobytes() == ref.g.tobytes())
            total += 1
            big += rep.largestRegion > 256
            if not ok:
                bad += 1
                print("MISMATCH", seed, kind, shape, mode, flush=True)
print(f"cases {total} (largest region > 256 slots in {big}) mismatches {bad}")
sys.exit(1 if bad else 0)
