"""Timing of the persistence-driven mode on a BASELINE config (GPU pairs of
both polarities at epsilon = inf and 1% of the range, persistence_simplify at
1%), next to the CPU oracle's pairs_sweep on the same field.
Usage: python tools/pairs_bench.py [cfg] [--no-cpu]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_00083_b200 as P  # noqa: E402
from paper_2009_00083_b200 import synthetic as S  # noqa: E402

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = S.CONFIGS[cfgn]
f = S.make_field(cfgn, 0).ravel().astype(np.float32)
mesh = P.build_grid_triangulation(cfg.dims)
fd = torch.from_numpy(f).cuda()
F = P.compute_order_field(P.ScalarField(mesh, fd))
eps1 = 0.01 * float(f.max() - f.min())


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t) * 1e3)
    return min(ts), r


for kind in ("max", "min"):
    for eps in (float("inf"), eps1):
        ms, pp = timed(lambda: P.compute_extremum_saddle_pairs(mesh, fd, F, kind, eps))
        print(f"cfg{cfgn} pairs {kind} eps={eps:.4g}: {ms:.2f} ms, {pp.extrema.numel()} extrema, "
              f"{int((pp.saddles >= 0).sum())} pairs")
ms, (g, G, (a, b), rep) = timed(lambda: P.persistence_simplify(mesh, fd, eps1))
print(f"cfg{cfgn} persistence_simplify eps=1%: {ms:.2f} ms (ok={rep.ok}, survivors {a.survivors.numel()} max "
      f"/ {b.survivors.numel()} min, regions {rep.regionCount})")
if "--no-cpu" not in sys.argv:
    from oracle import lts_oracle as O
    rank = F.rank32.cpu().numpy()
    t = time.perf_counter()
    O.pairs(cfg.dims, rank, f.astype(np.float64), "max", eps1)
    print(f"cfg{cfgn} CPU oracle pairs_sweep max eps=1%: {(time.perf_counter() - t) * 1e3:.1f} ms (1 core)")
