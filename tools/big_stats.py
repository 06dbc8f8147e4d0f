"""Per-region counters of the CTA flood kernel (lts_debug_big_stats) for one
pass of a BASELINE config: steps, global-rule commits, flood cycles.

    python tools/big_stats.py CFG [max|min]
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2009_00083_b200 as P  # noqa: E402
from paper_2009_00083_b200 import _native as N, synthetic as S  # noqa: E402

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 3
kind = sys.argv[2] if len(sys.argv) > 2 else "max"
cfg = S.CONFIGS[cfgn]
f = torch.from_numpy(S.make_field(cfgn, 0).ravel()).cuda()
mesh = P.build_grid_triangulation(cfg.dims)
F = P.compute_order_field(P.ScalarField(mesh, f))
mn, mx = P.extrema(mesh, F)
pm, pn = S.select_preserved(F.rank32.cpu().numpy(), mx.cpu().numpy(), mn.cpu().numpy(), cfg.n_keep_max,
                            cfg.n_keep_min)
pres = P.ConstraintSet(preserveMinima=pn, preserveMaxima=pm)
if kind == "min":
    F = P.remove_pass(mesh, F, pres, "max").new_order
P.remove_pass(mesh, F, pres, kind)
L = N.load()
L.lts_debug_big_stats(1, None, 0)
torch.cuda.synchronize()
t = time.time()
pr = P.remove_pass(mesh, F, pres, kind)
torch.cuda.synchronize()
print(f"cfg{cfgn} {kind} pass wall ms {(time.time() - t) * 1e3:.1f}", pr.report)
out = np.zeros(256 * 24, np.int64)
L.lts_debug_big_stats(0, out.ctypes.data_as(ctypes.c_void_p), 256)
out = out.reshape(256, 24)
print("k | block steps, cands, committed, warp steps | global attempts, steps, commits | flood Mcyc | nit"
      " | cycles per block step: gather probe cut commit | per global attempt | per warp step"
      " | warp gather probe commit")
for r in out[:10]:
    st = max(r[1], 1)
    print(r[0], "|", r[1], r[2], r[3], r[16], "|", r[18], r[5], r[6], "|", round(r[4] / 1e6, 2), "|", r[7], "|",
          *(r[8:12] // st), "|", r[17] // max(r[18], 1), "|", r[19] // max(r[16], 1), "|",
          *(r[20:23] // max(r[16], 1)))
nz = out[out[:, 0] > 0]
print("regions recorded", len(nz), "sum k", nz[:, 0].sum(), "sum flood Mcyc", nz[:, 4].sum() / 1e6,
      "max", nz[:, 4].max() / 1e6, "sum steps", nz[:, 1].sum() + nz[:, 5].sum())
