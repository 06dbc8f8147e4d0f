"""Per-region counters of the CTA flood kernel for one maxima pass."""
import os, sys, ctypes, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2009_00083_b200 as P
from paper_2009_00083_b200 import _native as N, synthetic as S
cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 3
kind = sys.argv[2] if len(sys.argv) > 2 else "max"
cfg = S.CONFIGS[cfgn]
f = torch.from_numpy(S.make_field(cfgn, 0).ravel()).cuda()
mesh = P.build_grid_triangulation(cfg.dims)
F = P.compute_order_field(P.ScalarField(mesh, f))
mn, mx = P.extrema(mesh, F)
pm, pn = S.select_preserved(F.rank32.cpu().numpy(), mx.cpu().numpy(), mn.cpu().numpy(), cfg.n_keep_max, cfg.n_keep_min)
pres = P.ConstraintSet(preserveMinima=pn, preserveMaxima=pm)
P.remove_pass(mesh, F, pres, kind)
L = N.load()
L.lts_debug_big_stats(1, None, 0)
torch.cuda.synchronize()
t = time.time()
pr = P.remove_pass(mesh, F, pres, kind)
torch.cuda.synchronize(); print("pass wall ms", (time.time() - t) * 1e3, pr.report)
out = np.zeros(256 * 24, np.int64)
L.lts_debug_big_stats(0, out.ctypes.data_as(ctypes.c_void_p), 256)
out = out.reshape(256, 24)
print("k steps cands committed flood_Mcyc nit | per-step cycles: gather probe cut commit")
for r in out[:12]:
    st = max(r[1], 1)
    print(r[0], r[1], r[2], r[3], round(r[4] / 1e6, 2), r[7], "|", *(r[8:12] // st),
          "| j<=8:", r[12], "j<=32:", r[13], "sum ceil(j/32):", r[14], "unpreempted:", r[15], "sum ceil(j/64):", r[16])
nz = out[out[:, 0] > 0]
print("regions", len(nz), "sum flood Mcyc", nz[:, 4].sum() / 1e6, "max", nz[:, 4].max() / 1e6)
