"""One full LTS pass on a BASELINE config (default cfg3 256^3), for ncu.
Usage: python tools/profile_step.py [cfg] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_00083_b200 as P  # noqa: E402
from paper_2009_00083_b200 import synthetic as S  # noqa: E402

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = S.CONFIGS[cfgn]
f = torch.from_numpy(S.make_field(cfgn, 0).ravel()).cuda()
mesh = P.build_grid_triangulation(cfg.dims)
F = P.compute_order_field(P.ScalarField(mesh, f))
mn, mx = P.extrema(mesh, F)
pm, pn = S.select_preserved(F.rank32.cpu().numpy(), mx.cpu().numpy(), mn.cpu().numpy(),
                            cfg.n_keep_max, cfg.n_keep_min)
pm = torch.from_numpy(pm).cuda()
pn = torch.from_numpy(pn).cuda()
for _ in range(reps):
    g, G, rep = P.simplify_raw(mesh, f, pm, pn)
torch.cuda.synchronize()
print("ok", rep.ok, rep.outer_iterations)
