import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2009_00083_b200 as P
from paper_2009_00083_b200 import _native as N, synthetic as S
cfg = S.CONFIGS[3]
f = torch.from_numpy(S.make_field(3, 0).ravel()).cuda()
mesh = P.build_grid_triangulation(cfg.dims)
L = N.load()
P.compute_order_field(P.ScalarField(mesh, f))
L.lts_debug_big_stats(1, None, -1)
P.compute_order_field(P.ScalarField(mesh, f))
torch.cuda.synchronize()
out = np.zeros(8, np.int64)
L.lts_debug_big_stats(0, out.ctypes.data_as(ctypes.c_void_p), -1)
tiles = 4 * ((mesh.n + 4095) // 4096)
print("per-tile cycles by phase (init, hist, rank, lookback, scatter, write):", (out[1:7] / tiles).astype(int))
