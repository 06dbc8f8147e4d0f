import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2009_00083_b200 as P
from paper_2009_00083_b200 import _native as N, synthetic as S
cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = S.CONFIGS[cfgn]
f = torch.from_numpy(S.make_field(cfgn, 0).ravel()).cuda()
mesh = P.build_grid_triangulation(cfg.dims)
ws = N.workspace(mesh.grid_dims, f.device)
kms = (ctypes.c_double * 4)()
L = N.load()
for _ in range(2):
    N.check(L.lts_bench_kernels(N.ptr(f), mesh.dim, N.dims_arg(mesh.grid_dims), 10, kms, N.ptr(ws), ws.numel(), N.stream_ptr()))
n = mesh.n
print("sort ms %.4f  -> %.0f GB/s (64 B/voxel)" % (kms[0], 64 * n / kms[0] / 1e6))
print("classify ms %.4f -> %.0f GB/s (5 B/voxel)" % (kms[1], 5 * n / kms[1] / 1e6))
print("classify+ptr ms %.4f -> %.0f GB/s (9 B/voxel)" % (kms[2], 9 * n / kms[2] / 1e6))
