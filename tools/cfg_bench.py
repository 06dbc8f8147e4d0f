"""Full LTS pass on each BASELINE config (seed 0) on the GPU, checked against
the pinned oracle digests in tests/golden/full_hashes.json.

    python tools/cfg_bench.py [configs...] [--repeat R]

Prints one JSON line per config: device ms per pass (CUDA events, inputs in
HBM), phase split, flood statistics and whether G / g match the digests.
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2009_00083_b200 as P  # noqa: E402
from paper_2009_00083_b200 import synthetic as S  # noqa: E402

HASHES = json.load(open(os.path.join(ROOT, "tests", "golden", "full_hashes.json")))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run(cfg, repeat):
    C = S.CONFIGS[cfg]
    t0 = time.time()
    f = S.make_field(cfg, 0).ravel()
    tgen = time.time() - t0
    mesh = P.build_grid_triangulation(C.dims)
    fd = torch.from_numpy(f).cuda()
    F = P.compute_order_field(P.ScalarField(mesh, fd))
    mn, mx = P.extrema(mesh, F)
    pm, pn = S.select_preserved(F.rank32.cpu().numpy(), mx.cpu().numpy(), mn.cpu().numpy(),
                                C.n_keep_max, C.n_keep_min)
    pm_d, pn_d = torch.from_numpy(pm).cuda(), torch.from_numpy(pn).cuda()
    opt = P.SimplifyOptions(collectTiming=True)
    g = torch.empty_like(fd)
    G = torch.empty(mesh.n, dtype=torch.int32, device="cuda")
    P.simplify_raw(mesh, fd, pm_d, pn_d, None, opt, g, G)  # warm-up
    torch.cuda.synchronize()
    ms, rep = [], None
    for _ in range(repeat):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _, _, rep = P.simplify_raw(mesh, fd, pm_d, pn_d, None, opt, g, G)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    r = P.engine._report(rep)
    ref = HASHES.get(str(cfg), {})
    out = {"config": C.name, "n": mesh.n, "ms": ms, "voxels_per_s": mesh.n / (min(ms) * 1e-3),
           "phase_ms": {k: round(v, 3) for k, v in r.phase_ms.items()},
           "outer": r.outerIterations, "maxNI": r.maxNI, "largest": r.largestRegion,
           "G_match": sha(G.cpu().numpy()) == ref.get("G_sha"),
           "g_match": sha(g.cpu().numpy()) == ref.get("g_sha"), "gen_s": round(tgen, 1)}
    print(json.dumps(out), flush=True)
    # free this config's buffers and workspace before the next config allocates its own
    del fd, F, g, G, pm_d, pn_d
    P._native.release_workspaces()
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", type=int, default=[1, 2, 3, 4, 5])
    ap.add_argument("--repeat", type=int, default=1)
    a = ap.parse_args()
    for c in a.configs:
        run(c, a.repeat)
