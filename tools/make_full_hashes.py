"""Run the CPU oracle on the full-size BASELINE configs and record SHA-256
digests of its outputs in tests/golden/full_hashes.json (key "C" for seed 0,
"C_sS" for seed S).

    python tools/make_full_hashes.py [--seeds 0 1 2] [configs...]

The GPU tests (tests/test_gpu_fullsize.py) regenerate each field with the same
seeded generator and compare the digests of the GPU outputs: full-size
bit-exact parity without committing 64-512 MiB fixtures.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import lts_oracle as O  # noqa: E402
from paper_2009_00083_b200 import synthetic as S  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "full_hashes.json")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main(cfgs, seeds):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for c, seed in [(c, s) for s in seeds for c in cfgs]:
        cfg = S.CONFIGS[c]
        t0 = time.time()
        f = S.make_field(c, seed).ravel()
        tg = time.time() - t0
        dims = cfg.dims
        t0 = time.time()
        rank, inv = O.order_field(f)
        mn, mx = O.extrema(dims, rank, 8)
        pm, pn = S.select_preserved(rank, mx, mn, cfg.n_keep_max, cfg.n_keep_min)
        t1 = time.time()
        res = O.simplify(dims, f, pm, pn, nthreads=8, F=rank)
        t2 = time.time()
        rec = dict(
            config=cfg.name, cfg=c, seed=seed, dims=list(dims), f_sha=sha(f), F_sha=sha(rank),
            pres_max_sha=sha(pm), pres_min_sha=sha(pn), n_pres=[int(pm.size), int(pn.size)],
            maxima=int(mx.size), minima=int(mn.size),
            G_sha=sha(res.G_rank.astype(np.int32)), g_sha=sha(res.g.astype(np.float32)),
            ok=bool(res.ok), outer=int(res.outer_iterations), restored=int(res.restored),
            passes=[dict(kind=p.kind, seeds=p.seeds, regions=p.regions, claimed=p.claimed,
                         largest=p.largest, n_iter_max=p.n_iter_max, capped=p.capped,
                         seconds={k: round(v, 3) for k, v in p.seconds.items()}) for p in res.passes],
            oracle_seconds=dict(generate=round(tg, 2), order_and_classify=round(t1 - t0, 2),
                                simplify=round(t2 - t1, 2)),
        )
        data[str(c) if seed == 0 else f"{c}_s{seed}"] = rec
        json.dump(data, open(OUT, "w"), indent=1)
        print(json.dumps(rec)[:600], flush=True)


if __name__ == "__main__":
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", type=int, default=[1, 2, 3])
    ap.add_argument("--seeds", nargs="*", type=int, default=[0])
    a = ap.parse_args()
    main(a.configs, a.seeds)
