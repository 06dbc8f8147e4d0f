"""Oracle digests of the full-size persistence pairings (reference
pairs_sweep, _kernels.py:309-421, restated in oracle/lts_oracle.c and pinned to
the reference by tests/golden/make_pairs_golden.py) for cfg1-3, seed 0, both
polarities, epsilon = inf and 1 % of the value range ->
tests/golden/full_pairs.json (checked by tests/test_pairs.py on the GPU)."""
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

OUT = os.path.join(ROOT, "tests", "golden", "full_pairs.json")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.int64).tobytes()).hexdigest()


def main(cfgs):
    data = {}
    for c in cfgs:
        f = S.make_field(c, 0).ravel()
        dims = S.CONFIGS[c].dims
        rank, _ = O.order_field(f)
        vals = f.astype(np.float64)
        rng = float(vals.max() - vals.min())
        for kind in ("max", "min"):
            for tag, eps in (("inf", float("inf")), ("1pct", 0.01 * rng)):
                t0 = time.time()
                seeds, sad, err = O.pairs(dims, rank, vals, kind, eps)
                assert err == 0
                data[f"cfg{c}_{kind}_{tag}"] = dict(cfg=c, seed=0, kind=kind, eps=eps, count=int(seeds.size),
                                                    paired=int((sad >= 0).sum()), extrema_sha=sha(seeds),
                                                    saddles_sha=sha(sad), oracle_s=round(time.time() - t0, 3))
                print(c, kind, tag, data[f"cfg{c}_{kind}_{tag}"], flush=True)
    json.dump(data, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [1, 2, 3])
