"""CPU-only checks of the boundary: the C-ABI library loads and exports every
symbol declared in include/lts_sm100.h; host-side metadata matches the
reference tables; the product path refuses to run without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "lts_sm100.h")).read()
    return sorted(set(re.findall(r"\b(lts_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    from paper_2009_00083_b200 import _native as N
    L = N.load()
    names = _declared()
    assert "lts_simplify" in names and "lts_order_field" in names
    for name in names:
        assert hasattr(L, name), name
    assert L.lts_version().startswith(b"lts_sm100")


def test_workspace_size_and_bad_dims():
    from paper_2009_00083_b200 import _native as N
    L = N.load()
    nb = ctypes.c_size_t(0)
    assert L.lts_workspace_size(3, N.dims_arg((256, 256, 256)), ctypes.byref(nb)) == 0
    assert nb.value > 16 ** 3
    assert L.lts_workspace_size(4, N.dims_arg((2, 2, 2)), ctypes.byref(nb)) == N.E_BAD_DIMS
    assert L.lts_workspace_size(2, N.dims_arg((1, 5)), ctypes.byref(nb)) == N.E_BAD_DIMS


def test_link_tables_match_oracle_restatement():
    from paper_2009_00083_b200 import grid_link_tables
    from oracle import lts_oracle as O
    for d in (2, 3):
        offs, pairs = grid_link_tables(d)
        o2, p2 = O.grid_tables(d)
        np.testing.assert_array_equal(offs, o2)
        np.testing.assert_array_equal(pairs, p2)


def test_mesh_errors_and_neighbors():
    import paper_2009_00083_b200 as P
    with pytest.raises(P.MeshError):
        P.build_grid_triangulation((1, 4))
    with pytest.raises(P.MeshError):
        P.build_grid_triangulation((2, 2, 2, 2))
    m = P.build_grid_triangulation((2, 2))
    assert sorted(m.neighbors(0).tolist()) == [1, 2, 3]  # SPEC.md:45 example
    m = P.build_grid_triangulation((5, 5))
    assert sorted(m.neighbors(12).tolist()) == sorted([11, 13, 7, 17, 18, 6])
    m = P.build_grid_triangulation((3, 3, 3))
    assert m.degree(13) == 14


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2009_00083_b200 as P
    m = P.build_grid_triangulation((4, 4))
    with pytest.raises(Exception):
        P.ScalarField(m, np.zeros(16, np.float32))


def test_synthetic_generators_small():
    from paper_2009_00083_b200 import synthetic as S
    a = S.cfg1(0, N=32)
    b = S.cfg1(0, N=32)
    assert a.dtype == np.float32 and a.shape == (32, 32) and np.array_equal(a, b)
    assert S.cfg2(3, N=8).shape == (8, 8, 8)
    assert S.CONFIGS[3].dims == (256, 256, 256)


def test_generators_match_full_size_digests():
    """cfg1/cfg2 generators reproduce the fields the oracle digests were made
    from (tests/golden/full_hashes.json)."""
    import hashlib
    import json
    from paper_2009_00083_b200 import synthetic as S
    data = json.load(open(os.path.join(ROOT, "tests", "golden", "full_hashes.json")))
    for c in (1, 2):
        f = S.make_field(c, 0).ravel()
        assert hashlib.sha256(f.tobytes()).hexdigest() == data[str(c)]["f_sha"]


def test_oracle_matches_full_size_cfg1_digest():
    """The pinned CPU oracle reproduces its own full-size cfg1 digest."""
    import hashlib
    import json
    from oracle import lts_oracle as O
    from paper_2009_00083_b200 import synthetic as S
    data = json.load(open(os.path.join(ROOT, "tests", "golden", "full_hashes.json")))["1"]
    C = S.CONFIGS[1]
    f = S.make_field(1, 0).ravel()
    rank, _ = O.order_field(f)
    mn, mx = O.extrema(C.dims, rank)
    pm, pn = S.select_preserved(rank, mx, mn, C.n_keep_max, C.n_keep_min)
    res = O.simplify(C.dims, f, pm, pn)
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    assert sha(res.G_rank.astype(np.int32)) == data["G_sha"]
    assert sha(res.g) == data["g_sha"]


def test_select_preserved_top_k():
    from paper_2009_00083_b200 import synthetic as S
    rank = np.array([5, 0, 3, 9, 1, 7, 2, 8, 4, 6])
    mx = np.array([0, 3, 5, 7])
    mn = np.array([1, 4, 6])
    pm, pn = S.select_preserved(rank, mx, mn, 2, 1)
    assert pm.tolist() == [3, 7] and pn.tolist() == [1]


def test_grid_size_limit_matches_library():
    """One n limit on both sides of the boundary (MeshError / LTS_E_BAD_DIMS):
    the device path packs rank << 4 | stencil index into 32 bits."""
    import paper_2009_00083_b200 as P
    P.build_grid_triangulation((512, 512, 512))  # 2^27: allowed
    with pytest.raises(P.MeshError):
        P.build_grid_triangulation((513, 512, 512))
    assert P.triangulation.MAX_GRID_VERTICES == 1 << 27


def test_simplify_options_validation():
    import paper_2009_00083_b200 as P
    assert P.SimplifyOptions().zeta is None  # contract D1 by default
    with pytest.raises(ValueError):
        P.SimplifyOptions(maxIterations=0)
    with pytest.raises(ValueError):
        P.SimplifyOptions(threadCount=-1)
    with pytest.raises(TypeError):
        P.SimplifyOptions(zeta=1e-12)
    # the reference's ZetaPolicy default (order.py:77)
    assert P.ZetaPolicy().mode is P.ZetaMode.RELATIVE_EPSILON
    assert P.ZetaPolicy().step(2.0) == 2e-12
    assert P.ZetaPolicy(P.ZetaMode.ULP_DECREMENT).step(2.0) == 0.0


def test_float64_exactness_check_host_side():
    from paper_2009_00083_b200.order import _to_f32_exact
    from paper_2009_00083_b200 import FieldError
    a = np.array([0.5, 1.25, -3.0, 2.0 ** 100], np.float64)
    assert _to_f32_exact(a).dtype == np.float32
    with pytest.raises(FieldError):
        _to_f32_exact(np.array([0.1], np.float64))  # not a float32
    assert _to_f32_exact(np.array([0.1], np.float32)).dtype == np.float32


def test_bench_cli_refuses_nothing_on_cpu_parse():
    """bench.py parses --gpus N and re-launches itself under torchrun when it
    is not already a torchrun rank (checked by reading its argument handling)."""
    src = open(os.path.join(ROOT, "bench.py")).read()
    assert "torch.distributed.run" in src and "--nproc-per-node" in src
