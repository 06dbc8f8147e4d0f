"""SFG / SFGB field files, preserve lists and the command line surface
(SPEC.md:529-628).  CPU tests cover the formats and usage errors; the GPU test
runs simplify -> verify through files and checks the output against the CPU
oracle."""
import json
import os

import numpy as np
import pytest

from paper_2009_00083_b200 import cli
from paper_2009_00083_b200 import io as sio
from paper_2009_00083_b200.errors import FieldError, MeshError


def test_sfg_spec_example():
    dims, v = sio.read_sfg("SFG 2 2 2\n0 1 2 3")
    assert dims == (2, 2) and v.tolist() == [0.0, 1.0, 2.0, 3.0]


def test_sfg_round_trip_float32_exact():
    rng = np.random.default_rng(0)
    v = rng.standard_normal(7 * 5 * 3).astype(np.float32)
    v[:4] = [np.float32(3.4e38), np.float32(-1e-45), np.float32(0.1), np.float32(-0.0)]
    dims = (7, 5, 3)
    d2, back = sio.read_sfg(sio.write_sfg(dims, v))
    assert d2 == dims
    assert back.astype(np.float32).tobytes() == v.tobytes()


def test_sfgb_round_trip(tmp_path):
    v = np.random.default_rng(1).random(6 * 4) * 1e3
    p = str(tmp_path / "f.sfgb")
    sio.write_field(p, (6, 4), v)
    dims, back = sio.read_sfgb(open(p, "rb").read())
    assert dims == (6, 4) and np.array_equal(back, v)
    d3, b32 = sio.read_field(p)
    assert d3 == (6, 4) and b32.dtype == np.float32


def test_sfg_errors_name_the_line():
    with pytest.raises(FieldError, match="line 2"):
        sio.read_sfg("SFG 2 2 2\n0 1 2")
    with pytest.raises(FieldError, match="line 3"):
        sio.read_sfg("SFG 2 2 2\n0 1\n2 x")
    with pytest.raises(FieldError, match="not finite"):
        sio.read_sfg("SFG 2 2 1\n0 nan")
    with pytest.raises(MeshError, match="line 1"):
        sio.read_sfg("SFG 4 2 2\n0 1 2 3")
    with pytest.raises(MeshError):
        sio.read_sfg("XYZ 2 2 2\n0 1 2 3")
    with pytest.raises(FieldError):
        sio.read_sfgb(b"SFGB 2 2 2\n" + b"\0" * 8)


def test_preserve_list():
    assert sio.read_preserve_list("0\n24\n", 25).tolist() == [0, 24]
    assert sio.read_preserve_list("# comment\n\n3\n3\n", 5).tolist() == [3]
    with pytest.raises(FieldError, match="25"):
        sio.read_preserve_list("0\n25\n", 25)
    assert sio.read_preserve_list(sio.write_preserve_list([4, 1]), 9).tolist() == [1, 4]


def test_cli_usage_errors(tmp_path):
    f = str(tmp_path / "f.sfg")
    open(f, "w").write("SFG 2 2 2\n0 1 2 3\n")
    for argv in (["bench", "--input", f, "--epsilon", "1%"],
                 ["simplify", "--input", f, "--output", f + ".o", "--epsilon", "1%", "--preserve", f],
                 ["simplify", "--input", f, "--output", f + ".o"],
                 ["simplify", "--input", f, "--output", f + ".o", "--preserve", f, "--keep-max", "1",
                  "--keep-min", "1"],
                 ["nosuch"]):
        with pytest.raises(SystemExit) as e:
            cli.main(argv)
        assert e.value.code == 2


def test_cli_synth(tmp_path):
    p = str(tmp_path / "cfg1.sfgb")
    assert cli.main(["synth", "--config", "1", "--seed", "0", "--output", p]) == 0
    from paper_2009_00083_b200 import synthetic as S
    dims, v = sio.read_field(p)
    assert dims == (512, 512)
    assert v.tobytes() == S.make_field(1, 0).ravel().astype(np.float32).tobytes()


@pytest.mark.gpu
def test_cli_simplify_verify_matches_oracle(tmp_path):
    from oracle import lts_oracle as O
    rng = np.random.default_rng(11)
    f = (np.round(rng.random((30, 34)) * 25) / 25).astype(np.float32)  # ties on purpose
    dims = (34, 30)
    src = str(tmp_path / "f.sfg")
    sio.write_field(src, dims, f.ravel())
    rank, _ = O.order_field(f.ravel())
    mn, mx = O.extrema(dims, rank)
    pm = mx[np.argsort(rank[mx])[-4:]]
    pn = mn[np.argsort(rank[mn])[:3]]
    plist = str(tmp_path / "keep.txt")
    open(plist, "w").write(sio.write_preserve_list(np.concatenate([pm, pn])))
    out, order, rep = (str(tmp_path / x) for x in ("g.sfg", "G.npy", "r.json"))
    assert cli.main(["simplify", "--input", src, "--preserve", plist, "--output", out,
                     "--order-out", order, "--report", rep]) == 0
    ref = O.simplify(dims, f.ravel(), np.sort(pm), np.sort(pn))
    _, g = sio.read_field(out)
    assert g.tobytes() == ref.g.tobytes()
    assert np.array_equal(np.load(order), ref.G_rank)
    assert json.load(open(rep))["ok"]
    assert cli.main(["verify", "--original", src, "--simplified", out, "--order", order,
                     "--preserve", plist]) == 0
    # a tampered order (swap the preserved maximum with a neighbour) fails verification
    G = np.load(order)
    v = int(pm[-1])
    u = v + 1 if (v + 1) % dims[0] else v - 1
    G[[u, v]] = G[[v, u]]
    np.save(order, G)
    assert cli.main(["verify", "--original", src, "--simplified", out, "--order", order,
                     "--preserve", plist]) == 1


@pytest.mark.gpu
def test_cli_persistence_commands(tmp_path):
    """simplify --epsilon E% (persistence-driven), diagram and curve JSON."""
    f = (np.round(np.random.default_rng(12).random((26, 30)) * 40) / 40).astype(np.float32)
    dims = (30, 26)
    src = str(tmp_path / "f.sfgb")
    sio.write_field(src, dims, f.ravel())
    out, rep, dia, cur = (str(tmp_path / x) for x in ("g.sfg", "r.json", "d.json", "c.json"))
    assert cli.main(["simplify", "--input", src, "--epsilon", "20%", "--output", out, "--report", rep]) == 0
    _, g = sio.read_field(out)
    assert float(np.abs(g.astype(np.float64) - f.ravel()).max()) <= 0.2 * float(f.max() - f.min())
    assert cli.main(["diagram", "--input", src, "--output", dia]) == 0
    d = json.load(open(dia))
    pol = {"MaxSaddle": 0, "MinSaddle": 0}
    for e in d:
        pol[e["polarity"]] += 1
        if e["saddleVertex"] is not None:
            assert e["persistence"] >= 0  # 0 only between tied values (quantised field)
    glob = [e for e in d if e["saddleVertex"] is None]
    assert len(glob) == 2  # epsilon = infinity: only the global pair survives per polarity
    assert cli.main(["curve", "--input", src, "--output", cur]) == 0
    c = json.load(open(cur))
    assert c[0]["count"] == len(d) and all(a["count"] >= b["count"] for a, b in zip(c, c[1:]))
