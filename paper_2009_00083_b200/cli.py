"""Command line surface of the LTS path (cli module).

    python -m paper_2009_00083_b200.cli simplify --input F --preserve LIST --output G
            [--order-out O.npy] [--report R.json] [--no-restore] [--max-iterations N]
    python -m paper_2009_00083_b200.cli simplify --input F --keep-max K --keep-min K --output G
    python -m paper_2009_00083_b200.cli verify --original F --simplified G --order O.npy --preserve LIST
    python -m paper_2009_00083_b200.cli bench --input F (--preserve LIST | --keep-max K --keep-min K)
            [--repeat N]
    python -m paper_2009_00083_b200.cli simplify --input F --epsilon E[%] --output G
    python -m paper_2009_00083_b200.cli diagram --input F [--epsilon E[%]] --output D.json
            [--polarity max|min|both]
    python -m paper_2009_00083_b200.cli curve --input F --output C.json
    python -m paper_2009_00083_b200.cli synth --config C [--seed S] --output F

Fields are SFG text or SFGB binary (``paper_2009_00083_b200.io``); the
preserve list holds vertex ids of maxima and minima of the input order, one per
line, split by classification.  ``--keep-max/--keep-min`` select the K highest
maxima / K lowest minima of the input order instead (the BASELINE
configs' selection rule).  ``--epsilon E`` (field units, or ``E%`` of the
value range) selects the persistence-driven mode instead: every
extremum less persistent than E is removed (SPEC persistence module).
``--threads`` is accepted and ignored (the work runs on the GPU).
Exit codes: 0 success, 1 verification failure, 2 usage.
"""
from __future__ import annotations

import argparse
import json
import sys

import numpy as np

from . import io as sio
from .errors import ConstraintNotExtremum, FieldError, MeshError


def _load(path):
    import torch

    from .triangulation import build_grid_triangulation
    dims, v = sio.read_field(path)
    mesh = build_grid_triangulation(dims)
    return dims, mesh, torch.from_numpy(v).cuda()


def _constraints(args, mesh, fd):
    """ConstraintSet from --preserve LIST or --keep-max/--keep-min."""
    from . import ConstraintSet, ScalarField, compute_order_field, extrema
    F = compute_order_field(ScalarField(mesh, fd))
    mn, mx = extrema(mesh, F)
    mn, mx = mn.cpu().numpy(), mx.cpu().numpy()
    if args.preserve:
        with open(args.preserve) as fh:
            ids = sio.read_preserve_list(fh.read(), mesh.n)
        pmax = np.intersect1d(ids, mx)
        pmin = np.intersect1d(ids, mn)
        other = np.setdiff1d(ids, np.union1d(pmax, pmin))
        if other.size:
            raise ConstraintNotExtremum(f"vertex {int(other[0])} of the preserve list is not an extremum of the input")
    else:
        from .synthetic import select_preserved
        pmax, pmin = select_preserved(F.rank32.cpu().numpy(), mx, mn, args.keep_max, args.keep_min)
    return F, ConstraintSet(preserveMinima=pmin, preserveMaxima=pmax)


def _need_selection(ap, args, epsilon_ok=False):
    chosen = [args.epsilon is not None, bool(args.preserve), args.keep_max is not None or args.keep_min is not None]
    if sum(chosen) != 1:
        ap.error("give exactly one of --epsilon, --preserve LIST, or --keep-max K --keep-min K")
    if args.epsilon is not None and not epsilon_ok:
        ap.error("--epsilon is not accepted by this subcommand")
    if chosen[2] and (args.keep_max is None or args.keep_min is None):
        ap.error("--keep-max and --keep-min go together")


def _epsilon(text, fd) -> float:
    """E (field units) or E% of the value range."""
    t = str(text).strip()
    try:
        if t.endswith("%"):
            return float(t[:-1]) / 100.0 * float(fd.max() - fd.min())
        return float(t)
    except ValueError:
        raise FieldError(f"--epsilon {t!r} is not a number or a percentage") from None


def cmd_simplify(ap, args) -> int:
    _need_selection(ap, args, epsilon_ok=True)
    from . import ConstraintSet, SimplifyOptions, persistence_simplify, simplify_field
    dims, mesh, fd = _load(args.input)
    opt = SimplifyOptions(restoreInteriorExtrema=not args.no_restore, maxIterations=args.max_iterations)
    if args.epsilon is not None:
        eps = _epsilon(args.epsilon, fd)
        if eps < 0:
            ap.error("--epsilon must be >= 0")
        g, G, (pmax, pmin), rep = persistence_simplify(mesh, fd, eps, opt)
        cs = ConstraintSet(preserveMinima=pmin.survivors.cpu().numpy(), preserveMaxima=pmax.survivors.cpu().numpy())
    else:
        F, cs = _constraints(args, mesh, fd)
        g, G, rep = simplify_field(mesh, fd, cs, opt, order=F)
    sio.write_field(args.output, dims, g.values.cpu().numpy())
    if args.order_out:
        np.save(args.order_out, G.rank32.cpu().numpy().astype(np.int64))
    if args.report:
        d = {"ok": rep.ok, "outerIterations": rep.outerIterations, "restored": rep.restored,
             "regionCount": rep.regionCount, "largestRegion": rep.largestRegion, "maxNI": rep.maxNI,
             "capped": rep.capped, "linf": rep.linf, "phase_ms": rep.phase_ms,
             "passes": [p.__dict__ for p in rep.passes],
             "preserved": {"maxima": int(len(cs.preserveMaxima)), "minima": int(len(cs.preserveMinima))}}
        with open(args.report, "w") as fh:
            json.dump(d, fh, indent=1, default=float)
    return 0 if rep.ok else 1


def cmd_verify(ap, args) -> int:
    from . import ConstraintSet, extrema, order_from_ranks, verify_constraints
    dims, mesh, fd = _load(args.original)
    dims2, gv = sio.read_field(args.simplified)
    if tuple(dims2) != tuple(dims):
        print(f"grid mismatch: {dims} vs {dims2}", file=sys.stderr)
        return 1
    G = order_from_ranks(np.load(args.order))
    with open(args.preserve) as fh:
        ids = sio.read_preserve_list(fh.read(), mesh.n)
    mn, mx = extrema(mesh, G)
    mn, mx = mn.cpu().numpy(), mx.cpu().numpy()
    # the requested sets are read off the ids: a preserved maximum of f is a
    # maximum of G, so split by the input order's classification
    from . import ScalarField, compute_order_field
    Fmn, Fmx = extrema(mesh, compute_order_field(ScalarField(mesh, fd)))
    cs = ConstraintSet(preserveMinima=np.intersect1d(ids, Fmn.cpu().numpy()),
                       preserveMaxima=np.intersect1d(ids, Fmx.cpu().numpy()))
    v = verify_constraints(mesh, G, cs)
    f = fd.cpu().numpy()
    fz = np.where(f == 0, np.float32(0), f)
    inv = G.inverse.cpu().numpy().astype(np.int64)
    checks = {
        "constraints": bool(v.ok),
        "values_are_copies": bool(np.all(np.isin(gv, fz))),
        "g_realises_G": bool(np.all(np.diff(gv[inv]) >= 0)),
    }
    out = dict(checks, linf=float(np.abs(gv.astype(np.float64) - f).max()) if f.size else 0.0,
               maxima=int(mx.size), minima=int(mn.size))
    print(json.dumps(out))
    return 0 if all(checks.values()) else 1


def cmd_bench(ap, args) -> int:
    _need_selection(ap, args)
    import torch

    from . import SimplifyOptions, simplify_raw
    from .engine import _report
    dims, mesh, fd = _load(args.input)
    F, cs = _constraints(args, mesh, fd)
    pm = torch.as_tensor(np.asarray(cs.preserveMaxima, np.int64)).cuda()
    pn = torch.as_tensor(np.asarray(cs.preserveMinima, np.int64)).cuda()
    opt = SimplifyOptions(collectTiming=True)
    simplify_raw(mesh, fd, pm, pn, F.rank32, opt)  # warm-up
    torch.cuda.synchronize()
    ms, phases = [], []
    for _ in range(args.repeat):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _, _, rep = simplify_raw(mesh, fd, pm, pn, None, opt)
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
        phases.append(_report(rep).phase_ms)
    best = int(np.argmin(ms))
    print(json.dumps({"input": args.input, "dims": list(dims), "n": mesh.n, "ms": ms,
                      "voxels_per_s": mesh.n / (min(ms) / 1e3), "phase_ms": phases[best]}))
    return 0


def _pairs(mesh, fd, polarity, eps):
    from . import ScalarField, compute_extremum_saddle_pairs, compute_order_field
    f = ScalarField(mesh, fd)
    F = compute_order_field(f)
    kinds = ["max", "min"] if polarity == "both" else [polarity]
    return [compute_extremum_saddle_pairs(mesh, f, F, k, eps) for k in kinds]


def cmd_diagram(ap, args) -> int:
    """Diagram JSON: pairs below epsilon plus the survivors
    (saddleVertex null); a survivor's persistence is the value range for the
    global extremum (the global pair convention) and null for the
    others when epsilon is finite."""
    dims, mesh, fd = _load(args.input)
    eps = _epsilon(args.epsilon, fd) if args.epsilon is not None else float("inf")
    f = fd.cpu().numpy().astype(np.float64)
    vr = float(f.max() - f.min())
    out = []
    for pp in _pairs(mesh, fd, args.polarity, eps):
        pol = "MaxSaddle" if pp.polarity == "max" else "MinSaddle"
        ext = pp.extrema.cpu().numpy()
        sad = pp.saddles.cpu().numpy()
        glob_ext = int(ext[np.argmax(f[ext])]) if pp.polarity == "max" else int(ext[np.argmin(f[ext])])
        for e, sv in zip(ext.tolist(), sad.tolist()):
            if sv >= 0:
                out.append({"extremumVertex": e, "saddleVertex": sv, "birth": f[e], "death": f[sv],
                            "persistence": abs(f[e] - f[sv]), "polarity": pol})
            else:
                out.append({"extremumVertex": e, "saddleVertex": None, "birth": f[e], "death": None,
                            "persistence": vr if e == glob_ext else None, "polarity": pol})
    with open(args.output, "w") as fh:
        json.dump(out, fh)
    return 0


def cmd_curve(ap, args) -> int:
    """Curve JSON: both polarities, full diagram."""
    from . import persistence_curve
    dims, mesh, fd = _load(args.input)
    vr = float(fd.max() - fd.min())
    thr, cnt = persistence_curve(_pairs(mesh, fd, "both", float("inf")), value_range=vr)
    with open(args.output, "w") as fh:
        json.dump([{"threshold": float(t), "count": int(c)} for t, c in zip(thr, cnt)], fh)
    return 0


def cmd_synth(ap, args) -> int:
    from .synthetic import CONFIGS, make_field
    if args.config not in CONFIGS:
        ap.error(f"--config must be one of {sorted(CONFIGS)}")
    f = make_field(args.config, args.seed)
    sio.write_field(args.output, CONFIGS[args.config].dims, f.ravel())
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="paper_2009_00083_b200.cli", description=__doc__.split("\n")[0])
    sub = ap.add_subparsers(dest="cmd", required=True)

    def selection(p):
        p.add_argument("--preserve", help="vertex ids to preserve, one per line")
        p.add_argument("--keep-max", type=int, help="preserve the K highest maxima")
        p.add_argument("--keep-min", type=int, help="preserve the K lowest minima")
        p.add_argument("--epsilon", help="persistence threshold E or E%% of the value range")
        p.add_argument("--threads", help="accepted for compatibility; ignored")

    p = sub.add_parser("simplify")
    p.add_argument("--input", required=True)
    p.add_argument("--output", required=True)
    p.add_argument("--order-out")
    p.add_argument("--report")
    p.add_argument("--no-restore", action="store_true")
    p.add_argument("--max-iterations", type=int, default=100)
    selection(p)
    p = sub.add_parser("verify")
    p.add_argument("--original", required=True)
    p.add_argument("--simplified", required=True)
    p.add_argument("--order", required=True, help="order field of the simplified output (.npy)")
    p.add_argument("--preserve", required=True)
    p = sub.add_parser("bench")
    p.add_argument("--input", required=True)
    p.add_argument("--repeat", type=int, default=5)
    selection(p)
    p = sub.add_parser("diagram")
    p.add_argument("--input", required=True)
    p.add_argument("--output", required=True)
    p.add_argument("--epsilon")
    p.add_argument("--polarity", choices=["max", "min", "both"], default="both")
    p = sub.add_parser("curve")
    p.add_argument("--input", required=True)
    p.add_argument("--output", required=True)
    p = sub.add_parser("synth")
    p.add_argument("--config", type=int, required=True)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--output", required=True)
    args = ap.parse_args(argv)
    try:
        return {"simplify": cmd_simplify, "verify": cmd_verify, "bench": cmd_bench, "diagram": cmd_diagram,
                "curve": cmd_curve, "synth": cmd_synth}[args.cmd](ap, args)
    except (FieldError, MeshError, ConstraintNotExtremum, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
