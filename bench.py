"""Benchmark of the full LTS pass (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 3] [--seed 0]

A "step" is one full LTS pass (SPEC simplify_field: order field -> classify ->
maxima/minima passes -> restore/verify -> realize) over the 256^3 float32
field of BASELINE config 3, inputs resident in HBM.  Prints ONE JSON line.

  value  whole-job voxels/s, device-timed (CUDA events per step, L2 flushed
         between steps outside the event window), max over ranks
  e2e    the same metric through the public API with host buffers: pinned
         H2D of f + preserve lists, D2H of g and G, inside the timed region
  roofline  dominant kernel of the step vs MEASURED_PEAKS.json HBM GB/s
  cpu_baseline  the CPU oracle (C port of the reference kernels + SPEC glue)
         running the same full pass on the same field (rank 0 only), with
         the host CPU model and the threads used
  configs  one warm-up + one timed full pass of each other BASELINE config
         (cfg1, cfg2, cfg4, cfg5), with their parity against the oracle
         digests of tests/golden/full_hashes.json

--impl reference runs the CPU oracle port (the reference is Python/numba and
does not travel to the GPU box) on the same full pass per step.
Multi-GPU: one process per GPU (torchrun), independent replicas
("replicas only"): the path has no data exchange.  `--gpus N`
without torchrun re-launches itself under torch.distributed.run.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "simplified voxels/sec (full LTS pass) at 256^3 fp32; kernel HBM GB/s vs peak"
UNIT = "voxels/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p is not None:
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx = max(mx, float(f[1]))
            except ValueError:
                continue
            for nm, val in zip(names, f[2:6]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        load = [x for x in sm if x > 0.5 * mx] if mx else sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_workload(f3d: np.ndarray, cfg):
    """The benchmark's own workload for the CPU legs: the full field and the
    same preserve lists (top-K maxima / bottom-K minima of F)."""
    from paper_2009_00083_b200 import synthetic as S
    from oracle import lts_oracle as O
    dims = tuple(f3d.shape[::-1])
    fr = np.ascontiguousarray(f3d.ravel())
    rank, _ = O.order_field(fr)
    mn, mx = O.extrema(dims, rank, os.cpu_count())
    pm, pn = S.select_preserved(rank, mx, mn, cfg.n_keep_max, cfg.n_keep_min)
    return dims, fr, pm, pn


def run_oracle(dims, fr, pm, pn, threads):
    from oracle import lts_oracle as O
    t0 = time.perf_counter()
    res = O.simplify(dims, fr, pm, pn, nthreads=threads)
    dt = time.perf_counter() - t0
    assert res.ok
    return dt


def workload_config(cfg, args, n, npres, world):
    """The `config` object both arms print (same workload, same keys)."""
    return {"workload": f"{cfg.name} full LTS pass", "grid": list(cfg.dims), "n": n, "seed": args.seed,
            "preserve": [int(npres[0]), int(npres[1])],
            "parallelism": "replicas" if world > 1 else "single",
            "l2": "flushed between steps (256 MiB write, outside the per-step events)"}


def reference_arm(args):
    """The reference's CPU path (the pinned C port of its numba kernels + the
    SPEC glue, oracle/) on the SAME workload as our arm: the full cfg3 pass
    over the whole 256^3 field with the same preserve lists, every host
    thread (OpenMP where the reference uses prange; discover, sort and the
    realisation sweep are sequential as in the reference).  The C port has no
    JIT, so one untimed pass stands in for the warm-up steps."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    from paper_2009_00083_b200 import synthetic as S
    cfg = S.CONFIGS[args.config]
    f3d = S.make_field(args.config, args.seed)
    dims, fr, pm, pn = cpu_workload(f3d, cfg)
    threads = os.cpu_count() or 1
    if args.warmup > 0:
        run_oracle(dims, fr, pm, pn, threads)
    ts = [run_oracle(dims, fr, pm, pn, threads) for _ in range(args.steps)]
    t = sum(ts) / len(ts)
    v = fr.size / t
    sample = (f"the full workload: {cfg.name} field (seed {args.seed}), {fr.size} voxels, "
              f"preserve {pm.size} max / {pn.size} min, one full LTS pass per step "
              f"({t:.1f} s each); host CPU {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": workload_config(cfg, args, fr.size, (pm.size, pn.size), world),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def other_configs(dev, budget_s: float):
    """One warm-up + one timed full pass (device-resident, CUDA events) of each
    other BASELINE config, each checked against its oracle digest.  Configs are
    skipped once the block has used `budget_s` seconds of wall time."""
    import hashlib

    import torch

    import paper_2009_00083_b200 as P
    from paper_2009_00083_b200 import _native as N
    from paper_2009_00083_b200 import synthetic as S
    hp = os.path.join(ROOT, "tests", "golden", "full_hashes.json")
    digests = json.load(open(hp)) if os.path.exists(hp) else {}
    out = {}
    t_start = time.time()
    for c in (1, 2, 4, 5):
        if time.time() - t_start > budget_s:
            out[S.CONFIGS[c].name] = {"skipped": "time budget of the configs block used up"}
            continue
        C = S.CONFIGS[c]
        f = S.make_field(c, 0).ravel()
        mesh = P.build_grid_triangulation(C.dims)
        fd = torch.from_numpy(f).to(dev)
        F = P.compute_order_field(P.ScalarField(mesh, fd))
        mn, mx = P.extrema(mesh, F)
        pm, pn = S.select_preserved(F.rank32.cpu().numpy(), mx.cpu().numpy(), mn.cpu().numpy(),
                                    C.n_keep_max, C.n_keep_min)
        pm_d, pn_d = torch.from_numpy(pm).to(dev), torch.from_numpy(pn).to(dev)
        g = torch.empty_like(fd)
        G = torch.empty(mesh.n, dtype=torch.int32, device=dev)
        opt = P.SimplifyOptions(collectTiming=True)
        P.simplify_raw(mesh, fd, pm_d, pn_d, None, opt, g, G)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        _, _, rep = P.simplify_raw(mesh, fd, pm_d, pn_d, None, opt, g, G)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        r = P.engine._report(rep)
        d = digests.get(str(c), {})
        out[C.name] = {
            "n": mesh.n, "ms_per_pass": ms, "value": mesh.n / (ms * 1e-3), "unit": UNIT,
            "preserve": [int(pm.size), int(pn.size)], "outer": r.outerIterations, "maxNI": r.maxNI,
            "largest_region": r.largestRegion,
            "phases_ms": {k: round(v, 3) for k, v in r.phase_ms.items()},
            "G_matches_oracle": hashlib.sha256(G.cpu().numpy().tobytes()).hexdigest() == d.get("G_sha"),
            "g_matches_oracle": hashlib.sha256(g.cpu().numpy().tobytes()).hexdigest() == d.get("g_sha"),
            "oracle_cpu_s": (d.get("oracle_seconds") or {}).get("simplify"),
        }
        del fd, F, g, G
        N.release_workspaces()  # the next config allocates its own workspace into free memory
        torch.cuda.empty_cache()
    return out


def large_field_kernels(dev, hbm):
    """Order-field sort and classification timed on a cfg5-shaped 512^3 field."""
    import torch

    import paper_2009_00083_b200 as P
    from paper_2009_00083_b200 import _native as N
    Nn = 512
    r = np.random.default_rng(0)
    waves = [(r.integers(1, 7, 3), r.uniform(0, 2 * np.pi), r.uniform(0.2, 1.0)) for _ in range(8)]
    x = torch.arange(Nn, dtype=torch.float64, device=dev)
    f = torch.empty((Nn, Nn, Nn), dtype=torch.float32, device=dev)
    gen = torch.Generator(device=dev)
    gen.manual_seed(5)
    for z0 in range(0, Nn, 64):
        z = x[z0:z0 + 64].view(-1, 1, 1)
        s = torch.zeros((z.shape[0], Nn, Nn), dtype=torch.float64, device=dev)
        for k, ph, a in waves:
            s += a * torch.sin(2 * np.pi * (int(k[0]) * x.view(1, 1, -1) + int(k[1]) * x.view(1, -1, 1)
                                            + int(k[2]) * z) / Nn + ph)
        s += torch.randn(s.shape, dtype=torch.float64, device=dev, generator=gen) * 0.02
        f[z0:z0 + 64] = s.float()
    mesh = P.build_grid_triangulation((Nn, Nn, Nn))
    ws = N.workspace(mesh.grid_dims, dev)
    kms = (ctypes.c_double * 4)()
    N.check(N.load().lts_bench_kernels(N.ptr(f.view(-1)), 3, N.dims_arg(mesh.grid_dims), 10, kms, N.ptr(ws),
                                       ws.numel(), N.stream_ptr()))
    n = mesh.n
    del ws
    N._ws_cache.clear()
    torch.cuda.empty_cache()
    out = {"config": "cfg5-3d-512-sin8 shape and distribution (waves as synthetic.cfg5, noise drawn "
                     "on the device)", "n": n}
    for key, ms, b in (("order_sort", kms[0], 64), ("classify", kms[1], 5), ("classify_ascent", kms[2], 9)):
        gbs = b * n / (ms * 1e-3) / 1e9
        out[key] = {"ms": ms, "bytes_per_voxel": b, "achieved_gbs": gbs, "frac": gbs / hbm}
    return out


def grid2d_kernels(dev, hbm):
    """Order-field sort and classification timed on cfg4's 4096^2 field (the
    2-D stencil path: six neighbours, tile kernel)."""
    import torch

    import paper_2009_00083_b200 as P
    from paper_2009_00083_b200 import _native as N
    from paper_2009_00083_b200 import synthetic as S
    C = S.CONFIGS[4]
    f = torch.from_numpy(S.make_field(4, 0).ravel()).to(dev)
    mesh = P.build_grid_triangulation(C.dims)
    ws = N.workspace(mesh.grid_dims, dev)
    kms = (ctypes.c_double * 4)()
    N.check(N.load().lts_bench_kernels(N.ptr(f), 2, N.dims_arg(mesh.grid_dims), 10, kms, N.ptr(ws), ws.numel(),
                                       N.stream_ptr()))
    n = mesh.n
    del ws
    N.release_workspaces()
    torch.cuda.empty_cache()
    out = {"config": C.name, "n": n}
    for key, ms, b in (("order_sort", kms[0], 64), ("classify", kms[1], 5), ("classify_ascent", kms[2], 9)):
        gbs = b * n / (ms * 1e-3) / 1e9
        out[key] = {"ms": ms, "bytes_per_voxel": b, "achieved_gbs": gbs, "frac": gbs / hbm}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-large", action="store_true", help="skip the 512^3 kernel roofline block")
    ap.add_argument("--no-configs", action="store_true", help="skip the other-configs block")
    ap.add_argument("--configs-budget", type=float, default=240.0,
                    help="wall seconds after which the other-configs block stops starting configs")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (rendezvous on 127.0.0.1)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", os.environ.get("MASTER_PORT", "29517"),
               os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if args.impl == "reference":
        return reference_arm(args)

    import torch
    import paper_2009_00083_b200 as P
    from paper_2009_00083_b200 import _native as N
    from paper_2009_00083_b200 import synthetic as S

    from paper_2009_00083_b200 import replicas as R
    rank, world, local = R.env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    R.init("nccl", dev)

    cfg = S.CONFIGS[args.config]
    f3d = S.make_field(args.config, args.seed)
    f_host = torch.from_numpy(f3d.ravel()).pin_memory()
    n = f_host.numel()
    mesh = P.build_grid_triangulation(cfg.dims)
    f_dev = f_host.to(dev)
    # preserve lists: harness work outside the timed region
    F = P.compute_order_field(P.ScalarField(mesh, f_dev))
    mn, mx = P.extrema(mesh, F)
    pm, pn = S.select_preserved(F.rank32.cpu().numpy(), mx.cpu().numpy(), mn.cpu().numpy(),
                                cfg.n_keep_max, cfg.n_keep_min)
    pm_d = torch.from_numpy(pm).to(dev)
    pn_d = torch.from_numpy(pn).to(dev)
    g = torch.empty(n, dtype=torch.float32, device=dev)
    G = torch.empty(n, dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    opt_timed = P.SimplifyOptions(collectTiming=True)
    opt = P.SimplifyOptions()

    def step(o):
        return P.simplify_raw(mesh, f_dev, pm_d, pn_d, None, o, g, G)

    for _ in range(args.warmup):
        step(opt)
    torch.cuda.synchronize()

    # ---- device-resident timed region -------------------------------------
    stream = torch.cuda.current_stream()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    launches0 = N.kernel_launches()
    R.barrier()
    torch.cuda.synchronize()
    with Clocks(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record(stream)
            step(opt)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
    launches = N.kernel_launches() - launches0
    step_ms = [a.elapsed_time(b) for a, b in evs]
    t_ms = R.max_over_ranks(sum(step_ms), dev)
    R.barrier()
    ms_per_step = t_ms / args.steps
    value = R.job_throughput(n, world, ms_per_step)

    # ---- phase breakdown (library CUDA events on the launching stream) ------
    flush.zero_()
    _, _, rep = step(opt_timed)
    phases = {name: round(float(rep.phase_ms[i]), 4) for i, name in enumerate(N.PHASES)}
    report = P.engine._report(rep)

    # ---- kernel rooflines: order-field sort and classification -------------
    hbm, peak_kind = peaks()
    ws = N.workspace(mesh.grid_dims, dev)
    L = N.load()
    dims = N.dims_arg(mesh.grid_dims)

    kms = (ctypes.c_double * 4)()
    N.check(L.lts_bench_kernels(N.ptr(f_dev), mesh.dim, dims, 10, kms, N.ptr(ws), ws.numel(),
                                N.stream_ptr()))
    sort_ms, cls_ms, clsptr_ms = kms[0], kms[1], kms[2]
    # algorithmic bytes per voxel: sort 64 B (hist read 4; pass 1
    # read 4 write 8; passes 2-3 read 8 write 8; pass 4 read 8, write inverse 4
    # + rank 4), classification 5 B (rank read 4, flags write 1)
    sort_gbs = 64.0 * n / (sort_ms * 1e-3) / 1e9
    cls_gbs = 5.0 * n / (cls_ms * 1e-3) / 1e9
    traffic = {}
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp))
    kernels = {
        "order_sort": {"ms": sort_ms, "bytes_per_voxel": 64, "achieved_gbs": sort_gbs,
                       "frac": sort_gbs / hbm, "traffic": traffic.get("order_sort")},
        "classify": {"ms": cls_ms, "bytes_per_voxel": 5, "achieved_gbs": cls_gbs,
                     "frac": cls_gbs / hbm, "traffic": traffic.get("classify")},
        "classify_ascent": {"ms": clsptr_ms, "bytes_per_voxel": 9,
                            "achieved_gbs": 9.0 * n / (clsptr_ms * 1e-3) / 1e9,
                            "frac": 9.0 * n / (clsptr_ms * 1e-3) / 1e9 / hbm,
                            "traffic": traffic.get("classify_ascent")},
    }
    # dominant kernels: the large-region floods (k_big_flood for the smooth
    # mid-sized regions beside k_lv_coop, the level-parallel floods of the rough
    # and the largest regions), timed together by the library with CUDA events
    # on the streams they run on.  Algorithmic bytes per flooded region slot:
    # its neighbour-key row (4 K B), its key -> index entry (4 B) and its label
    # (4 B); DESIGN.md section 4.
    K = 14 if mesh.dim == 3 else 6
    flood_ms = float(rep.phase_ms[9])
    flood_launches = int(rep.phase_ms[N.PH_FLOOD_LAUNCHES])
    flood_slots = float(rep.phase_ms[N.PH_FLOOD_SLOTS])
    per_launch_ms = flood_ms / max(flood_launches, 1)
    flood_bytes = (4.0 * K + 8.0) * flood_slots / max(flood_launches, 1)
    flood_gbs = flood_bytes / (per_launch_ms * 1e-3) / 1e9 if per_launch_ms > 0 else 0.0
    roofline = {"bound": "hbm", "kernel": "k_big_flood || k_lv_coop", "achieved": flood_gbs, "peak": hbm,
                "unit": "GB/s", "frac": flood_gbs / hbm, "traffic": traffic.get("k_big_flood || k_lv_coop", traffic.get("k_big_flood")),
                "peak_source": peak_kind, "launches": flood_launches, "ms_per_launch": per_launch_ms,
                "bytes_per_launch": flood_bytes,
                "share_of_step": flood_ms / phases["total"] if phases["total"] else None,
                "slots_per_s": flood_slots / (flood_ms * 1e-3) if flood_ms > 0 else None,
                "note": "latency-bound exact priority floods: one CTA per smooth region (about one L2 "
                        "round trip and five barriers per batched step) beside the level-parallel "
                        "decomposition (one grid barrier per phase); DESIGN.md section 4a"}

    # ---- end to end through the public API with host buffers ---------------
    g_host = torch.empty(n, dtype=torch.float32).pin_memory()
    G_host = torch.empty(n, dtype=torch.int32).pin_memory()
    pm_h = torch.from_numpy(pm).pin_memory()
    pn_h = torch.from_numpy(pn).pin_memory()
    # the public host-buffer call (engine.simplify_field_host -> lts_simplify_host):
    # pinned f and preserve lists in, pinned g and G out, every copy inside
    pres_h = P.ConstraintSet(preserveMinima=pn_h.numpy(), preserveMaxima=pm_h.numpy())
    with torch.cuda.device(dev):
        gq, Gq, _ = P.simplify_field_host(mesh, f_host, pres_h, opt, g_host, G_host, device=dev)
    torch.cuda.synchronize()
    # the host outputs equal the device-resident call's
    assert torch.equal(G_host, G.cpu()) and g_host.numpy().tobytes() == g.cpu().numpy().tobytes()

    def e2e_step():
        P.simplify_field_host(mesh, f_host, pres_h, opt, g_host, G_host, device=dev)

    e2e_step()
    torch.cuda.synchronize()
    e_ms = []
    for _ in range(max(3, min(args.steps, 5))):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        e2e_step()
        b.record(stream)
        torch.cuda.synchronize()
        e_ms.append(a.elapsed_time(b))
    e2e_t = R.max_over_ranks(sum(e_ms) / len(e_ms), dev)
    e2e = {"value": R.job_throughput(n, world, e2e_t), "unit": UNIT,
           "h2d_bytes_per_step": 4 * n + 8 * (pm.size + pn.size), "d2h_bytes_per_step": 8 * n,
           "ms_per_step": e2e_t}

    # ---- kernel rooflines at BASELINE's large-field roofline config ----------
    # cfg5 (512^3): the same eight waves as synthetic.cfg5 (numpy draws), the
    # N(0, 0.02) noise drawn on the device (torch generator) so the field is
    # built in well under a second; kernels as above (rank 0, N = 1).
    kernels_large = kernels_2d = None
    if rank == 0 and world == 1 and not args.no_large:
        kernels_large = large_field_kernels(dev, hbm)
        kernels_2d = grid2d_kernels(dev, hbm)

    # ---- other BASELINE configs (rank 0, N = 1) -------------------------------
    configs = None
    if rank == 0 and world == 1 and not args.no_configs:
        configs = other_configs(dev, args.configs_budget)

    # ---- CPU baseline (rank 0, N = 1): the same full pass on the host --------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        dims_s, fr, pms, pns = cpu_workload(f3d, cfg)
        threads = os.cpu_count() or 1
        dt = run_oracle(dims_s, fr, pms, pns, threads)
        cpu = {"value": fr.size / dt, "unit": UNIT, "cores": threads, "kind": "port",
               "cpu_model": cpu_model(),
               "sample": (f"the full workload ({cfg.name}, {fr.size} voxels, preserve {pms.size} max / "
                          f"{pns.size} min), one full pass, {dt:.1f} s; OpenMP in classify/localize, "
                          f"discover/sort/realize sequential as in the reference")}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(cfg, args, n, (pm.size, pn.size), world),
            "e2e": e2e, "gpu_launches": int(launches), "roofline": roofline, "kernels": kernels,
            "kernels_large": kernels_large, "kernels_2d": kernels_2d,
            "phases_ms": phases, "cpu_baseline": cpu, "clocks": clk.summary(), "configs": configs,
            "report": {"ok": report.ok, "outer": report.outerIterations,
                       "passes": [p.__dict__ for p in report.passes]},
            "step_ms": step_ms,
        }
        print(json.dumps(line), flush=True)
    R.shutdown()


if __name__ == "__main__":
    main()
