#!/usr/bin/env python
"""J-FFT PCG throughput on B200 (BASELINE.json metric: GDOF-iterations/s, fp64,
3-D 512^3, and the fraction of the HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload 3d512|3d128|2d2048] [--kind green-jacobi|green]

A "step" is one fixed-length PCG solve (``--iters`` iterations, eta = -1 so
no early exit) over the resident synthetic problem: BASELINE config 4, a
512^3 crack-disc damage field (E = (1-phi)^2 + 1e-4, nu = 0.3, eps_xx = 1),
Green-Jacobi preconditioner.  value = d * N * iterations * K / time / 1e9.
Only the PCG iterations are credited; each step's init (k = 0 preconditioner
application) and the final mean subtraction run inside the timed region.

--impl reference times the reference algorithm's CPU implementation (the
NumPy oracle port, oracle/jfft_oracle.py -- the reference is pure Python and
cannot be built into oracle/_ref) on the host's cores with the same metric.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

WORKLOADS = {
    # name: (d, n, generator, eps_bar)
    "3d512": (3, 512, "cracks", [1.0, 0, 0, 0, 0, 0]),
    "3d128": (3, 128, "spheres", [1.0, 0, 0, 0, 0, 0]),
    "3d256": (3, 256, "cracks", [1.0, 0, 0, 0, 0, 0]),
    "2d2048": (2, 2048, "bernoulli20", [0.0, 0.0, np.sqrt(2.0) * 0.5]),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="3d512", choices=sorted(WORKLOADS))
    ap.add_argument("--kind", default="green-jacobi", choices=["green-jacobi", "green"])
    ap.add_argument("--iters", type=int, default=50,
                    help="PCG iterations per step (SURVEY 8d throughput mode: 50 at 512^3)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="use the distributed (slab) library path even at N = 1")
    return ap.parse_args()


def peak_hbm():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(
                        ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                         "--format=csv,noheader,nounits"], capture_output=True, text=True,
                        timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for k, nm in enumerate(names):
                if len(r) > 5 + k and r[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# reference arm: the oracle port on the host cores
# ---------------------------------------------------------------------------
_W = {}


def _ref_worker_init(d, n, kind, seed):
    from oracle import jfft_oracle as X
    from paper_2508_02613_b200 import microstructures as ms
    lam, mu = ms.lame_from_poisson()
    if d == 3:
        rho = ms.crack_discs(n, count=max(1, 64 * n ** 3 // 512 ** 3), seed=seed)
        eb = np.array([1.0, 0, 0, 0, 0, 0])
    else:
        rho = ms.bernoulli_smoothed(n, 20, 1e4, seed)
        eb = np.array([0.0, 0.0, np.sqrt(2.0) * 0.5])
    c = X.isotropic_stiffness(d, lam, mu)
    h = X.pixel_size((n,) * d, (1.0,) * d)
    _W.update(X=X, rho=rho, c=c, h=h, kind=kind,
              blocks=X.assemble_green((n,) * d, (1.0,) * d, c),
              inv=X.assemble_jacobi(rho, c, h), rhs=X.assemble_rhs(rho, c, h, eb))


def _ref_worker_solve(iters):
    X = _W["X"]
    t0 = time.perf_counter()
    X.pcg(_W["rho"], _W["c"], _W["h"], _W["rhs"], _W["kind"], _W["blocks"], _W["inv"],
          eta=-1.0, max_iter=iters)
    return time.perf_counter() - t0


def cpu_sample_n(d):
    """the CPU baseline runs the oracle at 128^3 (BASELINE config
    3's size) on a sample of the workload generator; 2-D at 1024^2."""
    return 128 if d == 3 else 1024


def host_info():
    """CPU model, core count, NumPy / BLAS versions and the BLAS thread
    setting of the host the CPU arm runs on."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = "unknown"
    try:
        cfg = np.show_config(mode="dicts")
        b = cfg.get("Build Dependencies", {}).get("blas", {})
        blas = f"{b.get('name', '?')} {b.get('version', '?')}"
    except Exception:
        pass
    mem = os.sysconf("SC_PHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    return {"cpu_model": model, "nproc": os.cpu_count(), "host_mem_gb": round(mem / 2 ** 30, 1),
            "numpy": np.__version__, "blas": blas,
            "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS", "unset")}


def run_reference(args, rank):
    if rank != 0:
        return None
    import multiprocessing as mp
    d, nfull, _, _ = WORKLOADS[args.workload]
    n = cpu_sample_n(d)
    info = host_info()
    # one single-threaded oracle solve per core, as many as host memory holds
    # (a 128^3 oracle solve peaks at ~4 GB)
    per_proc_gb = 4.5 if d == 3 else 1.0
    cores = max(1, min(os.cpu_count() or 1, int(info["host_mem_gb"] * 0.8 // per_proc_gb)))
    iters = 2
    os.environ["OPENBLAS_NUM_THREADS"] = "1"  # NumPy's kernels here are single-threaded anyway
    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=_ref_worker_init, initargs=(d, n, args.kind, 0)) as pool:
        for _ in range(max(args.warmup, 0)):
            pool.map(_ref_worker_solve, [1] * cores)
        t0 = time.perf_counter()
        for _ in range(args.steps):
            pool.map(_ref_worker_solve, [iters] * cores)
        dt = time.perf_counter() - t0
    dof_it = d * n ** d * iters * cores * args.steps
    value = dof_it / dt / 1e9
    sample = (f"{cores} concurrent single-threaded oracle PCG solves ({args.kind}) of the "
              f"{n}^{d} sample per step, {iters} iterations each (the {nfull}^{d} cell needs "
              f"~60 GB and ~150 s per iteration in the NumPy oracle)")
    line = {
        "impl": "reference", "metric": metric_name(args), "value": value, "unit": "GDOF-it/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_of(args),
        "cpu_baseline": {"value": value, "unit": "GDOF-it/s", "cores": cores, "kind": "port",
                         "sample": sample, "host": info},
        "e2e": {"value": value, "unit": "GDOF-it/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    return line


def cpu_baseline_single(args):
    """The oracle port, 1 core, a bounded sample of the workload (rank 0, N=1)."""
    d = WORKLOADS[args.workload][0]
    n = cpu_sample_n(d)
    _ref_worker_init(d, n, args.kind, 0)
    _ref_worker_solve(1)
    iters = 3
    t = _ref_worker_solve(iters)
    return {"value": d * n ** d * iters / t / 1e9, "unit": "GDOF-it/s", "cores": 1,
            "kind": "port",
            "sample": f"oracle PCG ({args.kind}) on a {n}^{d} sample of the workload "
                      f"generator, {iters} iterations, {t:.1f} s, numpy single-threaded "
                      "(1 core used)",
            "host": host_info()}


def metric_name(args):
    d, n, _, _ = WORKLOADS[args.workload]
    return f"J-FFT PCG GDOF-iterations/s (fp64, {d}D {n}^{d})"


def config_of(args):
    d, n, gen, _ = WORKLOADS[args.workload]
    return {"workload": f"{args.workload}-{gen}-{args.kind}", "d": d, "n": n,
            "kind": args.kind, "iterations_per_step": args.iters,
            "mode": "fixed-iteration throughput (eta=-1); parity solves are in tests/",
            "l2": "inputs larger than L2 (one vector field = %.1f GiB)" % (d * n ** d * 8 / 2 ** 30),
            "parallelism": "replicas" if args.gpus > 1 else "single"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def build_problem(args, torch, dev):
    from paper_2508_02613_b200 import _native as N
    from paper_2508_02613_b200 import microstructures as ms
    d, n, gen, eb = WORKLOADS[args.workload]
    lam, mu = ms.lame_from_poisson()
    shape = (n,) * d
    if gen == "cracks":
        rho = ms.crack_discs_device(n, seed=0, device=dev)
    elif gen == "spheres":
        rho = torch.from_numpy(ms.random_spheres(n, seed=0)).to(dev)
    else:
        rho = torch.from_numpy(ms.bernoulli_smoothed(n, 20, 1e4, 0)).to(dev)
    gh = N.GridHandle(d, shape, (1.0,) * d, device=torch.cuda.current_device())
    gh.set_stream(torch.cuda.current_stream().cuda_stream)
    N.register_grid(gh)  # the public-API (e2e) leg shares this context
    op = N.OpHandle(gh, rho.data_ptr(), lam, mu, where=N.DEVICE)
    green = N.GreenHandle(gh, lam, mu)
    jac = N.JacobiHandle(op) if args.kind == "green-jacobi" else None
    rhs = torch.empty((d,) + shape, dtype=torch.float64, device=dev)
    ebv = np.ascontiguousarray(eb, dtype=np.float64)
    N.check(N.load().jfftb_assemble_rhs(op.ptr, N.dptr(ebv), rhs.data_ptr(), N.DEVICE))
    x = torch.empty_like(rhs)
    torch.cuda.synchronize()
    return dict(d=d, n=n, N=n ** d, gh=gh, op=op, green=green, jac=jac, rhs=rhs, x=x, rho=rho,
                lam=lam, mu=mu, eb=ebv)


def run_ours(args, rank, world):
    import torch
    import torch.distributed as dist
    from paper_2508_02613_b200 import _native as N
    from paper_2508_02613_b200 import roofline as R
    from paper_2508_02613_b200.solver import pcg_device

    dev = torch.device("cuda", torch.cuda.current_device())
    P = build_problem(args, torch, dev)
    d, Nn = P["d"], P["N"]

    def step():
        pcg_device(P["op"], args.kind, P["green"], P["jac"], P["rhs"].data_ptr(),
                   P["x"].data_ptr(), -1.0, args.iters)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(torch.cuda.current_device())
    clocks.start()
    N.launch_count(reset=True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = N.launch_count(reset=True)
    # stage breakdown from one extra, separately profiled step (the timed
    # steps above run without the per-stage events)
    P["gh"].profile_start()
    step()
    torch.cuda.synchronize()
    stage_ms, prof_iters = P["gh"].profile_read(stop=True)
    ms_total = ev0.elapsed_time(ev1)
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    iters_total = args.iters * args.steps
    value = world * d * Nn * iters_total / (ms_total / 1e3) / 1e9

    # ---- roofline: whole iteration (north star) and dominant stage --------
    peak, peak_src = peak_hbm()
    per_iter_ms = ms_total / iters_total
    alg_iter = R.algorithmic_bytes(args.kind, d, Nn)
    # power-of-two grids run the fused FFT passes (fused.cu) unless disabled
    fused_path = (all(k & (k - 1) == 0 and 16 <= k <= 2048 for k in P["gh"].shape)
                  and os.environ.get("JFFTB_DISABLE_FUSED") != "1")
    stages = {}
    for k, nm in enumerate(R.STAGES):
        if prof_iters:
            avg = stage_ms[k] / prof_iters
            b = R.kernel_bytes(nm, args.kind, d, Nn, fused=fused_path)
            stages[nm] = {"ms": avg, "share": stage_ms[k] / max(stage_ms.sum(), 1e-30),
                          "alg_bytes": b, "GBps": (b / (avg / 1e3) / 1e9) if avg > 0 and b else None}
    ours = {k: v for k, v in stages.items() if not k.startswith("fft")}
    dom_all = max(stages, key=lambda k: stages[k]["ms"]) if stages else None
    dom = max(ours, key=lambda k: ours[k]["ms"]) if ours else None
    traffic = None
    tpath = os.path.join(REPO, "profiles", "traffic.json")
    if dom and os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"{args.workload}:{args.kind}:{dom}")
        except Exception:
            traffic = None
    roof = None
    if dom:
        ach = stages[dom]["GBps"]
        roof = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak if ach else None, "traffic": traffic,
                "alg_bytes_per_launch": stages[dom]["alg_bytes"], "ms_per_launch": stages[dom]["ms"],
                "peak_source": peak_src,
                "note": f"dominant stage overall: {dom_all} "
                        f"({stages[dom_all]['share']:.0%} of the iteration)"}
    ach_it = alg_iter / (per_iter_ms / 1e3) / 1e9
    roof_it = {"bound": "hbm", "achieved": ach_it, "peak": peak, "unit": "GB/s",
               "frac": ach_it / peak, "frac_of_8TBps": ach_it / 8000.0,
               "alg_bytes_per_iteration": alg_iter, "ms_per_iteration": per_iter_ms,
               "model": "fused minimum (18d+1)U / (14d+1)U, SURVEY 8(d)"}

    # ---- e2e through the public API with host (pinned) buffers -----------
    e2e = e2e_pg = None
    if args.e2e_steps > 0:
        e2e = run_e2e(args, P, torch, world)
        # the reference hands over plain (pageable) NumPy arrays
        e2e_pg = run_e2e(args, P, torch, world, pageable=True)

    line = {
        "metric": metric_name(args), "value": value, "unit": "GDOF-it/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE.json config generator; see DESIGN.md)",
        "config": config_of(args), "roofline": roof, "roofline_iteration": roof_it,
        "stages_ms_per_iteration": {k: round(v["ms"], 4) for k, v in stages.items()},
        "e2e": e2e, "e2e_pageable": e2e_pg, "gpu_launches": int(launches), "clocks": clk,
    }
    return line


def weak_shape(n, world):
    """Per-GPU work fixed at n^3 nodes: 2 -> (n, 2n, n), 4 -> (n, 2n, 2n),
    8 -> (2n)^3 (= BASELINE config 5, 1024^3 on 8 GPUs for n = 512).  Axis 1
    (the slab axis) and axis 2 grow before axis 0: the axis-0 passes hold a
    whole column per tile and lose their 128-byte row segments at n0 = 2n
    (measured per rank: 20.1 ms per iteration on (1024, 256, 512) against
    18.3 ms on 512^3)."""
    shape = [n, n, n]
    w, a = world, 0
    order = (1, 2, 0)
    while w > 1:
        shape[order[a % 3]] *= 2
        w //= 2
        a += 1
    return tuple(shape)


def run_dist(args, rank, world):
    """N > 1 (or --dist): the slab-decomposed solver inside libjfftb200
    (csrc/dist.cu via paper_2508_02613_b200.dist): fused passes per rank,
    NCCL halo rows / all-to-all / all-gathers on the solver's stream, device
    scalars; weak scaling (the 512^3 cell per GPU)."""
    import torch
    import torch.distributed as dist
    from paper_2508_02613_b200 import _native as N
    from paper_2508_02613_b200 import dist as Dm
    from paper_2508_02613_b200 import microstructures as ms
    from paper_2508_02613_b200 import roofline as R
    d, n, gen, eb = WORKLOADS[args.workload]
    assert d == 3, "slab decomposition is 3-D; 2-D runs as replicas"
    shape = weak_shape(n, world)
    lengths = tuple(k / n for k in shape)  # same pixel size as the 1-GPU cell
    dev = torch.device("cuda", torch.cuda.current_device())
    lam, mu = ms.lame_from_poisson()
    count = int(round(64 * (shape[0] * shape[1] * shape[2]) / 512 ** 3))
    lo, hi = Dm.slab_rows(shape[1], world, rank)
    rho = ms.crack_discs_device(shape, count=count, seed=0, device=dev, rows=(lo, hi))
    comm = Dm.Comm.nccl_from_torch()
    solver = Dm.DistSolver(comm, shape, lengths, rho.contiguous(), lam, mu, kind=args.kind)
    del rho
    rhs = solver.assemble_rhs(np.asarray(eb, dtype=np.float64), device=torch.empty(1, device=dev))
    x = torch.empty_like(rhs)
    torch.cuda.synchronize()

    def step():
        solver.pcg(rhs, eta=-1.0, max_iter=args.iters, x_out=x)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    dist.barrier()
    clocks = Clocks(torch.cuda.current_device())
    clocks.start()
    N.launch_count(reset=True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    dist.barrier()
    clk = clocks.stop()
    launches = N.launch_count(reset=True)
    t = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    Ng = shape[0] * shape[1] * shape[2]
    iters_total = args.iters * args.steps
    value = 3 * Ng * iters_total / (ms_total / 1e3) / 1e9
    peak, peak_src = peak_hbm()
    per_iter_ms = ms_total / iters_total
    alg = R.algorithmic_bytes(args.kind, 3, Ng // world)  # per GPU
    ach = alg / (per_iter_ms / 1e3) / 1e9
    roof = {"bound": "hbm", "kernel": "pcg-iteration (distributed, per GPU)", "achieved": ach,
            "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": None,
            "alg_bytes_per_launch": alg, "ms_per_launch": per_iter_ms, "peak_source": peak_src}
    # e2e: the rhs from pinned host memory and the solution back, every step,
    # through the same public call with host buffers
    rhs_h = torch.empty(rhs.shape, dtype=torch.float64, pin_memory=True)
    rhs_h.copy_(rhs)
    x_h = torch.empty_like(rhs_h, pin_memory=True)
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(max(args.e2e_steps, 1)):
        solver.pcg(rhs_h.numpy(), eta=-1.0, max_iter=args.iters, x_out=x_h.numpy())
    te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_v = 3 * Ng * args.iters * max(args.e2e_steps, 1) / float(te.item()) / 1e9
    cfg = config_of(args)
    cfg.update({"shape": list(shape), "parallelism": f"slab{world} (axis-1 real slabs / k0 "
                "spectral slabs in libjfftb200; NCCL halo rows + all-to-all + all-gather)",
                "nodes_per_gpu": Ng // world})
    return {
        "metric": metric_name(args), "value": value, "unit": "GDOF-it/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded crack-disc field on the weak-scaled cell; see DESIGN.md)",
        "config": cfg, "roofline": roof, "roofline_iteration": roof,
        "e2e": {"value": e2e_v, "unit": "GDOF-it/s",
                "h2d_bytes_per_step": int(rhs.numel() * 8 * world),
                "d2h_bytes_per_step": int(rhs.numel() * 8 * world)},
        "gpu_launches": int(launches), "clocks": clk,
    }


def run_e2e(args, P, torch, world, pageable=False):
    from paper_2508_02613_b200 import grid as G
    from paper_2508_02613_b200.material import isotropic_material
    from paper_2508_02613_b200.operators import make_operator, op_handle
    from paper_2508_02613_b200.preconditioners import GreenOperator, JacobiDiagonal, Preconditioner
    from paper_2508_02613_b200.solver import pcg
    d, n = P["d"], P["n"]
    grid = G.make_grid(n, (1.0,) * d)
    mat = isotropic_material(P["lam"], P["mu"], d)
    # density and rhs live in pinned host memory (the caller's buffers)
    rho_h = torch.empty(P["rho"].shape, dtype=torch.float64, pin_memory=not pageable)
    rho_h.copy_(P["rho"])
    rhs_h = torch.empty(P["rhs"].shape, dtype=torch.float64, pin_memory=not pageable)
    rhs_h.copy_(P["rhs"])
    if pageable:  # plain NumPy arrays, as the reference's callers hold them
        rho_h, rhs_h = rho_h.numpy().copy(), rhs_h.numpy().copy()
        rho_np, rhs_np = rho_h, rhs_h
    else:
        rho_np, rhs_np = rho_h.numpy(), rhs_h.numpy()
    op = make_operator(G.ScalarField(grid, rho_np), mat)
    op_handle(op)  # operator assembly (density upload) is setup, as in the reference
    green = GreenOperator(grid, mat, P["green"])
    jac = JacobiDiagonal(grid, P["jac"]) if P["jac"] is not None else None
    pre = Preconditioner(args.kind, green=green, jacobi=jac)
    rhs = G.VectorField(grid, rhs_np)
    pcg(op, rhs, pre, green, eta=-1.0, max_iter=args.iters)  # warm
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        rep = pcg(op, rhs, pre, green, eta=-1.0, max_iter=args.iters)
        _ = float(rep.solution.values[0].ravel()[0])
    dt = time.perf_counter() - t0
    value = world * d * n ** d * args.iters * args.e2e_steps / dt / 1e9
    nbytes = d * n ** d * 8
    return {"value": value, "unit": "GDOF-it/s", "h2d_bytes_per_step": nbytes,
            "d2h_bytes_per_step": nbytes + 8 * (args.iters + 1),
            "api": "paper_2508_02613_b200.pcg(op, rhs, preconditioner, green) host VectorField "
                   f"({'pageable NumPy' if pageable else 'pinned'}), solution returned on the "
                   "host (a fresh NumPy array)"}


def _json_stdout():
    """The driver reads exactly one JSON line from stdout.  Libraries may
    print to file descriptor 1 (NCCL's version banner under torchrun), so fd 1
    is pointed at stderr for the whole run and the result line goes to a
    duplicate of the original stdout."""
    sys.stdout.flush()
    out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    return out


def _emit(out, line):
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    args = parse()
    out = _json_stdout()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        line = run_reference(args, rank)
        if line is not None:
            _emit(out, line)
        return
    import torch
    import torch.distributed as dist
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ["JFFTB_DEVICE"] = str(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if (world > 1 or args.dist) and WORKLOADS[args.workload][0] == 3:
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            dist.init_process_group("nccl", rank=0, world_size=1,
                                    device_id=torch.device("cuda", local))
        line = run_dist(args, rank, world)
    else:
        line = run_ours(args, rank, world)
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline_single(args)
        _emit(out, line)
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
