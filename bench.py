#!/usr/bin/env python
"""Benchmark of the hot path: mixed-precision preconditioned BiCGStab on the operational-size grid.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C5]

One STEP = one pass of every SURVEY.md §8(a) row over the resident synthetic problem:
    eg_solver_set_operator (a1: diagonal scaling of the 7 fp64 bands)  +
    eg_solve(b, x0 = 0, tol = 0, maxit = 8)  (a2 entry, 8 x a3-a10, a11 true-residual verification)
value = BiCGStab iterations per second of the whole job = 8 * K / (device time of K steps),
max over ranks.  For N > 1 (torchrun) the grid is split into latitude bands (strong scaling).

Timing: CUDA events on the solver's stream, barrier + synchronize on both sides.  Inputs are far
larger than L2 (46.8 GB of algorithmic traffic per iteration at C5), so no L2 flush is needed.
The `--impl reference` arm times the CPU oracle (oracle/) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BiCGStab iters/s & time-to-solve, 2560×1920×70 fp32; achieved HBM GB/s"
ITERS_PER_STEP = 8
# algorithmic HBM bytes per grid point per BiCGStab iteration:
# 18 vector + 12 band + 2 x accesses: MIXED 136, FP64 256, FP32 128
B_ALG = {"mixed": 136, "fp64": 256, "fp32": 128}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class Clocks:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line).  The sampler is
    started before the region; only samples whose timestamps fall inside [mark_start, mark_end]
    are summarised."""

    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.p = None
        self.t0 = self.t1 = None
        self.lines = []

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(1.0)  # let the sampler come up before the timed region
        except Exception:
            self.p = None
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def __exit__(self, *a):
        if self.p is not None:
            time.sleep(0.2)
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
                self.lines = [l for l in out.splitlines() if l.strip()]
            except Exception:
                self.p.kill()

    def summary(self):
        import datetime
        sm, mx, reasons, n_all = [], 0.0, set(), 0
        for l in self.lines:
            f = [t.strip() for t in l.split(",")]
            if len(f) < 8:
                continue
            n_all += 1
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                ts = None
            if ts is not None and self.t0 is not None and not (self.t0 - 0.05 <= ts <= self.t1 + 0.05):
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no nvidia-smi sample in window"],
                    "samples_total": n_all}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def spawn_ranks(n):
    """`--gpus N` without a launcher: re-exec this script under torch.distributed.run with N ranks on
    this node (127.0.0.1 rendezvous), exactly as the driver launches it; rank 0 prints the line."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.stdout.flush()
    os.execv(sys.executable, cmd)


def dist_init(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        backend = "gloo" if args.impl == "reference" else "nccl"
        if backend == "nccl":
            import torch
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
        print(f"bench.py: rank {rank}/{ws} process group backend {dist.get_backend()}", file=sys.stderr, flush=True)
    return ws, rank, local


def oracle_sample(prob, precision, target_s=12.0):
    """Time the CPU oracle on a bounded latitude sample of the workload (same nx, nz, recipe): the
    step (oracle_scale + oracle_solve(tol=0, maxit=8)) on the rows of a 2560 x R x 70 sample, R
    chosen so the step takes ~target_s.  Per-iteration work is proportional to the points, so
    value = iterations / wall * (sample points / grid points) is the full grid's iters/s.
    Returns dict(value, seconds = the sample step's own wall time, ...)."""
    import gen
    import oracle
    rows = 8
    g = (prob.nx, rows, prob.nz)
    sub = prob.with_(ny=rows)
    bands, b = gen.host(sub)
    ahat, diag = oracle.scale(g, bands, precision)
    t0 = time.perf_counter()
    oracle.solve(g, precision, ahat, diag, b, tol=0.0, maxit=1)
    t1 = time.perf_counter() - t0
    # choose rows (multiple of 8, <= ny) and iterations so the run is ~target_s
    rows = int(max(8, min(prob.ny, 8 * round(rows * target_s / max(t1, 1e-3) / ITERS_PER_STEP / 8))))
    g = (prob.nx, rows, prob.nz)
    sub = prob.with_(ny=rows)
    bands, b = gen.host(sub)
    t0 = time.perf_counter()
    ahat, diag = oracle.scale(g, bands, precision)
    x, hist, info = oracle.solve(g, precision, ahat, diag, b, tol=0.0, maxit=ITERS_PER_STEP)
    dt = time.perf_counter() - t0
    frac = (prob.nx * rows * prob.nz) / prob.n
    return {
        "value": info.iters / dt * frac, "unit": "iter/s", "cores": oracle.threads(), "kind": "oracle",
        "cpu_model": cpu_model(),
        "sample": (f"oracle_scale + oracle_solve({precision}, tol=0, maxit={ITERS_PER_STEP}) on a "
                   f"{prob.nx}x{rows}x{prob.nz} latitude sample ({frac:.4f} of the grid) generated "
                   f"with the same recipe; {dt:.2f} s wall; iters/s scaled by the point ratio"),
        "sample_grid": [prob.nx, rows, prob.nz], "sample_fraction": frac,
        "seconds": dt,
    }


def run_reference(args, prob, ws, rank):
    """The reference arm: the CPU oracle as it stands, on this host's cores, each step a bounded
    latitude sample of the workload (oracle_sample).  ms_per_step is the sample step's own wall
    time (what this run spent), value the full grid's iters/s it implies (scaled by the point
    ratio).  Under torchrun only rank 0 works and prints; the other ranks exit without work."""
    if rank != 0:
        return
    import oracle  # the reference arm is the CPU oracle
    oracle.set_threads(os.cpu_count() or 1)  # all host cores, also under torchrun (OMP_NUM_THREADS=1)
    t_run = time.perf_counter()
    for _ in range(args.warmup):
        oracle_sample(prob, args.precision, target_s=min(1.0, args.ref_seconds))
    # each step ~ref_seconds, but the whole K-step run bounded to ~2 minutes
    per_step = min(args.ref_seconds, max(0.5, 120.0 / max(args.steps, 1)))
    vals, secs = [], []
    last = None
    for _ in range(args.steps):
        last = oracle_sample(prob, args.precision, target_s=per_step)
        vals.append(last["value"])
        secs.append(last["seconds"])
    v = statistics.median(vals)
    cfg = config_dict(args, prob, ws)
    cfg["reference_sample"] = (f"each step: the same step on a {last['sample_grid'][0]}x{last['sample_grid'][1]}x"
                               f"{last['sample_grid'][2]} latitude sample ({last['sample_fraction']:.4f} of the grid); "
                               "value scaled to the full grid by the point ratio")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "iter/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * statistics.median(secs),
        "full_grid_ms_per_step_extrapolated": 1000.0 * ITERS_PER_STEP / v,
        "wall_s": time.perf_counter() - t_run,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": DTYPE[args.precision],
        "data": "synthetic", "config": cfg,
        "cpu_baseline": {k: last[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model")},
        "e2e": {"value": v, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


DTYPE = {"mixed": "f32 (x, global sums f64)", "fp64": "f64", "fp32": "f32"}


def config_dict(args, prob, ws):
    return {
        "workload": (f"{args.config}: {prob.nx}x{prob.ny}x{prob.nz} seed {prob.seed}, "
                     f"c_v~U({prob.cv[0]:g},{prob.cv[1]:g}), {args.precision}, step = set_operator + "
                     f"solve(tol=0, maxit={ITERS_PER_STEP})"),
        "grid": [prob.nx, prob.ny, prob.nz], "precision": args.precision,
        "iters_per_step": ITERS_PER_STEP, "parallelism": f"latitude-bands x{ws}",
        "l2": "inputs larger than L2 (no flush needed)", "data": "synthetic (seeded generator, gen/)",
    }


def run_ours(args, prob, ws, rank, local):
    import numpy as np
    import torch

    import gen
    import paper_1811_03852_b200 as egs

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    group = None
    if ws > 1:
        import torch.distributed as dist
        group = dist.group.WORLD
    j0, j1 = egs.band_rows(prob.ny, rank, ws) if ws > 1 else (0, prob.ny)
    nloc = (j1 - j0) * prob.nx * prob.nz
    stream = torch.cuda.Stream(dev)
    with torch.cuda.stream(stream):
        bands = torch.empty((7, nloc), dtype=torch.float64, device=dev)
        b = torch.empty(nloc, dtype=torch.float64, device=dev)
        gen.device(prob, bands, b, j0, j1, stream=stream)
        x = torch.empty(nloc, dtype=torch.float64, device=dev)
        s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, args.precision, group=group, stream=stream,
                       batch=True)
    transport = s.transport  # latitude bands: "p2p" (NVLink peer memory) or "nccl"; one GPU: "none"

    def barrier():
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()

    def step(flags, bb=b, xx=x):
        s.set_operator(bands)
        _, info, _ = s.solve(bb, tol=0.0, maxit=ITERS_PER_STEP, flags=flags, out=xx)
        return info

    def timed(nsteps, flags, bb=b, xx=x):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        infos = [step(flags, bb, xx) for _ in range(nsteps)]
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        ms = ev0.elapsed_time(ev1)
        if ws > 1:
            import torch.distributed as dist
            t = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, infos

    # warm-up (also captures the CUDA graph), then the timed region with per-kernel events
    for _ in range(args.warmup):
        step(egs.EG_SOLVE_PROFILE)
    s.profile_reset()
    with Clocks(local) as clk:
        clk.mark_start()
        ms, infos = timed(args.steps, egs.EG_SOLVE_PROFILE)
        clk.mark_end()
    prof = s.profile()
    iters = sum(i.iters for i in infos)
    value = iters / (ms / 1000.0)
    launches = sum(v[1] for v in prof.values())

    # dominant kernel roofline (algorithmic bytes / average CUDA-event duration)
    peak, peak_src = peaks()
    kname, (kms, kn, kbytes) = max(((k, v) for k, v in prof.items() if v[1] > 0), key=lambda kv: kv[1][0])
    achieved = kbytes / (kms / kn / 1000.0) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(args.precision, {}).get(kname)
        except Exception:
            traffic = None
    kernels = {k: {"avg_ms": v[0] / v[1], "launches": v[1], "alg_GBps": v[2] / (v[0] / v[1] / 1e3) / 1e9,
                   "share": v[0] / sum(w[0] for w in prof.values())} for k, v in prof.items() if v[1] > 0}

    # graph-replay timing (no per-kernel events) for comparison
    ms_graph, infos_g = timed(args.steps, 0)
    iters_g = sum(i.iters for i in infos_g)

    # end to end through the public C-ABI with HOST buffers: every step uploads its b from pinned host
    # memory and downloads its x.  (1) eg_solve_batch over the K steps, which overlaps the transfers
    # of neighbouring steps with the solves (the headline e2e); (2) K blocking eg_solve calls.
    hb = [torch.empty(nloc, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    for h in hb:
        h.copy_(b)
    hx = [torch.empty(nloc, dtype=torch.float64, pin_memory=True) for _ in range(2)]
    bs_e = [hb[k % 2] for k in range(args.steps)]
    xs_e = [hx[k % 2] for k in range(args.steps)]
    s.solve_batch(bs_e[:2], xs_e[:2], bands=bands, tol=0.0, maxit=ITERS_PER_STEP)  # warm-up

    def timed_batch(nsteps):
        bb_ = [hb[k % 2] for k in range(nsteps)]
        xx_ = [hx[k % 2] for k in range(nsteps)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        torch.cuda.synchronize(dev)
        e0.record(stream)
        inf_ = s.solve_batch(bb_, xx_, bands=bands, tol=0.0, maxit=ITERS_PER_STEP)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        barrier()
        ms_ = e0.elapsed_time(e1)
        if ws > 1:
            import torch.distributed as dist
            t_ = torch.tensor([ms_], dtype=torch.float64, device=dev)
            dist.all_reduce(t_, op=dist.ReduceOp.MAX)
            ms_ = float(t_.item())
        return ms_, inf_

    ms_e2e, infos_e = timed_batch(args.steps)
    iters_e = sum(i.iters for i in infos_e)
    # the same pipeline over 16 steps: the first upload and the last download amortised
    ms_e2e16, infos_e16 = timed_batch(16)
    iters_e16 = sum(i.iters for i in infos_e16)
    step(0, hb[0].numpy(), hx[0].numpy())
    ms_e2e_blk, infos_eb = timed(args.steps, 0, hb[0].numpy(), hx[0].numpy())
    iters_eb = sum(i.iters for i in infos_eb)

    # time-to-solution at the operational tolerance, one solve, device events
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    barrier()
    ev0.record(stream)
    s.set_operator(bands)
    _, tinfo, thist = s.solve(b, tol=1e-4, maxit=200, out=x)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    tts = ev0.elapsed_time(ev1)

    # the paper's own preconditioner (NEXT-1): red-black tri-SOR, 3 sweeps, omega = 1.5,
    # same step and timing; reported beside the headline, which uses C^-1 = T^-1 (reading A-3)
    tri = None
    if not args.no_trisor:
        with torch.cuda.stream(stream):
            st_ = egs.Solver((prob.nx, prob.ny, prob.nz), bands, args.precision, group=group, stream=stream,
                             trisor=True)
            st_.set_preconditioner("trisor", sweeps=3, omega=1.5)
        s_main = s
        s = st_
        step(0)
        ms_t, infos_t = timed(args.steps, 0)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        st_.set_operator(bands)
        _, tinfo_t, _ = st_.solve(b, tol=1e-4, maxit=200, out=x)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        # algorithmic bytes of one step (every launch's, from one profiled step) against the timed rate
        st_.profile_reset()
        pinfo = step(egs.EG_SOLVE_PROFILE)
        ptri = st_.profile()
        step_bytes = sum(v[1] * v[2] for v in ptri.values())
        tri_value = sum(i.iters for i in infos_t) / (ms_t / 1000.0)
        tri_gbps = step_bytes / (ms_t / args.steps / 1000.0) / 1e9
        tri = {"preconditioner": "red-black tri-SOR, 3 sweeps, omega 1.5 (P:243-258)",
               "value": tri_value, "unit": "iter/s",
               "ms_per_step": ms_t / args.steps,
               "step_roofline": {"alg_bytes_per_step": step_bytes,
                                 "alg_bytes_per_point_per_iteration": step_bytes / max(pinfo.iters, 1) / prob.n,
                                 "achieved_GBps": tri_gbps, "frac": tri_gbps / peaks()[0],
                                 "note": "algorithmic bytes of every launch of one profiled step (set_operator, "
                                         "entry, 8 iterations, verification) over the timed step time"},
               "restarts_in_timed_region": int(sum(i.restarts for i in infos_t)),
               "note": "fixed 8 iterations per step; with this preconditioner R falls below the fp32 floor "
                       "within the step, so restarts (r recomputed in fp64) are part of the timed work",
               "time_to_solution": {"tol": 1e-4, "ms": ev0.elapsed_time(ev1), "iters": tinfo_t.iters,
                                    "true_R": tinfo_t.true_R}}
        s = s_main
        del st_
        torch.cuda.empty_cache()


    if rank != 0:
        return
    n = prob.n
    line = {
        "metric": METRIC, "value": value, "unit": "iter/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": DTYPE[args.precision], "data": "synthetic",
        "config": dict(config_dict(args, prob, ws), transport=transport),
        "roofline": {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                     "peak_source": peak_src,
                     "peak_note": "the measured copy bandwidth (1:1 read:write); a read-dominated kernel "
                                  "(the stencils read 8 bytes per byte written) can exceed it: frac > 1",
                     "alg_bytes_per_launch": kbytes},
        "iteration_roofline": {"alg_bytes_per_point": B_ALG[args.precision],
                               "achieved_GBps": B_ALG[args.precision] * n * value / 1e9,
                               "frac": B_ALG[args.precision] * n * value / 1e9 / peak,
                               "note": "whole step incl. a1/a2/a11 and control, per iteration"},
        "step_roofline": {"alg_bytes_per_step": sum(v[1] * v[2] for v in prof.values()) / args.steps,
                          "achieved_GBps": sum(v[1] * v[2] for v in prof.values()) / (ms / 1000.0) / 1e9,
                          "frac": sum(v[1] * v[2] for v in prof.values()) / (ms / 1000.0) / 1e9 / peak,
                          "note": "algorithmic bytes of every launch in the timed steps (set_operator, entry, "
                                  "8 iterations, verification) over the timed time"},
        "kernels": kernels,
        "graph_replay": {"value": iters_g / (ms_graph / 1000.0), "ms_per_step": ms_graph / args.steps},
        "e2e": {"value": iters_e / (ms_e2e / 1000.0), "unit": "iter/s",
                "h2d_bytes_per_step": 8 * nloc, "d2h_bytes_per_step": 8 * nloc,
                "ms_per_step": ms_e2e / args.steps,
                "api": "eg_solve_batch (C ABI) over the K steps with pinned host b / x: each step = "
                       "set_operator + solve; uploads / downloads of neighbouring steps overlap the solves",
                "steady_16_steps": {"value": iters_e16 / (ms_e2e16 / 1000.0), "ms_per_step": ms_e2e16 / 16,
                                    "note": "eg_solve_batch over 16 steps (not the K timed steps)"},
                "blocking": {"value": iters_eb / (ms_e2e_blk / 1000.0), "ms_per_step": ms_e2e_blk / args.steps,
                             "api": "K separate eg_solve calls with host buffers (transfers not overlapped)"}},
        "time_to_solution": {"tol": 1e-4, "ms": tts, "iters": tinfo.iters, "converged": tinfo.converged,
                             "true_R": tinfo.true_R, "history": [float(v) for v in thist],
                             "includes": "set_operator + solve (a1-a11)"},
        "trisor": tri,
        "gpu_launches": int(launches),
        "restarts_in_timed_region": int(sum(i.restarts for i in infos)),
        "clocks": clk.summary(),
    }
    if ws == 1 and not args.no_cpu_baseline:
        cb = oracle_sample(prob, args.precision, target_s=args.ref_seconds)
        line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model")}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--precision", default="mixed", choices=["mixed", "fp64", "fp32"])
    ap.add_argument("--ref-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-trisor", action="store_true", help="skip the tri-SOR preconditioner block")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args.gpus)           # does not return
    ws, rank, local = dist_init(args)
    if ws != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}; measuring {ws} rank(s)", file=sys.stderr)
    if rank == 0:  # one build, not one per rank racing on the same files
        subprocess.check_call(["make", "-s", "all"], cwd=ROOT, stdout=subprocess.DEVNULL)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    import gen
    prob = gen.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, prob, ws, rank)
    else:
        run_ours(args, prob, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
