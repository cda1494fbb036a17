"""every BASELINE.json config on one GPU, with the CPU oracle beside it.

Per (config, precision): iterations to tol 1e-4 on the GPU and in the oracle, GPU time to solution
(set_operator + solve, CUDA events), GPU iters/s of a fixed 8-iteration solve (graph replay),
HBM fraction of that rate (136 / 256 B per point per iteration against MEASURED_PEAKS hbm_gbs),
the oracle's tol-1e-4 wall time on all host cores and, for C1 / C2, on one core.

    python scripts/results_table.py [--out profiles/r02_results_table.json]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import oracle  # noqa: E402
import paper_1811_03852_b200 as egs  # noqa: E402

B_ALG = {"mixed": 136, "fp64": 256}
RUNS = [("C1", "mixed"), ("C1", "fp64"), ("C2", "mixed"), ("C2", "fp64"), ("C3", "mixed"), ("C4", "mixed"),
        ("C5", "mixed"), ("C5", "fp64")]


def peak():
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6650.0


def gpu_row(prob, mode):
    g = (prob.nx, prob.ny, prob.nz)
    bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
    b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    gen.device(prob, bands, b)
    x = torch.empty_like(b)
    s = egs.Solver(g, bands, mode)
    s.solve(b, tol=1e-4, maxit=200, out=x)
    s.solve(b, tol=0.0, maxit=8, out=x)

    def timed(fn, reps=3):
        best = 1e30
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            out = fn()
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return best, out

    tts, (xx, info, hist) = timed(lambda: (s.set_operator(bands), s.solve(b, tol=1e-4, maxit=200, out=x))[1])
    t8, (_, i8, _) = timed(lambda: s.solve(b, tol=0.0, maxit=8, out=x))
    s.profile_reset()
    s.solve(b, tol=0.0, maxit=1, flags=egs.EG_SOLVE_PROFILE, out=x)
    fused = s.profile()["phase_A"][1] > 0
    rate = i8.iters / (t8 / 1e3)
    row = {"gpu_iters": info.iters, "gpu_true_R": info.true_R, "gpu_tts_ms": tts, "gpu_iter_per_s": rate,
           "hbm_frac": B_ALG[mode] * prob.n * rate / 1e9 / peak(), "schedule": "fused" if fused else "5-kernel"}
    s.close()
    del s, bands, b, x
    torch.cuda.empty_cache()
    return row


def oracle_row(prob, mode, single):
    g = (prob.nx, prob.ny, prob.nz)
    hb, hr = gen.host(prob)
    out = {}
    for label, threads in (("all", os.cpu_count() or 1),) + ((("one", 1),) if single else ()):
        oracle.set_threads(threads)
        t0 = time.perf_counter()
        ahat, diag = oracle.scale(g, hb, mode)
        _, _, io = oracle.solve(g, mode, ahat, diag, hr, tol=1e-4, maxit=200)
        out[f"oracle_s_{label}"] = time.perf_counter() - t0
        out["oracle_iters"] = io.iters
        del ahat, diag
    oracle.set_threads(os.cpu_count() or 1)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "results_table.json"))
    a = ap.parse_args()
    rows = []
    for cfg, mode in RUNS:
        prob = gen.CONFIGS[cfg]
        r = {"config": cfg, "grid": [prob.nx, prob.ny, prob.nz], "precision": mode}
        r.update(gpu_row(prob, mode))
        r.update(oracle_row(prob, mode, single=cfg in ("C1", "C2")))
        rows.append(r)
        print(json.dumps(r), flush=True)
    meta = {"gpu": torch.cuda.get_device_name(0), "cpu_cores": os.cpu_count(),
            "cpu_model": next((l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")), "?"),
            "peak_GBps": peak()}
    json.dump({"meta": meta, "rows": rows}, open(a.out, "w"), indent=1)
    print(json.dumps(meta))


if __name__ == "__main__":
    main()
