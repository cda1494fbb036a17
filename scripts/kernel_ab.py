"""A/B per-kernel timing on one problem: variants selected by environment variables read at solver
creation (e.g. EG_NO_TMEM).  Variants are interleaved round by round to cancel clock drift.

    python scripts/kernel_ab.py --variants "tmem:EG_NO_TMEM=0" "smem:EG_NO_TMEM=1" --rounds 4
"""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
import paper_1811_03852_b200 as egs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--precision", default="mixed")
ap.add_argument("--variants", nargs="+", default=["base:"])
ap.add_argument("--rounds", type=int, default=4)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--maxit", type=int, default=8)
a = ap.parse_args()

prob = gen.CONFIGS[a.config]
st = torch.cuda.Stream()
solvers = {}
with torch.cuda.stream(st):
    bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
    b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    gen.device(prob, bands, b, stream=st)
    x = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    for v in a.variants:
        name, _, envs = v.partition(":")
        saved = {}
        for kv in filter(None, envs.split(",")):
            k, _, val = kv.partition("=")
            saved[k] = os.environ.get(k)
            os.environ[k] = val
        solvers[name] = egs.Solver((prob.nx, prob.ny, prob.nz), bands, a.precision, stream=st)
        for k, val in saved.items():
            if val is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = val

res = {n: {} for n in solvers}
steps_ms = {n: [] for n in solvers}
for r in range(a.rounds + 1):
    for n, s in solvers.items():
        s.profile_reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(a.steps):
            s.set_operator(bands)
            s.solve(b, tol=0.0, maxit=a.maxit, flags=egs.EG_SOLVE_PROFILE, out=x)
        e1.record(st)
        torch.cuda.synchronize()
        if r == 0:
            continue  # warm-up round
        steps_ms[n].append(e0.elapsed_time(e1) / a.steps)
        for k, (ms, cnt, by) in s.profile().items():
            if cnt:
                res[n].setdefault(k, []).append((ms / cnt, by))
for n in solvers:
    print(f"== {n}: ms/step median {statistics.median(steps_ms[n]):.3f}  "
          f"-> {a.maxit * 1000 / statistics.median(steps_ms[n]):.2f} it/s")
    for k, lst in res[n].items():
        t = statistics.median(v[0] for v in lst)
        by = lst[0][1]
        print(f"   {k:15s} {t:.4f} ms  {by / t / 1e6:8.0f} GB/s   (min {min(v[0] for v in lst):.4f})")
