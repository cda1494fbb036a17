"""Stress the fused march kernels for races: many repeated fixed-iteration solves must give bitwise
identical x and histories (and equal the 5-kernel schedule's)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1811_03852_b200 as egs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="C5,C4,C3")
ap.add_argument("--reps", type=int, default=40)
ap.add_argument("--maxit", type=int, default=8)
ap.add_argument("--precision", default="mixed")
ap.add_argument("--tol", type=float, default=0.0)
ap.add_argument("--fresh-out", action="store_true", help="a new output tensor per solve (graph re-capture)")
a = ap.parse_args()
bad = 0
for name in a.configs.split(","):
    prob = gen.CONFIGS[name]
    bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
    b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    gen.device(prob, bands, b)
    g = (prob.nx, prob.ny, prob.nz)
    os.environ["EG_NO_FUSE"] = "1"
    ref = egs.Solver(g, bands, a.precision)
    os.environ.pop("EG_NO_FUSE")
    x0, _, h0 = ref.solve(b, tol=a.tol, maxit=a.maxit)
    del ref
    s = egs.Solver(g, bands, a.precision)
    nd = 0
    keep = []
    for r in range(a.reps):
        x, info, h = s.solve(b, tol=a.tol, maxit=a.maxit, out=None if a.fresh_out else x0.clone())
        if a.fresh_out:
            keep.append(x)  # keep the buffers alive so the next solve gets a new pointer
        if not (torch.equal(x, x0) and np.array_equal(h, h0)):
            nd += 1
            print(f"{name} rep {r}: MISMATCH max|dx| {float((x - x0).abs().max()):.3e}", flush=True)
    print(f"{name}: {a.reps - nd}/{a.reps} repetitions bitwise equal to the 5-kernel schedule", flush=True)
    bad += nd
    del s, bands, b, x0
    torch.cuda.empty_cache()
sys.exit(1 if bad else 0)
