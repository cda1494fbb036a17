"""One short step of the hot path for ncu: C5 (2560x1920x70) set_operator + solve(tol=0, maxit).

    python scripts/profile_step.py [--config C5] [--precision mixed] [--maxit 2] [--flags 2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
import paper_1811_03852_b200 as egs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--precision", default="mixed")
ap.add_argument("--maxit", type=int, default=2)
ap.add_argument("--flags", type=int, default=egs.EG_SOLVE_NO_GRAPH)
a = ap.parse_args()
prob = gen.CONFIGS[a.config]
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
    b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    gen.device(prob, bands, b, stream=st)
    s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, a.precision, stream=st)
    s.set_operator(bands)                               # warm-up step (graph capture), as the bench does
    s.solve(b, tol=0.0, maxit=a.maxit, flags=a.flags)
    s.set_operator(bands)
    x, info, hist = s.solve(b, tol=0.0, maxit=a.maxit, flags=a.flags)
torch.cuda.synchronize()
print("iters", info.iters, "hist", list(hist))
