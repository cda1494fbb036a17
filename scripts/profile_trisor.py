"""One short tri-SOR solve at C5 for ncu (NEXT-1): set_operator + solve(tol=0, maxit)."""
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
ap.add_argument("--sweeps", type=int, default=3)
ap.add_argument("--omega", type=float, default=1.5)
ap.add_argument("--maxit", type=int, default=1)
ap.add_argument("--precision", default="mixed")
a = ap.parse_args()
prob = gen.CONFIGS[a.config]
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
    b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    gen.device(prob, bands, b, stream=st)
    s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, a.precision, stream=st, trisor=True)
    s.set_preconditioner("trisor", sweeps=a.sweeps, omega=a.omega)  # (colour-split copies: trisor=True)
    x, info, hist = s.solve(b, tol=0.0, maxit=a.maxit, flags=egs.EG_SOLVE_NO_GRAPH)
torch.cuda.synchronize()
print("iters", info.iters, "hist", list(hist))
