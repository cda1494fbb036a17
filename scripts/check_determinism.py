"""Run-to-run determinism and fused-vs-5-kernel bitwise equality at full size (C5 by default)."""
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
ap.add_argument("--tol", type=float, default=1e-6)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
prob = gen.CONFIGS[a.config]
bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
gen.device(prob, bands, b)
g = (prob.nx, prob.ny, prob.nz)
res = []
for fuse in (True, False):
    if not fuse:
        os.environ["EG_NO_FUSE"] = "1"
    s = egs.Solver(g, bands, "mixed")
    os.environ.pop("EG_NO_FUSE", None)
    for r in range(a.reps):
        x, info, h = s.solve(b, tol=a.tol, maxit=200)
        res.append((fuse, r, info.iters, info.restarts, info.true_R, list(h), x.clone()))
        print(f"fused={fuse} rep={r}: iters {info.iters} restarts {info.restarts} true_R {info.true_R:.6e} "
              f"hist {[f'{v:.6e}' for v in h]}", flush=True)
    del s
    torch.cuda.empty_cache()
x0 = res[0][6]
for fuse, r, it, rs, tr, h, x in res:
    print(fuse, r, "x bitwise equal to first:", torch.equal(x, x0), "max|dx|", float((x - x0).abs().max()))
