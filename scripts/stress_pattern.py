"""Reproduce check_determinism's allocation pattern (new output tensor per solve, earlier ones
dropped) many times; count solves whose x differs from the first."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1811_03852_b200 as egs  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 50
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
prob = gen.CONFIGS["C5"]
bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
gen.device(prob, bands, b)
s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, "mixed")
x0 = None
bad = 0
for r in range(reps):
    if r % 7 == 3:
        s.set_operator(bands)
    x, info, h = s.solve(b, tol=tol, maxit=200)
    if x0 is None:
        x0 = x.clone()
        it0 = info.iters
    elif not torch.equal(x, x0):
        bad += 1
        print(f"rep {r}: iters {info.iters} (first {it0}) restarts {info.restarts} max|dx| {float((x - x0).abs().max()):.3e}", flush=True)
print(f"{reps - bad}/{reps} equal", flush=True)
