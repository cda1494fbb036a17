"""The README's Python example, runnable (python scripts/readme_example.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch, gen, paper_1811_03852_b200 as egs

prob = gen.CONFIGS["C3"]                                  # 640x480x70, seeded synthetic operator
bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
gen.device(prob, bands, b)                                # C, E, W, N, S, U, D; layout i + nx*(k + nz*j)

s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, "mixed")   # a1: scale the operator
x, info, hist = s.solve(b, tol=1e-4, maxit=200)                # a2-a11; x fp64, hist = R per iteration
s.set_preconditioner("trisor", sweeps=3, omega=1.5)            # the paper's tri-SOR (NEXT-1)
x, info, hist = s.solve(b, tol=1e-6)
y = s.apply(torch.randn(prob.n, device="cuda"))                # y = Ahat x (fp32 in MIXED)

# a time-step sequence with host buffers, transfers overlapped with the solves
sb = egs.Solver((prob.nx, prob.ny, prob.nz), bands, "mixed", batch=True)
bs = [b.cpu().pin_memory() for _ in range(4)]
xs = [torch.empty(prob.n, dtype=torch.float64).pin_memory() for _ in range(4)]
infos = sb.solve_batch(bs, xs, bands=bands, tol=1e-4)
print(info, [i.iters for i in infos])
