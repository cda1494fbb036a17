"""Per-kernel table of a profiled tri-SOR(3, 1.5) solve at C5 (NEXT-1): average time per launch,
algorithmic bytes per launch and the implied GB/s (EG_SOLVE_PROFILE events)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch, gen
import paper_1811_03852_b200 as egs
prob = gen.CONFIGS["C5"]
bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
gen.device(prob, bands, b)
s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, "mixed", trisor=True)
s.set_preconditioner("trisor", sweeps=3, omega=1.5)
x = torch.empty(prob.n, dtype=torch.float64, device="cuda")
s.solve(b, tol=0.0, maxit=8, out=x)
s.profile_reset()
s.solve(b, tol=0.0, maxit=8, out=x, flags=egs.EG_SOLVE_PROFILE)
p = s.profile()
for k, (ms, n, by) in p.items():
    if n: print(f"{k:16s} n={n:4d} avg {ms/n:8.3f} ms  {by/1e9:7.2f} GB/launch  {by*n/ms/1e6 if ms else 0:7.0f} GB/s")
