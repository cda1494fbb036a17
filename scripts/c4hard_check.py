import os, sys
sys.path.insert(0, "/root/repo")
import torch, gen, paper_1811_03852_b200 as egs
prob = gen.CONFIGS["C4"].with_(cv=(5.0, 20.0), dl=(1e-4, 1e-3))
bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
gen.device(prob, bands, b)
s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, "mixed")
for tol in (1e-4, 1e-6):
    x, info, hist = s.solve(b, tol=tol, maxit=200)
    print(os.environ.get("EGSOLVE_LIB", "cur"), tol, info.iters, info.restarts, info.true_R, float(x.double().norm()))
