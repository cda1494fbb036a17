import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import gen, paper_1811_03852_b200 as egs
prob = gen.Problem(64, 48, 20, seed=46, cv=(5.0, 20.0), dl=(1e-3, 1e-2))
bands, b = gen.host(prob)
for mode in ("fp64", "mixed", "fp32"):
    for flags in (0, egs.EG_SOLVE_NO_GRAPH):
        s = egs.Solver((prob.nx, prob.ny, prob.nz), torch.from_numpy(bands).cuda(), mode)
        s.set_preconditioner("trisor", 3, 1.5)
        x, info, h = s.solve(torch.from_numpy(b).cuda(), tol=1e-4, maxit=30, flags=flags, raise_on_error=False, check_every=1)
        print(mode, flags, info, np.array2string(h, precision=3))
