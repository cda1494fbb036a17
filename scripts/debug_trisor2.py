import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import gen, paper_1811_03852_b200 as egs
prob = gen.Problem(64, 48, 20, seed=46, cv=(5.0, 20.0), dl=(1e-3, 1e-2))
bands, b = gen.host(prob)
bd = torch.from_numpy(bands).cuda()
for mode in ("mixed", "fp64"):
    s = egs.Solver((prob.nx, prob.ny, prob.nz), bd, mode)
    dt = torch.float32 if mode != "fp64" else torch.float64
    C = bd[0]
    r = (torch.from_numpy(b).cuda() / C).to(dt)
    for sw, om in ((1, 1.0), (3, 1.5)):
        s.set_preconditioner("trisor", sw, om)
        z = s.precondition(r)
        v = s.apply(z)
        sig = float((r.double() * v.double()).sum())
        print(mode, sw, om, "z finite", bool(torch.isfinite(z).all()), "sigma", sig, "|z|", float(z.double().norm()))
        for sw2 in (1, 3):
            s.set_preconditioner("trisor", sw2, om)
            x, info, h = s.solve(torch.from_numpy(b).cuda(), tol=1e-4, maxit=3, raise_on_error=False, flags=egs.EG_SOLVE_NO_GRAPH, check_every=1)
            print("   solve sweeps", sw2, info.status, info.iters, info.breakdowns, h)
