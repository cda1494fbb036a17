"""Solves of a few problems (argument: fp64 | mixed | fp32), printed as hashes of x, the history and
a preconditioner application: run under two builds (EGSOLVE_LIB) to check that a change is bitwise
neutral."""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1811_03852_b200 as egs  # noqa: E402

MODE = sys.argv[1] if len(sys.argv) > 1 else "fp64"
for prob in [gen.CONFIGS["C1"], gen.Problem(200, 37, 13, seed=8), gen.CONFIGS["C2"], gen.Problem(96, 24, 13, seed=17)]:
    bands, b = gen.host(prob)
    g = (prob.nx, prob.ny, prob.nz)
    for pre in ("tridiag", "trisor"):
        s = egs.Solver(g, torch.from_numpy(bands).cuda(), MODE, trisor=True)
        s.set_preconditioner(pre)
        x, info, hist = s.solve(torch.from_numpy(b).cuda(), tol=1e-10, maxit=80, restart_every=7)
        z = s.precondition(torch.from_numpy(b).cuda().to(s.vdtype))
        h = hashlib.sha1(x.cpu().numpy().tobytes() + hist.tobytes() + z.cpu().numpy().tobytes()).hexdigest()[:16]
        print(f"{prob.nx}x{prob.ny}x{prob.nz} {pre}: iters {info.iters} {h}")
