"""Run-to-run determinism of the TMA tri-SOR sweeps at scale: repeated tri-SOR(3, 1.5) solves
(set_operator + solve, graph replay) must give bitwise the same x, MIXED and FP64."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1811_03852_b200 as egs  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for name, mode in (("C4", "mixed"), ("C3", "fp64"), ("C5", "mixed")):
    prob = gen.CONFIGS[name].with_(cv=(5.0, 20.0), dl=(1e-4, 1e-3))
    bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
    b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    x = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    gen.device(prob, bands, b)
    s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, mode, trisor=True)
    s.set_preconditioner("trisor", sweeps=3, omega=1.5)
    s.set_operator(bands)
    _, i0, h0 = s.solve(b, tol=1e-6, maxit=40, out=x)
    ref = x.clone()
    bad = 0
    for _ in range(reps):
        s.set_operator(bands)
        _, i1, h1 = s.solve(b, tol=1e-6, maxit=40, out=x)
        bad += int(not torch.equal(x, ref) or i1.iters != i0.iters)
    print(f"{name} {mode}: {reps - bad}/{reps} repetitions bitwise equal ({i0.iters} iterations)", flush=True)
    s.close()
    del s, bands, b, x, ref
    torch.cuda.empty_cache()
