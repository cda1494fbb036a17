"""Fused (march) vs 5-kernel schedule: time of fixed 8-iteration solves per config (CUDA events)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1811_03852_b200 as egs  # noqa: E402

for name in sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]:
    prob = gen.CONFIGS[name]
    bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
    b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    x = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    gen.device(prob, bands, b)
    res = {}
    for fuse in (True, False):
        if not fuse:
            os.environ["EG_NO_FUSE"] = "1"
        s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, "mixed")
        os.environ.pop("EG_NO_FUSE", None)
        s.solve(b, tol=0.0, maxit=8, out=x)
        best = 1e30
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            s.solve(b, tol=0.0, maxit=8, out=x)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        res[fuse] = best
        del s
    print(f"{name} {prob.nx}x{prob.ny}x{prob.nz}: fused {res[True]:.3f} ms, 5-kernel {res[False]:.3f} ms "
          f"(per iteration incl. entry/verify: {res[True] / 8:.3f} vs {res[False] / 8:.3f})", flush=True)
    del bands, b, x
    torch.cuda.empty_cache()
