import os, sys
sys.path.insert(0, "/root/repo")
import torch, gen
import paper_1811_03852_b200 as egs
prob = gen.CONFIGS["C5"]
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
    b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    x = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    gen.device(prob, bands, b, stream=st)
    s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, "mixed", stream=st)
    for rep in range(4):
        for flags in (0, egs.EG_SOLVE_PROFILE):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.profile_reset()
            e0.record(st)
            s.set_operator(bands)
            _, info, h = s.solve(b, tol=1e-4, maxit=200, out=x, flags=flags)
            e1.record(st)
            torch.cuda.synchronize()
            msg = f"rep {rep} flags {flags}: {e0.elapsed_time(e1):.2f} ms iters {info.iters}"
            if flags:
                p = s.profile()
                msg += " | " + " ".join(f"{k}:{v[0]:.2f}/{v[1]}" for k, v in p.items() if v[1])
            print(msg, flush=True)
