"""Cost of the multi-rank machinery measured on one GPU, per iteration: the same band-sized problem
(a C4 / C5 band for P ranks, timed as a whole grid) solved on the single-GPU path, and through the
1-rank multi-rank path (EG_FORCE_NCCL=1: split finalisers, split update) with the P2P transport
(group kernels push their sums to the gather buffer and stamp flags; the logic kernel waits) or
the NCCL transport (ncclAllGather of the sums on a 1-rank communicator).  Per-iteration time =
(t(maxit=48) - t(maxit=8)) / 40, fixed iterations, CUDA graph replay, best of 5.  Ghost rows do
not exist with one rank, so this isolates the reductions' transport."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1811_03852_b200 as egs  # noqa: E402

VARIANTS = [("single GPU", {}), ("1-rank P2P", {"EG_FORCE_NCCL": "1"}),
            ("1-rank NCCL", {"EG_FORCE_NCCL": "1", "EG_P2P": "0"})]


def timed(s, b, x, it):
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        s.solve(b, tol=0.0, maxit=it, out=x)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for cfg, P in [("C4", 8), ("C4", 1), ("C5", 8), ("C5", 1)]:
    base = gen.CONFIGS[cfg]
    prob = base.with_(ny=base.ny // P)
    for mode in ("mixed", "fp64"):
        bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
        b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
        x = torch.empty(prob.n, dtype=torch.float64, device="cuda")
        gen.device(prob, bands, b)
        res = []
        for name, env in VARIANTS:
            os.environ.update(env)
            s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, mode)
            for k in env:
                os.environ.pop(k, None)
            s.solve(b, tol=0.0, maxit=8, out=x)
            per = (timed(s, b, x, 48) - timed(s, b, x, 8)) / 40 * 1000.0
            res.append(per)
            print(f"{cfg} band P={P} ({prob.nx}x{prob.ny}x{prob.nz}) {mode:5s} {name:12s} [{s.transport}]: "
                  f"{per:8.1f} us/iteration (+{per - res[0]:5.1f} us vs single GPU)", flush=True)
            s.close()
        del bands, b, x
        torch.cuda.empty_cache()

# per-kernel breakdown at the C4 P = 8 band (profiled solves: serialised on one stream, events per kernel)
if True:
    base = gen.CONFIGS["C4"]
    prob = base.with_(ny=base.ny // 8)
    bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
    b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    x = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    gen.device(prob, bands, b)
    for name, env in VARIANTS:
        os.environ.update(env)
        s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, "mixed")
        for k in env:
            os.environ.pop(k, None)
        s.solve(b, tol=0.0, maxit=8, out=x)
        s.profile_reset()
        s.solve(b, tol=0.0, maxit=40, out=x, flags=egs.EG_SOLVE_PROFILE)
        p = s.profile()
        tot = sum(v[0] for v in p.values())
        print(f"profile C4 band P=8 mixed {name:12s}: " + ", ".join(
            f"{k} {1000 * v[0] / 40:.1f}us/it ({v[1] / 40:.2f}/it)" for k, v in p.items() if v[1] > 0)
            + f"; sum {1000 * tot / 40:.1f} us/it", flush=True)
        s.close()
