"""Per-rank work of the latitude-band decomposition, measured on one GPU: a band of ny/P rows of a
BASELINE config (default C5: 2560 x 1920/P x 70; `--config C4`) timed as a whole problem (fixed 8 iterations, CUDA events), for the fused
schedule with each strip count and for the 5-kernel schedule.  The halo exchange and the
all-gather are not included (they need P GPUs)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1811_03852_b200 as egs  # noqa: E402

args = sys.argv[1:]
cfg = "C5"
if args and args[0] == "--config":
    cfg, args = args[1], args[2:]
quick = "--quick" in args          # default schedules only (no strip sweep)
args = [a for a in args if a != "--quick"]
base = gen.CONFIGS[cfg]
for P in [int(a) for a in (args or ["1", "2", "4", "8"])]:
    prob = base.with_(ny=base.ny // P)
    bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
    b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    x = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    gen.device(prob, bands, b)
    variants = [("5-kernel", {"EG_NO_FUSE": "1"}), ("fused default", {})] + \
        ([] if quick else [(f"fused strips={k}", {"EG_MARCH_STRIPS": str(k)}) for k in (1, 2, 3, 4, 5, 6)])
    for name, env in variants:
        for k in ("EG_NO_FUSE", "EG_MARCH_STRIPS"):
            os.environ.pop(k, None)
        os.environ.update(env)
        s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, "mixed")
        for k in env:
            os.environ.pop(k, None)
        s.solve(b, tol=0.0, maxit=8, out=x)
        best = 1e30
        for _ in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            s.solve(b, tol=0.0, maxit=8, out=x)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        s.profile_reset()
        s.solve(b, tol=0.0, maxit=8, out=x, flags=egs.EG_SOLVE_PROFILE)
        p = s.profile()
        kt = " ".join(f"{k} {p[k][0] / p[k][1]:.4f}" for k in p if p[k][1] > 0)
        print(f"P={P} ({prob.nx}x{prob.ny}x{prob.nz}) {name:18s}: solve(8) {best:.3f} ms, "
              f"{best / 8 * P:.3f} ms x P per iteration; {kt}", flush=True)
        s.close()
        del s
    del bands, b, x
    torch.cuda.empty_cache()
