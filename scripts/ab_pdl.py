"""A/B of programmatic dependent launch (EG_PDL) per config and precision: best of 7 fixed
40-iteration solves (graph replay), in this process with the environment as given."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1811_03852_b200 as egs  # noqa: E402

out = {}
for cfg in sys.argv[1].split(","):
    for mode in sys.argv[2].split(","):
        prob = gen.CONFIGS[cfg]
        bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
        b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
        gen.device(prob, bands, b)
        s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, mode)
        x = torch.empty(prob.n, dtype=torch.float64, device="cuda")
        it = 40 if prob.n < 3e7 else 8
        s.solve(b, tol=0.0, maxit=it, out=x)
        best = 1e9
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            s.solve(b, tol=0.0, maxit=it, out=x)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[f"{cfg}-{mode}"] = round(1000 * best / it, 2)  # us per iteration (incl. entry / verify share)
        s.close()
        del bands, b, x
        torch.cuda.empty_cache()
print(os.environ.get("EG_PDL", "0"), json.dumps(out), flush=True)
