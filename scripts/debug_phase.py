"""Small fused-phase probe: one solve on a chosen grid, printing progress (run under `timeout`)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
import paper_1811_03852_b200 as egs  # noqa: E402

nx, ny, nz = (int(v) for v in sys.argv[1:4])
maxit = int(sys.argv[4]) if len(sys.argv) > 4 else 2
prob = gen.Problem(nx, ny, nz, seed=1)
bands, b = gen.host(prob)
s = egs.Solver((nx, ny, nz), torch.from_numpy(bands).cuda(), "mixed")
print("created", flush=True)
t = time.time()
x, info, h = s.solve(torch.from_numpy(b).cuda(), tol=0.0, maxit=maxit, flags=egs.EG_SOLVE_NO_GRAPH,
                     check_every=1)
torch.cuda.synchronize()
print("solved", info, list(h), time.time() - t, flush=True)
