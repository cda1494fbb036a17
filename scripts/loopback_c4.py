"""C4 (or --config) on P latitude bands through the loopback group, a few fixed iterations: a
target for ncu (per-kernel durations of the band machinery: k_edge_rows, k_p2p_wait, k_push_rows,
edge-row k_stencil, finalisers), which cannot be timed with events on the shared stream."""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1811_03852_b200 as egs  # noqa: E402

args = sys.argv[1:]
cfg = args[args.index("--config") + 1] if "--config" in args else "C4"
P = int(args[args.index("--P") + 1]) if "--P" in args else 8
mode = args[args.index("--mode") + 1] if "--mode" in args else "mixed"
prob = gen.CONFIGS[cfg]
bands, bh = gen.host(prob)
row = prob.nx * prob.nz
uid = egs.loopback_id(P)
sv = []
for r in range(P):
    j0, j1 = egs.band_rows(prob.ny, r, P)
    sv.append((egs.Solver((prob.nx, prob.ny, prob.nz),
                          torch.from_numpy(np.ascontiguousarray(bands[:, j0 * row:j1 * row])).cuda(), mode,
                          dist=(r, P, uid)), torch.from_numpy(bh[j0 * row:j1 * row].copy()).cuda()))
ts = [threading.Thread(target=lambda q=q: q[0].solve(q[1], tol=0.0, maxit=3)) for q in sv]
for t in ts:
    t.start()
for t in ts:
    t.join()
torch.cuda.synchronize()
print(cfg, P, mode, sv[0][0].transport, "ok")
