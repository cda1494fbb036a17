"""Small invocations of every kernel family, for compute-sanitizer (one --tool per gpurun call):
fused phases (EG_FUSE=1; fp32 and FP64 kernels), the 5-kernel schedule, FP64 / FP32, tri-SOR (TMA
sweeps), apply, precondition, solve_batch with host buffers, a caller-given rhat0 (k_shadow), and
2 latitude bands through the loopback transport (overlapped halo, split update)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1811_03852_b200 as egs  # noqa: E402

prob = gen.Problem(136, 12, 13, seed=3)
bands, b = gen.host(prob)
g = (prob.nx, prob.ny, prob.nz)
bd = torch.from_numpy(bands).cuda()
bt = torch.from_numpy(b).cuda()
for mode in ("mixed", "fp32", "fp64"):
    for fuse in ("1", "0"):
        os.environ["EG_FUSE" if fuse == "1" else "EG_NO_FUSE"] = "1"
        s = egs.Solver(g, bd, mode, trisor=True, batch=True)
        os.environ.pop("EG_FUSE", None)
        os.environ.pop("EG_NO_FUSE", None)
        x, info, h = s.solve(bt, tol=1e-6, maxit=12, restart_every=4)
        print(mode, fuse, info.iters, info.status, flush=True)
        x, info, h = s.solve(bt, tol=1e-6, maxit=12, rhat0=bt / 3.0)
        print(mode, fuse, "rhat0", info.iters, info.status, flush=True)
        v = torch.ones(prob.n, dtype=s.vdtype, device="cuda")
        s.apply(v)
        s.precondition(v)
        s.set_preconditioner("trisor", sweeps=2, omega=1.5)
        x, info, h = s.solve(bt, tol=1e-6, maxit=6)
        s.precondition(v)
        print(mode, fuse, "trisor", info.iters, info.status, flush=True)
        s.set_preconditioner("tridiag")
        hb = [np.ascontiguousarray(b), np.ascontiguousarray(2 * b)]
        hx = [np.empty(prob.n), np.empty(prob.n)]
        s.solve_batch(hb, hx, bands=bd, tol=0.0, maxit=3)
        s.close()
# two latitude bands on one GPU (loopback): k_edge_rows, overlapped ghost rows, edge stencils, split update
import threading  # noqa: E402
for mode, fuse in (("mixed", "1"), ("fp64", "0")):
    os.environ["EG_FUSE" if fuse == "1" else "EG_NO_FUSE"] = "1"
    uid = egs.loopback_id(2)
    row = prob.nx * prob.nz
    sv = []
    for r in range(2):
        j0, j1 = egs.band_rows(prob.ny, r, 2)
        sv.append((egs.Solver(g, torch.from_numpy(np.ascontiguousarray(bands[:, j0 * row:j1 * row])).cuda(), mode,
                              dist=(r, 2, uid)), torch.from_numpy(b[j0 * row:j1 * row].copy()).cuda()))
    os.environ.pop("EG_FUSE", None)
    os.environ.pop("EG_NO_FUSE", None)
    ts = [threading.Thread(target=lambda q=q: q[0].solve(q[1], tol=1e-6, maxit=10, restart_every=4)) for q in sv]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    print(mode, "bands", flush=True)
torch.cuda.synchronize()
print("ok")
