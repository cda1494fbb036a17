"""Stress of the latitude-band path on one GPU: C3 (or --config) on P loopback bands with the P2P
transport, where the band-edge kernels run on each rank's side stream CONCURRENTLY with the phase
kernels on the shared stream (real overlap, unlike the stream-ordered pushes): many solves with
restarts, each compared bitwise with the single-GPU solve.  Prints one line per solve."""
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
cfg = args[args.index("--config") + 1] if "--config" in args else "C3"
P = int(args[args.index("--P") + 1]) if "--P" in args else 4
reps = int(args[args.index("--reps") + 1]) if "--reps" in args else 6
mode = args[args.index("--mode") + 1] if "--mode" in args else "mixed"
trisor = "--trisor" in args  # the tri-SOR preconditioner (P2P half-sweep halos)
prob = gen.CONFIGS[cfg]
bands, bh = gen.host(prob)
g = (prob.nx, prob.ny, prob.nz)
row = prob.nx * prob.nz
ref = egs.Solver(g, torch.from_numpy(bands).cuda(), mode, trisor=trisor)
uid = egs.loopback_id(P)
sv = []
for r in range(P):
    j0, j1 = egs.band_rows(prob.ny, r, P)
    sv.append((egs.Solver(g, torch.from_numpy(np.ascontiguousarray(bands[:, j0 * row:j1 * row])).cuda(), mode,
                          dist=(r, P, uid), trisor=trisor), slice(j0 * row, j1 * row)))
if trisor:
    for q in [ref] + [v[0] for v in sv]:
        q.set_preconditioner("trisor", sweeps=3, omega=1.5)
print(cfg, P, mode, "tri-SOR" if trisor else "T^-1", sv[0][0].transport, flush=True)
rng = np.random.default_rng(7)
bad = 0
for rep in range(reps):
    b = bh * (1.0 + 0.3 * rng.standard_normal()) + 0.01 * rng.standard_normal(prob.n)
    kw = dict(tol=float(rng.choice([1e-5, 1e-7, 0.0])), maxit=int(rng.integers(20, 80)),
              restart_every=int(rng.choice([0, 7, 13])))
    x1, i1, h1 = ref.solve(torch.from_numpy(b).cuda(), **kw)
    outs = [None] * P

    def work(r):
        s, sl = sv[r]
        outs[r] = s.solve(torch.from_numpy(np.ascontiguousarray(b[sl])).cuda(), **kw)
    ts = [threading.Thread(target=work, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    xP = torch.cat([o[0] for o in outs])
    same = torch.equal(xP, x1) and all(np.array_equal(o[2], h1) for o in outs) and \
        all(o[1].iters == i1.iters and o[1].restarts == i1.restarts for o in outs)
    bad += not same
    print(f"rep {rep}: {kw} iters {i1.iters} restarts {i1.restarts} -> {'bitwise' if same else 'MISMATCH'}", flush=True)
print("stress", "FAILED" if bad else "ok", flush=True)
sys.exit(1 if bad else 0)
