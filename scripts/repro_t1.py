"""table1-shaped rare-event hunt (scripts/studies.py table1 --hard): per date, the fused MIXED solver
does set_operator + solve at 1e-3 and 1e-4, then the 5-kernel MIXED solver, then FP64.  Reports
solves where fused and 5-kernel x differ.  Options: nograph, nofp64, sync."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1811_03852_b200 as egs  # noqa: E402

opts = set(sys.argv[1:])
dates = 22
base = gen.CONFIGS["C4"].with_(cv=(5.0, 20.0), dl=(1e-4, 1e-3))
g = (base.nx, base.ny, base.nz)
st = torch.cuda.Stream()
bad = tot = 0
flags = egs.EG_SOLVE_NO_GRAPH if "nograph" in opts else 0
with torch.cuda.stream(st):
    bands = torch.empty((7, base.n), dtype=torch.float64, device="cuda")
    b = torch.empty(base.n, dtype=torch.float64, device="cuda")
    x = torch.empty(base.n, dtype=torch.float64, device="cuda")
    xs = {"fu": x, "un": torch.empty_like(x) if "sepx" in opts else x, "64": x}
    gen.device(base, bands, b, stream=st)
    if "uu" in opts:
        os.environ["EG_NO_FUSE"] = "1"
    fu = egs.Solver(g, bands, "mixed", stream=st)
    os.environ.pop("EG_NO_FUSE", None)
    if "ff" not in opts:
        os.environ["EG_NO_FUSE"] = "1"
    un = egs.Solver(g, bands, "mixed", stream=st)
    os.environ.pop("EG_NO_FUSE", None)
    print("first solver fused:", fu.profile is not None and "uu" not in opts, "second fused:", "ff" in opts, flush=True)
    d64 = None if "nofp64" in opts else egs.Solver(g, bands, "fp64", stream=st)
    import ctypes
    seen = hasattr(egs.lib(), "eg_debug_seen")
    print("debug record:", seen, egs._SO, flush=True)
    if seen:
        L = egs.lib()
        L.eg_debug_seen.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        L.eg_debug_seen(base.n, None, None)
        cb, cn = ctypes.c_ulonglong(), ctypes.c_ulonglong()
    for d in range(dates):
        gen.device(base.with_(seed=4 + d % 11), bands, b, stream=st)
        res = {}
        for name, s in (("fu", fu), ("un", un), ("64", d64)):
            if s is None:
                continue
            for tol in (1e-3, 1e-4):
                if "sync" in opts:
                    torch.cuda.synchronize()
                s.set_operator(bands)
                xo = xs[name]
                _, info, h = s.solve(b, tol=tol, maxit=200, out=xo, flags=flags)
                res[(name, tol)] = (xo.clone(), info.iters, info.restarts, h.copy())
                if seen and name == "fu":
                    L.eg_debug_seen(0, ctypes.byref(cb), ctypes.byref(cn))
                    if cb.value or d == 0:
                        print(f"date {d} tol {tol:g}: {cb.value} of {cn.value} cross-CTA z reads stale", flush=True)
        for tol in (1e-3, 1e-4):
            tot += 1
            a, c = res[("fu", tol)], res[("un", tol)]
            if not torch.equal(a[0], c[0]):
                bad += 1
                ha, hc = a[3], c[3]
                fd = next((i for i in range(min(len(ha), len(hc))) if ha[i] != hc[i]), None)
                print(f"date {d} tol {tol:g}: fused {a[1]} it {a[2]} rs | 5-kernel {c[1]} it {c[2]} rs | "
                      f"max|dx| {float((a[0] - c[0]).abs().max()):.2e} | first hist diff at {fd}: "
                      f"{ha[fd] if fd is not None else ''} vs {hc[fd] if fd is not None else ''}", flush=True)
print(f"{opts or ''}: {bad} / {tot} fused solves differ", flush=True)
