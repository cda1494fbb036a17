"""Cycle accounting of the fused march kernels (debug build with -DMA_TRACE, see DESIGN.md §Fused phases).

    EGSOLVE_LIB=build/libegsolve_trace.so python scripts/march_trace.py [--config C5] [--which A|B]
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1811_03852_b200 as egs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--which", default="B")
a = ap.parse_args()
prob = gen.CONFIGS[a.config]
bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
gen.device(prob, bands, b)
s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, "mixed")
# maxit 2: the second iteration is not "fresh" (p, v are read); phase A is the last march launch
# when the solve stops right after it, so run A-only via NO_GRAPH + maxit and read what is last
x, info, hist = s.solve(b, tol=0.0, maxit=2, flags=egs.EG_SOLVE_NO_GRAPH)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (1024 * 16))()
assert egs.lib().eg_debug_march_trace(buf, 1024 * 16) == 0
t = np.frombuffer(buf, dtype=np.uint64).reshape(2, 512, 16).astype(np.float64)[0 if a.which == "A" else 1]
ncta = int((t[:, 0] > 0).sum())
t = t[:ncta]
names = ["S total", " S halo copy (wait hready)", " S stage waits", "-", " S boundary-row sync", " S wait z(r_m+1) from F",
         " S stencil pass", "-", " S reduce", "PRODUCER empty-wait", "PRODUCER total", "F total",
         " F stage waits", " F wait sread (S behind)", " F back subst", " F elimination"]
print(f"CTAs {ncta}; cycles per CTA (mean / min / max) of the last phase {a.which} launch")
for q, nm in enumerate(names):
    print(f"  {nm:22s} {t[:, q].mean():14.0f} {t[:, q].min():14.0f} {t[:, q].max():14.0f}  {100 * t[:, q].mean() / t[:, 0].mean():5.1f}%")
