"""Stage split of the fused phase kernels' two TMA rings (EG_MARCH_FST_A / _B = elimination-ring
stages, the rest of the shared memory goes to the stencil ring): phase A / B kernel times at C5."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import gen  # noqa: E402
import paper_1811_03852_b200 as egs  # noqa: E402

prob = gen.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C5"]
bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
x = torch.empty(prob.n, dtype=torch.float64, device="cuda")
gen.device(prob, bands, b)
settings = [(None, None)] + [(str(a), str(a + 3)) for a in range(3, 9)]
for fa, fb in settings:
    for k, v in (("EG_MARCH_FST_A", fa), ("EG_MARCH_FST_B", fb)):
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v
    s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, "mixed")
    s.solve(b, tol=0.0, maxit=8, out=x, flags=egs.EG_SOLVE_PROFILE)
    s.profile_reset()
    for _ in range(3):
        s.solve(b, tol=0.0, maxit=8, out=x, flags=egs.EG_SOLVE_PROFILE)
    p = s.profile()
    a, bb = p["phase_A"], p["phase_B"]
    print(f"F stages A={fa} B={fb}: phase_A {a[0] / a[1]:.3f} ms  phase_B {bb[0] / bb[1]:.3f} ms", flush=True)
    s.close()
    del s
    torch.cuda.empty_cache()
