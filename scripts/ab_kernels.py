"""A/B timing of library variants (EGSOLVE_LIB builds from scripts/build_variant.sh): per-kernel
average times of a C5 bench step (set_operator + solve(tol=0, maxit=8), EG_SOLVE_PROFILE events),
each variant in its own process.   python scripts/ab_kernels.py build/libegsolve_a.so build/libegsolve_b.so ..."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, json
sys.path.insert(0, ROOT)
import torch, gen, paper_1811_03852_b200 as egs
prob = gen.CONFIGS[os.environ.get("CFG", "C5")]
prec = os.environ.get("PREC", "mixed")
bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda"); b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
gen.device(prob, bands, b); x = torch.empty_like(b)
s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, prec)
for _ in range(2):
    s.set_operator(bands); s.solve(b, tol=0.0, maxit=8, out=x, flags=egs.EG_SOLVE_PROFILE)
s.profile_reset()
for _ in range(4):
    s.set_operator(bands); s.solve(b, tol=0.0, maxit=8, out=x, flags=egs.EG_SOLVE_PROFILE)
p = s.profile()
print(json.dumps({k: [round(v[0] / v[1], 4), round(v[2] / (v[0] / v[1]) / 1e6, 1)] for k, v in p.items() if v[1]}))
'''.replace("ROOT", repr(ROOT))
for lib in sys.argv[1:]:
    env = dict(os.environ, EGSOLVE_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), out.stdout.strip() or out.stderr[-500:], flush=True)
