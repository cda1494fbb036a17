"""A/B of environment knobs on one config / band: per-kernel average times (EG_SOLVE_PROFILE) and
the graph-replay solve(8) time, each setting in its own process.
    python scripts/ab_env.py CFG P PREC "ENV1=a,ENV2=b" "ENV1=c" ...   (P: band of ny/P rows)"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, json
sys.path.insert(0, ROOT)
import torch, gen, paper_1811_03852_b200 as egs
cfg, P, prec = sys.argv[1], int(sys.argv[2]), sys.argv[3]
base = gen.CONFIGS[cfg]
prob = base.with_(ny=base.ny // P)
bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda"); b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
gen.device(prob, bands, b); x = torch.empty_like(b)
s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, prec)
s.solve(b, tol=0.0, maxit=8, out=x)
best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(); s.solve(b, tol=0.0, maxit=8, out=x); e1.record(); torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
s.profile_reset()
for _ in range(3):
    s.solve(b, tol=0.0, maxit=8, out=x, flags=egs.EG_SOLVE_PROFILE)
p = s.profile()
print(f"solve(8) {best:.3f} ms", json.dumps({k: round(v[0] / v[1], 4) for k, v in p.items() if v[1]}))
'''.replace("ROOT", repr(ROOT))
cfg, P, prec = sys.argv[1], sys.argv[2], sys.argv[3]
for setting in sys.argv[4:]:
    env = dict(os.environ)
    for kv in filter(None, setting.split(",")):
        k, v = kv.split("=", 1)
        env[k] = v
    out = subprocess.run([sys.executable, "-c", CHILD, cfg, P, prec], env=env, capture_output=True, text=True)
    print(f"{cfg} P={P} {prec} [{setting}]", out.stdout.strip() or out.stderr[-600:], flush=True)
