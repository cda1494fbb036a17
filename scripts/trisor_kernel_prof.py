import os, sys
sys.path.insert(0, "/root/repo")
import torch, gen, paper_1811_03852_b200 as egs
prob = gen.CONFIGS["C5"]
bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
x = torch.empty(prob.n, dtype=torch.float64, device="cuda")
gen.device(prob, bands, b)
for mode, env in (("mixed", {}), ("mixed", {"EG_NO_SOR_TMA": "1"}), ("fp64", {})):
    os.environ.pop("EG_NO_SOR_TMA", None); os.environ.update(env)
    s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, mode, trisor=True)
    s.set_preconditioner("trisor", sweeps=3, omega=1.5)
    s.solve(b, tol=0.0, maxit=2, out=x, flags=egs.EG_SOLVE_PROFILE)
    s.profile_reset()
    s.solve(b, tol=0.0, maxit=2, out=x, flags=egs.EG_SOLVE_PROFILE)
    p = s.profile()
    print(mode, env, {k: (round(v[0]/v[1],3), v[1], round(v[2]/(v[0]/v[1]/1e3)/1e9)) for k, v in p.items() if v[1]}, flush=True)
    s.close(); del s; torch.cuda.empty_cache()
