# ncu full captures of the FP64 phase-A / phase-B kernels: fused (march64) and 5-kernel (Thomas)
mkdir -p gpurun_out
CMD="python scripts/profile_step.py --maxit 3 --flags 0 --precision fp64"
timeout 300 $CMD > gpurun_out/p64.log 2>&1; echo plain rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_march64" -s 2 -c 2 \
    -o gpurun_out/r02_fp64_march -f $CMD > gpurun_out/ncu64a.log 2>&1; echo ncu1 rc $?
EG_NO_FUSE=1 timeout 300 $CMD > gpurun_out/p64b.log 2>&1; echo plain2 rc $?
EG_NO_FUSE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_thomas|k_stencil" -s 4 -c 4 \
    -o gpurun_out/r02_fp64_5k -f $CMD > gpurun_out/ncu64b.log 2>&1; echo ncu2 rc $?
for P in 1; do
  for cfg in C4 C5; do
    python - <<PY
import os, sys, torch
sys.path.insert(0, ".")
import gen, paper_1811_03852_b200 as egs
prob = gen.CONFIGS["$cfg"]
bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda"); b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
gen.device(prob, bands, b)
x = torch.empty_like(b)
for env in ({"EG_NO_FUSE": "1"}, {}):
    os.environ.pop("EG_NO_FUSE", None); os.environ.update(env)
    s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, "fp64")
    os.environ.pop("EG_NO_FUSE", None)
    s.solve(b, tol=0.0, maxit=8, out=x)
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record(); s.solve(b, tol=0.0, maxit=8, out=x); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    s.profile_reset(); s.solve(b, tol=0.0, maxit=8, out=x, flags=egs.EG_SOLVE_PROFILE); p = s.profile()
    print("$cfg fp64", env, f"solve(8) {best:.2f} ms", {k: round(v[0] / v[1], 3) for k, v in p.items() if v[1]}, flush=True)
    s.close(); del s
PY
  done
done
