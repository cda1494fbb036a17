# One GPU call: the driver's bench command (N=1, K=20, W=5) in MIXED and FP64, then the ncu launch
# list of one C5 bench-shaped step (set_operator + solve(tol=0, maxit=8)) and a full capture of the
# fused phase kernels, the update and the verification pass.  TAG names the output files.
# Each ncu command runs only after the same command exited 0 without ncu.
TAG=${TAG:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 900 python bench.py --steps ${STEPS:-20} --warmup ${WARMUP:-5} > gpurun_out/${TAG}_bench_mixed.json 2> gpurun_out/${TAG}_bench_mixed.err; echo bench mixed rc $?
if [ "${FP64:-1}" = "1" ]; then
  timeout 900 python bench.py --steps ${STEPS:-20} --warmup ${WARMUP:-5} --precision fp64 --no-cpu-baseline > gpurun_out/${TAG}_bench_fp64.json 2> gpurun_out/${TAG}_bench_fp64.err; echo bench fp64 rc $?
fi
if [ "${NCU:-1}" = "1" ]; then
  CMD="python scripts/profile_step.py --maxit 8 --flags 0"
  timeout 300 $CMD > gpurun_out/prof_plain.log 2>&1; echo plain rc $?
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc $?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_march|k_update|k_start" -s 4 -c 5 \
      -o gpurun_out/${TAG}_full -f $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc $?
  tail -2 gpurun_out/ncu_full.log
fi
