# ncu evidence for profiles/: launch list with per-launch time and DRAM bytes of one C5 step
# (set_operator + solve(tol=0, maxit=8), the bench step), then a full capture of the fused phase
# kernels and the update.  Each ncu command runs after the same command exited 0 without ncu.
mkdir -p gpurun_out
CMD="python scripts/profile_step.py --maxit 8"
timeout 300 $CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_march|k_update" -s 3 -c 3 \
    -o gpurun_out/prof_r01_march -f $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc $?
tail -2 gpurun_out/ncu_full.log
