# ncu evidence for profiles/: launch list with per-launch time and DRAM bytes of one C5 step, then a
# full capture of the update (dominant) kernel.  Each ncu command runs after the same command exited 0.
mkdir -p gpurun_out
CMD="python scripts/profile_step.py --maxit 3"
timeout 300 $CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_update|k_stencil|k_thomas_tm" -s 3 -c 5 \
    -o gpurun_out/prof_r01 -f $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc $?
