# ncu full capture of kernels matching $KREGEX (after a plain run of the same command exits 0)
mkdir -p gpurun_out
CMD="python scripts/profile_step.py ${PROF_ARGS:-}"
timeout 300 $CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_thomas}" -s ${KSKIP:-0} -c ${KCOUNT:-2} \
    -o gpurun_out/${NCU_OUT:-prof_full} -f $CMD > gpurun_out/ncu_full.log 2>&1; echo ncu rc $?
tail -3 gpurun_out/ncu_full.log
