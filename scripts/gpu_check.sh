# one GPU call: tests, smoke, bench, then ncu (launch list + full capture of the top kernels)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
tail -25 gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc $?; tail -3 gpurun_out/smoke.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc $?
tail -3 gpurun_out/bench.err; cat gpurun_out/bench.json
if [ "${NCU:-0}" = "1" ]; then
  timeout 300 python scripts/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/launches.csv python scripts/profile_step.py > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc $?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_thomas|k_update|k_stencil" -c 4 \
      -o gpurun_out/prof_full -f python scripts/profile_step.py > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc $?
  tail -3 gpurun_out/ncu_full.log
fi
