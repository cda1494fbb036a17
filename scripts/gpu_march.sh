# fused-phase iteration loop: bitwise parity tests, bench, cycle trace (debug build)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "fused" > gpurun_out/fused.log 2>&1; echo rc $?; tail -2 gpurun_out/fused.log
bash scripts/gpu_bench.sh
if [ -f build/libegsolve_trace.so ]; then
  EGSOLVE_LIB=build/libegsolve_trace.so timeout 300 python scripts/march_trace.py --which A
  EGSOLVE_LIB=build/libegsolve_trace.so timeout 300 python scripts/march_trace.py --which B
fi
