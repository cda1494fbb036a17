# one GPU call: the GPU test suite (optionally a subset: TESTS="tests/x.py", KEXPR="pytest -k expression"), smoke
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
if [ -n "${KEXPR:-}" ]; then KARGS=(-k "$KEXPR"); else KARGS=(); fi
timeout ${PYT_TIMEOUT:-1500} python -m pytest ${TESTS:-tests} -x -q -m gpu ${PYTEST_ARGS:-} "${KARGS[@]}" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc $?
tail -30 gpurun_out/pytest_gpu.log
if [ "${SMOKE:-1}" = "1" ]; then
  timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke rc $?; tail -3 gpurun_out/smoke.log
fi
