# Mutation checks of the latitude-band tests: each build drops one mechanism the band path relies
# on; the band tests must fail with it (and pass with the real library).  One GPU call:
#   bash scripts/build_mutants.sh here (nvcc), then under gpurun: bash scripts/mutation_checks.sh
mkdir -p gpurun_out
T="tests/test_gpu_p2p.py tests/test_gpu_loopback.py"
for v in NO_EDGE_STENCIL NO_HALO_PUSH NO_VCOPY NO_SWEEP_PUSH; do
  lib=build/libegsolve_mut_$v.so
  r=$(EGSOLVE_LIB=$lib EG_P2P_TIMEOUT_MS=2000 timeout 900 python -m pytest -q -m gpu $T 2>&1 | tail -1)
  echo "EG_MUTATE_$v: $r"
done
r=$(timeout 900 python -m pytest -q -m gpu $T 2>&1 | tail -1)
echo "real library: $r"
