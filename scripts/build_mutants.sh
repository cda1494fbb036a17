# the mutation builds of scripts/mutation_checks.sh (build/libegsolve_mut_*.so)
set -e
cd "$(dirname "$0")/.."
for v in NO_EDGE_STENCIL NO_HALO_PUSH NO_VCOPY NO_SWEEP_PUSH; do
  bash scripts/build_variant.sh mut_$v "-DEG_MUTATE_$v"
done
