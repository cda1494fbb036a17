# build an A/B variant of libegsolve.so with extra -D flags: scripts/build_variant.sh NAME "-DFOO=1 -DBAR=2"
# (load it with EGSOLVE_LIB=build/libegsolve_NAME.so)
set -e
cd "$(dirname "$0")/.."
NCCL_DIR=$(python -c "import nvidia.nccl,os;print(list(nvidia.nccl.__path__)[0])")
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $2 \
  -Iinclude -I$NCCL_DIR/include -shared -o build/libegsolve_$1.so paper_1811_03852_b200/csrc/egsolve.cu \
  -L$NCCL_DIR/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL_DIR/lib -lcudart
