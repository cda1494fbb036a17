# Build everything in-tree (the .so files travel to the GPU box with the gpurun snapshot).
#   gen/libeggen.so                       seeded input generator (host C + CUDA), test/bench infra
#   oracle/liboracle.so                   CPU oracle (plain C, -ffp-contract=off), test infra
#   paper_1811_03852_b200/libegsolve.so   the product: sm_100a kernels behind the C ABI
NVCC    ?= /usr/local/cuda/bin/nvcc
CUDA    ?= /usr/local/cuda
ARCH    := -gencode arch=compute_100a,code=sm_100a
PY      ?= python
NCCL_DIR := $(shell $(PY) -c "import nvidia.nccl,os;print(list(nvidia.nccl.__path__)[0])" 2>/dev/null)
BUILD   := build

PKG     := paper_1811_03852_b200
CSRC    := $(wildcard $(PKG)/csrc/*.cu) $(wildcard $(PKG)/csrc/*.cuh) $(wildcard $(PKG)/csrc/*.h) include/egsolve.h
NVFLAGS := $(ARCH) -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v --expt-relaxed-constexpr

all: gen/libeggen.so oracle/liboracle.so $(PKG)/libegsolve.so

$(BUILD):
	mkdir -p $(BUILD)

gen/libeggen.so: gen/eggen_host.c gen/eggen_cuda.cu gen/eggen.h gen/eggen_formula.h | $(BUILD)
	gcc -O2 -fPIC -fopenmp -ffp-contract=off -c gen/eggen_host.c -o $(BUILD)/eggen_host.o
	$(NVCC) $(ARCH) -O3 -fmad=false -Xcompiler -fPIC -c gen/eggen_cuda.cu -o $(BUILD)/eggen_cuda.o
	$(NVCC) $(ARCH) -shared -o $@ $(BUILD)/eggen_host.o $(BUILD)/eggen_cuda.o -Xcompiler -fopenmp -lcudart

oracle/liboracle.so: oracle/oracle.c oracle/oracle.h
	gcc -O2 -fPIC -fopenmp -ffp-contract=off -shared -o $@ oracle/oracle.c -lm

$(PKG)/libegsolve.so: $(CSRC) | $(BUILD)
	$(NVCC) $(NVFLAGS) -Iinclude -I$(NCCL_DIR)/include -c $(PKG)/csrc/egsolve.cu -o $(BUILD)/egsolve.o 2> $(BUILD)/ptxas.log || (cat $(BUILD)/ptxas.log; false)
	$(NVCC) $(ARCH) -shared -o $@ $(BUILD)/egsolve.o -L$(NCCL_DIR)/lib -l:libnccl.so.2 -Xlinker -rpath=$(NCCL_DIR)/lib -lcudart

clean:
	rm -rf $(BUILD) gen/libeggen.so oracle/liboracle.so $(PKG)/libegsolve.so

.PHONY: all clean

# debug build with per-CTA cycle accounting of the fused phase kernels (scripts/march_trace.py)
trace: $(CSRC) | $(BUILD)
	$(NVCC) $(NVFLAGS) -DMA_TRACE -Iinclude -I$(NCCL_DIR)/include -shared -o $(BUILD)/libegsolve_trace.so $(PKG)/csrc/egsolve.cu -L$(NCCL_DIR)/lib -l:libnccl.so.2 -Xlinker -rpath=$(NCCL_DIR)/lib -lcudart 2> $(BUILD)/ptxas_trace.log || (cat $(BUILD)/ptxas_trace.log; false)

.PHONY: trace
