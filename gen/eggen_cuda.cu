/* eggen_cuda.cu — device side of the seeded problem generator (see eggen.h).
 * Same per-point formula as eggen_host.c (eggen_formula.h), FMA-free, so the bits match. */
#include <cuda_runtime.h>
#include <stdlib.h>
#include "eggen.h"
#include "eggen_formula.h"

__global__ void eggen_kernel(uint64_t seed, int64_t nx, int64_t ny, int64_t nz, double ch_lo,
                             double ch_w, double cv_lo, double cv_w, double dl_lo, double dl_w,
                             const double* __restrict__ coslat, int64_t j_begin, int64_t nrows,
                             double* __restrict__ bands, double* __restrict__ b) {
    const int64_t row = nx * nz;
    const int64_t nloc = nrows * row;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nloc;
         q += (int64_t)gridDim.x * blockDim.x) {
        int64_t jl = q / row;
        int64_t rem = q - jl * row;
        int64_t k = rem / nx;
        int64_t i = rem - k * nx;
        int64_t j = j_begin + jl;
        double v[8];
        gen_point(seed, nx, ny, nz, ch_lo, ch_w, cv_lo, cv_w, dl_lo, dl_w, coslat[j], i, j, k, v);
#pragma unroll
        for (int d = 0; d < 7; ++d) bands[(int64_t)d * nloc + q] = v[d];
        if (b) b[q] = v[7];
    }
}

extern "C" int eggen_device(const eggen_params* p, int64_t j_begin, int64_t j_end, double* bands,
                            double* b, void* stream) {
    if (!p || !bands || p->nx < 1 || p->ny < 1 || p->nz < 1 || j_begin < 0 || j_end > p->ny ||
        j_begin > j_end)
        return -1;
    cudaStream_t st = (cudaStream_t)stream;
    double* cl_h = (double*)malloc(sizeof(double) * (size_t)p->ny);
    if (!cl_h) return -1;
    eggen_coslat(p->ny, cl_h);
    double* cl_d = nullptr;
    if (cudaMallocAsync(&cl_d, sizeof(double) * p->ny, st) != cudaSuccess) { free(cl_h); return -2; }
    cudaMemcpyAsync(cl_d, cl_h, sizeof(double) * p->ny, cudaMemcpyHostToDevice, st);
    int64_t nrows = j_end - j_begin;
    int64_t nloc = nrows * p->nx * p->nz;
    if (nloc > 0) {
        int dev = 0, nsm = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
        int64_t blocks = (nloc + 255) / 256;
        if (blocks > (int64_t)nsm * 16) blocks = (int64_t)nsm * 16;
        eggen_kernel<<<(unsigned)blocks, 256, 0, st>>>(
            p->seed, p->nx, p->ny, p->nz, p->ch_lo, p->ch_hi - p->ch_lo, p->cv_lo,
            p->cv_hi - p->cv_lo, p->dl_lo, p->dl_hi - p->dl_lo, cl_d, j_begin, nrows, bands, b);
    }
    cudaFreeAsync(cl_d, st);
    cudaError_t e = cudaStreamSynchronize(st);  /* cl_h must outlive the async copy */
    free(cl_h);
    return (e == cudaSuccess && cudaGetLastError() == cudaSuccess) ? 0 : -2;
}
