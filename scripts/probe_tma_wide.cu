// probe_tma_wide.cu — phase A's streaming pattern with 256-column tiles (1 KB box rows for the fp32
// arrays, 2 KB for (U,D), 4 KB for (E,W,N,S)) instead of 128: does the DRAM side reward longer
// contiguous segments?  Same 52 B/pt and the same per-SM bytes in flight as probe_tma_stream.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I../paper_1811_03852_b200/csrc -I../include probe_tma_wide.cu -o probe_tma_wide -lcuda
//   ./probe_tma_wide [strips=14] [stages per ring=5] [tile=256]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "march.cuh"

using namespace eg;

struct Maps { CUtensorMap r, p, v, rh, b2, b4; };
constexpr int KS = MA_KS;

template <int TW>
__global__ void __launch_bounds__(288, 1) k_wide(int nx, int nz, int nyl, int T, int strips, int NS, float* __restrict__ po,
                                                 float* __restrict__ zo, float* __restrict__ vo,
                                                 const __grid_constant__ Maps maps) {
    constexpr int FSF = KS * (3 * TW + 2 * TW), SSF = KS * (4 * TW + TW);  // floats per stage
    constexpr int NB = TW / 128;  // boxes per array row (box inner <= 256 elements)
    extern __shared__ __align__(128) unsigned char smraw[];
    __shared__ __align__(8) uint64_t fullF[16], emptyF[16], fullS[16], emptyS[16];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int t = blockIdx.x % T, strip = blockIdx.x / T;
    const int ja = (int)((int64_t)strip * nyl / strips), jb = (int)((int64_t)(strip + 1) * nyl / strips);
    const int L = jb - ja, i0 = t * TW, NZ8 = (nz + 7) / 8 * 8;
    float* stF = reinterpret_cast<float*>(smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u));
    float* stS = stF + (size_t)NS * FSF;
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            mbar_init(&fullF[s], 1); mbar_init(&emptyF[s], 128);
            mbar_init(&fullS[s], 1); mbar_init(&emptyS[s], 128);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 8) {
        if (lane == 0) {
            int fs = 0, fr = 0, ss = 0, sr = 0;
            for (int m = 0; m < L; ++m)
                for (int k0 = 0; k0 < NZ8; k0 += KS) {
                    const int j = ja + m;
                    if (sr > 0) mbar_wait_sleep(&emptyS[ss], (uint32_t)((sr - 1) & 1), 32);
                    mbar_expect_tx(&fullS[ss], SSF * 4);
                    float* sb = stS + (size_t)ss * SSF;
                    for (int b = 0; b < NB; ++b) tma3(sb + b * KS * 512, &maps.b4, 2 * i0 + 256 * b, k0, j, &fullS[ss]);
                    tma3(sb + KS * 4 * TW, &maps.rh, i0, k0, j, &fullS[ss]);
                    if (++ss == NS) { ss = 0; ++sr; }
                    if (fr > 0) mbar_wait_sleep(&emptyF[fs], (uint32_t)((fr - 1) & 1), 32);
                    mbar_expect_tx(&fullF[fs], FSF * 4);
                    float* fb = stF + (size_t)fs * FSF;
                    tma3(fb, &maps.r, i0, k0, j, &fullF[fs]);
                    tma3(fb + KS * TW, &maps.p, i0, k0, j, &fullF[fs]);
                    tma3(fb + 2 * KS * TW, &maps.v, i0, k0, j, &fullF[fs]);
                    for (int b = 0; b < NB; ++b) tma3(fb + 3 * KS * TW + b * KS * 256, &maps.b2, i0 + 128 * b, k0, j, &fullF[fs]);
                    if (++fs == NS) { fs = 0; ++fr; }
                }
        }
        return;
    }
    const bool isF = warp >= 4;
    const int c = tid & 127;
    int slot = 0;
    uint32_t ph = 0;
    for (int m = 0; m < L; ++m) {
        const int64_t rowoff = (int64_t)(ja + m) * nz * nx + i0;
        for (int k0 = 0; k0 < NZ8; k0 += KS) {
            if (isF) {
                mbar_wait(&fullF[slot], ph);
                const float* sb = stF + (size_t)slot * FSF;
                float a[KS][TW / 128], z[KS][TW / 128];
#pragma unroll
                for (int l = 0; l < KS; ++l)
#pragma unroll
                    for (int h = 0; h < TW / 128; ++h) {
                        const int col = c + 128 * h;
                        a[l][h] = sb[l * TW + col] + sb[KS * TW + l * TW + col];
                        z[l][h] = sb[2 * KS * TW + l * TW + col] + sb[3 * KS * TW + l * 2 * TW + 2 * col];
                    }
                fence_proxy_async_smem();
                mbar_arrive(&emptyF[slot]);
                if (++slot == NS) { slot = 0; ph ^= 1u; }
#pragma unroll
                for (int l = 0; l < KS; ++l)
                    if (k0 + l < nz)
#pragma unroll
                        for (int h = 0; h < TW / 128; ++h) {
                            __stcg(po + rowoff + (int64_t)(k0 + l) * nx + c + 128 * h, a[l][h]);
                            __stcg(zo + rowoff + (int64_t)(k0 + l) * nx + c + 128 * h, z[l][h]);
                        }
            } else {
                mbar_wait(&fullS[slot], ph);
                const float* sb = stS + (size_t)slot * SSF;
                float a[KS][TW / 128];
#pragma unroll
                for (int l = 0; l < KS; ++l)
#pragma unroll
                    for (int h = 0; h < TW / 128; ++h) {
                        const int col = c + 128 * h;
                        const float4 e = *reinterpret_cast<const float4*>(sb + l * 4 * TW + 4 * col);
                        a[l][h] = e.x + e.y + e.z + e.w + sb[KS * 4 * TW + l * TW + col];
                    }
                fence_proxy_async_smem();
                mbar_arrive(&emptyS[slot]);
                if (++slot == NS) { slot = 0; ph ^= 1u; }
#pragma unroll
                for (int l = 0; l < KS; ++l)
                    if (k0 + l < nz)
#pragma unroll
                        for (int h = 0; h < TW / 128; ++h) __stcg(vo + rowoff + (int64_t)(k0 + l) * nx + c + 128 * h, a[l][h]);
            }
        }
    }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static bool enc(EncFn f, CUtensorMap* m, void* base, int64_t inner, int64_t nz, int64_t nyl, int esz, int box0) {
    const cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)nz, (cuuint64_t)nyl};
    const cuuint64_t str[2] = {(cuuint64_t)(inner * esz), (cuuint64_t)(inner * nz * esz)};
    const cuuint32_t box[3] = {(cuuint32_t)box0, (cuuint32_t)KS, 1u};
    const cuuint32_t es[3] = {1u, 1u, 1u};
    return f(m, esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, base, dims, str, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int main(int argc, char** argv) {
    const int nx = 2560, ny = 1920, nz = 70;
    const int strips = argc > 1 ? atoi(argv[1]) : 14;
    const int NS = argc > 2 ? atoi(argv[2]) : 5;
    const int TW = argc > 3 ? atoi(argv[3]) : 256;
    const int64_t n = (int64_t)nx * ny * nz;
    const int T = nx / TW;
    float *r, *p, *v, *rh, *b2, *b4, *po, *zo, *vo;
    cudaMalloc(&r, n * 4); cudaMalloc(&p, n * 4); cudaMalloc(&v, n * 4); cudaMalloc(&rh, n * 4);
    cudaMalloc(&b2, n * 8); cudaMalloc(&b4, n * 16);
    cudaMalloc(&po, n * 4); cudaMalloc(&zo, n * 4); cudaMalloc(&vo, n * 4);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
    EncFn f = (EncFn)fn;
    Maps maps;
    const int bw = TW > 256 ? 256 : TW;
    bool ok = enc(f, &maps.r, r, nx, nz, ny, 4, TW) && enc(f, &maps.p, p, nx, nz, ny, 4, TW) &&
              enc(f, &maps.v, v, nx, nz, ny, 4, TW) && enc(f, &maps.rh, rh, nx, nz, ny, 4, TW) &&
              enc(f, &maps.b2, b2, nx, nz, ny, 8, 128) && enc(f, &maps.b4, b4, 2 * nx, nz, ny, 8, 256);
    (void)bw;
    if (!ok) { printf("encode failed\n"); return 1; }
    const int FSF = KS * 5 * TW, SSF = KS * 5 * TW;
    const size_t smem = (size_t)NS * (FSF + SSF) * 4 + 128;
    auto kern = TW == 256 ? k_wide<256> : k_wide<128>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = strips * T;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int it = 0; it < 2; ++it) kern<<<grid, 288, smem>>>(nx, nz, ny, T, strips, NS, po, zo, vo, maps);
    cudaEventRecord(a);
    const int reps = 10;
    for (int it = 0; it < reps; ++it) kern<<<grid, 288, smem>>>(nx, nz, ny, T, strips, NS, po, zo, vo, maps);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    printf("tile=%d strips=%d grid=%d stages=%d+%d smem=%zu KB: %.3f ms  %.0f GB/s  %s\n", TW, strips, grid, NS, NS,
           smem / 1024, ms, 52.0 * n / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
