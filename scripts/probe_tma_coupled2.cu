// probe_tma_coupled2.cu — probe_tma_coupled.cu generalised to the tile width: phase A's access
// pattern and F / S lockstep with TW = 128-column tiles (one CTA per SM, today's phase kernels) or
// TW = 64-column tiles with TWO CTAs per SM (two independent lockstep pipelines sharing an SM, the
// same number of compute warps per SM).  Question: does the second pipeline hide the lockstep?
//   ./probe_tma_coupled2 TW strips stagesF stagesS ring_kb dF dS
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "march.cuh"

using namespace eg;

struct Maps { CUtensorMap r, p, v, rh, b2, b4; };

template <int TW, int MINB>
__global__ void __launch_bounds__((2 * TW / 32 + 2) * 32, MINB) k_probe(int nx, int nz, int nyl, int T, int strips, int NSF,
                                                                        int NSS, float* __restrict__ po, float* __restrict__ zo,
                                                                        float* __restrict__ vo, const __grid_constant__ Maps maps,
                                                                        float* sink, int dF, int dS) {
    constexpr int KS = MA_KS, CONS = TW, NW = TW / 32;
    constexpr int SF = KS * 5 * TW;  // floats per stage (both rings)
    extern __shared__ __align__(128) unsigned char smraw[];
    __shared__ __align__(8) uint64_t fullF[MA_MAX_STAGES], emptyF[MA_MAX_STAGES];
    __shared__ __align__(8) uint64_t fullS[MA_MAX_STAGES], emptyS[MA_MAX_STAGES];
    __shared__ __align__(8) uint64_t sreadq[2][32], zreadyq[4];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int t = blockIdx.x % T, strip = blockIdx.x / T;
    const int ja = (int)((int64_t)strip * nyl / strips), jb = (int)((int64_t)(strip + 1) * nyl / strips);
    const int L = jb - ja;
    const int i0 = t * TW;
    const int NZ8 = (nz + 7) / 8 * 8;
    float* stF = reinterpret_cast<float*>(smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u));
    float* stS = stF + (size_t)NSF * SF;
    if (tid == 0) {
        for (int s = 0; s < NSF; ++s) { mbar_init(&fullF[s], 1); mbar_init(&emptyF[s], CONS); }
        for (int s = 0; s < NSS; ++s) { mbar_init(&fullS[s], 1); mbar_init(&emptyS[s], CONS); }
        for (int q = 0; q < 32; ++q) { mbar_init(&sreadq[0][q], CONS); mbar_init(&sreadq[1][q], CONS); }
        for (int q = 0; q < 4; ++q) mbar_init(&zreadyq[q], CONS);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp >= 2 * NW) {  // producers: warp 2NW the F ring, warp 2NW+1 the S ring
        const bool doF = warp == 2 * NW;
        if (lane == 0) {
            int fs = 0, fr = 0, ss = 0, sr = 0;
            const uint32_t bv = KS * TW * 4, bb2 = 2 * bv, bb4 = 4 * bv;
            for (int m = 0; m < L; ++m)
                for (int k0 = 0; k0 < NZ8; k0 += KS) {
                    const int j = ja + m;
                    if (!doF) {
                        if (sr > 0) mbar_wait_sleep(&emptyS[ss], (uint32_t)((sr - 1) & 1), 32);
                        mbar_expect_tx(&fullS[ss], bb4 + bv);
                        float* sb = stS + (size_t)ss * SF;
                        tma3(sb, &maps.b4, 2 * i0, k0, j, &fullS[ss]);
                        tma3(sb + KS * 4 * TW, &maps.rh, i0, k0, j, &fullS[ss]);
                        if (++ss == NSS) { ss = 0; ++sr; }
                    } else {
                        if (fr > 0) mbar_wait_sleep(&emptyF[fs], (uint32_t)((fr - 1) & 1), 32);
                        mbar_expect_tx(&fullF[fs], 3u * bv + bb2);
                        float* fb = stF + (size_t)fs * SF;
                        tma3(fb, &maps.r, i0, k0, j, &fullF[fs]);
                        tma3(fb + KS * TW, &maps.p, i0, k0, j, &fullF[fs]);
                        tma3(fb + 2 * KS * TW, &maps.v, i0, k0, j, &fullF[fs]);
                        tma3(fb + 3 * KS * TW, &maps.b2, i0, k0, j, &fullF[fs]);
                        if (++fs == NSF) { fs = 0; ++fr; }
                    }
                }
        }
        return;
    }
    const bool isF = warp >= NW;
    const int col = tid % TW;
    int slot = 0;
    uint32_t ph = 0;
    float acc = 0.f;
    auto spin = [&](int cyc) {
        if (cyc <= 0) return;
        const long long t0 = clock64();
        while (clock64() - t0 < cyc) acc += 1e-30f;
    };
    const int lead = 2;
    for (int m = 0; m < L; ++m) {
        const int64_t rowoff = (int64_t)(ja + m) * nz * nx + i0 + col;
        if (!isF) {
            if (m == 0) mbar_wait(&zreadyq[0], 0u);
            if (m + 1 < L) mbar_wait(&zreadyq[(m + 1) & 3], (uint32_t)(((m + 1) >> 2) & 1));
        }
        for (int k0 = 0; k0 < NZ8; k0 += KS) {
            const int q = k0 / KS;
            if (isF) {
                if (m >= lead) mbar_wait(&sreadq[(m - lead) & 1][q], (uint32_t)(((m - lead) >> 1) & 1));
                mbar_wait(&fullF[slot], ph);
                const float* sb = stF + (size_t)slot * SF;
                float a[KS], b[KS];
#pragma unroll
                for (int l = 0; l < KS; ++l) {
                    const float2 ud = *reinterpret_cast<const float2*>(sb + 3 * KS * TW + l * 2 * TW + 2 * col);
                    a[l] = sb[l * TW + col] + sb[KS * TW + l * TW + col] * ud.x;
                    b[l] = sb[2 * KS * TW + l * TW + col] + ud.y;
                }
                fence_proxy_async_smem();
                mbar_arrive(&emptyF[slot]);
                if (++slot == NSF) { slot = 0; ph ^= 1u; }
                spin(dF);
#pragma unroll
                for (int l = 0; l < KS; ++l)
                    if (k0 + l < nz) {
                        __stcg(po + rowoff + (int64_t)(k0 + l) * nx, a[l]);
                        __stcg(zo + rowoff + (int64_t)(k0 + l) * nx, b[l]);
                    }
            } else {
                mbar_wait(&fullS[slot], ph);
                const float* sb = stS + (size_t)slot * SF;
                float a[KS];
#pragma unroll
                for (int l = 0; l < KS; ++l) {
                    const float4 e = *reinterpret_cast<const float4*>(sb + l * 4 * TW + 4 * col);
                    a[l] = e.x + e.y + e.z + e.w + sb[KS * 4 * TW + l * TW + col];
                }
                fence_proxy_async_smem();
                mbar_arrive(&emptyS[slot]);
                if (++slot == NSS) { slot = 0; ph ^= 1u; }
                mbar_arrive(&sreadq[m & 1][q]);
                spin(dS);
#pragma unroll
                for (int l = 0; l < KS; ++l)
                    if (k0 + l < nz) __stcg(vo + rowoff + (int64_t)(k0 + l) * nx, a[l]);
            }
        }
        if (isF) mbar_arrive(&zreadyq[m & 3]);  // F: row m done
    }
    if (acc != 0.f) sink[0] = acc;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static bool enc(EncFn f, CUtensorMap* m, void* base, int64_t inner, int64_t nz, int64_t nyl, int esz, int box0) {
    const cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)nz, (cuuint64_t)nyl};
    const cuuint64_t str[2] = {(cuuint64_t)(inner * esz), (cuuint64_t)(inner * nz * esz)};
    const cuuint32_t box[3] = {(cuuint32_t)box0, (cuuint32_t)MA_KS, 1u};
    const cuuint32_t es[3] = {1u, 1u, 1u};
    return f(m, esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, base, dims, str, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int TW, int MINB>
int run(int strips, int NSF, int NSS, int ring_kb, int dF, int dS) {
    const int nx = 2560, ny = 1920, nz = 70;
    const int64_t n = (int64_t)nx * ny * nz;
    const int T = nx / TW;
    float *r, *p, *v, *rh, *b2, *b4, *po, *zo, *vo, *sink;
    cudaMalloc(&r, n * 4); cudaMalloc(&p, n * 4); cudaMalloc(&v, n * 4); cudaMalloc(&rh, n * 4);
    cudaMalloc(&b2, n * 8); cudaMalloc(&b4, n * 16);
    cudaMalloc(&po, n * 4); cudaMalloc(&zo, n * 4); cudaMalloc(&vo, n * 4); cudaMalloc(&sink, 64);
    for (float* a : {r, p, v, rh, po, zo, vo}) cudaMemset(a, 0, n * 4);
    cudaMemset(b2, 0, n * 8);
    cudaMemset(b4, 0, n * 16);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
    EncFn f = (EncFn)fn;
    Maps maps;
    bool ok = enc(f, &maps.r, r, nx, nz, ny, 4, TW) && enc(f, &maps.p, p, nx, nz, ny, 4, TW) &&
              enc(f, &maps.v, v, nx, nz, ny, 4, TW) && enc(f, &maps.rh, rh, nx, nz, ny, 4, TW) &&
              enc(f, &maps.b2, b2, nx, nz, ny, 8, TW) && enc(f, &maps.b4, b4, 2 * nx, nz, ny, 8, 2 * TW);
    if (!ok) { printf("encode failed\n"); return 1; }
    const size_t smem = (size_t)(NSF + NSS) * MA_KS * 5 * TW * 4 + (size_t)ring_kb * 1024 + 128;
    cudaFuncSetAttribute(k_probe<TW, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int occ = 0;
    const int threads = (2 * TW / 32 + 2) * 32;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_probe<TW, MINB>, threads, smem);
    const int grid = strips * T;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int it = 0; it < 2; ++it)
        k_probe<TW, MINB><<<grid, threads, smem>>>(nx, nz, ny, T, strips, NSF, NSS, po, zo, vo, maps, sink, dF, dS);
    cudaEventRecord(a);
    const int reps = 10;
    for (int it = 0; it < reps; ++it)
        k_probe<TW, MINB><<<grid, threads, smem>>>(nx, nz, ny, T, strips, NSF, NSS, po, zo, vo, maps, sink, dF, dS);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    printf("TW=%d grid=%d (occ %d/SM) dF=%d dS=%d strips=%d stages %d+%d smem=%zu KB: %.3f ms  %.0f GB/s (52 B/pt)  %s\n", TW,
           grid, occ, dF, dS, strips, NSF, NSS, smem / 1024, ms, 52.0 * n / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
    cudaFree(r); cudaFree(p); cudaFree(v); cudaFree(rh); cudaFree(b2); cudaFree(b4);
    cudaFree(po); cudaFree(zo); cudaFree(vo); cudaFree(sink);
    return e == cudaSuccess ? 0 : 1;
}

int main(int argc, char** argv) {
    const int TW = argc > 1 ? atoi(argv[1]) : 128;
    const int strips = argc > 2 ? atoi(argv[2]) : 7;
    const int NSF = argc > 3 ? atoi(argv[3]) : 6, NSS = argc > 4 ? atoi(argv[4]) : 5;
    const int ring_kb = argc > 5 ? atoi(argv[5]) : 112;
    const int dF = argc > 6 ? atoi(argv[6]) : 0, dS = argc > 7 ? atoi(argv[7]) : 0;
    return TW == 64 ? run<64, 2>(strips, NSF, NSS, ring_kb, dF, dS) : run<128, 1>(strips, NSF, NSS, ring_kb, dF, dS);
}
