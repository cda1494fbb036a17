// probe_tma_pair.cu — phase A's TMA stream (probe_tma_stream.cu) with the two tiles of a CTA pair
// (a cluster of 2 adjacent tiles of one strip) loaded by ONE producer, back to back: box t into
// this CTA's stage, box t+1 into the peer's (shared::cluster destination and mbarrier).  Does the
// DRAM side reward adjacent 512-B segments issued together, like one 1-KB segment?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -I../paper_1811_03852_b200/csrc -I../include probe_tma_pair.cu -o probe_tma_pair -lcuda
//   ./probe_tma_pair [stagesF=6] [stagesS=5] [pair=1]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "march.cuh"

using namespace eg;

struct Maps { CUtensorMap r, p, v, rh, b2, b4; };

__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void tma3_c(uint32_t dst, const CUtensorMap* map, int c0, int k0, int j, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(k0), "r"(j), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void expect_tx_c(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.relaxed.cluster.shared::cluster.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void arrive_c(uint32_t bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void arrive_c_relaxed(uint32_t bar) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cta_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(MA_THREADS, 1)
    k_pair(int nx, int nz, int nyl, int T, int strips, int NSF, int NSS, float* __restrict__ po, float* __restrict__ zo,
           float* __restrict__ vo, const __grid_constant__ Maps maps, int pair) {
    constexpr int SF = ma_stage_floats(1), KS = MA_KS;
    extern __shared__ __align__(128) unsigned char smp[];
    __shared__ __align__(8) uint64_t fullF[MA_MAX_STAGES], emptyF[MA_MAX_STAGES];
    __shared__ __align__(8) uint64_t fullS[MA_MAX_STAGES], emptyS[MA_MAX_STAGES];
    __shared__ __align__(8) uint64_t pemptyF[MA_MAX_STAGES], pemptyS[MA_MAX_STAGES];  // pair = 2: the peer's relay
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t rk = cta_rank();
    const int t = blockIdx.x % T, strip = blockIdx.x / T;
    const int ja = (int)((int64_t)strip * nyl / strips), jb = (int)((int64_t)(strip + 1) * nyl / strips);
    const int L = jb - ja;
    const int i0 = t * 128;
    const int NZ8 = (nz + 7) / 8 * 8;
    float* stF = reinterpret_cast<float*>(smp + ((128u - (smem_u32(smp) & 127u)) & 127u));
    float* stS = stF + (size_t)NSF * SF;
    if (tid == 0) {
        // the rank-0 CTA's empty barriers count both CTAs' consumers
        // one arrival per consumer warp of both CTAs (after the warp's reads, __syncwarp)
        const int ec = (pair == 1 ? 2 : 1) * MA_CONS / 32;
        for (int s = 0; s < NSF; ++s) { mbar_init(&fullF[s], 1); mbar_init(&emptyF[s], ec); mbar_init(&pemptyF[s], 1); }
        for (int s = 0; s < NSS; ++s) { mbar_init(&fullS[s], 1); mbar_init(&emptyS[s], ec); mbar_init(&pemptyS[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cluster_sync();
    if ((warp == 8 || warp == 10) && pair >= 2 && rk == 1) {  // relay: local empty -> the producer CTA
        if (lane == 0) {
            const bool isF = warp == 8;
            const int NS = isF ? NSF : NSS;
            uint64_t* empty = isF ? emptyF : emptyS;
            uint64_t* pempty = isF ? pemptyF : pemptyS;
            int slot = 0, round = 0;
            for (int m = 0; m < L; ++m)
                for (int k0 = 0; k0 < NZ8; k0 += KS) {
                    mbar_wait_sleep(&empty[slot], (uint32_t)(round & 1), 32);
                    if (pair == 3) arrive_c_relaxed(mapa_u32(smem_u32(&pempty[slot]), 0));
                    else arrive_c(mapa_u32(smem_u32(&pempty[slot]), 0));
                    if (++slot == NS) { slot = 0; ++round; }
                }
        }
    } else if ((warp == 8 || warp == 10) && (rk == 0 || !pair)) {
        if (lane == 0) {
            const bool isF = warp == 8;
            const int NS = isF ? NSF : NSS;
            uint64_t* full = isF ? fullF : fullS;
            uint64_t* empty = isF ? emptyF : emptyS;
            uint64_t* pempty = isF ? pemptyF : pemptyS;
            float* st = isF ? stF : stS;
            int slot = 0, round = 0;
            for (int m = 0; m < L; ++m)
                for (int k0 = 0; k0 < NZ8; k0 += KS) {
                    const int j = ja + m;
                    if (round > 0) mbar_wait_sleep(&empty[slot], (uint32_t)((round - 1) & 1), 32);
                    if (round > 0 && pair >= 2) mbar_wait_sleep(&pempty[slot], (uint32_t)((round - 1) & 1), 32);
                    const uint32_t bytes = isF ? 3u * MA_BOX_V + MA_BOX_B2 : MA_BOX_B4 + MA_BOX_V;
                    for (uint32_t c = 0; c < (pair ? 2u : 1u); ++c) {  // this CTA's tile (, then the peer's)
                        const uint32_t tgt = pair ? c : rk;
                        const uint32_t bar = mapa_u32(smem_u32(&full[slot]), tgt);
                        const uint32_t dst = mapa_u32(smem_u32(st + (size_t)slot * SF), tgt);
                        const int ic = i0 + 128 * (int)c;
                        expect_tx_c(bar, bytes);
                        if (isF) {
                            tma3_c(dst, &maps.r, ic, k0, j, bar);
                            tma3_c(dst + 4 * KS * 128, &maps.p, ic, k0, j, bar);
                            tma3_c(dst + 8 * KS * 128, &maps.v, ic, k0, j, bar);
                            tma3_c(dst + 12 * KS * 128, &maps.b2, ic, k0, j, bar);
                        } else {
                            tma3_c(dst, &maps.b4, 2 * ic, k0, j, bar);
                            tma3_c(dst + 4 * KS * 512, &maps.rh, ic, k0, j, bar);
                        }
                    }
                    if (++slot == NS) { slot = 0; ++round; }
                }
        }
    } else if (warp < 8) {
        const bool isF = warp >= 4;
        const int col = tid & 127;
        int slot = 0;
        uint32_t ph = 0;
        for (int m = 0; m < L; ++m) {
            const int64_t rowoff = (int64_t)(ja + m) * nz * nx + i0 + col;
            for (int k0 = 0; k0 < NZ8; k0 += KS) {
                if (isF) {
                    mbar_wait(&fullF[slot], ph);
                    const float* sb = stF + (size_t)slot * SF;
                    float a[KS], b[KS];
#pragma unroll
                    for (int l = 0; l < KS; ++l) {
                        const float2 ud = *reinterpret_cast<const float2*>(sb + 3 * KS * 128 + l * 256 + 2 * col);
                        a[l] = sb[l * 128 + col] + sb[KS * 128 + l * 128 + col] * ud.x;
                        b[l] = sb[2 * KS * 128 + l * 128 + col] + ud.y;
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if (pair >= 2) mbar_arrive(&emptyF[slot]);  // CTA-local; the relay forwards it
                        else arrive_c(mapa_u32(smem_u32(&emptyF[slot]), pair ? 0u : rk));
                    }
                    if (++slot == NSF) { slot = 0; ph ^= 1u; }
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
                        const float4 e = *reinterpret_cast<const float4*>(sb + l * 512 + 4 * col);
                        a[l] = e.x + e.y + e.z + e.w + sb[KS * 512 + l * 128 + col];
                    }
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        if (pair >= 2) mbar_arrive(&emptyS[slot]);
                        else arrive_c(mapa_u32(smem_u32(&emptyS[slot]), pair ? 0u : rk));
                    }
                    if (++slot == NSS) { slot = 0; ph ^= 1u; }
#pragma unroll
                    for (int l = 0; l < KS; ++l)
                        if (k0 + l < nz) __stcg(vo + rowoff + (int64_t)(k0 + l) * nx, a[l]);
                }
            }
        }
    }
    cluster_sync();  // no CTA leaves while the peer may still arrive on its barriers
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
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int main(int argc, char** argv) {
    const int nx = 2560, ny = 1920, nz = 70, strips = 7;
    const int NSF = argc > 1 ? atoi(argv[1]) : 6;
    const int NSS = argc > 2 ? atoi(argv[2]) : 5;
    const int pair = argc > 3 ? atoi(argv[3]) : 1;
    const int64_t n = (int64_t)nx * ny * nz;
    const int T = nx / 128;
    float *r, *p, *v, *rh, *b2, *b4, *po, *zo, *vo;
    cudaMalloc(&r, n * 4); cudaMalloc(&p, n * 4); cudaMalloc(&v, n * 4); cudaMalloc(&rh, n * 4);
    cudaMalloc(&b2, n * 8); cudaMalloc(&b4, n * 16);
    cudaMalloc(&po, n * 4); cudaMalloc(&zo, n * 4); cudaMalloc(&vo, n * 4);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
    EncFn f = (EncFn)fn;
    Maps maps;
    bool ok = enc(f, &maps.r, r, nx, nz, ny, 4, 128) && enc(f, &maps.p, p, nx, nz, ny, 4, 128) &&
              enc(f, &maps.v, v, nx, nz, ny, 4, 128) && enc(f, &maps.rh, rh, nx, nz, ny, 4, 128) &&
              enc(f, &maps.b2, b2, nx, nz, ny, 8, 128) && enc(f, &maps.b4, b4, 2 * nx, nz, ny, 8, 256);
    if (!ok) { printf("encode failed\n"); return 1; }
    const size_t smem = (size_t)(NSF + NSS) * ma_stage_bytes(1) + 112 * 1024 + 128;  // + the phase kernels' z ring
    cudaFuncSetAttribute(k_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = strips * T;
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(MA_THREADS);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at;
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = 2; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
        cfg.attrs = &at;
        cfg.numAttrs = 1;
        int nclu = 0;
        cudaError_t eo = cudaOccupancyMaxActiveClusters(&nclu, (void*)k_pair, &cfg);
        printf("max active 2-CTA clusters: %d (%s); grid needs %d\n", nclu, cudaGetErrorString(eo), grid / 2);
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int it = 0; it < 2; ++it) k_pair<<<grid, MA_THREADS, smem>>>(nx, nz, ny, T, strips, NSF, NSS, po, zo, vo, maps, pair);
    cudaError_t e0 = cudaDeviceSynchronize();
    if (e0 != cudaSuccess) { printf("launch failed: %s\n", cudaGetErrorString(e0)); return 1; }
    cudaEventRecord(a);
    const int reps = 10;
    for (int it = 0; it < reps; ++it) k_pair<<<grid, MA_THREADS, smem>>>(nx, nz, ny, T, strips, NSF, NSS, po, zo, vo, maps, pair);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    printf("pair=%d: strips=%d grid=%d stages=%d+%d smem=%zu KB: %.3f ms  %.0f GB/s (52 B/pt)  %s\n", pair, strips, grid, NSF, NSS,
           smem / 1024, ms, 52.0 * n / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
