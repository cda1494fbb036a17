// probe_tma_coupled.cu — phase A's access pattern with the phase kernel's CONSUMER COUPLING:
// probe_tma_stream.cu plus (a) a busy delay of dF / dS cycles per stage for the F / S consumers
// (their arithmetic) and (b) the march's lockstep: F consumes row x stage q only after S consumed
// row x-2 stage q (sread, couple bit 2), and S starts row m only after F finished row m+1 (zready,
// couple bit 1; couple = 3 is the phase kernels').  With extra
// ring_kb shared memory it mimics the z ring; the question is how much deeper rings would buy.
//   ./probe_tma_coupled strips stagesF stagesS ring_kb dF dS couple
// (based on probe_tma_stream.cu, whose header follows)
// probe_tma_stream.cu — how fast can phase A's access pattern stream on its own?
//
// Same grid (strips x 128-column tiles, one CTA per SM), same TMA boxes (128 columns x MA_KS
// levels of r, p, v, (U,D) for the "F" ring and (E,W,N,S), rhat0 for the "S" ring), same stage
// sizes and 52 B / point (40 read, 12 written) as k_march<MODE,1>, but the consumer warps only
// touch the data (no Thomas, no stencil, no coupling between the F and S warps).  If this runs
// well above phase A's 6.2 TB/s, the phase kernel loses time in its compute / coupling; if not,
// the access pattern and ring depth are the limit.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1811_03852_b200/csrc \
//        -I../include probe_tma_stream.cu -o probe_tma_stream -lcuda   (binary git-ignored)
//   ./probe_tma_stream [strips=7] [stagesF=6] [stagesS=5] [ring_kb=112]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#include "march.cuh"

using namespace eg;

struct Maps { CUtensorMap r, p, v, rh, b2, b4; };

__global__ void __launch_bounds__(MA_THREADS, 1) k_probe(int nx, int nz, int nyl, int T, int strips, int NSF,
                                                         int NSS, float* __restrict__ po, float* __restrict__ zo,
                                                         float* __restrict__ vo, const __grid_constant__ Maps maps,
                                                         float* sink, int split, int dF, int dS, int couple, int lead) {
    constexpr int SF = ma_stage_floats(1), KS = MA_KS;
    extern __shared__ __align__(128) unsigned char smraw[];
    __shared__ __align__(8) uint64_t fullF[MA_MAX_STAGES], emptyF[MA_MAX_STAGES];
    __shared__ __align__(8) uint64_t fullS[MA_MAX_STAGES], emptyS[MA_MAX_STAGES];
    __shared__ __align__(8) uint64_t sreadq[2][32], zreadyq[4];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int t = blockIdx.x % T, strip = blockIdx.x / T;
    const int ja = (int)((int64_t)strip * nyl / strips), jb = (int)((int64_t)(strip + 1) * nyl / strips);
    const int L = jb - ja;
    const int i0 = t * 128;
    const int NZ8 = (nz + 7) / 8 * 8;
    float* stF = reinterpret_cast<float*>(smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u));
    float* stS = stF + (size_t)NSF * SF;
    if (tid == 0) {
        for (int s = 0; s < NSF; ++s) { mbar_init(&fullF[s], 1); mbar_init(&emptyF[s], MA_CONS); }
        for (int s = 0; s < NSS; ++s) { mbar_init(&fullS[s], 1); mbar_init(&emptyS[s], MA_CONS); }
        for (int q = 0; q < 32; ++q) { mbar_init(&sreadq[0][q], MA_CONS); mbar_init(&sreadq[1][q], MA_CONS); }
        for (int q = 0; q < 4; ++q) mbar_init(&zreadyq[q], MA_CONS);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == 8 || warp == 10) {  // warp 8: both rings in a fixed interleave (split = 0), or the F ring only
        const bool doS = warp == 8 ? !split : true, doF = warp == 8;
        if (warp == 10 && !split) return;
        if (lane == 0) {
            int fs = 0, fr = 0, ss = 0, sr = 0;
            for (int m = 0; m < L; ++m)
                for (int k0 = 0; k0 < NZ8; k0 += KS) {
                    const int j = ja + m;
                    if (doS) {
                    if (sr > 0) mbar_wait_sleep(&emptyS[ss], (uint32_t)((sr - 1) & 1), 32);
                    mbar_expect_tx(&fullS[ss], MA_BOX_B4 + MA_BOX_V);
                    float* sb = stS + (size_t)ss * SF;
                    tma3(sb, &maps.b4, 2 * i0, k0, j, &fullS[ss]);
                    tma3(sb + KS * 512, &maps.rh, i0, k0, j, &fullS[ss]);
                    if (++ss == NSS) { ss = 0; ++sr; }
                    }
                    if (!doF) continue;
                    if (fr > 0) mbar_wait_sleep(&emptyF[fs], (uint32_t)((fr - 1) & 1), 32);
                    mbar_expect_tx(&fullF[fs], 3u * MA_BOX_V + MA_BOX_B2);
                    float* fb = stF + (size_t)fs * SF;
                    tma3(fb, &maps.r, i0, k0, j, &fullF[fs]);
                    tma3(fb + KS * 128, &maps.p, i0, k0, j, &fullF[fs]);
                    tma3(fb + 2 * KS * 128, &maps.v, i0, k0, j, &fullF[fs]);
                    tma3(fb + 3 * KS * 128, &maps.b2, i0, k0, j, &fullF[fs]);
                    if (++fs == NSF) { fs = 0; ++fr; }
                }
        }
        return;
    }
    if (warp >= 9) return;  // (MA_THREADS also counts the phase kernels' publisher and halo warps)
    const bool isF = warp >= 4;
    const int col = tid & 127;
    int slot = 0;
    uint32_t ph = 0;
    float acc = 0.f;
    auto spin = [&](int cyc) {
        if (cyc <= 0) return;
        const long long t0 = clock64();
        while (clock64() - t0 < cyc) acc += 1e-30f;
    };
    for (int m = 0; m < L; ++m) {
        const int64_t rowoff = (int64_t)(ja + m) * nz * nx + i0 + col;
        if ((couple & 1) && !isF) {  // S: z(r_m) and z(r_{m+1}) complete
            // sets of 4 rows: F is at most `lead` rows ahead, so a set's phase never runs 2 ahead
            if (m == 0) mbar_wait(&zreadyq[0], 0u);
            if (m + 1 < L) mbar_wait(&zreadyq[(m + 1) & 3], (uint32_t)(((m + 1) >> 2) & 1));
        }
        for (int k0 = 0; k0 < NZ8; k0 += KS) {
            const int q = k0 / KS;
            if (isF) {
                if ((couple & 2) && m >= lead) mbar_wait(&sreadq[(m - lead) & 1][q], (uint32_t)(((m - lead) >> 1) & 1));
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
                    const float4 e = *reinterpret_cast<const float4*>(sb + l * 512 + 4 * col);
                    a[l] = e.x + e.y + e.z + e.w + sb[KS * 512 + l * 128 + col];
                }
                fence_proxy_async_smem();
                mbar_arrive(&emptyS[slot]);
                if (++slot == NSS) { slot = 0; ph ^= 1u; }
                if (couple & 2) mbar_arrive(&sreadq[m & 1][q]);
                spin(dS);
#pragma unroll
                for (int l = 0; l < KS; ++l)
                    if (k0 + l < nz) __stcg(vo + rowoff + (int64_t)(k0 + l) * nx, a[l]);
            }
        }
        if ((couple & 1) && isF) mbar_arrive(&zreadyq[m & 3]);  // F: row m done
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

int main(int argc, char** argv) {
    const int nx = 2560, ny = 1920, nz = 70;
    const int strips = argc > 1 ? atoi(argv[1]) : 7;
    const int NSF = argc > 2 ? atoi(argv[2]) : 6;
    const int NSS = argc > 3 ? atoi(argv[3]) : 5;
    const int ring_kb = argc > 4 ? atoi(argv[4]) : 0;  // extra smem to mimic the z ring
    const int split = 1;                               // one producer warp per ring (as the phase kernels)
    const int dF = argc > 5 ? atoi(argv[5]) : 0, dS = argc > 6 ? atoi(argv[6]) : 0, couple = argc > 7 ? atoi(argv[7]) : 3;
    const int lead = argc > 8 ? atoi(argv[8]) : 2;  // rows the F consumers run ahead of the S consumers
    const int64_t n = (int64_t)nx * ny * nz;
    const int T = nx / 128;
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
    bool ok = enc(f, &maps.r, r, nx, nz, ny, 4, 128) && enc(f, &maps.p, p, nx, nz, ny, 4, 128) &&
              enc(f, &maps.v, v, nx, nz, ny, 4, 128) && enc(f, &maps.rh, rh, nx, nz, ny, 4, 128) &&
              enc(f, &maps.b2, b2, nx, nz, ny, 8, 128) && enc(f, &maps.b4, b4, 2 * nx, nz, ny, 8, 256);
    if (!ok) { printf("encode failed\n"); return 1; }
    const size_t smem = (size_t)(NSF + NSS) * ma_stage_bytes(1) + (size_t)ring_kb * 1024 + 128;
    cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int grid = strips * T;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int it = 0; it < 2; ++it)
        k_probe<<<grid, MA_THREADS, smem>>>(nx, nz, ny, T, strips, NSF, NSS, po, zo, vo, maps, sink, split, dF, dS, couple, lead);
    cudaEventRecord(a);
    const int reps = 10;
    for (int it = 0; it < reps; ++it)
        k_probe<<<grid, MA_THREADS, smem>>>(nx, nz, ny, T, strips, NSF, NSS, po, zo, vo, maps, sink, split, dF, dS, couple, lead);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    ms /= reps;
    printf("lead=%d couple=%d dF=%d dS=%d strips=%d stagesF=%d stagesS=%d smem=%zu KB: %.3f ms  %.0f GB/s (52 B/pt)  %s\n", lead,
           couple, dF, dS, strips, NSF, NSS, smem / 1024, ms, 52.0 * n / (ms * 1e-3) / 1e9, cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
