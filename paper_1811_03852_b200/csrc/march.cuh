// march.cuh — fused phase kernels of the BiCGStab iteration (fp32 working precision, one GPU).
//
//   phase A (rows a3 + a4):  p = r + beta (p - omega v);  z = T^-1 p;  v = Ahat z;  partial rhat0 . v
//   phase B (rows a6 + a7):  s = r - alpha v;  z_s = T^-1 s;  t = Ahat z_s;  partials t.s, t.t, s.s
//
// The 5-kernel schedule moves 164 B / point / iteration because each stencil re-reads z (or z_s)
// and the (U, D) bands its Thomas solve has just read.  Here one persistent CTA per SM owns a
// 128-column tile of a STRIP of latitude rows and MARCHES through it row by row.  At step n it
//   1. forward-eliminates row r_n (the update that forms the right-hand side is fused in), keeping
//      the factors c'_k, the bands U_k, D_k (and s_k in phase B) in its TMEM lanes,
//   2. back-substitutes z(r_n) into a 3-row shared-memory ring (and writes z to HBM for the
//      update kernel), publishes a ready flag for (r_n, tile),
//   3. applies the stencil to row r_{n-1}: centre / N / S values come from the ring, E / W halo
//      columns from the neighbouring tiles' z in L2 (after their flags), U / D from TMEM.
// Every HBM byte is therefore read or written once: 52 B / point for phase A, 44 B for phase B,
// with the 40 B update that is 136 B / point / iteration, the algorithmic minimum with the paper's
// three global sums.
//
// The inputs a CTA streams (r, p, v, (U,D) for the elimination; (E,W,N,S), rhat0 for the stencil)
// do not depend on its arithmetic, so two producer warps stream them with TMA tensor copies into
// rings of MA_KS-level stages (mbarrier full / empty pairs) far ahead of the consumer warps.  The
// arithmetic, its order and the reduction slots are those of k_thomas_tm + k_stencil, so the fused
// schedule is bitwise identical to the 5-kernel one (tests/test_gpu_parity.py).
//
// Strips alternate direction (even: ascending rows, odd: descending), so a strip's first row
// neighbours the adjacent strip's first row and its last row the other neighbour's last row.  A
// CTA only ever waits for Thomas results that never wait themselves on the waiting CTA's later
// work, so with all CTAs co-resident (grid <= #SMs, one CTA per SM) the march cannot deadlock.
// The producer issues one TMA box (128 columns x MA_KB levels) per array per stage.
// Requires: nx % 4 == 0 (16-byte TMA strides), 7 * ceil8(nz) <= 512 TMEM columns, tiles <= #SMs.
// Multi-GPU: the band's first / last rows' neighbours are the ghost rows -1 / nyl of z, which the
// exchange (k_edge_rows + NCCL on a communication stream) fills WHILE this kernel runs: the stencil
// of those two rows (which read them) is computed but not stored (MarchGeo.skip_lo / skip_hi), and
// k_stencil redoes the two rows after the exchange, bitwise the same arithmetic.
#pragma once
#include <cuda.h>  // CUtensorMap (the host encodes the maps through cudaGetDriverEntryPointByVersion)

#include "kernels.cuh"

namespace eg {

constexpr int MA_KB = 8;                               // levels per stage
constexpr int MA_CONS = 128;                           // consumer threads: one column each
constexpr int MA_THREADS = 2 * MA_CONS + 128;          // stencil + Thomas warps, 2 producers, publisher, halo
// stage = one MA_KB-level chunk of one row.  Elimination ring: r, (p,) v, (U, D); stencil ring:
// (E, W, N, S) (, rhat0): 640 floats / level in phase A, 512 in phase B, for both rings
constexpr int MA_KS = 4;  // levels per stage: a chunk of MA_KB levels is two stages (finer refill)
constexpr int ma_stage_floats(int kind) { return MA_KS * (kind == 1 ? 640 : 512); }
constexpr int ma_stage_bytes(int kind) { return 4 * ma_stage_floats(kind); }
constexpr int MA_MAX_STAGES = 16;
constexpr int MA_RING_W = 130;                         // W halo | 128 columns | E halo

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void cons_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }  // stencil warps
__device__ __forceinline__ int ld_volatile(const int* p) {
    int v;
    asm volatile("ld.volatile.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void tm_ld8_nw(uint32_t taddr, float (&c)[8]) {  // no wait::ld
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
#pragma unroll
    for (int e = 0; e < 8; ++e) c[e] = __uint_as_float(r[e]);
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred P;\n"
        "MA_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n"
        " @!P bra MA_WAIT_%=;\n}\n" ::"r"(smem_u32(b)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred P;\n"
        " mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n"
        " selp.u32 %0, 1, 0, P;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
// waits of the producer / publisher warps back off so that they do not take issue slots from the
// consumer warp sharing their SM sub-partition
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity, int ns) {
    while (!mbar_test(b, parity)) __nanosleep(ns);
}
// A/B knob (build flag MA_WAIT_MODE): 0 = the producers / publisher poll with a back-off sleep;
// 1 = producers wait with try_wait (suspended in hardware until the phase completes); 2 = both
#ifndef MA_WAIT_MODE
#define MA_WAIT_MODE 0
#endif
#if MA_WAIT_MODE >= 1
#define MA_PROD_WAIT(b, p) mbar_wait((b), (p))
#else
#define MA_PROD_WAIT(b, p) mbar_wait_sleep((b), (p), 32)
#endif
#if MA_WAIT_MODE >= 2
#define MA_PUB_WAIT(b, p) mbar_wait((b), (p))
#else
#define MA_PUB_WAIT(b, p) mbar_wait_sleep((b), (p), 256)
#endif
// a consumer's generic-proxy reads of a stage must be ordered before the TMA (async proxy) that
// refills it: without this fence the refill can land before the reads are performed (observed as a
// rare run-to-run difference at full size; scripts/repro_t1.py)
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
// one TMA box (c0 .. c0+box0-1, k0 .. k0+7, row j) of a 3D tensor map into shared memory; elements
// outside the tensor (the ragged last tile, levels >= nz) are zero-filled and cost no HBM traffic
__device__ __forceinline__ void tma3(void* dst, const CUtensorMap* map, int c0, int k0, int j, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(k0), "r"(j), "r"(smem_u32(b))
        : "memory");
}

// tensor maps of the streamed arrays, [nyl][nz][nx] views with 128 x MA_KS x 1 boxes; (U, D) and
// (E, W, N, S) are viewed as 8-byte elements: [nyl][nz][nx] and [nyl][nz][2 nx]
struct MarchMaps {
    CUtensorMap r, p, v, rh, b2, b4;
};
constexpr uint32_t MA_BOX_V = 128 * MA_KS * 4;       // one fp32 array
constexpr uint32_t MA_BOX_B2 = 2 * MA_BOX_V;
constexpr uint32_t MA_BOX_B4 = 4 * MA_BOX_V;

// TMEM allocation of all 512 columns (one CTA per SM is guaranteed by the shared-memory request)
__device__ __forceinline__ uint32_t tm_alloc512(uint32_t* slot) {
    if ((threadIdx.x >> 5) == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    return *slot;
}

// the same fixed-order CTA sum as block_sum_d (4 warps), over the consumer warps only
template <int NQ>
__device__ __forceinline__ void cons_sum_d(double (&v)[NQ], double* sm, uint32_t r32) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        double a = v[q];
        const bool f = (r32 >> q) & 1u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_down_sync(0xffffffffu, a, o);
            if (f) a = (double)(float)a;
        }
        if (lane == 0) sm[q * 32 + wid] = a;
    }
    cons_bar();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const bool f = (r32 >> q) & 1u;
            double t = sm[q * 32];
            for (int w = 1; w < MA_CONS / 32; ++w) {
                t += sm[q * 32 + w];
                if (f) t = (double)(float)t;
            }
            v[q] = t;
        }
    }
}

// -DMA_TRACE: per-CTA cycle accounting of thread 0 (consumer) and the producer lane (debug builds)
#ifdef MA_TRACE
__device__ unsigned long long g_ma_trace[1024 * 16];
#define MA_CLK(v) const long long v = clock64()
#define MA_ADD(slot, t0) tr[slot] += clock64() - (t0)
#else
#define MA_CLK(v)
#define MA_ADD(slot, t0)
#endif

// -DMA_JITTER (debug builds): pseudo-random delays at the synchronisation points, to expose races
#ifdef MA_JITTER
__device__ __forceinline__ void ma_jitter(uint32_t salt) {
    uint32_t h = (uint32_t)clock() * 2654435761u ^ (salt * 40503u) ^ (blockIdx.x * 2246822519u) ^ threadIdx.x;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13;
    if ((h & 7u) == 0u) __nanosleep(h >> 20 & 2047u);
}
#define MA_J(salt) ma_jitter(salt)
#else
#define MA_J(salt)
#endif


// tcgen05 accesses of one warp role are ordered against the other role's through the mbarriers
// only with these fences (a run-to-run race at full size without them: scripts/stress_march.py)
#ifdef MA_NO_TMEM_FENCE
#define MA_TFENCE_BEFORE()
#define MA_TFENCE_AFTER()
#else
#define MA_TFENCE_BEFORE() asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory")
#define MA_TFENCE_AFTER() asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory")
#endif

struct MarchGeo {
    int strips;                  // latitude strips; grid = strips * tiles CTAs
    int fst_a, sst_a;            // phase A: stages of the elimination / stencil input rings
    int fst_b, sst_b;            // phase B
    int skip_lo, skip_hi;        // latitude bands: local row 0 / nyl-1 has a neighbouring rank, whose
                                 // ghost row arrives during the launch: its stencil is not stored
                                 // here (k_stencil on the edge rows redoes it after the exchange)
};
constexpr int MA_MAX_CH = 9;     // chunks per column (nz <= 72)

// KIND 1: phase A, KIND 2: phase B.  grid strips*tiles, block MA_THREADS: warps 0-3 stencil (S),
// warps 4-7 Thomas (F; warp 4+w shares TMEM lanes, i.e. columns, with S warp w), warps 8 / 10 TMA producers,
// warp 9 publisher.  Dynamic shared memory: the two stage rings + 3*ceil8(nz)*130*4 B z ring + 128 B
// of alignment slack (padded so that only one CTA fits an SM).
//
// Schedule of a strip r_0, r_1, ..., r_{L-1} (r_{-1}, r_L: the neighbouring strips' rows):
//   F: T(r_0), T(r_1), then per step m: elimination(r_{m+2}) chunk by chunk, back substitution
//   S: per step m: [wait z(r_{m+1})] stencil(r_m) chunk by chunk, dot partials
//   (T = forward elimination + back substitution)
// Ring slot x % 3 holds z(r_x); TMEM slot x & 1 holds U, D (and s) of r_x.  The elimination of
// r_{m+2} overwrites, level by level and column by column, exactly the ring entries (z(r_{m-1})) and
// TMEM entries (row r_m) that the stencil of r_m reads in the same chunk: the F warps store a chunk
// only after the S warps have read it (mbarrier sread[chunk], one phase per step).  The S warps
// start step m+1 only when F has finished z(r_{m+2}) (mbarrier zready[x & 1]).
// Levels are padded to a multiple of MA_KB: the TMA zero-fills levels >= nz, which the elimination
// turns into c' = y = z = 0 (m = 1), so every chunk is branch-free; global stores are masked.
// The publisher warp turns "z(r_x) stored" (mbarrier zdone) into the ready flag with a gpu-scope
// release, keeping the fence latency off the compute warps; halo columns of r_{m+1} are fetched
// late in step m, one step before they are needed.
template <int MODE, int KIND>
__global__ void __launch_bounds__(MA_THREADS, 1) k_march(Geo g, Vecs<MODE> vv, MarchGeo mg, int* __restrict__ flags,
                                                            const __grid_constant__ MarchMaps maps) {
    static_assert(sizeof(typename Prec<MODE>::V) == 4, "fp32 working precision only");
    using V = float;
    constexpr int NQ = KIND == 1 ? 1 : 3;
    constexpr int KB = MA_KB;
    constexpr int SF = ma_stage_floats(KIND);
    constexpr int KS = MA_KS;
    constexpr int OFF_P = KS * 128;                          // p after r
    constexpr int OFF_V = (KIND == 1 ? 2 : 1) * KS * 128;   // v after r (, p)
    constexpr int OFF_B2 = (KIND == 1 ? 3 : 2) * KS * 128;  // (U, D) after r, (p,) v
    constexpr int OFF_RH = KS * 512;                         // rhat0 after (E, W, N, S)
    extern __shared__ __align__(128) unsigned char smtma[];
    __shared__ __align__(8) uint64_t fullF[MA_MAX_STAGES], emptyF[MA_MAX_STAGES];
    __shared__ __align__(8) uint64_t fullS[MA_MAX_STAGES], emptyS[MA_MAX_STAGES];
    __shared__ __align__(8) uint64_t sread[MA_MAX_CH], zready[2], zdone[2];
    __shared__ __align__(8) uint64_t hready[2], hfree[2], pubd[2];
    __shared__ float hbuf[2][2][8 * MA_MAX_CH];  // E / W halo columns of rows r_x, slot x & 1
    __shared__ uint32_t tm_slot;
    __shared__ double red[32 * 3];
    DevState* st = vv.st;
    pdl_wait();  // (programmatic dependent launch: the finaliser before has finished)
    if (st->halt != H_RUN) return;  // uniform
    const int epoch = st->epoch;
    const bool fresh = KIND == 1 && st->fresh != 0;
    float beta = 0.f, omega = 0.f, alpha = 0.f;
    if (KIND == 1) {
        beta = fresh ? 0.f : (float)st->beta_v;
        omega = (float)st->omega_v;
    } else {
        alpha = (float)st->alpha_v;
    }
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nx = (int)g.nx, nz = (int)g.nz, nyl = (int)g.nyl;
    const int T = g.tiles;
    const int NSF = KIND == 1 ? mg.fst_a : mg.fst_b, NSS = KIND == 1 ? mg.sst_a : mg.sst_b;
    const int t = blockIdx.x % T, strip = blockIdx.x / T;
    const int ja = (int)((int64_t)strip * nyl / mg.strips), jb = (int)((int64_t)(strip + 1) * nyl / mg.strips);
    const int L = jb - ja;
    const int dir = (strip & 1) ? -1 : 1;
    const int rfirst = dir > 0 ? ja : jb - 1;
    const int i0 = t * 128;
    const int w = min(128, nx - i0);  // columns of this tile (a multiple of 4)
    const int nch = (nz + KB - 1) / KB;
    const int NZ8 = nch * KB;
    // TMA destinations must be 128-byte aligned; the dynamic region follows the static one
    float* stF = reinterpret_cast<float*>(smtma + ((128u - (smem_u32(smtma) & 127u)) & 127u));
    float* stS = stF + (size_t)NSF * SF;
    float* ring = stS + (size_t)NSS * SF;  // [3][NZ8][130]
    const int ring_slot = NZ8 * MA_RING_W;

    if (tid == 0) {
        // consumer-side barriers count every thread of a role (128): each thread releases its own
        // shared / global / TMEM accesses, nothing relies on a warp-level hand-off to lane 0
        for (int s = 0; s < NSF; ++s) { mbar_init(&fullF[s], 1); mbar_init(&emptyF[s], MA_CONS); }
        for (int s = 0; s < NSS; ++s) { mbar_init(&fullS[s], 1); mbar_init(&emptyS[s], MA_CONS); }
        for (int c = 0; c < MA_MAX_CH; ++c) mbar_init(&sread[c], MA_CONS);
        for (int b = 0; b < 2; ++b) { mbar_init(&zready[b], MA_CONS); mbar_init(&zdone[b], MA_CONS); }
        for (int b = 0; b < 2; ++b) { mbar_init(&hready[b], 32); mbar_init(&hfree[b], MA_CONS); mbar_init(&pubd[b], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const uint32_t tbase = tm_alloc512(&tm_slot);  // contains __syncthreads()
    auto row_of = [&](int n) { return rfirst + dir * n; };
#ifdef MA_TRACE
    long long tr[16] = {0};
#endif
    MA_CLK(t_all);

    // ------------------------------------------------------------------ producer warps
    // warp 8 fills the elimination ring, warp 10 the stencil ring: one ring never waits for room in
    // the other (a single producer in a fixed interleave starves one role whenever the other lags)
    if (warp == 8 || warp == 10) {
        if (lane == 0 && L > 0) {
            int fslot = 0, fround = 0, sslot = 0, sround = 0;
            // elimination inputs of row jr, levels k0..k0+7: r, (p, v) or v, (U, D)
            auto fwd_stage = [&](int jr, int k0) {
                MA_CLK(t0);
                if (fround > 0) MA_PROD_WAIT(&emptyF[fslot], (uint32_t)((fround - 1) & 1));
                MA_ADD(9, t0);
                uint64_t* fb = &fullF[fslot];
                MA_J(1);
                mbar_expect_tx(fb, (KIND == 1 ? (fresh ? 1u : 3u) : 2u) * MA_BOX_V + MA_BOX_B2);
                float* sb = stF + (size_t)fslot * SF;
                tma3(sb, &maps.r, i0, k0, jr, fb);
                if (KIND == 1 && !fresh) tma3(sb + OFF_P, &maps.p, i0, k0, jr, fb);
                if (KIND == 2 || !fresh) tma3(sb + OFF_V, &maps.v, i0, k0, jr, fb);
                tma3(sb + OFF_B2, &maps.b2, i0, k0, jr, fb);
                if (++fslot == NSF) { fslot = 0; ++fround; }
            };
            // stencil inputs of row jr: (E, W, N, S), rhat0 (phase A)
            auto sten_stage = [&](int jr, int k0) {
                MA_CLK(t0);
                if (sround > 0) MA_PROD_WAIT(&emptyS[sslot], (uint32_t)((sround - 1) & 1));
                MA_ADD(9, t0);
                uint64_t* fb = &fullS[sslot];
                MA_J(2);
                mbar_expect_tx(fb, MA_BOX_B4 + (KIND == 1 ? MA_BOX_V : 0u));
                float* sb = stS + (size_t)sslot * SF;
                tma3(sb, &maps.b4, 2 * i0, k0, jr, fb);
                if (KIND == 1) tma3(sb + OFF_RH, &maps.rh, i0, k0, jr, fb);
                if (++sslot == NSS) { sslot = 0; ++sround; }
            };
            for (int m = 0; m < L; ++m)
                for (int k0 = 0; k0 < NZ8; k0 += KS) {
                    if (warp == 8) fwd_stage(row_of(m), k0);
                    else sten_stage(row_of(m), k0);
                }
        }
#ifdef MA_TRACE
        if (lane == 0 && warp == 8) {
            MA_ADD(10, t_all);
            for (int q = 9; q < 11; ++q) g_ma_trace[(KIND - 1) * 512 * 16 + blockIdx.x * 16 + q] = tr[q];
        }
#endif
        return;  // the compute warps keep the CTA (and its TMEM) alive until every stage has landed
    }
    // ------------------------------------------------------------------ publisher warp
    if (warp == 9) {
        if (lane == 0)
            for (int x = 0; x < L; ++x) {
                MA_PUB_WAIT(&zdone[x & 1], (uint32_t)((x >> 1) & 1));
                MA_J(3);
                st_release(flags + (int64_t)row_of(x) * T + t, epoch);  // gpu-scope release: z(r_x)
                mbar_arrive(&pubd[x & 1]);
            }
        return;
    }
    // ------------------------------------------------------------------ halo warp
    // E / W halo columns of r_x (the neighbouring tiles' z, after their ready flags) into hbuf[x & 1],
    // well ahead of the stencil of r_x: the stencil warps never wait on another CTA mid-step
    const int tW = (t == 0) ? T - 1 : t - 1, tE = (t + 1 == T) ? 0 : t + 1;
    const int iWg = (i0 == 0) ? nx - 1 : i0 - 1;         // W halo column (tile t-1, periodic)
    const int iEg = (i0 + min(128, nx - i0) == nx) ? 0 : i0 + min(128, nx - i0);  // E halo column
    if (warp == 11) {
        V* __restrict__ Zh = KIND == 1 ? vv.z : vv.zs;
        for (int x = 0; x < L; ++x) {
            if (x >= 2) mbar_wait_sleep(&hfree[x & 1], (uint32_t)(((x - 2) >> 1) & 1), 64);  // copied out
            const int jr = row_of(x);
            if (lane < 2) {
                const int* f = flags + (int64_t)jr * T + (lane == 0 ? tW : tE);
                while (ld_acquire(f) != epoch) __nanosleep(64);
            }
            __syncwarp();
            for (int k = lane; k < nz; k += 32) {
                const V* zg = Zh + (int64_t)jr * g.row + (int64_t)k * nx;
                hbuf[x & 1][0][k] = __ldcg(zg + iWg);
                hbuf[x & 1][1][k] = __ldcg(zg + iEg);
            }
            mbar_arrive(&hready[x & 1]);  // every lane releases its own stores
        }
        return;
    }

    // ------------------------------------------------------------------ compute warps (S and F)
    const bool isF = warp >= 4;
    const int col = tid & 127;
    const bool act = col < w;
    const bool uni = w == 128;  // every lane owns a column (all tiles but a ragged last one)
    const int i = i0 + (act ? col : w - 1);  // inactive lanes compute on zero-filled data, never store
    const uint32_t tl = tbase + ((uint32_t)((warp & 3) * 32) << 16);
    // TMEM column map (per lane = per column): c' | U(2 slots) | D(2 slots) | s(2 slots, phase B)
    auto tU = [&](int slot) { return tl + (uint32_t)(NZ8 + slot * 2 * NZ8); };
    auto tD = [&](int slot) { return tl + (uint32_t)(NZ8 + slot * 2 * NZ8 + NZ8); };
    auto tS = [&](int slot) { return tl + (uint32_t)(5 * NZ8 + slot * NZ8); };
    V* __restrict__ Zw = KIND == 1 ? vv.z : vv.zs;
    auto slot_ptr = [&](int x) { return ring + (size_t)(((x % 3) + 3) % 3) * ring_slot; };

    if (isF) {
        // ============================ Thomas warps ============================
        V* __restrict__ Pw = KIND == 1 ? vv.p : vv.s;
        int cslot = 0;
        uint32_t cphase = 0;
        V cprev = 0.f, yprev = 0.f;
        struct FwdIn { float rr[KB], pp[KB], vq[KB], uu[KB], dd[KB]; };
        // one chunk of the elimination of row r_x: f = update, factors; y -> ring, c'/U/D/s -> TMEM,
        // f -> HBM.  sync_step >= 0: wait until the S warps have read this chunk in step sync_step.
        auto fwd_chunk = [&](int k0, int c, float* zr, V* pw, int us, int sync_step) {
            FwdIn in;
#pragma unroll
            for (int h = 0; h < KB / KS; ++h) {  // the chunk's stages
                MA_CLK(t0);
                mbar_wait(&fullF[cslot], cphase);
                MA_ADD(12, t0);
                MA_J(4);
                const float* sb = stF + (size_t)cslot * SF;
#pragma unroll
                for (int l = 0; l < KS; ++l) {
                    const int e = h * KS + l;
                    in.rr[e] = sb[l * 128 + col];
                    if (KIND == 1) in.pp[e] = fresh ? in.rr[e] : sb[OFF_P + l * 128 + col];
                    in.vq[e] = (KIND == 1 && fresh) ? in.rr[e] : sb[OFF_V + l * 128 + col];
                    const float2 ud = *reinterpret_cast<const float2*>(sb + OFF_B2 + l * 256 + 2 * col);
                    in.uu[e] = ud.x;
                    in.dd[e] = ud.y;
                }
                fence_proxy_async_smem();
                mbar_arrive(&emptyF[cslot]);
                if (++cslot == NSF) { cslot = 0; cphase ^= 1u; }
            }
            float cb[KB], yb[KB], fb[KB];
#pragma unroll
            for (int e = 0; e < KB; ++e) {
                const int k = k0 + e;
                const V f = KIND == 1 ? fmaf(beta, fmaf(-omega, in.vq[e], in.pp[e]), in.rr[e])
                                      : fmaf(-alpha, in.vq[e], in.rr[e]);
                const V inv = rcp_fast<V>(fmaf(-in.dd[e], cprev, 1.f));
                const V cc = k == 0 ? in.uu[e] : in.uu[e] * inv;
                const V y = k == 0 ? f : fmaf(-in.dd[e], yprev, f) * inv;
                cb[e] = cc; yb[e] = y; fb[e] = f;
                cprev = cc;
                yprev = y;
            }
            V* pk = pw + (int64_t)k0 * nx;
            if (uni && k0 + KB <= nz) {  // warp-uniform: a full chunk of a full tile
#pragma unroll
                for (int e = 0; e < KB; ++e) __stcg(pk + e * nx, fb[e]);
            } else {
#pragma unroll
                for (int e = 0; e < KB; ++e)
                    if (act && k0 + e < nz) __stcg(pk + e * nx, fb[e]);
            }
            tm_st8(tl + (uint32_t)k0, cb);
            if (sync_step >= 0) {  // the S warps read U, D, s (TMEM slot us) and z(r_{m-1}) of this chunk
                MA_CLK(t1);
                mbar_wait(&sread[c], (uint32_t)(sync_step & 1));
                MA_TFENCE_AFTER();
                MA_J(5);
                MA_ADD(13, t1);
            }
#pragma unroll
            for (int e = 0; e < KB; ++e) zr[(k0 + e) * MA_RING_W] = yb[e];
            tm_st8(tU(us) + (uint32_t)k0, in.uu);
            tm_st8(tD(us) + (uint32_t)k0, in.dd);
            if (KIND == 2) tm_st8(tS(us) + (uint32_t)k0, fb);
        };
        // back substitution of row r_x (y in ring row zr): z -> ring (in place) and HBM
        auto back_row = [&](float* zr, V* zw, int x) {
            MA_CLK(t0);
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            V zn = 0.f;  // z(NZ8) = 0; padded levels have c' = y = 0
            for (int k0 = NZ8 - KB; k0 >= 0; k0 -= KB) {
                float cb[KB], yb[KB];
                tm_ld8_nw(tl + (uint32_t)k0, cb);
#pragma unroll
                for (int e = 0; e < KB; ++e) yb[e] = zr[(k0 + e) * MA_RING_W];
                tm_wait_ld();
#pragma unroll
                for (int e = KB - 1; e >= 0; --e) {
                    zn = fmaf(-cb[e], zn, yb[e]);
                    yb[e] = zn;
                }
#pragma unroll
                for (int e = 0; e < KB; ++e) zr[(k0 + e) * MA_RING_W] = yb[e];
                V* zk = zw + (int64_t)k0 * nx;
                if (uni && k0 + KB <= nz) {
#pragma unroll
                    for (int e = 0; e < KB; ++e) __stcg(zk + e * nx, yb[e]);
                } else {
#pragma unroll
                    for (int e = 0; e < KB; ++e)
                        if (act && k0 + e < nz) __stcg(zk + e * nx, yb[e]);
                }
            }
            // TMEM writes of this row (U, D, s) are ordered before the S warps' reads by the fence
            MA_TFENCE_BEFORE();
            mbar_arrive(&zready[x & 1]);  // the S warps may read z(r_x) from the ring
            // the publisher may release the ready flag: these arrivals (release, CTA scope) and its
            // wait (acquire) order every thread's z stores before its gpu-scope release of the flag.
            // zdone[x & 1] must not run two phases ahead of the publisher: r_{x-2} published first.
            if (x >= 2) mbar_wait(&pubd[x & 1], (uint32_t)(((x - 2) >> 1) & 1));
            mbar_arrive(&zdone[x & 1]);
            MA_ADD(14, t0);
        };
        auto T_row = [&](int x, int sync_step) {
            const int jr = row_of(x);
            float* zr = slot_ptr(x) + 1 + col;
            V* pw = Pw + (int64_t)jr * g.row + i;
            cprev = yprev = 0.f;
            MA_CLK(t0);
            for (int c = 0; c < nch; ++c) fwd_chunk(c * KB, c, zr, pw, x & 1, sync_step);
            MA_ADD(15, t0);
            back_row(zr, Zw + (int64_t)jr * g.row + i, x);
        };
        T_row(0, -1);
        if (L >= 2) T_row(1, -1);
        for (int m = 0; m + 2 < L; ++m) T_row(m + 2, m);
    } else {
        // ============================ stencil warps ============================
        V* __restrict__ Yw = KIND == 1 ? vv.v : vv.t;
        const int64_t per_q = (int64_t)nyl * T;
        int cslot = 0;
        uint32_t cphase = 0;
        auto wait_flag = [&](int row, int tile) {
            const int* f = flags + (int64_t)row * T + tile;
            while (ld_acquire(f) != epoch) __nanosleep(40);
        };
        // a whole row of z from another strip (rows r_{-1}, r_L) into ring row dst (own column)
        auto load_row = [&](float* dst, int row) {
            const V* src = Zw + (int64_t)row * g.row + i;
            for (int k = 0; k < nz; ++k) dst[k * MA_RING_W] = __ldcg(src + (int64_t)k * nx);
        };
        // E / W halo of r_x from hbuf into its ring slot (threads k = tid < nz), then free hbuf[x & 1]
        auto copy_halo = [&](int x) {
            if (tid < nz) {
                mbar_wait(&hready[x & 1], (uint32_t)((x >> 1) & 1));
                float* zr = slot_ptr(x);
                zr[tid * MA_RING_W] = hbuf[x & 1][0][tid];
                zr[tid * MA_RING_W + w + 1] = hbuf[x & 1][1][tid];
            }
            mbar_arrive(&hfree[x & 1]);
        };
        for (int m = 0; m < L; ++m) {
            const int j = row_of(m);
            const int64_t jg = g.j0 + j;
            const bool hasN = jg < g.ny - 1, hasS = jg > 0;
            // ---- z(r_m), z(r_{m+1}) complete (F warps) ----
            MA_CLK(t_z);
            if (m == 0) mbar_wait(&zready[0], 0u);
            if (m + 1 < L) mbar_wait(&zready[(m + 1) & 1], (uint32_t)(((m + 1) >> 1) & 1));
            MA_TFENCE_AFTER();
            MA_J(6);
            MA_ADD(5, t_z);
            float* zC0 = slot_ptr(m);
            float* zN0 = hasN ? (dir > 0 ? slot_ptr(m + 1) : slot_ptr(m - 1)) : zC0;
            float* zS0 = hasS ? (dir > 0 ? slot_ptr(m - 1) : slot_ptr(m + 1)) : zC0;
            // ---- rows outside the strip (first / last step) and the first halo: synchronous ----
            MA_CLK(t_sync);
            const bool ld_prev = m == 0 && (dir > 0 ? hasS : hasN);       // r_{-1} exists
            const bool ld_next = m == L - 1 && (dir > 0 ? hasN : hasS);   // r_L exists
            if (m == 0 || ld_next) {
                if (tid == 0) {
                    // rows of a neighbouring rank sit in the ghost rows -1 / nyl, exchanged before
                    // the launch: no flag
                    if (ld_prev && j - dir >= 0 && j - dir < nyl) wait_flag(j - dir, t);
                    if (ld_next && j + dir >= 0 && j + dir < nyl) wait_flag(j + dir, t);
                }
                cons_bar();
                if (m == 0) copy_halo(0);
                if (ld_prev) load_row(slot_ptr(m - 1) + 1 + col, j - dir);
                if (ld_next) load_row(slot_ptr(m + 1) + 1 + col, j + dir);
                cons_bar();
            }
            MA_ADD(4, t_sync);
            MA_CLK(t_st);
            const float* zC = zC0 + 1 + col;
            const float* zN = zN0 + 1 + col;
            const float* zS = zS0 + 1 + col;
            V* yw = Yw + (int64_t)j * g.row + i;
            const bool keep = !((j == 0 && mg.skip_lo) || (j == nyl - 1 && mg.skip_hi));  // warp-uniform
            const int us = m & 1;
            double acc[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
            V zprev = 0.f;
            for (int c = 0; c < nch; ++c) {
                const int k0 = c * KB;
                // U, D (, s) of r_m from TMEM, bands / rhat0 from the stage, z from the ring
                float ub[KB], db[KB], sv[KB];
                tm_ld8_nw(tU(us) + (uint32_t)k0, ub);
                tm_ld8_nw(tD(us) + (uint32_t)k0, db);
                if (KIND == 2) tm_ld8_nw(tS(us) + (uint32_t)k0, sv);
                float4 b4[KB];
                float ax[KB], zc[KB + 1], zE[KB], zW[KB], zNv[KB], zSv[KB], av[KB];
                int sl[KB / KS];
#pragma unroll
                for (int h = 0; h < KB / KS; ++h) {  // the chunk's stages
                    MA_CLK(t0);
                    mbar_wait(&fullS[cslot], cphase);
                    MA_ADD(2, t0);
                    MA_J(7);
                    const float* sbS = stS + (size_t)cslot * SF;
#pragma unroll
                    for (int l = 0; l < KS; ++l) {
                        b4[h * KS + l] = *reinterpret_cast<const float4*>(sbS + l * 512 + 4 * col);
                        if (KIND == 1) ax[h * KS + l] = sbS[OFF_RH + l * 128 + col];
                    }
                    sl[h] = cslot;
                    if (++cslot == NSS) { cslot = 0; cphase ^= 1u; }
                }
#pragma unroll
                for (int e = 0; e < KB; ++e) {
                    const int ko = (k0 + e) * MA_RING_W;
                    zc[e] = zC[ko];
                    zE[e] = zC[ko + 1];
                    zW[e] = zC[ko - 1];
                    zNv[e] = zN[ko];
                    zSv[e] = zS[ko];
                }
                zc[KB] = zC[min(k0 + KB, nz - 1) * MA_RING_W];
                tm_wait_ld();
                MA_TFENCE_BEFORE();
                MA_J(8);
                fence_proxy_async_smem();
#pragma unroll
                for (int h = 0; h < KB / KS; ++h) mbar_arrive(&emptyS[sl[h]]);
                mbar_arrive(&sread[c]);  // the F warps may now overwrite this chunk
                if (KIND == 2) {
#pragma unroll
                    for (int e = 0; e < KB; ++e) ax[e] = sv[e];
                }
#pragma unroll
                for (int e = 0; e < KB; ++e) {
                    const int k = k0 + e;
                    const V zp = (k + 1 < nz) ? zc[e + 1] : zc[e];  // multiplied by U = 0 on the top level
                    V a = zc[e];
                    a = fmaf(b4[e].x, zE[e], a);
                    a = fmaf(b4[e].y, zW[e], a);
                    a = fmaf(b4[e].z, zNv[e], a);
                    a = fmaf(b4[e].w, zSv[e], a);
                    a = fmaf(ub[e], zp, a);
                    a = fmaf(db[e], zprev, a);  // zprev = 0 at k = 0 (D = 0 there)
                    zprev = zc[e];
                    av[e] = a;
                    if (act && k < nz) {
                        if (KIND == 1) {
                            acc_dot<MODE>(acc[0], ax[e], a);
                        } else {
                            acc_dot<MODE>(acc[0], a, ax[e]);
                            acc_dot<MODE>(acc[1], a, a);
                            acc_dot<MODE>(acc[2], ax[e], ax[e]);
                        }
                    }
                }
                V* yk = yw + (int64_t)k0 * nx;
                if (!keep) {
                } else if (uni && k0 + KB <= nz) {
#pragma unroll
                    for (int e = 0; e < KB; ++e) __stcg(yk + e * nx, av[e]);
                } else {
#pragma unroll
                    for (int e = 0; e < KB; ++e)
                        if (act && k0 + e < nz) __stcg(yk + e * nx, av[e]);
                }
            }
            MA_ADD(6, t_st);
            MA_CLK(t_red);
            cons_sum_d<NQ>(acc, red, MODE == 2 ? 0x7u : 0x0u);  // contains cons_bar()
            if (tid == 0 && keep) {
#pragma unroll
                for (int q = 0; q < NQ; ++q) vv.slots[q * per_q + (int64_t)j * T + t] = acc[q];
            }
            if (m + 1 < L) {
                MA_CLK(t_h);
                copy_halo(m + 1);
                MA_ADD(1, t_h);
            }
            cons_bar();  // ring halo and `red` are rewritten by the next step
            MA_ADD(8, t_red);
        }
    }
    // ---- all compute warps: release TMEM ----
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    asm volatile("bar.sync 2, 256;" ::: "memory");
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase) : "memory");
    }
#ifdef MA_TRACE
    if (tid == 0) {
        MA_ADD(0, t_all);
        for (int q = 0; q < 9; ++q) g_ma_trace[(KIND - 1) * 512 * 16 + blockIdx.x * 16 + q] = tr[q];
    }
    if (tid == 128) {
        MA_ADD(11, t_all);
        for (int q = 11; q < 16; ++q) g_ma_trace[(KIND - 1) * 512 * 16 + blockIdx.x * 16 + q] = tr[q];
    }
#endif
}

}  // namespace eg
