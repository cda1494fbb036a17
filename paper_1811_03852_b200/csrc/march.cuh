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
// do not depend on its arithmetic, so a producer warp streams them with TMA tensor copies into a
// ring of MA_KB-level stages (mbarrier full / empty pairs) far ahead of the four consumer warps.  The
// arithmetic, its order and the reduction slots are those of k_thomas_tm + k_stencil, so the fused
// schedule is bitwise identical to the 5-kernel one (tests/test_gpu_parity.py).
//
// Strips alternate direction (even: ascending rows, odd: descending), so a strip's first row
// neighbours the adjacent strip's first row and its last row the other neighbour's last row.  A
// CTA only ever waits for Thomas results that never wait themselves on the waiting CTA's later
// work, so with all CTAs co-resident (grid <= #SMs, one CTA per SM) the march cannot deadlock.
// The producer issues one TMA box (128 columns x MA_KB levels) per array per stage.
// Requires: nx % 4 == 0 (16-byte TMA strides), 7 * ceil8(nz) <= 512 TMEM columns, tiles <= #SMs.
#pragma once
#include <cuda.h>  // CUtensorMap (the host encodes the maps through cudaGetDriverEntryPointByVersion)

#include "kernels.cuh"

namespace eg {

constexpr int MA_KB = 8;                               // levels per stage
constexpr int MA_CONS = 128;                           // consumer threads: one column each
constexpr int MA_THREADS = MA_CONS + 64;               // + a producer and a publisher warp
// stage = one MA_KB-level chunk: phase A: r, p, v, (U,D) or (E,W,N,S), rhat0 (640 floats / level);
// phase B: r, v, (U,D) or (E,W,N,S) (512 floats / level)
constexpr int ma_stage_floats(int kind) { return MA_KB * (kind == 1 ? 640 : 512); }
constexpr int ma_stage_bytes(int kind) { return 4 * ma_stage_floats(kind); }
constexpr int MA_MAX_STAGES = 8;
constexpr int MA_RING_W = 130;                         // W halo | 128 columns | E halo

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void cons_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
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

// tensor maps of the streamed arrays, [nyl][nz][nx] views with 128 x MA_KB x 1 boxes; (U, D) and
// (E, W, N, S) are viewed as 8-byte elements: [nyl][nz][nx] and [nyl][nz][2 nx]
struct MarchMaps {
    CUtensorMap r, p, v, rh, b2, b4;
};
constexpr uint32_t MA_BOX_V = 128 * MA_KB * 4;       // one fp32 array
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

struct MarchGeo {
    int strips;            // latitude strips; grid = strips * tiles CTAs
    int stages_a, stages_b;  // pipeline depth of phase A / phase B
};

// KIND 1: phase A, KIND 2: phase B.  grid strips*tiles, block MA_THREADS (4 consumer warps, a TMA
// producer warp, a publisher warp), dynamic shared memory stages*20 KB + 3*ceil8(nz)*130*4 B + 128 B
// of alignment slack (padded so that only one CTA fits an SM).
//
// Consumer schedule of a strip r_0, r_1, ..., r_{L-1} (r_{-1}, r_L: the neighbouring strips' rows):
//   prologue:   T(r_0), T(r_1)                           T = forward elimination + back substitution
//   step m:     for each MA_KB-level chunk: stencil(r_m) chunk, then elimination(r_{m+2}) chunk
//               [the two are independent: the elimination's latency-bound recurrence interleaves
//               with the stencil's streaming arithmetic]; back substitution of r_{m+2}
// Ring slot x % 3 holds z(r_x); TMEM slot x & 1 holds U, D (and s) of r_x.  The elimination of
// r_{m+2} overwrites, level by level and in the same thread, exactly the ring entries (z(r_{m-1}),
// own column) and TMEM entries (row r_m) that the stencil of r_m has just read.
// Levels are padded to a multiple of MA_KB: the TMA zero-fills levels >= nz, which the elimination
// turns into c' = y = z = 0 (m = 1), so every chunk is branch-free; global stores are masked.
// The publisher warp turns "z(r_x) stored" (an mbarrier the consumer warps arrive on) into the
// ready flag with a gpu-scope release, keeping the fence latency off the consumers' path; halo
// columns of r_{m+1} are fetched in the middle of step m, one step before they are needed.
template <int MODE, int KIND>
__global__ void __launch_bounds__(MA_THREADS, 1) k_march(Geo g, Vecs<MODE> vv, MarchGeo mg, int* __restrict__ flags,
                                                            const __grid_constant__ MarchMaps maps) {
    static_assert(sizeof(typename Prec<MODE>::V) == 4, "fp32 working precision only");
    using V = float;
    constexpr int NQ = KIND == 1 ? 1 : 3;
    constexpr int KB = MA_KB;
    extern __shared__ __align__(128) unsigned char smraw[];
    __shared__ __align__(8) uint64_t full[MA_MAX_STAGES], empty[MA_MAX_STAGES], zdone[2];
    __shared__ uint32_t tm_slot;
    __shared__ double red[32 * 3];
    DevState* st = vv.st;
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
    constexpr int SF = ma_stage_floats(KIND);
    constexpr int OFF_B2 = (KIND == 1 ? 3 : 2) * MA_KB * 128;  // (U, D) after r, (p,) v
    const int T = g.tiles, NS = KIND == 1 ? mg.stages_a : mg.stages_b;
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
    float* stages = reinterpret_cast<float*>(smraw + ((128u - (smem_u32(smraw) & 127u)) & 127u));
    float* ring = stages + (size_t)NS * SF;  // [3][NZ8][130]
    const int ring_slot = NZ8 * MA_RING_W;

    if (tid == 0) {
        for (int s = 0; s < NS; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], MA_CONS / 32); }
        mbar_init(&zdone[0], MA_CONS / 32);
        mbar_init(&zdone[1], MA_CONS / 32);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    const uint32_t tbase = tm_alloc512(&tm_slot);  // contains __syncthreads()
    auto row_of = [&](int n) { return rfirst + dir * n; };
#ifdef MA_TRACE
    long long tr[16] = {0};
#endif
    MA_CLK(t_all);

    // ------------------------------------------------------------------ producer warp
    if (warp == MA_CONS / 32) {
        if (lane == 0 && L > 0) {
            int slot = 0, round = 0;  // stage ring position (no runtime divisions in the loop)
            auto acquire = [&](uint32_t bytes) -> float* {
                MA_CLK(t0);
                if (round > 0) mbar_wait_sleep(&empty[slot], (uint32_t)((round - 1) & 1), 32);
                MA_ADD(9, t0);
                mbar_expect_tx(&full[slot], bytes);
                return stages + (size_t)slot * SF;
            };
            auto advance = [&]() {
                if (++slot == NS) { slot = 0; ++round; }
            };
            // elimination inputs of row jr, levels k0..k0+7: r, (p, v) or v, (U, D)
            auto fwd_stage = [&](int jr, int k0) {
                const uint32_t bytes = (KIND == 1 ? (fresh ? 1u : 3u) : 2u) * MA_BOX_V + MA_BOX_B2;
                float* sb = acquire(bytes);
                uint64_t* fb = &full[slot];
                tma3(sb, &maps.r, i0, k0, jr, fb);
                if (KIND == 1 && !fresh) tma3(sb + KB * 128, &maps.p, i0, k0, jr, fb);
                if (KIND == 2 || !fresh) tma3(sb + (KIND == 1 ? 2 : 1) * KB * 128, &maps.v, i0, k0, jr, fb);
                tma3(sb + OFF_B2, &maps.b2, i0, k0, jr, fb);
                advance();
            };
            // stencil inputs of row jr: (E, W, N, S), rhat0 (phase A)
            auto sten_stage = [&](int jr, int k0) {
                float* sb = acquire(MA_BOX_B4 + (KIND == 1 ? MA_BOX_V : 0u));
                uint64_t* fb = &full[slot];
                tma3(sb, &maps.b4, 2 * i0, k0, jr, fb);
                if (KIND == 1) tma3(sb + KB * 512, &maps.rh, i0, k0, jr, fb);
                advance();
            };
            for (int c = 0; c < nch; ++c) fwd_stage(row_of(0), c * KB);
            if (L >= 2)
                for (int c = 0; c < nch; ++c) fwd_stage(row_of(1), c * KB);
            for (int m = 0; m < L; ++m)
                for (int c = 0; c < nch; ++c) {
                    sten_stage(row_of(m), c * KB);
                    if (m + 2 < L) fwd_stage(row_of(m + 2), c * KB);
                }
        }
#ifdef MA_TRACE
        if (lane == 0) {
            MA_ADD(10, t_all);
            for (int q = 9; q < 11; ++q) g_ma_trace[blockIdx.x * 16 + q] = tr[q];
        }
#endif
        return;  // the consumers keep the CTA (and its TMEM) alive until every stage has landed
    }
    // ------------------------------------------------------------------ publisher warp
    if (warp == MA_CONS / 32 + 1) {
        if (lane == 0)
            for (int x = 0; x < L; ++x) {
                mbar_wait_sleep(&zdone[x & 1], (uint32_t)((x >> 1) & 1), 256);
                st_release(flags + (int64_t)row_of(x) * T + t, epoch);  // gpu-scope release: z(r_x)
            }
        return;
    }

    // ------------------------------------------------------------------ consumer warps
    const bool act = tid < w;
    const bool uni = w == 128;  // every consumer lane owns a column (all tiles but a ragged last one)
    const int i = i0 + (act ? tid : w - 1);  // inactive lanes compute on zero-filled data, never store
    const uint32_t tl = tbase + ((uint32_t)(warp * 32) << 16);
    // TMEM column map (per lane = per column): c' | U(2 slots) | D(2 slots) | s(2 slots, phase B)
    auto tU = [&](int slot) { return tl + (uint32_t)(NZ8 + slot * 2 * NZ8); };
    auto tD = [&](int slot) { return tl + (uint32_t)(NZ8 + slot * 2 * NZ8 + NZ8); };
    auto tS = [&](int slot) { return tl + (uint32_t)(5 * NZ8 + slot * NZ8); };
    V* __restrict__ Pw = KIND == 1 ? vv.p : vv.s;
    V* __restrict__ Zw = KIND == 1 ? vv.z : vv.zs;
    V* __restrict__ Yw = KIND == 1 ? vv.v : vv.t;
    const int64_t per_q = (int64_t)nyl * T;
    const int iWg = (i0 == 0) ? nx - 1 : i0 - 1;       // W halo column (tile t-1, periodic)
    const int iEg = (i0 + w == nx) ? 0 : i0 + w;        // E halo column (tile t+1, periodic)
    const int tW = (t == 0) ? T - 1 : t - 1, tE = (t + 1 == T) ? 0 : t + 1;
    auto slot_ptr = [&](int x) { return ring + (size_t)(((x % 3) + 3) % 3) * ring_slot; };
    int cslot = 0;
    uint32_t cphase = 0;  // stage ring position of the consumers
    auto stage_wait = [&](int& taken) -> const float* {
        taken = cslot;
        MA_CLK(t0);
        mbar_wait(&full[cslot], cphase);
        MA_ADD(2, t0);
        const float* sb = stages + (size_t)cslot * SF;
        if (++cslot == NS) { cslot = 0; cphase ^= 1u; }
        return sb;
    };
    auto stage_release = [&](int taken) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[taken]);
    };

    // forward elimination of one chunk of row jr (inputs in stage sb): f = update, Thomas factors;
    // y -> ring (own column), c' / U / D / s -> TMEM slot us, f -> HBM (p or s)
    V cprev = 0.f, yprev = 0.f;
    auto fwd_chunk = [&](const float* sb, int k0, float* zr, V* pw, int us) {
        float rr[KB], pp[KB], vq[KB], uu[KB], dd[KB];
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            rr[e] = sb[e * 128 + tid];
            if (KIND == 1) pp[e] = fresh ? rr[e] : sb[KB * 128 + e * 128 + tid];
            vq[e] = (KIND == 1 && fresh) ? rr[e] : sb[(KIND == 1 ? 2 : 1) * KB * 128 + e * 128 + tid];
            const float2 ud = *reinterpret_cast<const float2*>(sb + OFF_B2 + e * 256 + 2 * tid);
            uu[e] = ud.x;
            dd[e] = ud.y;
        }
        float cb[KB], yb[KB], fb[KB];
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            const int k = k0 + e;
            const V f = KIND == 1 ? fmaf(beta, fmaf(-omega, vq[e], pp[e]), rr[e]) : fmaf(-alpha, vq[e], rr[e]);
            const V inv = rcp_fast<V>(fmaf(-dd[e], cprev, 1.f));
            const V c = k == 0 ? uu[e] : uu[e] * inv;
            const V y = k == 0 ? f : fmaf(-dd[e], yprev, f) * inv;
            cb[e] = c; yb[e] = y; fb[e] = f;
            cprev = c;
            yprev = y;
        }
        V* pk = pw + (int64_t)k0 * nx;
        if (uni && k0 + KB <= nz) {  // warp-uniform: a full chunk of a full tile
#pragma unroll
            for (int e = 0; e < KB; ++e) pk[e * nx] = fb[e];
        } else {
#pragma unroll
            for (int e = 0; e < KB; ++e)
                if (act && k0 + e < nz) pk[e * nx] = fb[e];
        }
#pragma unroll
        for (int e = 0; e < KB; ++e) zr[(k0 + e) * MA_RING_W] = yb[e];
        tm_st8(tl + (uint32_t)k0, cb);
        tm_st8(tU(us) + (uint32_t)k0, uu);
        tm_st8(tD(us) + (uint32_t)k0, dd);
        if (KIND == 2) tm_st8(tS(us) + (uint32_t)k0, fb);
    };
    // back substitution of the row whose y sits in ring row zr: z -> ring (in place) and HBM
    auto back_row = [&](float* zr, V* zw) {
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
                for (int e = 0; e < KB; ++e) zk[e * nx] = yb[e];
            } else {
#pragma unroll
                for (int e = 0; e < KB; ++e)
                    if (act && k0 + e < nz) zk[e * nx] = yb[e];
            }
        }
    };
    auto fwd_row = [&](int x) {  // prologue: elimination of r_x alone, then back substitution
        const int jr = row_of(x);
        float* zr = slot_ptr(x) + 1 + tid;
        V* pw = Pw + (int64_t)jr * g.row + i;
        cprev = yprev = 0.f;
        for (int c = 0; c < nch; ++c) {
            int g0;
            const float* sb = stage_wait(g0);
            fwd_chunk(sb, c * KB, zr, pw, x & 1);
            stage_release(g0);
        }
        back_row(zr, Zw + (int64_t)jr * g.row + i);
        __syncwarp();
        if (lane == 0) mbar_arrive(&zdone[x & 1]);
    };
    // wait for flag(row, tile) == epoch (thread 0), then a consumer barrier
    auto wait_flag = [&](int row, int tile) {
        const int* f = flags + (int64_t)row * T + tile;
        while (ld_acquire(f) != epoch) __nanosleep(40);
    };
    // a whole row of z from another strip (rows r_{-1}, r_L) into ring row dst (own column)
    auto load_row = [&](float* dst, int row) {
        const V* src = Zw + (int64_t)row * g.row + i;
        for (int k = 0; k < nz; ++k) dst[k * MA_RING_W] = __ldcg(src + (int64_t)k * nx);
    };

    MA_CLK(t_pro);
    fwd_row(0);
    if (L >= 2) fwd_row(1);
    MA_ADD(1, t_pro);
    float hw = 0.f, he = 0.f;  // prefetched halo values of r_{m+1} (thread k = tid < nz)
    for (int m = 0; m < L; ++m) {
        const int j = row_of(m);
        const int64_t jg = g.j0 + j;
        const bool hasN = jg < g.ny - 1, hasS = jg > 0;
        float* zC0 = slot_ptr(m);
        // ring rows of j+1 and j-1: r_{m+1} (slot m+1) and r_{m-1} (slot m-1) in marching order
        float* zN0 = hasN ? (dir > 0 ? slot_ptr(m + 1) : slot_ptr(m - 1)) : zC0;
        float* zS0 = hasS ? (dir > 0 ? slot_ptr(m - 1) : slot_ptr(m + 1)) : zC0;
        // ---- rows outside the strip (first / last step) and the first halo: synchronous ----
        MA_CLK(t_sync);
        const bool ld_prev = m == 0 && (dir > 0 ? hasS : hasN);       // r_{-1} exists
        const bool ld_next = m == L - 1 && (dir > 0 ? hasN : hasS);   // r_L exists
        if (m == 0 || ld_next) {
            if (tid == 0) {
                if (m == 0) { wait_flag(j, tW); wait_flag(j, tE); }
                if (ld_prev) wait_flag(j - dir, t);
                if (ld_next) wait_flag(j + dir, t);
            }
            cons_bar();
            if (m == 0 && tid < nz) {
                const V* zg = Zw + (int64_t)j * g.row + (int64_t)tid * nx;
                zC0[tid * MA_RING_W] = __ldcg(zg + iWg);
                zC0[tid * MA_RING_W + w + 1] = __ldcg(zg + iEg);
            }
            if (ld_prev) load_row(slot_ptr(m - 1) + 1 + tid, j - dir);
            if (ld_next) load_row(slot_ptr(m + 1) + 1 + tid, j + dir);
            cons_bar();
        }
        MA_ADD(4, t_sync);
        // ---- combined pass: stencil(r_m) || elimination(r_{m+2}) ----
        MA_CLK(t_comb);
        const bool fw = m + 2 < L;
        const int jf = fw ? row_of(m + 2) : j;
        float* zrF = slot_ptr(m + 2) + 1 + tid;
        V* pwF = Pw + (int64_t)jf * g.row + i;
        const float* zC = zC0 + 1 + tid;
        const float* zN = zN0 + 1 + tid;
        const float* zS = zS0 + 1 + tid;
        V* yw = Yw + (int64_t)j * g.row + i;
        const int us = m & 1;
        double acc[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
        V zprev = 0.f;
        cprev = yprev = 0.f;
        for (int c = 0; c < nch; ++c) {
            const int k0 = c * KB;
            if (c == nch / 2 && m + 1 < L) {  // halo of r_{m+1} (published during step m-1)
                MA_CLK(t_h);
                if (tid == 0) {
                    const int jn = row_of(m + 1);
                    wait_flag(jn, tW);
                    wait_flag(jn, tE);
                    // zdone[x & 1] may run at most one phase ahead of the publisher: it must have
                    // published r_m before the consumers arrive for r_{m+2} on the same barrier
                    if (m + 2 < L) wait_flag(j, t);
                }
                cons_bar();
                if (tid < nz) {
                    const V* zg = Zw + (int64_t)row_of(m + 1) * g.row + (int64_t)tid * nx;
                    hw = __ldcg(zg + iWg);
                    he = __ldcg(zg + iEg);
                }
                MA_ADD(4, t_h);
            }
            // stencil inputs: U, D (, s) of r_m from TMEM, bands / rhat0 from the stage, z from the ring
            float ub[KB], db[KB], sv[KB];
            tm_ld8_nw(tU(us) + (uint32_t)k0, ub);
            tm_ld8_nw(tD(us) + (uint32_t)k0, db);
            if (KIND == 2) tm_ld8_nw(tS(us) + (uint32_t)k0, sv);
            int gS, gF = 0;
            const float* sbS = stage_wait(gS);
            const float* sbF = fw ? stage_wait(gF) : nullptr;
            float4 b4[KB];
            float ax[KB], zc[KB + 1], zE[KB], zW[KB], zNv[KB], zSv[KB], av[KB];
#pragma unroll
            for (int e = 0; e < KB; ++e) {
                const int ko = (k0 + e) * MA_RING_W;
                b4[e] = *reinterpret_cast<const float4*>(sbS + e * 512 + 4 * tid);
                if (KIND == 1) ax[e] = sbS[KB * 512 + e * 128 + tid];
                zc[e] = zC[ko];
                zE[e] = zC[ko + 1];
                zW[e] = zC[ko - 1];
                zNv[e] = zN[ko];
                zSv[e] = zS[ko];
            }
            zc[KB] = zC[min(k0 + KB, nz - 1) * MA_RING_W];
            tm_wait_ld();
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
            if (uni && k0 + KB <= nz) {
#pragma unroll
                for (int e = 0; e < KB; ++e) yk[e * nx] = av[e];
            } else {
#pragma unroll
                for (int e = 0; e < KB; ++e)
                    if (act && k0 + e < nz) yk[e * nx] = av[e];
            }
            if (fw) fwd_chunk(sbF, k0, zrF, pwF, us);
            stage_release(gS);
            if (fw) stage_release(gF);
        }
        MA_ADD(6, t_comb);
        MA_CLK(t_red);
        cons_sum_d<NQ>(acc, red, MODE == 2 ? 0x7u : 0x0u);  // contains cons_bar()
        if (tid == 0) {
#pragma unroll
            for (int q = 0; q < NQ; ++q) vv.slots[q * per_q + (int64_t)j * T + t] = acc[q];
        }
        MA_ADD(8, t_red);
        if (fw) {
            MA_CLK(t_back);
            back_row(zrF, Zw + (int64_t)jf * g.row + i);
            __syncwarp();
            if (lane == 0) mbar_arrive(&zdone[(m + 2) & 1]);
            MA_ADD(3, t_back);
        }
        if (m + 1 < L && tid < nz) {
            float* zn1 = slot_ptr(m + 1);
            zn1[tid * MA_RING_W] = hw;
            zn1[tid * MA_RING_W + w + 1] = he;
        }
        cons_bar();  // ring rows / halo and `red` are rewritten by the next step
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    cons_bar();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase) : "memory");
    }
#ifdef MA_TRACE
    if (tid == 0) {
        MA_ADD(0, t_all);
        for (int q = 0; q < 9; ++q) g_ma_trace[blockIdx.x * 16 + q] = tr[q];
    }
#endif
}

}  // namespace eg
