// sor_tma.cuh — TMA-fed, persistent red-black tri-SOR half-sweep (NEXT-1, Eq. 7), fp32 vectors.
//
// One half-sweep updates the columns (i, j) with (i + j) % 2 == colour:
//   rhs_k = (1 - omega) (T x_old)_k + omega (f_k - (E x_E + W x_W + N x_N + S x_S)_k),  x_col = T^-1 rhs
// (k_sor_half in kernels.cuh has the same arithmetic, operation for operation, so both give bitwise
// the same x).  Every value a half-sweep reads from x has the other colour or is the updated
// column's own old value, so CTAs never depend on one another.
//
// This kernel serves every half-sweep after the first sweep's red half.  x lives COLOUR-SPLIT
// during the sweeps (xs: per row and level, the nx/2 columns of colour 0 then those of colour 1;
// ghosted rows -1 / nyl), like f and the bands, so every array an item touches is contiguous for
// its 128 columns: the own colour's old x (levels k0-1 .. k0+4), the other colour's x in the row
// (E / W neighbours, with a 4-wide box on each side for the tile's edge columns and the periodic
// wrap) and in the rows j-1 / j+1 (N / S), f, (E,W,N,S), (U,D).  An item writes only its own
// colour's 128 values per level (no half-written natural sectors).  The last half-sweep of an
// application (FINAL) writes z in natural order instead: both colours as (red, black) pairs, the
// other colour's values kept in TMEM from the forward pass.
// Work item = (latitude row, 128 columns of one colour), one column per consumer thread; a producer
// warp streams 4-level stages with 3-D TMA boxes.  c', y (and for FINAL the other colour) live in
// TMEM.  Persistent grid (2 CTAs / SM); stage release is ordered before the TMA refill by
// fence.proxy.async (see march.cuh).
#pragma once
#include "march.cuh"

namespace eg {

constexpr int SO_KS = 4;                  // levels per stage
constexpr int SO_CONS = 128;              // consumer threads (columns of one colour per item)
constexpr int SO_THREADS = SO_CONS + 32;  // + the producer warp
constexpr int SO_TILE = 256;              // natural columns per item
// stage layout (floats; every TMA destination 128-byte aligned)
constexpr int SO_XO = 0;                               // own colour [KS+2][128], levels k0-1 ..
constexpr int SO_XT = SO_XO + (SO_KS + 2) * 128;       // other colour, row j [KS][128]
constexpr int SO_XHW = SO_XT + SO_KS * 128;            // other colour, 4 columns W of the tile [KS][4]
constexpr int SO_XHE = SO_XHW + 32;                    // other colour, 4 columns E of the tile [KS][4]
constexpr int SO_XN = SO_XHE + 32;                     // other colour, row j+1 [KS][128]
constexpr int SO_XS = SO_XN + SO_KS * 128;             // other colour, row j-1 [KS][128]
constexpr int SO_F = SO_XS + SO_KS * 128;              // [KS][128]
constexpr int SO_B4 = SO_F + SO_KS * 128;              // [KS][512]
constexpr int SO_B2 = SO_B4 + SO_KS * 512;             // [KS][256]
constexpr int SO_STAGE_FLOATS = SO_B2 + SO_KS * 256;
constexpr int SO_STAGES = 4;
constexpr int SO_MAX_NZ8 = 72;
constexpr uint32_t SO_BOX_XO = (SO_KS + 2) * 128 * 4, SO_BOX_XR = SO_KS * 128 * 4, SO_BOX_XH = SO_KS * 4 * 4;
constexpr uint32_t SO_BOX_F = SO_KS * 128 * 4, SO_BOX_B4 = SO_KS * 512 * 4, SO_BOX_B2 = SO_KS * 256 * 4;

// tensor maps: xs (ghosted, colour-split) with (128, KS+2), (128, KS) and (4, KS) boxes; f split
// (128, KS); (E,W,N,S) split as u64 (256, KS); (U,D) split as u64 (128, KS)
struct SorMaps {
    CUtensorMap xo6, x4, xh, f, b4, b2;
};

// grid: persistent (2 CTAs / SM), block SO_THREADS, dynamic smem SO_STAGES * SO_STAGE_FLOATS * 4 + 128.
// xs: the colour-split ghosted x's row 0 (own colour updated in place unless FINAL); z: the natural
// output's row 0 (written when FINAL).  FIRST: the black half of the first sweep (x_old = 0:
// rhs = omega (f - H x); the red neighbours and f were written by k_sor_first_red).
template <int MODE, bool FIRST>
__global__ void __launch_bounds__(SO_THREADS, 2) k_sor_tma(Geo g, Vecs<MODE> vv, float* __restrict__ xs,
                                                            float* __restrict__ z, int colour, int final_,
                                                            double omega_d, int check_halt,
                                                            const __grid_constant__ SorMaps maps) {
    static_assert(sizeof(typename Prec<MODE>::V) == 4, "fp32 working precision only");
    using V = float;
    extern __shared__ __align__(128) unsigned char smtma[];
    __shared__ __align__(8) uint64_t full[SO_STAGES], empty[SO_STAGES];
    __shared__ uint32_t tm_slot;
    if (check_halt && vv.st->halt != H_RUN) return;  // uniform
    const V om = (V)omega_d, om1 = (V)(1.0 - omega_d);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nx = (int)g.nx, nz = (int)g.nz, nyl = (int)g.nyl;
    const int nh = nx / 2;                          // columns per colour
    const int tiles = (nh + SO_CONS - 1) / SO_CONS;
    const int64_t items = (int64_t)tiles * nyl;
    const int NZ8 = (nz + 7) / 8 * 8;  // levels padded to whole 8-level TMEM chunks
    const int oc = colour ^ 1;          // the other colour
    float* stages = reinterpret_cast<float*>(smtma + ((128u - (smem_u32(smtma) & 127u)) & 127u));
    if (tid == 0) {
        for (int q = 0; q < SO_STAGES; ++q) { mbar_init(&full[q], 1); mbar_init(&empty[q], SO_CONS); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // 256 TMEM columns: c' [0, 72), y [72, 144), the other colour (FINAL) [144, 216)
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(&tm_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tbase = tm_slot;
    const int nstage = NZ8 / SO_KS;  // even

    if (warp == SO_CONS / 32) {  // ------------------------------------------------ producer
        if (lane == 0) {
            int slot = 0, round = 0;
            for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
                const int jl = (int)(it / tiles), t = (int)(it % tiles);
                const int64_t jg = g.j0 + jl;
                const int m0 = t * SO_CONS;
                const int w = min(SO_CONS, nh - m0);
                const int cs = colour * nh + m0, co = oc * nh + m0;  // split columns of the tile
                const int hW = oc * nh + (m0 == 0 ? nh : m0) - 4;      // box ending at the W neighbour
                const int hE = oc * nh + (m0 + w == nh ? 0 : m0 + w);  // box starting at the E neighbour
                const bool hasN = jg < g.ny - 1, hasS = jg > 0;
                for (int q = 0; q < nstage; ++q) {
                    const int k0 = q * SO_KS;
                    if (round > 0) mbar_wait_sleep(&empty[slot], (uint32_t)((round - 1) & 1), 32);
                    uint64_t* fb = &full[slot];
                    const uint32_t bytes = (FIRST ? 0u : SO_BOX_XO) + SO_BOX_XR + 2 * SO_BOX_XH +
                                           (hasN ? SO_BOX_XR : 0u) + (hasS ? SO_BOX_XR : 0u) + SO_BOX_F +
                                           SO_BOX_B4 + SO_BOX_B2;
                    mbar_expect_tx(fb, bytes);
                    float* sb = stages + (size_t)slot * SO_STAGE_FLOATS;
                    // xs maps span the ghosted rows -1 .. nyl: local row r is coordinate r + 1
                    if (!FIRST) tma3(sb + SO_XO, &maps.xo6, cs, k0 - 1, jl + 1, fb);
                    tma3(sb + SO_XT, &maps.x4, co, k0, jl + 1, fb);
                    tma3(sb + SO_XHW, &maps.xh, hW, k0, jl + 1, fb);
                    tma3(sb + SO_XHE, &maps.xh, hE, k0, jl + 1, fb);
                    if (hasN) tma3(sb + SO_XN, &maps.x4, co, k0, jl + 2, fb);
                    if (hasS) tma3(sb + SO_XS, &maps.x4, co, k0, jl, fb);
                    tma3(sb + SO_F, &maps.f, cs, k0, jl, fb);
                    tma3(sb + SO_B4, &maps.b4, 2 * cs, k0, jl, fb);
                    tma3(sb + SO_B2, &maps.b2, cs, k0, jl, fb);
                    if (++slot == SO_STAGES) { slot = 0; ++round; }
                }
            }
        }
    } else {  // ------------------------------------------------------------------ consumers
        const uint32_t tl = tbase + ((uint32_t)(warp * 32) << 16);
        int slot = 0;
        uint32_t phase = 0;
        for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
            const int jl = (int)(it / tiles), t = (int)(it % tiles);
            const int64_t jg = g.j0 + jl;
            const int m0 = t * SO_CONS;
            const int w = min(SO_CONS, nh - m0);
            const bool hasN = jg < g.ny - 1, hasS = jg > 0;
            const int par = (int)((jg + colour) & 1);  // natural column of split m: 2 m + par
            const bool act = tid < w;
            // the other colour's E neighbour is its split column m + par, the W one m + par - 1
            const bool eh = par == 1 && tid + 1 >= w, wh = par == 0 && tid == 0;
            V cprev = 0.f, yprev = 0.f;
            for (int k8 = 0; k8 < NZ8; k8 += 8) {  // two stages = one 8-level TMEM chunk
                float cb[8], yb[8], ob[8];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int k0 = k8 + h * SO_KS;
                    mbar_wait(&full[slot], phase);
                    const float* sb = stages + (size_t)slot * SO_STAGE_FLOATS;
                    float xm[SO_KS], xc[SO_KS], xp[SO_KS], xE[SO_KS], xW[SO_KS], xN[SO_KS], xS[SO_KS], f[SO_KS];
                    float xo[SO_KS];
                    float4 b4[SO_KS];
                    float2 b2[SO_KS];
#pragma unroll
                    for (int l = 0; l < SO_KS; ++l) {
                        if (!FIRST) {
                            const float* xr = sb + SO_XO + (l + 1) * 128;  // own colour, level k0 + l
                            xm[l] = xr[tid - 128];
                            xc[l] = xr[tid];
                            xp[l] = xr[tid + 128];
                        }
                        const float* xt = sb + SO_XT + l * 128;
                        xo[l] = xt[tid];  // the other colour in the same natural pair
                        xE[l] = eh ? sb[SO_XHE + l * 4] : xt[tid + par];
                        xW[l] = wh ? sb[SO_XHW + l * 4 + 3] : xt[tid + par - 1];
                        xN[l] = hasN ? sb[SO_XN + l * 128 + tid] : xE[l];  // poles: the zero N / S band reads x_E
                        xS[l] = hasS ? sb[SO_XS + l * 128 + tid] : xE[l];
                        f[l] = sb[SO_F + l * 128 + tid];
                        b4[l] = *reinterpret_cast<const float4*>(sb + SO_B4 + l * 512 + 4 * tid);
                        b2[l] = *reinterpret_cast<const float2*>(sb + SO_B2 + l * 256 + 2 * tid);
                    }
                    fence_proxy_async_smem();
                    mbar_arrive(&empty[slot]);
                    if (++slot == SO_STAGES) { slot = 0; phase ^= 1u; }
#pragma unroll
                    for (int l = 0; l < SO_KS; ++l) {
                        const int k = k0 + l;
                        V hx = b4[l].x * xE[l];
                        hx = fmaf(b4[l].y, xW[l], hx);
                        hx = fmaf(b4[l].z, xN[l], hx);
                        hx = fmaf(b4[l].w, xS[l], hx);
                        V rhs;
                        if (FIRST) {
                            rhs = om * (f[l] - hx);
                        } else {
                            const V xup = k + 1 < nz ? xp[l] : xc[l];  // U = 0 on the top level
                            V tx = xc[l];
                            tx = fmaf(b2[l].x, xup, tx);
                            tx = fmaf(b2[l].y, xm[l], tx);  // D = 0 (and x(-1) = 0) at k = 0
                            rhs = fmaf(om1, tx, om * (f[l] - hx));
                        }
                        const V u = b2[l].x, d = b2[l].y;
                        V c, y;
                        if (k == 0) {
                            c = u;
                            y = rhs;
                        } else {
                            const V inv = rcp_fast<V>(fmaf(-d, cprev, 1.f));
                            c = u * inv;
                            y = fmaf(-d, yprev, rhs) * inv;
                        }
                        cb[h * SO_KS + l] = c;
                        yb[h * SO_KS + l] = y;
                        ob[h * SO_KS + l] = xo[l];
                        cprev = c;
                        yprev = y;
                    }
                }
                tm_st8(tl + (uint32_t)k8, cb);
                tm_st8(tl + (uint32_t)(SO_MAX_NZ8 + k8), yb);
                if (final_) tm_st8(tl + (uint32_t)(2 * SO_MAX_NZ8 + k8), ob);  // warp-uniform
            }
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            // back substitution from the top (padded levels: c' = y = 0 as in the march kernels)
            V zn = 0.f;
            float* xsw = xs + (int64_t)jl * g.row + colour * nh + m0 + (act ? tid : 0);
            float* zw = z + (int64_t)jl * g.row + 2 * (m0 + (act ? tid : 0));
            for (int k8 = NZ8 - 8; k8 >= 0; k8 -= 8) {
                float cc[8], yy[8], oo[8];
                tm_ld8_nw(tl + (uint32_t)k8, cc);
                tm_ld8_nw(tl + (uint32_t)(SO_MAX_NZ8 + k8), yy);
                if (final_) tm_ld8_nw(tl + (uint32_t)(2 * SO_MAX_NZ8 + k8), oo);
                tm_wait_ld();
#pragma unroll
                for (int e = 7; e >= 0; --e) {
                    const int k = k8 + e;
                    zn = (k == nz - 1) ? yy[e] : fmaf(-cc[e], zn, yy[e]);
                    if (k >= nz) zn = 0.f;
                    if (act && k < nz) {
                        if (final_) {  // natural (2 m, 2 m + 1) = (own, other) or (other, own)
                            const float2 pr = par ? make_float2(oo[e], zn) : make_float2(zn, oo[e]);
                            *reinterpret_cast<float2*>(zw + (int64_t)k * nx) = pr;
                        } else {
                            xsw[(int64_t)k * nx] = zn;
                        }
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tbase) : "memory");
    }
}

// FP64 counterpart of k_sor_tma (same items, colour-split x, FINAL natural write), arithmetic as
// k_sor_half<0, ...> operation for operation (so the FP64 tri-SOR result is bitwise unchanged).
// Doubles double the stage: 4 stages of 4 levels (48 KB each) fill one CTA per SM; (E,W,N,S) of the
// 128 colour columns come as two 256-element boxes; c', y and (FINAL) the other colour live in TMEM
// as pairs of 32-bit words (c' [0, 144), y [144, 288), other [288, 432) of a 512-column allocation).
constexpr int S6_KS = 4;
constexpr int S6_STAGES = 4;
constexpr int S6_THREADS = SO_CONS + 32;
constexpr int S6_XO = 0;                               // own colour [KS+2][128]
constexpr int S6_XT = S6_XO + (S6_KS + 2) * 128;       // other colour, row j [KS][128]
constexpr int S6_XHW = S6_XT + S6_KS * 128;            // [KS][4] (32 reserved: 128-byte aligned)
constexpr int S6_XHE = S6_XHW + 32;
constexpr int S6_XN = S6_XHE + 32;                     // other colour, row j+1 [KS][128]
constexpr int S6_XS = S6_XN + S6_KS * 128;             // other colour, row j-1 [KS][128]
constexpr int S6_F = S6_XS + S6_KS * 128;              // [KS][128]
constexpr int S6_B4L = S6_F + S6_KS * 128;             // [KS][64 columns x 4]
constexpr int S6_B4H = S6_B4L + S6_KS * 256;           // [KS][64 columns x 4]
constexpr int S6_B2 = S6_B4H + S6_KS * 256;            // [KS][128 columns x 2]
constexpr int S6_STAGE_DOUBLES = S6_B2 + S6_KS * 256;
constexpr uint32_t S6_BOX_XO = (S6_KS + 2) * 128 * 8, S6_BOX_XR = S6_KS * 128 * 8, S6_BOX_XH = S6_KS * 4 * 8;
constexpr uint32_t S6_BOX_F = S6_KS * 128 * 8, S6_BOX_B = S6_KS * 256 * 8;
constexpr int S6_SMEM = S6_STAGES * S6_STAGE_DOUBLES * 8 + 128;

// maps: xs (ghosted, colour-split) with (128, KS+2), (128, KS), (4, KS) boxes; f split (128, KS);
// (E,W,N,S) split [nyl][nz][4 nx] with (256, KS) boxes; (U, D) split [nyl][nz][2 nx] with (256, KS)
struct SorMaps64 {
    CUtensorMap xo6, x4, xh, f, b4, b2;
};

__device__ __forceinline__ void split_d(double v, float& lo, float& hi) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    lo = __uint_as_float((uint32_t)b);
    hi = __uint_as_float((uint32_t)(b >> 32));
}
__device__ __forceinline__ double join_d(float lo, float hi) {
    return __longlong_as_double((long long)(((unsigned long long)__float_as_uint(hi) << 32) | __float_as_uint(lo)));
}

// grid: persistent (one CTA / SM), block S6_THREADS, dynamic smem S6_SMEM.  FIRST: the black half of
// the first sweep after k_sor_first_red<0, KIND> (rhs = omega (f - H x); the own column is not read).
template <bool FIRST>
__global__ void __launch_bounds__(S6_THREADS, 1) k_sor_tma64(Geo g, Vecs<0> vv, double* __restrict__ xs,
                                                              double* __restrict__ z, int colour, int final_,
                                                              double omega_d, int check_halt,
                                                              const __grid_constant__ SorMaps64 maps) {
    using V = double;
    extern __shared__ __align__(128) unsigned char smtma[];
    __shared__ __align__(8) uint64_t full[S6_STAGES], empty[S6_STAGES];
    __shared__ uint32_t tm_slot;
    if (check_halt && vv.st->halt != H_RUN) return;  // uniform
    const V om = (V)omega_d, om1 = (V)(1.0 - omega_d);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nx = (int)g.nx, nz = (int)g.nz, nyl = (int)g.nyl;
    const int nh = nx / 2;
    const int tiles = (nh + SO_CONS - 1) / SO_CONS;
    const int64_t items = (int64_t)tiles * nyl;
    const int NZ4 = (nz + S6_KS - 1) / S6_KS * S6_KS;
    const int oc = colour ^ 1;
    V* stages = reinterpret_cast<V*>(smtma + ((128u - (smem_u32(smtma) & 127u)) & 127u));
    if (tid == 0) {
        for (int q = 0; q < S6_STAGES; ++q) { mbar_init(&full[q], 1); mbar_init(&empty[q], SO_CONS); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tm_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tbase = tm_slot;
    const int nstage = NZ4 / S6_KS;

    if (warp == SO_CONS / 32) {  // ------------------------------------------------ producer
        if (lane == 0) {
            int slot = 0, round = 0;
            for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
                const int jl = (int)(it / tiles), t = (int)(it % tiles);
                const int64_t jg = g.j0 + jl;
                const int m0 = t * SO_CONS;
                const int w = min(SO_CONS, nh - m0);
                const int cs = colour * nh + m0, co = oc * nh + m0;
                const int hW = oc * nh + (m0 == 0 ? nh : m0) - 4;
                const int hE = oc * nh + (m0 + w == nh ? 0 : m0 + w);
                const bool hasN = jg < g.ny - 1, hasS = jg > 0;
                for (int q = 0; q < nstage; ++q) {
                    const int k0 = q * S6_KS;
                    if (round > 0) mbar_wait_sleep(&empty[slot], (uint32_t)((round - 1) & 1), 32);
                    uint64_t* fb = &full[slot];
                    const uint32_t bytes = (FIRST ? 0u : S6_BOX_XO) + S6_BOX_XR + 2 * S6_BOX_XH +
                                           (hasN ? S6_BOX_XR : 0u) + (hasS ? S6_BOX_XR : 0u) + S6_BOX_F + 3 * S6_BOX_B;
                    mbar_expect_tx(fb, bytes);
                    V* sb = stages + (size_t)slot * S6_STAGE_DOUBLES;
                    if (!FIRST) tma3(sb + S6_XO, &maps.xo6, cs, k0 - 1, jl + 1, fb);
                    tma3(sb + S6_XT, &maps.x4, co, k0, jl + 1, fb);
                    tma3(sb + S6_XHW, &maps.xh, hW, k0, jl + 1, fb);
                    tma3(sb + S6_XHE, &maps.xh, hE, k0, jl + 1, fb);
                    if (hasN) tma3(sb + S6_XN, &maps.x4, co, k0, jl + 2, fb);
                    if (hasS) tma3(sb + S6_XS, &maps.x4, co, k0, jl, fb);
                    tma3(sb + S6_F, &maps.f, cs, k0, jl, fb);
                    tma3(sb + S6_B4L, &maps.b4, 4 * cs, k0, jl, fb);
                    tma3(sb + S6_B4H, &maps.b4, 4 * cs + 256, k0, jl, fb);
                    tma3(sb + S6_B2, &maps.b2, 2 * cs, k0, jl, fb);
                    if (++slot == S6_STAGES) { slot = 0; ++round; }
                }
            }
        }
    } else {  // ------------------------------------------------------------------ consumers
        const uint32_t tl = tbase + ((uint32_t)(warp * 32) << 16);
        int slot = 0;
        uint32_t phase = 0;
        const int b4off = tid < 64 ? S6_B4L + 4 * tid : S6_B4H + 4 * (tid - 64);  // this column's (E,W,N,S)
        for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
            const int jl = (int)(it / tiles), t = (int)(it % tiles);
            const int64_t jg = g.j0 + jl;
            const int m0 = t * SO_CONS;
            const int w = min(SO_CONS, nh - m0);
            const bool hasN = jg < g.ny - 1, hasS = jg > 0;
            const int par = (int)((jg + colour) & 1);
            const bool act = tid < w;
            const bool eh = par == 1 && tid + 1 >= w, wh = par == 0 && tid == 0;
            V cprev = 0.0, yprev = 0.0;
            for (int q = 0; q < nstage; ++q) {
                const int k0 = q * S6_KS;
                mbar_wait(&full[slot], phase);
                const V* sb = stages + (size_t)slot * S6_STAGE_DOUBLES;
                float cw[2 * S6_KS], yw[2 * S6_KS], ow[2 * S6_KS];
#pragma unroll
                for (int l = 0; l < S6_KS; ++l) {
                    const int k = k0 + l;
                    const V* xt = sb + S6_XT + l * 128;
                    const V xE = eh ? sb[S6_XHE + l * 4] : xt[tid + par];
                    const V xW = wh ? sb[S6_XHW + l * 4 + 3] : xt[tid + par - 1];
                    const V xN = hasN ? sb[S6_XN + l * 128 + tid] : xE;
                    const V xS = hasS ? sb[S6_XS + l * 128 + tid] : xE;
                    const V f = sb[S6_F + l * 128 + tid];
                    const double2 e01 = *reinterpret_cast<const double2*>(sb + b4off + l * 256);
                    const double2 e23 = *reinterpret_cast<const double2*>(sb + b4off + l * 256 + 2);
                    const double2 ud = *reinterpret_cast<const double2*>(sb + S6_B2 + l * 256 + 2 * tid);
                    V hx = e01.x * xE;
                    hx = fma(e01.y, xW, hx);
                    hx = fma(e23.x, xN, hx);
                    hx = fma(e23.y, xS, hx);
                    V rhs;
                    if (FIRST) {
                        rhs = om * (f - hx);
                    } else {
                        const V* xr = sb + S6_XO + (l + 1) * 128;  // own colour, level k
                        const V xm = xr[tid - 128], xc = xr[tid], xp = xr[tid + 128];
                        const V xup = k + 1 < nz ? xp : xc;  // U = 0 on the top level
                        V tx = xc;
                        tx = fma(ud.x, xup, tx);
                        tx = fma(ud.y, xm, tx);  // D = 0 (and x(-1) = 0) at k = 0
                        rhs = fma(om1, tx, om * (f - hx));
                    }
                    V c, y;
                    if (k == 0) {
                        c = ud.x;
                        y = rhs;
                    } else {
                        const V inv = rcp_fast<V>(fma(-ud.y, cprev, (V)1));
                        c = ud.x * inv;
                        y = fma(-ud.y, yprev, rhs) * inv;
                    }
                    if (k >= nz) c = y = 0.0;  // padded levels: z = 0 above the top
                    split_d(c, cw[2 * l], cw[2 * l + 1]);
                    split_d(y, yw[2 * l], yw[2 * l + 1]);
                    split_d(xt[tid], ow[2 * l], ow[2 * l + 1]);  // the other colour of the natural pair
                    cprev = c;
                    yprev = y;
                }
                fence_proxy_async_smem();
                mbar_arrive(&empty[slot]);
                if (++slot == S6_STAGES) { slot = 0; phase ^= 1u; }
                tm_st8(tl + (uint32_t)(2 * k0), cw);
                tm_st8(tl + (uint32_t)(144 + 2 * k0), yw);
                if (final_) tm_st8(tl + (uint32_t)(288 + 2 * k0), ow);  // warp-uniform
            }
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            V zn = 0.0;
            V* xsw = xs + (int64_t)jl * g.row + colour * nh + m0 + (act ? tid : 0);
            V* zw = z + (int64_t)jl * g.row + 2 * (m0 + (act ? tid : 0));
            for (int k0 = NZ4 - S6_KS; k0 >= 0; k0 -= S6_KS) {
                float cc[8], yy[8], oo[8];
                tm_ld8_nw(tl + (uint32_t)(2 * k0), cc);
                tm_ld8_nw(tl + (uint32_t)(144 + 2 * k0), yy);
                if (final_) tm_ld8_nw(tl + (uint32_t)(288 + 2 * k0), oo);
                tm_wait_ld();
#pragma unroll
                for (int e = S6_KS - 1; e >= 0; --e) {
                    const int k = k0 + e;
                    const V yk = join_d(yy[2 * e], yy[2 * e + 1]);
                    zn = (k == nz - 1) ? yk : fma(-join_d(cc[2 * e], cc[2 * e + 1]), zn, yk);
                    if (k >= nz) zn = 0.0;
                    if (act && k < nz) {
                        if (final_) {
                            const V ov = join_d(oo[2 * e], oo[2 * e + 1]);
                            const double2 pr = par ? make_double2(ov, zn) : make_double2(zn, ov);
                            *reinterpret_cast<double2*>(zw + (int64_t)k * nx) = pr;
                        } else {
                            xsw[(int64_t)k * nx] = zn;
                        }
                    }
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase) : "memory");
    }
}

// FP64 Thomas solve of the 5-kernel schedule (a3 / a6 / precondition), TMA-fed: the FP64 analogue of
// the fp32 path's TMEM Thomas, with the same arithmetic as k_thomas_tm64<KIND> operation for
// operation (bitwise the same p / s and z).  Item = (latitude row, 128 natural columns), one column
// per consumer thread; a producer warp streams 4-level stages of r, (p, v) / v / fin and (U, D) with
// 3-D TMA boxes; c' and y live in TMEM as word pairs (c' [0, 144), y [144, 288)); one CTA per SM.
// KIND 0: f = fin;  1: p = r + beta (p - omega v), f = p (r only on a fresh iteration);  2: s = r -
// alpha v, f = s.
constexpr int T6_KS = 4;
constexpr int T6_STAGES = 6;
constexpr int T6_THREADS = SO_CONS + 32;
constexpr int T6_A = 0;                        // r (or fin) [KS][128]
constexpr int T6_P = T6_A + T6_KS * 128;       // p [KS][128]
constexpr int T6_V = T6_P + T6_KS * 128;       // v [KS][128]
constexpr int T6_UD = T6_V + T6_KS * 128;      // (U, D) [KS][256]
constexpr int T6_STAGE_DOUBLES = T6_UD + T6_KS * 256;
constexpr uint32_t T6_BOX_V = T6_KS * 128 * 8, T6_BOX_UD = T6_KS * 256 * 8;
constexpr int T6_SMEM = T6_STAGES * T6_STAGE_DOUBLES * 8 + 128;

// maps: r, p, v, fin natural (128, KS); (U, D) natural [nyl][nz][2 nx] (256, KS)
struct ThomasMaps64 {
    CUtensorMap a, p, v, ud;
};

template <int KIND>
__global__ void __launch_bounds__(T6_THREADS, 1) k_thomas_tma64(Geo g, Vecs<0> vv, double* __restrict__ zout,
                                                                 const __grid_constant__ ThomasMaps64 maps) {
    pdl_enter();  // (EG_PDL: the iteration may launch this kernel programmatically)
    using V = double;
    extern __shared__ __align__(128) unsigned char smtma[];
    __shared__ __align__(8) uint64_t full[T6_STAGES], empty[T6_STAGES];
    __shared__ uint32_t tm_slot;
    V beta = 0, omega = 0, alpha = 0;
    bool fresh = false;
    if (KIND != 0) {
        const DevState* st = vv.st;
        if (st->halt != H_RUN) return;  // uniform
        if (KIND == 1) {
            fresh = st->fresh != 0;
            beta = st->beta_v;
            omega = st->omega_v;
        } else {
            alpha = st->alpha_v;
        }
    }
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nx = (int)g.nx, nz = (int)g.nz, nyl = (int)g.nyl;
    const int tiles = (nx + 127) / 128;
    const int64_t items = (int64_t)tiles * nyl;
    const int NZ4 = (nz + T6_KS - 1) / T6_KS * T6_KS;
    V* stages = reinterpret_cast<V*>(smtma + ((128u - (smem_u32(smtma) & 127u)) & 127u));
    if (tid == 0) {
        for (int q = 0; q < T6_STAGES; ++q) { mbar_init(&full[q], 1); mbar_init(&empty[q], SO_CONS); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tm_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tbase = tm_slot;
    const int nstage = NZ4 / T6_KS;
    const bool rpv = KIND == 1 && !fresh;  // p and v are read

    if (warp == SO_CONS / 32) {  // ------------------------------------------------ producer
        if (lane == 0) {
            int slot = 0, round = 0;
            for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
                const int jl = (int)(it / tiles), t = (int)(it % tiles);
                const int i0 = t * 128;
                for (int q = 0; q < nstage; ++q) {
                    const int k0 = q * T6_KS;
                    if (round > 0) mbar_wait_sleep(&empty[slot], (uint32_t)((round - 1) & 1), 32);
                    uint64_t* fb = &full[slot];
                    const uint32_t bytes = T6_BOX_V * (1u + (rpv ? 2u : 0u) + (KIND == 2 ? 1u : 0u)) + T6_BOX_UD;
                    mbar_expect_tx(fb, bytes);
                    V* sb = stages + (size_t)slot * T6_STAGE_DOUBLES;
                    tma3(sb + T6_A, &maps.a, i0, k0, jl, fb);
                    if (rpv) tma3(sb + T6_P, &maps.p, i0, k0, jl, fb);
                    if (rpv || KIND == 2) tma3(sb + T6_V, &maps.v, i0, k0, jl, fb);
                    tma3(sb + T6_UD, &maps.ud, 2 * i0, k0, jl, fb);
                    if (++slot == T6_STAGES) { slot = 0; ++round; }
                }
            }
        }
    } else {  // ------------------------------------------------------------------ consumers
        const uint32_t tl = tbase + ((uint32_t)(warp * 32) << 16);
        int slot = 0;
        uint32_t phase = 0;
        for (int64_t it = blockIdx.x; it < items; it += gridDim.x) {
            const int jl = (int)(it / tiles), t = (int)(it % tiles);
            const int i = t * 128 + tid;
            const bool act = i < nx;
            const int64_t base = (int64_t)jl * g.row + (act ? i : 0);
            V* __restrict__ Pw = (KIND == 1 ? vv.p : vv.s) + base;
            V cprev = 0.0, yprev = 0.0;
            for (int q = 0; q < nstage; ++q) {
                const int k0 = q * T6_KS;
                mbar_wait(&full[slot], phase);
                const V* sb = stages + (size_t)slot * T6_STAGE_DOUBLES;
                float cw[2 * T6_KS], yw[2 * T6_KS];
                V fv[T6_KS];
#pragma unroll
                for (int l = 0; l < T6_KS; ++l) {
                    const int k = k0 + l;
                    const V a = sb[T6_A + l * 128 + tid];
                    V f;
                    if (KIND == 0) f = a;
                    else if (KIND == 1) f = fresh ? a : fma(beta, fma(-omega, sb[T6_V + l * 128 + tid], sb[T6_P + l * 128 + tid]), a);
                    else f = fma(-alpha, sb[T6_V + l * 128 + tid], a);
                    const double2 ud = *reinterpret_cast<const double2*>(sb + T6_UD + l * 256 + 2 * tid);
                    V c, y;
                    if (k == 0) {
                        c = ud.x;
                        y = f;
                    } else {
                        const V inv = rcp_fast<V>(fma(-ud.y, cprev, (V)1));
                        c = ud.x * inv;
                        y = fma(-ud.y, yprev, f) * inv;
                    }
                    if (k >= nz) c = y = 0.0;  // padded levels: z = 0 above the top
                    fv[l] = f;
                    split_d(c, cw[2 * l], cw[2 * l + 1]);
                    split_d(y, yw[2 * l], yw[2 * l + 1]);
                    cprev = c;
                    yprev = y;
                }
                fence_proxy_async_smem();
                mbar_arrive(&empty[slot]);
                if (++slot == T6_STAGES) { slot = 0; phase ^= 1u; }
                if (KIND != 0) {
#pragma unroll
                    for (int l = 0; l < T6_KS; ++l)
                        if (act && k0 + l < nz) Pw[(int64_t)(k0 + l) * nx] = fv[l];
                }
                tm_st8(tl + (uint32_t)(2 * k0), cw);
                tm_st8(tl + (uint32_t)(144 + 2 * k0), yw);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            V zn = 0.0;
            V* zw = zout + base;
            for (int k0 = NZ4 - T6_KS; k0 >= 0; k0 -= T6_KS) {
                float cc[8], yy[8];
                tm_ld8_nw(tl + (uint32_t)(2 * k0), cc);
                tm_ld8_nw(tl + (uint32_t)(144 + 2 * k0), yy);
                tm_wait_ld();
#pragma unroll
                for (int e = T6_KS - 1; e >= 0; --e) {
                    const int k = k0 + e;
                    const V yk = join_d(yy[2 * e], yy[2 * e + 1]);
                    zn = (k == nz - 1) ? yk : fma(-join_d(cc[2 * e], cc[2 * e + 1]), zn, yk);
                    if (k >= nz) zn = 0.0;
                    if (act && k < nz) zw[(int64_t)k * nx] = zn;
                }
            }
            asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase) : "memory");
    }
}

// The red half of the first sweep (x = 0 before it: rhs = omega f) fused with forming f for BOTH
// colours: thread m owns the natural column pair (2m, 2m+1) of a row, reads r, p, v (or fin) for
// both with 8-byte loads, writes p / s (KIND 1 / 2) for both and f colour-split for both, and solves
// the pair's red column.  The black half then reads f colour-split (k_sor_tma<FIRST>), so r, p, v are
// read once per application instead of once per colour.  Arithmetic as k_sor_half<KIND, true>.
// grid (ceil(nx/2 / 128), nyl), block 128, dynamic smem 2 * nz * 128 * 4.
#ifndef FR_PF
#define FR_PF 16
#endif
template <int MODE, int KIND>
__global__ void __launch_bounds__(128) k_sor_first_red(Geo g, Vecs<MODE> vv, const typename Prec<MODE>::V* __restrict__ fin,
                                                       typename Prec<MODE>::V* __restrict__ x, double omega_d,
                                                       Split<typename Prec<MODE>::V> sp,
                                                       typename Prec<MODE>::V* __restrict__ xsplit) {
    using V = typename Prec<MODE>::V;
    constexpr int KB = 4;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int W = blockDim.x, tid = threadIdx.x;
    V* cps = reinterpret_cast<V*>(smraw);
    V* ys = cps + g.nz * W;
    V beta = 0, omega_b = 0, alpha = 0;
    bool fresh = false;
    if (KIND != 0) {
        const DevState* st = vv.st;
        if (st->halt != H_RUN) return;
        if (KIND == 1) {
            fresh = st->fresh != 0;
            beta = (V)st->beta_v;
            omega_b = (V)st->omega_v;
        } else {
            alpha = (V)st->alpha_v;
        }
    }
    const V om = (V)omega_d;
    const int nx = (int)g.nx, nz = (int)g.nz;
    const int m = blockIdx.x * W + tid;
    if (m >= nx / 2) return;
    const int64_t jl = blockIdx.y, jg = g.j0 + jl;
    const int red = (int)(jg & 1);  // which of the pair (2m, 2m+1) is red: (i + jg) % 2 == 0
    const int64_t rb = jl * g.row;
    const int64_t q0 = rb + 2 * m;  // natural index of the pair
    const V* __restrict__ A0 = (KIND == 0 ? fin : vv.r) + q0;
    const V* __restrict__ Pp = (KIND == 1 && fresh ? vv.r : vv.p) + q0;
    const V* __restrict__ Vv = (KIND == 1 && fresh ? vv.r : vv.v) + q0;
    if (KIND == 1 && fresh) beta = 0;
    V* __restrict__ Fw = (KIND == 1 ? vv.p : vv.s) + q0;
    V* __restrict__ Fr = sp.f + rb + m;                           // colour 0 (red) half of the row
    V* __restrict__ Fb = sp.f + rb + nx / 2 + m;                  // colour 1 (black)
    const V* __restrict__ b2 = sp.b2 + 2 * (rb + m);              // red colour-split (U, D)
    // x of the red column: into the colour-split x (xsplit, the fp32 TMA sweeps), else as whole
    // (red, black) pairs of the natural x, the black one 0 (x = 0 before the first sweep; the black
    // half overwrites it): full 32-byte sectors either way, no read-for-merge of partial ones
    V* __restrict__ Xw = x + q0;
    V* __restrict__ Xs = xsplit ? xsplit + rb + m : nullptr;  // colour 0 (red) half of the row
    auto st_pair = [&](int64_t o, V xr) {
        if (Xs) {
            Xs[o] = xr;
            return;
        }
        VecN<V, 2> pr;
        pr.v[0] = red ? (V)0 : xr;
        pr.v[1] = red ? xr : (V)0;
        stv<2>(Xw + o, pr);
    };
    VecN<V, 2> ca[KB], cp[KB], cv[KB], na[KB], np[KB], nv[KB];
    VecN<V, 2> cu[KB], nu[KB];
#pragma unroll
    for (int e = 0; e < KB; ++e)
#pragma unroll
        for (int c = 0; c < 2; ++c) ca[e].v[c] = cp[e].v[c] = cv[e].v[c] = na[e].v[c] = np[e].v[c] = nv[e].v[c] =
            cu[e].v[c] = nu[e].v[c] = 0.f;
    const bool pf_lane = (tid & (32 / (2 * (int)sizeof(V)) - 1)) == 0;  // one L2 prefetch per 32-byte sector
    auto load = [&](int k0, VecN<V, 2>(&a)[KB], VecN<V, 2>(&p)[KB], VecN<V, 2>(&v)[KB], VecN<V, 2>(&u)[KB]) {
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            const int o = min(k0 + e, nz - 1) * nx;
            if (FR_PF > 0 && pf_lane && k0 + e + FR_PF < nz) {  // FR_PF levels ahead
                const int of = (k0 + e + FR_PF) * nx;
                pf_l2(A0 + of);
                if (KIND == 1) { pf_l2(Pp + of); pf_l2(Vv + of); }
                if (KIND == 2) pf_l2(Vv + of);
                pf_l2(b2 + 2 * of);
            }
            a[e] = ldv<2>(A0 + o);
            if (KIND == 1) { p[e] = ldv<2>(Pp + o); v[e] = ldv<2>(Vv + o); }
            if (KIND == 2) v[e] = ldv<2>(Vv + o);
            u[e] = ldv<2>(b2 + 2 * o);
        }
    };
    load(0, ca, cp, cv, cu);
    V cprev = 0, yprev = 0;
    for (int k0 = 0; k0 < nz; k0 += KB) {
        if (k0 + KB < nz) load(k0 + KB, na, np, nv, nu);
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            const int k = k0 + e;
            if (k < nz) {
                VecN<V, 2> f;
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    if (KIND == 1) f.v[c] = fma(beta, fma(-omega_b, cv[e].v[c], cp[e].v[c]), ca[e].v[c]);
                    else if (KIND == 2) f.v[c] = fma(-alpha, cv[e].v[c], ca[e].v[c]);
                    else f.v[c] = ca[e].v[c];
                }
                if (KIND != 0) stv<2>(Fw + k * nx, f);
                Fr[k * nx] = f.v[red];
                Fb[k * nx] = f.v[red ^ 1];
                const V hx = 0;
                const V rhs = om * (f.v[red] - hx);
                const V u = cu[e].v[0], d = cu[e].v[1];
                V c, y;
                if (k == 0) {
                    c = u;
                    y = rhs;
                } else {
                    const V inv = rcp_fast<V>(fma(-d, cprev, (V)1));
                    c = u * inv;
                    y = fma(-d, yprev, rhs) * inv;
                }
                cps[k * W + tid] = c;
                ys[k * W + tid] = y;
                cprev = c;
                yprev = y;
            }
        }
#pragma unroll
        for (int e = 0; e < KB; ++e) { ca[e] = na[e]; cp[e] = np[e]; cv[e] = nv[e]; cu[e] = nu[e]; }
    }
    V zn = yprev;
    st_pair((int64_t)(nz - 1) * nx, zn);
    for (int k = nz - 2; k >= 0; --k) {
        zn = fma(-cps[k * W + tid], zn, ys[k * W + tid]);
        st_pair((int64_t)k * nx, zn);
    }
}

}  // namespace eg
