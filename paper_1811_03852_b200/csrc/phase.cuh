// phase.cuh — fused "phase" kernels: vector update + Thomas (T^-1) + stencil (Ahat) + dot partials,
// fp32 working precision, one GPU (DESIGN.md §Fused phases).
//
//   phase A (a3 + a4):  p = r + beta (p - omega v);  z = T^-1 p;  v = Ahat z;  partial rhat0 . v
//   phase B (a6 + a7):  s = r - alpha v;  z_s = T^-1 s;  t = Ahat z_s;  partials t.s, t.t, s.s
//
// The unfused schedule writes z to HBM and reads it back (plus U, D a second time) in the stencil
// kernel: 164 B / point / iteration.  Here the stencil runs right behind the Thomas solves, as a
// wavefront over latitude rows, so the z rows (and U, D) it reads were written / read moments ago
// and come from L2: 52 + 44 + 40 (update) = 136 B / point of HBM traffic, the algorithmic minimum
// with the paper's three global sums.
//
// Persistent kernel, 4 CTAs / SM of 128 threads (one longitude column per thread, 128-column tiles
// as in the unfused kernels, so the reduction slots and the finaliser are the same).  Work items
// m = 0 .. (rows+1)*T-1 are taken in increasing order from an atomic counter; item m = (j, t) does
//   1. the Thomas solve of row j+1, tile t (factors in TMEM, y in shared memory), writes p / s and
//      z / z_s, then publishes flag[j+1][t] = epoch (release);
//   2. waits until rows j-1, j, j+1 of tiles t-1, t, t+1 (periodic) are published (acquire), then
//      applies the stencil to row j, tile t, reading z / z_s (and s) through L2 (ld.global.cg: other
//      CTAs wrote them), and writes v / t and the row-tile dot partials.
// A dependency is always on an item whose index is < m + T, so with more than T resident CTAs the
// smallest waiting item can always complete: no deadlock.  p and v are updated in place: the
// Thomas of row j+1 reads p(j+1), v(j+1) and is the only writer of p(j+1); v(j+1) is rewritten
// only by the stencil of row j+1, which waits for flag[j+1][t].
// `epoch` comes from DevState and is bumped by every finaliser (monotonic across solves), so flags
// never need resetting; the work counter is reset by the finaliser that precedes each launch.
#pragma once
#include "kernels.cuh"

namespace eg {

constexpr int WAVE_THREADS = 128;

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int MODE, int KIND>
__global__ void __launch_bounds__(WAVE_THREADS, 4) k_wave(Geo g, Vecs<MODE> vv, int* __restrict__ flags) {
    using V = float;
    static_assert(sizeof(typename Prec<MODE>::V) == 4, "fp32 working precision only");
    constexpr int NQ = KIND == 1 ? 1 : 3;
    constexpr int SKB = 4;
    extern __shared__ __align__(16) unsigned char smraw[];
    __shared__ uint32_t tm_base;
    __shared__ int s_item;
    __shared__ double red[32 * 3];
    DevState* st = vv.st;
    if (st->halt != H_RUN) return;  // uniform: before any collective
    const int epoch = st->epoch;
    float beta = 0.f, omega = 0.f, alpha = 0.f;
    bool fresh = false;
    if (KIND == 1) {
        fresh = st->fresh != 0;
        beta = (float)st->beta_v;
        omega = (float)st->omega_v;
    } else {
        alpha = (float)st->alpha_v;
    }
    const uint32_t base = tm_alloc128(&tm_base);
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t taddr = base + ((uint32_t)(warp * 32) << 16);
    float* ys = reinterpret_cast<float*>(smraw);
    const int nx = (int)g.nx, nz = (int)g.nz, nyl = (int)g.nyl;
    const int T = g.tiles;
    const int total = (nyl + 1) * T;
    V* Zout = KIND == 1 ? vv.z : vv.zs;   // z or z_s
    V* Yout = KIND == 1 ? vv.v : vv.t;    // v or t
    const V* Aux = KIND == 1 ? vv.rh : vv.s;

    for (;;) {
        if (tid == 0) s_item = atomicAdd(&st->wave_ctr, 1);
        __syncthreads();
        const int m = s_item;
        if (m >= total) break;  // uniform
        const int j = m / T - 1, t = m % T;
        const int i_raw = t * 128 + tid;
        const bool act = i_raw < nx;
        const int i = act ? i_raw : nx - 1;
        // ---- 1. Thomas of row j+1 -------------------------------------------------------------
        if (j + 1 < nyl) {
            thomas_tm_tile<MODE, KIND>(g, vv, (int64_t)(j + 1) * g.row, i, act, taddr, ys, beta, omega, alpha,
                                       fresh, nullptr, Zout);
            __threadfence();
            __syncthreads();
            if (tid == 0) st_release(flags + (int64_t)(j + 1) * T + t, epoch);
        }
        // ---- 2. stencil of row j ----------------------------------------------------------------
        if (j >= 0) {
            const int64_t jg = g.j0 + j;
            if (tid == 0) {
                const int r0 = jg > 0 ? j - 1 : j, r1 = jg < g.ny - 1 ? j + 1 : j;
                for (int r = r0; r <= r1; ++r)
                    for (int dt = -1; dt <= 1; ++dt) {
                        const int tt = (t + dt + T) % T;
                        const int* f = flags + (int64_t)r * T + tt;
                        while (ld_acquire(f) != epoch) __nanosleep(64);
                    }
            }
            __syncthreads();
            double acc[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
            if (act) {
                const int64_t rb = (int64_t)j * g.row;
                const int iE = (i + 1 == nx) ? 0 : i + 1, iW = (i == 0) ? nx - 1 : i - 1;
                const V* zc = Zout + rb + i;
                const V* zE = Zout + rb + iE;
                const V* zW = Zout + rb + iW;
                const V* zN = (jg < g.ny - 1) ? zc + g.row : zc;
                const V* zS = (jg > 0) ? zc - g.row : zc;
                const V* __restrict__ b4 = vv.B4 + 4 * (rb + i);
                const V* __restrict__ b2 = vv.B2 + 2 * (rb + i);
                const V* ax = Aux + rb + i;
                V* yo = Yout + rb + i;
                constexpr int NA = 12;
                V cur[SKB][NA], nxt[SKB][NA];
#pragma unroll
                for (int e = 0; e < SKB; ++e)
#pragma unroll
                    for (int a = 0; a < NA; ++a) cur[e][a] = nxt[e][a] = 0.f;
                V zup_c = 0.f, zup_n = 0.f;
                // z / z_s and s were written by other CTAs in this launch: read them through L2
                auto load = [&](int k0, V(&b)[SKB][NA], V& zup) {
#pragma unroll
                    for (int e = 0; e < SKB; ++e) {
                        const int o = min(k0 + e, nz - 1) * nx;
                        const VecN<V, 4> h4 = ldv<4>(b4 + 4 * o);
                        const VecN<V, 2> h2 = ldv<2>(b2 + 2 * o);
                        b[e][0] = h4.v[0]; b[e][1] = h4.v[1]; b[e][2] = h4.v[2];
                        b[e][3] = h4.v[3]; b[e][4] = h2.v[0]; b[e][5] = h2.v[1];
                        b[e][6] = __ldcg(zc + o); b[e][7] = __ldcg(zE + o); b[e][8] = __ldcg(zW + o);
                        b[e][9] = __ldcg(zN + o); b[e][10] = __ldcg(zS + o);
                        b[e][11] = KIND == 1 ? ax[o] : __ldcg(ax + o);
                    }
                    zup = __ldcg(zc + min(k0 + SKB, nz - 1) * nx);
                };
                load(0, cur, zup_c);
                V zprev = 0.f;
                for (int k0 = 0; k0 < nz; k0 += SKB) {
                    if (k0 + SKB < nz) load(k0 + SKB, nxt, zup_n);
#pragma unroll
                    for (int e = 0; e < SKB; ++e) {
                        const int k = k0 + e;
                        if (k < nz) {
                            const V zm = e == 0 ? zprev : cur[e - 1][6];
                            const V zp = e + 1 < SKB ? cur[e + 1][6] : zup_c;  // U = 0 at k = nz-1
                            V a = cur[e][6];
                            a = fmaf(cur[e][0], cur[e][7], a);
                            a = fmaf(cur[e][1], cur[e][8], a);
                            a = fmaf(cur[e][2], cur[e][9], a);
                            a = fmaf(cur[e][3], cur[e][10], a);
                            a = fmaf(cur[e][4], zp, a);
                            a = fmaf(cur[e][5], zm, a);
                            yo[k * nx] = a;
                            if (KIND == 1) {
                                acc_dot<MODE>(acc[0], cur[e][11], a);
                            } else {
                                const V sv = cur[e][11];
                                acc_dot<MODE>(acc[0], a, sv);
                                acc_dot<MODE>(acc[1], a, a);
                                acc_dot<MODE>(acc[2], sv, sv);
                            }
                        }
                    }
                    zprev = cur[SKB - 1][6];
#pragma unroll
                    for (int e = 0; e < SKB; ++e)
#pragma unroll
                        for (int a = 0; a < NA; ++a) cur[e][a] = nxt[e][a];
                    zup_c = zup_n;
                }
            }
            block_sum_d<NQ>(acc, red, MODE == 2 ? 0x7u : 0x0u);  // contains __syncthreads()
            if (tid == 0) {
                const int64_t per_q = (int64_t)nyl * T;
#pragma unroll
                for (int q = 0; q < NQ; ++q) vv.slots[q * per_q + (int64_t)j * T + t] = acc[q];
            }
        }
        __syncthreads();  // s_item is rewritten at the top of the next item
    }
    tm_free128(base);
}

}  // namespace eg
