// kernels.cuh — sm_100a kernels of the BiCGStab hot path.
//
// Unfused 5-kernel iteration schedule:
//   thomas_p  : p = r + beta (p - omega v);  z = T^-1 p            (a3)
//   stencil_A : v = Ahat z;  partial sigma = rhat0 . v             (a4)
//   fin_A     : alpha = rho / sigma                                 (a5)
//   thomas_s  : s = r - alpha v;  z_s = T^-1 s                      (a6)
//   stencil_B : t = Ahat z_s;  partials t.s, t.t, s.s               (a7)
//   fin_B     : omega = t.s / t.t, s-step exit test                 (a8)
//   update    : x += alpha z + omega z_s;  r = s - omega t;
//               partials rhat0 . r, r . r                           (a9)
//   fin_C     : beta, R, history, convergence / breakdown / restart (a10)
// plus scale (a1), start (a2 / a11: bhat, r = round(bhat - Ahat x) in fp64) and the finalisers.
//
// Memory layout: every field is longitude-fastest, q = i + nx*(k + nz*jl); the
// scaled bands are packed per point as B4[q] = (E, W, N, S) and B2[q] = (U, D) so one 16-byte and
// one 8-byte load (fp32) fetch all six.  Column kernels give each thread CPT consecutive columns and
// walk the levels k, prefetching KB levels ahead into registers (double-buffered batches) so that
// every warp keeps many independent loads in flight while it runs the per-column recurrences.
//
// Every reducing kernel writes one partial per (latitude row, 128-column tile) slot; the finaliser
// sums slots in a fixed order inside 8 fixed latitude row-groups, then the groups in order, so sums
// are bitwise reproducible run to run and for any number of GPUs.
#pragma once
#include "common.cuh"

namespace eg {

struct Geo {
    int64_t nx, ny, nz;  // global grid
    int64_t row;         // nx*nz: one latitude row
    int64_t nyl;         // local rows
    int64_t j0;          // global index of local row 0
    int64_t n;           // nyl*row
    int tiles;           // 128-column tiles per row (= reduction slots per row)
    int G, g_lo, g_hi;   // reduction row-groups: all, and this rank's [g_lo, g_hi)
    int quad;            // finalisers: each slot is 4 warp sums ((w0 + w1) + w2) + w3 (the FP64 phase
                         // kernels' 64-column half-slots, march64.cuh)
};

constexpr int RW = 128;  // columns per CTA of the row-tiled kernels (one reduction slot each)

template <int MODE>
struct Vecs {
    using V = typename Prec<MODE>::V;
    using X = typename Prec<MODE>::X;
    const V* B4;                     // [n][4] scaled (E, W, N, S); the unit diagonal is not stored
    const V* B2;                     // [n][2] scaled (U, D)
    const double* diag;              // a_C, fp64 (scales b only)
    double* bhat;                    // D_g^-1 b, fp64
    X* x;                            // iterate
    const X* xg_lo;                  // x ghost row below local row 0 (multi-GPU)
    const X* xg_hi;                  // x ghost row above local row nyl-1
    V *r, *rh, *p, *v, *s, *t;
    V *z, *zs;                       // row 0 of ghosted arrays: rows -1 and nyl exist
    double* slots;                   // [NQ][nyl][tiles]
    DevState* st;
};

// ---- aligned vector access ----
template <class T, int N>
struct alignas(sizeof(T) * N) VecN { T v[N]; };

template <int N, class T>
__device__ __forceinline__ VecN<T, N> ldv(const T* p) { return *reinterpret_cast<const VecN<T, N>*>(p); }
template <int N, class T>
__device__ __forceinline__ void stv(T* p, const VecN<T, N>& a) { *reinterpret_cast<VecN<T, N>*>(p) = a; }

// Programmatic dependent launch: a kernel launched with programmatic stream serialization may
// start while the previous kernel in the stream still runs; it waits here (a no-op otherwise)
// before it reads anything that kernel writes, and lets its own dependents launch early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// first thing of a kernel the iteration may launch programmatically (EG_PDL): wait for the previous
// kernel's completion (a no-op for a normal launch), then let the next one launch and wait likewise
__device__ __forceinline__ void pdl_enter() {
    pdl_wait();
    pdl_launch_dependents();
}

// L2 prefetch of a future level (no register cost): the register batches then see L2 latency
__device__ __forceinline__ void pf_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// L2 prefetch distance (levels) of the shared-memory-factor Thomas kernel (the FP64 path), 0 = off
#ifndef TH_PF
#define TH_PF 16
#endif

// FP32 mode keeps its global sums in binary32: emulate exactly by rounding after every add
template <int MODE> __device__ __forceinline__ double rs(double a) {
    return MODE == 2 ? (double)(float)a : a;
}

// fixed-order CTA sum of NQ doubles; quantities whose bit is set in r32 are summed in binary32
template <int NQ>
__device__ __forceinline__ void block_sum_d(double (&v)[NQ], double* sm, uint32_t r32) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
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
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const bool f = (r32 >> q) & 1u;
            double t = sm[q * 32];
            for (int w = 1; w < nw; ++w) {
                t += sm[q * 32 + w];
                if (f) t = (double)(float)t;
            }
            v[q] = t;
        }
    }
}

template <int NQ>
__device__ __forceinline__ void write_slots(const Geo& g, double* slots, double (&acc)[NQ],
                                            uint32_t r32, int64_t row = -1) {
    __shared__ double sm[32 * NQ];
    block_sum_d<NQ>(acc, sm, r32);
    if (threadIdx.x == 0) {
        const int64_t per_q = g.nyl * g.tiles;
        const int64_t jl = row >= 0 ? row : (int64_t)blockIdx.y;
#pragma unroll
        for (int q = 0; q < NQ; ++q) slots[q * per_q + jl * g.tiles + blockIdx.x] = acc[q];
    }
}

// the local rows a row-tiled launch covers: row = lo + blockIdx.y * step (all rows: {0, 1}; the
// band-edge rows of a latitude band: {0, nyl - 1}; the interior: {1, 1})
struct RowMap {
    int lo, step;
};
constexpr RowMap ALL_ROWS{0, 1};

// product of two V values summed into an S accumulator held as double: the product rounded, then
// the sum rounded (oracle_dot's s = rs(s + rs(a b))) — in binary32 for FP32 mode, binary64 otherwise
// (exact product for fp32 operands).  Written with the _rn intrinsics, which the compiler never
// contracts into an FMA: a contraction (legal for a plain a * b + s) would skip the product's
// rounding in some kernels and not in others, and the kernels that compute the same partials
// (phase kernels, the 5-kernel stencil, the band-edge stencil) must agree bitwise.
template <int MODE, class V>
__device__ __forceinline__ void acc_dot(double& acc, V a, V b) {
    if (MODE == 2) acc = (double)__fadd_rn((float)acc, __fmul_rn((float)a, (float)b));
    else acc = __dadd_rn(acc, __dmul_rn((double)a, (double)b));
}

// ---------------------------------------------------------------------------------------------
// a1: scale bands (Eq. 5): ahat_d = round_V(a_d / a_C) (binary64 IEEE division), packed
// into B4 / B2; diag = a_C.  Validation flags: 2 = a_C zero or non-finite, 1 = non-finite band or a
// nonzero band at an absent neighbour.  grid (ceil(nx/256), nz, nyl), block 256.
struct Bands7 { const double* b[7]; };

template <class V>
__global__ void __launch_bounds__(256) k_scale(Geo g, Bands7 in, V* __restrict__ B4, V* __restrict__ B2,
                                               double* __restrict__ diag, int* __restrict__ err,
                                               V* __restrict__ B4s, V* __restrict__ B2s) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.nx) return;
    const int64_t k = blockIdx.y, jl = blockIdx.z, jg = g.j0 + jl;
    const int64_t q = jl * g.row + k * g.nx + i;
    const double c = in.b[0][q];
    double a[6];
#pragma unroll
    for (int d = 0; d < 6; ++d) a[d] = in.b[d + 1][q];
    int e = 0;
    if (c == 0.0 || !isfinite(c)) e |= 2;
    const bool present[6] = {true, true, jg < g.ny - 1, jg > 0, k < g.nz - 1, k > 0};
    VecN<V, 4> h4;
    VecN<V, 2> h2;
#pragma unroll
    for (int d = 0; d < 6; ++d) {
        if (!isfinite(a[d]) || (!present[d] && a[d] != 0.0)) e |= 1;
        const V v = (V)(a[d] / c);  // IEEE binary64 division, then one rounding to V
        if (d < 4) h4.v[d] = v;
        else h2.v[d - 4] = v;
    }
    stv<4>(B4 + 4 * q, h4);
    stv<2>(B2 + 2 * q, h2);
    if (B4s) {  // the colour-split copies of the red-black tri-SOR sweeps (k_split_bands' layout)
        const int64_t qs = jl * g.row + k * g.nx + ((i + jg) & 1) * (g.nx / 2) + (i >> 1);
        stv<4>(B4s + 4 * qs, h4);
        stv<2>(B2s + 2 * qs, h2);
    }
    diag[q] = c;
    if (e) atomicOr(err, e);
}

// ---------------------------------------------------------------------------------------------
// a2 / a11 (entry, restart, verification):  bhat = b / diag (ENTRY);
//   res = bhat - Ahat x with fp64 accumulation (bands promoted);  r = rhat0 = round_V(res)
// partials: q0 = ||bhat||^2 (ENTRY), q1 = ||res||^2 (fp64, true residual), q2 = r . r (S).
// XZERO: x = 0 (written at ENTRY), res = bhat, no operator application.  WRITE = false: verification
// only (true residual norm, r / rhat0 untouched).  grid (tiles, nyl), RW.
#ifndef ST_KB
#define ST_KB 2
#endif
// L2 prefetch distance (levels) of k_start's operator pass (restart / verification / warm entry):
// (measured slower at 8 / 16 / 32 levels: 0 = off)
#ifndef START_PF
#define START_PF 0
#endif
template <int MODE, bool ENTRY, bool XZERO, bool WRITE = true>
__global__ void __launch_bounds__(RW) k_start(Geo g, Vecs<MODE> vv, const double* __restrict__ b) {
    using V = typename Prec<MODE>::V;
    using X = typename Prec<MODE>::X;
    constexpr int KB = XZERO ? 8 : ST_KB;
    double acc[3] = {0.0, 0.0, 0.0};
    const int i = blockIdx.x * RW + threadIdx.x;
    const int64_t jl = blockIdx.y, jg = g.j0 + jl;
    if (i < g.nx) {
        const int nx = (int)g.nx, nz = (int)g.nz;
        const int64_t rb = jl * g.row;
        const int iE = (i + 1 == nx) ? 0 : i + 1, iW = (i == 0) ? nx - 1 : i - 1;
        const X* __restrict__ xc = vv.x + rb + i;
        const X* __restrict__ xE = vv.x + rb + iE;
        const X* __restrict__ xW = vv.x + rb + iW;
        // N/S neighbour rows: local, ghost (multi-GPU), or the centre row at a pole (zero band)
        const X* __restrict__ xN = (jg == g.ny - 1) ? xc : (jl + 1 < g.nyl ? xc + g.row : vv.xg_hi + i);
        const X* __restrict__ xS = (jg == 0) ? xc : (jl > 0 ? xc - g.row : vv.xg_lo + i);
        const V* __restrict__ b4 = vv.B4 + 4 * (rb + i);
        const V* __restrict__ b2 = vv.B2 + 2 * (rb + i);
        const double* __restrict__ bp = (ENTRY ? b : vv.bhat) + rb + i;
        const double* __restrict__ dp = vv.diag + rb + i;
        double* __restrict__ bh_out = vv.bhat + rb + i;
        X* __restrict__ xo = vv.x + rb + i;
        V* __restrict__ ro = vv.r + rb + i;
        V* __restrict__ rho = vv.rh + rb + i;
        // per level: fp64 values (bhat, diag, x, xE, xW, xN, xS) and the six bands kept in the
        // working precision (promoted when used): fewer registers per buffered level
        constexpr int ND = XZERO ? 2 : 7, NB = XZERO ? 1 : 6;
        double cd[KB][ND], nd[KB][ND];
        V cbd[KB][NB], nbd[KB][NB];
#pragma unroll
        for (int e = 0; e < KB; ++e) {
#pragma unroll
            for (int a = 0; a < ND; ++a) cd[e][a] = nd[e][a] = 0.0;
#pragma unroll
            for (int a = 0; a < NB; ++a) cbd[e][a] = nbd[e][a] = (V)0;
        }
        double xup_c = 0, xup_n = 0;
        auto load = [&](int k0, double(&c)[KB][ND], V(&cb)[KB][NB], double& xup) {
#pragma unroll
            for (int e = 0; e < KB; ++e) {
                const int k = k0 + e;
                if (k < nz) {
                    const int o = k * nx;
                    c[e][0] = bp[o];
                    c[e][1] = ENTRY ? dp[o] : 1.0;
                    if (!XZERO) {
                        const VecN<V, 4> h4 = ldv<4>(b4 + 4 * o);
                        const VecN<V, 2> h2 = ldv<2>(b2 + 2 * o);
                        cb[e][0] = h4.v[0]; cb[e][1] = h4.v[1]; cb[e][2] = h4.v[2]; cb[e][3] = h4.v[3];
                        cb[e][4] = h2.v[0]; cb[e][5] = h2.v[1];
                        c[e][2] = (double)xc[o]; c[e][3] = (double)xE[o]; c[e][4] = (double)xW[o];
                        c[e][5] = (double)xN[o]; c[e][6] = (double)xS[o];
                        if (START_PF > 0 && k + START_PF < nz) {  // warp-uniform
                            const int of = (k + START_PF) * nx;
                            const int l = threadIdx.x & 31;
                            if ((l * (int)sizeof(X)) % 32 == 0) pf_l2(xc + of);
                            if ((l * 8) % 32 == 0) pf_l2(bp + of);
                            if ((l * 4 * (int)sizeof(V)) % 32 == 0) pf_l2(b4 + 4 * of);
                            if ((l * 2 * (int)sizeof(V)) % 32 == 0) pf_l2(b2 + 2 * of);
                        }
                    }
                }
            }
            if (!XZERO) xup = (k0 + KB < nz) ? (double)xc[(k0 + KB) * nx] : 0.0;
        };
        load(0, cd, cbd, xup_c);
        double xprev = 0.0;
        for (int k0 = 0; k0 < nz; k0 += KB) {
            if (k0 + KB < nz) load(k0 + KB, nd, nbd, xup_n);
#pragma unroll
            for (int e = 0; e < KB; ++e) {
                const int k = k0 + e;
                if (k < nz) {
                    const int o = k * nx;
                    double bh = cd[e][0];
                    if (ENTRY) {
                        bh = bh / cd[e][1];
                        bh_out[o] = bh;
                        if (MODE == 2) {
                            const float b32 = (float)bh;
                            acc[0] = (double)__fadd_rn((float)acc[0], __fmul_rn(b32, b32));
                        } else {
                            acc[0] = __dadd_rn(acc[0], __dmul_rn(bh, bh));
                        }
                    }
                    double res;
                    if (XZERO) {
                        res = bh;  // x = 0 is not stored: DevState.xzero (the first update starts from 0)
                    } else {
                        const double xm = e == 0 ? xprev : cd[e - 1][2];
                        const double xp = e + 1 < KB ? (k + 1 < nz ? cd[e + 1][2] : 0.0) : xup_c;
                        double ax = cd[e][2];
                        ax += (double)cbd[e][0] * cd[e][3];
                        ax += (double)cbd[e][1] * cd[e][4];
                        ax += (double)cbd[e][2] * cd[e][5];
                        ax += (double)cbd[e][3] * cd[e][6];
                        ax += (double)cbd[e][4] * xp;
                        ax += (double)cbd[e][5] * xm;
                        res = bh - ax;
                    }
                    acc[1] += res * res;
                    if (WRITE) {
                        const V rv = (V)res;
                        ro[o] = rv;
                        rho[o] = rv;
                        acc_dot<MODE>(acc[2], rv, rv);
                    }
                }
            }
            if (!XZERO) xprev = cd[KB - 1][2];
#pragma unroll
            for (int e = 0; e < KB; ++e) {
#pragma unroll
                for (int a = 0; a < ND; ++a) cd[e][a] = nd[e][a];
#pragma unroll
                for (int a = 0; a < NB; ++a) cbd[e][a] = nbd[e][a];
            }
            xup_c = xup_n;
        }
    }
    write_slots<3>(g, vv.slots, acc, MODE == 2 ? 0x5u : 0x0u);
}

// ---------------------------------------------------------------------------------------------
// a11 verification (the true residual norm of the current x, nothing written), two columns per
// thread (nx even): k_start<MODE, false, false, false>'s per-point arithmetic (res = bhat - Ahat x
// with fp64 accumulation, the same operation order per point) with 16-byte loads of x, bhat and the
// (U, D) pairs and 32 bytes of (E, W, N, S) per level, half the load instructions per byte.  Each
// thread sums its two columns level by level (a fixed order; the sum differs from the one-column
// kernel's only in rounding).  grid (tiles, nyl), RW / 2 threads.
template <int MODE>
__global__ void __launch_bounds__(RW / 2) k_verify2(Geo g, Vecs<MODE> vv) {
    using V = typename Prec<MODE>::V;
    using X = typename Prec<MODE>::X;
    constexpr int KB = 2;
    double acc[3] = {0.0, 0.0, 0.0};
    const int i = blockIdx.x * RW + 2 * threadIdx.x;
    const int64_t jl = blockIdx.y, jg = g.j0 + jl;
    if (i < g.nx) {
        const int nx = (int)g.nx, nz = (int)g.nz;
        const int64_t rb = jl * g.row;
        const int iE = (i + 2 == nx) ? 0 : i + 2, iW = (i == 0) ? nx - 1 : i - 1;
        const X* __restrict__ xc = vv.x + rb + i;
        const X* __restrict__ xE = vv.x + rb + iE;
        const X* __restrict__ xW = vv.x + rb + iW;
        const X* __restrict__ xN = (jg == g.ny - 1) ? xc : (jl + 1 < g.nyl ? xc + g.row : vv.xg_hi + i);
        const X* __restrict__ xS = (jg == 0) ? xc : (jl > 0 ? xc - g.row : vv.xg_lo + i);
        const V* __restrict__ b4 = vv.B4 + 4 * (rb + i);
        const V* __restrict__ b2 = vv.B2 + 2 * (rb + i);
        const double* __restrict__ bp = vv.bhat + rb + i;
        // per level: bhat[2], x[2], xE, xW, xN[2], xS[2] (fp64) and 2 x 6 bands (working precision)
        double cd[KB][10], nd[KB][10];
        V cb[KB][12], nb[KB][12];
#pragma unroll
        for (int e = 0; e < KB; ++e) {
#pragma unroll
            for (int a = 0; a < 10; ++a) cd[e][a] = nd[e][a] = 0.0;
#pragma unroll
            for (int a = 0; a < 12; ++a) cb[e][a] = nb[e][a] = (V)0;
        }
        double xup_c[2] = {0.0, 0.0}, xup_n[2] = {0.0, 0.0};
        auto load = [&](int k0, double (&c)[KB][10], V (&bb)[KB][12], double (&xup)[2]) {
#pragma unroll
            for (int e = 0; e < KB; ++e) {
                const int k = k0 + e;
                if (k < nz) {
                    const int o = k * nx;
                    const VecN<double, 2> bh = ldv<2>(bp + o);
                    const VecN<X, 2> x2 = ldv<2>(xc + o);
                    const VecN<X, 2> n2 = ldv<2>(xN + o);
                    const VecN<X, 2> s2 = ldv<2>(xS + o);
                    const VecN<V, 4> h0 = ldv<4>(b4 + 4 * o), h1 = ldv<4>(b4 + 4 * o + 4);
                    const VecN<V, 4> u2 = ldv<4>(b2 + 2 * o);
                    c[e][0] = bh.v[0]; c[e][1] = bh.v[1];
                    c[e][2] = (double)x2.v[0]; c[e][3] = (double)x2.v[1];
                    c[e][4] = (double)xE[o]; c[e][5] = (double)xW[o];
                    c[e][6] = (double)n2.v[0]; c[e][7] = (double)n2.v[1];
                    c[e][8] = (double)s2.v[0]; c[e][9] = (double)s2.v[1];
#pragma unroll
                    for (int a = 0; a < 4; ++a) { bb[e][a] = h0.v[a]; bb[e][6 + a] = h1.v[a]; }
                    bb[e][4] = u2.v[0]; bb[e][5] = u2.v[1]; bb[e][10] = u2.v[2]; bb[e][11] = u2.v[3];
                }
            }
            if (k0 + KB < nz) {
                const VecN<X, 2> up = ldv<2>(xc + (k0 + KB) * nx);
                xup[0] = (double)up.v[0];
                xup[1] = (double)up.v[1];
            } else {
                xup[0] = xup[1] = 0.0;
            }
        };
        load(0, cd, cb, xup_c);
        double xprev[2] = {0.0, 0.0};
        for (int k0 = 0; k0 < nz; k0 += KB) {
            if (k0 + KB < nz) load(k0 + KB, nd, nb, xup_n);
#pragma unroll
            for (int e = 0; e < KB; ++e) {
                const int k = k0 + e;
                if (k < nz) {
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const double xm = e == 0 ? xprev[c] : cd[e - 1][2 + c];
                        const double xp = e + 1 < KB ? (k + 1 < nz ? cd[e + 1][2 + c] : 0.0) : xup_c[c];
                        const double xe = c == 0 ? cd[e][3] : cd[e][4];   // column i+1 / i+2
                        const double xw = c == 0 ? cd[e][5] : cd[e][2];   // column i-1 / i
                        const V* bb = cb[e] + 6 * c;
                        double ax = cd[e][2 + c];
                        ax += (double)bb[0] * xe;
                        ax += (double)bb[1] * xw;
                        ax += (double)bb[2] * cd[e][6 + c];
                        ax += (double)bb[3] * cd[e][8 + c];
                        ax += (double)bb[4] * xp;
                        ax += (double)bb[5] * xm;
                        const double res = cd[e][c] - ax;
                        acc[1] += res * res;
                    }
                }
            }
            xprev[0] = cd[KB - 1][2];
            xprev[1] = cd[KB - 1][3];
#pragma unroll
            for (int e = 0; e < KB; ++e) {
#pragma unroll
                for (int a = 0; a < 10; ++a) cd[e][a] = nd[e][a];
#pragma unroll
                for (int a = 0; a < 12; ++a) cb[e][a] = nb[e][a];
            }
            xup_c[0] = xup_n[0];
            xup_c[1] = xup_n[1];
        }
    }
    write_slots<3>(g, vv.slots, acc, MODE == 2 ? 0x5u : 0x0u);
}

// ---------------------------------------------------------------------------------------------
// a3 / a6 / precondition: per-column Thomas solve fused with the vector update that
// produces its right-hand side.  KIND 0: f = fin;  1: p = r + beta (p - omega v), f = p;
// 2: s = r - alpha v, f = s.  Each thread owns CPT consecutive columns (independent recurrences,
// vector loads); the forward-elimination factors c'_k, y_k live in shared memory laid out
// [k][column] (conflict-free).  grid (ceil(nx/W), nyl), W = blockDim*CPT columns,
// dynamic smem 2*nz*W*sizeof(V).
//   c'_0 = U_0, y_0 = f_0;  k >= 1: m = 1 - D_k c'_{k-1}, c'_k = U_k / m, y_k = (f_k - D_k y_{k-1}) / m
//   z_{nz-1} = y_{nz-1};    z_k = y_k - c'_k z_{k+1}
template <int MODE, int KIND, int CPT>
__global__ void __launch_bounds__(128) k_thomas(Geo g, Vecs<MODE> vv,
                                                const typename Prec<MODE>::V* __restrict__ fin,
                                                typename Prec<MODE>::V* __restrict__ zout) {
    pdl_enter();  // (EG_PDL: the iteration may launch this kernel programmatically)
    using V = typename Prec<MODE>::V;
    // levels per batch; the next batch is in flight while the current one is eliminated.  Occupancy
    // is bounded by the shared-memory factors (3 CTAs / SM), not registers, so batches are deep.
    constexpr int KB = (sizeof(V) == 4 ? 16 : 8) / CPT;
    using VC = VecN<V, CPT>;
    using VU = VecN<V, 2 * CPT>;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int W = blockDim.x * CPT, tid = threadIdx.x;
    V* cps = reinterpret_cast<V*>(smraw);
    V* ys = cps + g.nz * W;
    V beta = 0, omega = 0, alpha = 0;
    bool fresh = false;
    if (KIND != 0) {
        const DevState* st = vv.st;
        if (st->halt != H_RUN) return;
        if (KIND == 1) {
            fresh = st->fresh != 0;
            beta = (V)st->beta_v;
            omega = (V)st->omega_v;
        } else {
            alpha = (V)st->alpha_v;
        }
    }
    const int i = blockIdx.x * W + tid * CPT;
    if (i >= g.nx) return;
    const int64_t base = (int64_t)blockIdx.y * g.row + i;
    const int nx = (int)g.nx;
    const int nz = (int)g.nz;
    const V* __restrict__ A0 = (KIND == 0 ? fin : vv.r) + base;
    const V* __restrict__ Pp = vv.p + base;
    const V* __restrict__ Vv = vv.v + base;
    const V* __restrict__ UD = vv.B2 + 2 * base;
    V* __restrict__ Pw = (KIND == 1 ? vv.p : vv.s) + base;
    V* __restrict__ Zw = zout + base;
    const int sc = tid * CPT;  // this thread's first column in the shared-memory rows
    VC ca[KB], cp[KB], cv[KB], na[KB], np[KB], nv[KB];
    VU cu[KB], nu[KB];
#pragma unroll
    for (int e = 0; e < KB; ++e)
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            ca[e].v[c] = cp[e].v[c] = cv[e].v[c] = na[e].v[c] = np[e].v[c] = nv[e].v[c] = (V)0;
            cu[e].v[2 * c] = cu[e].v[2 * c + 1] = nu[e].v[2 * c] = nu[e].v[2 * c + 1] = (V)0;
        }
    auto load = [&](int k0, VC(&a)[KB], VC(&p)[KB], VC(&v)[KB], VU(&u)[KB]) {
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            const int k = k0 + e;
            if (k < nz) {
                const int o = k * nx;
                a[e] = ldv<CPT>(A0 + o);
                if (KIND == 1 && !fresh) { p[e] = ldv<CPT>(Pp + o); v[e] = ldv<CPT>(Vv + o); }
                if (KIND == 2) v[e] = ldv<CPT>(Vv + o);
                u[e] = ldv<2 * CPT>(UD + 2 * o);
            }
            if (TH_PF > 0 && k + TH_PF < nz) {  // warp-uniform: L2 prefetch TH_PF levels ahead
                const int of = (k + TH_PF) * nx;
                const int l = threadIdx.x & 31;
                if ((l * CPT * (int)sizeof(V)) % 32 == 0) {  // one per 32-byte sector
                    pf_l2(A0 + of);
                    if (KIND == 1) { pf_l2(Pp + of); pf_l2(Vv + of); }
                    if (KIND == 2) pf_l2(Vv + of);
                }
                if ((l * 2 * CPT * (int)sizeof(V)) % 32 == 0) pf_l2(UD + 2 * of);
            }
        }
    };
    load(0, ca, cp, cv, cu);
    V cprev[CPT], yprev[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) cprev[c] = yprev[c] = (V)0;
    for (int k0 = 0; k0 < nz; k0 += KB) {
        if (k0 + KB < nz) load(k0 + KB, na, np, nv, nu);
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            const int k = k0 + e;
            if (k < nz) {
                VC f, cc, yy;
#pragma unroll
                for (int c = 0; c < CPT; ++c) {
                    if (KIND == 0) f.v[c] = ca[e].v[c];
                    else if (KIND == 1) f.v[c] = fresh ? ca[e].v[c] : fma(beta, fma(-omega, cv[e].v[c], cp[e].v[c]), ca[e].v[c]);
                    else f.v[c] = fma(-alpha, cv[e].v[c], ca[e].v[c]);
                    const V u = cu[e].v[2 * c], d = cu[e].v[2 * c + 1];
                    if (k == 0) {
                        cc.v[c] = u;
                        yy.v[c] = f.v[c];
                    } else {
                        const V inv = rcp_fast<V>(fma(-d, cprev[c], (V)1));
                        cc.v[c] = u * inv;
                        yy.v[c] = fma(-d, yprev[c], f.v[c]) * inv;
                    }
                    cprev[c] = cc.v[c];
                    yprev[c] = yy.v[c];
                }
                if (KIND != 0) stv<CPT>(Pw + k * nx, f);
                stv<CPT>(cps + k * W + sc, cc);
                stv<CPT>(ys + k * W + sc, yy);
            }
        }
#pragma unroll
        for (int e = 0; e < KB; ++e) { ca[e] = na[e]; cp[e] = np[e]; cv[e] = nv[e]; cu[e] = nu[e]; }
    }
    VC zn;
#pragma unroll
    for (int c = 0; c < CPT; ++c) zn.v[c] = yprev[c];
    stv<CPT>(Zw + (nz - 1) * nx, zn);
#pragma unroll 4
    for (int k = nz - 2; k >= 0; --k) {
        const VC cc = ldv<CPT>(cps + k * W + sc), yy = ldv<CPT>(ys + k * W + sc);
#pragma unroll
        for (int c = 0; c < CPT; ++c) zn.v[c] = fma(-cc.v[c], zn.v[c], yy.v[c]);
        stv<CPT>(Zw + k * nx, zn);
    }
}

// ---------------------------------------------------------------------------------------------
// Same Thomas solve (fp32 working precision), with the elimination factors c'_k kept in TENSOR
// MEMORY instead of shared memory.  TMEM (256 KB / SM) is otherwise idle in this memory-bound
// solver: each thread owns one TMEM lane (warp w -> lanes 32w..32w+31) and stores / reloads its
// column's c'_k eight levels at a time (tcgen05.st / tcgen05.ld .32x32b.x8); y_k stays in shared
// memory ([k][column], conflict-free).  Per 128-column CTA: 128 TMEM columns + nz*512 B of shared
// memory, so 4 CTAs (16 warps) fit on an SM instead of 3 (12 warps at 2 columns / thread with
// both factors in shared memory, i.e. 6 warps): twice the loads in flight.  Dynamic shared memory
// is padded to 50 KB (+1 KB reserved per CTA) so that at most 4 CTAs (= 4 x 128 = all 512 TMEM columns) are ever resident
// on an SM and tcgen05.alloc never waits.  Requires nz <= 128.  grid (ceil(nx/128), nyl), 128 thr.
constexpr int TM_SMEM = 50 * 1024;
// L2 prefetch distances in levels (0 = off) of the Thomas, stencil and update kernels
#ifndef TM_PF
#define TM_PF 16
#endif
#ifndef ST_PF
#define ST_PF 0
#endif
#ifndef UP_PF
#define UP_PF 0
#endif

__device__ __forceinline__ void tm_st8(uint32_t taddr, const float (&c)[8]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
        "r"(__float_as_uint(c[0])), "r"(__float_as_uint(c[1])), "r"(__float_as_uint(c[2])),
        "r"(__float_as_uint(c[3])), "r"(__float_as_uint(c[4])), "r"(__float_as_uint(c[5])),
        "r"(__float_as_uint(c[6])), "r"(__float_as_uint(c[7]))
        : "memory");
}

__device__ __forceinline__ void tm_ld8(uint32_t taddr, float (&c)[8]) {
    uint32_t r[8];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int e = 0; e < 8; ++e) c[e] = __uint_as_float(r[e]);
}

// TMEM allocation of 128 columns by warp 0 (with the fence / barrier / fence hand-off) and release
__device__ __forceinline__ uint32_t tm_alloc128(uint32_t* slot) {
    if ((threadIdx.x >> 5) == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    return *slot;
}

__device__ __forceinline__ void tm_free128(uint32_t base) {
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(base) : "memory");
    }
}

// One 128-column tile of one latitude row: f = update(inputs), z = T^-1 f, with c'_k in this
// thread's TMEM lane and y_k in shared memory ys[k][128].  All 128 threads of the CTA call it
// (warp-collective TMEM access); `act` masks columns beyond nx.  KIND as in k_thomas.
template <int MODE, int KIND, bool WRITE_F = true>
__device__ __forceinline__ void thomas_tm_tile(const Geo& g, const Vecs<MODE>& vv, int64_t row_base, int i,
                                               bool act, uint32_t taddr, float* ys, float beta, float omega,
                                               float alpha, bool fresh, const float* __restrict__ fin,
                                               float* __restrict__ zout) {
    using V = float;
    constexpr int KB = 8;
    const int tid = threadIdx.x;
    const int nx = (int)g.nx, nz = (int)g.nz;
    const int64_t base = row_base + i;
    const V* __restrict__ A0 = (KIND == 0 ? fin : vv.r) + base;
    // p = v = 0 after a (re)start: read r in their place with beta = 0, so the update is exactly
    // f = r + 0*(r - omega r) = r without a data-dependent branch
    const V* __restrict__ Pp = (KIND == 1 && fresh ? vv.r : vv.p) + base;
    const V* __restrict__ Vv = (KIND == 1 && fresh ? vv.r : vv.v) + base;
    if (KIND == 1 && fresh) beta = 0.f;
    const V* __restrict__ UD = vv.B2 + 2 * base;
    V* __restrict__ Pw = (KIND == 1 ? vv.p : vv.s) + base;
    V* __restrict__ Zw = zout + base;
    V ca[KB], cp[KB], cv[KB], na[KB], np[KB], nv[KB];
    VecN<V, 2> cu[KB], nu[KB];
#pragma unroll
    for (int e = 0; e < KB; ++e) {
        ca[e] = cp[e] = cv[e] = na[e] = np[e] = nv[e] = 0.f;
        cu[e].v[0] = cu[e].v[1] = nu[e].v[0] = nu[e].v[1] = 0.f;
    }
    auto load = [&](int k0, V(&a)[KB], V(&p)[KB], V(&v)[KB], VecN<V, 2>(&u)[KB]) {
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            const int o = min(k0 + e, nz - 1) * nx;  // tail levels re-read the last one (L1 hit)
            a[e] = A0[o];
            if (KIND == 1) { p[e] = Pp[o]; v[e] = Vv[o]; }
            if (KIND == 2) v[e] = Vv[o];
            u[e] = ldv<2>(UD + 2 * o);
            if (TM_PF > 0 && k0 + e + TM_PF < nz) {  // warp-uniform condition
                const int of = (k0 + e + TM_PF) * nx;
                if ((tid & 7) == 0) {  // one prefetch per 32-byte sector of each array
                    pf_l2(A0 + of);
                    if (KIND == 1) { pf_l2(Pp + of); pf_l2(Vv + of); }
                    if (KIND == 2) pf_l2(Vv + of);
                    pf_l2(UD + 2 * of);
                    pf_l2(UD + 2 * of + 8);
                }
            }
        }
    };
    load(0, ca, cp, cv, cu);
    V cprev = 0.f, yprev = 0.f;
    for (int k0 = 0; k0 < nz; k0 += KB) {
        if (k0 + KB < nz) load(k0 + KB, na, np, nv, nu);
        float cb[KB];
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            const int k = k0 + e;
            cb[e] = 0.f;
            if (k < nz) {
                V f;
                if (KIND == 0) f = ca[e];
                else if (KIND == 1) f = fmaf(beta, fmaf(-omega, cv[e], cp[e]), ca[e]);
                else f = fmaf(-alpha, cv[e], ca[e]);
                if (KIND != 0 && WRITE_F && act) Pw[k * nx] = f;
                const V u = cu[e].v[0], d = cu[e].v[1];
                V c, y;
                if (k == 0) {
                    c = u;
                    y = f;
                } else {
                    const V inv = rcp_fast<V>(fmaf(-d, cprev, 1.f));
                    c = u * inv;
                    y = fmaf(-d, yprev, f) * inv;
                }
                cb[e] = c;
                ys[k * 128 + tid] = y;
                cprev = c;
                yprev = y;
            }
        }
        tm_st8(taddr + (uint32_t)k0, cb);
#pragma unroll
        for (int e = 0; e < KB; ++e) { ca[e] = na[e]; cp[e] = np[e]; cv[e] = nv[e]; cu[e] = nu[e]; }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    V zn = yprev;
    if (act) Zw[(nz - 1) * nx] = zn;
    for (int k0 = ((nz - 1) / KB) * KB; k0 >= 0; k0 -= KB) {
        float cb[KB];
        tm_ld8(taddr + (uint32_t)k0, cb);
#pragma unroll
        for (int e = KB - 1; e >= 0; --e) {
            const int k = k0 + e;
            if (k <= nz - 2) {
                zn = fmaf(-cb[e], zn, ys[k * 128 + tid]);
                if (act) Zw[k * nx] = zn;
            }
        }
    }
}

template <int MODE, int KIND>
__global__ void __launch_bounds__(128, 4) k_thomas_tm(Geo g, Vecs<MODE> vv, const float* __restrict__ fin,
                                                      float* __restrict__ zout) {
    pdl_enter();  // (EG_PDL: the iteration may launch this kernel programmatically)
    static_assert(sizeof(typename Prec<MODE>::V) == 4, "fp32 working precision only");
    extern __shared__ __align__(16) unsigned char smraw[];
    __shared__ uint32_t tm_base;
    float beta = 0.f, omega = 0.f, alpha = 0.f;
    bool fresh = false;
    if (KIND != 0) {
        const DevState* st = vv.st;
        if (st->halt != H_RUN) return;  // uniform: before any collective
        if (KIND == 1) {
            fresh = st->fresh != 0;
            beta = (float)st->beta_v;
            omega = (float)st->omega_v;
        } else {
            alpha = (float)st->alpha_v;
        }
    }
    const uint32_t base = tm_alloc128(&tm_base);
    const int warp = threadIdx.x >> 5;
    const int nx = (int)g.nx;
    const int i_raw = blockIdx.x * 128 + threadIdx.x;
    const bool act = i_raw < nx;
    const int i = act ? i_raw : nx - 1;  // inactive lanes read a valid column, never store
    thomas_tm_tile<MODE, KIND>(g, vv, (int64_t)blockIdx.y * g.row, i, act, base + ((uint32_t)(warp * 32) << 16),
                               reinterpret_cast<float*>(smraw), beta, omega, alpha, fresh, fin, zout);
    tm_free128(base);
}

// FP64 Thomas with the elimination factors c'_k in TENSOR MEMORY (two 32-bit columns per level;
// 256 columns per 128-column CTA, so at most two CTAs per SM, which the shared-memory request also
// enforces) and y_k in shared memory [k][128]: 8 warps per SM instead of the 6 the two
// shared-memory factor arrays allow, plus an L2 prefetch TM_PF levels ahead.  Same recurrence,
// operation for operation, as k_thomas<0>.  KIND as in k_thomas.  grid (ceil(nx/128), nyl), 128 thr.
constexpr int TM64_SMEM = 80 * 1024;  // >= nz * 128 * 8 (nz <= 80); > 228 KB / 3
template <int KIND>
__global__ void __launch_bounds__(128, 2) k_thomas_tm64(Geo g, Vecs<0> vv, const double* __restrict__ fin,
                                                        double* __restrict__ zout) {
    pdl_enter();  // (EG_PDL: the iteration may launch this kernel programmatically)
    using V = double;
    constexpr int KB = 4;
    extern __shared__ __align__(16) unsigned char smraw[];
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
    if ((threadIdx.x >> 5) == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tm_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tbase = tm_slot;
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t tl = tbase + ((uint32_t)(warp * 32) << 16);
    const int nx = (int)g.nx, nz = (int)g.nz;
    const int i_raw = blockIdx.x * 128 + tid;
    const bool act = i_raw < nx;
    const int i = act ? i_raw : nx - 1;  // inactive lanes read a valid column, never store
    const int64_t base = (int64_t)blockIdx.y * g.row + i;
    const V* __restrict__ A0 = (KIND == 0 ? fin : vv.r) + base;
    const V* __restrict__ Pp = vv.p + base;
    const V* __restrict__ Vv = vv.v + base;
    const V* __restrict__ UD = vv.B2 + 2 * base;
    V* __restrict__ Pw = (KIND == 1 ? vv.p : vv.s) + base;
    V* __restrict__ Zw = zout + base;
    V* ys = reinterpret_cast<V*>(smraw);
    V ca[KB], cp[KB], cv[KB], na[KB], np[KB], nv[KB];
    VecN<V, 2> cu[KB], nu[KB];
#pragma unroll
    for (int e = 0; e < KB; ++e) {
        ca[e] = cp[e] = cv[e] = na[e] = np[e] = nv[e] = 0.0;
        cu[e].v[0] = cu[e].v[1] = nu[e].v[0] = nu[e].v[1] = 0.0;
    }
    auto load = [&](int k0, V(&a)[KB], V(&p)[KB], V(&v)[KB], VecN<V, 2>(&u)[KB]) {
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            const int o = min(k0 + e, nz - 1) * nx;  // tail levels re-read the last one (L1 hit)
            a[e] = A0[o];
            if (KIND == 1 && !fresh) { p[e] = Pp[o]; v[e] = Vv[o]; }
            if (KIND == 2) v[e] = Vv[o];
            u[e] = ldv<2>(UD + 2 * o);
            if (TM_PF > 0 && k0 + e + TM_PF < nz) {  // warp-uniform
                const int of = (k0 + e + TM_PF) * nx;
                if ((tid & 3) == 0) {  // one prefetch per 32-byte sector of each array
                    pf_l2(A0 + of);
                    if (KIND == 1) { pf_l2(Pp + of); pf_l2(Vv + of); }
                    if (KIND == 2) pf_l2(Vv + of);
                }
                if ((tid & 1) == 0) pf_l2(UD + 2 * of);
            }
        }
    };
    load(0, ca, cp, cv, cu);
    V cprev = 0, yprev = 0;
    for (int k0 = 0; k0 < nz; k0 += KB) {
        if (k0 + KB < nz) load(k0 + KB, na, np, nv, nu);
        float cw[2 * KB];  // the c'_k as pairs of 32-bit words
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            const int k = k0 + e;
            V c = 0;
            if (k < nz) {
                V f;
                if (KIND == 0) f = ca[e];
                else if (KIND == 1) f = fresh ? ca[e] : fma(beta, fma(-omega, cv[e], cp[e]), ca[e]);
                else f = fma(-alpha, cv[e], ca[e]);
                if (KIND != 0 && act) Pw[k * nx] = f;
                const V u = cu[e].v[0], d = cu[e].v[1];
                V y;
                if (k == 0) {
                    c = u;
                    y = f;
                } else {
                    const V inv = rcp_fast<V>(fma(-d, cprev, (V)1));
                    c = u * inv;
                    y = fma(-d, yprev, f) * inv;
                }
                ys[k * 128 + tid] = y;
                cprev = c;
                yprev = y;
            }
            const unsigned long long cb = __double_as_longlong(c);
            cw[2 * e] = __uint_as_float((uint32_t)cb);
            cw[2 * e + 1] = __uint_as_float((uint32_t)(cb >> 32));
        }
        tm_st8(tl + (uint32_t)(2 * k0), cw);
#pragma unroll
        for (int e = 0; e < KB; ++e) { ca[e] = na[e]; cp[e] = np[e]; cv[e] = nv[e]; cu[e] = nu[e]; }
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
    V zn = yprev;
    if (act) Zw[(nz - 1) * nx] = zn;
    for (int k0 = ((nz - 1) / KB) * KB; k0 >= 0; k0 -= KB) {
        float cw[2 * KB];
        tm_ld8(tl + (uint32_t)(2 * k0), cw);
#pragma unroll
        for (int e = KB - 1; e >= 0; --e) {
            const int k = k0 + e;
            if (k <= nz - 2) {
                const V c = __longlong_as_double((long long)(((unsigned long long)__float_as_uint(cw[2 * e + 1]) << 32) |
                                                             __float_as_uint(cw[2 * e])));
                zn = fma(-c, zn, ys[k * 128 + tid]);
                if (act) Zw[k * nx] = zn;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tbase) : "memory");
    }
}

// ---- latitude bands: the band-edge rows ----
// Only two rows per band, so these kernels are latency-bound, not bandwidth-bound: a column walk
// over nz levels issues nz dependent rounds of loads.  They stage instead: every thread of a wide
// CTA loads its share of the levels at once into shared memory, a few threads then run the serial
// part from shared memory, and the results leave in parallel.  Same arithmetic as the full-band
// kernels, operation for operation (bitwise equal results).
constexpr int ER_COLS = 64;       // columns per CTA of the edge-row kernels (one P2P flag each)
constexpr int ER_THREADS = 512;   // 8 level lanes x 64 columns
constexpr int ER_MAXL = 16;       // levels per lane: nz <= 128 (the fused schedule's limit)
inline size_t er_smem_bytes(int64_t nz) { return (size_t)5 * nz * ER_COLS * sizeof(float); }

// P2P transport (pp.on): this CTA's ER_COLS columns of the band's edge row go straight into the
// neighbour's ghost row through peer memory (side 0: local row 0 -> rank-1's ghost row nyl; side 1:
// row nyl-1 -> rank+1's ghost row -1), then the tile's flag in the neighbour's workspace is stamped
// with the epoch (release, system scope).  a: 0 = z, 1 = z_s.  zrow: the local row, written by this
// CTA before the call (a __syncthreads precedes).  Columns ER_COLS * blockIdx.x + [0, ER_COLS).
template <class V>
__device__ __forceinline__ void push_edge_tile(const Geo& g, const P2P& pp, int a, int side, const V* zrow,
                                               int epoch) {
    V* dst = (V*)(side == 0 ? pp.dst_lo[a] : pp.dst_hi[a]);
    int* fl = side == 0 ? pp.fdst_lo : pp.fdst_hi;
    if (dst == nullptr || fl == nullptr) return;  // no neighbour on this side (uniform per CTA)
    const int c = threadIdx.x % ER_COLS, kl = threadIdx.x / ER_COLS, nl = blockDim.x / ER_COLS;
    const int i = blockIdx.x * ER_COLS + c;
#ifndef EG_MUTATE_NO_HALO_PUSH  // mutation check of the P2P tests (scripts/build_variant.sh): flags only
    if (i < g.nx)
        for (int k = kl; k < (int)g.nz; k += nl) dst[(int64_t)k * g.nx + i] = zrow[(int64_t)k * g.nx + i];
#endif
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        // the receiver's flags [a][side'][tile]: our row 0 is its ghost row nyl (side' 1), and back
        st_release_sys(fl + (a * 2 + (side == 0 ? 1 : 0)) * pp.tiles + blockIdx.x, epoch);
    }
}

// Fused schedule, latitude bands: z (KIND 1) / z_s (KIND 2) of the band's first and last rows,
// ahead of / beside the phase kernel (which recomputes these rows bitwise identically and is the
// one that writes z, p / s for them), so that they reach the neighbours' ghost rows while it runs.
// zout: scratch rows [2][row] (row 0, row nyl-1); P2P: pushed to the neighbours from here.
// The update f and the Thomas solve of thomas_tm_tile, operation for operation: 512 threads load
// f and (U, D) of all levels of 64 columns into shared memory (8 levels at a time), 64 threads run
// the elimination and back substitution there, 512 threads store.
// grid (ceil(nx/64), 2): blockIdx.y 0 -> local row 0, 1 -> local row nyl-1.  smem er_smem_bytes.
template <int MODE, int KIND>
__global__ void __launch_bounds__(ER_THREADS) k_edge_rows(Geo g, Vecs<MODE> vv, float* __restrict__ zout, P2P pp,
                                                          float* pv_edge) {
    static_assert(sizeof(typename Prec<MODE>::V) == 4, "fp32 working precision only");
    extern __shared__ __align__(16) float ersm[];
    const DevState* st = vv.st;
    if (st->halt != H_RUN) return;
    float beta = 0.f, omega = 0.f, alpha = 0.f;
    bool fresh = false;
    if (KIND == 1) {
        fresh = st->fresh != 0;
        beta = (float)st->beta_v;
        omega = (float)st->omega_v;
    } else {
        alpha = (float)st->alpha_v;
    }
    const int nx = (int)g.nx, nz = (int)g.nz;
    float* F = ersm;                      // f, then z   [nz][64]
    float* U = ersm + nz * ER_COLS;
    float* D = U + nz * ER_COLS;
    float* C = D + nz * ER_COLS;          // c'
    float* Y = C + nz * ER_COLS;          // y
    const int c = threadIdx.x % ER_COLS, kl = threadIdx.x / ER_COLS;
    constexpr int NL = ER_THREADS / ER_COLS;
    const int i_raw = blockIdx.x * ER_COLS + c;
    const bool act = i_raw < nx;
    const int i = act ? i_raw : nx - 1;  // inactive lanes read a valid column, never store
    const int64_t row = blockIdx.y == 0 ? 0 : g.nyl - 1;
    const int64_t base = row * g.row + i;
    const float* __restrict__ A0 = vv.r + base;
    // p = v = 0 after a (re)start: read r in their place with beta = 0 (as thomas_tm_tile).
    // z (KIND 1) with pv_edge: p and v of the edge rows come from the band-edge copies [p, v][2][row]
    // (this kernel's own p of the last iteration, the edge-row stencil's v), not from p / v, which
    // the phase kernel running beside it rewrites; the new p goes back to the copy
    const int64_t eb = (int64_t)blockIdx.y * g.row + i;
    const float* Pp = KIND == 1 && fresh ? vv.r + base : (KIND == 1 && pv_edge ? pv_edge + eb : vv.p + base);
    const float* Vv = KIND == 1 && fresh ? vv.r + base
                      : (KIND == 1 && pv_edge ? pv_edge + 2 * g.row + eb : vv.v + base);
    if (KIND == 1 && fresh) beta = 0.f;
    const float* __restrict__ UD = vv.B2 + 2 * base;
    {  // all of this thread's levels (<= ER_MAXL) loaded before any is used: one round of latency
        float a_[ER_MAXL], p_[ER_MAXL], v_[ER_MAXL];
        VecN<float, 2> ud_[ER_MAXL];
#pragma unroll
        for (int e = 0; e < ER_MAXL; ++e) {
            const int64_t o = (int64_t)min(kl + e * NL, nz - 1) * nx;
            a_[e] = A0[o];
            v_[e] = Vv[o];
            p_[e] = KIND == 1 ? Pp[o] : 0.f;
            ud_[e] = ldv<2>(UD + 2 * o);
        }
#pragma unroll
        for (int e = 0; e < ER_MAXL; ++e) {
            const int k = kl + e * NL;
            if (k < nz) {
                float f;
                if (KIND == 1) f = fmaf(beta, fmaf(-omega, v_[e], p_[e]), a_[e]);
                else f = fmaf(-alpha, v_[e], a_[e]);
                if (KIND == 1 && pv_edge && act) pv_edge[eb + (int64_t)k * nx] = f;  // p of this row, for the next one
                F[k * ER_COLS + c] = f;
                U[k * ER_COLS + c] = ud_[e].v[0];
                D[k * ER_COLS + c] = ud_[e].v[1];
            }
        }
    }
    __syncthreads();
    if (threadIdx.x < ER_COLS) {
        float cprev = 0.f, yprev = 0.f;
#pragma unroll 8
        for (int k = 0; k < nz; ++k) {
            const float u = U[k * ER_COLS + c], d = D[k * ER_COLS + c], f = F[k * ER_COLS + c];
            float cc, y;
            if (k == 0) {
                cc = u;
                y = f;
            } else {
                const float inv = rcp_fast<float>(fmaf(-d, cprev, 1.f));
                cc = u * inv;
                y = fmaf(-d, yprev, f) * inv;
            }
            C[k * ER_COLS + c] = cc;
            Y[k * ER_COLS + c] = y;
            cprev = cc;
            yprev = y;
        }
        float zn = yprev;
        F[(nz - 1) * ER_COLS + c] = zn;
#pragma unroll 8
        for (int k = nz - 2; k >= 0; --k) {
            zn = fmaf(-C[k * ER_COLS + c], zn, Y[k * ER_COLS + c]);
            F[k * ER_COLS + c] = zn;
        }
    }
    __syncthreads();
    float* zrow = zout + (int64_t)blockIdx.y * g.row;
    if (act)
        for (int k = kl; k < nz; k += NL) zrow[(int64_t)k * nx + i] = F[k * ER_COLS + c];
    if (pp.on) {
        __syncthreads();
        push_edge_tile<float>(g, pp, KIND - 1, (int)blockIdx.y, zrow, *(volatile const int*)&st->epoch);
    }
}

// P2P transport, 5-kernel schedule: push the edge rows of z (a = 0) / z_s (a = 1) that the Thomas
// kernel just wrote.  grid (ceil(nx/64), 2), 256 threads; blockIdx.y = side as in push_edge_tile.
template <class V>
__global__ void __launch_bounds__(256) k_push_rows(Geo g, const V* __restrict__ z, const DevState* st, P2P pp, int a) {
    if (st->halt != H_RUN) return;
    const int64_t row = blockIdx.y == 0 ? 0 : g.nyl - 1;
    push_edge_tile<V>(g, pp, a, (int)blockIdx.y, z + row * g.row, *(volatile const int*)&st->epoch);
}

// P2P transport, tri-SOR (NEXT-1): the halo after every red-black half-sweep (and the sequenced
// halos outside the iteration: x before a restart / the verification, the input of
// eg_apply_operator).  k_push_sweep pushes rows 0 / nyl-1 of an array (which: 0 z, 1 z_s, 2 the
// colour-split x, 3 the ghost rows of x) into
// the neighbours' ghost rows and stamps their flags [seq & 1][side][tile] with seq + 1; k_wait_sweep
// waits for the neighbours' stamps of the same seq, then advances this rank's counter (*tcount,
// every rank the same sequence of half-sweeps).  Two flag buffers: a rank's push seq + 2 needs its
// wait seq + 1, i.e. the neighbour's push seq + 1, made after that neighbour's wait seq.  The ghost
// data itself is single-buffered: a push overwrites the neighbour's ghost row while that
// neighbour's next half-sweep may read it, but that half-sweep reads only the other colour, whose
// values the push rewrites unchanged (a half-sweep updates one colour).  check_halt: inside a
// solve (KIND != 0) the sweeps of a halted iteration return early, and so do both kernels.
template <class V>
__global__ void __launch_bounds__(256) k_push_sweep(Geo g, const V* __restrict__ arr, const DevState* st, P2P pp, int which,
                                                    int check_halt) {
    if (check_halt && st->halt != H_RUN) return;
    V* dst = (V*)(blockIdx.y == 0 ? (which == 3 ? pp.dst_lo_xg : which == 2 ? pp.dst_lo_x : pp.dst_lo[which])
                                   : (which == 3 ? pp.dst_hi_xg : which == 2 ? pp.dst_hi_x : pp.dst_hi[which]));
    int* fl = blockIdx.y == 0 ? pp.tdst_lo : pp.tdst_hi;
    if (dst == nullptr || fl == nullptr) return;
    const int seq = *(volatile const int*)pp.tcount;
    const int64_t row = blockIdx.y == 0 ? 0 : g.nyl - 1;
    const V* src = arr + row * g.row;
    const int c = threadIdx.x % ER_COLS, kl = threadIdx.x / ER_COLS, nl = blockDim.x / ER_COLS;
    const int i = blockIdx.x * ER_COLS + c;
#ifndef EG_MUTATE_NO_SWEEP_PUSH  // mutation check of the tri-SOR P2P test (scripts/build_variant.sh)
    if (i < g.nx)
        for (int k = kl; k < (int)g.nz; k += nl) dst[(int64_t)k * g.nx + i] = src[(int64_t)k * g.nx + i];
#endif
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        // our row 0 is rank-1's ghost row nyl (its side 1), our row nyl-1 rank+1's ghost row -1
        st_release_sys(fl + ((seq & 1) * 2 + (blockIdx.y == 0 ? 1 : 0)) * pp.tiles + blockIdx.x, seq + 1);
    }
}
__global__ void __launch_bounds__(256) k_wait_sweep(DevState* st, P2P pp, int check_halt, int wlo, int whi) {
    if (check_halt && st->halt != H_RUN) return;
    const int seq = *(volatile const int*)pp.tcount;
    bool bad = false;
    for (int t = threadIdx.x; t < 2 * pp.tiles; t += blockDim.x) {
        const int side = t / pp.tiles;
        if (side == 0 ? !wlo : !whi) continue;
        if (!wait_flag_sys(pp.tflag + (seq & 1) * 2 * pp.tiles + t, seq + 1, pp.timeout_ns)) bad = true;
    }
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0) {
        *pp.tcount = seq + 1;
        if (bad) st->halt = H_PEER_TIMEOUT;
    }
}

// The P2P wait of an edge-row stencil CTA (128 columns = flags 2 blockIdx.x, 2 blockIdx.x + 1):
// the neighbours' pushes of this epoch into the ghost row(s) its row reads.  hw: this rank's halo
// flags of the array [side][tiles64] (NULL: no wait).  false on timeout.
struct HWait {
    const int* f;
    int tiles64;
    int wlo, whi;      // rank-1 / rank+1 exist
    long long timeout_ns;
};
__device__ __forceinline__ bool edge_wait(const HWait& hw, int64_t jl, int64_t nyl, int epoch) {
    bool ok = true;
    for (int h = 0; h < 2; ++h) {
        const int t = 2 * (int)blockIdx.x + h;
        if (t >= hw.tiles64) break;
        if (hw.wlo && jl == 0) ok = wait_flag_sys(hw.f + t, epoch, hw.timeout_ns) && ok;
        if (hw.whi && jl == nyl - 1) ok = wait_flag_sys(hw.f + hw.tiles64 + t, epoch, hw.timeout_ns) && ok;
    }
    return ok;
}

// ---------------------------------------------------------------------------------------------
// NEXT-1: one half-sweep of the tri-SOR preconditioner (Eq. 7) in red-black column
// order, over the columns (i, j) with (i + j) % 2 == colour:
//   rhs_k = (1 - omega) (T x_old)_k + omega (f_k - (E x_E + W x_W + N x_N + S x_S)_k)
//   x_col = T^-1 rhs                                   (Thomas, factors in shared memory)
// The horizontal neighbours of a column all have the other colour, so they are either the values
// of the previous sweep (red half) or of this sweep's red half (black half): in-place updates are
// race-free.  FIRST (sweep 1, x = 0): no T x_old term, and the red half needs no neighbours
// (rhs = omega f); with KIND 1 / 2 the first sweep also forms f = p (or s) for its colour's columns
// and stores it (later sweeps read it back with KIND 0).  Thread m of row j owns column
// i = 2m + ((j + colour) & 1); grid (ceil(nx/2 / W), nyl), dynamic smem 2*nz*W*sizeof(V).
// Colour-split copies (EG_FEATURE_TRISOR): split[c] holds, per (row, level), the nx/2 values of
// the columns of colour c in order, so a half-sweep thread m reads split + (jl*nz*nx +
// c*nx/2 + m) + k*nx: every loaded sector is used, where the natural arrays waste half of each.
template <class V>
struct Split {
    const V* b4;  // (E, W, N, S) per point, colour-split
    const V* b2;  // (U, D)
    V* f;         // the sweep's right-hand side (written by the first sweep, read by the others)
};

template <class V>
__global__ void __launch_bounds__(256) k_split_bands(Geo g, const V* __restrict__ B4, const V* __restrict__ B2,
                                                     V* __restrict__ B4s, V* __restrict__ B2s) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.nx) return;
    const int64_t k = blockIdx.y, jl = blockIdx.z, jg = g.j0 + jl;
    const int64_t q = jl * g.row + k * g.nx + i;
    const int64_t qs = jl * g.row + k * g.nx + ((i + jg) & 1) * (g.nx / 2) + (i >> 1);
    stv<4>(B4s + 4 * qs, ldv<4>(B4 + 4 * q));
    stv<2>(B2s + 2 * qs, ldv<2>(B2 + 2 * q));
}

template <int MODE, int KIND, bool FIRST>
__global__ void __launch_bounds__(128) k_sor_half(Geo g, Vecs<MODE> vv, const typename Prec<MODE>::V* __restrict__ fin,
                                                  typename Prec<MODE>::V* __restrict__ x, int colour,
                                                  double omega_d, int check_halt, Split<typename Prec<MODE>::V> sp) {
    using V = typename Prec<MODE>::V;
    constexpr int KB = sizeof(V) == 4 ? 4 : 2;
    constexpr int NA = 13;  // f, x(k), x(k+1) [own], xE, xW, xN, xS, E, W, N, S, U, D
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
    } else if (check_halt && vv.st->halt != H_RUN) {
        return;
    }
    const V om = (V)omega_d, om1 = (V)(1.0 - omega_d);
    const int nx = (int)g.nx, nz = (int)g.nz;
    const int m = blockIdx.x * W + tid;
    if (m >= nx / 2) return;
    const int64_t jl = blockIdx.y, jg = g.j0 + jl;
    const int i = 2 * m + (int)((jg + colour) & 1);
    const int iE = (i + 1 == nx) ? 0 : i + 1, iW = (i == 0) ? nx - 1 : i - 1;
    const int64_t rb = jl * g.row;
    const V* __restrict__ xc = x + rb + i;
    const V* __restrict__ xE = x + rb + iE;
    const V* __restrict__ xW = x + rb + iW;
    // at the poles the absent N / S neighbour (zero band) reads the E neighbour instead: it has the
    // other colour, so it is already written even in the first sweep (the own column is not)
    const V* __restrict__ xN = (jg < g.ny - 1) ? xc + g.row : xE;
    const V* __restrict__ xS = (jg > 0) ? xc - g.row : xE;
    const bool split = sp.b4 != nullptr;  // uniform
    const int64_t qs = rb + (int64_t)colour * (nx / 2) + m;  // colour-split index (per-level stride nx)
    const V* __restrict__ b4 = split ? sp.b4 + 4 * qs : vv.B4 + 4 * (rb + i);
    const V* __restrict__ b2 = split ? sp.b2 + 2 * qs : vv.B2 + 2 * (rb + i);
    const V* __restrict__ A0 = (!FIRST && split) ? sp.f + qs : (KIND == 0 ? fin : vv.r) + rb + i;
    const V* __restrict__ Pp = (KIND == 1 && fresh ? vv.r : vv.p) + rb + i;
    const V* __restrict__ Vv = (KIND == 1 && fresh ? vv.r : vv.v) + rb + i;
    if (KIND == 1 && fresh) beta = 0;
    V* __restrict__ Fw = (KIND == 1 ? vv.p : vv.s) + rb + i;
    V* __restrict__ Fs = split ? sp.f + qs : nullptr;
    V* __restrict__ Xw = x + rb + i;
    const bool need_nbr = !(FIRST && colour == 0);
    V cur[KB][NA], nxt[KB][NA];
#pragma unroll
    for (int e = 0; e < KB; ++e)
#pragma unroll
        for (int a = 0; a < NA; ++a) cur[e][a] = nxt[e][a] = (V)0;
    auto load = [&](int k0, V(&b)[KB][NA]) {
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            const int k = min(k0 + e, nz - 1);
            const int o = k * nx;
            if (KIND == 1) b[e][0] = fma(beta, fma(-omega_b, Vv[o], Pp[o]), A0[o]);
            else if (KIND == 2) b[e][0] = fma(-alpha, Vv[o], A0[o]);
            else b[e][0] = A0[o];
            if (!FIRST) {
                b[e][1] = xc[o];
                b[e][2] = xc[min(k + 1, nz - 1) * nx];
            }
            if (need_nbr) {
                b[e][3] = xE[o]; b[e][4] = xW[o]; b[e][5] = xN[o]; b[e][6] = xS[o];
                const VecN<V, 4> h4 = ldv<4>(b4 + 4 * o);
                b[e][7] = h4.v[0]; b[e][8] = h4.v[1]; b[e][9] = h4.v[2]; b[e][10] = h4.v[3];
            }
            const VecN<V, 2> h2 = ldv<2>(b2 + 2 * o);
            b[e][11] = h2.v[0]; b[e][12] = h2.v[1];
        }
    };
    load(0, cur);
    V cprev = 0, yprev = 0, xprev = 0;
    for (int k0 = 0; k0 < nz; k0 += KB) {
        if (k0 + KB < nz) load(k0 + KB, nxt);
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            const int k = k0 + e;
            if (k < nz) {
                const V f = cur[e][0];
                if (FIRST && KIND != 0) Fw[k * nx] = f;
                if (FIRST && split) Fs[k * nx] = f;  // the later sweeps read f colour-split
                V rhs;
                V hx = 0;
                if (need_nbr) {
                    hx = cur[e][7] * cur[e][3];
                    hx = fma(cur[e][8], cur[e][4], hx);
                    hx = fma(cur[e][9], cur[e][5], hx);
                    hx = fma(cur[e][10], cur[e][6], hx);
                }
                if (FIRST) {
                    rhs = om * (f - hx);
                } else {
                    V tx = cur[e][1];
                    tx = fma(cur[e][11], cur[e][2], tx);   // U x(k+1): U = 0 on the top level
                    tx = fma(cur[e][12], xprev, tx);      // D x(k-1): D = 0 at k = 0
                    rhs = fma(om1, tx, om * (f - hx));
                    xprev = cur[e][1];
                }
                const V u = cur[e][11], d = cur[e][12];
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
        for (int e = 0; e < KB; ++e)
#pragma unroll
            for (int a = 0; a < NA; ++a) cur[e][a] = nxt[e][a];
    }
    V zn = yprev;
    Xw[(nz - 1) * nx] = zn;
    for (int k = nz - 2; k >= 0; --k) {
        zn = fma(-cps[k * W + tid], zn, ys[k * W + tid]);
        Xw[k * nx] = zn;
    }
}

// ---------------------------------------------------------------------------------------------
// a4 / a7 / apply: y = Ahat z (unit diagonal + 6 bands; periodic i; absent neighbours contribute 0)
// DOTS 0: none;  1: sigma = aux . y (aux = rhat0);  2: t.s, t.t, s.s (aux = s).
// Thread per column walking k.  Loads of KB levels (B4, B2, z centre / E / W / N / S, aux) are
// issued as one batch into registers while the previous batch is combined (double-buffered
// register prefetch).  Absent N/S neighbours at the poles read the centre row instead (a valid
// address) and are multiplied by their zero band (validated at create); the top / bottom U / D
// bands are zero the same way.  grid (tiles, nyl), block RW.
template <int MODE, int DOTS>
__global__ void __launch_bounds__(RW, 4) k_stencil(Geo g, Vecs<MODE> vv,
                                                const typename Prec<MODE>::V* __restrict__ z,
                                                typename Prec<MODE>::V* __restrict__ y,
                                                const typename Prec<MODE>::V* __restrict__ aux, RowMap rm) {
    pdl_enter();  // (EG_PDL: the iteration may launch this kernel programmatically)
    using V = typename Prec<MODE>::V;
    if (DOTS != 0 && vv.st->halt != H_RUN) return;
    constexpr int NQ = DOTS == 2 ? 3 : 1;
    constexpr int KB = sizeof(V) == 4 ? 4 : 2;
    constexpr int NA = DOTS ? 12 : 11;
    double acc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
    const int i = blockIdx.x * RW + threadIdx.x;
    const int64_t jl = rm.lo + (int64_t)blockIdx.y * rm.step, jg = g.j0 + jl;
    if (i < g.nx) {
        const int nx = (int)g.nx, nz = (int)g.nz;
        const int64_t rb = jl * g.row;
        const int iE = (i + 1 == nx) ? 0 : i + 1, iW = (i == 0) ? nx - 1 : i - 1;
        const V* __restrict__ zc = z + rb + i;
        const V* __restrict__ zE = z + rb + iE;
        const V* __restrict__ zW = z + rb + iW;
        const V* __restrict__ zN = (jg < g.ny - 1) ? zc + g.row : zc;
        const V* __restrict__ zS = (jg > 0) ? zc - g.row : zc;
        const V* __restrict__ b4 = vv.B4 + 4 * (rb + i);
        const V* __restrict__ b2 = vv.B2 + 2 * (rb + i);
        const V* __restrict__ ax = DOTS ? aux + rb + i : zc;
        V* __restrict__ yo = y + rb + i;
        V cur[KB][NA], nxt[KB][NA];
#pragma unroll
        for (int e = 0; e < KB; ++e)
#pragma unroll
            for (int a = 0; a < NA; ++a) cur[e][a] = nxt[e][a] = (V)0;
        V zup_c = 0, zup_n = 0;
        auto load = [&](int k0, V(&b)[KB][NA], V& zup) {
#pragma unroll
            for (int e = 0; e < KB; ++e) {
                const int o = min(k0 + e, nz - 1) * nx;  // tail levels re-read the last one
                const VecN<V, 4> h4 = ldv<4>(b4 + 4 * o);
                const VecN<V, 2> h2 = ldv<2>(b2 + 2 * o);
                b[e][0] = h4.v[0]; b[e][1] = h4.v[1]; b[e][2] = h4.v[2];
                b[e][3] = h4.v[3]; b[e][4] = h2.v[0]; b[e][5] = h2.v[1];
                b[e][6] = zc[o]; b[e][7] = zE[o]; b[e][8] = zW[o];
                b[e][9] = zN[o]; b[e][10] = zS[o];
                if (DOTS) b[e][NA - 1] = ax[o];
                if (ST_PF > 0 && k0 + e + ST_PF < nz) {  // warp-uniform
                    const int of = (k0 + e + ST_PF) * nx;
                    const int l = threadIdx.x & 31;
                    if ((l & 7) == 0) {  // one per 32-byte sector: z, aux, B2
                        pf_l2(zc + of);
                        if (DOTS) pf_l2(ax + of);
                        pf_l2(b2 + 2 * of);
                    }
                    if ((l & 1) == 0) pf_l2(b4 + 4 * of);  // B4: 16 B per point
                }
            }
            zup = zc[min(k0 + KB, nz - 1) * nx];  // multiplied by U = 0 on the top level
        };
        load(0, cur, zup_c);
        V zprev = 0;
        for (int k0 = 0; k0 < nz; k0 += KB) {
            if (k0 + KB < nz) load(k0 + KB, nxt, zup_n);
#pragma unroll
            for (int e = 0; e < KB; ++e) {
                const int k = k0 + e;
                if (k < nz) {
                    const V zm = e == 0 ? zprev : cur[e - 1][6];
                    const V zp = e + 1 < KB ? cur[e + 1][6] : zup_c;  // U = 0 at k = nz-1
                    V a = cur[e][6];
                    a = fma(cur[e][0], cur[e][7], a);
                    a = fma(cur[e][1], cur[e][8], a);
                    a = fma(cur[e][2], cur[e][9], a);
                    a = fma(cur[e][3], cur[e][10], a);
                    a = fma(cur[e][4], zp, a);
                    a = fma(cur[e][5], zm, a);
                    yo[k * nx] = a;
                    if (DOTS == 1) {
                        acc_dot<MODE>(acc[0], cur[e][NA - 1], a);
                    } else if (DOTS == 2) {
                        const V sv = cur[e][NA - 1];
                        acc_dot<MODE>(acc[0], a, sv);
                        acc_dot<MODE>(acc[1], a, a);
                        acc_dot<MODE>(acc[2], sv, sv);
                    }
                }
            }
            zprev = cur[KB - 1][6];
#pragma unroll
            for (int e = 0; e < KB; ++e)
#pragma unroll
                for (int a = 0; a < NA; ++a) cur[e][a] = nxt[e][a];
            zup_c = zup_n;
        }
    }
    if (DOTS != 0) write_slots<NQ>(g, vv.slots, acc, MODE == 2 ? 0x7u : 0x0u, jl);
}

// The stencil (and its dot-product slots) of a few rows — the band-edge rows of latitude bands,
// after their ghost rows arrived.  Two rows are too few for k_stencil's column walk (nz dependent
// rounds of loads in 24 CTAs), so one latency-short kernel, k_edge_stencil:
//  * every CTA computes y = Ahat z at 4 levels of 128 columns of one row, one point per thread
//    (grid (tiles, rows, ceil(nz / 4))): a single round of loads.  With the P2P transport it first
//    waits (hw.f != NULL) for the neighbours' pushes of this epoch, which may land while the grid
//    runs, so z is read through L2 (ld.global.cg);
//  * the last CTA to finish a (tile, row) — an arrival counter per (row, tile) in ctr, reset by it —
//    loads y and aux of every level of its 128 columns into shared memory (one round, L2) and its
//    first 128 threads add their column's terms in level order, then the CTA's slot: k_stencil's
//    sums operation for operation (the other 384 threads join the CTA sum with zero partials: a sum
//    that starts at +0.0 is never -0.0, so adding +0.0 leaves every bit).
// Bitwise equal to k_stencil's y and slots.  Dynamic smem: es_smem_bytes.
constexpr int ES_KC = 64;  // levels staged per round of the dot pass
template <int MODE>
inline size_t es_smem_bytes() { return (size_t)2 * ES_KC * RW * sizeof(typename Prec<MODE>::V); }
template <int MODE, int DOTS>
__global__ void __launch_bounds__(512) k_edge_stencil(Geo g, Vecs<MODE> vv, const typename Prec<MODE>::V* __restrict__ z,
                                                      typename Prec<MODE>::V* __restrict__ y,
                                                      const typename Prec<MODE>::V* __restrict__ aux, RowMap rm, HWait hw,
                                                      int* __restrict__ ctr, typename Prec<MODE>::V* ycopy) {
    using V = typename Prec<MODE>::V;
    extern __shared__ __align__(16) unsigned char essm[];
    if (vv.st->halt != H_RUN) return;
    const int64_t jl = rm.lo + (int64_t)blockIdx.y * rm.step, jg = g.j0 + jl;
    __shared__ int flag;
    if (hw.f != nullptr) {
        if (threadIdx.x == 0) flag = edge_wait(hw, jl, g.nyl, *(volatile const int*)&vv.st->epoch);
        __syncthreads();
        if (!flag) {
            if (threadIdx.x == 0) vv.st->halt = H_PEER_TIMEOUT;
            return;
        }
        __syncthreads();
    }
    const int c = threadIdx.x % RW;
    const int i = blockIdx.x * RW + c;
    const int nx = (int)g.nx, nz = (int)g.nz;
    const int64_t rb = jl * g.row;
    {
        const int k = (int)blockIdx.z * 4 + (int)threadIdx.x / RW;
        if (i < nx && k < nz) {
            const int iE = (i + 1 == nx) ? 0 : i + 1, iW = (i == 0) ? nx - 1 : i - 1;
            const V* zc = z + rb + i;
            const V* zN = (jg < g.ny - 1) ? zc + g.row : zc;
            const V* zS = (jg > 0) ? zc - g.row : zc;
            const int o = k * nx;
            const VecN<V, 4> h4 = ldv<4>(vv.B4 + 4 * (rb + i + o));
            const VecN<V, 2> h2 = ldv<2>(vv.B2 + 2 * (rb + i + o));
            const V zp = __ldcg(zc + min(k + 1, nz - 1) * nx);  // multiplied by U = 0 on the top level
            const V zm = k == 0 ? (V)0 : __ldcg(zc + (k - 1) * nx);
            V a = __ldcg(zc + o);
            a = fma(h4.v[0], __ldcg(z + rb + iE + o), a);
            a = fma(h4.v[1], __ldcg(z + rb + iW + o), a);
            a = fma(h4.v[2], __ldcg(zN + o), a);
            a = fma(h4.v[3], __ldcg(zS + o), a);
            a = fma(h2.v[0], zp, a);
            a = fma(h2.v[1], zm, a);
            y[rb + i + o] = a;
#ifndef EG_MUTATE_NO_VCOPY  // mutation check of the band-edge copies (scripts/build_variant.sh)
            if (ycopy) {  // v of the band-edge rows for k_edge_rows (slot 0: row 0, slot 1: row nyl-1)
                if (jl == 0) ycopy[i + o] = a;
                if (jl == g.nyl - 1) ycopy[g.row + i + o] = a;
            }
#endif
        }
    }
    if (DOTS == 0) return;
    // the last CTA of this (tile, row) to arrive sums the column terms
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();  // this CTA's y before its arrival
        int* cp = ctr + blockIdx.y * gridDim.x + blockIdx.x;
        flag = atomicAdd(cp, 1) == (int)gridDim.z - 1;
        if (flag) *cp = 0;  // every CTA of the (tile, row) has arrived: ready for the next launch
    }
    __syncthreads();
    if (!flag) return;
    __threadfence();
    constexpr int NQ = DOTS == 2 ? 3 : 1;
    V* sy = reinterpret_cast<V*>(essm);
    V* sx = sy + ES_KC * RW;
    double acc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
    constexpr int PER = ES_KC * RW / 512;  // elements per thread per round
    for (int k0 = 0; k0 < nz; k0 += ES_KC) {
        const int kn = min(ES_KC, nz - k0);
        V ty[PER], tx[PER];
#pragma unroll
        for (int u = 0; u < PER; ++u) {  // all loads of the round first: [level][column], coalesced
            const int e = threadIdx.x + u * 512, kk = e / RW, ii = blockIdx.x * RW + e % RW;
            if (kk < kn && ii < nx) {
                const int64_t q = rb + ii + (int64_t)(k0 + kk) * nx;
                ty[u] = __ldcg(y + q);
                tx[u] = aux[q];
            }
        }
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int e = threadIdx.x + u * 512, kk = e / RW, ii = blockIdx.x * RW + e % RW;
            if (kk < kn && ii < nx) {
                sy[e] = ty[u];
                sx[e] = tx[u];
            }
        }
        __syncthreads();
        if (threadIdx.x < RW && i < nx) {
            for (int kk = 0; kk < kn; ++kk) {
                const V a = sy[kk * RW + c], sv = sx[kk * RW + c];
                if (DOTS == 1) {
                    acc_dot<MODE>(acc[0], sv, a);
                } else {
                    acc_dot<MODE>(acc[0], a, sv);
                    acc_dot<MODE>(acc[1], a, a);
                    acc_dot<MODE>(acc[2], sv, sv);
                }
            }
        }
        __syncthreads();
    }
    write_slots<NQ>(g, vv.slots, acc, MODE == 2 ? 0x7u : 0x0u, jl);
}

// ---------------------------------------------------------------------------------------------
// a9: x += alpha z + omega z_s (X precision, scalars unrounded, A-10); r = s - omega t;
// partials rhat0 . r, r . r.  On an s-step exit only x += alpha z.  CPT columns per thread,
// double-buffered register batches of KB levels.  grid (tiles, nyl), block RW / CPT.
// PART 0: both updates.  Latitude bands split it so that the x half runs beside reduction 3
// (its all-gather) on a side stream: PART 1 = r and its partials, PART 2 = x only, which reads the
// control snapshot reduction 2 left (xs_*), because reduction 3 rewrites halt / sexit / xzero
// while it runs.  The arithmetic of each half is PART 0's.
// KBX > 0 overrides the batch depth (levels per register batch; same operations in the same order):
// shallower batches use fewer registers, so more CTAs fit an SM when the grid is only a few waves.
template <int MODE, int CPT, int PART = 0, int KBX = 0>
__global__ void __launch_bounds__(RW) k_update(Geo g, Vecs<MODE> vv) {
    using V = typename Prec<MODE>::V;
    using X = typename Prec<MODE>::X;
    constexpr int KB0 = (sizeof(V) == 4 ? 8 : 4) / CPT > 0 ? (sizeof(V) == 4 ? 8 : 4) / CPT : 1;
    constexpr int KB = KBX > 0 ? KBX : KB0;
    constexpr bool DO_X = PART != 1, DO_R = PART != 2;
    using VC = VecN<V, CPT>;
    using XC = VecN<X, CPT>;
    const DevState* st = vv.st;
    pdl_enter();
    if (PART == 2 ? st->xs_run == 0 : st->halt != H_RUN) return;
    const bool sexit = (PART == 2 ? st->xs_sexit : st->sexit) != 0;
    const bool xz = (PART == 2 ? st->xs_xzero : st->xzero) != 0;  // x = 0 (not stored): first update after x0 = 0
    if (PART == 1 && sexit) return;
    const X alpha = (X)st->alpha, omega = (X)st->omega;
    const V omega_v = (V)st->omega_v;
    double acc[2] = {0.0, 0.0};
    const int i = blockIdx.x * RW + threadIdx.x * CPT;
    if (i < g.nx) {
        const int nx = (int)g.nx, nz = (int)g.nz;
        const int64_t base = (int64_t)blockIdx.y * g.row + i;
        X* __restrict__ xp = vv.x + base;
        const V* __restrict__ zp = vv.z + base;
        const V* __restrict__ zsp = vv.zs + base;
        const V* __restrict__ sp = vv.s + base;
        const V* __restrict__ tp = vv.t + base;
        const V* __restrict__ rhp = vv.rh + base;
        V* __restrict__ rp = vv.r + base;
        if (sexit) {  // (PART 0 / 2)
            for (int k = 0; k < nz; ++k) {
                XC xv;
#pragma unroll
                for (int c = 0; c < CPT; ++c) xv.v[c] = (X)0;
                if (!xz) xv = ldv<CPT>(xp + k * nx);
                const VC zv = ldv<CPT>(zp + k * nx);
#pragma unroll
                for (int c = 0; c < CPT; ++c) xv.v[c] = fma(alpha, (X)zv.v[c], xv.v[c]);
                stv<CPT>(xp + k * nx, xv);
            }
        } else {
            XC cx[KB], nxv[KB];
            VC cz[KB], czs[KB], cs[KB], ct[KB], crh[KB];
            VC nz_[KB], nzs[KB], ns[KB], nt[KB], nrh[KB];
#pragma unroll
            for (int e = 0; e < KB; ++e)
#pragma unroll
                for (int c = 0; c < CPT; ++c) {
                    cx[e].v[c] = nxv[e].v[c] = (X)0;
                    cz[e].v[c] = czs[e].v[c] = cs[e].v[c] = ct[e].v[c] = crh[e].v[c] = (V)0;
                    nz_[e].v[c] = nzs[e].v[c] = ns[e].v[c] = nt[e].v[c] = nrh[e].v[c] = (V)0;
                }
            auto load = [&](int k0, XC(&x_)[KB], VC(&z_)[KB], VC(&zs_)[KB], VC(&s_)[KB], VC(&t_)[KB],
                            VC(&rh_)[KB]) {
#pragma unroll
                for (int e = 0; e < KB; ++e) {
                    const int o = min(k0 + e, nz - 1) * nx;  // tail levels re-read the last one
                    if (DO_X) {
                        if (!xz) x_[e] = ldv<CPT>(xp + o);  // else stays 0
                        z_[e] = ldv<CPT>(zp + o); zs_[e] = ldv<CPT>(zsp + o);
                    }
                    if (DO_R) { s_[e] = ldv<CPT>(sp + o); t_[e] = ldv<CPT>(tp + o); rh_[e] = ldv<CPT>(rhp + o); }
                    if (UP_PF > 0 && k0 + e + UP_PF < nz) {  // warp-uniform
                        const int of = (k0 + e + UP_PF) * nx;
                        const int l = threadIdx.x & 31;
                        if ((l * CPT * (int)sizeof(V)) % 32 == 0) {
                            if (DO_X) { pf_l2(zp + of); pf_l2(zsp + of); }
                            if (DO_R) { pf_l2(sp + of); pf_l2(tp + of); pf_l2(rhp + of); }
                        }
                        if (DO_X && (l * CPT * (int)sizeof(X)) % 32 == 0) pf_l2(xp + of);
                    }
                }
            };
            load(0, cx, cz, czs, cs, ct, crh);
            for (int k0 = 0; k0 < nz; k0 += KB) {
                if (k0 + KB < nz) load(k0 + KB, nxv, nz_, nzs, ns, nt, nrh);
#pragma unroll
                for (int e = 0; e < KB; ++e) {
                    const int k = k0 + e;
                    if (k < nz) {
                        const int o = k * nx;
                        XC xv;
                        VC rv;
#pragma unroll
                        for (int c = 0; c < CPT; ++c) {
                            if (DO_X) xv.v[c] = fma(omega, (X)czs[e].v[c], fma(alpha, (X)cz[e].v[c], cx[e].v[c]));
                            if (DO_R) {
                                rv.v[c] = fma(-omega_v, ct[e].v[c], cs[e].v[c]);
                                acc_dot<MODE>(acc[0], crh[e].v[c], rv.v[c]);
                                acc_dot<MODE>(acc[1], rv.v[c], rv.v[c]);
                            }
                        }
                        if (DO_X) stv<CPT>(xp + o, xv);
                        if (DO_R) stv<CPT>(rp + o, rv);
                    }
                }
#pragma unroll
                for (int e = 0; e < KB; ++e) {
                    cx[e] = nxv[e]; cz[e] = nz_[e]; czs[e] = nzs[e]; cs[e] = ns[e]; ct[e] = nt[e]; crh[e] = nrh[e];
                }
            }
        }
    }
    if (DO_R && !sexit) write_slots<2>(g, vv.slots, acc, MODE == 2 ? 0x3u : 0x0u);
}

// ---------------------------------------------------------------------------------------------
// Finalisers.  fin_groups: warp w sums quantity (w % NQ) of local group (w / NQ): lane l sums the
// group's (row, tile) slots l, l+32, l+64, ... in 16 fixed chains, then a fixed shuffle tree.
// fin_logic (thread 0): groups in order -> totals -> BiCGStab scalars and control flags.
enum Which { W_START = 0, W_A = 1, W_B = 2, W_C = 3, W_VERIFY = 4, W_SHADOW = 5 };
// quantities per slot row of each finaliser: A sigma | B t.s, t.t, s.s | C rhat0.r, r.r |
// START / VERIFY ||bhat||^2, ||res||^2 (fp64), r.r | SHADOW rhat0.r, rhat0.rhat0
__host__ __device__ constexpr int fin_nq(int which) {
    return which == W_A ? 1 : (which == W_C || which == W_SHADOW) ? 2 : 3;
}
// FP32 mode: which of them are binary32 sums (bit q); the true residual stays fp64
template <int MODE>
__host__ __device__ constexpr uint32_t fin_r32(int which) {
    return MODE != 2 ? 0x0u : (which == W_START || which == W_VERIFY) ? 0x5u : which == W_SHADOW ? 0x3u : 0x7u;
}

// breakdown test of rho at a (re)start and after an iteration (A-12): exactly 0, non-finite, or
// |rho| < eps_V ||rhat0|| ||r|| ("scalar weights ... close to or equal to zero")
__device__ __forceinline__ bool rho_breakdown(double rho, double rh_norm, double rr, double eps) {
    return rho == 0.0 || !isfinite(rho) || fabs(rho) < eps * rh_norm * sqrt(rr);
}

template <int NQ>
__device__ __forceinline__ void fin_groups(const Geo& g, const double* __restrict__ slots, uint32_t r32,
                                           double* __restrict__ gsum) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int gl = w / NQ, qq = w % NQ;
    if (gl >= g.g_hi - g.g_lo) return;
    const int gi = g.g_lo + gl;
    const int64_t rb = (int64_t)gi * g.ny / g.G - g.j0, re = (int64_t)(gi + 1) * g.ny / g.G - g.j0;
    const int64_t L = (re - rb) * g.tiles;
    const double* src = slots + (int64_t)qq * g.nyl * g.tiles + rb * g.tiles;
    const bool f = (r32 >> qq) & 1u;
    // lane l sums slots l + 32 m for m = 0, 1, 2, ... into FC chains (m mod FC; the FC loads of a
    // round are independent, so a round costs one L2 latency), combined by a fixed pairwise tree:
    // coalesced, latency-tolerant, and the same tree for any launch / rank count
    constexpr int FC = 16;
    double ac[FC];
#pragma unroll
    for (int c = 0; c < FC; ++c) ac[c] = 0.0;
    int64_t e = lane;
    for (; e + 32 * (FC - 1) < L; e += 32 * FC) {
        double v[FC];
#pragma unroll
        for (int c = 0; c < FC; ++c) v[c] = src[e + 32 * c];
#pragma unroll
        for (int c = 0; c < FC; ++c) {
            ac[c] += v[c];
            if (f) ac[c] = (double)(float)ac[c];
        }
    }
#pragma unroll
    for (int c = 0; c < FC; ++c) {  // the last partial round
        if (e + 32 * c < L) {
            ac[c] += src[e + 32 * c];
            if (f) ac[c] = (double)(float)ac[c];
        }
    }
#pragma unroll
    for (int h = FC / 2; h > 0; h >>= 1) {
#pragma unroll
        for (int c = 0; c < h; ++c) {
            ac[c] += ac[c + h];
            if (f) ac[c] = (double)(float)ac[c];
        }
    }
    double s = ac[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_down_sync(0xffffffffu, s, o);
        if (f) s = (double)(float)s;
    }
    if (lane == 0) gsum[gl * NQ + qq] = s;
}

// The same sums as fin_groups, with the chains spread over threads: one CTA of FIN_THREADS = 512
// threads per group, thread (c, l) = (chain, lane) adds the group's slots l + 32 c + 512 m in order
// of m (exactly lane l's chain c of fin_groups), then warp q combines the chains of quantity q with
// fin_groups' pairwise tree and shuffle tree: bitwise the same group sums, ~16x the parallelism.
constexpr int FIN_THREADS = 512;
template <int NQ>
__device__ __forceinline__ void fin_group_par(const Geo& g, const double* __restrict__ slots, uint32_t r32, int gl,
                                              double* __restrict__ gsum) {
    constexpr int FC = 16;
    __shared__ double chain[NQ][FC][32];
    const int lane = threadIdx.x & 31, c = threadIdx.x >> 5;
    const int gi = g.g_lo + gl;
    const int64_t rb = (int64_t)gi * g.ny / g.G - g.j0, re = (int64_t)(gi + 1) * g.ny / g.G - g.j0;
    const int64_t L = (re - rb) * g.tiles;
    const int sw = g.quad ? 4 : 1;  // doubles per slot
    // a chain's slots are loaded FB at a time (independent loads in flight), then added in order
    constexpr int FB = 8;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        const double* src = slots + ((int64_t)q * g.nyl * g.tiles + rb * g.tiles) * sw;
        const bool f = (r32 >> q) & 1u;
        double ac = 0.0;
        for (int64_t e0 = lane + 32 * c; e0 < L; e0 += (int64_t)32 * FC * FB) {
            double v[FB];
#pragma unroll
            for (int u = 0; u < FB; ++u) {
                const int64_t e = e0 + (int64_t)32 * FC * u;
                if (e >= L) {
                    v[u] = 0.0;
                } else if (sw == 4) {  // k_stencil's CTA order over its four warps
                    const double4 h = *reinterpret_cast<const double4*>(src + 4 * e);
                    v[u] = ((h.x + h.y) + h.z) + h.w;
                } else {
                    v[u] = src[e];
                }
            }
#pragma unroll
            for (int u = 0; u < FB; ++u) {
                if (e0 + (int64_t)32 * FC * u < L) {
                    ac += v[u];
                    if (f) ac = (double)(float)ac;
                }
            }
        }
        chain[q][c][lane] = ac;
    }
    __syncthreads();
    if (c < NQ) {
        const int q = c;
        const bool f = (r32 >> q) & 1u;
        double ac[FC];
#pragma unroll
        for (int k = 0; k < FC; ++k) ac[k] = chain[q][k][lane];
#pragma unroll
        for (int h = FC / 2; h > 0; h >>= 1) {
#pragma unroll
            for (int k = 0; k < h; ++k) {
                ac[k] += ac[k + h];
                if (f) ac[k] = (double)(float)ac[k];
            }
        }
        double sv = ac[0];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            sv += __shfl_down_sync(0xffffffffu, sv, o);
            if (f) sv = (double)(float)sv;
        }
        if (lane == 0) {
            gsum[gl * NQ + q] = sv;
            __threadfence();  // visible device-wide before this CTA's arrival (k_fin's last-CTA logic)
        }
    }
}

template <int MODE, int WHICH>
__device__ __forceinline__ void fin_logic(const Geo& g, const double* __restrict__ gall, DevState* st,
                                          int first) {
    constexpr int NQ = fin_nq(WHICH);
    const uint32_t r32 = fin_r32<MODE>(WHICH);
    using V = typename Prec<MODE>::V;
    double tot[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        double t = 0.0;
        const bool f = (r32 >> q) & 1u;
        for (int gi = 0; gi < g.G; ++gi) {
            t += gall[gi * NQ + q];
            if (f) t = (double)(float)t;
        }
        tot[q] = t;
    }
    if (WHICH == W_VERIFY) {  // true residual of the current x only (A-6)
        const double rt = sqrt(tot[1]) / st->nb;
        st->true_R = rt;
        st->halt = !isfinite(rt) ? H_NONFINITE : (rt < st->tol ? H_START_CONVERGED : H_VERIFY_FAILED);
        return;
    }
    if (WHICH == W_START) {
        if (first) {
            double nb = sqrt(tot[0]);
            nb = rs<MODE>(nb);
            st->nb = nb;
            if (!(nb > 0.0) || !isfinite(nb)) { st->halt = nb == 0.0 ? H_DEGENERATE : H_NONFINITE; return; }
        }
        const double rt = sqrt(tot[1]) / st->nb;
        if (!isfinite(rt)) { st->halt = H_NONFINITE; return; }
        st->true_R = rt;
        if (first) { st->hist[0] = rt; st->final_R = rt; }
        st->rho = tot[2];  // rhat0 = r (A-1, A-11); eg_solve's rhat0 replaces it next (W_SHADOW)
        st->rh_norm = sqrt(tot[2]);
        st->rr0 = tot[2];
        st->beta = 0.0; st->beta_v = 0.0;
        st->omega = 1.0; st->omega_v = 1.0;
        st->fresh = 1;
        st->sexit = 0;
        st->last_start = st->iter;
        if (rt < st->tol) st->halt = H_START_CONVERGED;
        else if (st->iter >= st->maxit) st->halt = H_START_MAXIT;
        else if (rho_breakdown(st->rho, st->rh_norm, tot[2], st->eps_v)) st->halt = H_BD_ABORT;
        else st->halt = H_RUN;
        return;
    }
    if (st->halt != H_RUN) return;
    if (WHICH == W_SHADOW) {  // a caller-given rhat0 at the first start: rho = rhat0 . r
        st->rho = tot[0];
        st->rh_norm = sqrt(tot[1]);
        if (rho_breakdown(st->rho, st->rh_norm, st->rr0, st->eps_v) || !isfinite(st->rh_norm)) st->halt = H_BD_ABORT;
        return;
    }
    if (WHICH == W_A) {
        const double sigma = tot[0];
        if (sigma == 0.0 || !isfinite(sigma)) { st->halt = H_BD_ABORT; return; }
        const double alpha = rs<MODE>(st->rho / sigma);
        st->alpha = alpha;
        st->alpha_v = (double)(V)alpha;
    } else if (WHICH == W_B) {
        const double ts = tot[0], tt = tot[1], ss = tot[2];
        const double Rs = sqrt(ss) / st->nb;
        if (Rs < st->tol) { st->sexit = 1; st->Rs = Rs; return; }
        if (tt == 0.0 || !isfinite(tt) || !isfinite(ts)) { st->halt = H_BD_ABORT; return; }
        const double omega = rs<MODE>(ts / tt);
        st->omega = omega;
        st->omega_v = (double)(V)omega;
    } else {  // W_C
        const int it = st->iter + 1;
        st->iter = it;
        st->xzero = 0;  // the update has stored x
        if (st->sexit) {
            st->hist[it % HIST_CAP] = st->Rs;
            st->final_R = st->Rs;
            st->sexit = 0;
            st->halt = H_CONVERGED;
            return;
        }
        const double rho_n = tot[0], rr = tot[1];
        const double R = sqrt(rr) / st->nb;
        st->hist[it % HIST_CAP] = R;
        st->final_R = R;
        if (!isfinite(R)) { st->halt = H_NONFINITE; return; }
        if (R < st->tol) { st->halt = H_CONVERGED; return; }
        if (rho_breakdown(rho_n, st->rh_norm, rr, st->eps_v) || st->omega == 0.0) {
            st->halt = H_BD_END;
            return;
        }
        const double beta = rs<MODE>(rs<MODE>(rho_n / st->rho) * rs<MODE>(st->alpha / st->omega));
        st->beta = beta;
        st->beta_v = (double)(V)beta;
        st->rho = rho_n;
        st->fresh = 0;
        if (st->restart_every > 0 && it - st->last_start == st->restart_every) st->halt = H_RESTART;
        else if (it >= st->maxit) st->halt = H_MAXIT;
    }
}

// after reduction 2 (W_B): the control state the x half of a split update (k_update PART 2) runs on,
// which reduction 3 does not touch (it rewrites halt / sexit / xzero while that half may still run)
__device__ __forceinline__ void x_snapshot(DevState* st) {
    st->xs_run = st->halt == H_RUN;
    st->xs_sexit = st->sexit;
    st->xs_xzero = st->xzero;
}

// one-kernel finaliser: one CTA per (local) reduction group, the last CTA to finish runs the logic.
// One GPU: all G groups are local.  Latitude bands with the P2P transport (pp.on, NCCL ranks):
// every CTA also pushes its group's sums to every rank (p2p_push_group) and the last CTA waits for
// all G groups' words of this reduction (p2p_gather) before the logic — the all-gather inside the
// finaliser, one launch per reduction as on one GPU.
template <int WHICH> __device__ __forceinline__ bool fin_no_sums(const DevState* st);
template <int WHICH>
__device__ __forceinline__ void p2p_push_group(const Geo& g, const P2P& pp, const double* gsum, int gl, int seq);
template <int WHICH>
__device__ __forceinline__ bool p2p_gather(const Geo& g, const P2P& pp, int seq, double* gs);

template <int MODE, int WHICH>
__global__ void __launch_bounds__(FIN_THREADS) k_fin(Geo g, const double* __restrict__ slots, DevState* st,
                                                     double* __restrict__ gsum, int first, P2P pp) {
    constexpr int NQ = fin_nq(WHICH);
    const uint32_t r32 = fin_r32<MODE>(WHICH);
    pdl_wait();
    pdl_launch_dependents();  // the next kernel may launch (and wait) while this small grid runs
    // halt / sexit / epoch / gseq are read once, before this CTA's arrival: only the last CTA to
    // arrive (after every CTA has read them) writes the state, so every CTA takes the same branch
    // and stamps its pushes alike
    const int halt0 = *(volatile const int*)&st->halt;
    const int sexit0 = *(volatile const int*)&st->sexit;
    const int epoch = *(volatile const int*)&st->epoch;
    const int gseq = *(volatile const int*)&st->gseq;
    if (WHICH != W_START && WHICH != W_VERIFY && halt0 != H_RUN) {  // (then nobody writes but this)
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            st->epoch = epoch + 1;  // every finaliser launch bumps the epoch (stamps the next phase launch)
            if (WHICH == W_B) x_snapshot(st);
        }
        return;
    }
    // s-step exit (W_C): no sums needed, but every CTA still arrives so that the counter is reset
    const bool sums = !(WHICH == W_C && sexit0);
    if (sums) fin_group_par<NQ>(g, slots, r32, blockIdx.x, gsum);
    __shared__ int last;
    __shared__ double gs[8 * 3];
    __syncthreads();
    if (pp.on && sums) p2p_push_group<WHICH>(g, pp, gsum, blockIdx.x, gseq);
    if (threadIdx.x == 0) {
        __threadfence();  // this group's sums before the arrival
        last = atomicAdd(&st->fin_ctr, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    bool ok = true;
    if (pp.on && sums) ok = p2p_gather<WHICH>(g, pp, gseq, gs);
    if (threadIdx.x == 0) {
        __threadfence();
        st->fin_ctr = 0;
        st->epoch = epoch + 1;
        if (sums) st->gseq = gseq + 1;
        if (!ok) {
            st->halt = H_PEER_TIMEOUT;
        } else {
            fin_logic<MODE, WHICH>(g, pp.on && sums ? gs : gsum, st, first);
        }
        if (WHICH == W_B) x_snapshot(st);
    }
}

// The P2P all-gather of the group sums (pp.on): every fp64 sum travels as two 64-bit words
// ((seq + 1) << 32 | one 32-bit half) into every rank's gather buffer (its own included) at
// [seq & 1][global group][q][half], seq = DevState.gseq, the number of summing finalisers so far
// (the same on every rank, kept across solves).  No fence: an aligned 64-bit store is single-copy
// atomic, so a word whose stamp matches holds this reduction's half.  Two buffers, alternating
// strictly: a rank can run at most one reduction ahead of a slower one, because its next needs the
// slower rank's push of the current one, which that rank makes after consuming the previous one
// (DESIGN.md §7 P2P).  (A stamp per pushing reduction, not the epoch: halted finalisers bump the
// epoch without pushing, so epochs of consecutive pushes can share a parity.)
template <int WHICH>
__device__ __forceinline__ bool fin_no_sums(const DevState* st) {  // k_fin_groups' early exits
    return (WHICH != W_START && WHICH != W_VERIFY && st->halt != H_RUN) || (WHICH == W_C && st->sexit);
}
constexpr int P2P_GWORDS = 8 * 3 * 2;  // words per parity buffer: [group][q][half]
// after fin_group_par + __syncthreads: this CTA's group (local index gl) to every rank
template <int WHICH>
__device__ __forceinline__ void p2p_push_group(const Geo& g, const P2P& pp, const double* gsum, int gl, int seq) {
    constexpr int NQ = fin_nq(WHICH);
    const int t = threadIdx.x;
    if (t < pp.nranks * NQ * 2) {  // one word per thread: rank r, sum q, half h
        const int r = t / (NQ * 2), q = (t >> 1) % NQ, h = t & 1;
        const unsigned stamp = (unsigned)seq + 1u + (pp.fault ? 2u : 0u);  // fault injection: a wrong stamp
        const unsigned long long bits =
            (unsigned long long)__double_as_longlong(((volatile const double*)gsum)[gl * NQ + q]);
        const unsigned half = h ? (unsigned)(bits >> 32) : (unsigned)bits;
        st_relaxed_sys_u64(pp.gall[r] + ((unsigned)seq & 1u) * P2P_GWORDS + ((g.g_lo + gl) * 3 + q) * 2 + h,
                           ((unsigned long long)stamp << 32) | half);
    }
}
// all G groups' sums of reduction seq from this rank's gather buffer into gs[G * NQ] (shared), the
// words polled by the CTA's threads in parallel; false if one did not arrive within the timeout.
// Called by every thread of the CTA.
template <int WHICH>
__device__ __forceinline__ bool p2p_gather(const Geo& g, const P2P& pp, int seq, double* gs) {
    constexpr int NQ = fin_nq(WHICH);
    __shared__ unsigned gw[P2P_GWORDS];
    const unsigned long long* b = pp.gall[pp.rank] + ((unsigned)seq & 1u) * P2P_GWORDS;
    const unsigned stamp = (unsigned)seq + 1u;
    bool bad = false;
    for (int w = threadIdx.x; w < g.G * NQ * 2; w += blockDim.x) {
        const int gi = w / (NQ * 2), rem = w % (NQ * 2);
        const unsigned long long* src = b + (gi * 3 + (rem >> 1)) * 2 + (rem & 1);
        unsigned long long v = ld_relaxed_sys_u64(src);
        if ((unsigned)(v >> 32) != stamp) {
            const unsigned long long t0 = globaltimer_ns();
            while ((unsigned)((v = ld_relaxed_sys_u64(src)) >> 32) != stamp) {
                __nanosleep(100);
                if ((long long)(globaltimer_ns() - t0) > pp.timeout_ns) { bad = true; break; }
            }
        }
        gw[w] = (unsigned)v;
    }
    bad = __syncthreads_or(bad);
    if (threadIdx.x == 0 && !bad)
        for (int e = 0; e < g.G * NQ; ++e)
            gs[e] = __longlong_as_double((long long)(((unsigned long long)gw[2 * e + 1] << 32) | gw[2 * e]));
    __syncthreads();
    return !bad;
}

// two-kernel finaliser of the NCCL / loopback transports: local groups -> (ncclAllGather, or the
// loopback copies) -> logic; with the loopback P2P transport the group kernel pushes and the logic
// kernel gathers, a host barrier between them ordering every rank's pushes ahead of every wait on
// the one shared stream.  grid: one CTA per local group.
template <int MODE, int WHICH>
__global__ void __launch_bounds__(FIN_THREADS) k_fin_groups(Geo g, const double* __restrict__ slots,
                                                            const DevState* st, double* __restrict__ gsum, P2P pp) {
    constexpr int NQ = fin_nq(WHICH);
    const uint32_t r32 = fin_r32<MODE>(WHICH);
    if (fin_no_sums<WHICH>(st)) return;
    fin_group_par<NQ>(g, slots, r32, blockIdx.x, gsum);
    if (pp.on) {
        __syncthreads();
        p2p_push_group<WHICH>(g, pp, gsum, blockIdx.x, *(volatile const int*)&st->gseq);
    }
}

template <int MODE, int WHICH>
__global__ void k_fin_logic(Geo g, const double* __restrict__ gall, DevState* st, int first, P2P pp) {
    __shared__ double gs[8 * 3];
    const int epoch = *(volatile const int*)&st->epoch;
    const int gseq = *(volatile const int*)&st->gseq;
    const bool sums = !fin_no_sums<WHICH>(st);
    const bool p2p = pp.on && sums;
    const bool ok = p2p ? p2p_gather<WHICH>(g, pp, gseq, gs) : true;
    if (threadIdx.x == 0) {
        st->epoch = epoch + 1;
        if (sums) st->gseq = gseq + 1;
        if (!ok) {
            st->halt = H_PEER_TIMEOUT;
        } else {
            fin_logic<MODE, WHICH>(g, p2p ? gs : gall, st, first);
        }
        if (WHICH == W_B) x_snapshot(st);
    }
}

// ---------------------------------------------------------------------------------------------
// A caller-given shadow residual at the first start (eg_solve_params.rhat0; BiCGStab leaves r̂0 free,
// A-1 takes r̂0 = r0 by default): rhat0 = round_V(sh); partials rhat0 . r (S), rhat0 . rhat0 (S).
// Rare (a test / fault-injection hook), so a plain column walk.  grid (tiles, nyl), RW.
template <int MODE>
__global__ void __launch_bounds__(RW) k_shadow(Geo g, Vecs<MODE> vv, const double* __restrict__ sh) {
    using V = typename Prec<MODE>::V;
    double acc[2] = {0.0, 0.0};
    const int i = blockIdx.x * RW + threadIdx.x;
    if (i < g.nx) {
        const int64_t rb = (int64_t)blockIdx.y * g.row + i;
        for (int k = 0; k < (int)g.nz; ++k) {
            const int64_t q = rb + (int64_t)k * g.nx;
            const V h = (V)sh[q];
            vv.rh[q] = h;
            acc_dot<MODE>(acc[0], h, vv.r[q]);
            acc_dot<MODE>(acc[1], h, h);
        }
    }
    write_slots<2>(g, vv.slots, acc, fin_r32<MODE>(W_SHADOW));
}

template <class A, class B>
__global__ void k_convert(const A* __restrict__ src, B* __restrict__ dst, int64_t n) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x)
        dst[q] = (B)src[q];
}

}  // namespace eg
