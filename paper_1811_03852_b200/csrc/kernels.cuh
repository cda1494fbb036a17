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
// Every reducing kernel writes one partial per (latitude row, column tile) slot; the finaliser sums
// slots in a fixed order inside 8 fixed latitude row-groups, then the groups in order, so sums are
// bitwise reproducible run to run and for any number of GPUs.
#pragma once
#include "common.cuh"

namespace eg {

struct Geo {
    int64_t nx, ny, nz;  // global grid
    int64_t row;         // nx*nz: one latitude row
    int64_t nyl;         // local rows
    int64_t j0;          // global index of local row 0
    int64_t n;           // nyl*row
    int tiles;           // column tiles of width RW per row (reduction slots per row)
    int G, g_lo, g_hi;   // reduction row-groups: all, and this rank's [g_lo, g_hi)
};

constexpr int RW = 128;  // columns per CTA of the row-tiled kernels (= threads per CTA)

template <int MODE>
struct Vecs {
    using V = typename Prec<MODE>::V;
    using X = typename Prec<MODE>::X;
    const V *E, *W, *N, *S, *U, *D;  // scaled bands (unit diagonal not stored)
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
                                            uint32_t r32) {
    __shared__ double sm[32 * NQ];
    block_sum_d<NQ>(acc, sm, r32);
    if (threadIdx.x == 0) {
        const int64_t per_q = g.nyl * g.tiles;
#pragma unroll
        for (int q = 0; q < NQ; ++q) slots[q * per_q + blockIdx.y * g.tiles + blockIdx.x] = acc[q];
    }
}

// product of two V values summed into an S accumulator held as double (exact product for fp32
// operands; FP32 mode rounds product and sum to binary32 like the oracle)
template <int MODE, class V>
__device__ __forceinline__ void acc_dot(double& acc, V a, V b) {
    if (MODE == 2) acc = rs<MODE>(acc + (double)(float)((double)a * (double)b));
    else acc += (double)a * (double)b;
}

// ---------------------------------------------------------------------------------------------
// a1: scale bands (Eq. 5).  grid (ceil(nx/256), nz, nyl), block 256.
struct Bands7 { const double* b[7]; };

template <class V>
__global__ void __launch_bounds__(256) k_scale(Geo g, Bands7 in, V* __restrict__ E, V* __restrict__ W,
                                               V* __restrict__ N, V* __restrict__ S,
                                               V* __restrict__ U, V* __restrict__ D,
                                               double* __restrict__ diag, int* __restrict__ err) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= g.nx) return;
    const int64_t k = blockIdx.y, jl = blockIdx.z, jg = g.j0 + jl;
    const int64_t q = jl * g.row + k * g.nx + i;
    const double c = in.b[0][q];
    int e = 0;
    if (c == 0.0 || !isfinite(c)) e |= 2;
    V* out[6] = {E, W, N, S, U, D};
    const bool present[6] = {true, true, jg < g.ny - 1, jg > 0, k < g.nz - 1, k > 0};
#pragma unroll
    for (int d = 0; d < 6; ++d) {
        const double a = in.b[d + 1][q];
        if (!isfinite(a) || (!present[d] && a != 0.0)) e |= 1;
        out[d][q] = (V)(a / c);  // IEEE binary64 division, then one rounding to V
    }
    diag[q] = c;
    if (e) atomicOr(err, e);
}

// ---------------------------------------------------------------------------------------------
// a2 / a11 (entry, restart, verification):  bhat = b / diag (entry only);
//   res = bhat - Ahat x with fp64 accumulation (bands promoted);  r = rhat0 = round_V(res)
// partials: q0 = ||bhat||^2 (entry), q1 = ||res||^2 (fp64, true residual), q2 = r . r (S)
// grid (tiles, nyl), block RW.
template <int MODE>
__global__ void __launch_bounds__(RW) k_start(Geo g, Vecs<MODE> vv, const double* __restrict__ b,
                                              int entry, int xzero) {
    using V = typename Prec<MODE>::V;
    using X = typename Prec<MODE>::X;
    const int64_t i = (int64_t)blockIdx.x * RW + threadIdx.x;
    const int64_t jl = blockIdx.y, jg = g.j0 + jl;
    double acc[3] = {0.0, 0.0, 0.0};
    if (i < g.nx) {
        const bool hasN = jg < g.ny - 1, hasS = jg > 0;
        const int64_t iE = (i + 1 == g.nx) ? 0 : i + 1, iW = (i == 0) ? g.nx - 1 : i - 1;
        const int64_t rb = jl * g.row;
        for (int64_t k = 0; k < g.nz; ++k) {
            const int64_t q = rb + k * g.nx + i;
            double bh;
            if (entry) {
                bh = b[q] / vv.diag[q];
                vv.bhat[q] = bh;
                if (MODE == 2) {
                    const double b32 = (double)(float)bh;
                    acc[0] = rs<MODE>(acc[0] + (double)(float)(b32 * b32));
                } else {
                    acc[0] += bh * bh;
                }
            } else {
                bh = vv.bhat[q];
            }
            double res;
            if (xzero) {
                res = bh;
                if (entry) vv.x[q] = (X)0;
            } else {
                const int64_t lk = k * g.nx;
                double ax = (double)vv.x[q];
                ax += (double)vv.E[q] * (double)vv.x[rb + lk + iE];
                ax += (double)vv.W[q] * (double)vv.x[rb + lk + iW];
                if (hasN) {
                    const double xn = (jl + 1 < g.nyl) ? (double)vv.x[q + g.row] : (double)vv.xg_hi[lk + i];
                    ax += (double)vv.N[q] * xn;
                }
                if (hasS) {
                    const double xs = (jl > 0) ? (double)vv.x[q - g.row] : (double)vv.xg_lo[lk + i];
                    ax += (double)vv.S[q] * xs;
                }
                if (k + 1 < g.nz) ax += (double)vv.U[q] * (double)vv.x[q + g.nx];
                if (k > 0) ax += (double)vv.D[q] * (double)vv.x[q - g.nx];
                res = bh - ax;
            }
            const V rv = (V)res;
            vv.r[q] = rv;
            vv.rh[q] = rv;
            acc[1] += res * res;
            acc_dot<MODE>(acc[2], rv, rv);
        }
    }
    write_slots<3>(g, vv.slots, acc, MODE == 2 ? 0x5u : 0x0u);
}

// ---------------------------------------------------------------------------------------------
// a3 / a6 / precondition: per-column Thomas solve fused with the vector update that
// produces its right-hand side.  KIND 0: f = fin;  1: p = r + beta (p - omega v), f = p;
// 2: s = r - alpha v, f = s.  The forward-elimination factors c'_k and y_k live in shared memory
// laid out [k][thread] (conflict-free).  grid (ceil(nx/blockDim), nyl), dynamic smem 2*nz*blockDim*V.
template <int MODE, int KIND>
__global__ void __launch_bounds__(128) k_thomas(Geo g, Vecs<MODE> vv,
                                                const typename Prec<MODE>::V* __restrict__ fin,
                                                typename Prec<MODE>::V* __restrict__ zout) {
    using V = typename Prec<MODE>::V;
    // levels loaded per batch; the next batch is in flight while the current one is eliminated
    // (one DRAM round trip per level otherwise makes the recurrence latency bound)
    constexpr int KB = sizeof(V) == 4 ? 8 : 4;
    extern __shared__ __align__(16) unsigned char smraw[];
    const int W = blockDim.x, tid = threadIdx.x;
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
    const int64_t i = (int64_t)blockIdx.x * W + tid;
    if (i >= g.nx) return;
    const int64_t base = (int64_t)blockIdx.y * g.row + i;
    const int64_t nx = g.nx;
    const int nz = (int)g.nz;
    const V* __restrict__ A0 = KIND == 0 ? fin : vv.r;
    const V* __restrict__ Pp = vv.p;
    const V* __restrict__ Vv = vv.v;
    const V* __restrict__ Uu = vv.U;
    const V* __restrict__ Dd = vv.D;
    V ca[KB], cp[KB], cv[KB], cu[KB], cd[KB];
    V na[KB], np[KB], nv[KB], nu[KB], nd[KB];
#pragma unroll
    for (int e = 0; e < KB; ++e) { ca[e] = cp[e] = cv[e] = cu[e] = cd[e] = (V)0; na[e] = np[e] = nv[e] = nu[e] = nd[e] = (V)0; }
    auto load = [&](int k0, V(&a)[KB], V(&p)[KB], V(&v)[KB], V(&u)[KB], V(&d)[KB]) {
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            const int k = k0 + e;
            if (k < nz) {
                const int64_t q = base + (int64_t)k * nx;
                a[e] = A0[q];
                if (KIND == 1 && !fresh) { p[e] = Pp[q]; v[e] = Vv[q]; }
                if (KIND == 2) v[e] = Vv[q];
                u[e] = Uu[q];
                d[e] = Dd[q];
            }
        }
    };
    load(0, ca, cp, cv, cu, cd);
    V cp_prev = 0, y_prev = 0;
    for (int k0 = 0; k0 < nz; k0 += KB) {
        if (k0 + KB < nz) load(k0 + KB, na, np, nv, nu, nd);
#pragma unroll
        for (int e = 0; e < KB; ++e) {
            const int k = k0 + e;
            if (k < nz) {
                const int64_t q = base + (int64_t)k * nx;
                V f;
                if (KIND == 0) {
                    f = ca[e];
                } else if (KIND == 1) {
                    f = fresh ? ca[e] : fma(beta, fma(-omega, cv[e], cp[e]), ca[e]);
                    vv.p[q] = f;
                } else {
                    f = fma(-alpha, cv[e], ca[e]);
                    vv.s[q] = f;
                }
                V c, y;
                if (k == 0) {
                    c = cu[e];
                    y = f;
                } else {
                    const V inv = rcp<V>(fma(-cd[e], cp_prev, (V)1));
                    c = cu[e] * inv;
                    y = fma(-cd[e], y_prev, f) * inv;
                }
                cps[k * W + tid] = c;
                ys[k * W + tid] = y;
                cp_prev = c;
                y_prev = y;
            }
        }
#pragma unroll
        for (int e = 0; e < KB; ++e) { ca[e] = na[e]; cp[e] = np[e]; cv[e] = nv[e]; cu[e] = nu[e]; cd[e] = nd[e]; }
    }
    V zn = y_prev;
    zout[base + (int64_t)(nz - 1) * nx] = zn;
#pragma unroll 4
    for (int k = nz - 2; k >= 0; --k) {
        zn = fma(-cps[k * W + tid], zn, ys[k * W + tid]);
        zout[base + (int64_t)k * nx] = zn;
    }
}

// ---------------------------------------------------------------------------------------------
// a4 / a7 / apply: y = Ahat z (unit diagonal + 6 bands; periodic i; absent neighbours skipped)
// DOTS 0: none;  1: sigma = aux . y (aux = rhat0);  2: t.s, t.t, s.s (aux = s).
// Thread per column walking k; z(k-1), z(k), z(k+1) carried in registers.  grid (tiles, nyl).
template <int MODE, int DOTS>
__global__ void __launch_bounds__(RW) k_stencil(Geo g, Vecs<MODE> vv,
                                                const typename Prec<MODE>::V* __restrict__ z,
                                                typename Prec<MODE>::V* __restrict__ y,
                                                const typename Prec<MODE>::V* __restrict__ aux) {
    using V = typename Prec<MODE>::V;
    if (DOTS != 0 && vv.st->halt != H_RUN) return;
    constexpr int NQ = DOTS == 2 ? 3 : 1;
    double acc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
    const int64_t i = (int64_t)blockIdx.x * RW + threadIdx.x;
    const int64_t jl = blockIdx.y, jg = g.j0 + jl;
    if (i < g.nx) {
        const bool hasN = jg < g.ny - 1, hasS = jg > 0;
        const int64_t nx = g.nx, row = g.row;
        const int nz = (int)g.nz;
        const int64_t iE = (i + 1 == nx) ? 0 : i + 1, iW = (i == 0) ? nx - 1 : i - 1;
        const int64_t rb = jl * row;
        V zm = 0, z0 = z[rb + i];
#pragma unroll 2
        for (int k = 0; k < nz; ++k) {
            const int64_t lk = rb + (int64_t)k * nx;
            const int64_t q = lk + i;
            const V zp = (k + 1 < nz) ? z[q + nx] : (V)0;
            V a = z0;
            a = fma(vv.E[q], z[lk + iE], a);
            a = fma(vv.W[q], z[lk + iW], a);
            if (hasN) a = fma(vv.N[q], z[q + row], a);
            if (hasS) a = fma(vv.S[q], z[q - row], a);
            if (k + 1 < nz) a = fma(vv.U[q], zp, a);
            if (k > 0) a = fma(vv.D[q], zm, a);
            y[q] = a;
            if (DOTS == 1) {
                acc_dot<MODE>(acc[0], aux[q], a);
            } else if (DOTS == 2) {
                const V sv = aux[q];
                acc_dot<MODE>(acc[0], a, sv);
                acc_dot<MODE>(acc[1], a, a);
                acc_dot<MODE>(acc[2], sv, sv);
            }
            zm = z0;
            z0 = zp;
        }
    }
    if (DOTS != 0) write_slots<NQ>(g, vv.slots, acc, MODE == 2 ? 0x7u : 0x0u);
}

// ---------------------------------------------------------------------------------------------
// a9: x += alpha z + omega z_s (X precision, scalars unrounded, A-10); r = s - omega t;
// partials rhat0 . r, r . r.  On an s-step exit only x += alpha z.  grid (tiles, nyl).
template <int MODE>
__global__ void __launch_bounds__(RW) k_update(Geo g, Vecs<MODE> vv) {
    using V = typename Prec<MODE>::V;
    using X = typename Prec<MODE>::X;
    const DevState* st = vv.st;
    if (st->halt != H_RUN) return;
    const bool sexit = st->sexit != 0;
    const X alpha = (X)st->alpha, omega = (X)st->omega;
    const V omega_v = (V)st->omega_v;
    double acc[2] = {0.0, 0.0};
    const int64_t i = (int64_t)blockIdx.x * RW + threadIdx.x;
    if (i < g.nx) {
        const int64_t base = (int64_t)blockIdx.y * g.row + i;
        const int nz = (int)g.nz;
        if (sexit) {
            for (int k = 0; k < nz; ++k) {
                const int64_t q = base + (int64_t)k * g.nx;
                vv.x[q] = fma(alpha, (X)vv.z[q], vv.x[q]);
            }
        } else {
#pragma unroll 4
            for (int k = 0; k < nz; ++k) {
                const int64_t q = base + (int64_t)k * g.nx;
                vv.x[q] = fma(omega, (X)vv.zs[q], fma(alpha, (X)vv.z[q], vv.x[q]));
                const V rq = fma(-omega_v, vv.t[q], vv.s[q]);
                vv.r[q] = rq;
                acc_dot<MODE>(acc[0], vv.rh[q], rq);
                acc_dot<MODE>(acc[1], rq, rq);
            }
        }
    }
    if (!sexit) write_slots<2>(g, vv.slots, acc, MODE == 2 ? 0x3u : 0x0u);
}

// ---------------------------------------------------------------------------------------------
// Finalisers.  fin_groups: warp w sums quantity (w % NQ) of local group (w / NQ): lanes take fixed
// contiguous chunks of the group's (row, tile) slots, then a fixed shuffle tree.
// fin_logic (thread 0): groups in order -> totals -> BiCGStab scalars and control flags.
enum Which { W_START = 0, W_A = 1, W_B = 2, W_C = 3 };

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
    const int64_t c = (L + 31) / 32, e0 = lane * c, e1 = min(L, e0 + c);
    double s = 0.0;
    for (int64_t e = e0; e < e1; ++e) {
        s += src[e];
        if (f) s = (double)(float)s;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_down_sync(0xffffffffu, s, o);
        if (f) s = (double)(float)s;
    }
    if (lane == 0) gsum[gl * NQ + qq] = s;
}

template <int MODE, int WHICH>
__device__ __forceinline__ void fin_logic(const Geo& g, const double* __restrict__ gall, DevState* st,
                                          int first) {
    constexpr int NQ = WHICH == W_A ? 1 : (WHICH == W_C ? 2 : 3);
    const uint32_t r32 = MODE == 2 ? (WHICH == W_START ? 0x5u : 0x7u) : 0x0u;
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
        st->rho = tot[2];
        st->rh_norm = sqrt(tot[2]);
        st->beta = 0.0; st->beta_v = 0.0;
        st->omega = 1.0; st->omega_v = 1.0;
        st->fresh = 1;
        st->sexit = 0;
        st->last_start = st->iter;
        if (rt < st->tol) st->halt = H_START_CONVERGED;
        else if (st->iter >= st->maxit) st->halt = H_START_MAXIT;
        else st->halt = H_RUN;
        return;
    }
    if (st->halt != H_RUN) return;
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
        if (rho_n == 0.0 || !isfinite(rho_n) || fabs(rho_n) < st->eps_v * st->rh_norm * sqrt(rr) ||
            st->omega == 0.0) {
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

// single-GPU finaliser: groups + logic in one CTA (1024 threads)
template <int MODE, int WHICH>
__global__ void __launch_bounds__(1024) k_fin(Geo g, const double* __restrict__ slots, DevState* st,
                                              double* __restrict__ gsum, int first) {
    constexpr int NQ = WHICH == W_A ? 1 : (WHICH == W_C ? 2 : 3);
    const uint32_t r32 = MODE == 2 ? (WHICH == W_START ? 0x5u : 0x7u) : 0x0u;
    if (WHICH != W_START && st->halt != H_RUN) return;
    if (WHICH == W_C && st->sexit) {  // s-step exit: no sums needed
        if (threadIdx.x == 0) fin_logic<MODE, WHICH>(g, gsum, st, first);
        return;
    }
    fin_groups<NQ>(g, slots, r32, gsum);
    __syncthreads();
    if (threadIdx.x == 0) fin_logic<MODE, WHICH>(g, gsum, st, first);
}

// multi-GPU: local groups -> (NCCL all-gather) -> logic
template <int MODE, int WHICH>
__global__ void __launch_bounds__(1024) k_fin_groups(Geo g, const double* __restrict__ slots,
                                                     const DevState* st, double* __restrict__ gsum) {
    constexpr int NQ = WHICH == W_A ? 1 : (WHICH == W_C ? 2 : 3);
    const uint32_t r32 = MODE == 2 ? (WHICH == W_START ? 0x5u : 0x7u) : 0x0u;
    if (WHICH != W_START && st->halt != H_RUN) return;
    if (WHICH == W_C && st->sexit) return;
    fin_groups<NQ>(g, slots, r32, gsum);
}

template <int MODE, int WHICH>
__global__ void k_fin_logic(Geo g, const double* __restrict__ gall, DevState* st, int first) {
    if (threadIdx.x == 0) fin_logic<MODE, WHICH>(g, gall, st, first);
}

// ---------------------------------------------------------------------------------------------
template <class A, class B>
__global__ void k_convert(const A* __restrict__ src, B* __restrict__ dst, int64_t n) {
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n;
         q += (int64_t)gridDim.x * blockDim.x)
        dst[q] = (B)src[q];
}

}  // namespace eg
