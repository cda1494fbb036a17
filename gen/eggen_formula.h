/*
 * eggen_formula.h — the per-point draw shared by eggen_host.c and eggen_cuda.cu (generator-internal;
 * neither the solver nor the oracle includes this file).  See eggen.h for the recipe and citations.
 *
 * Every operation is an exact integer op or a single correctly-rounded IEEE double +,-,*,/,sqrt,
 * written through GEN_ADD / GEN_MUL / GEN_DIV / GEN_SQRT so that the device build can never
 * contract into an FMA.  That is what makes host and device bits identical.  The logarithm and
 * cosine of the Box-Muller draw are therefore evaluated here from those operations (series of a
 * fixed length), not by libm / CUDA's math library, whose last bits differ.
 */
#ifndef EGGEN_FORMULA_H
#define EGGEN_FORMULA_H
#include <stdint.h>

#if defined(__CUDACC__)
#define GEN_FN __host__ __device__ static inline
#if defined(__CUDA_ARCH__)
#define GEN_ADD(a, b) __dadd_rn((a), (b))
#define GEN_MUL(a, b) __dmul_rn((a), (b))
#define GEN_DIV(a, b) __ddiv_rn((a), (b))
#define GEN_SQRT(a) __dsqrt_rn(a)
#else
#include <math.h>
#define GEN_ADD(a, b) ((a) + (b))
#define GEN_MUL(a, b) ((a) * (b))
#define GEN_DIV(a, b) ((a) / (b))
#define GEN_SQRT(a) sqrt(a)
#endif
#else
#include <math.h>
#define GEN_FN static inline
#define GEN_ADD(a, b) ((a) + (b))
#define GEN_MUL(a, b) ((a) * (b))
#define GEN_DIV(a, b) ((a) / (b))
#define GEN_SQRT(a) sqrt(a)
#endif

/* SplitMix64 finaliser (Steele, Lea & Flood 2014 constants). */
GEN_FN uint64_t gen_mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* u(seed, s, q) = (mix(mix(seed*2^8 + s) ^ q) >> 11) * 2^-53  — exact, in [0,1). */
GEN_FN double gen_u(uint64_t seed, uint64_t s, uint64_t q) {
    uint64_t h = gen_mix(gen_mix(seed * 256ull + s) ^ q);
    return (double)(h >> 11) * 0x1.0p-53;
}

GEN_FN double gen_fabs(double a) { return a < 0.0 ? -a : a; }

/* ln x for 0 < x <= 1 (normal doubles): x = m 2^e exactly (bit fields), m in [sqrt(1/2), sqrt(2)),
 * ln x = e ln 2 + 2 atanh(t), t = (m - 1) / (m + 1), |t| < 0.172, atanh by 16 terms of its series
 * (the remainder is < 1e-26 relative).  Within a few ulp of the true value. */
GEN_FN double gen_log(double x) {
    union { double d; uint64_t u; } v;
    v.d = x;
    int64_t e = (int64_t)((v.u >> 52) & 0x7ff) - 1023;
    v.u = (v.u & 0x000fffffffffffffull) | 0x3ff0000000000000ull;  /* m in [1, 2) */
    double m = v.d;
    if (m > 1.4142135623730951) { m = GEN_MUL(m, 0.5); e += 1; }
    const double t = GEN_DIV(GEN_ADD(m, -1.0), GEN_ADD(m, 1.0));
    const double t2 = GEN_MUL(t, t);
    double sum = 0.0;
    for (int k = 15; k >= 0; --k) sum = GEN_ADD(GEN_DIV(1.0, (double)(2 * k + 1)), GEN_MUL(t2, sum));
    return GEN_ADD(GEN_MUL((double)e, 0.6931471805599453), GEN_MUL(2.0, GEN_MUL(t, sum)));
}

/* cos(2 pi u) for 0 <= u < 1: folded to w in [0, 1/4] (exact subtractions) with the sign, then the
 * Taylor series of cos(2 pi w) to theta^28 (the remainder at theta = pi/2 is < 1e-21). */
GEN_FN double gen_cos2pi(double u) {
    double w = u > 0.5 ? GEN_ADD(1.0, -u) : u;  /* cos(2 pi (1 - u)) = cos(2 pi u) */
    double sg = 1.0;
    if (w > 0.25) { w = GEN_ADD(0.5, -w); sg = -1.0; }  /* cos(2 pi (1/2 - w)) = -cos(2 pi w) */
    const double th = GEN_MUL(6.283185307179586, w);
    const double th2 = GEN_MUL(th, th);
    double sum = 1.0;
    for (int k = 14; k >= 1; --k)
        sum = GEN_ADD(1.0, GEN_MUL(GEN_DIV(-th2, (double)((2 * k - 1) * (2 * k))), sum));
    return GEN_MUL(sg, sum);
}

/* streams: 0 c_h, 1 c_v, 2 delta, 3-4 the two uniforms of b's Box-Muller draw */
enum { GEN_S_CH = 0, GEN_S_CV = 1, GEN_S_DL = 2, GEN_S_B0 = 3, GEN_S_B1 = 4 };

/* One point.  out: C,E,W,N,S,U,D,b. */
GEN_FN void gen_point(uint64_t seed, int64_t nx, int64_t ny, int64_t nz,
                      double ch_lo, double ch_w, double cv_lo, double cv_w,
                      double dl_lo, double dl_w, double cl_j,
                      int64_t i, int64_t j, int64_t k, double out[8]) {
    uint64_t q = (uint64_t)(i + nx * (k + nz * j));
    double ch = GEN_ADD(ch_lo, GEN_MUL(ch_w, gen_u(seed, GEN_S_CH, q)));
    double cv = GEN_ADD(cv_lo, GEN_MUL(cv_w, gen_u(seed, GEN_S_CV, q)));
    double dl = GEN_ADD(dl_lo, GEN_MUL(dl_w, gen_u(seed, GEN_S_DL, q)));
    double e = -GEN_MUL(ch, cl_j);
    double w = e;
    double n = (j < ny - 1) ? -ch : 0.0;
    double s = (j > 0) ? -ch : 0.0;
    double u = (k < nz - 1) ? -cv : 0.0;
    double d = (k > 0) ? -cv : 0.0;
    double sum = GEN_ADD(gen_fabs(e), gen_fabs(w));
    sum = GEN_ADD(sum, gen_fabs(n));
    sum = GEN_ADD(sum, gen_fabs(s));
    sum = GEN_ADD(sum, gen_fabs(u));
    sum = GEN_ADD(sum, gen_fabs(d));
    double c = GEN_MUL(sum, GEN_ADD(1.0, dl));
    /* b ~ N(0,1) by Box-Muller (BASELINE.json): sqrt(-2 ln(1 - u3)) cos(2 pi u4),
     * 1 - u3 in [2^-53, 1] */
    const double u3 = gen_u(seed, GEN_S_B0, q), u4 = gen_u(seed, GEN_S_B1, q);
    const double rad = GEN_SQRT(GEN_MUL(-2.0, gen_log(GEN_ADD(1.0, -u3))));
    out[0] = c; out[1] = e; out[2] = w; out[3] = n; out[4] = s; out[5] = u; out[6] = d;
    out[7] = GEN_MUL(rad, gen_cos2pi(u4));
}

#endif
