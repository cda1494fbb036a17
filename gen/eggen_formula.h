/*
 * eggen_formula.h — the per-point draw shared by eggen_host.c and eggen_cuda.cu (generator-internal;
 * neither the solver nor the oracle includes this file).  See eggen.h for the recipe and citations.
 *
 * Every operation is an exact integer op or a single correctly-rounded IEEE double +,-,*, written
 * through GEN_ADD / GEN_MUL so that the device build can never contract into an FMA.  That is
 * what makes host and device bits identical.
 */
#ifndef EGGEN_FORMULA_H
#define EGGEN_FORMULA_H
#include <stdint.h>

#if defined(__CUDACC__)
#define GEN_FN __host__ __device__ static inline
#if defined(__CUDA_ARCH__)
#define GEN_ADD(a, b) __dadd_rn((a), (b))
#define GEN_MUL(a, b) __dmul_rn((a), (b))
#else
#define GEN_ADD(a, b) ((a) + (b))
#define GEN_MUL(a, b) ((a) * (b))
#endif
#else
#define GEN_FN static inline
#define GEN_ADD(a, b) ((a) + (b))
#define GEN_MUL(a, b) ((a) * (b))
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

/* streams: 0 c_h, 1 c_v, 2 delta, 3..14 the twelve uniforms of b */
enum { GEN_S_CH = 0, GEN_S_CV = 1, GEN_S_DL = 2, GEN_S_B0 = 3, GEN_NB = 12 };

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
    /* b ~ Irwin-Hall(12) - 6: mean 0, variance 1 (stand-in for N(0,1)) */
    double acc = 0.0;
    for (int m = 0; m < GEN_NB; ++m) acc = GEN_ADD(acc, gen_u(seed, GEN_S_B0 + m, q));
    out[0] = c; out[1] = e; out[2] = w; out[3] = n; out[4] = s; out[5] = u; out[6] = d;
    out[7] = GEN_ADD(acc, -6.0);
}

#endif
