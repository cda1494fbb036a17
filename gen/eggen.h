/*
 * eggen.h — seeded synthetic ENDGame-shaped Helmholtz problems (test/bench INPUT GENERATOR).
 *
 * This module is the one thing the CUDA path (paper_1811_03852_b200/) and the CPU oracle
 * (oracle/) both consume.  It holds NONE of the solver's arithmetic: no diagonal scaling, no
 * stencil application, no tridiagonal solve, no Krylov step.  It only draws coefficients and a
 * right-hand side from a counter-based hash, following BASELINE.json's config recipe:
 *
 *   "A is a 7-point variable-coefficient stencil ... Horizontal off-diagonals are -c_h*cos(lat)
 *    in E/W and -c_h in N/S, with c_h ~ U(0.5,1.5) per point. Vertical off-diagonals are -c_v
 *    with c_v ~ U(5,50) per point. diag = (sum of |off-diagonals|)*(1+delta), delta ~
 *    U(0.01,0.1). b ~ N(0,1), x0 = 0"                                         (BASELINE.json)
 *
 * which stands in for the paper's UM Helmholtz matrix: "7-band structure similar to ... the
 * Laplacian", "non-symmetric and ... not constant coefficient", vertical
 * coupling much stronger than horizontal.  DESIGN.md §"Input recipe" states
 * every reading taken here (cell-centred latitudes, one c_h/c_v per point for both directions,
 * zeros at absent neighbours, b by Box-Muller with a portable logarithm and cosine).
 *
 * Layout of every field ("IKJ", longitude fastest):  q = i + nx*(k + nz*j)
 *   i in [0,nx)  longitude, periodic;  k in [0,nz) level;  j in [0,ny) latitude.
 * Band order: 0=C (centre/diagonal), 1=E (i+1), 2=W (i-1), 3=N (j+1), 4=S (j-1), 5=U (k+1), 6=D (k-1).
 *
 * Bitwise contract: eggen_host and eggen_device produce IDENTICAL bits for identical params,
 * because every value is built from exact integer hashing plus correctly rounded IEEE
 * +,-,*,/,sqrt (no fused multiply-add on either side; ln and cos from fixed-length series of those)
 * and one host-computed cos(lat) table.
 */
#ifndef EGGEN_H
#define EGGEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    int64_t nx, ny, nz;       /* global grid */
    uint64_t seed;            /* BASELINE.json configs use seeds 0..4 */
    double ch_lo, ch_hi;      /* c_h ~ U(ch_lo, ch_hi) */
    double cv_lo, cv_hi;      /* c_v ~ U(cv_lo, cv_hi) */
    double dl_lo, dl_hi;      /* delta ~ U(dl_lo, dl_hi) */
} eggen_params;

/* Fill BASELINE.json's default ranges: c_h U(0.5,1.5), c_v U(5,50), delta U(0.01,0.1). */
void eggen_default_params(eggen_params* p, int64_t nx, int64_t ny, int64_t nz, uint64_t seed);

/* cos(lat_j), lat_j = -pi/2 + (j+1/2)*pi/ny (cell centres; > 0 at the poles). Host libm. */
void eggen_coslat(int64_t ny, double* out);

/* SplitMix64 finaliser and the uniform draw u(seed, stream, q) in [0,1), exposed for tests. */
uint64_t eggen_mix(uint64_t z);
double eggen_uniform(uint64_t seed, uint64_t stream, uint64_t q);

/* One grid point: out[0..6] = C,E,W,N,S,U,D and out[7] = b at global (i,j,k). */
void eggen_point(const eggen_params* p, const double* coslat, int64_t i, int64_t j, int64_t k,
                 double out[8]);

/* Rows [j_begin, j_end) of the global grid, host memory.  bands = 7 consecutive arrays of
 * n_loc = (j_end-j_begin)*nx*nz doubles (band d at bands + d*n_loc); b = n_loc doubles (may be NULL).
 * Returns 0, or -1 on bad arguments.  OpenMP over rows (counter-based, so thread-count independent). */
int eggen_host(const eggen_params* p, int64_t j_begin, int64_t j_end, double* bands, double* b);

/* Same rows generated on the current CUDA device into device memory, stream-ordered on `stream`
 * (a cudaStream_t, NULL = legacy default).  Returns 0, -1 bad args, -2 CUDA error. */
int eggen_device(const eggen_params* p, int64_t j_begin, int64_t j_end, double* bands, double* b,
                 void* stream);

#ifdef __cplusplus
}
#endif
#endif
