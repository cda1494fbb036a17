/* eggen_host.c — host side of the seeded problem generator (see eggen.h). */
#include "eggen.h"
#include "eggen_formula.h"
#include <math.h>
#include <stddef.h>
#include <stdlib.h>

void eggen_default_params(eggen_params* p, int64_t nx, int64_t ny, int64_t nz, uint64_t seed) {
    p->nx = nx; p->ny = ny; p->nz = nz; p->seed = seed;
    p->ch_lo = 0.5;  p->ch_hi = 1.5;
    p->cv_lo = 5.0;  p->cv_hi = 50.0;
    p->dl_lo = 0.01; p->dl_hi = 0.1;
}

void eggen_coslat(int64_t ny, double* out) {
    const double pi = 3.14159265358979323846;
    for (int64_t j = 0; j < ny; ++j) out[j] = cos(-pi / 2.0 + ((double)j + 0.5) * pi / (double)ny);
}

uint64_t eggen_mix(uint64_t z) { return gen_mix(z); }
double eggen_uniform(uint64_t seed, uint64_t stream, uint64_t q) { return gen_u(seed, stream, q); }

void eggen_point(const eggen_params* p, const double* coslat, int64_t i, int64_t j, int64_t k,
                 double out[8]) {
    gen_point(p->seed, p->nx, p->ny, p->nz, p->ch_lo, p->ch_hi - p->ch_lo, p->cv_lo,
              p->cv_hi - p->cv_lo, p->dl_lo, p->dl_hi - p->dl_lo, coslat[j], i, j, k, out);
}

int eggen_host(const eggen_params* p, int64_t j_begin, int64_t j_end, double* bands, double* b) {
    if (!p || !bands || p->nx < 1 || p->ny < 1 || p->nz < 1 || j_begin < 0 || j_end > p->ny ||
        j_begin > j_end)
        return -1;
    const int64_t nx = p->nx, nz = p->nz, row = nx * nz;
    const int64_t nloc = (j_end - j_begin) * row;
    double* cl = (double*)malloc(sizeof(double) * (size_t)p->ny);
    if (!cl) return -1;
    eggen_coslat(p->ny, cl);
#pragma omp parallel for schedule(static)
    for (int64_t j = j_begin; j < j_end; ++j) {
        for (int64_t k = 0; k < nz; ++k) {
            for (int64_t i = 0; i < nx; ++i) {
                double v[8];
                eggen_point(p, cl, i, j, k, v);
                int64_t q = i + nx * k + row * (j - j_begin);
                for (int d = 0; d < 7; ++d) bands[(int64_t)d * nloc + q] = v[d];
                if (b) b[q] = v[7];
            }
        }
    }
    free(cl);
    return 0;
}
