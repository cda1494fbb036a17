/*
 * oracle.c — plain, slow, obviously-correct CPU oracle.  TEST INFRASTRUCTURE ONLY (see oracle.h):
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg use it.
 *
 * Written from the paper (PAPER.md line numbers "P:L") and the readings in DESIGN.md; no blocking,
 * no fusion, no reordering beyond what the definitions state.  OpenMP only splits independent
 * latitude rows; every sum has one fixed order, so results do not depend on the thread count.
 */
#include "oracle.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int oracle_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ---- precision helpers (32-bit storage and arithmetic except x and the sums) ---- */

/* round to the working (vector) precision V */
static double rv(int mode, double a) { return mode == OR_FP64 ? a : (double)(float)a; }
/* round to the solution precision X: 64-bit in FP64 and MIXED ("the pressure field is kept as a
 * 64-bit data-type"), 32-bit in FP32 */
static double rx(int mode, double a) { return mode == OR_FP32 ? (double)(float)a : a; }
/* round to the global-sum precision S: 64-bit except FP32 ("reverted to 64-bit") */
static double rs(int mode, double a) { return mode == OR_FP32 ? (double)(float)a : a; }

/* ---- grid connectivity: 7-point stencil, periodic longitude, zero-flux lat / vertical ---- */

enum { E_ = 0, W_ = 1, N_ = 2, S_ = 3, U_ = 4, D_ = 5 };

/* neighbour of (i,j,k) in direction d; returns 0 when the neighbour is absent */
static int nbr(int64_t nx, int64_t ny, int64_t nz, int d, int64_t i, int64_t j, int64_t k,
               int64_t* q) {
    switch (d) {
        case E_: i = (i + 1) % nx; break;
        case W_: i = (i + nx - 1) % nx; break;
        case N_: if (j == ny - 1) return 0; j = j + 1; break;
        case S_: if (j == 0) return 0; j = j - 1; break;
        case U_: if (k == nz - 1) return 0; k = k + 1; break;
        case D_: if (k == 0) return 0; k = k - 1; break;
    }
    *q = i + nx * (k + nz * j);
    return 1;
}

/* ---- a1: diagonal scaling, Eq. 5 ---- */

int oracle_scale(int64_t nx, int64_t ny, int64_t nz, const double* bands7, int mode,
                 double* ahat6, double* diag) {
    if (nx < 3 || ny < 1 || nz < 1 || mode < 0 || mode > 2) return OR_ERR_ARG;
    const int64_t n = nx * ny * nz;
    for (int64_t j = 0; j < ny; ++j)
        for (int64_t k = 0; k < nz; ++k)
            for (int64_t i = 0; i < nx; ++i) {
                int64_t q = i + nx * (k + nz * j);
                double c = bands7[q];
                if (c == 0.0 || !isfinite(c)) return OR_ERR_SINGULAR_DIAG;
                diag[q] = c;
                for (int d = 0; d < 6; ++d) {
                    double a = bands7[(int64_t)(d + 1) * n + q];
                    int64_t qn;
                    if (!isfinite(a)) return OR_ERR_ARG;
                    if (!nbr(nx, ny, nz, d, i, j, k, &qn) && a != 0.0) return OR_ERR_ARG;
                    ahat6[(int64_t)d * n + q] = rv(mode, a / c);
                }
            }
    return OR_OK;
}

/* ---- (c1) the scaled operator ---- */

void oracle_apply(int64_t nx, int64_t ny, int64_t nz, const double* ahat6, const double* x,
                  double* y) {
    const int64_t n = nx * ny * nz;
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < ny; ++j)
        for (int64_t k = 0; k < nz; ++k)
            for (int64_t i = 0; i < nx; ++i) {
                int64_t q = i + nx * (k + nz * j), qn;
                double acc = x[q];                         /* unit diagonal of D_g^-1 A */
                for (int d = 0; d < 6; ++d)
                    if (nbr(nx, ny, nz, d, i, j, k, &qn)) acc = acc + ahat6[(int64_t)d * n + q] * x[qn];
                y[q] = acc;
            }
}

void oracle_apply_wp(int64_t nx, int64_t ny, int64_t nz, int mode, const double* ahat6,
                     const double* x, double* y) {
    const int64_t n = nx * ny * nz;
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < ny; ++j)
        for (int64_t k = 0; k < nz; ++k)
            for (int64_t i = 0; i < nx; ++i) {
                int64_t q = i + nx * (k + nz * j), qn;
                double acc = x[q];
                for (int d = 0; d < 6; ++d)
                    if (nbr(nx, ny, nz, d, i, j, k, &qn))
                        acc = rv(mode, acc + rv(mode, ahat6[(int64_t)d * n + q] * x[qn]));
                y[q] = acc;
            }
}

void oracle_residual64(int64_t nx, int64_t ny, int64_t nz, const double* ahat6, const double* bhat,
                       const double* x, double* r) {
    const int64_t n = nx * ny * nz;
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < ny; ++j)
        for (int64_t k = 0; k < nz; ++k)
            for (int64_t i = 0; i < nx; ++i) {
                int64_t q = i + nx * (k + nz * j), qn;
                double acc = x[q];
                for (int d = 0; d < 6; ++d)
                    if (nbr(nx, ny, nz, d, i, j, k, &qn)) acc = acc + ahat6[(int64_t)d * n + q] * x[qn];
                r[q] = bhat[q] - acc;
            }
}

/* ---- (c1) T^-1 per column: "the lower/upper-factorisation of the matrix T" ---- */

void oracle_thomas(int64_t nx, int64_t ny, int64_t nz, int mode, const double* ahat6,
                   const double* f, double* z) {
    const int64_t n = nx * ny * nz;
    const double* U = ahat6 + (int64_t)U_ * n;
    const double* D = ahat6 + (int64_t)D_ * n;
#pragma omp parallel
    {
        double* cp = (double*)malloc(sizeof(double) * (size_t)nz);
        double* y = (double*)malloc(sizeof(double) * (size_t)nz);
#pragma omp for schedule(static)
        for (int64_t j = 0; j < ny; ++j)
            for (int64_t i = 0; i < nx; ++i) {
#define Q(k) ((i) + nx * ((k) + nz * (j)))
                cp[0] = U[Q(0)];
                y[0] = f[Q(0)];
                for (int64_t k = 1; k < nz; ++k) {
                    double m = rv(mode, 1.0 - rv(mode, D[Q(k)] * cp[k - 1]));
                    cp[k] = rv(mode, U[Q(k)] / m);
                    y[k] = rv(mode, rv(mode, f[Q(k)] - rv(mode, D[Q(k)] * y[k - 1])) / m);
                }
                z[Q(nz - 1)] = y[nz - 1];
                for (int64_t k = nz - 2; k >= 0; --k)
                    z[Q(k)] = rv(mode, y[k] - rv(mode, cp[k] * z[Q(k + 1)]));
#undef Q
            }
        free(cp);
        free(y);
    }
}

/* ---- NEXT-1: tri-SOR, Eq. 7, red-black column ordering ---- */

int oracle_trisor(int64_t nx, int64_t ny, int64_t nz, int mode, const double* ahat6, const double* f,
                  int sweeps, double omega, const double* x_init, double* x) {
    if (nx < 3 || nx % 2 != 0 || sweeps < 0) return OR_ERR_ARG;
    const int64_t n = nx * ny * nz;
    const double* U = ahat6 + (int64_t)U_ * n;
    const double* D = ahat6 + (int64_t)D_ * n;
    for (int64_t q = 0; q < n; ++q) x[q] = x_init ? rv(mode, x_init[q]) : 0.0;
    double* rhs = (double*)malloc(sizeof(double) * (size_t)nz);
    double* cp = (double*)malloc(sizeof(double) * (size_t)nz);
    double* y = (double*)malloc(sizeof(double) * (size_t)nz);
    for (int sw = 0; sw < sweeps; ++sw)
        for (int colour = 0; colour < 2; ++colour)
            for (int64_t j = 0; j < ny; ++j)
                for (int64_t i = 0; i < nx; ++i) {
                    if ((i + j) % 2 != colour) continue;
#define Q(k) ((i) + nx * ((k) + nz * (j)))
                    /* rhs = (1 - omega) T x_old + omega (f - H x) */
                    for (int64_t k = 0; k < nz; ++k) {
                        double tx = x[Q(k)];
                        if (k + 1 < nz) tx = rv(mode, tx + rv(mode, U[Q(k)] * x[Q(k + 1)]));
                        if (k > 0) tx = rv(mode, tx + rv(mode, D[Q(k)] * x[Q(k - 1)]));
                        double hx = 0.0;
                        for (int d = E_; d <= S_; ++d) {
                            int64_t qn;
                            if (nbr(nx, ny, nz, d, i, j, k, &qn))
                                hx = rv(mode, hx + rv(mode, ahat6[(int64_t)d * n + Q(k)] * x[qn]));
                        }
                        rhs[k] = rv(mode, rv(mode, (1.0 - omega) * tx) + rv(mode, omega * rv(mode, f[Q(k)] - hx)));
                    }
                    /* x_col = T^-1 rhs (same recurrence as oracle_thomas) */
                    cp[0] = U[Q(0)];
                    y[0] = rhs[0];
                    for (int64_t k = 1; k < nz; ++k) {
                        double m = rv(mode, 1.0 - rv(mode, D[Q(k)] * cp[k - 1]));
                        cp[k] = rv(mode, U[Q(k)] / m);
                        y[k] = rv(mode, rv(mode, rhs[k] - rv(mode, D[Q(k)] * y[k - 1])) / m);
                    }
                    x[Q(nz - 1)] = y[nz - 1];
                    for (int64_t k = nz - 2; k >= 0; --k) x[Q(k)] = rv(mode, y[k] - rv(mode, cp[k] * x[Q(k + 1)]));
#undef Q
                }
    free(rhs);
    free(cp);
    free(y);
    return OR_OK;
}

/* ---- global sums ---- */

double oracle_dot(int64_t nx, int64_t ny, int64_t nz, int mode, const double* a, const double* b) {
    const int64_t row = nx * nz;
    double* part = (double*)malloc(sizeof(double) * (size_t)ny);
#pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < ny; ++j) {
        double s = 0.0;
        for (int64_t t = 0; t < row; ++t) s = rs(mode, s + rs(mode, a[j * row + t] * b[j * row + t]));
        part[j] = s;
    }
    double tot = 0.0;
    for (int64_t j = 0; j < ny; ++j) tot = rs(mode, tot + part[j]);
    free(part);
    return tot;
}

/* ---- BiCGStab, right-preconditioned ("post-conditioned") ---- */

int oracle_solve(int64_t nx, int64_t ny, int64_t nz, int mode, const double* ahat6,
                 const double* diag, const double* b, const double* x0, const oracle_params* prm,
                 double* x, double* hist, oracle_info* info) {
    const int64_t n = nx * ny * nz;
    oracle_info inf;
    memset(&inf, 0, sizeof inf);
    if (nx < 3 || ny < 1 || nz < 1 || mode < 0 || mode > 2 || !prm || prm->maxit < 0 ||
        (prm->sor_sweeps > 0 && nx % 2 != 0)) {
        inf.status = OR_ERR_ARG;
        if (info) *info = inf;
        return OR_ERR_ARG;
    }
    const double tol = prm->tol;
    const int maxit = prm->maxit;
    const double eps_v = (mode == OR_FP64) ? 0x1.0p-53 : 0x1.0p-24; /* reading A-12 */
    double* bhat = (double*)malloc(sizeof(double) * n);
    double* r64 = (double*)malloc(sizeof(double) * n);
    double* r = (double*)malloc(sizeof(double) * n);
    double* rh = (double*)malloc(sizeof(double) * n);
    double* p = (double*)malloc(sizeof(double) * n);
    double* v = (double*)malloc(sizeof(double) * n);
    double* s = (double*)malloc(sizeof(double) * n);
    double* t = (double*)malloc(sizeof(double) * n);
    double* z = (double*)malloc(sizeof(double) * n);
    double* zs = (double*)malloc(sizeof(double) * n);
    int status = OR_OK;
    if (!bhat || !r64 || !r || !rh || !p || !v || !s || !t || !z || !zs) {
        status = OR_ERR_NOMEM;
        goto out;
    }

    /* entry: bhat = D_g^-1 b, "performed outside the solver" */
    for (int64_t q = 0; q < n; ++q) bhat[q] = b[q] / diag[q];
    for (int64_t q = 0; q < n; ++q) r[q] = rv(mode, bhat[q]);
    double nb = sqrt(oracle_dot(nx, ny, nz, mode, mode == OR_FP32 ? r : bhat, mode == OR_FP32 ? r : bhat));
    nb = rs(mode, nb);
    if (!(nb > 0.0) || !isfinite(nb)) { status = nb == 0.0 ? OR_ERR_DEGENERATE_RHS : OR_ERR_NONFINITE; goto out; }
    for (int64_t q = 0; q < n; ++q) x[q] = x0 ? rx(mode, x0[q]) : 0.0;

    int i = 0;              /* completed iterations */
    int last_start = 0;     /* i at the last (re)start, for the mandatory restart (A-11) */
    int bd_at = -1;         /* completed-iteration count at the last breakdown (A-12) */
    int first = 1;
    int use_shadow = prm->shadow != 0;  /* the caller's rhat0 at the first start only */
    double rho = 0, alpha = 0, omega = 1, beta = 0, rh_norm = 0;
    int fresh = 1;

start:
    /* (re)start: r = round_V(bhat - Ahat x) with 64-bit accumulation (A-6, A-11) */
    oracle_residual64(nx, ny, nz, ahat6, bhat, x, r64);
    {
        double rt = sqrt(oracle_dot(nx, ny, nz, OR_FP64, r64, r64)) / nb;
        if (!isfinite(rt)) { status = OR_ERR_NONFINITE; goto done; }
        inf.true_R = rt;
        if (first) { hist[0] = rt; inf.final_R = rt; first = 0; }
        if (rt < tol) { inf.converged = 1; goto done; }
        if (i >= maxit) goto done;
    }
    for (int64_t q = 0; q < n; ++q) {
        r[q] = rv(mode, r64[q]);
        rh[q] = use_shadow ? rv(mode, prm->shadow[q]) : r[q];   /* rhat0 = r0 (A-1) unless given */
    }
    use_shadow = 0;
    rho = oracle_dot(nx, ny, nz, mode, rh, r);
    rh_norm = sqrt(oracle_dot(nx, ny, nz, mode, rh, rh));
    beta = 0.0;
    omega = 1.0;
    fresh = 1;              /* p = v = 0, so p_1 = r (A-11) */
    last_start = i;
    {   /* the breakdown test of rho (A-12) applies at a (re)start too: r orthogonal to rhat0 */
        const double rr0 = oracle_dot(nx, ny, nz, mode, r, r);
        if (rho == 0.0 || !isfinite(rho) || !isfinite(rh_norm) || fabs(rho) < eps_v * rh_norm * sqrt(rr0))
            goto breakdown;
    }

    while (i < maxit) {
        const int it = i + 1;
        /* p = r + beta (p - omega v) */
        if (fresh) {
            for (int64_t q = 0; q < n; ++q) p[q] = r[q];
        } else {
            const double bv = rv(mode, beta), ov = rv(mode, omega);
            for (int64_t q = 0; q < n; ++q)
                p[q] = rv(mode, r[q] + rv(mode, bv * rv(mode, p[q] - rv(mode, ov * v[q]))));
        }
        /* z = C^-1 p  (C^-1 = T^-1, reading A-3; or tri-SOR, NEXT-1), v = Ahat z */
        if (prm->sor_sweeps > 0) oracle_trisor(nx, ny, nz, mode, ahat6, p, prm->sor_sweeps, prm->sor_omega, 0, z);
        else oracle_thomas(nx, ny, nz, mode, ahat6, p, z);
        if (prm->precond_scale != 1.0)
            for (int64_t q = 0; q < n; ++q) z[q] = rv(mode, prm->precond_scale * z[q]);
        oracle_apply_wp(nx, ny, nz, mode, ahat6, z, v);
        double sigma = oracle_dot(nx, ny, nz, mode, rh, v);
        if (sigma == 0.0 || !isfinite(sigma)) goto breakdown;   /* P:537-541, A-12 */
        alpha = rs(mode, rho / sigma);
        {
            const double av = rv(mode, alpha);
            for (int64_t q = 0; q < n; ++q) s[q] = rv(mode, r[q] - rv(mode, av * v[q]));
        }
        if (prm->sor_sweeps > 0) oracle_trisor(nx, ny, nz, mode, ahat6, s, prm->sor_sweeps, prm->sor_omega, 0, zs);
        else oracle_thomas(nx, ny, nz, mode, ahat6, s, zs);
        if (prm->precond_scale != 1.0)
            for (int64_t q = 0; q < n; ++q) zs[q] = rv(mode, prm->precond_scale * zs[q]);
        oracle_apply_wp(nx, ny, nz, mode, ahat6, zs, t);
        double ss = oracle_dot(nx, ny, nz, mode, s, s);
        double ts = oracle_dot(nx, ny, nz, mode, t, s);
        double tt = oracle_dot(nx, ny, nz, mode, t, t);
        double Rs = sqrt(ss) / nb;
        if (Rs < tol) {                                          /* s-step exit (A-7) */
            for (int64_t q = 0; q < n; ++q) x[q] = rx(mode, x[q] + rx(mode, alpha * z[q]));
            i = it;
            hist[i] = Rs;
            inf.final_R = Rs;
            goto converged;
        }
        if (tt == 0.0 || !isfinite(tt) || !isfinite(ts)) goto breakdown;
        omega = rs(mode, ts / tt);
        /* x = x + alpha z + omega z_s in the solution precision (A-10: scalars unrounded) */
        for (int64_t q = 0; q < n; ++q)
            x[q] = rx(mode, rx(mode, x[q] + rx(mode, alpha * z[q])) + rx(mode, omega * zs[q]));
        {
            const double ov = rv(mode, omega);
            for (int64_t q = 0; q < n; ++q) r[q] = rv(mode, s[q] - rv(mode, ov * t[q]));
        }
        double rho_n = oracle_dot(nx, ny, nz, mode, rh, r);
        double rr = oracle_dot(nx, ny, nz, mode, r, r);
        i = it;
        hist[i] = sqrt(rr) / nb;                                 /* Eq. 9 */
        inf.final_R = hist[i];
        if (!isfinite(hist[i])) { status = OR_ERR_NONFINITE; goto done; }
        if (hist[i] < tol) goto converged;                       /* R < R_c */
        if (rho_n == 0.0 || !isfinite(rho_n) || fabs(rho_n) < eps_v * rh_norm * sqrt(rr) ||
            omega == 0.0)
            goto breakdown;
        beta = rs(mode, rs(mode, rho_n / rho) * rs(mode, alpha / omega));
        rho = rho_n;
        fresh = 0;
        bd_at = -1;
        if (prm->restart_every > 0 && i - last_start == prm->restart_every) {
            inf.restarts++;
            goto start;
        }
    }
    goto done;  /* maxit reached: true_R below */

breakdown:
    inf.breakdowns++;
    if (bd_at == i) { status = OR_ERR_BREAKDOWN; goto done; }   /* two in a row, no progress */
    bd_at = i;
    inf.restarts++;
    goto start;

converged:
    /* verify with the true residual (A-6); if it fails and iterations remain, restart */
    oracle_residual64(nx, ny, nz, ahat6, bhat, x, r64);
    inf.true_R = sqrt(oracle_dot(nx, ny, nz, OR_FP64, r64, r64)) / nb;
    if (inf.true_R < tol) { inf.converged = 1; goto done_nores; }
    if (i >= maxit) goto done_nores;
    inf.restarts++;
    goto start;

done:
    if (status == OR_OK && !inf.converged && i >= maxit && maxit > 0) {
        oracle_residual64(nx, ny, nz, ahat6, bhat, x, r64);
        inf.true_R = sqrt(oracle_dot(nx, ny, nz, OR_FP64, r64, r64)) / nb;
    }
done_nores:
    inf.iters = i;
out:
    inf.status = status;
    if (info) *info = inf;
    free(bhat); free(r64); free(r); free(rh); free(p); free(v); free(s); free(t); free(z); free(zs);
    return status;
}
