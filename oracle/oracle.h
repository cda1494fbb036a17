/*
 * oracle.h — CPU ORACLE of the hot path of Maynard & Walters, "Precision of the ENDGame:
 * Mixed-precision arithmetic in the iterative solver of the Unified Model" (arXiv 1811.03852).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load, call or link anything under oracle/.  The product path
 * (paper_1811_03852_b200/) never does, and the two share no code, header, table or helper.
 *
 * Citations "P:L" are lines of PAPER.md (the paper's LaTeX); "§8(c)" is SURVEY.md's reading table,
 * restated in DESIGN.md §Readings.
 *
 * Every field uses the generator's layout q = i + nx*(k + nz*j) (longitude fastest, then level,
 * then latitude); longitude is periodic, latitude and vertical are zero-flux (absent neighbours).
 * Scaled band order in ahat6: 0=E (i+1), 1=W (i-1), 2=N (j+1), 3=S (j-1), 4=U (k+1), 5=D (k-1).
 *
 * Precision modes:
 *   OR_FP64  = 0  everything 64-bit ("DP", Table 1)
 *   OR_MIXED = 1  x 64-bit; bands, Krylov vectors and their arithmetic 32-bit; global sums 64-bit
 *   OR_FP32  = 2  everything 32-bit incl. global sums (the "original" MP solver / toy-model SP)
 * All values are carried in C doubles; "rounded to working precision" = (double)(float)v, applied
 * after every single +,-,*,/ — this reproduces IEEE binary32 arithmetic exactly, because binary64
 * has more than 2*24+2 significand bits (no double-rounding error for one basic operation).
 * Built with -ffp-contract=off: no fused multiply-add anywhere.
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py (dense numpy / scipy
 * solves, closed forms, special cases, invariants); see DESIGN.md §Oracle pins.
 */
#ifndef EG_ORACLE_H
#define EG_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum { OR_FP64 = 0, OR_MIXED = 1, OR_FP32 = 2 };
enum {
    OR_OK = 0,
    OR_ERR_ARG = 1,
    OR_ERR_SINGULAR_DIAG = 2,
    OR_ERR_DEGENERATE_RHS = 3,
    OR_ERR_BREAKDOWN = 4,
    OR_ERR_NONFINITE = 5,
    OR_ERR_NOMEM = 6
};

/* a1 — diagonal scaling "outside the solver" (Eq. 5): ahat_d = a_d / a_C (IEEE
 * binary64 division) rounded to working precision; diag = a_C kept in binary64.
 * bands7 = 7 consecutive arrays C,E,W,N,S,U,D of n = nx*ny*nz.  ahat6 = 6 arrays E..D.
 * Errors: OR_ERR_SINGULAR_DIAG if some a_C is 0 or non-finite; OR_ERR_ARG if a band is nonzero at
 * an absent neighbour or the grid is invalid (nx < 3). */
int oracle_scale(int64_t nx, int64_t ny, int64_t nz, const double* bands7, int mode,
                 double* ahat6, double* diag);

/* (c1) apply: y_q = x_q + sum_d ahat_d(q) * x_nbr_d(q), absent neighbours contribute 0,
 * evaluated in binary64 in the order x, E, W, N, S, U, D. */
void oracle_apply(int64_t nx, int64_t ny, int64_t nz, const double* ahat6, const double* x,
                  double* y);

/* same sum, every operation rounded to the working precision of `mode` (the solver's matvec). */
void oracle_apply_wp(int64_t nx, int64_t ny, int64_t nz, int mode, const double* ahat6,
                     const double* x, double* y);

/* (c1) precondition: z = T^{-1} f per column (i,j), T = tridiag(D_k, 1, U_k) from ahat6's U/D
 * bands, by the Thomas recurrence without pivoting, every operation rounded to the
 * working precision of `mode`:
 *   c'_0 = U_0, y_0 = f_0;  k>=1: m = 1 - D_k c'_{k-1}; c'_k = U_k/m; y_k = (f_k - D_k y_{k-1})/m
 *   z_{nz-1} = y_{nz-1};    k = nz-2..0: z_k = y_k - c'_k z_{k+1}                          */
void oracle_thomas(int64_t nx, int64_t ny, int64_t nz, int mode, const double* ahat6,
                   const double* f, double* z);

/* NEXT-1: tri-SOR preconditioner (Eq. 7) in red-black column ordering:
 *   (T + omega L) x_n = (1 - omega) T x_{n-1} + omega (f - U x_{n-1}),   Ahat = L + T + U (Eq. 6)
 * Columns (i, j) are coloured (i + j) % 2 (red = 0 first, then black = 1; nx must be even so the
 * periodic seam keeps the colouring).  For every column of the current colour, in place:
 *   rhs_k = (1 - omega) (T x)_k + omega (f_k - sum_{E,W,N,S} ahat_h x_nbr)   (current neighbours)
 *   x_col = T^-1 rhs                                                        (Thomas, as above)
 * i.e. L couples a column to already-updated neighbours and U to not-yet-updated ones (reading
 * DESIGN.md NEXT-1).  x starts from x_init (NULL = 0: the fixed linear preconditioner of BiCGStab).
 * Every operation rounded to the working precision of `mode`.  Returns OR_ERR_ARG for odd nx. */
int oracle_trisor(int64_t nx, int64_t ny, int64_t nz, int mode, const double* ahat6, const double* f,
                  int sweeps, double omega, const double* x_init, double* x);

/* r = bhat - Ahat x in binary64 (bands promoted), the restart / verification residual. */
void oracle_residual64(int64_t nx, int64_t ny, int64_t nz, const double* ahat6, const double* bhat,
                       const double* x, double* r);

/* Global sum of a_q*b_q "local summation performed first": per latitude row j a
 * sequential sum in q order, then the row sums in j order.  Accumulated in binary64 for
 * OR_FP64/OR_MIXED (products of binary32 operands are exact in binary64), in binary32 for OR_FP32. */
double oracle_dot(int64_t nx, int64_t ny, int64_t nz, int mode, const double* a, const double* b);

typedef struct {
    double tol;            /* R_c; 0 = run exactly maxit iterations   */
    int32_t maxit;
    int32_t restart_every; /* mandatory restart period, 150 in the UM; <=0 off */
    double precond_scale;  /* test hook: M^-1 -> precond_scale * T^-1 (A-3); 1 */
    int32_t sor_sweeps;    /* 0: M^-1 = T^-1 (hot path, A-3); > 0: tri-SOR with this many sweeps */
    double sor_omega;      /* tri-SOR over-relaxation (1.5 in the UM) */
    const double* shadow;  /* NULL: rhat0 = r0 (reading A-1).  Else rhat0 = round_V(shadow) at the
                              FIRST start only (BiCGStab leaves rhat0 free; restarts use r, A-11) */
} oracle_params;

typedef struct {
    int32_t iters, converged, restarts, breakdowns, status;
    double final_R, true_R;
} oracle_info;

/* Right-("post-")preconditioned BiCGStab on Ahat x = bhat with M^-1 = T^-1, following the
 * step-by-step reading in DESIGN.md §Oracle algorithm, P:230-288, P:337-348,
 * P:537-557.  At every (re)start, rho = rhat0 . r is put to the same breakdown test as after an
 * iteration (A-12: 0, non-finite, or |rho| < eps_V ||rhat0|| ||r||, "scalar weights ... close to or
 * equal to zero"); a breakdown there restarts (with rhat0 = r) like any other.
 * b, x0 (may be NULL = 0) and x are binary64 arrays of n.  hist has >= maxit+1
 * entries: hist[0] = true relative residual of x0, hist[i] = R after iteration i.
 * Returns an OR_* status (also in info->status). */
int oracle_solve(int64_t nx, int64_t ny, int64_t nz, int mode, const double* ahat6,
                 const double* diag, const double* b, const double* x0, const oracle_params* prm,
                 double* x, double* hist, oracle_info* info);

/* Number of OpenMP threads the oracle will use (1 when built without OpenMP). */
int oracle_threads(void);

#ifdef __cplusplus
}
#endif
#endif
