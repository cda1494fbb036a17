"""Pins of the oracle's BiCGStab: direct solves, special cases, exact
metamorphic identities, the M-matrix spectral bound, and the paper's MP-vs-DP observations."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

import gen
import oracle
from _dense import dense_Ahat, dense_T, sparse_from_bands
from _golden import paper_observations

OBS = paper_observations()


def _setup(prob, mode):
    g = (prob.nx, prob.ny, prob.nz)
    bands, b = gen.host(prob)
    ahat, diag = oracle.scale(g, bands, mode)
    return g, bands, b, ahat, diag


def _sigfig_agree(a, b, k):
    return abs(a - b) <= 5.0 * 10.0 ** (-k) * abs(b)


# ---------------- against direct solves ----------------

@pytest.mark.parametrize("prob", [gen.Problem(4, 3, 2, seed=21), gen.Problem(8, 6, 4, seed=22),
                                  gen.Problem(16, 12, 6, seed=23)])
def test_fp64_solve_matches_numpy_dense(prob):
    g, bands, b, ahat, diag = _setup(prob, "fp64")
    x, hist, info = oracle.solve(g, "fp64", ahat, diag, b, tol=1e-12, maxit=200)
    assert info.status == 0 and info.converged and info.true_R < 1e-12
    A = sparse_from_bands(g, bands[0], bands[1:]).toarray()
    xd = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xd) <= 1e-9 * np.linalg.norm(xd)


def test_fp64_solve_matches_scipy_superlu_C1():
    prob = gen.CONFIGS["C1"]
    g, bands, b, ahat, diag = _setup(prob, "fp64")
    x, hist, info = oracle.solve(g, "fp64", ahat, diag, b, tol=1e-12, maxit=200)
    assert info.converged and info.true_R < 1e-12
    A = sparse_from_bands(g, bands[0], bands[1:]).tocsc()
    xd = spla.spsolve(A, b)
    assert np.linalg.norm(x - xd) <= 1e-9 * np.linalg.norm(xd)
    # the unscaled residual too (reading A-5)
    assert np.linalg.norm(b - A @ x) <= 1e-11 * np.linalg.norm(b)


@pytest.mark.parametrize("mode,tol", [("mixed", 1e-4), ("fp64", 1e-4), ("fp32", 1e-4)])
def test_tol_solve_accuracy_C1(mode, tol):
    prob = gen.CONFIGS["C1"]
    g, bands, b, ahat, diag = _setup(prob, mode)
    x, hist, info = oracle.solve(g, mode, ahat, diag, b, tol=tol, maxit=200)
    assert info.converged and info.true_R < tol and hist[-1] < tol
    assert np.all(hist[:-1] >= tol)                 # stops at the first iterate below R_c
    A = sparse_from_bands(g, bands[0], bands[1:]).tocsc()
    xd = spla.spsolve(A, b)
    # error bounded by cond-ish * tol; generous 10*tol reading of BASELINE.json's bar
    assert np.linalg.norm(x - xd) <= 10 * tol * np.linalg.norm(xd)


# ---------------- special cases ----------------

@pytest.mark.parametrize("mode,rt", [("fp64", 1e-14), ("mixed", 1e-5)])
def test_no_horizontal_coupling_converges_in_one_iteration(mode, rt):
    """c_h = 0: Ahat = T so M^-1 Ahat = I; alpha = 1 and the s-step exits at iteration 1 with
    x = T^-1 bhat."""
    prob = gen.Problem(12, 8, 10, seed=5, ch=(0.0, 0.0))
    g, bands, b, ahat, diag = _setup(prob, mode)
    x, hist, info = oracle.solve(g, mode, ahat, diag, b, tol=1e-4, maxit=50)
    assert info.converged and info.iters == 1
    a64, _ = oracle.scale(g, bands, "fp64")
    xd = np.linalg.solve(dense_T(g, a64), b / diag)
    assert np.linalg.norm(x - xd) <= rt * np.linalg.norm(xd)


def test_exact_initial_guess_needs_zero_iterations():
    prob = gen.Problem(16, 12, 6, seed=24)
    g, bands, b, ahat, diag = _setup(prob, "fp64")
    xd = spla.spsolve(sparse_from_bands(g, bands[0], bands[1:]).tocsc(), b)
    x, hist, info = oracle.solve(g, "fp64", ahat, diag, b, x0=xd, tol=1e-6, maxit=50)
    assert info.converged and info.iters == 0 and len(hist) == 1 and hist[0] < 1e-6
    assert np.array_equal(x, xd)


def test_degenerate_and_nonfinite_rhs():
    prob = gen.Problem(8, 6, 4, seed=25)
    g, bands, b, ahat, diag = _setup(prob, "mixed")
    _, _, info = oracle.solve(g, "mixed", ahat, diag, np.zeros_like(b))
    assert info.status == 3                              # DEGENERATE_RHS
    bb = b.copy(); bb[3] = np.nan
    _, _, info = oracle.solve(g, "mixed", ahat, diag, bb)
    assert info.status == 5                              # NONFINITE


# ---------------- exact (bitwise) metamorphic identities ----------------

@pytest.mark.parametrize("mode", ["fp64", "mixed", "fp32"])
def test_power_of_two_rhs_scaling_is_exact(mode):
    prob = gen.Problem(16, 12, 10, seed=26)
    g, bands, b, ahat, diag = _setup(prob, mode)
    x1, h1, i1 = oracle.solve(g, mode, ahat, diag, b, tol=1e-5, maxit=100)
    x2, h2, i2 = oracle.solve(g, mode, ahat, diag, 8.0 * b, tol=1e-5, maxit=100)
    assert i1.iters == i2.iters and np.array_equal(h1, h2) and np.array_equal(8.0 * x1, x2)


@pytest.mark.parametrize("mode", ["fp64", "mixed"])
def test_row_scaling_of_A_and_b_is_invisible(mode):
    """D_g^-1 scaling "outside the solver": multiplying row q of A and b_q by 2^k
    leaves Ahat and bhat, hence everything, bitwise unchanged."""
    prob = gen.Problem(16, 12, 10, seed=27)
    g, bands, b, ahat, diag = _setup(prob, mode)
    rng = np.random.default_rng(0)
    f = 2.0 ** rng.integers(-6, 7, prob.n)
    a2, d2 = oracle.scale(g, bands * f[None, :], mode)
    assert np.array_equal(a2, ahat)
    x1, h1, _ = oracle.solve(g, mode, ahat, diag, b, tol=1e-5, maxit=100)
    x2, h2, _ = oracle.solve(g, mode, a2, d2, b * f, tol=1e-5, maxit=100)
    assert np.array_equal(h1, h2) and np.array_equal(x1, x2)


@pytest.mark.parametrize("mode", ["fp64", "mixed"])
def test_preconditioner_scale_invariance(mode):
    """Reading A-3: one Eq. 7 sweep from 0 gives omega*T^-1 r; BiCGStab is invariant to a constant
    factor on M^-1 (bitwise for powers of two), so dropping omega only rescales the preconditioner."""
    prob = gen.Problem(16, 12, 10, seed=28)
    g, bands, b, ahat, diag = _setup(prob, mode)
    x1, h1, i1 = oracle.solve(g, mode, ahat, diag, b, tol=1e-5, maxit=100)
    x2, h2, i2 = oracle.solve(g, mode, ahat, diag, b, tol=1e-5, maxit=100, precond_scale=2.0)
    assert np.array_equal(x1, x2) and np.array_equal(h1, h2)
    # omega = 1.5 is not a power of two: same iterations, x within rounding
    x3, h3, i3 = oracle.solve(g, mode, ahat, diag, b, tol=1e-5, maxit=100, precond_scale=1.5)
    assert i3.iters == i1.iters
    assert np.linalg.norm(x3 - x1) <= (1e-12 if mode == "fp64" else 1e-5) * np.linalg.norm(x1)


# ---------------- spectral bound of the preconditioned operator ----------------

@pytest.mark.parametrize("prob", [gen.Problem(6, 4, 5, seed=29), gen.Problem(12, 8, 5, seed=30, cv=(5, 500))])
def test_mmatrix_spectral_bound(prob):
    """Ahat = I - N_v - N_h is a strictly diagonally dominant M-matrix, so T^-1 >= 0 and every
    eigenvalue of T^-1 Ahat lies in the disk |lambda - 1| <= 1 - min_p (T^-1 d)_p < 1, d = Ahat·1
    (SURVEY.md §8(d)).  Built column by column from the oracle's own thomas/apply."""
    g, bands, b, ahat, diag = _setup(prob, "fp64")
    n = prob.n
    M = np.empty((n, n))
    for c in range(n):
        e = np.zeros(n); e[c] = 1.0
        M[:, c] = oracle.thomas(g, "fp64", ahat, oracle.apply(g, ahat, e))
    d = oracle.apply(g, ahat, np.ones(n))
    tinv_d = oracle.thomas(g, "fp64", ahat, d)
    rho = 1.0 - tinv_d.min()
    assert 0 < rho < 1
    lam = np.linalg.eigvals(M)
    assert np.max(np.abs(lam - 1.0)) <= rho + 1e-12
    assert np.min(np.linalg.inv(dense_T(g, ahat))) >= -1e-15       # T^-1 >= 0


# ---------------- control flow: fixed iterations, restarts ----------------

def test_tol_zero_runs_exactly_maxit():
    prob = gen.CONFIGS["C1"]
    g, bands, b, ahat, diag = _setup(prob, "mixed")
    x, hist, info = oracle.solve(g, "mixed", ahat, diag, b, tol=0.0, maxit=8)
    assert info.iters == 8 and not info.converged and info.restarts == 0
    assert len(hist) == 9 and np.all(np.isfinite(hist)) and hist[0] == 1.0


def test_mandatory_restart_bookkeeping():
    prob = gen.Problem(32, 24, 10, seed=31)
    g, bands, b, ahat, diag = _setup(prob, "fp64")
    x0, h0, i0 = oracle.solve(g, "fp64", ahat, diag, b, tol=1e-8, maxit=200, restart_every=0)
    x1, h1, i1 = oracle.solve(g, "fp64", ahat, diag, b, tol=1e-8, maxit=200, restart_every=3)
    assert i1.converged and i1.true_R < 1e-8
    assert i1.restarts == (i1.iters - 1) // 3
    assert np.array_equal(h1[:4], h0[:4])                 # identical until the first restart
    assert np.linalg.norm(x1 - x0) <= 1e-6 * np.linalg.norm(x0)


def test_recurrence_tracks_true_residual():
    """|R_rec - R_true| / R_true <= 1e-3 while R >= 100 eps; and the running minimum of the
    true residual falls at least once in every 5 iterations (reading A-17, never monotone R)."""
    prob = gen.CONFIGS["C1"]
    g, bands, b, ahat, diag = _setup(prob, "fp64")
    true = []
    for m in range(1, 9):
        _, hist, info = oracle.solve(g, "fp64", ahat, diag, b, tol=0.0, maxit=m)
        assert abs(hist[m] - info.true_R) <= 1e-3 * info.true_R
        true.append(info.true_R)
    run_min = np.minimum.accumulate(true)
    for s in range(len(true) - 5):
        assert run_min[s + 5] < run_min[s]


# ---------------- the paper's MP-vs-DP observations (Table 1) ----------------

@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("tol", [OBS["original_tol"], OBS["operational_tol"]])
def test_mixed_and_fp64_identical_iteration_counts(seed, tol):
    prob = gen.Problem(64, 48, 10, seed=seed)
    g, bands, b, a64, d64 = _setup(prob, "fp64")
    a32, d32 = oracle.scale(g, bands, "mixed")
    _, h64, i64 = oracle.solve(g, "fp64", a64, d64, b, tol=tol, maxit=200)
    _, h32, i32 = oracle.solve(g, "mixed", a32, d32, b, tol=tol, maxit=200)
    assert i64.converged and i32.converged
    assert i32.iters == i64.iters
    assert _sigfig_agree(h32[1], h64[1], OBS["mp_dp_sigfigs_after_iteration_1"])
    for a, c in zip(h32, h64):
        if c < 1e-3:
            break
        assert _sigfig_agree(a, c, OBS["mp_dp_sigfigs_at_halting"])
    assert _sigfig_agree(h32[-1], h64[-1], OBS["mp_dp_sigfigs_at_halting"])


@pytest.mark.slow
def test_mixed_and_fp64_identical_iteration_counts_C2():
    prob = gen.CONFIGS["C2"]
    g, bands, b, a64, d64 = _setup(prob, "fp64")
    a32, d32 = oracle.scale(g, bands, "mixed")
    _, h64, i64 = oracle.solve(g, "fp64", a64, d64, b, tol=1e-4, maxit=200)
    _, h32, i32 = oracle.solve(g, "mixed", a32, d32, b, tol=1e-4, maxit=200)
    assert i64.converged and i32.converged and i32.iters == i64.iters
    assert _sigfig_agree(h32[-1], h64[-1], 4)
