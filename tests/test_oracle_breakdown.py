"""Pins of the oracle's breakdown / restart branch (reading A-12; restart P:553-557).

Each case is built so that the scalar that breaks down is EXACTLY zero by arithmetic a reader can
check by hand (tests/_cases.py: dyadic values, identity or ring operators), and the expected
outcome follows from the algorithm's definition, not from the oracle:

* Ahat = I (nz = 1, no coupling): z = p = r and v = Ahat z = r, so sigma = rhat0 . v = rho and
  alpha = 1 exactly; s = r - v = 0 and t = 0.  With tol = 0 the s-step exit is not taken
  (R_s = 0 is not < 0), t.t = 0 is a breakdown; the restart from the unchanged x = 0 repeats it:
  two breakdowns without progress = EG_ERR_BREAKDOWN, 0 iterations, 1 restart.  With tol > 0 the
  s-step exits at iteration 1 with x = alpha z = bhat.
* r0 = 0 (x0 the exact solution, tol = 0): rho = 0 at the start, twice.
* a caller-given rhat0 with sigma = 0 in the first iteration, or with rho = 0 at the first start:
  one breakdown, then a restart from x = 0 with rhat0 = r, which IS the plain solve: x and the
  history bitwise those of the solve without rhat0, one more restart, one breakdown.
* rho = 2^-30 ||rhat0|| ||r0||: a breakdown under the binary32 threshold eps_V = 2^-24 (MIXED, FP32)
  but not under the binary64 one, 2^-53 (FP64), where the solve runs with the given rhat0.
"""
import numpy as np
import pytest

import oracle
from _cases import (NX, NY, dyadic_rhs, identity_operator, ring_operator, shadow_rho_tiny,
                    shadow_rho_zero, shadow_sigma_zero, unit_rhs)
from _dense import sparse_from_bands

MODES = ["fp64", "mixed", "fp32"]
G = (NX, NY, 1)
TOL = {"fp64": 1e-8, "mixed": 1e-6, "fp32": 1e-5}


def _solve(bands, b, mode, **kw):
    ahat, diag = oracle.scale(G, bands, mode)
    return oracle.solve(G, mode, ahat, diag, b, **kw)


@pytest.mark.parametrize("mode", MODES)
def test_identity_operator_tol0_breaks_down_twice(mode):
    x, h, info = _solve(identity_operator(), dyadic_rhs(), mode, tol=0.0, maxit=10)
    assert info.status == oracle.STATUS_CODES["ERR_BREAKDOWN"]
    assert (info.iters, info.breakdowns, info.restarts, info.converged) == (0, 2, 1, False)
    assert np.all(x == 0.0) and h[0] == pytest.approx(1.0, rel=1e-7)


@pytest.mark.parametrize("mode", MODES)
def test_identity_operator_s_step_exit(mode):
    b = dyadic_rhs()
    x, h, info = _solve(identity_operator(c=2.0), b, mode, tol=1e-6, maxit=10)
    assert info.status == 0 and info.converged and (info.iters, info.breakdowns, info.restarts) == (1, 0, 0)
    assert np.array_equal(x, b / 2.0) and h[1] == 0.0 and info.true_R == 0.0


@pytest.mark.parametrize("mode", MODES)
def test_exact_initial_guess_tol0_breaks_down_at_start(mode):
    b = dyadic_rhs(seed=1)
    x0 = b / 2.0
    x, h, info = _solve(identity_operator(c=2.0), b, mode, x0=x0, tol=0.0, maxit=10)
    assert info.status == oracle.STATUS_CODES["ERR_BREAKDOWN"]
    assert (info.iters, info.breakdowns, info.restarts) == (0, 2, 1)
    assert np.array_equal(x, x0) and h[0] == 0.0


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("shadow", [shadow_sigma_zero, shadow_rho_zero], ids=["sigma0", "rho0"])
def test_given_shadow_breakdown_restarts_into_the_plain_solve(mode, shadow):
    bands, b, sh = ring_operator(), unit_rhs(), shadow()
    # the hand arithmetic of tests/_cases.py, checked with an independent dense assembly
    A = sparse_from_bands(G, bands[0], bands[1:]).toarray()
    if shadow is shadow_sigma_zero:
        assert sh @ b == 1.0 and sh @ (A @ b) == 0.0        # rho = 1, sigma = 0 (T = I, r0 = b)
    else:
        assert sh @ b == 0.0                                 # rho = 0
    xp, hp, ip = _solve(bands, b, mode, tol=TOL[mode], maxit=100)
    x, h, info = _solve(bands, b, mode, tol=TOL[mode], maxit=100, rhat0=sh)
    assert ip.status == 0 and ip.converged and ip.breakdowns == 0
    assert info.status == 0 and info.converged
    assert info.breakdowns == 1 and info.restarts == ip.restarts + 1 and info.iters == ip.iters
    assert np.array_equal(x, xp) and np.array_equal(h, hp)
    xd = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xd) <= 10 * TOL[mode] * np.linalg.norm(xd)


@pytest.mark.parametrize("mode", MODES)
def test_rho_threshold_depends_on_the_working_precision(mode):
    bands, b, sh = ring_operator(), unit_rhs(), shadow_rho_tiny()
    assert sh @ b == 2.0 ** -30
    xp, hp, ip = _solve(bands, b, mode, tol=TOL[mode], maxit=100)
    x, h, info = _solve(bands, b, mode, tol=TOL[mode], maxit=100, rhat0=sh)
    assert info.status == 0 and info.converged and info.true_R < TOL[mode]
    if mode == "fp64":      # 2^-30 > 2^-53: no breakdown, the given rhat0 is used
        assert info.breakdowns == 0 and not np.array_equal(h, hp)
    else:                   # 2^-30 < 2^-24: breakdown at the start, then the plain solve
        assert info.breakdowns == 1 and np.array_equal(x, xp) and np.array_equal(h, hp)


def test_shadow_equal_to_r0_is_the_default():
    """rhat0 = r0 given explicitly reproduces the default solve bitwise (reading A-1)."""
    import gen
    prob = gen.Problem(16, 12, 6, seed=31)
    bands, b = gen.host(prob)
    g = (prob.nx, prob.ny, prob.nz)
    for mode in MODES:
        ahat, diag = oracle.scale(g, bands, mode)
        x1, h1, i1 = oracle.solve(g, mode, ahat, diag, b, tol=1e-5, maxit=100)
        x2, h2, i2 = oracle.solve(g, mode, ahat, diag, b, tol=1e-5, maxit=100, rhat0=b / diag)
        assert i1.iters == i2.iters and np.array_equal(x1, x2) and np.array_equal(h1, h2), mode
