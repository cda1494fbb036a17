"""Pins of the oracle's NEXT-1 tri-SOR preconditioner (Eq. 7), red-black order.

The reference is Eq. 7 itself in dense matrix form: with the columns ordered red (i+j even) before
black, L (U) holds the couplings of a column to columns earlier (later) in that order — for the
horizontal 7-point couplings this means black->red couplings are in L and red->black in U — and
    (T + omega L) x_n = (1 - omega) T x_{n-1} + omega (f - U x_{n-1})
is solved with numpy.linalg.solve.  The oracle instead sweeps columns in place with Thomas solves.
"""
import numpy as np
import pytest

import gen
import oracle
from _dense import dense_Ahat, dense_T, idx

GRIDS = [gen.Problem(4, 3, 3, seed=41), gen.Problem(6, 4, 5, seed=42), gen.Problem(8, 5, 4, seed=43)]


def _setup(prob, mode="fp64"):
    g = (prob.nx, prob.ny, prob.nz)
    bands, b = gen.host(prob)
    ahat, diag = oracle.scale(g, bands, mode)
    return g, ahat, diag, b


def _dense_eq7(g, ahat, f, sweeps, omega, x0=None):
    nx, ny, nz = g
    n = nx * ny * nz
    A = dense_Ahat(g, ahat)
    T = dense_T(g, ahat)
    H = A - T
    colour = np.empty(n, int)
    for j in range(ny):
        for k in range(nz):
            for i in range(nx):
                colour[idx(nx, ny, nz, i, j, k)] = (i + j) % 2
    # L: coupling of row q to a column of an earlier colour; U: to the same or a later colour
    earlier = colour[:, None] > colour[None, :]
    L = np.where(earlier, H, 0.0)
    U = H - L
    x = np.zeros(n) if x0 is None else x0.copy()
    for _ in range(sweeps):
        x = np.linalg.solve(T + omega * L, (1 - omega) * (T @ x) + omega * (f - U @ x))
    return x


@pytest.mark.parametrize("prob", GRIDS)
@pytest.mark.parametrize("sweeps,omega", [(1, 1.0), (1, 1.5), (3, 1.5), (2, 0.7)])
def test_trisor_is_eq7_in_red_black_order(prob, sweeps, omega):
    g, ahat, _, _ = _setup(prob)
    f = np.random.default_rng(1).standard_normal(prob.n)
    z = oracle.trisor(g, "fp64", ahat, f, sweeps=sweeps, omega=omega)
    zd = _dense_eq7(g, ahat, f, sweeps, omega)
    assert np.linalg.norm(z - zd) <= 1e-12 * np.linalg.norm(zd)


def test_no_horizontal_coupling_reduces_to_thomas():
    """c_h = 0: L = U = 0, so one sweep with omega = 1 is exactly T^-1 f (bitwise)."""
    prob = gen.Problem(8, 6, 10, seed=44, ch=(0.0, 0.0))
    g, ahat, _, _ = _setup(prob, "mixed")
    f = np.random.default_rng(2).standard_normal(prob.n).astype(np.float32).astype(np.float64)
    assert np.array_equal(oracle.trisor(g, "mixed", ahat, f, sweeps=1, omega=1.0), oracle.thomas(g, "mixed", ahat, f))


def test_exact_solution_is_a_fixed_point_and_sweeps_converge():
    prob = GRIDS[1]
    g, ahat, _, _ = _setup(prob)
    f = np.random.default_rng(3).standard_normal(prob.n)
    xs = np.linalg.solve(dense_Ahat(g, ahat), f)
    x1 = oracle.trisor(g, "fp64", ahat, f, sweeps=1, omega=1.5, x_init=xs)
    assert np.linalg.norm(x1 - xs) <= 1e-12 * np.linalg.norm(xs)
    # the stationary iteration converges to Ahat^-1 f (M-matrix, omega = 1)
    x = oracle.trisor(g, "fp64", ahat, f, sweeps=400, omega=1.0)
    assert np.linalg.norm(x - xs) <= 1e-10 * np.linalg.norm(xs)


def test_trisor_is_linear_and_rejects_odd_nx():
    prob = GRIDS[2]
    g, ahat, _, _ = _setup(prob)
    rng = np.random.default_rng(4)
    f1, f2 = rng.standard_normal(prob.n), rng.standard_normal(prob.n)
    lhs = oracle.trisor(g, "fp64", ahat, 2.0 * f1 + f2)
    rhs = 2.0 * oracle.trisor(g, "fp64", ahat, f1) + oracle.trisor(g, "fp64", ahat, f2)
    assert np.linalg.norm(lhs - rhs) <= 1e-13 * np.linalg.norm(rhs)
    odd = gen.Problem(5, 3, 3, seed=45)
    go, ao, _, _ = _setup(odd)
    with pytest.raises(oracle.OracleError):
        oracle.trisor(go, "fp64", ao, np.ones(odd.n))


@pytest.mark.parametrize("mode", ["fp64", "mixed"])
def test_solve_with_trisor_preconditioner(mode):
    """BiCGStab with the paper's preconditioner (3 sweeps, omega = 1.5) reaches the same solution in
    no more iterations than with T^-1 on a harder operator."""
    prob = gen.Problem(32, 24, 20, seed=46, cv=(5.0, 20.0), dl=(1e-3, 1e-2))
    g, ahat, diag, b = _setup(prob, mode)
    x1, h1, i1 = oracle.solve(g, mode, ahat, diag, b, tol=1e-6 if mode == "fp64" else 1e-5, maxit=300)
    x3, h3, i3 = oracle.solve(g, mode, ahat, diag, b, tol=1e-6 if mode == "fp64" else 1e-5, maxit=300,
                              sor_sweeps=3, sor_omega=1.5)
    assert i1.converged and i3.converged
    assert i3.iters <= i1.iters
    # the same solution: both within 50 tol of the direct (SuperLU) solve.  The error of a solve
    # stopped at R < tol is bounded by cond(Ahat) R, loose here (delta down to 1e-3); the T^-1 solve
    # of this seed sits at 12 tol, the tri-SOR one at 0.5 tol
    import scipy.sparse.linalg as spla
    from _dense import sparse_from_bands
    bands, _ = gen.host(prob)
    xd = spla.spsolve(sparse_from_bands(g, bands[0], bands[1:]).tocsc(), b)
    tol = 1e-6 if mode == "fp64" else 1e-5
    for x in (x1, x3):
        assert np.linalg.norm(x - xd) <= 50 * tol * np.linalg.norm(xd)
