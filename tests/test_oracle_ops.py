"""Pins of the oracle's exact sub-steps: scaling, apply, Thomas, global sums.

Each pin comes from outside the oracle: an independently assembled numpy/scipy matrix, a closed
form, an invariant, or a special case that reduces to a textbook result.
"""
import math

import numpy as np
import pytest

import gen
import oracle
from _dense import dense_A, dense_Ahat, dense_T, transpose_apply

GRIDS = [gen.Problem(4, 3, 2, seed=11), gen.Problem(5, 4, 3, seed=12), gen.Problem(16, 12, 6, seed=13)]


def _setup(prob, mode="fp64"):
    g = (prob.nx, prob.ny, prob.nz)
    bands, b = gen.host(prob)
    ahat, diag = oracle.scale(g, bands, mode)
    return g, bands, b, ahat, diag


# ---------------- a1: diagonal scaling (Eq. 5) ----------------

@pytest.mark.parametrize("prob", GRIDS)
def test_scale_is_D_inverse_A(prob):
    g, bands, _, ahat, diag = _setup(prob)
    A = dense_A(g, bands)
    Ah = dense_Ahat(g, ahat)
    assert np.array_equal(diag, bands[0])
    # D^-1 A with unit diagonal, entry for entry (IEEE division on both sides)
    np.testing.assert_array_equal(Ah, A / np.diag(A)[:, None])


def test_scale_rounds_to_fp32_in_mixed():
    prob = GRIDS[1]
    g, bands, _, a64, _ = _setup(prob, "fp64")
    a32, _ = oracle.scale(g, bands, "mixed")
    assert np.array_equal(a32, a64.astype(np.float32).astype(np.float64))


def test_scale_spec_example_and_errors():
    # aC = 2, aE = 1 -> ahat_E = 0.5
    g = (4, 3, 2)
    n = 24
    bands = np.zeros((7, n))
    bands[0] = 2.0
    bands[1] = 1.0
    ahat, diag = oracle.scale(g, bands, "fp64")
    assert np.all(ahat[0] == 0.5) and np.all(ahat[1:] == 0) and np.all(diag == 2)
    bad = bands.copy(); bad[0, 5] = 0.0
    with pytest.raises(oracle.OracleError) as e:
        oracle.scale(g, bad, "fp64")
    assert e.value.status == 2                       # singular diagonal
    bad = bands.copy(); bad[3, 23] = 1.0             # N band at j = ny-1 (absent neighbour)
    with pytest.raises(oracle.OracleError) as e:
        oracle.scale(g, bad, "fp64")
    assert e.value.status == 1
    with pytest.raises(oracle.OracleError):
        oracle.scale((2, 3, 2), np.ones((7, 12)), "fp64")   # nx < 3 (reading A-19)


# ---------------- (c1) apply ----------------

@pytest.mark.parametrize("prob", GRIDS)
def test_apply_matches_dense(prob):
    g, _, _, ahat, _ = _setup(prob)
    x = np.random.default_rng(prob.seed).standard_normal(prob.n)
    y = oracle.apply(g, ahat, x)
    yd = dense_Ahat(g, ahat) @ x
    assert np.linalg.norm(y - yd) <= 1e-14 * np.linalg.norm(yd)


@pytest.mark.parametrize("prob", GRIDS + [gen.CONFIGS["C1"], gen.Problem(7, 5, 1, seed=3)])
def test_apply_closed_form_on_ones(prob):
    """A·1 = diag - sum|off| (all off-diagonals negative) => Ahat·1 = delta/(1+delta) pointwise;
    covers the periodic seam, the poles, top/bottom and the scaling at once."""
    g, _, _, ahat, _ = _setup(prob)
    y = oracle.apply(g, ahat, np.ones(prob.n))
    q = np.arange(prob.n)
    dl = 0.01 + 0.09 * np.array([gen.uniform(prob.seed, 2, int(t)) for t in q])
    np.testing.assert_allclose(y, dl / (1 + dl), rtol=0, atol=4e-15)
    _, _, _, a32, _ = _setup(prob, "mixed")
    y32 = oracle.apply_wp(g, "mixed", a32, np.ones(prob.n))
    np.testing.assert_allclose(y32, dl / (1 + dl), rtol=0, atol=1e-6)


@pytest.mark.parametrize("prob", GRIDS)
def test_apply_adjoint_identity(prob):
    g, _, _, ahat, _ = _setup(prob)
    rng = np.random.default_rng(1)
    x, y = rng.standard_normal(prob.n), rng.standard_normal(prob.n)
    lhs = y @ oracle.apply(g, ahat, x)
    rhs = transpose_apply(g, ahat, y) @ x
    assert abs(lhs - rhs) <= 1e-13 * (abs(lhs) + 1)


def test_operator_symmetry_structure():
    prob = gen.Problem(5, 4, 3, seed=4)
    g = (5, 4, 3)
    bands, _ = gen.host(prob)
    A = dense_A(g, bands)
    assert np.array_equal(A != 0, A.T != 0)          # structural symmetry incl. the seam
    assert not np.array_equal(A, A.T)                # "the matrix is non-symmetric"
    # constant coefficients: the Laplacian / Boussinesq limit is exactly symmetric
    const = prob.with_(ch=(1.0, 1.0), cv=(20.0, 20.0))
    Ac = dense_A(g, gen.host(const)[0])
    assert np.array_equal(Ac, Ac.T)


def test_apply_wp_fp64_is_apply_and_fp32_error_bound():
    prob = GRIDS[2]
    g, _, _, ahat, _ = _setup(prob)
    x = np.random.default_rng(2).standard_normal(prob.n)
    assert np.array_equal(oracle.apply_wp(g, "fp64", ahat, x), oracle.apply(g, ahat, x))
    _, _, _, a32, _ = _setup(prob, "mixed")
    x32 = x.astype(np.float32).astype(np.float64)
    ywp = oracle.apply_wp(g, "mixed", a32, x32)
    assert np.array_equal(ywp, ywp.astype(np.float32))           # binary32 values
    y64 = oracle.apply(g, a32, x32)
    absum = np.abs(x32) + np.abs(dense_Ahat(g, a32) - np.eye(prob.n)) @ np.abs(x32)
    assert np.all(np.abs(ywp - y64) <= 14 * 2.0**-24 * absum)


# ---------------- (c1) Thomas: z = T^-1 f per column ----------------

@pytest.mark.parametrize("prob", GRIDS + [gen.Problem(4, 3, 70, seed=9)])
def test_thomas_matches_dense_lu(prob):
    g, _, _, ahat, _ = _setup(prob)
    f = np.random.default_rng(3).standard_normal(prob.n)
    z = oracle.thomas(g, "fp64", ahat, f)
    zd = np.linalg.solve(dense_T(g, ahat), f)
    assert np.max(np.abs(z - zd)) <= 1e-12 * np.max(np.abs(zd))


@pytest.mark.parametrize("nz", [2, 10, 70])
def test_thomas_fp32_residual_bound(nz):
    prob = gen.Problem(8, 6, nz, seed=nz)
    g, _, _, a32, _ = _setup(prob, "mixed")
    f = np.random.default_rng(4).standard_normal(prob.n).astype(np.float32).astype(np.float64)
    z = oracle.thomas(g, "mixed", a32, f)
    assert np.array_equal(z, z.astype(np.float32))
    res = dense_T(g, a32) @ z - f
    # S:225 bound 10*nz*eps on each column
    assert np.max(np.abs(res)) / np.max(np.abs(f)) <= 10 * nz * 2.0**-24


@pytest.mark.parametrize("nz,a,m", [(10, 0.3, 1), (70, 0.45, 3), (33, 0.2, 7)])
def test_thomas_closed_form_sine_modes(nz, a, m):
    """T = tridiag(-a, 1, -a) has eigenvectors sin(pi m (k+1)/(nz+1)) with eigenvalue
    1 - 2a cos(pi m/(nz+1)): the textbook tridiagonal-Toeplitz closed form."""
    nx, ny = 3, 2
    n = nx * ny * nz
    ahat = np.zeros((6, n))
    k = np.tile(np.repeat(np.arange(nz), nx), ny)
    ahat[4] = np.where(k < nz - 1, -a, 0.0)
    ahat[5] = np.where(k > 0, -a, 0.0)
    f = np.sin(np.pi * m * (k + 1) / (nz + 1))
    z = oracle.thomas((nx, ny, nz), "fp64", ahat, f)
    lam = 1 - 2 * a * math.cos(math.pi * m / (nz + 1))
    np.testing.assert_allclose(z, f / lam, rtol=1e-13, atol=1e-15)


def test_thomas_special_cases():
    prob = GRIDS[1]
    g, _, _, ahat, _ = _setup(prob)
    f = np.random.default_rng(5).standard_normal(prob.n)
    a0 = ahat.copy(); a0[4:] = 0.0
    assert np.array_equal(oracle.thomas(g, "fp64", a0, f), f)          # U = D = 0 -> z = f
    g1 = (prob.nx, prob.ny, 1)
    p1 = gen.Problem(prob.nx, prob.ny, 1, seed=3)
    _, _, _, a1, _ = _setup(p1)
    f1 = f[: p1.n]
    assert np.array_equal(oracle.thomas(g1, "fp64", a1, f1), f1)        # nz = 1 -> z = f


# ---------------- global sums ----------------

def test_dot_small_integers_exact():
    g = (4, 1, 1)
    assert oracle.dot(g, "fp64", np.array([1.0, 2, 3, 4]), np.ones(4)) == 10.0
    assert oracle.dot(g, "fp32", np.array([1.0, 2, 3, 4]), np.ones(4)) == 10.0
    rng = np.random.default_rng(6)
    a = rng.integers(-1000, 1000, 3 * 5 * 7).astype(np.float64)
    b = rng.integers(-1000, 1000, 3 * 5 * 7).astype(np.float64)
    assert oracle.dot((3, 5, 7), "mixed", a, b) == float(np.sum(a.astype(np.int64) * b.astype(np.int64)))


def test_dot_fp64_accumulation_error_bound():
    rng = np.random.default_rng(7)
    g = (64, 48, 10)
    a = rng.standard_normal(30720).astype(np.float32).astype(np.float64)
    b = rng.standard_normal(30720).astype(np.float32).astype(np.float64)
    exact = math.fsum((a * b).tolist())            # products of binary32 are exact in binary64
    err = abs(oracle.dot(g, "mixed", a, b) - exact)
    assert err <= 30720 * 2.0**-53 * float(np.sum(np.abs(a * b)))
    err32 = abs(oracle.dot(g, "fp32", a, b) - exact)
    assert err32 <= 30720 * 2.0**-24 * float(np.sum(np.abs(a * b)))
    assert err32 > err                              # 32-bit sums are genuinely 32-bit


def test_dot_rows_first_then_across_rows():
    """"local summation performed first, then ... a reduction": per-row partials, then
    rows in order.  In binary32, 1e8 absorbs a following +1, so a flat sequential sum of
    [1e8, 1 x 7 | 1 x 8] gives 1e8 while rows-first gives 1e8 + 8 (exactly representable)."""
    g = (8, 2, 1)           # two rows of 8 points
    a = np.array([1e8] + [1.0] * 15, dtype=np.float64)
    assert oracle.dot(g, "fp32", a, np.ones(16)) == 100000008.0
    assert oracle.dot(g, "fp64", a, np.ones(16)) == 100000015.0
