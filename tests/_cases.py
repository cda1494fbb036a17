"""Hand-built inputs for the breakdown / restart cases (input generators only: no solver arithmetic).

Both the oracle pins (tests/test_oracle_breakdown.py) and the GPU parity tests
(tests/test_gpu_breakdown.py) build their inputs here.  Every value is a small dyadic rational
(a few significant bits), so the dot products of the first iteration are exact in binary32 and
binary64 whatever the summation order: the scalar that breaks down is exactly 0 on both sides, not
merely small.  The paper's operational failure mode is "scalar weights ... close to or equal to
zero", handled by a restart; reading A-12 fixes the test.
"""
import numpy as np

NX, NY = 128, 8   # one 128-column tile, 8 reduction row-groups of one row each; nz = 1


def _q(i, j, nx=NX):
    return i + nx * j          # nz = 1: q = i + nx*(k + nz*j)


def identity_operator(nx=NX, ny=NY, c=2.0):
    """nz = 1 and no horizontal coupling: A = c I, so Ahat = I and T = I (M^-1 Ahat = I).
    Returns bands7 [7, n] (C, E, W, N, S, U, D)."""
    n = nx * ny
    bands = np.zeros((7, n))
    bands[0] = c
    return bands


def ring_operator(nx=NX, ny=NY, a=0.25):
    """nz = 1, unit diagonal, E = W = -a, no N/S coupling: every latitude row is an independent
    periodic ring, Ahat = I - a (shift_E + shift_W), T = I."""
    n = nx * ny
    bands = np.zeros((7, n))
    bands[0] = 1.0
    bands[1] = -a
    bands[2] = -a
    return bands


def dyadic_rhs(nx=NX, ny=NY, seed=0):
    """b with values k/8, k in [-32, 32] \\ {0}: products and sums of the first iteration are exact."""
    rng = np.random.default_rng(seed)
    k = rng.integers(1, 33, size=nx * ny) * rng.choice([-1, 1], size=nx * ny)
    return k.astype(np.float64) / 8.0


def unit_rhs(nx=NX, ny=NY):
    """b = e_0 (the first point of row 0)."""
    b = np.zeros(nx * ny)
    b[_q(0, 0, nx)] = 1.0
    return b


def shadow_sigma_zero(nx=NX, ny=NY):
    """With ring_operator(a = 1/4) and b = e_0: r0 = e_0, v = Ahat T^-1 r0 = e_0 - e_1/4 - e_{nx-1}/4,
    so rhat0 = e_0 + 2 e_1 + 2 e_{nx-1} gives rho = rhat0 . r0 = 1 and sigma = rhat0 . v =
    1 - 1/2 - 1/2 = 0 exactly in the first iteration."""
    s = np.zeros(nx * ny)
    s[_q(0, 0, nx)] = 1.0
    s[_q(1, 0, nx)] = 2.0
    s[_q(nx - 1, 0, nx)] = 2.0
    return s


def shadow_rho_zero(nx=NX, ny=NY):
    """b = e_0: rhat0 = e_1 + e_5 is orthogonal to r0, rho = 0 at the first start."""
    s = np.zeros(nx * ny)
    s[_q(1, 0, nx)] = 1.0
    s[_q(5, 0, nx)] = 1.0
    return s


def shadow_rho_tiny(nx=NX, ny=NY):
    """b = e_0: rhat0 = 2^-30 e_0 + e_5, rho = 2^-30 ~ 2^-30 ||rhat0|| ||r0||: below the binary32
    threshold eps_V = 2^-24 (MIXED, FP32) and above the binary64 one (2^-53, FP64)."""
    s = np.zeros(nx * ny)
    s[_q(0, 0, nx)] = 2.0 ** -30
    s[_q(5, 0, nx)] = 1.0
    return s
