"""Seeded generator: determinism, the BASELINE.json recipe's invariants, and SplitMix64 vectors."""
import numpy as np
import pytest

import gen

SMALL = [gen.Problem(4, 3, 2, seed=7), gen.Problem(16, 12, 6, seed=1), gen.CONFIGS["C1"]]


def test_splitmix64_published_vectors():
    # SplitMix64 (Steele, Lea & Flood 2014) from state 0: first two outputs
    assert gen.mix(0) == 0xE220A8397B1DCDAF
    assert gen.mix(0x9E3779B97F4A7C15) == 0x6E789E6AA1B965F4


def test_uniform_range_and_exactness():
    us = np.array([gen.uniform(3, s, q) for s in range(3) for q in range(2000)])
    assert us.min() >= 0.0 and us.max() < 1.0
    # 53-bit dyadic rationals
    assert np.all(us * 2.0**53 == np.floor(us * 2.0**53))
    assert abs(us.mean() - 0.5) < 0.02


@pytest.mark.parametrize("prob", SMALL)
def test_determinism_and_seed_dependence(prob):
    b1, r1 = gen.host(prob)
    b2, r2 = gen.host(prob)
    assert np.array_equal(b1, b2) and np.array_equal(r1, r2)
    b3, r3 = gen.host(prob.with_(seed=prob.seed + 1))
    assert not np.array_equal(b1, b3) and not np.array_equal(r1, r3)


@pytest.mark.parametrize("prob", SMALL)
def test_recipe_invariants(prob):
    nx, ny, nz = prob.nx, prob.ny, prob.nz
    bands, b = gen.host(prob)
    C, E, W, N, S, U, D = [x.reshape(ny, nz, nx) for x in bands]
    cl = gen.coslat(ny)
    assert np.all(cl > 0) and np.allclose(cl, cl[::-1], rtol=0, atol=1e-15)
    # zeros at absent neighbours, negative couplings elsewhere
    assert np.all(N[-1] == 0) and np.all(S[0] == 0) and np.all(U[:, -1] == 0) and np.all(D[:, 0] == 0)
    assert np.all(N[:-1] < 0) and np.all(S[1:] < 0) and np.all(U[:, :-1] < 0) and np.all(D[:, 1:] < 0)
    assert np.array_equal(E, W) and np.all(E < 0)
    # one c_h per point: N = S = -c_h in the interior; E = -c_h cos(lat_j)
    if ny > 2:
        assert np.array_equal(N[1:-1], S[1:-1])
        ch = -N[1:-1]
        assert np.allclose(E[1:-1], -ch * cl[1:-1, None, None], rtol=1e-15)
        assert ch.min() >= 0.5 and ch.max() < 1.5
    if nz > 2:
        cv = -U[:, 1:-1]
        assert np.array_equal(U[:, 1:-1], D[:, 1:-1])
        assert cv.min() >= prob.cv[0] and cv.max() < prob.cv[1]
    # diag / sum|off| - 1 = delta in [0.01, 0.1]
    off = np.abs(E) + np.abs(W) + np.abs(N) + np.abs(S) + np.abs(U) + np.abs(D)
    delta = C / off - 1.0
    assert delta.min() >= 0.01 - 1e-14 and delta.max() <= 0.1 + 1e-14
    # the delta drawn from stream 2 (independent recomputation)
    q = np.arange(prob.n)
    dl = np.array([0.01 + 0.09 * gen.uniform(prob.seed, 2, int(t)) for t in q[:: max(1, prob.n // 500)]])
    assert np.allclose(delta.reshape(-1)[:: max(1, prob.n // 500)], dl, rtol=0, atol=4e-15)


def test_rhs_moments():
    _, b = gen.host(gen.Problem(64, 48, 20, seed=5))
    assert abs(b.mean()) < 0.02 and abs(b.var() - 1.0) < 0.02
    assert b.min() >= -6 and b.max() <= 6


@pytest.mark.parametrize("prob", SMALL)
def test_point_matches_rows(prob):
    bands, b = gen.host(prob)
    cl = gen.coslat(prob.ny)
    rng = np.random.default_rng(0)
    for _ in range(20):
        i, j, k = rng.integers(prob.nx), rng.integers(prob.ny), rng.integers(prob.nz)
        q = i + prob.nx * (k + prob.nz * j)
        v = gen.point(prob, int(i), int(j), int(k), cl)
        assert np.array_equal(v[:7], bands[:, q]) and v[7] == b[q]


def test_row_slices_match_full():
    prob = gen.Problem(8, 10, 3, seed=2)
    full, bf = gen.host(prob)
    part, bp = gen.host(prob, 3, 7)
    row = prob.nx * prob.nz
    assert np.array_equal(part, full[:, 3 * row:7 * row]) and np.array_equal(bp, bf[3 * row:7 * row])


@pytest.mark.gpu
@pytest.mark.parametrize("prob", [gen.Problem(33, 17, 5, seed=3), gen.CONFIGS["C2"]])
def test_device_generator_bitwise_equals_host(prob):
    import torch
    bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
    b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    gen.device(prob, bands, b)
    hb, hr = gen.host(prob)
    assert np.array_equal(bands.cpu().numpy(), hb) and np.array_equal(b.cpu().numpy(), hr)


@pytest.mark.gpu
@pytest.mark.parametrize("rows", [(0, 5), (5, 11), (11, 17), (8, 9)])
def test_device_generator_band_equals_host_rows(rows):
    """A latitude band generated on the device (what each rank of bench.py does) is bitwise the
    host generator's rows of the global problem."""
    import torch
    prob = gen.Problem(33, 17, 5, seed=3)
    j0, j1 = rows
    row = prob.nx * prob.nz
    nloc = (j1 - j0) * row
    bands = torch.empty((7, nloc), dtype=torch.float64, device="cuda")
    b = torch.empty(nloc, dtype=torch.float64, device="cuda")
    gen.device(prob, bands, b, j0, j1)
    hb, hr = gen.host(prob)
    assert np.array_equal(bands.cpu().numpy(), hb[:, j0 * row:j1 * row])
    assert np.array_equal(b.cpu().numpy(), hr[j0 * row:j1 * row])


def test_rhs_is_box_muller_normal():
    """b = sqrt(-2 ln(1 - u3)) cos(2 pi u4) from streams 3 and 4 (BASELINE.json's b ~ N(0,1),
    SURVEY.md §8(d)): the generator's portable ln / cos agree with numpy's libm to a few ulp, and
    the sample moments are those of N(0,1)."""
    prob = gen.Problem(64, 48, 10, seed=0)
    _, b = gen.host(prob)
    q = np.arange(0, prob.n, 7)
    u3 = np.array([gen.uniform(prob.seed, 3, int(t)) for t in q])
    u4 = np.array([gen.uniform(prob.seed, 4, int(t)) for t in q])
    ref = np.sqrt(-2.0 * np.log(1.0 - u3)) * np.cos(2.0 * np.pi * u4)
    assert np.max(np.abs(b[q] - ref)) <= 1e-14
    big = gen.host(gen.Problem(192, 144, 70, seed=1))[1]
    assert abs(big.mean()) < 5e-3 and abs(big.var() - 1.0) < 5e-3
    assert abs(np.mean(big ** 3)) < 1e-2 and abs(np.mean(big ** 4) - 3.0) < 2e-2   # skew 0, kurtosis 3
