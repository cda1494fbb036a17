"""Parity at BASELINE.json's full operational size (C5: 2560 x 1920 x 70, 344 M unknowns), in the
launch configuration bench.py times (the default solver, CUDA-graph replay, generator on device).

* apply / precondition: sampled latitude rows (poles, seam rows, interior) against the oracle run
  on a 3-row sub-grid around each sampled row (the sub-grid's artificial edges are decoupled; rows
  outside the sample are never compared).
* tri-SOR precondition (NEXT-1, 3 sweeps, omega 1.5, on the TMA sweep kernels): sampled rows
  against the oracle's sweeps on a window of rows around each; information travels one row per
  half-sweep, so a row at least 7 rows inside the window is exact (the window's decoupled edges
  cannot reach it in 6 half-sweeps); windows start on an even row (the colouring's parity).
* solve (MIXED, tol 1e-4): the full CPU oracle solve of the same inputs (about 70 GB of host RAM
  and a minute on the GPU box's cores) — iterations within 2, ||dx||/||x|| <= 10 tol, and the GPU's
  x has oracle-recomputed true residual < tol.  The same at C3 and C4 (MIXED, the default solver:
  fused phase kernels) and at C5 in the FP64 variant (BASELINE.json config 5's "fp64 variant"; the
  Table 1 DP column), where the fixed-iteration histories must agree to 1e-10.
"""
import numpy as np
import pytest

import gen
import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
egs = pytest.importorskip("paper_1811_03852_b200")

C5 = gen.CONFIGS["C5"]
ROWS = [0, 1, 959, 960, 1918, 1919]


@pytest.fixture(scope="module")
def c5():
    prob = C5
    bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
    b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    gen.device(prob, bands, b)
    s = egs.Solver((prob.nx, prob.ny, prob.nz), bands, "mixed")
    yield prob, bands, b, s
    s.close()


def _subgrid_oracle(prob, j, mode):
    """scaled bands of rows [j0, j1) around j with the artificial edges decoupled"""
    j0, j1 = max(0, j - 1), min(prob.ny, j + 2)
    row = prob.nx * prob.nz
    bands, _ = gen.host(prob, j0, j1)
    if j0 > 0:
        bands[4, :row] = 0.0     # S band of the first sub-grid row
    if j1 < prob.ny:
        bands[3, -row:] = 0.0    # N band of the last sub-grid row
    ahat, _ = oracle.scale((prob.nx, j1 - j0, prob.nz), bands, mode)
    return j0, j1, ahat


def test_c5_apply_and_precondition_sampled_rows(c5):
    prob, bands, b, s = c5
    row = prob.nx * prob.nz
    g = torch.Generator(device="cuda").manual_seed(5)
    x = torch.randn(prob.n, generator=g, device="cuda", dtype=torch.float32)
    y = s.apply(x)
    z = s.precondition(x)
    torch.cuda.synchronize()
    for j in ROWS:
        j0, j1, ahat = _subgrid_oracle(prob, j, "mixed")
        xs = x[j0 * row:j1 * row].double().cpu().numpy()
        yo = oracle.apply((prob.nx, j1 - j0, prob.nz), ahat, xs)[(j - j0) * row:(j - j0 + 1) * row]
        yg = y[j * row:(j + 1) * row].double().cpu().numpy()
        assert np.linalg.norm(yg - yo) <= 1e-6 * np.linalg.norm(yo), j
        zo = oracle.thomas((prob.nx, j1 - j0, prob.nz), "fp64", ahat, xs)[(j - j0) * row:(j - j0 + 1) * row]
        zg = z[j * row:(j + 1) * row].double().cpu().numpy()
        assert np.linalg.norm(zg - zo) <= 1e-5 * np.linalg.norm(zo), j


def test_c5_trisor_precondition_sampled_rows(c5):
    prob, bands, b, _ = c5
    row = prob.nx * prob.nz
    st = egs.Solver((prob.nx, prob.ny, prob.nz), bands, "mixed", trisor=True)
    st.set_preconditioner("trisor", sweeps=3, omega=1.5)
    g = torch.Generator(device="cuda").manual_seed(7)
    x = torch.randn(prob.n, generator=g, device="cuda", dtype=torch.float32)
    z = st.precondition(x)
    torch.cuda.synchronize()
    W = 8
    for j in (0, 3, 960, 1919):
        j0 = max(0, j - W)
        j0 -= j0 % 2                      # same colouring parity as the full grid
        j1 = min(prob.ny, j + W + 1)
        hb, _ = gen.host(prob, j0, j1)
        if j0 > 0:
            hb[4, :row] = 0.0             # decouple the window's artificial edges
        if j1 < prob.ny:
            hb[3, -row:] = 0.0
        gw = (prob.nx, j1 - j0, prob.nz)
        ahat, _ = oracle.scale(gw, hb, "mixed")
        xs = x[j0 * row:j1 * row].double().cpu().numpy()
        zo = oracle.trisor(gw, "fp64", ahat, xs, sweeps=3, omega=1.5)[(j - j0) * row:(j - j0 + 1) * row]
        zg = z[j * row:(j + 1) * row].double().cpu().numpy()
        assert np.linalg.norm(zg - zo) <= 1e-5 * np.linalg.norm(zo), j
    st.close()


def test_c5_solve_matches_full_oracle(c5):
    prob, bands, b, s = c5
    x, info, hist = s.solve(b, tol=1e-4, maxit=200)
    assert info.converged and info.true_R < 1e-4
    xg = x.cpu().numpy()
    del x
    hb, hrhs = gen.host(prob)
    assert np.array_equal(hrhs, b.cpu().numpy())           # the device generator's bits
    g = (prob.nx, prob.ny, prob.nz)
    ahat, diag = oracle.scale(g, hb, "mixed")
    del hb
    xo, ho, io = oracle.solve(g, "mixed", ahat, diag, hrhs, tol=1e-4, maxit=200)
    assert io.converged and abs(info.iters - io.iters) <= 2
    assert np.linalg.norm(xg - xo) <= 10 * 1e-4 * np.linalg.norm(xo)
    # the GPU's x against the oracle's fp64 residual on the fp32-rounded operator it iterated with
    bhat = hrhs / diag
    r = oracle.residual64(g, ahat, bhat, xg)
    assert np.linalg.norm(r) / np.linalg.norm(bhat) < 1e-4
    n = min(len(hist), len(ho))
    assert np.allclose(hist[:n], ho[:n], rtol=1e-3)


def _full_oracle_parity(prob, mode, tol=1e-4, hist_rtol=None):
    g = (prob.nx, prob.ny, prob.nz)
    bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
    b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    gen.device(prob, bands, b)
    s = egs.Solver(g, bands, mode)
    if mode != "fp64":   # the production path at these sizes: the fused phase kernels
        s.profile_reset()
        s.solve(b, tol=0.0, maxit=1, flags=egs.EG_SOLVE_PROFILE)
        assert s.profile()["phase_A"][1] == 1
    x, info, hist = s.solve(b, tol=tol, maxit=200)
    hf = None
    if hist_rtol is not None:
        _, _, hf = s.solve(b, tol=0.0, maxit=6)
    xg = x.cpu().numpy()
    s.close()
    del x, s, bands, b
    torch.cuda.empty_cache()
    hb, hrhs = gen.host(prob)
    ahat, diag = oracle.scale(g, hb, mode)
    del hb
    xo, ho, io = oracle.solve(g, mode, ahat, diag, hrhs, tol=tol, maxit=200)
    assert info.converged and info.true_R < tol and io.converged
    assert abs(info.iters - io.iters) <= 2
    assert np.linalg.norm(xg - xo) <= 10 * tol * np.linalg.norm(xo)
    bhat = hrhs / diag
    r = oracle.residual64(g, ahat, bhat, xg)
    assert np.linalg.norm(r) / np.linalg.norm(bhat) < tol
    del xo
    if hist_rtol is not None:
        _, hfo, _ = oracle.solve(g, mode, ahat, diag, hrhs, tol=0.0, maxit=6)
        keep = hfo >= 1e-5
        assert np.all(np.abs(hf[keep] - hfo[keep]) <= hist_rtol * hfo[keep])
    return info, io


@pytest.mark.parametrize("cfg", ["C3", "C4"])
def test_solve_matches_full_oracle_default_path(cfg):
    """BASELINE.json configs 3 and 4 (MIXED, tol 1e-4) on the default (fused) path."""
    _full_oracle_parity(gen.CONFIGS[cfg], "mixed", hist_rtol=1e-3)


def test_c5_fp64_solve_matches_full_oracle():
    """BASELINE.json config 5's fp64 variant: the all-fp64 solve against the fp64 oracle."""
    _full_oracle_parity(C5, "fp64", hist_rtol=1e-10)
