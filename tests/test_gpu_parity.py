"""GPU parity: the CUDA path through the C ABI against the CPU oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): apply rel-L2 <= 1e-13 (fp64) / <= 1e-6 (fp32, against the
oracle's fp64 evaluation of the same fp32 inputs); precondition <= 1e-12 / 1e-5;
solve: iterations within +-2, true residual < tol, ||x_gpu - x_orc|| / ||x_orc|| <= 10 tol,
fixed-iteration histories within 1e-3 (mixed / fp32) and 1e-10 (fp64) while R >= 1e-5.
"""
import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
egs = pytest.importorskip("paper_1811_03852_b200")

RAGGED = gen.Problem(200, 37, 13, seed=8)     # nx not a multiple of the 128-column tile, odd rows
SMALLEST = gen.Problem(3, 1, 1, seed=9)       # degenerate: one latitude row, one level
# columns at and past the kernels' limits: nz = 81 (> 80, the FP64 TMEM Thomas), 129 (> 128, the
# fp32 TMEM Thomas), 200 (the shared-memory Thomas with 32-column CTAs)
DEEP = [gen.Problem(64, 5, 81, seed=18), gen.Problem(64, 5, 129, seed=19), gen.Problem(40, 6, 200, seed=20)]
CASES = [gen.CONFIGS["C1"], RAGGED, gen.Problem(130, 9, 70, seed=10), SMALLEST] + DEEP
MODES = ["fp64", "mixed", "fp32"]


def _vnp(mode):
    return np.float64 if mode == "fp64" else np.float32


def _make(prob, mode, env=None, monkeypatch=None):
    bands, b = gen.host(prob)
    bd = torch.from_numpy(bands).cuda()
    # poison the caching allocator with NaN so that a read of an unwritten workspace element shows up
    junk = torch.full((4 * 7 * prob.n + (1 << 20),), float("nan"), dtype=torch.float64, device="cuda")
    del junk
    for k, v in (env or {}).items():
        monkeypatch.setenv(k, v)
    s = egs.Solver((prob.nx, prob.ny, prob.nz), bd, mode)
    for k in (env or {}):
        monkeypatch.delenv(k)
    return s, bands, b


def _uses_fused(s, b):
    """True iff the solver's iteration runs the fused phase kernels (one profiled iteration)."""
    s.profile_reset()
    s.solve(b, tol=0.0, maxit=1, flags=egs.EG_SOLVE_PROFILE)
    return s.profile()["phase_A"][1] == 1


def _rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


@pytest.mark.parametrize("prob", CASES, ids=lambda p: f"{p.nx}x{p.ny}x{p.nz}")
@pytest.mark.parametrize("mode", MODES)
def test_apply_parity(prob, mode):
    s, bands, _ = _make(prob, mode)
    g = (prob.nx, prob.ny, prob.nz)
    ahat, _ = oracle.scale(g, bands, mode)
    x = np.random.default_rng(1).standard_normal(prob.n).astype(_vnp(mode))
    y = s.apply(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
    yo = oracle.apply(g, ahat, x.astype(np.float64))
    assert _rel(y, yo) <= (1e-13 if mode == "fp64" else 1e-6)


@pytest.mark.parametrize("prob", CASES, ids=lambda p: f"{p.nx}x{p.ny}x{p.nz}")
@pytest.mark.parametrize("mode", MODES)
def test_precondition_parity(prob, mode):
    s, bands, _ = _make(prob, mode)
    g = (prob.nx, prob.ny, prob.nz)
    ahat, _ = oracle.scale(g, bands, mode)
    r = np.random.default_rng(2).standard_normal(prob.n).astype(_vnp(mode))
    z = s.precondition(torch.from_numpy(r).cuda()).cpu().numpy().astype(np.float64)
    zo = oracle.thomas(g, "fp64", ahat, r.astype(np.float64))
    assert _rel(z, zo) <= (1e-12 if mode == "fp64" else 1e-5)


FUSED_ODD = gen.Problem(128, 37, 13, seed=11)   # one 128-column tile, odd ny / nz
FUSED_THIN = gen.Problem(192, 3, 70, seed=12)   # fewer rows than the per-CTA row ranges
# below 2^18 points the default is the 5-kernel schedule: these cases force the fused phase kernels
# (march.cuh for fp32 vectors, march64.cuh for FP64)
FORCE_FUSED = (FUSED_ODD, FUSED_THIN)


@pytest.mark.parametrize("prob", [gen.CONFIGS["C1"], RAGGED, gen.Problem(130, 9, 70, seed=10), FUSED_ODD,
                                  FUSED_THIN] + DEEP, ids=lambda p: f"{p.nx}x{p.ny}x{p.nz}")
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("tol", [1e-3, 1e-4])
def test_solve_parity(prob, mode, tol, monkeypatch):
    fused = prob in FORCE_FUSED
    s, bands, b = _make(prob, mode, {"EG_FUSE": "1"} if fused else None, monkeypatch)
    if fused:
        assert _uses_fused(s, torch.from_numpy(b).cuda())
    g = (prob.nx, prob.ny, prob.nz)
    ahat, diag = oracle.scale(g, bands, mode)
    xo, ho, io = oracle.solve(g, mode, ahat, diag, b, tol=tol, maxit=200)
    x, info, h = s.solve(torch.from_numpy(b).cuda(), tol=tol, maxit=200)
    x = x.cpu().numpy()
    assert info.converged and io.converged
    assert abs(info.iters - io.iters) <= 2
    assert info.true_R < tol
    # true residual recomputed independently by the oracle in fp64 on the fp64 operator
    a64, d64 = oracle.scale(g, bands, "fp64")
    rt = oracle.residual64(g, a64, b / d64, x)
    assert np.linalg.norm(rt) / np.linalg.norm(b / d64) < tol
    assert _rel(x, xo) <= 10 * tol


@pytest.mark.parametrize("prob", [gen.CONFIGS["C1"], RAGGED, FUSED_ODD], ids=lambda p: f"{p.nx}x{p.ny}x{p.nz}")
@pytest.mark.parametrize("mode", MODES)
def test_fixed_iteration_history_parity(prob, mode, monkeypatch):
    s, bands, b = _make(prob, mode, {"EG_FUSE": "1"} if prob in FORCE_FUSED else None, monkeypatch)
    g = (prob.nx, prob.ny, prob.nz)
    ahat, diag = oracle.scale(g, bands, mode)
    _, ho, io = oracle.solve(g, mode, ahat, diag, b, tol=0.0, maxit=8)
    _, info, h = s.solve(torch.from_numpy(b).cuda(), tol=0.0, maxit=8)
    assert info.iters == io.iters == 8 and not info.converged
    keep = ho >= 1e-5
    rt = 1e-10 if mode == "fp64" else 1e-3
    assert np.all(np.abs(h[keep] - ho[keep]) <= rt * ho[keep])


def test_c2_mixed_vs_fp64_iteration_match():
    """BASELINE config 2: fp32 (mixed) solve vs all-fp64 solve, identical iteration counts."""
    prob = gen.CONFIGS["C2"]
    bands, b = gen.host(prob)
    bd = torch.from_numpy(bands).cuda()
    bt = torch.from_numpy(b).cuda()
    g = (prob.nx, prob.ny, prob.nz)
    res = {}
    for mode in ("mixed", "fp64"):
        s = egs.Solver(g, bd, mode)
        x, info, h = s.solve(bt, tol=1e-4, maxit=200)
        res[mode] = (x.cpu().numpy(), info, h)
        ahat, diag = oracle.scale(g, bands, mode)
        xo, ho, io = oracle.solve(g, mode, ahat, diag, b, tol=1e-4, maxit=200)
        assert abs(info.iters - io.iters) <= 2 and info.true_R < 1e-4
        assert _rel(res[mode][0], xo) <= 1e-3
    assert res["mixed"][1].iters == res["fp64"][1].iters
    assert abs(res["mixed"][2][1] - res["fp64"][2][1]) <= 5e-7 * res["fp64"][2][1]


def test_determinism_and_host_buffers():
    prob = RAGGED
    s, bands, b = _make(prob, "mixed")
    x1, i1, h1 = s.solve(torch.from_numpy(b).cuda(), tol=1e-5, maxit=100)
    x2, i2, h2 = s.solve(torch.from_numpy(b).cuda(), tol=1e-5, maxit=100)
    assert torch.equal(x1, x2) and np.array_equal(h1, h2)
    x3, i3, h3 = s.solve(b.copy(), tol=1e-5, maxit=100)            # host numpy in / out
    assert isinstance(x3, np.ndarray) and np.array_equal(x3, x1.cpu().numpy()) and np.array_equal(h3, h1)
    xg, ig, hg = s.solve(torch.from_numpy(b).cuda(), tol=1e-5, maxit=100, flags=egs.EG_SOLVE_NO_GRAPH)
    assert torch.equal(xg, x1) and np.array_equal(hg, h1)            # graph replay == direct launch


@pytest.mark.parametrize("fused", [False, True], ids=["5-kernel", "fused"])
@pytest.mark.parametrize("mode", MODES)
def test_warm_start_parity(mode, fused, monkeypatch):
    """Warm start (x0 != 0, the NEXT-4 workflow): the entry computes r0 = round(bhat - Ahat x0) with
    fp64 accumulation (k_start<ENTRY, !XZERO>) and the solve continues from x0.  Against the oracle's
    solve from the same x0: counts within +-2, x within 10 tol, and the fixed-iteration history."""
    prob = gen.Problem(128, 40, 20, seed=41)
    s, bands, b = _make(prob, mode, {"EG_FUSE": "1"} if fused else {"EG_NO_FUSE": "1"}, monkeypatch)
    g = (prob.nx, prob.ny, prob.nz)
    ahat, diag = oracle.scale(g, bands, mode)
    # x0: the oracle's 2-iteration iterate of a perturbed right-hand side (nonzero everywhere, smooth)
    x0, _, _ = oracle.solve(g, mode, ahat, diag, 1.1 * b + 0.01, tol=0.0, maxit=2)
    bt, x0t = torch.from_numpy(b).cuda(), torch.from_numpy(x0).cuda()
    if fused:
        assert _uses_fused(s, bt)
    tol = 1e-5 if mode != "fp32" else 1e-4
    xo, ho, io = oracle.solve(g, mode, ahat, diag, b, x0=x0, tol=tol, maxit=200)
    x, info, h = s.solve(bt, x0=x0t, tol=tol, maxit=200)
    assert io.converged and info.converged and abs(info.iters - io.iters) <= 2 and info.true_R < tol
    # true R of x0: fp64 sums, except FP32 mode's ||bhat|| (a binary32 sum, order-dependent rounding)
    assert h[0] == pytest.approx(ho[0], rel=1e-5 if mode == "fp32" else 1e-12)
    assert _rel(x.cpu().numpy(), xo) <= 10 * tol
    _, hf, _ = oracle.solve(g, mode, ahat, diag, b, x0=x0, tol=0.0, maxit=6)
    _, infof, hg = s.solve(bt, x0=x0t, tol=0.0, maxit=6)
    keep = hf >= 1e-5
    rt = 1e-10 if mode == "fp64" else 1e-3
    assert np.all(np.abs(hg[keep] - hf[keep]) <= rt * hf[keep])


def test_warm_start_and_zero_iterations():
    prob = gen.CONFIGS["C1"]
    s, bands, b = _make(prob, "fp64")
    x, info, _ = s.solve(torch.from_numpy(b).cuda(), tol=1e-10, maxit=200)
    x2, info2, h2 = s.solve(torch.from_numpy(b).cuda(), x0=x.clone(), tol=1e-8, maxit=200)
    assert info2.iters == 0 and info2.converged and torch.equal(x2, x)


@pytest.mark.parametrize("mode", MODES)
def test_solution_stays_zero_without_iterations(mode):
    """From x0 = 0 the entry does not store x (the first update starts from 0): a solve that stops
    before any update must still return exactly x = 0 in a NaN-poisoned output buffer (converged at
    the start with tol > R_0 = 1, or maxit = 0), and the host-buffer path must agree."""
    prob = gen.CONFIGS["C1"]
    s, bands, b = _make(prob, mode)
    bt = torch.from_numpy(b).cuda()
    for tol, maxit in ((2.0, 200), (1e-6, 0)):
        out = torch.full((prob.n,), float("nan"), dtype=torch.float64, device="cuda")
        x, info, h = s.solve(bt, tol=tol, maxit=maxit, out=out)
        assert info.iters == 0 and bool(torch.all(x == 0.0)), (tol, maxit)
        xh = np.full(prob.n, np.nan)
        xh, info_h, _ = s.solve(b, tol=tol, maxit=maxit, out=xh)
        assert info_h.iters == 0 and np.all(xh == 0.0)
    # one iteration from x0 = 0 equals one iteration from an explicit zero x0
    x1, i1, h1 = s.solve(bt, tol=0.0, maxit=1)
    x2, i2, h2 = s.solve(bt, x0=torch.zeros(prob.n, dtype=torch.float64, device="cuda"), tol=0.0, maxit=1)
    assert np.array_equal(h1, h2) and torch.equal(x1, x2)


def test_power_of_two_scaling_bitwise():
    prob = RAGGED
    s, bands, b = _make(prob, "mixed")
    x1, i1, h1 = s.solve(torch.from_numpy(b).cuda(), tol=1e-5, maxit=100)
    x2, i2, h2 = s.solve(torch.from_numpy(4.0 * b).cuda(), tol=1e-5, maxit=100)
    assert np.array_equal(h1, h2) and torch.equal(4.0 * x1, x2)


def test_restart_bookkeeping_matches_oracle():
    prob = gen.Problem(64, 48, 10, seed=3)
    s, bands, b = _make(prob, "fp64")
    g = (prob.nx, prob.ny, prob.nz)
    ahat, diag = oracle.scale(g, bands, "fp64")
    _, ho, io = oracle.solve(g, "fp64", ahat, diag, b, tol=1e-9, maxit=200, restart_every=3)
    _, info, h = s.solve(torch.from_numpy(b).cuda(), tol=1e-9, maxit=200, restart_every=3)
    assert info.restarts == io.restarts and info.iters == io.iters and info.converged


def test_error_paths():
    prob = gen.Problem(16, 8, 4, seed=4)
    bands, b = gen.host(prob)
    g = (prob.nx, prob.ny, prob.nz)
    bad = bands.copy(); bad[0, 7] = 0.0
    with pytest.raises(egs.EgError) as e:
        egs.Solver(g, torch.from_numpy(bad).cuda(), "mixed")
    assert e.value.status == 2
    bad = bands.copy(); bad[5, prob.nx * (prob.nz - 1)] = -1.0      # U band on the top level
    with pytest.raises(egs.EgError) as e:
        egs.Solver(g, torch.from_numpy(bad).cuda(), "mixed")
    assert e.value.status == 1
    s = egs.Solver(g, torch.from_numpy(bands).cuda(), "mixed")
    with pytest.raises(egs.EgError) as e:
        s.solve(torch.zeros(prob.n, dtype=torch.float64, device="cuda"))
    assert e.value.status == 3
    # the degenerate right-hand side leaves x = 0 (the entry does not store it; the exit does)
    out = torch.full((prob.n,), float("nan"), dtype=torch.float64, device="cuda")
    _, info, _ = s.solve(torch.zeros(prob.n, dtype=torch.float64, device="cuda"), out=out, raise_on_error=False)
    assert info.status == 3 and bool(torch.all(out == 0.0))
    bb = b.copy(); bb[5] = np.nan
    _, info, _ = s.solve(torch.from_numpy(bb).cuda(), raise_on_error=False)
    assert info.status == 5
    # argument validation (EG_ERR_ARG before any device work), then the handle still solves
    bt = torch.from_numpy(b).cuda()
    for kw in (dict(maxit=-1), dict(tol=float("nan")), dict(tol=-1.0)):
        with pytest.raises(egs.EgError) as e:
            s.solve(bt, **kw)
        assert e.value.status == 1, kw
    for args in (("trisor", 0, 1.5), ("trisor", 3, 2.0), ("trisor", 3, 0.0), ("nonsense", 3, 1.5)):
        with pytest.raises((egs.EgError, KeyError)):
            s.set_preconditioner(*args)
    podd = gen.Problem(15, 8, 4, seed=4)  # nx odd: no red-black colouring
    bo, _ = gen.host(podd)
    so = egs.Solver((podd.nx, podd.ny, podd.nz), torch.from_numpy(bo).cuda(), "mixed")
    with pytest.raises(egs.EgError) as e:
        so.set_preconditioner("trisor")
    assert e.value.status == 1
    x, info, _ = s.solve(bt, tol=1e-6, maxit=50)
    assert info.status == 0 and info.converged


def test_no_horizontal_coupling_one_iteration():
    prob = gen.Problem(130, 6, 10, seed=5, ch=(0.0, 0.0))
    s, bands, b = _make(prob, "mixed")
    x, info, h = s.solve(torch.from_numpy(b).cuda(), tol=1e-4, maxit=20)
    assert info.iters == 1 and info.converged


def test_profile_counts_kernels():
    prob = gen.CONFIGS["C1"]
    s, bands, b = _make(prob, "mixed")
    s.profile_reset()
    s.solve(torch.from_numpy(b).cuda(), tol=0.0, maxit=4, flags=egs.EG_SOLVE_PROFILE)
    p = s.profile()
    fused = p["phase_A"][1] > 0
    names = ("phase_A", "phase_B", "update_xr") if fused else (
        "thomas_p", "stencil_dot_A", "thomas_s", "stencil_dot_B", "update_xr")
    for k in names:
        assert p[k][1] == 4 and p[k][0] > 0 and p[k][2] > 0


@pytest.mark.parametrize("mode", ["mixed", "fp64"])
@pytest.mark.parametrize("transport", ["p2p", "nccl"])
def test_multirank_finaliser_path_bitwise_equal(mode, transport, monkeypatch):
    """EG_FORCE_NCCL=1 runs one GPU through the multi-rank path (local row-group sums -> the
    all-gather -> logic kernel, captured in the iteration graph): by the group kernels' own pushes
    and flags (P2P transport, the default) or ncclAllGather (EG_P2P=0).  The fixed grouping makes
    it bitwise identical to the single-GPU finaliser."""
    prob = RAGGED
    bands, b = gen.host(prob)
    g = (prob.nx, prob.ny, prob.nz)
    bd = torch.from_numpy(bands).cuda()
    s1 = egs.Solver(g, bd, mode)
    x1, i1, h1 = s1.solve(torch.from_numpy(b).cuda(), tol=1e-6, maxit=100)
    monkeypatch.setenv("EG_FORCE_NCCL", "1")
    monkeypatch.setenv("EG_FUSE", "1")
    if transport == "nccl":
        monkeypatch.setenv("EG_P2P", "0")
    s2 = egs.Solver(g, bd, mode)
    monkeypatch.delenv("EG_FORCE_NCCL")
    monkeypatch.delenv("EG_FUSE")
    monkeypatch.delenv("EG_P2P", raising=False)
    assert s2.transport == transport and s1.transport == "none"
    x2, i2, h2 = s2.solve(torch.from_numpy(b).cuda(), tol=1e-6, maxit=100)
    assert i1.iters == i2.iters and np.array_equal(h1, h2) and torch.equal(x1, x2)
    if mode == "mixed":  # the fused phases run on the multi-rank path too (edge rows + ghost rows)
        s2.profile_reset()
        s2.solve(torch.from_numpy(b).cuda(), tol=0.0, maxit=2, flags=egs.EG_SOLVE_PROFILE)
        assert s2.profile()["phase_A"][1] == 2
    y1 = s1.apply(torch.ones(prob.n, dtype=s1.vdtype, device="cuda"))
    y2 = s2.apply(torch.ones(prob.n, dtype=s2.vdtype, device="cuda"))
    assert torch.equal(y1, y2)


MARCH_CASES = [gen.CONFIGS["C1"], RAGGED, FUSED_ODD, FUSED_THIN, gen.CONFIGS["C2"],
               gen.Problem(388, 23, 70, seed=13),   # 4 tiles (last one 4 columns wide), nz = 70
               gen.Problem(8, 5, 1, seed=14),       # one level: the Thomas solve is the identity
               gen.Problem(132, 6, 72, seed=15)]    # the deepest column the fused kernels take


@pytest.mark.parametrize("prob", MARCH_CASES, ids=lambda p: f"{p.nx}x{p.ny}x{p.nz}")
@pytest.mark.parametrize("mode", ["mixed", "fp32", "fp64"])
@pytest.mark.parametrize("strips", [None, 1, 2, 3])
def test_fused_phases_match_unfused_schedule(prob, mode, strips, monkeypatch):
    """The fused marching phase kernels (march.cuh for fp32 vectors, march64.cuh for FP64: Thomas +
    stencil of a latitude strip per CTA, the default from 2^18 local points; EG_FUSE=1 forces them
    here) compute z, v, s, t with the same operations as the 5-kernel schedule (EG_NO_FUSE=1) and
    write the same reduction sums (FP64: 64-column half-slots combined in k_stencil's warp order), so
    the solve is bitwise identical, whatever the number of strips (EG_MARCH_STRIPS: one-row strips,
    one strip per tile column, odd counts whose strips alternate direction)."""
    bands, b = gen.host(prob)
    g = (prob.nx, prob.ny, prob.nz)
    bd = torch.from_numpy(bands).cuda()
    bt = torch.from_numpy(b).cuda()
    if strips is not None:
        monkeypatch.setenv("EG_MARCH_STRIPS", str(strips))
    monkeypatch.setenv("EG_FUSE", "1")   # small grids default to the 5-kernel schedule
    s1 = egs.Solver(g, bd, mode)
    monkeypatch.delenv("EG_FUSE")
    monkeypatch.delenv("EG_MARCH_STRIPS", raising=False)
    monkeypatch.setenv("EG_NO_FUSE", "1")
    s2 = egs.Solver(g, bd, mode)
    monkeypatch.delenv("EG_NO_FUSE")
    # fixed iterations; to tolerance; with a restart every 3 iterations (fresh phase A each time)
    for tol, maxit, rs in ((0.0, 8, 150), (1e-5, 100, 150), (0.0, 10, 3)):
        x1, i1, h1 = s1.solve(bt, tol=tol, maxit=maxit, restart_every=rs)
        x2, i2, h2 = s2.solve(bt, tol=tol, maxit=maxit, restart_every=rs)
        assert i1.iters == i2.iters and i1.restarts == i2.restarts
        assert np.array_equal(h1, h2) and torch.equal(x1, x2)
    for s, fused in ((s1, True), (s2, False)):
        s.profile_reset()
        s.solve(bt, tol=0.0, maxit=3, flags=egs.EG_SOLVE_PROFILE)
        p = s.profile()
        assert (p["phase_A"][1], p["phase_B"][1], p["thomas_p"][1]) == ((3, 3, 0) if fused else (0, 0, 3))


@pytest.mark.parametrize("prob", [gen.Problem(130, 9, 70, seed=10), gen.Problem(64, 8, 73, seed=16)],
                         ids=lambda p: f"{p.nx}x{p.ny}x{p.nz}")
def test_fused_phases_fall_back_outside_their_domain(prob):
    """nx % 4 != 0 (16-byte TMA strides) or nz > 72 (TMEM columns): the 5-kernel schedule runs."""
    s, _, b = _make(prob, "mixed")
    s.profile_reset()
    s.solve(torch.from_numpy(b).cuda(), tol=0.0, maxit=2, flags=egs.EG_SOLVE_PROFILE)
    p = s.profile()
    assert p["phase_A"][1] == 0 and p["thomas_p"][1] == 2


# nx = 130 / 132 / 136: the second colour's colour-split rows start at byte 260 / 264 / 272 (fp32),
# 520 / 528 / 544 (FP64); the TMA sweeps need a 16-byte boundary there and fall back otherwise
TRISOR_CASES = [gen.Problem(64, 48, 10, seed=0), gen.Problem(130, 9, 70, seed=10), gen.Problem(128, 37, 13, seed=11),
                gen.Problem(132, 7, 13, seed=21), gen.Problem(136, 7, 70, seed=22),
                gen.Problem(64, 6, 100, seed=24)]  # nz > 72: the TMA sweeps' TMEM limit, k_sor_half runs


@pytest.mark.parametrize("prob", TRISOR_CASES, ids=lambda p: f"{p.nx}x{p.ny}x{p.nz}")
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("sweeps,omega", [(1, 1.0), (3, 1.5)])
def test_trisor_precondition_parity(prob, mode, sweeps, omega):
    """NEXT-1: the GPU red-black tri-SOR sweeps against the oracle's Eq. 7 sweeps, on the natural
    arrays and on the colour-split copies (EG_FEATURE_TRISOR), which give bitwise the same z."""
    s, bands, _ = _make(prob, mode)
    s.set_preconditioner("trisor", sweeps=sweeps, omega=omega)
    g = (prob.nx, prob.ny, prob.nz)
    ahat, _ = oracle.scale(g, bands, mode)
    f = np.random.default_rng(3).standard_normal(prob.n).astype(_vnp(mode))
    z = s.precondition(torch.from_numpy(f).cuda())
    zo = oracle.trisor(g, "fp64", ahat, f.astype(np.float64), sweeps=sweeps, omega=omega)
    assert _rel(z.cpu().numpy().astype(np.float64), zo) <= (1e-12 if mode == "fp64" else 1e-5)
    st = egs.Solver(g, torch.from_numpy(bands).cuda(), mode, trisor=True)
    st.set_preconditioner("trisor", sweeps=sweeps, omega=omega)
    assert torch.equal(st.precondition(torch.from_numpy(f).cuda()), z)


@pytest.mark.parametrize("mode", MODES)
def test_trisor_solve_parity(mode):
    prob = gen.Problem(64, 48, 20, seed=46, cv=(5.0, 20.0), dl=(1e-3, 1e-2))
    s, bands, b = _make(prob, mode)
    s.set_preconditioner("trisor", sweeps=3, omega=1.5)
    g = (prob.nx, prob.ny, prob.nz)
    ahat, diag = oracle.scale(g, bands, mode)
    tol = 1e-4
    xo, ho, io = oracle.solve(g, mode, ahat, diag, b, tol=tol, maxit=200, sor_sweeps=3, sor_omega=1.5)
    x, info, h = s.solve(torch.from_numpy(b).cuda(), tol=tol, maxit=200)
    assert info.converged and io.converged and abs(info.iters - io.iters) <= 2 and info.true_R < tol
    assert _rel(x.cpu().numpy(), xo) <= 10 * tol
    st = egs.Solver(g, torch.from_numpy(bands).cuda(), mode, trisor=True)   # colour-split copies
    st.set_preconditioner("trisor", sweeps=3, omega=1.5)
    xs, infos, hs = st.solve(torch.from_numpy(b).cuda(), tol=tol, maxit=200)
    assert infos.iters == info.iters and np.array_equal(hs, h) and torch.equal(xs, x)
    st.set_operator(torch.from_numpy(bands).cuda() * 2.0)   # new operator -> split copies refreshed
    xs2, infos2, _ = st.solve(torch.from_numpy(b).cuda() * 2.0, tol=tol, maxit=200)
    assert infos2.iters == info.iters and torch.equal(xs2, x)  # (2A) x = 2b: same scaled system
    s.set_preconditioner("tridiag")
    _, info1, _ = s.solve(torch.from_numpy(b).cuda(), tol=tol, maxit=200)
    assert info.iters < info1.iters      # the paper's preconditioner is the stronger one
    with pytest.raises(egs.EgError):
        _make(gen.Problem(65, 4, 4, seed=1), mode)[0].set_preconditioner("trisor")   # odd nx


def test_fused_phases_repeatable_at_scale(monkeypatch):
    """Race check of the fused phase kernels on a multi-strip grid (C3: 5 tiles x 29 strips of
    ~17 rows): repeated solves, each with a new output buffer (so the iteration graph is
    re-captured), are bitwise identical to one another and to the 5-kernel schedule."""
    prob = gen.CONFIGS["C3"]
    bands = torch.empty((7, prob.n), dtype=torch.float64, device="cuda")
    b = torch.empty(prob.n, dtype=torch.float64, device="cuda")
    gen.device(prob, bands, b)
    g = (prob.nx, prob.ny, prob.nz)
    monkeypatch.setenv("EG_NO_FUSE", "1")
    ref = egs.Solver(g, bands, "mixed")
    monkeypatch.delenv("EG_NO_FUSE")
    x0, i0, h0 = ref.solve(b, tol=1e-6, maxit=200)
    s = egs.Solver(g, bands, "mixed")
    keep = []
    for _ in range(6):
        x, info, h = s.solve(b, tol=1e-6, maxit=200)
        keep.append(x)
        assert info.iters == i0.iters and np.array_equal(h, h0) and torch.equal(x, x0)


def test_fused_phases_repeatable_table1_sequence():
    """Regression test for a stage-refill race (fixed with fence.proxy.async before each stage
    release): two fused solvers driven like the Table 1 study (set_operator + solve at 1e-3, then
    at 1e-4, per date) on the hard operator at C4 size must agree bitwise.  Before the fix about one
    solve in six differed."""
    base = gen.CONFIGS["C4"].with_(cv=(5.0, 20.0), dl=(1e-4, 1e-3))
    g = (base.nx, base.ny, base.nz)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        bands = torch.empty((7, base.n), dtype=torch.float64, device="cuda")
        b = torch.empty(base.n, dtype=torch.float64, device="cuda")
        x = torch.empty(base.n, dtype=torch.float64, device="cuda")
        gen.device(base, bands, b, stream=st)
        sv = [egs.Solver(g, bands, "mixed", stream=st) for _ in range(2)]
        for d in range(6):
            gen.device(base.with_(seed=4 + d), bands, b, stream=st)
            out = {}
            for si, s in enumerate(sv):
                for tol in (1e-3, 1e-4):
                    s.set_operator(bands)
                    _, info, h = s.solve(b, tol=tol, maxit=200, out=x)
                    out[(si, tol)] = (x.clone(), info.iters, h)
            for tol in (1e-3, 1e-4):
                (x0, i0, h0), (x1, i1, h1) = out[(0, tol)], out[(1, tol)]
                assert i0 == i1 and np.array_equal(h0, h1) and torch.equal(x0, x1), (d, tol)


def test_solve_batch_matches_individual_solves():
    """eg_solve_batch overlaps the transfers of neighbouring solves (copy streams, two staging
    buffers each for b and x): every solve's x, iteration count and status are those of the
    individual eg_solve call, for pinned host, pageable (numpy) and device buffers, with and without
    re-scaling the operator before each solve."""
    prob = gen.Problem(128, 40, 20, seed=17)
    bands, b0 = gen.host(prob)
    g = (prob.nx, prob.ny, prob.nz)
    bd = torch.from_numpy(bands).cuda()
    s = egs.Solver(g, bd, "mixed", batch=True)
    rng = np.random.default_rng(5)
    bs = [b0 * (1.0 + 0.1 * k) + 0.01 * rng.standard_normal(prob.n) for k in range(5)]
    ref = [s.solve(torch.from_numpy(v).cuda(), tol=1e-6, maxit=100) for v in bs]
    # pinned host buffers, operator re-scaled before every solve
    hb = [torch.from_numpy(v).pin_memory() for v in bs]
    hx = [torch.empty(prob.n, dtype=torch.float64).pin_memory() for _ in bs]
    infos = s.solve_batch(hb, hx, bands=bd, tol=1e-6, maxit=100)
    for (x, i, _), xh, ib in zip(ref, hx, infos):
        assert ib.iters == i.iters and ib.converged and torch.equal(xh, x.cpu())
    # pageable numpy and device buffers
    nx_ = [np.empty(prob.n) for _ in bs]
    s.solve_batch(bs, nx_, tol=1e-6, maxit=100)
    dx = [torch.empty(prob.n, dtype=torch.float64, device="cuda") for _ in bs]
    s.solve_batch([torch.from_numpy(v).cuda() for v in bs], dx, tol=1e-6, maxit=100)
    for (x, _, _), xn, xd in zip(ref, nx_, dx):
        assert np.array_equal(xn, x.cpu().numpy()) and torch.equal(xd, x)
    assert s.solve_batch([], [], tol=1e-6) == []
    with pytest.raises(egs.EgError):   # no EG_FEATURE_BATCH staging in the workspace
        egs.Solver(g, bd, "mixed").solve_batch(hb[:1], hx[:1], tol=1e-6)


def test_solve_batch_stops_at_the_first_failing_solve():
    """A degenerate right-hand side in the middle of a sequence: the earlier solves complete with
    their usual results, the batch returns that solve's status and reports how many completed."""
    prob = gen.Problem(64, 16, 10, seed=18)
    bands, b0 = gen.host(prob)
    g = (prob.nx, prob.ny, prob.nz)
    s = egs.Solver(g, torch.from_numpy(bands).cuda(), "mixed", batch=True)
    bs = [b0, 2.0 * b0, np.zeros(prob.n), b0]
    xs = [np.full(prob.n, np.nan) for _ in bs]
    with pytest.raises(egs.EgError) as e:
        s.solve_batch(bs, xs, tol=1e-6, maxit=50)
    assert e.value.status == 3
    infos = s.solve_batch(bs, xs, tol=1e-6, maxit=50, raise_on_error=False)
    assert len(infos) == 2 and all(i.converged and i.status == 0 for i in infos)
    x0, _, _ = s.solve(torch.from_numpy(b0).cuda(), tol=1e-6, maxit=50)
    assert np.array_equal(xs[0], x0.cpu().numpy()) and np.array_equal(xs[1], 2.0 * xs[0])
    assert np.isnan(xs[3]).all()  # never started


def test_concurrent_fused_solves_on_two_streams(monkeypatch):
    """Two handles solving at the same time from two threads, each on its own stream, with the fused
    phase kernels (which need all their CTAs resident): the library serialises such solves, so both
    finish and give bitwise the results of the same solves run one after the other."""
    import threading
    monkeypatch.setenv("EG_FUSE", "1")
    probs = [gen.Problem(192, 144, 70, seed=1), gen.Problem(256, 96, 70, seed=2)]
    sts = [torch.cuda.Stream() for _ in probs]
    solvers, rhs = [], []
    for p, st in zip(probs, sts):
        bands, b = gen.host(p)
        solvers.append(egs.Solver((p.nx, p.ny, p.nz), torch.from_numpy(bands).cuda(), "mixed", stream=st))
        rhs.append(torch.from_numpy(b).cuda())
    torch.cuda.synchronize()
    seq = [s.solve(b, tol=0.0, maxit=12)[0].clone() for s, b in zip(solvers, rhs)]
    outs = [torch.empty_like(x) for x in seq]
    errs = []

    def run(k):
        try:
            for _ in range(5):
                solvers[k].solve(rhs[k], tol=0.0, maxit=12, out=outs[k])
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=run, args=(k,)) for k in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(120)
    assert not any(t.is_alive() for t in ts) and not errs
    torch.cuda.synchronize()
    assert all(torch.equal(o, x) for o, x in zip(outs, seq))


@pytest.mark.parametrize("prob", [gen.CONFIGS["C1"], gen.Problem(200, 37, 13, seed=8), gen.Problem(388, 23, 70, seed=13)],
                         ids=lambda p: f"{p.nx}x{p.ny}x{p.nz}")
def test_fp64_thomas_tma_matches_tmem_kernel(prob, monkeypatch):
    """The FP64 iteration's Thomas solves on the TMA-fed kernel (k_thomas_tma64, the default for
    nz <= 72) give bitwise the results of the TMEM-factor kernel (EG_NO_THOMAS_TMA=1).  (5-kernel
    schedule: the FP64 fused phase kernels take over some of these grids by default.)"""
    monkeypatch.setenv("EG_NO_FUSE", "1")
    bands, b = gen.host(prob)
    g = (prob.nx, prob.ny, prob.nz)
    bd = torch.from_numpy(bands).cuda()
    bt = torch.from_numpy(b).cuda()
    s1 = egs.Solver(g, bd, "fp64")
    monkeypatch.setenv("EG_NO_THOMAS_TMA", "1")
    s2 = egs.Solver(g, bd, "fp64")
    monkeypatch.delenv("EG_NO_THOMAS_TMA")
    for kw in (dict(tol=1e-10, maxit=60, restart_every=5), dict(tol=0.0, maxit=8)):
        x1, i1, h1 = s1.solve(bt, **kw)
        x2, i2, h2 = s2.solve(bt, **kw)
        assert i1.iters == i2.iters and np.array_equal(h1, h2) and torch.equal(x1, x2)
    s1.profile_reset()
    s1.solve(bt, tol=0.0, maxit=2, flags=egs.EG_SOLVE_PROFILE)
    assert s1.profile()["thomas_p"][1] == 2


@pytest.mark.parametrize("mode", ["mixed", "fp64"])
def test_trisor_split_bands_from_set_operator_bitwise(mode):
    """With tri-SOR selected, set_operator writes the colour-split band copies in the scaling pass;
    otherwise they are derived before the first solve (never inside the captured iteration graph).
    Both give bitwise the same solve, graph replay or not."""
    prob = gen.Problem(136, 20, 13, seed=23)
    bands, b = gen.host(prob)
    g = (prob.nx, prob.ny, prob.nz)
    bd = torch.from_numpy(bands).cuda()
    bt = torch.from_numpy(b).cuda()
    s1 = egs.Solver(g, bd, mode, trisor=True)
    s1.set_preconditioner("trisor", sweeps=3, omega=1.5)      # split copies derived at the solve
    x1, i1, h1 = s1.solve(bt, tol=1e-8, maxit=40)
    s2 = egs.Solver(g, 2.0 * bd, mode, trisor=True)            # another operator first
    s2.set_preconditioner("trisor", sweeps=3, omega=1.5)
    s2.solve(bt, tol=1e-8, maxit=40)
    s2.set_operator(bd)                                        # split copies written by the scaling pass
    x2, i2, h2 = s2.solve(bt, tol=1e-8, maxit=40)
    x3, i3, h3 = s2.solve(bt, tol=1e-8, maxit=40, flags=egs.EG_SOLVE_NO_GRAPH)
    assert i1.iters == i2.iters == i3.iters and np.array_equal(h1, h2) and np.array_equal(h1, h3)
    assert torch.equal(x1, x2) and torch.equal(x1, x3)


# seeded random shapes (ragged tiles, odd / tiny rows and levels, both schedules): apply, precondition
# and a short solve against the oracle; FP64 / MIXED / FP32 in turn
_RNG = np.random.default_rng(2026)
RANDOM_SHAPES = [gen.Problem(int(_RNG.integers(3, 300)), int(_RNG.integers(1, 40)), int(_RNG.integers(1, 90)),
                             seed=100 + k) for k in range(12)]


@pytest.mark.parametrize("k", range(len(RANDOM_SHAPES)))
def test_random_shapes_parity(k, monkeypatch):
    prob = RANDOM_SHAPES[k]
    mode = MODES[k % 3]
    env = {"EG_FUSE": "1"} if k % 2 == 0 else {"EG_NO_FUSE": "1"}
    s, bands, b = _make(prob, mode, env, monkeypatch)
    g = (prob.nx, prob.ny, prob.nz)
    ahat, diag = oracle.scale(g, bands, mode)
    x = np.random.default_rng(k).standard_normal(prob.n).astype(_vnp(mode))
    y = s.apply(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
    assert _rel(y, oracle.apply(g, ahat, x.astype(np.float64))) <= (1e-13 if mode == "fp64" else 1e-6)
    z = s.precondition(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
    assert _rel(z, oracle.thomas(g, "fp64", ahat, x.astype(np.float64))) <= (1e-12 if mode == "fp64" else 1e-5)
    tol = 1e-4
    xo, ho, io = oracle.solve(g, mode, ahat, diag, b, tol=tol, maxit=200)
    xg, info, h = s.solve(torch.from_numpy(b).cuda(), tol=tol, maxit=200)
    assert io.converged and info.converged and abs(info.iters - io.iters) <= 2 and info.true_R < tol
    assert _rel(xg.cpu().numpy(), xo) <= 10 * tol


@pytest.mark.parametrize("mode", ["mixed", "fp32", "fp64"])
@pytest.mark.parametrize("sched", ["EG_FUSE", "EG_NO_FUSE"])
def test_programmatic_dependent_launch_bitwise(mode, sched, monkeypatch):
    """EG_PDL=1 (programmatic dependent launches of the iteration's kernels, fused or 5-kernel
    schedule) changes no result."""
    prob = gen.Problem(256, 40, 30, seed=33)
    bands, b = gen.host(prob)
    g = (prob.nx, prob.ny, prob.nz)
    bd, bt = torch.from_numpy(bands).cuda(), torch.from_numpy(b).cuda()
    monkeypatch.setenv(sched, "1")
    s1 = egs.Solver(g, bd, mode)
    monkeypatch.setenv("EG_PDL", "1")
    s2 = egs.Solver(g, bd, mode)
    for kw in (dict(tol=0.0, maxit=8), dict(tol=1e-6, maxit=100, restart_every=4)):
        x1, i1, h1 = s1.solve(bt, **kw)
        x2, i2, h2 = s2.solve(bt, **kw)
        assert i1.iters == i2.iters and np.array_equal(h1, h2) and torch.equal(x1, x2)


_RNG_T = np.random.default_rng(1853)
RANDOM_TRISOR = [gen.Problem(2 * int(_RNG_T.integers(2, 150)), int(_RNG_T.integers(1, 40)), int(_RNG_T.integers(1, 90)),
                             seed=200 + k) for k in range(8)]  # nx even: red-black tri-SOR


@pytest.mark.parametrize("k", range(len(RANDOM_TRISOR)))
def test_random_trisor_parity(k):
    """NEXT-1 on seeded random shapes (nz up to 89: both the TMA sweeps and k_sor_half): the
    tri-SOR sweeps against the oracle's Eq. 7 sweeps, natural and colour-split arrays bitwise equal,
    and a tri-SOR solve that converges with the oracle's solution."""
    prob = RANDOM_TRISOR[k]
    mode = MODES[k % 3]
    sweeps, omega = (3, 1.5) if k % 2 == 0 else (2, 1.2)
    s, bands, b = _make(prob, mode)
    s.set_preconditioner("trisor", sweeps=sweeps, omega=omega)
    g = (prob.nx, prob.ny, prob.nz)
    ahat, diag = oracle.scale(g, bands, mode)
    f = np.random.default_rng(k).standard_normal(prob.n).astype(_vnp(mode))
    z = s.precondition(torch.from_numpy(f).cuda())
    zo = oracle.trisor(g, "fp64", ahat, f.astype(np.float64), sweeps=sweeps, omega=omega)
    assert _rel(z.cpu().numpy().astype(np.float64), zo) <= (1e-12 if mode == "fp64" else 1e-5), (prob, mode)
    st = egs.Solver(g, torch.from_numpy(bands).cuda(), mode, trisor=True)
    st.set_preconditioner("trisor", sweeps=sweeps, omega=omega)
    assert torch.equal(st.precondition(torch.from_numpy(f).cuda()), z), (prob, mode)
    tol = 1e-4
    xo, ho, io = oracle.solve(g, mode, ahat, diag, b, tol=tol, maxit=200)
    xg, info, h = st.solve(torch.from_numpy(b).cuda(), tol=tol, maxit=200)
    assert info.converged and info.true_R < tol, (prob, mode, info)
    assert _rel(xg.cpu().numpy(), xo) <= 50 * tol, (prob, mode)
