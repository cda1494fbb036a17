"""GPU parity of the breakdown / restart branch (reading A-12; restart P:553-557) against
the oracle, on the hand-built cases of tests/_cases.py whose breakdowns are exact zeros (pinned by
tests/test_oracle_breakdown.py).  Status, iteration count, restart and breakdown counts must EQUAL
the oracle's; x within the solve tolerance of the oracle's; a breakdown of a caller-given rhat0
restarts into the plain solve, bitwise.  Run on the 5-kernel schedule, the fused phase kernels
(EG_FUSE=1), the multi-rank finaliser path (EG_FORCE_NCCL=1) and the in-process 2-rank bands."""
import threading

import numpy as np
import pytest

import oracle
from _cases import (NX, NY, dyadic_rhs, identity_operator, ring_operator, shadow_rho_tiny,
                    shadow_rho_zero, shadow_sigma_zero, unit_rhs)

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
egs = pytest.importorskip("paper_1811_03852_b200")

MODES = ["fp64", "mixed", "fp32"]
G = (NX, NY, 1)
TOL = {"fp64": 1e-8, "mixed": 1e-6, "fp32": 1e-5}
SCHEDULES = {"5-kernel": {"EG_NO_FUSE": "1"}, "fused": {"EG_FUSE": "1"}, "nccl1": {"EG_FORCE_NCCL": "1"}}


def _solver(bands, mode, env, monkeypatch):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    s = egs.Solver(G, torch.from_numpy(bands).cuda(), mode)
    for k in env:
        monkeypatch.delenv(k)
    return s


def _oracle(bands, b, mode, **kw):
    ahat, diag = oracle.scale(G, bands, mode)
    return oracle.solve(G, mode, ahat, diag, b, **kw)


def _same_counts(info, io):
    assert (info.status, info.iters, info.restarts, info.breakdowns, bool(info.converged)) == \
        (io.status, io.iters, io.restarts, io.breakdowns, bool(io.converged))


@pytest.mark.parametrize("sched", list(SCHEDULES))
@pytest.mark.parametrize("mode", MODES)
def test_identity_operator_tol0_breakdown_error(mode, sched, monkeypatch):
    bands, b = identity_operator(), dyadic_rhs()
    s = _solver(bands, mode, SCHEDULES[sched], monkeypatch)
    out = torch.full((b.size,), float("nan"), dtype=torch.float64, device="cuda")
    x, info, h = s.solve(torch.from_numpy(b).cuda(), tol=0.0, maxit=10, out=out, raise_on_error=False)
    xo, ho, io = _oracle(bands, b, mode, tol=0.0, maxit=10)
    assert io.status == 4
    _same_counts(info, io)
    assert bool(torch.all(x == 0.0))
    with pytest.raises(egs.EgError) as e:
        s.solve(torch.from_numpy(b).cuda(), tol=0.0, maxit=10)
    assert e.value.status == 4


@pytest.mark.parametrize("sched", list(SCHEDULES))
@pytest.mark.parametrize("mode", MODES)
def test_identity_operator_s_step_exit(mode, sched, monkeypatch):
    bands, b = identity_operator(c=2.0), dyadic_rhs()
    s = _solver(bands, mode, SCHEDULES[sched], monkeypatch)
    x, info, h = s.solve(torch.from_numpy(b).cuda(), tol=1e-6, maxit=10)
    xo, ho, io = _oracle(bands, b, mode, tol=1e-6, maxit=10)
    _same_counts(info, io)
    assert np.array_equal(x.cpu().numpy(), xo) and h[1] == 0.0


@pytest.mark.parametrize("mode", MODES)
def test_exact_initial_guess_tol0_breakdown_at_start(mode, monkeypatch):
    bands, b = identity_operator(c=2.0), dyadic_rhs(seed=1)
    x0 = b / 2.0
    s = _solver(bands, mode, {}, monkeypatch)
    x, info, h = s.solve(torch.from_numpy(b).cuda(), x0=torch.from_numpy(x0).cuda(), tol=0.0, maxit=10,
                         raise_on_error=False)
    _, _, io = _oracle(bands, b, mode, x0=x0, tol=0.0, maxit=10)
    _same_counts(info, io)
    assert np.array_equal(x.cpu().numpy(), x0)


@pytest.mark.parametrize("sched", list(SCHEDULES))
@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("shadow", [shadow_sigma_zero, shadow_rho_zero, shadow_rho_tiny],
                         ids=["sigma0", "rho0", "rho_tiny"])
def test_given_shadow_breakdown_parity(mode, sched, shadow, monkeypatch):
    bands, b, sh = ring_operator(), unit_rhs(), shadow()
    tol = TOL[mode]
    s = _solver(bands, mode, SCHEDULES[sched], monkeypatch)
    bt = torch.from_numpy(b).cuda()
    xp, ip, hp = s.solve(bt, tol=tol, maxit=100)
    x, info, h = s.solve(bt, tol=tol, maxit=100, rhat0=torch.from_numpy(sh).cuda())
    xo, ho, io = _oracle(bands, b, mode, tol=tol, maxit=100, rhat0=sh)
    _same_counts(info, io)
    xn = x.cpu().numpy()
    assert np.linalg.norm(xn - xo) <= 10 * tol * np.linalg.norm(xo)
    if io.breakdowns:        # the restart with rhat0 = r is the plain solve, bitwise
        assert info.breakdowns == 1 and info.restarts == ip.restarts + 1
        assert torch.equal(x, xp) and np.array_equal(h, hp)
    else:                    # FP64 with rho = 2^-30: the given rhat0 is used
        assert not np.array_equal(h, hp) and info.true_R < tol


def test_shadow_argument_validation(monkeypatch):
    bands, b = ring_operator(), unit_rhs()
    s = _solver(bands, "mixed", {}, monkeypatch)
    with pytest.raises(egs.EgError) as e:   # host memory is refused (device fp64 only)
        s.solve(torch.from_numpy(b).cuda(), tol=1e-6, rhat0=torch.from_numpy(shadow_rho_zero()))
    assert e.value.status == 1


@pytest.mark.parametrize("mode", ["mixed", "fp64"])
@pytest.mark.parametrize("P", [2, 4])
def test_shadow_breakdown_on_latitude_bands_bitwise(mode, P):
    """The same injected breakdowns on P latitude bands (in-process loopback transport): x, the
    history and every info field bitwise those of P = 1 (the W_SHADOW group sums and the restart
    bookkeeping go through the multi-rank finaliser path)."""
    bands, b, sh = ring_operator(), unit_rhs(), shadow_sigma_zero()
    ref_s = egs.Solver(G, torch.from_numpy(bands).cuda(), mode)
    xr, ir, hr = ref_s.solve(torch.from_numpy(b).cuda(), tol=TOL[mode], maxit=100, rhat0=torch.from_numpy(sh).cuda())
    assert ir.breakdowns == 1
    uid = egs.loopback_id(P)
    st = torch.cuda.Stream()
    row = NX
    res = [None] * P
    errs = []
    solvers = []
    with torch.cuda.stream(st):
        for r in range(P):
            j0, j1 = egs.band_rows(NY, r, P)
            solvers.append((egs.Solver(G, torch.from_numpy(np.ascontiguousarray(bands[:, j0 * row:j1 * row])).cuda(),
                                       mode, stream=st, dist=(r, P, uid)), j0, j1))

    def run(r):
        try:
            s, j0, j1 = solvers[r]
            with torch.cuda.stream(st):
                res[r] = s.solve(torch.from_numpy(b[j0 * row:j1 * row].copy()).cuda(), tol=TOL[mode], maxit=100,
                                 rhat0=torch.from_numpy(sh[j0 * row:j1 * row].copy()).cuda())
        except BaseException as e:  # noqa: BLE001
            errs.append(e)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(120)
    assert not errs
    torch.cuda.synchronize()
    x = torch.cat([res[r][0] for r in range(P)])
    for r in range(P):
        i = res[r][1]
        assert (i.iters, i.restarts, i.breakdowns, i.status) == (ir.iters, ir.restarts, ir.breakdowns, ir.status)
        assert np.array_equal(res[r][2], hr)
    assert torch.equal(x, xr)
