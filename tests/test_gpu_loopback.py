"""The latitude-band decomposition on ONE GPU through the
in-process loopback transport (eg_loopback_id): P solver handles, one per band, each driven by its
own host thread, exchanging ghost rows and group sums by device copies on one shared stream.

This runs every multi-rank kernel the NCCL path runs (k_edge_rows before the fused phase kernels,
ghost-row stencils, the fp64 x ghost rows at restart / verification, the row-group finaliser with
an all-gather, the tri-SOR colour halos) and checks the claim of A-23: x, the history and the
control decisions are bitwise identical for P = 1, 2, 4, 8.  No kernel of one rank ever waits for
another rank's kernel (B200_PROFILING.md), so this is safe on one GPU.
"""
import threading

import numpy as np
import pytest

import gen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
egs = pytest.importorskip("paper_1811_03852_b200")

RAGGED = gen.Problem(200, 37, 13, seed=8)    # uneven row-groups (37 rows in 8 groups), 2 tiles
CASES = [gen.CONFIGS["C1"], RAGGED, gen.Problem(136, 16, 70, seed=16)]


def _run_ranks(fns, timeout=600):
    out, errs = [None] * len(fns), [None] * len(fns)

    def work(i):
        try:
            out[i] = fns[i]()
        except BaseException as e:  # noqa: BLE001 - re-raised below
            errs[i] = e

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(fns))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
    assert not any(t.is_alive() for t in ts), "a loopback rank did not finish"
    for e in errs:
        if e is not None:
            raise e
    return out


class Bands:
    """P loopback solvers over the latitude bands of one problem (all on the default stream)."""

    def __init__(self, prob, mode, P, **kw):
        self.prob, self.P = prob, P
        self.bands, self.b = gen.host(prob)
        g = (prob.nx, prob.ny, prob.nz)
        row = prob.nx * prob.nz
        uid = egs.loopback_id(P)
        self.rows = [egs.band_rows(prob.ny, r, P) for r in range(P)]
        self.sl = [slice(j0 * row, j1 * row) for j0, j1 in self.rows]
        self.s = [egs.Solver(g, torch.from_numpy(np.ascontiguousarray(self.bands[:, sl])).cuda(), mode,
                             dist=(r, P, uid), **kw) for r, sl in enumerate(self.sl)]

    def close(self):
        for s in self.s:
            s.close()

    def solve(self, b=None, **kw):
        b = self.b if b is None else b
        bs = [torch.from_numpy(np.ascontiguousarray(b[sl])).cuda() for sl in self.sl]
        outs = [torch.full((s.n_local,), float("nan"), dtype=torch.float64, device="cuda") for s in self.s]
        torch.cuda.synchronize()
        res = _run_ranks([lambda r=r: self.s[r].solve(bs[r], out=outs[r], **kw) for r in range(self.P)])
        x = torch.cat([o for o, _, _ in res]).cpu().numpy()
        return x, [i for _, i, _ in res], [h for _, _, h in res]

    def call(self, name, v):
        parts = [v[sl].contiguous() for sl in self.sl]
        outs = [torch.empty_like(p) for p in parts]
        torch.cuda.synchronize()
        _run_ranks([lambda r=r: getattr(self.s[r], name)(parts[r], out=outs[r]) for r in range(self.P)])
        return torch.cat(outs)


def _same_info(a, b):
    return (a.iters, a.converged, a.restarts, a.breakdowns, a.status) == \
        (b.iters, b.converged, b.restarts, b.breakdowns, b.status) and \
        np.float64(a.final_R).tobytes() == np.float64(b.final_R).tobytes() and \
        np.float64(a.true_R).tobytes() == np.float64(b.true_R).tobytes()


@pytest.mark.parametrize("prob", CASES, ids=lambda p: f"{p.nx}x{p.ny}x{p.nz}")
@pytest.mark.parametrize("mode", ["mixed", "fp64", "fp32"])
@pytest.mark.parametrize("fuse", [True, False], ids=["fused", "5kernel"])
def test_loopback_solve_bitwise_equal_any_P(prob, mode, fuse, monkeypatch):
    # (FP64: P = 1 runs the fused FP64 phase kernels, P > 1 the 5-kernel schedule: bitwise equal too)
    monkeypatch.setenv("EG_FUSE" if fuse else "EG_NO_FUSE", "1")
    ref = Bands(prob, mode, 1)
    P_list = [p for p in (2, 4, 8) if min(8, prob.ny) % p == 0]
    runs = [Bands(prob, mode, P) for P in P_list]
    for kw in (dict(tol=1e-6, maxit=60, restart_every=3),   # restarts: fp64 x ghost rows
               dict(tol=0.0, maxit=8)):                     # fixed iterations (the bench's run)
        x1, i1, h1 = ref.solve(**kw)
        assert i1[0].status == 0 and i1[0].iters > 0
        for run in runs:
            xP, iP, hP = run.solve(**kw)
            for r in range(run.P):
                assert _same_info(iP[r], i1[0]), (run.P, r, iP[r], i1[0])
                assert np.array_equal(hP[r], h1[0]), (run.P, r)
            assert np.array_equal(xP, x1), run.P
    if fuse and mode != "fp64":  # the fused phase kernels did run on the multi-rank path
        s = runs[0].s
        for q in s:
            q.profile_reset()
        runs[0].solve(tol=0.0, maxit=2, flags=egs.EG_SOLVE_PROFILE)
        assert all(q.profile()["phase_A"][1] == 2 for q in s)
    for run in runs + [ref]:
        run.close()


@pytest.mark.parametrize("mode", ["mixed", "fp64"])
def test_loopback_apply_and_trisor_bitwise_equal(mode):
    """eg_apply_operator (ghost rows of the input) and the red-black tri-SOR preconditioner
    (one halo per colour per sweep) on bands equal the single-GPU results bitwise."""
    prob = gen.Problem(96, 24, 13, seed=17)  # nx even: red-black tri-SOR
    ref = Bands(prob, mode, 1, trisor=True)
    dt = torch.float64 if mode == "fp64" else torch.float32
    x = torch.from_numpy(np.random.default_rng(3).standard_normal(prob.n)).to(dt).cuda()
    y1 = ref.call("apply", x)
    for q in ref.s:
        q.set_preconditioner("trisor", sweeps=3, omega=1.5)
    z1 = ref.call("precondition", x)
    x1, i1, h1 = ref.solve(tol=1e-8, maxit=40)
    for P in (2, 4, 8):
        run = Bands(prob, mode, P, trisor=True)
        assert torch.equal(run.call("apply", x), y1), P
        for q in run.s:
            q.set_preconditioner("trisor", sweeps=3, omega=1.5)
        assert torch.equal(run.call("precondition", x), z1), P
        xP, iP, hP = run.solve(tol=1e-8, maxit=40)
        assert all(_same_info(i, i1[0]) for i in iP) and np.array_equal(xP, x1), P
        assert all(np.array_equal(h, h1[0]) for h in hP)
        run.close()
    ref.close()


def test_loopback_id_checks():
    prob = gen.CONFIGS["C1"]
    bands, _ = gen.host(prob)
    g = (prob.nx, prob.ny, prob.nz)
    row = prob.nx * prob.nz
    uid = egs.loopback_id(2)
    j0, j1 = egs.band_rows(prob.ny, 0, 4)
    bd = torch.from_numpy(np.ascontiguousarray(bands[:, j0 * row:j1 * row])).cuda()
    with pytest.raises(egs.EgError) as e:  # the id names 2 ranks, the decomposition 4
        egs.Solver(g, bd, "mixed", dist=(0, 4, uid))
    assert e.value.status == 1
    j0, j1 = egs.band_rows(prob.ny, 0, 2)
    bd0 = torch.from_numpy(np.ascontiguousarray(bands[:, j0 * row:j1 * row])).cuda()
    j0, j1 = egs.band_rows(prob.ny, 1, 2)
    bd1 = torch.from_numpy(np.ascontiguousarray(bands[:, j0 * row:j1 * row])).cuda()
    uid = egs.loopback_id(2)
    s0 = egs.Solver(g, bd0, "mixed", dist=(0, 2, uid))
    other = torch.cuda.Stream()
    with pytest.raises(egs.EgError) as e:  # ranks of one group must share the stream
        egs.Solver(g, bd1, "mixed", dist=(1, 2, uid), stream=other)
    assert e.value.status == 1
    s0.close()


def test_loopback_solve_batch_bitwise_equal():
    """eg_solve_batch on latitude bands (host buffers, operator re-scaled before each solve, copy
    streams per rank) gives each rank's rows of the single-GPU batch, bitwise."""
    prob = gen.CONFIGS["C1"]
    ref = Bands(prob, "mixed", 1, batch=True)
    run = Bands(prob, "mixed", 4, batch=True)
    rng = np.random.default_rng(9)
    bs = [ref.b * (1.0 + 0.25 * k) + 0.01 * rng.standard_normal(prob.n) for k in range(3)]

    def batch(B):
        xs = [[np.empty(sl.stop - sl.start) for _ in bs] for sl in B.sl]
        bds = [torch.from_numpy(np.ascontiguousarray(B.bands[:, sl])).cuda() for sl in B.sl]
        torch.cuda.synchronize()
        infos = _run_ranks([lambda r=r: B.s[r].solve_batch([np.ascontiguousarray(v[B.sl[r]]) for v in bs], xs[r],
                                                            bands=bds[r], tol=1e-6, maxit=60)
                            for r in range(B.P)])
        return [np.concatenate([xs[r][k] for r in range(B.P)]) for k in range(len(bs))], infos

    x1, i1 = batch(ref)
    x4, i4 = batch(run)
    for k in range(len(bs)):
        assert np.array_equal(x1[k], x4[k]), k
        assert all(_same_info(i4[r][k], i1[0][k]) for r in range(4))
    ref.close()
    run.close()
