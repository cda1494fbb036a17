"""The P2P transport of the latitude-band decomposition (include/egsolve.h eg_solver_transport,
DESIGN.md §7): the kernels that produce the band-edge rows and the row-group sums store them into
the other ranks' workspaces and stamp epoch flags; the consumers wait on those flags.

On one GPU this runs through the loopback group (the ranks' workspaces are buffers of this
process; host barriers order every push ahead of its wait on the shared stream, so no kernel ever
spins on another rank's kernel) and the 1-rank NCCL path (pushes to its own buffers).  Checked:
bitwise equality with the copy / NCCL transports and the single-GPU path, the flag reset at an
epoch wrap-around, the timeout of a wait nobody satisfies, and the CUDA IPC step of the NCCL
setup across two processes on this GPU.
"""
import ctypes
import multiprocessing as mp
import os

import numpy as np
import pytest

import gen
from test_gpu_loopback import Bands, _same_info

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
egs = pytest.importorskip("paper_1811_03852_b200")

CASES = [gen.Problem(200, 37, 13, seed=8),     # uneven row-groups, 2 tiles (ragged last tile)
         gen.Problem(136, 16, 70, seed=16)]    # deep columns


def _bands(prob, mode, P, p2p, monkeypatch, **kw):
    if not p2p:
        monkeypatch.setenv("EG_P2P", "0")
    B = Bands(prob, mode, P, **kw)
    monkeypatch.delenv("EG_P2P", raising=False)
    want = "loopback-p2p" if p2p else "loopback"
    assert all(q.transport == want for q in B.s)
    return B


@pytest.mark.parametrize("prob", CASES, ids=lambda p: f"{p.nx}x{p.ny}x{p.nz}")
@pytest.mark.parametrize("mode", ["mixed", "fp64", "fp32"])
@pytest.mark.parametrize("fuse", [True, False], ids=["fused", "5kernel"])
def test_p2p_matches_copy_transport_bitwise(prob, mode, fuse, monkeypatch):
    """Same values land in the same ghost rows and gather slots: x, history and every control
    decision equal bitwise between the P2P pushes and the host-barrier copies, for P = 2, 4, 8."""
    monkeypatch.setenv("EG_FUSE" if fuse else "EG_NO_FUSE", "1")
    for P in (2, 4, 8):
        if min(8, prob.ny) % P:
            continue
        cp = _bands(prob, mode, P, False, monkeypatch)
        pp = _bands(prob, mode, P, True, monkeypatch)
        for kw in (dict(tol=1e-6, maxit=60, restart_every=3), dict(tol=0.0, maxit=7)):
            xc, ic, hc = cp.solve(**kw)
            xp, ip, hp = pp.solve(**kw)
            assert ic[0].iters > 0
            assert all(_same_info(a, b) for a, b in zip(ip, ic)), (P, ip[0], ic[0])
            assert all(np.array_equal(a, b) for a, b in zip(hp, hc)), P
            assert np.array_equal(xp, xc), P
        cp.close()
        pp.close()


@pytest.mark.parametrize("mode", ["mixed", "fp64"])
def test_p2p_epoch_wraparound(mode, monkeypatch):
    """The epoch wrap-around (flags cleared, epochs restart at 1) forced before every solve: the
    ranks clear their P2P flags between barriers and repeated solves stay bitwise equal to a
    single-GPU solve (a stale flag accepted would hand a rank old ghost rows or sums)."""
    prob = CASES[0]
    monkeypatch.setenv("EG_FUSE", "1")
    ref = Bands(prob, mode, 1)
    x1, i1, h1 = ref.solve(tol=1e-6, maxit=40)
    monkeypatch.setenv("EG_EPOCH_WRAP_TEST", "1")
    run = _bands(prob, mode, 4, True, monkeypatch)
    for _ in range(3):
        xP, iP, hP = run.solve(tol=1e-6, maxit=40)
        assert all(_same_info(i, i1[0]) for i in iP) and np.array_equal(xP, x1)
        assert all(np.array_equal(h, h1[0]) for h in hP)
    run.close()
    ref.close()


def test_p2p_wait_timeout_reports_error(monkeypatch):
    """A group-sum flag that is never stamped (EG_P2P_FAULT=1) ends the solve with EG_ERR_NCCL after
    EG_P2P_TIMEOUT_MS instead of hanging; a new handle then solves normally."""
    prob = CASES[0]
    bands, b = gen.host(prob)
    g = (prob.nx, prob.ny, prob.nz)
    bd = torch.from_numpy(bands).cuda()
    bt = torch.from_numpy(b).cuda()
    monkeypatch.setenv("EG_FORCE_NCCL", "1")
    monkeypatch.setenv("EG_P2P_FAULT", "1")
    monkeypatch.setenv("EG_P2P_TIMEOUT_MS", "50")
    s = egs.Solver(g, bd, "mixed")
    monkeypatch.delenv("EG_P2P_FAULT")
    monkeypatch.delenv("EG_P2P_TIMEOUT_MS")
    assert s.transport == "p2p"
    with pytest.raises(egs.EgError) as e:
        s.solve(bt, tol=1e-6, maxit=20)
    assert e.value.status == 7 and "did not arrive" in str(e.value)
    s.close()
    s2 = egs.Solver(g, bd, "mixed")
    monkeypatch.delenv("EG_FORCE_NCCL")
    ref = egs.Solver(g, bd, "mixed")
    x2, i2, h2 = s2.solve(bt, tol=1e-6, maxit=40)
    x1, i1, h1 = ref.solve(bt, tol=1e-6, maxit=40)
    assert i1.iters == i2.iters and torch.equal(x1, x2) and np.array_equal(h1, h2)


def _ipc_child(rec, conn):
    """Second process: open the exported workspace slice, check its bytes, write a reply pattern."""
    import torch as t
    import paper_1811_03852_b200 as e
    t.cuda.init()
    L = e.lib()
    ptr, opened = ctypes.c_void_p(), ctypes.c_void_p()
    rc = L.eg_debug_ipc_open(rec, ctypes.byref(ptr), ctypes.byref(opened))
    if rc != 0:
        conn.send(("open", rc))
        return
    n = 4096
    # view the peer memory as a tensor through __cuda_array_interface__
    class _Arr:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr.value, False), "version": 3}
    got = t.as_tensor(_Arr(), device="cuda")
    ok = bool(t.equal(got.cpu(), t.arange(n, dtype=t.float64) * 0.5 + 3.0))
    got.copy_(t.arange(n, dtype=t.float64, device="cuda") * -2.0)
    t.cuda.synchronize()
    L.eg_debug_ipc_close(opened)
    conn.send(("ok", ok))


def test_cuda_ipc_of_a_caching_allocator_slice():
    """The NCCL setup's IPC step on one GPU across two processes: a slice at a nonzero offset
    inside a PyTorch caching-allocator block is exported (allocation base + offset) and opened by
    another process, which sees the same bytes and whose writes land here."""
    n = 4096
    blk = torch.full((3 * n + 37,), 7.25, dtype=torch.float64, device="cuda")  # one allocator block
    view = blk[n + 37:2 * n + 37]                                      # nonzero offset inside it
    view.copy_(torch.arange(n, dtype=torch.float64, device="cuda") * 0.5 + 3.0)
    torch.cuda.synchronize()
    rec = ctypes.create_string_buffer(80)
    assert egs.lib().eg_debug_ipc_export(ctypes.c_void_p(view.data_ptr()), rec) == 0
    ctx = mp.get_context("spawn")
    a, b = ctx.Pipe()
    pr = ctx.Process(target=_ipc_child, args=(bytes(rec.raw), b))
    pr.start()
    assert a.poll(300), "IPC child did not answer"
    msg = a.recv()
    pr.join(60)
    assert msg == ("ok", True), msg
    torch.cuda.synchronize()
    assert torch.equal(view.cpu(), torch.arange(n, dtype=torch.float64) * -2.0)
    assert bool((blk[:n + 37] == 7.25).all()) and bool((blk[2 * n + 37:] == 7.25).all())  # only the slice


@pytest.mark.parametrize("split", ["0", "1"])
def test_p2p_split_update_knob_bitwise(split, monkeypatch):
    """EG_SPLIT_UPDATE forces the update's x half onto the side stream (default off with P2P, on
    with copies): either way the bands reproduce the single-GPU solve bitwise."""
    prob = CASES[1]
    monkeypatch.setenv("EG_FUSE", "1")
    ref = Bands(prob, "mixed", 1)
    x1, i1, h1 = ref.solve(tol=1e-6, maxit=30, restart_every=4)
    monkeypatch.setenv("EG_SPLIT_UPDATE", split)
    for p2p in (True, False):
        run = _bands(prob, "mixed", 4, p2p, monkeypatch)
        xP, iP, hP = run.solve(tol=1e-6, maxit=30, restart_every=4)
        assert all(_same_info(i, i1[0]) for i in iP) and np.array_equal(xP, x1), (split, p2p)
        run.close()
    ref.close()


def test_p2p_with_programmatic_dependent_launch_bitwise(monkeypatch):
    """EG_PDL=1 (phase kernels, update and one-kernel finalisers may launch before their predecessor
    finished and wait on it in-kernel) on 4 bands: bitwise the default."""
    prob = CASES[0]
    monkeypatch.setenv("EG_FUSE", "1")
    base = _bands(prob, "mixed", 4, True, monkeypatch)
    x0, i0, h0 = base.solve(tol=1e-6, maxit=40, restart_every=5)
    base.close()
    monkeypatch.setenv("EG_PDL", "1")
    run = _bands(prob, "mixed", 4, True, monkeypatch)
    x1, i1, h1 = run.solve(tol=1e-6, maxit=40, restart_every=5)
    run.close()
    assert all(_same_info(a, b) for a, b in zip(i1, i0)) and np.array_equal(x1, x0)
    assert all(np.array_equal(a, b) for a, b in zip(h1, h0))


def test_random_band_shapes_bitwise():
    """Seeded random grids (ragged tiles, odd nx, 1-row bands, nz from 1 to 80), random precision,
    schedule and P: the P2P bands reproduce the single-GPU solve bitwise (x, history, info)."""
    import os
    rng = np.random.default_rng(1811)
    for case in range(16):
        nx = int(rng.integers(3, 300))
        ny = int(rng.integers(8, 41))
        nz = int(rng.integers(1, 73))
        mode = ["mixed", "fp64", "fp32"][case % 3]
        fuse = case % 2 == 0
        if fuse:  # the fused phase kernels need nx % 4 == 0 (16-byte TMA strides)
            nx = max(4, nx - nx % 4)
        P = int(rng.choice([2, 4, 8]))
        prob = gen.Problem(nx, ny, nz, seed=100 + case)
        os.environ["EG_FUSE" if fuse else "EG_NO_FUSE"] = "1"
        try:
            ref = Bands(prob, mode, 1)
            run = Bands(prob, mode, P)
        finally:
            os.environ.pop("EG_FUSE", None)
            os.environ.pop("EG_NO_FUSE", None)
        assert all(q.transport == "loopback-p2p" for q in run.s)
        kw = dict(tol=1e-6, maxit=25, restart_every=4)
        x1, i1, h1 = ref.solve(**kw)
        xP, iP, hP = run.solve(**kw)
        tag = (nx, ny, nz, mode, fuse, P)
        assert all(_same_info(i, i1[0]) for i in iP), tag
        assert np.array_equal(xP, x1), tag
        assert all(np.array_equal(h, h1[0]) for h in hP), tag
        ref.close()
        run.close()


@pytest.mark.parametrize("mode", ["mixed", "fp64", "fp32"])
def test_p2p_trisor_halos_bitwise(mode, monkeypatch):
    """The tri-SOR preconditioner (NEXT-1) on bands: the halo after every red-black half-sweep by
    P2P pushes + waits (k_push_sweep / k_wait_sweep) equals the copy transport and the single-GPU
    solve bitwise, for solves (with restarts: the x ghost rows go the same way) and for
    eg_precondition after a solve (the counter persists), with eg_apply_operator in between."""
    prob = gen.Problem(96, 24, 13, seed=17)  # nx even: red-black tri-SOR
    ref = Bands(prob, mode, 1, trisor=True)
    for q in ref.s:
        q.set_preconditioner("trisor", sweeps=3, omega=1.5)
    x1, i1, h1 = ref.solve(tol=1e-8, maxit=40, restart_every=9)
    dt = torch.float64 if mode == "fp64" else torch.float32
    xin = torch.from_numpy(np.random.default_rng(5).standard_normal(prob.n)).to(dt).cuda()
    z1 = ref.call("precondition", xin)
    y1 = ref.call("apply", xin)
    for P in (2, 4, 8):
        for p2p in (True, False):
            run = _bands(prob, mode, P, p2p, monkeypatch, trisor=True)
            for q in run.s:
                q.set_preconditioner("trisor", sweeps=3, omega=1.5)
            for _ in range(2):  # the second solve reuses the half-sweep counter
                xP, iP, hP = run.solve(tol=1e-8, maxit=40, restart_every=9)
                assert all(_same_info(i, i1[0]) for i in iP) and np.array_equal(xP, x1), (P, p2p)
                assert all(np.array_equal(h, h1[0]) for h in hP), (P, p2p)
            assert torch.equal(run.call("precondition", xin), z1), (P, p2p)
            assert torch.equal(run.call("apply", xin), y1), (P, p2p)  # (its halo: NCCL / copies, on z_s)
            run.close()
    ref.close()
