"""GPU checks of the C-ABI contract that need a device: features are explicit (eg_solver_create_ex;
a larger workspace never turns one on), and the fused phase kernels, whose CTAs wait on each other's
ready flags, are launched cooperatively: a grid that cannot be co-resident fails with EG_ERR_CUDA
instead of hanging, and the process keeps working afterwards."""
import ctypes

import numpy as np
import pytest

import gen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
egs = pytest.importorskip("paper_1811_03852_b200")


def _raw_create(prob, mode, features, extra_bytes=0, nbytes=None):
    L = egs.lib()
    bands, b = gen.host(prob)
    bd = torch.from_numpy(bands).cuda()
    g = egs._Grid(prob.nx, prob.ny, prob.nz)
    nb = ctypes.c_size_t()
    assert L.eg_workspace_bytes_ex(ctypes.byref(g), None, egs.PRECISIONS[mode], features, ctypes.byref(nb)) == 0
    size = (nb.value + extra_bytes) if nbytes is None else nbytes
    ws = torch.empty(size, dtype=torch.uint8, device="cuda")
    ptrs = (ctypes.c_void_p * 7)(*[bd[d].data_ptr() for d in range(7)])
    h = ctypes.c_void_p()
    rc = L.eg_solver_create_ex(ctypes.byref(g), None, ptrs, egs.PRECISIONS[mode], features,
                               ctypes.c_void_p(ws.data_ptr()), size,
                               ctypes.c_void_p(torch.cuda.current_stream().cuda_stream), ctypes.byref(h))
    return rc, h, (ws, bd, b)


def test_features_are_explicit():
    prob = gen.Problem(64, 16, 10, seed=3)
    L = egs.lib()
    g = egs._Grid(prob.nx, prob.ny, prob.nz)
    nbb = ctypes.c_size_t()
    L.eg_workspace_bytes_ex(ctypes.byref(g), None, egs.EG_MIXED, egs.EG_FEATURE_BATCH, ctypes.byref(nbb))
    # a workspace big enough for the batch staging, created without the feature: no batch support
    rc, h, keep = _raw_create(prob, "mixed", 0, nbytes=nbb.value)
    assert rc == 0
    b = keep[2]
    prm = egs._Params(1e-6, 50, 150, 0, 0, None)
    xs = (ctypes.c_void_p * 1)(np.empty(prob.n).ctypes.data)
    bs = (ctypes.c_void_p * 1)(b.ctypes.data)
    done = ctypes.c_int()
    assert L.eg_solve_batch(h, 1, bs, xs, None, ctypes.byref(prm), None, None, ctypes.byref(done)) == 8
    L.eg_solver_destroy(h)
    # asked for, but the workspace is too small for it
    rc, h, _ = _raw_create(prob, "mixed", egs.EG_FEATURE_BATCH, nbytes=nbb.value - 256)
    assert rc == 8 and not h.value
    # asked for with room: works, and bitwise equal to a plain solve
    rc, h, keep = _raw_create(prob, "mixed", egs.EG_FEATURE_BATCH | egs.EG_FEATURE_TRISOR)
    assert rc == 0
    xb = np.empty(prob.n)
    xs = (ctypes.c_void_p * 1)(xb.ctypes.data)
    assert L.eg_solve_batch(h, 1, bs, xs, None, ctypes.byref(prm), None, None, ctypes.byref(done)) == 0
    L.eg_solver_destroy(h)
    s = egs.Solver((prob.nx, prob.ny, prob.nz), keep[1], "mixed")
    x, _, _ = s.solve(torch.from_numpy(b).cuda(), tol=1e-6, maxit=50)
    assert np.array_equal(x.cpu().numpy(), xb)


def test_non_coresident_fused_grid_fails_cleanly(monkeypatch):
    """More latitude strips than SMs (a test-only knob): the cooperative launch of the fused phase
    kernel is refused -> EG_ERR_CUDA; the same handle type then still solves normally."""
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    prob = gen.Problem(128, 2 * nsm + 10, 10, seed=5)
    bands, b = gen.host(prob)
    bd, bt = torch.from_numpy(bands).cuda(), torch.from_numpy(b).cuda()
    g = (prob.nx, prob.ny, prob.nz)
    monkeypatch.setenv("EG_FUSE", "1")
    monkeypatch.setenv("EG_MARCH_STRIPS_UNSAFE", str(nsm + 20))     # one 128-column tile x (nsm + 20) strips
    s_bad = egs.Solver(g, bd, "mixed")
    monkeypatch.delenv("EG_MARCH_STRIPS_UNSAFE")
    s_ok = egs.Solver(g, bd, "mixed")
    monkeypatch.delenv("EG_FUSE")
    for flags in (0, egs.EG_SOLVE_NO_GRAPH):
        _, info, _ = s_bad.solve(bt, tol=1e-6, maxit=20, flags=flags, raise_on_error=False)
        assert info.status == 6, flags                                   # EG_ERR_CUDA, no hang
    x, info, _ = s_ok.solve(bt, tol=1e-6, maxit=20)
    assert info.status == 0 and info.converged
    monkeypatch.setenv("EG_NO_FUSE", "1")
    s_ref = egs.Solver(g, bd, "mixed")
    xr, ir, _ = s_ref.solve(bt, tol=1e-6, maxit=20)
    assert torch.equal(x, xr)


def test_aliasing_and_in_place_warm_start():
    """apply / precondition refuse overlapping input and output (EG_ERR_ARG); a warm start whose x0
    is the output buffer (in place) gives the same result as a separate x0."""
    prob = gen.Problem(64, 16, 10, seed=9)
    bands, b = gen.host(prob)
    s = egs.Solver((prob.nx, prob.ny, prob.nz), torch.from_numpy(bands).cuda(), "mixed")
    v = torch.randn(prob.n, device="cuda", dtype=torch.float32)
    for fn in (s.apply, s.precondition):
        with pytest.raises(egs.EgError) as e:
            fn(v, out=v)
        assert e.value.status == 1
    y = s.apply(v)                      # the handle keeps working
    assert torch.isfinite(y).all()
    bt = torch.from_numpy(b).cuda()
    x1, _, _ = s.solve(bt, tol=0.0, maxit=3)
    x0 = x1.clone()
    xa, ia, ha = s.solve(bt, x0=x0, tol=1e-7, maxit=50)
    xin = x1.clone()
    xb, ib, hb = s.solve(bt, x0=xin, tol=1e-7, maxit=50, out=xin)   # x0 is the output
    assert ia.iters == ib.iters and np.array_equal(ha, hb) and torch.equal(xa, xb) and xb.data_ptr() == xin.data_ptr()
