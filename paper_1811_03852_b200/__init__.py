"""B200-native mixed-precision BiCGStab for the ENDGame Helmholtz system (arXiv 1811.03852).

Thin ctypes binding over ``libegsolve.so`` (the C ABI in ``include/egsolve.h``): argument
marshalling only — every step of the solve runs in the library's sm_100a kernels.  PyTorch supplies
device memory (the workspace and all vectors are torch tensors), the CUDA stream, and
``torch.distributed`` for broadcasting the NCCL unique id of a latitude-band decomposition.
There is no CPU fallback: importing this package without the built extension raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.environ.get("EGSOLVE_LIB") or os.path.join(_HERE, "libegsolve.so")  # override: A/B builds

EG_FP64, EG_MIXED, EG_FP32 = 0, 1, 2
PRECISIONS = {"fp64": EG_FP64, "mixed": EG_MIXED, "fp32": EG_FP32}
EG_SOLVE_NO_GRAPH, EG_SOLVE_PROFILE = 1, 2
EG_FEATURE_TRISOR, EG_FEATURE_BATCH = 1, 2
STATUS = {0: "EG_OK", 1: "EG_ERR_ARG", 2: "EG_ERR_SINGULAR_DIAG", 3: "EG_ERR_DEGENERATE_RHS",
          4: "EG_ERR_BREAKDOWN", 5: "EG_ERR_NONFINITE", 6: "EG_ERR_CUDA", 7: "EG_ERR_NCCL",
          8: "EG_ERR_WORKSPACE"}
# symbols declared in include/egsolve.h (tests check the library exports all of them)
ABI_SYMBOLS = ("eg_workspace_bytes", "eg_workspace_bytes_ex", "eg_solver_create", "eg_solver_create_ex",
               "eg_solver_set_operator",
               "eg_solver_set_preconditioner", "eg_apply_operator", "eg_precondition",
               "eg_solve", "eg_solve_batch", "eg_solver_destroy", "eg_last_error", "eg_status_str",
               "eg_nccl_unique_id", "eg_loopback_id", "eg_num_kernels", "eg_kernel_name", "eg_profile_get",
               "eg_profile_reset", "eg_solver_transport", "eg_debug_ipc_export", "eg_debug_ipc_open",
               "eg_debug_ipc_close")


class EgError(RuntimeError):
    def __init__(self, status: int, detail: str = ""):
        super().__init__(f"{STATUS.get(status, status)}{': ' + detail if detail else ''}")
        self.status = status


class _Grid(ctypes.Structure):
    _fields_ = [("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64)]


class _Dist(ctypes.Structure):
    _fields_ = [("j_begin", ctypes.c_int64), ("j_end", ctypes.c_int64), ("rank", ctypes.c_int32),
                ("nranks", ctypes.c_int32), ("nccl_unique_id", ctypes.c_void_p)]


class _Params(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("maxit", ctypes.c_int32),
                ("restart_every", ctypes.c_int32), ("flags", ctypes.c_uint32),
                ("check_every", ctypes.c_int32), ("rhat0", ctypes.c_void_p)]


class _Info(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("restarts", ctypes.c_int32), ("breakdowns", ctypes.c_int32),
                ("status", ctypes.c_int32), ("final_R", ctypes.c_double),
                ("true_R", ctypes.c_double)]


@dataclass
class SolveInfo:
    iters: int
    converged: bool
    restarts: int
    breakdowns: int
    status: int
    final_R: float
    true_R: float


_lib = None


def lib():
    """Load libegsolve.so (raises if it is not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise ImportError(f"{_SO} is not built; run `make` (or __graft_entry__.build())")
        L = ctypes.CDLL(_SO)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.eg_workspace_bytes.argtypes = [ctypes.POINTER(_Grid), ctypes.POINTER(_Dist), i32,
                                         ctypes.POINTER(ctypes.c_size_t)]
        L.eg_workspace_bytes_ex.argtypes = [ctypes.POINTER(_Grid), ctypes.POINTER(_Dist), i32,
                                            ctypes.c_uint32, ctypes.POINTER(ctypes.c_size_t)]
        L.eg_solver_create.argtypes = [ctypes.POINTER(_Grid), ctypes.POINTER(_Dist),
                                       ctypes.POINTER(vp), i32, vp, ctypes.c_size_t, vp,
                                       ctypes.POINTER(vp)]
        L.eg_solver_create_ex.argtypes = [ctypes.POINTER(_Grid), ctypes.POINTER(_Dist),
                                          ctypes.POINTER(vp), i32, ctypes.c_uint32, vp, ctypes.c_size_t, vp,
                                          ctypes.POINTER(vp)]
        L.eg_solver_set_operator.argtypes = [vp, ctypes.POINTER(vp)]
        L.eg_solver_set_preconditioner.argtypes = [vp, i32, i32, ctypes.c_double]
        L.eg_apply_operator.argtypes = [vp, vp, vp]
        L.eg_precondition.argtypes = [vp, vp, vp]
        L.eg_solve.argtypes = [vp, vp, vp, ctypes.POINTER(_Params), vp, vp, ctypes.POINTER(_Info)]
        L.eg_solve_batch.argtypes = [vp, i32, ctypes.POINTER(vp), ctypes.POINTER(vp), ctypes.POINTER(vp),
                                     ctypes.POINTER(_Params), vp, ctypes.POINTER(_Info), ctypes.POINTER(i32)]
        L.eg_solver_destroy.argtypes = [vp]
        L.eg_solver_destroy.restype = None
        L.eg_last_error.argtypes = [vp]
        L.eg_last_error.restype = ctypes.c_char_p
        L.eg_status_str.argtypes = [i32]
        L.eg_status_str.restype = ctypes.c_char_p
        L.eg_nccl_unique_id.argtypes = [ctypes.c_char_p]
        L.eg_loopback_id.argtypes = [i32, ctypes.c_char_p]
        L.eg_num_kernels.restype = i32
        L.eg_kernel_name.argtypes = [i32]
        L.eg_kernel_name.restype = ctypes.c_char_p
        L.eg_profile_get.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_double),
                                     ctypes.POINTER(i64), ctypes.POINTER(ctypes.c_double)]
        L.eg_profile_reset.argtypes = [vp]
        L.eg_solver_transport.argtypes = [vp]
        L.eg_solver_transport.restype = i32
        L.eg_debug_ipc_export.argtypes = [vp, ctypes.c_char_p]
        L.eg_debug_ipc_open.argtypes = [ctypes.c_char_p, ctypes.POINTER(vp), ctypes.POINTER(vp)]
        L.eg_debug_ipc_close.argtypes = [vp]
        _lib = L
    return _lib


def band_rows(ny: int, rank: int, nranks: int):
    """Rows [j_begin, j_end) of rank's latitude band: whole reduction row-groups
    (G = min(8, ny) groups, group g = rows [g*ny//G, (g+1)*ny//G)); nranks must divide G."""
    G = min(8, ny)
    if nranks < 1 or G % nranks:
        raise ValueError(f"nranks={nranks} must divide the {G} reduction row-groups")
    per = G // nranks
    return (rank * per) * ny // G, ((rank + 1) * per) * ny // G


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    rc = lib().eg_nccl_unique_id(buf)
    if rc:
        raise EgError(rc, "ncclGetUniqueId")
    return buf.raw


def loopback_id(nranks: int) -> bytes:
    """Id of a new in-process loopback group (eg_loopback_id): pass it as
    Solver(..., dist=(rank, nranks, id)) for each rank, all on one stream, one thread per rank."""
    buf = ctypes.create_string_buffer(128)
    rc = lib().eg_loopback_id(nranks, buf)
    if rc:
        raise EgError(rc, "eg_loopback_id")
    return buf.raw


def _ptr(t) -> ctypes.c_void_p:
    if t is None:
        return ctypes.c_void_p(0)
    if isinstance(t, np.ndarray):
        assert t.flags.c_contiguous
        return ctypes.c_void_p(t.ctypes.data)
    assert t.is_contiguous()
    return ctypes.c_void_p(t.data_ptr())


class Solver:
    """One (local band of a) Helmholtz operator on the current CUDA device.

    grid: (nx, ny, nz) global.  bands: float64 CUDA tensor [7, n_local] (C,E,W,N,S,U,D; layout
    q = i + nx*(k + nz*j_local)).  precision: "fp64" | "mixed" | "fp32".  group: optional
    torch.distributed process group for a latitude-band decomposition (one rank per GPU).
    """

    def __init__(self, grid, bands, precision="mixed", group=None, stream=None, trisor=False, batch=False,
                 dist=None):
        """trisor=True sizes the workspace for the colour-split tri-SOR copies (EG_FEATURE_TRISOR);
        set_preconditioner("trisor") works either way, faster with them.  batch=True adds the
        staging buffers solve_batch needs (EG_FEATURE_BATCH).  dist=(rank, nranks, id) gives the
        decomposition explicitly instead of a process group (id: 128 bytes from nccl_unique_id()
        or loopback_id())."""
        import torch
        self.grid = tuple(int(v) for v in grid)
        nx, ny, nz = self.grid
        self.precision = precision
        self.mode = PRECISIONS[precision]
        self.vdtype = torch.float64 if self.mode == EG_FP64 else torch.float32
        self.device = bands.device
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self._uid = None
        uid = None
        if dist is not None:
            rank, nranks, uid = int(dist[0]), int(dist[1]), dist[2]
        elif group is not None:
            import torch.distributed as tdist
            rank, nranks = tdist.get_rank(group), tdist.get_world_size(group)
        else:
            rank, nranks = 0, 1
        self.rank, self.nranks = rank, nranks
        self.j_begin, self.j_end = band_rows(ny, rank, nranks) if nranks > 1 else (0, ny)
        self.n_local = (self.j_end - self.j_begin) * nx * nz
        if nranks > 1:
            if uid is None:
                import torch.distributed as tdist
                obj = [nccl_unique_id() if rank == 0 else None]
                tdist.broadcast_object_list(obj, src=tdist.get_global_rank(group, 0), group=group)
                uid = obj[0]
            self._uid = ctypes.create_string_buffer(uid, 128)
            self._dist = _Dist(self.j_begin, self.j_end, rank, nranks,
                               ctypes.cast(self._uid, ctypes.c_void_p))
            dptr = ctypes.byref(self._dist)
        else:
            self._dist = None
            dptr = None
        assert bands.dtype == torch.float64 and bands.is_cuda and bands.is_contiguous()
        assert tuple(bands.shape) == (7, self.n_local), (tuple(bands.shape), self.n_local)
        self._grid = _Grid(nx, ny, nz)
        nbytes = ctypes.c_size_t()
        self.features = (EG_FEATURE_TRISOR if trisor else 0) | (EG_FEATURE_BATCH if batch else 0)
        rc = lib().eg_workspace_bytes_ex(ctypes.byref(self._grid), dptr, self.mode, self.features,
                                         ctypes.byref(nbytes))
        if rc:
            raise EgError(rc, "eg_workspace_bytes_ex")
        self.workspace = torch.empty(nbytes.value, dtype=torch.uint8, device=self.device)
        ptrs = (ctypes.c_void_p * 7)(*[bands[d].data_ptr() for d in range(7)])
        h = ctypes.c_void_p()
        rc = lib().eg_solver_create_ex(ctypes.byref(self._grid), dptr, ptrs, self.mode, self.features,
                                       _ptr(self.workspace), nbytes.value,
                                       ctypes.c_void_p(self.stream.cuda_stream), ctypes.byref(h))
        if rc:
            raise EgError(rc, "eg_solver_create_ex")
        self._h = h

    # ---- lifetime ----
    def close(self):
        if getattr(self, "_h", None):
            lib().eg_solver_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc, what):
        if rc:
            raise EgError(rc, f"{what}: {lib().eg_last_error(self._h).decode()}")

    # ---- the C ABI calls ----
    def set_operator(self, bands):
        """a1 on a new operator of the same grid (eg_solver_set_operator)."""
        import torch
        assert bands.dtype == torch.float64 and bands.is_cuda and bands.is_contiguous()
        assert tuple(bands.shape) == (7, self.n_local)
        ptrs = (ctypes.c_void_p * 7)(*[bands[d].data_ptr() for d in range(7)])
        self._check(lib().eg_solver_set_operator(self._h, ptrs), "eg_solver_set_operator")

    def set_preconditioner(self, kind="tridiag", sweeps=3, omega=1.5):
        """NEXT-1: "tridiag" (C^-1 = T^-1, default) or "trisor" (red-black tri-SOR, Eq. 7)."""
        k = {"tridiag": 0, "trisor": 1}[kind]
        self._check(lib().eg_solver_set_preconditioner(self._h, k, int(sweeps), float(omega)),
                    "eg_solver_set_preconditioner")

    def apply(self, x, out=None):
        """y = Ahat x (working precision tensors, local rows)."""
        import torch
        assert x.dtype == self.vdtype and x.is_cuda and x.numel() == self.n_local
        y = out if out is not None else torch.empty_like(x)
        self._check(lib().eg_apply_operator(self._h, _ptr(x), _ptr(y)), "eg_apply_operator")
        return y

    def precondition(self, r, out=None):
        """z = T^-1 r per column (working precision tensors)."""
        import torch
        assert r.dtype == self.vdtype and r.is_cuda and r.numel() == self.n_local
        z = out if out is not None else torch.empty_like(r)
        self._check(lib().eg_precondition(self._h, _ptr(r), _ptr(z)), "eg_precondition")
        return z

    def solve(self, b, x0=None, tol=1e-4, maxit=200, restart_every=150, flags=0, check_every=0,
              out=None, raise_on_error=True, history=True, rhat0=None):
        """Solve; b / x0 / out may be CUDA tensors or (pinned) host tensors / numpy arrays (fp64).
        history=False skips the residual history (no host array of maxit + 1 doubles; returned as
        None).  rhat0: optional fp64 CUDA tensor, the shadow residual of the first start
        (eg_solve_params.rhat0; default r0).  Returns (x, SolveInfo, history[: iters+1] numpy)."""
        import torch
        if out is None:
            if isinstance(b, np.ndarray):
                out = np.empty(self.n_local, np.float64)
            else:
                out = torch.empty(self.n_local, dtype=torch.float64, device=b.device)
        if rhat0 is not None:
            assert rhat0.dtype == torch.float64 and rhat0.numel() == self.n_local  # device memory: checked by eg_solve
        hist = np.full(int(maxit) + 1, np.nan) if history else None
        prm = _Params(float(tol), int(maxit), int(restart_every), int(flags), int(check_every), _ptr(rhat0))
        info = _Info()
        rc = lib().eg_solve(self._h, _ptr(b), _ptr(x0), ctypes.byref(prm), _ptr(out),
                            _ptr(hist), ctypes.byref(info))
        inf = SolveInfo(info.iters, bool(info.converged), info.restarts, info.breakdowns,
                        info.status, info.final_R, info.true_R)
        if rc and raise_on_error:
            self._check(rc, "eg_solve")
        return out, inf, (hist[: inf.iters + 1] if history else None)

    def solve_batch(self, bs, xs, bands=None, tol=1e-4, maxit=200, restart_every=150, flags=0,
                    check_every=0, raise_on_error=True):
        """eg_solve_batch: solve for every b in `bs` into the matching `xs` (fp64; pinned host tensors
        or numpy arrays, or CUDA tensors), re-scaling `bands` (CUDA, as for set_operator) before each
        solve if given, with the transfers of neighbouring solves overlapped.  Needs batch=True at
        construction.  Returns the list of SolveInfo."""
        n = len(bs)
        assert len(xs) == n
        pb = (ctypes.c_void_p * max(n, 1))(*[_ptr(v).value for v in bs])
        px = (ctypes.c_void_p * max(n, 1))(*[_ptr(v).value for v in xs])
        pbands = None
        if bands is not None:
            pbands = (ctypes.c_void_p * 7)(*[bands[d].data_ptr() for d in range(7)])
        prm = _Params(float(tol), int(maxit), int(restart_every), int(flags), int(check_every), None)
        infos = (_Info * max(n, 1))()
        done = ctypes.c_int()
        rc = lib().eg_solve_batch(self._h, n, pb, px, pbands, ctypes.byref(prm), None, infos, ctypes.byref(done))
        out = [SolveInfo(i.iters, bool(i.converged), i.restarts, i.breakdowns, i.status, i.final_R, i.true_R)
               for i in list(infos)[: done.value]]
        if rc and raise_on_error:
            self._check(rc, "eg_solve_batch")
        return out

    # ---- profiling ----
    def profile(self):
        """{kernel: (total_ms, launches, algorithmic_bytes_per_launch)}"""
        out = {}
        for k in range(lib().eg_num_kernels()):
            ms, n, by = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double()
            lib().eg_profile_get(self._h, k, ctypes.byref(ms), ctypes.byref(n), ctypes.byref(by))
            out[lib().eg_kernel_name(k).decode()] = (ms.value, n.value, by.value)
        return out

    def profile_reset(self):
        lib().eg_profile_reset(self._h)

    TRANSPORTS = {0: "none", 1: "nccl", 2: "p2p", 3: "loopback", 4: "loopback-p2p"}

    @property
    def transport(self) -> str:
        """How the latitude bands exchange ghost rows and group sums (include/egsolve.h
        eg_solver_transport): "none" (one GPU), "nccl", "p2p", "loopback", "loopback-p2p"."""
        return self.TRANSPORTS[lib().eg_solver_transport(self._h)]
