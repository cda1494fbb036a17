"""CPU oracle of the paper's hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / ``--impl reference``
leg may import this package.  The product path (``paper_1811_03852_b200``) never imports it, and the
two share no code.  ctypes wrapper over ``oracle/liboracle.so`` (plain C, see ``oracle/oracle.h`` for
the citations of every function).  All arrays are float64 numpy arrays in the layout
q = i + nx*(k + nz*j); working-precision values are float64 arrays holding binary32 values.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
_SO = os.path.join(_HERE, "liboracle.so")

FP64, MIXED, FP32 = 0, 1, 2
MODES = {"fp64": FP64, "mixed": MIXED, "fp32": FP32}
STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_SINGULAR_DIAG", 3: "ERR_DEGENERATE_RHS",
          4: "ERR_BREAKDOWN", 5: "ERR_NONFINITE", 6: "ERR_NOMEM"}
STATUS_CODES = {v: k for k, v in STATUS.items()}


class _Params(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("maxit", ctypes.c_int32),
                ("restart_every", ctypes.c_int32), ("precond_scale", ctypes.c_double),
                ("sor_sweeps", ctypes.c_int32), ("sor_omega", ctypes.c_double),
                ("shadow", ctypes.POINTER(ctypes.c_double))]


class _Info(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("restarts", ctypes.c_int32), ("breakdowns", ctypes.c_int32),
                ("status", ctypes.c_int32), ("final_R", ctypes.c_double),
                ("true_R", ctypes.c_double)]


@dataclass
class Info:
    iters: int
    converged: bool
    restarts: int
    breakdowns: int
    status: int
    final_R: float
    true_R: float


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            subprocess.check_call(["make", "-s", "oracle/liboracle.so"], cwd=_ROOT)
        L = ctypes.CDLL(_SO)
        dp = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        L.oracle_scale.argtypes = [i64, i64, i64, dp, ctypes.c_int, dp, dp]
        L.oracle_scale.restype = ctypes.c_int
        L.oracle_apply.argtypes = [i64, i64, i64, dp, dp, dp]
        L.oracle_apply_wp.argtypes = [i64, i64, i64, ctypes.c_int, dp, dp, dp]
        L.oracle_thomas.argtypes = [i64, i64, i64, ctypes.c_int, dp, dp, dp]
        L.oracle_residual64.argtypes = [i64, i64, i64, dp, dp, dp, dp]
        L.oracle_dot.argtypes = [i64, i64, i64, ctypes.c_int, dp, dp]
        L.oracle_dot.restype = ctypes.c_double
        L.oracle_solve.argtypes = [i64, i64, i64, ctypes.c_int, dp, dp, dp, dp,
                                   ctypes.POINTER(_Params), dp, dp, ctypes.POINTER(_Info)]
        L.oracle_solve.restype = ctypes.c_int
        L.oracle_threads.restype = ctypes.c_int
        L.oracle_trisor.argtypes = [i64, i64, i64, ctypes.c_int, dp, dp, ctypes.c_int, ctypes.c_double, dp, dp]
        L.oracle_trisor.restype = ctypes.c_int
        _lib = L
    return _lib


def _dp(a):
    if a is None:
        return ctypes.cast(0, ctypes.POINTER(ctypes.c_double))
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _mode(m):
    return MODES[m] if isinstance(m, str) else int(m)


def threads() -> int:
    return int(lib().oracle_threads())


def set_threads(n: int) -> None:
    """OpenMP thread count of the oracle's row loops (results do not depend on it: per-row partial
    sums are added in row order).  For launchers that export OMP_NUM_THREADS=1 (torchrun)."""
    lib().omp_set_num_threads(ctypes.c_int(int(n)))


class OracleError(RuntimeError):
    def __init__(self, status):
        super().__init__(STATUS.get(status, str(status)))
        self.status = status


def scale(grid, bands7: np.ndarray, mode):
    """a1 (Eq. 5): returns (ahat6 [6, n], diag [n])."""
    nx, ny, nz = grid
    n = nx * ny * nz
    bands7 = np.ascontiguousarray(bands7, np.float64).reshape(7, n)
    ahat = np.empty((6, n), np.float64)
    diag = np.empty(n, np.float64)
    rc = lib().oracle_scale(nx, ny, nz, _dp(bands7), _mode(mode), _dp(ahat), _dp(diag))
    if rc != 0:
        raise OracleError(rc)
    return ahat, diag


def apply(grid, ahat6, x):
    """y = Ahat x evaluated in binary64."""
    nx, ny, nz = grid
    y = np.empty(nx * ny * nz, np.float64)
    lib().oracle_apply(nx, ny, nz, _dp(np.ascontiguousarray(ahat6)), _dp(np.ascontiguousarray(x, np.float64)), _dp(y))
    return y


def apply_wp(grid, mode, ahat6, x):
    nx, ny, nz = grid
    y = np.empty(nx * ny * nz, np.float64)
    lib().oracle_apply_wp(nx, ny, nz, _mode(mode), _dp(np.ascontiguousarray(ahat6)),
                          _dp(np.ascontiguousarray(x, np.float64)), _dp(y))
    return y


def thomas(grid, mode, ahat6, f):
    nx, ny, nz = grid
    z = np.empty(nx * ny * nz, np.float64)
    lib().oracle_thomas(nx, ny, nz, _mode(mode), _dp(np.ascontiguousarray(ahat6)),
                        _dp(np.ascontiguousarray(f, np.float64)), _dp(z))
    return z


def trisor(grid, mode, ahat6, f, sweeps=3, omega=1.5, x_init=None):
    """NEXT-1 tri-SOR (Eq. 7), red-black column ordering (see oracle.h)."""
    nx, ny, nz = grid
    z = np.empty(nx * ny * nz, np.float64)
    rc = lib().oracle_trisor(nx, ny, nz, _mode(mode), _dp(np.ascontiguousarray(ahat6)),
                             _dp(np.ascontiguousarray(f, np.float64)), int(sweeps), float(omega),
                             _dp(None if x_init is None else np.ascontiguousarray(x_init, np.float64)), _dp(z))
    if rc:
        raise OracleError(rc)
    return z


def residual64(grid, ahat6, bhat, x):
    nx, ny, nz = grid
    r = np.empty(nx * ny * nz, np.float64)
    lib().oracle_residual64(nx, ny, nz, _dp(np.ascontiguousarray(ahat6)), _dp(bhat), _dp(x), _dp(r))
    return r


def dot(grid, mode, a, b) -> float:
    nx, ny, nz = grid
    return float(lib().oracle_dot(nx, ny, nz, _mode(mode), _dp(np.ascontiguousarray(a, np.float64)),
                                  _dp(np.ascontiguousarray(b, np.float64))))


def solve(grid, mode, ahat6, diag, b, x0=None, tol=1e-4, maxit=200, restart_every=150,
          precond_scale=1.0, raise_on_error=False, sor_sweeps=0, sor_omega=1.5, rhat0=None):
    """BiCGStab (see oracle.h).  rhat0: optional shadow residual of the first start (default r0).
    Returns (x, hist[: iters+1], Info)."""
    nx, ny, nz = grid
    n = nx * ny * nz
    x = np.empty(n, np.float64)
    hist = np.full(maxit + 1, np.nan)
    sh = None if rhat0 is None else np.ascontiguousarray(rhat0, np.float64)
    prm = _Params(tol, maxit, restart_every, precond_scale, sor_sweeps, sor_omega, _dp(sh))
    info = _Info()
    rc = lib().oracle_solve(nx, ny, nz, _mode(mode), _dp(np.ascontiguousarray(ahat6)), _dp(diag),
                            _dp(np.ascontiguousarray(b, np.float64)),
                            _dp(None if x0 is None else np.ascontiguousarray(x0, np.float64)),
                            ctypes.byref(prm), _dp(x), _dp(hist), ctypes.byref(info))
    inf = Info(info.iters, bool(info.converged), info.restarts, info.breakdowns, info.status,
               info.final_R, info.true_R)
    if rc != 0 and raise_on_error:
        raise OracleError(rc)
    return x, hist[: inf.iters + 1], inf
