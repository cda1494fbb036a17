"""Seeded synthetic problem generator (test / bench INPUT infrastructure).

Thin ctypes wrapper over ``gen/libeggen.so`` (see ``gen/eggen.h`` for the recipe and its
citations).  It holds none of the solver's arithmetic: it only draws the seven unscaled bands
C,E,W,N,S,U,D and the right-hand side b of BASELINE.json's configs.  Both the CUDA path and the
CPU oracle are fed from here; the host and device generators produce identical bits.

Field layout everywhere: q = i + nx*(k + nz*j) (longitude fastest, then level, then latitude).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, replace

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
_SO = os.path.join(_HERE, "libeggen.so")


class _Params(ctypes.Structure):
    _fields_ = [
        ("nx", ctypes.c_int64), ("ny", ctypes.c_int64), ("nz", ctypes.c_int64),
        ("seed", ctypes.c_uint64),
        ("ch_lo", ctypes.c_double), ("ch_hi", ctypes.c_double),
        ("cv_lo", ctypes.c_double), ("cv_hi", ctypes.c_double),
        ("dl_lo", ctypes.c_double), ("dl_hi", ctypes.c_double),
    ]


@dataclass(frozen=True)
class Problem:
    """One generator configuration (global grid + seed + coefficient ranges)."""
    nx: int
    ny: int
    nz: int
    seed: int = 0
    ch: tuple = (0.5, 1.5)     # c_h ~ U(0.5, 1.5)
    cv: tuple = (5.0, 50.0)    # c_v ~ U(5, 50)   (config 5: U(5, 500))
    dl: tuple = (0.01, 0.1)    # delta ~ U(0.01, 0.1)

    @property
    def n(self) -> int:
        return self.nx * self.ny * self.nz

    def with_(self, **kw) -> "Problem":
        return replace(self, **kw)

    def _c(self) -> _Params:
        return _Params(self.nx, self.ny, self.nz, self.seed, self.ch[0], self.ch[1],
                       self.cv[0], self.cv[1], self.dl[0], self.dl[1])


# BASELINE.json "configs" (tol 1e-4, maxit 200 everywhere)
CONFIGS = {
    "C1": Problem(64, 48, 10, seed=0),
    "C2": Problem(192, 144, 70, seed=1),
    "C3": Problem(640, 480, 70, seed=2),
    "C4": Problem(1536, 1152, 70, seed=3),
    "C5": Problem(2560, 1920, 70, seed=4, cv=(5.0, 500.0)),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            subprocess.check_call(["make", "-s", "gen/libeggen.so"], cwd=_ROOT)
        L = ctypes.CDLL(_SO)
        P = ctypes.POINTER(_Params)
        dp = ctypes.POINTER(ctypes.c_double)
        L.eggen_coslat.argtypes = [ctypes.c_int64, dp]
        L.eggen_mix.argtypes = [ctypes.c_uint64]
        L.eggen_mix.restype = ctypes.c_uint64
        L.eggen_uniform.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64]
        L.eggen_uniform.restype = ctypes.c_double
        L.eggen_point.argtypes = [P, dp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, dp]
        L.eggen_host.argtypes = [P, ctypes.c_int64, ctypes.c_int64, dp, dp]
        L.eggen_host.restype = ctypes.c_int
        L.eggen_device.argtypes = [P, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p]
        L.eggen_device.restype = ctypes.c_int
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def coslat(ny: int) -> np.ndarray:
    out = np.empty(ny, np.float64)
    lib().eggen_coslat(ny, _dp(out))
    return out


def mix(z: int) -> int:
    return int(lib().eggen_mix(z))


def uniform(seed: int, stream: int, q: int) -> float:
    return float(lib().eggen_uniform(seed, stream, q))


def point(prob: Problem, i: int, j: int, k: int, cl: np.ndarray | None = None) -> np.ndarray:
    """[C,E,W,N,S,U,D,b] at global (i, j, k)."""
    if cl is None:
        cl = coslat(prob.ny)
    out = np.empty(8, np.float64)
    p = prob._c()
    lib().eggen_point(ctypes.byref(p), _dp(cl), i, j, k, _dp(out))
    return out


def host(prob: Problem, j_begin: int = 0, j_end: int | None = None):
    """Rows [j_begin, j_end): returns (bands [7, n_loc] float64, b [n_loc] float64)."""
    if j_end is None:
        j_end = prob.ny
    nloc = (j_end - j_begin) * prob.nx * prob.nz
    bands = np.empty((7, nloc), np.float64)
    b = np.empty(nloc, np.float64)
    p = prob._c()
    rc = lib().eggen_host(ctypes.byref(p), j_begin, j_end, _dp(bands), _dp(b))
    if rc != 0:
        raise ValueError(f"eggen_host failed ({rc})")
    return bands, b


def device(prob: Problem, bands, b, j_begin: int = 0, j_end: int | None = None, stream=None):
    """Fill device tensors bands [7, n_loc] float64 and b [n_loc] float64 (torch, CUDA) on `stream`
    (a torch.cuda.Stream or None = current stream).  Synchronous on return."""
    import torch
    if j_end is None:
        j_end = prob.ny
    nloc = (j_end - j_begin) * prob.nx * prob.nz
    assert bands.is_cuda and bands.dtype == torch.float64 and bands.is_contiguous()
    assert bands.numel() == 7 * nloc
    assert b is None or (b.is_cuda and b.dtype == torch.float64 and b.numel() == nloc)
    st = stream if stream is not None else torch.cuda.current_stream()
    p = prob._c()
    rc = lib().eggen_device(ctypes.byref(p), j_begin, j_end, ctypes.c_void_p(bands.data_ptr()),
                            ctypes.c_void_p(b.data_ptr() if b is not None else 0),
                            ctypes.c_void_p(st.cuda_stream))
    if rc != 0:
        raise RuntimeError(f"eggen_device failed ({rc})")
