"""CSR SpMV of the oracle-assembled matrix in plain C with OpenMP (oracle/csrc/spmv.c)
-- TEST / BASELINE INFRASTRUCTURE ONLY (see oracle/__init__.py): the host-core
sparse-matrix baseline of bench.py's cpu_baseline (BASELINE.md "CPU-baseline plan")."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "csrc", "spmv.c")
_SO = os.path.join(_HERE, "_spmv.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O3", "-fopenmp", "-fPIC", "-shared", "-o", _SO, _SRC])
    return _SO


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        vp = ctypes.c_void_p
        _lib.oracle_spmv_csr.argtypes = [ctypes.c_int64, vp, vp, vp, vp, vp, ctypes.c_int]
        _lib.oracle_spmv_csr.restype = None
        _lib.oracle_max_threads.restype = ctypes.c_int
    return _lib


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def spmv(M, x, y=None, nthreads: int = 1):
    """y = M x for a scipy CSR matrix M (int32 column indices, int64 row pointers)."""
    L = _load()
    rp = np.ascontiguousarray(M.indptr, dtype=np.int64)
    col = np.ascontiguousarray(M.indices, dtype=np.int32)
    val = np.ascontiguousarray(M.data, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    if y is None:
        y = np.empty(M.shape[0])
    L.oracle_spmv_csr(M.shape[0], rp.ctypes.data, col.ctypes.data, val.ctypes.data, x.ctypes.data, y.ctypes.data,
                      int(nthreads))
    return y, (rp, col, val)
