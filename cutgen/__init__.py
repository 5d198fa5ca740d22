"""cutgen — the shared, seeded input generator (geometry + quadrature arrays).

This package is the ONLY code shared by the CPU oracle (``oracle/``) and the
CUDA path (``paper_2404_07911_b200``).  It holds none of the operator's
arithmetic: it builds the Cartesian background mesh, classifies cells/faces
against a level set (Omega = {phi < 0}, §2.3) and writes the
unstructured volume / interface / cut-face quadrature rules by dimension
reduction, plus the seeded source vector ``u`` (SURVEY §8(d):
``numpy.random.default_rng(seed).uniform(-1, 1, n_dofs)``).

Configs C1..C5 follow BASELINE.json ``configs[0..4]``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_cutgen.so")
_SRC = os.path.join(_HERE, "csrc", "cutgen.cpp")


def build(force: bool = False) -> str:
    """Compile the generator (host C++, no CUDA)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread",
                               "-o", _SO, _SRC])
    return _SO


class _Params(ctypes.Structure):
    _fields_ = [("ls_type", ctypes.c_int32), ("ls_params", ctypes.c_double * 8),
                ("n_cells", ctypes.c_int32 * 3), ("lower", ctypes.c_double * 3),
                ("h", ctypes.c_double), ("q", ctypes.c_int32), ("max_depth", ctypes.c_int32),
                ("force_cut_cells", ctypes.c_int32), ("force_cut_faces", ctypes.c_int32),
                ("nthreads", ctypes.c_int32)]


class _Result(ctypes.Structure):
    _fields_ = [("n_active", ctypes.c_int64), ("active_ijk", ctypes.POINTER(ctypes.c_int32)),
                ("is_cut", ctypes.POINTER(ctypes.c_uint8)), ("n_cut", ctypes.c_int64),
                ("vol_ptr", ctypes.POINTER(ctypes.c_int64)), ("vol_pts", ctypes.POINTER(ctypes.c_double)),
                ("srf_ptr", ctypes.POINTER(ctypes.c_int64)), ("srf_pts", ctypes.POINTER(ctypes.c_double)),
                ("n_sfaces", ctypes.c_int64), ("sf_cells", ctypes.POINTER(ctypes.c_int32)),
                ("sf_axis", ctypes.POINTER(ctypes.c_uint8)), ("sf_ptr", ctypes.POINTER(ctypes.c_int64)),
                ("sf_pts", ctypes.POINTER(ctypes.c_double)), ("n_subdivided", ctypes.c_int64),
                ("n_nonmonotone", ctypes.c_int64)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.cutgen_generate.argtypes = [ctypes.POINTER(_Params), ctypes.POINTER(_Result)]
        _lib.cutgen_generate.restype = ctypes.c_int
        _lib.cutgen_free.argtypes = [ctypes.POINTER(_Result)]
    return _lib


@dataclass
class Problem:
    """Everything ``cutfem_setup`` consumes (include/cutfem.h ``cutfem_problem``)."""
    n_cells: tuple
    lower: tuple
    h: float
    degree: int
    active_ijk: np.ndarray          # int32 [n_active,3], block order (x slowest, z fastest)
    is_cut: np.ndarray              # uint8 [n_active]
    vol_ptr: np.ndarray             # int64 [n_cut+1]
    vol_pts: np.ndarray             # f64 [n_vol,4]  xi,eta,zeta,W (W physical JxW)
    srf_ptr: np.ndarray             # int64 [n_cut+1]
    srf_pts: np.ndarray             # f64 [n_srf,7]  xi,eta,zeta,nx,ny,nz,W
    sf_cells: np.ndarray            # int32 [n_sfaces,2] (minus=lower, plus=upper) block ids
    sf_axis: np.ndarray             # uint8 [n_sfaces]
    sf_ptr: np.ndarray              # int64 [n_sfaces+1]
    sf_pts: np.ndarray              # f64 [n_fp,3]  s,t (in-face axes ascending), W
    sipg_gamma: float               # sigma = sipg_gamma / h
    nitsche_tau: float              # tau = nitsche_tau / h
    gp_gamma: np.ndarray            # f64 [degree+1], GP weight gp_gamma[j]*h^(2j-1)
    name: str = ""
    gp_kind: int = 0                # 0 face ghost penalty, 1 volume ghost penalty (stable neighbour)
    tau_v: float = 1.0              # volume GP penalty tau_v
    level_set: dict = field(default_factory=dict)
    n_subdivided: int = 0
    n_nonmonotone: int = 0

    @property
    def n(self) -> int:
        return self.degree + 1

    @property
    def n_active(self) -> int:
        return int(self.active_ijk.shape[0])

    @property
    def n_cut(self) -> int:
        return int(self.vol_ptr.shape[0] - 1)

    @property
    def n_dofs(self) -> int:
        return self.n_active * self.n ** 3

    def seeded_u(self, seed: int) -> np.ndarray:
        return np.random.default_rng(seed).uniform(-1.0, 1.0, self.n_dofs)

    def summary(self) -> dict:
        return {"name": self.name, "degree": self.degree, "n_cells": list(self.n_cells),
                "n_active": self.n_active, "n_cut": self.n_cut, "n_dofs": self.n_dofs,
                "n_vol_pts": int(self.vol_pts.shape[0]), "n_srf_pts": int(self.srf_pts.shape[0]),
                "n_sfaces": int(self.sf_cells.shape[0]), "n_face_pts": int(self.sf_pts.shape[0]),
                "n_subdivided": self.n_subdivided, "n_nonmonotone": self.n_nonmonotone}


def _copy(ptr, n, dtype, shape):
    if n == 0:
        return np.zeros(shape, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True).reshape(shape)


def generate(level_set: dict, n_cells, lower, upper, degree: int, *, q: int | None = None,
             max_depth: int = 3, force_cut_cells: bool = False, force_cut_faces: bool = False,
             sipg_gamma: float | None = None, nitsche_tau: float | None = None,
             gp_gamma=None, nthreads: int = 0, name: str = "", gp_kind: int = 0, tau_v: float = 1.0) -> Problem:
    """Generate a problem.  ``level_set``: {"type": "sphere", "center": [..], "radius": r} |
    {"type": "gyroid", "c": c} | {"type": "plane", "normal": [..], "offset": o}.
    Penalties default to BASELINE.json: gamma = tau_D = 10 p^2, GP weights 0.1."""
    lib = _load()
    n_cells = tuple(int(v) for v in (n_cells if np.ndim(n_cells) else (n_cells,) * 3))
    lower = tuple(float(v) for v in (lower if np.ndim(lower) else (lower,) * 3))
    upper = tuple(float(v) for v in (upper if np.ndim(upper) else (upper,) * 3))
    hs = [(upper[i] - lower[i]) / n_cells[i] for i in range(3)]
    if max(hs) - min(hs) > 1e-14 * max(hs):
        raise ValueError("cells must be cubes")
    p = _Params()
    t = level_set["type"]
    if t == "sphere":
        p.ls_type = 0
        vals = list(level_set["center"]) + [level_set["radius"]]
    elif t == "gyroid":
        p.ls_type = 1
        vals = [level_set["c"]]
    elif t == "plane":
        p.ls_type = 2
        nrm = np.asarray(level_set["normal"], dtype=float)
        vals = list(nrm / np.linalg.norm(nrm)) + [level_set["offset"]]
    else:
        raise ValueError(t)
    for i, v in enumerate(vals):
        p.ls_params[i] = float(v)
    for i in range(3):
        p.n_cells[i] = n_cells[i]
        p.lower[i] = lower[i]
    p.h = hs[0]
    p.q = int(q if q is not None else degree + 1)
    p.max_depth = int(max_depth)
    p.force_cut_cells = int(force_cut_cells)
    p.force_cut_faces = int(force_cut_faces)
    p.nthreads = int(nthreads)
    r = _Result()
    rc = lib.cutgen_generate(ctypes.byref(p), ctypes.byref(r))
    if rc != 0:
        raise RuntimeError(f"cutgen_generate failed: {rc}")
    try:
        na, nc, nf = r.n_active, r.n_cut, r.n_sfaces
        vol_ptr = _copy(r.vol_ptr, nc + 1, np.int64, (nc + 1,))
        srf_ptr = _copy(r.srf_ptr, nc + 1, np.int64, (nc + 1,))
        sf_ptr = _copy(r.sf_ptr, nf + 1, np.int64, (nf + 1,))
        prob = Problem(
            n_cells=n_cells, lower=lower, h=hs[0], degree=int(degree),
            active_ijk=_copy(r.active_ijk, 3 * na, np.int32, (na, 3)),
            is_cut=_copy(r.is_cut, na, np.uint8, (na,)),
            vol_ptr=vol_ptr, vol_pts=_copy(r.vol_pts, 4 * int(vol_ptr[-1]), np.float64, (int(vol_ptr[-1]), 4)),
            srf_ptr=srf_ptr, srf_pts=_copy(r.srf_pts, 7 * int(srf_ptr[-1]), np.float64, (int(srf_ptr[-1]), 7)),
            sf_cells=_copy(r.sf_cells, 2 * nf, np.int32, (nf, 2)),
            sf_axis=_copy(r.sf_axis, nf, np.uint8, (nf,)),
            sf_ptr=sf_ptr, sf_pts=_copy(r.sf_pts, 3 * int(sf_ptr[-1]), np.float64, (int(sf_ptr[-1]), 3)),
            sipg_gamma=float(sipg_gamma if sipg_gamma is not None else 10.0 * degree ** 2),
            nitsche_tau=float(nitsche_tau if nitsche_tau is not None else 10.0 * degree ** 2),
            gp_gamma=np.asarray(gp_gamma if gp_gamma is not None else [0.1] * (degree + 1), dtype=np.float64),
            name=name, level_set=dict(level_set), gp_kind=int(gp_kind), tau_v=float(tau_v),
            n_subdivided=int(r.n_subdivided), n_nonmonotone=int(r.n_nonmonotone))
    finally:
        lib.cutgen_free(ctypes.byref(r))
    return prob


# ------------------------------------------------------------------ configs
SPHERE = {"type": "sphere", "center": [0.05, 0.03, 0.02], "radius": 0.7}
GYROID = {"type": "gyroid", "c": 0.3}
# C3 k-sweep meshes: N nearest to ~8M active DoFs per degree
C3_N = {1: 175, 2: 116, 3: 86, 4: 69, 5: 57, 6: 49, 7: 42, 8: 37}


def config(name: str, degree: int | None = None, **kw) -> Problem:
    """BASELINE.json configs: C1 (8^3, p=2), C2 (64^3, p=3), C3 (sweep, N per p),
    C4 (192^3, p=3), C5 (gyroid 96^3 of [0,1]^3, p=5)."""
    if name == "C1":
        return generate(SPHERE, 8, -1.0, 1.0, degree or 2, name="C1", **kw)
    if name == "C2":
        return generate(SPHERE, 64, -1.0, 1.0, degree or 3, name="C2", **kw)
    if name == "C3":
        p = degree or 3
        return generate(SPHERE, C3_N[p], -1.0, 1.0, p, name=f"C3p{p}", **kw)
    if name == "C4":
        return generate(SPHERE, 192, -1.0, 1.0, degree or 3, name="C4", **kw)
    if name == "C5":
        return generate(GYROID, 96, 0.0, 1.0, degree or 5, name="C5", **kw)
    raise ValueError(name)
