"""ctypes binding of libcutfem.so (include/cutfem.h).  Marshalling only."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
_SO = os.path.join(_HERE, "libcutfem.so")
_SRC_DIR = os.path.join(_HERE, "csrc")
_HDR = os.path.join(_ROOT, "include", "cutfem.h")

TERM_CELL, TERM_SIPG, TERM_NITSCHE, TERM_GP = 1, 2, 4, 8
TERM_ALL = 15

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]


def lib_path() -> str:
    return _SO


def _sources():
    return [os.path.join(_SRC_DIR, f) for f in sorted(os.listdir(_SRC_DIR))] + [_HDR]


def _nccl_dir() -> str:
    """NCCL shipped with torch (nvidia-nccl wheel): headers + libnccl.so.2."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is not None and spec.submodule_search_locations:
        return list(spec.submodule_search_locations)[0]
    raise RuntimeError("NCCL (nvidia.nccl) not found")


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile libcutfem.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    stale = force or not os.path.exists(_SO) or any(
        os.path.getmtime(s) > os.path.getmtime(_SO) for s in _sources())
    if stale:
        nccl = _nccl_dir()
        cmd = ["nvcc", *NVCC_FLAGS, "-I", os.path.join(_ROOT, "include"), "-I", os.path.join(nccl, "include"),
               "-o", _SO, os.path.join(_SRC_DIR, "cutfem.cu"), "-lcusparse", "-L", os.path.join(nccl, "lib"),
               "-l:libnccl.so.2", "-Xlinker", "-rpath=" + os.path.join(nccl, "lib")]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
    return _SO


class _Problem(ctypes.Structure):
    _fields_ = [
        ("n_cells", ctypes.c_int32 * 3), ("lower", ctypes.c_double * 3), ("h", ctypes.c_double),
        ("degree", ctypes.c_int32), ("n_active", ctypes.c_int64),
        ("active_ijk", ctypes.c_void_p), ("is_cut", ctypes.c_void_p),
        ("vol_ptr", ctypes.c_void_p), ("vol_pts", ctypes.c_void_p),
        ("srf_ptr", ctypes.c_void_p), ("srf_pts", ctypes.c_void_p),
        ("n_sfaces", ctypes.c_int64), ("sf_cells", ctypes.c_void_p), ("sf_axis", ctypes.c_void_p),
        ("sf_ptr", ctypes.c_void_p), ("sf_pts", ctypes.c_void_p),
        ("sipg_gamma", ctypes.c_double), ("nitsche_tau", ctypes.c_double),
        ("gp_gamma", ctypes.c_void_p), ("term_mask", ctypes.c_uint32),
        ("gp_kind", ctypes.c_int32), ("tau_v", ctypes.c_double),
    ]


class Stats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in (
        "n_active", "n_uncut", "n_cut", "n_vol_pts", "n_srf_pts", "n_face_pts", "n_faces_struct",
        "n_faces_cut", "n_faces_empty", "n_faces_gp", "n_dofs")] + [
        ("degree", ctypes.c_int32), ("device", ctypes.c_int32), ("dev_bytes", ctypes.c_int64),
        ("launches_per_apply", ctypes.c_int32), ("reserved", ctypes.c_int32),
        ("n_ext_dofs", ctypes.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "reserved"}


EXPORTS = ["cutfem_setup", "cutfem_apply", "cutfem_apply_kernel", "cutfem_apply_host", "cutfem_apply_host_batch",
           "cutfem_csr_assemble",
           "cutfem_csr_setup", "cutfem_csr_apply", "cutfem_csr_nnz", "cutfem_csr_download",
           "cutfem_stats", "cutfem_last_error", "cutfem_destroy", "cutfem_partition_x",
           "cutfem_local_build", "cutfem_local_free", "cutfem_nccl_unique_id", "cutfem_setup_dist",
           "cutfem_dist_info", "cutfem_rhs_const", "cutfem_cg", "cutfem_h1_setup", "cutfem_h1_ndofs",
           "cutfem_h1_map", "cutfem_h1_apply", "cutfem_h1_rhs_const", "cutfem_h1_stats", "cutfem_h1_destroy",
           "cutfem_pcg", "cutfem_diag", "cutfem_h1_pcg", "cutfem_h1_diag", "cutfem_mg_setup", "cutfem_mg_lambda",
           "cutfem_mg_set_lambda", "cutfem_mg_vcycle", "cutfem_mg_pcg", "cutfem_mg_smooth", "cutfem_mg_transfer",
           "cutfem_mg_destroy"]


PRECOND = {"none": 0, "jacobi": 1}
INNER = {"jacobi": 0, "block": 1}


class MGParams(ctypes.Structure):
    _fields_ = [("inner", ctypes.c_int32), ("smooth_degree", ctypes.c_int32), ("smooth_range", ctypes.c_double),
                ("coarse_degree", ctypes.c_int32), ("coarse_range", ctypes.c_double),
                ("eig_iters", ctypes.c_int32), ("eig_safety", ctypes.c_double)]


class _Local(ctypes.Structure):
    _fields_ = [("pb", _Problem), ("n_own", ctypes.c_int64), ("n_ghost_lo", ctypes.c_int64),
                ("n_ghost_hi", ctypes.c_int64), ("global_begin", ctypes.c_int64),
                ("plane_lo", ctypes.c_int64), ("plane_hi", ctypes.c_int64), ("storage", ctypes.c_void_p)]

_lib = None


def load(path: str | None = None):
    """Load libcutfem.so; raises if it is missing (no fallback path exists)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or os.environ.get("CUTFEM_LIB") or _SO
    if not os.path.exists(p):
        raise RuntimeError(f"libcutfem.so not built ({p}); run __graft_entry__.build()")
    L = ctypes.CDLL(p)
    vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
    L.cutfem_setup.argtypes = [ctypes.POINTER(_Problem), i32, ctypes.POINTER(vp)]
    L.cutfem_apply.argtypes = [vp, vp, vp, vp]
    L.cutfem_apply_host.argtypes = [vp, vp, vp, vp]
    L.cutfem_apply_host_batch.argtypes = [vp, vp, vp, ctypes.c_int64, vp]
    L.cutfem_apply_host_batch.restype = i32
    L.cutfem_apply_kernel.argtypes = [vp, ctypes.c_int, vp, vp, vp]
    L.cutfem_csr_assemble.argtypes = [vp, ctypes.POINTER(i64)]
    L.cutfem_csr_setup.argtypes = [vp, i64, vp, vp, vp]
    L.cutfem_csr_apply.argtypes = [vp, vp, vp, vp]
    L.cutfem_csr_nnz.argtypes = [vp]
    L.cutfem_csr_nnz.restype = i64
    L.cutfem_csr_download.argtypes = [vp, vp, vp, vp]
    L.cutfem_stats.argtypes = [vp, ctypes.POINTER(Stats)]
    L.cutfem_rhs_const.argtypes = [vp, ctypes.c_double, vp, vp]
    L.cutfem_cg.argtypes = [vp, vp, vp, ctypes.c_int, ctypes.c_double, vp, ctypes.POINTER(ctypes.c_int), vp]
    L.cutfem_last_error.restype = ctypes.c_char_p
    L.cutfem_destroy.argtypes = [vp]
    L.cutfem_partition_x.argtypes = [ctypes.POINTER(_Problem), ctypes.c_int, ctypes.c_double, vp]
    L.cutfem_local_build.argtypes = [ctypes.POINTER(_Problem), ctypes.c_int32, ctypes.c_int32,
                                     ctypes.POINTER(_Local)]
    L.cutfem_local_free.argtypes = [ctypes.POINTER(_Local)]
    L.cutfem_local_free.restype = None
    L.cutfem_nccl_unique_id.argtypes = [vp, i64]
    L.cutfem_setup_dist.argtypes = [ctypes.POINTER(_Problem), ctypes.c_int32, ctypes.c_int32, i32, i32, vp, i32,
                                    ctypes.POINTER(vp)]
    L.cutfem_dist_info.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.cutfem_debug_loopback.argtypes = [vp, vp, vp]
    L.cutfem_h1_setup.argtypes = [ctypes.POINTER(_Problem), i32, ctypes.POINTER(vp)]
    L.cutfem_h1_ndofs.argtypes = [vp, ctypes.POINTER(i64)]
    L.cutfem_h1_map.argtypes = [vp, vp]
    L.cutfem_h1_apply.argtypes = [vp, vp, vp, vp]
    L.cutfem_h1_rhs_const.argtypes = [vp, ctypes.c_double, vp, vp]
    L.cutfem_h1_stats.argtypes = [vp, ctypes.POINTER(Stats)]
    L.cutfem_h1_destroy.argtypes = [vp]
    pcg_args = [vp, vp, vp, ctypes.c_int, ctypes.c_double, ctypes.c_int, vp, ctypes.POINTER(ctypes.c_int), vp]
    L.cutfem_pcg.argtypes = pcg_args
    L.cutfem_h1_pcg.argtypes = pcg_args
    L.cutfem_diag.argtypes = [vp, vp, vp]
    L.cutfem_h1_diag.argtypes = [vp, vp, vp]
    L.cutfem_mg_setup.argtypes = [ctypes.POINTER(vp), ctypes.c_int32, ctypes.POINTER(MGParams), vp,
                                  ctypes.POINTER(vp)]
    L.cutfem_mg_lambda.argtypes = [vp, vp]
    L.cutfem_mg_set_lambda.argtypes = [vp, vp]
    L.cutfem_mg_vcycle.argtypes = [vp, vp, vp, vp]
    L.cutfem_mg_pcg.argtypes = [vp, vp, vp, ctypes.c_int, ctypes.c_double, vp, ctypes.POINTER(ctypes.c_int), vp]
    L.cutfem_mg_smooth.argtypes = [vp, ctypes.c_int32, vp, vp, ctypes.c_int32, ctypes.c_double, ctypes.c_double,
                                   ctypes.c_int32, vp]
    L.cutfem_mg_transfer.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, vp, vp, vp]
    L.cutfem_mg_destroy.argtypes = [vp]
    for name in ("cutfem_mg_setup", "cutfem_mg_lambda", "cutfem_mg_set_lambda", "cutfem_mg_vcycle", "cutfem_mg_pcg",
                 "cutfem_mg_smooth", "cutfem_mg_transfer", "cutfem_mg_destroy"):
        getattr(L, name).restype = i32
    for name in ("cutfem_setup", "cutfem_apply", "cutfem_apply_kernel", "cutfem_apply_host", "cutfem_csr_assemble",
                 "cutfem_csr_setup", "cutfem_csr_apply", "cutfem_csr_download", "cutfem_stats",
                 "cutfem_destroy", "cutfem_partition_x", "cutfem_local_build", "cutfem_nccl_unique_id",
                 "cutfem_setup_dist", "cutfem_dist_info", "cutfem_h1_setup", "cutfem_h1_ndofs", "cutfem_h1_map",
                 "cutfem_h1_apply", "cutfem_h1_rhs_const", "cutfem_h1_stats", "cutfem_h1_destroy",
                 "cutfem_pcg", "cutfem_diag", "cutfem_h1_pcg", "cutfem_h1_diag"):
        getattr(L, name).restype = i32
    if path is None:
        _lib = L
    return L


def _check(rc):
    if rc != 0:
        raise RuntimeError(f"cutfem error {rc}: {load().cutfem_last_error().decode()}")


def _ptr(a):
    return a.ctypes.data if a is not None and a.size else None


def _stream_ptr(stream):
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _marshal(prob, term_mask=TERM_ALL):
    """Problem fields -> _Problem (with the numpy arrays kept alive in `keep`)."""
    keep = {
        "ijk": np.ascontiguousarray(prob.active_ijk, dtype=np.int32),
        "cut": np.ascontiguousarray(prob.is_cut, dtype=np.uint8),
        "vp": np.ascontiguousarray(prob.vol_ptr, dtype=np.int64),
        "vx": np.ascontiguousarray(prob.vol_pts, dtype=np.float64),
        "sp": np.ascontiguousarray(prob.srf_ptr, dtype=np.int64),
        "sx": np.ascontiguousarray(prob.srf_pts, dtype=np.float64),
        "fc": np.ascontiguousarray(prob.sf_cells, dtype=np.int32),
        "fa": np.ascontiguousarray(prob.sf_axis, dtype=np.uint8),
        "fp": np.ascontiguousarray(prob.sf_ptr, dtype=np.int64),
        "fx": np.ascontiguousarray(prob.sf_pts, dtype=np.float64),
        "gp": np.ascontiguousarray(prob.gp_gamma, dtype=np.float64),
    }
    pb = _Problem()
    for i in range(3):
        pb.n_cells[i] = int(prob.n_cells[i])
        pb.lower[i] = float(prob.lower[i])
    pb.h = float(prob.h)
    pb.degree = int(prob.degree)
    pb.n_active = keep["ijk"].shape[0]
    pb.active_ijk, pb.is_cut = _ptr(keep["ijk"]), _ptr(keep["cut"])
    pb.vol_ptr, pb.vol_pts = _ptr(keep["vp"]), _ptr(keep["vx"])
    pb.srf_ptr, pb.srf_pts = _ptr(keep["sp"]), _ptr(keep["sx"])
    pb.n_sfaces = keep["fc"].shape[0]
    pb.sf_cells, pb.sf_axis = _ptr(keep["fc"]), _ptr(keep["fa"])
    pb.sf_ptr, pb.sf_pts = _ptr(keep["fp"]), _ptr(keep["fx"])
    pb.sipg_gamma, pb.nitsche_tau = float(prob.sipg_gamma), float(prob.nitsche_tau)
    pb.gp_gamma = _ptr(keep["gp"])
    pb.term_mask = int(term_mask)
    pb.gp_kind = int(getattr(prob, "gp_kind", 0))
    pb.tau_v = float(getattr(prob, "tau_v", 1.0))
    return pb, keep


def _arr(ptr, n, ctype, dtype, shape):
    if n == 0 or not ptr:
        return np.zeros(shape, dtype=dtype)
    return np.ctypeslib.as_array(ctypes.cast(ptr, ctypes.POINTER(ctype)), shape=(n,)).astype(dtype).reshape(shape)


def partition_x(prob, nparts: int, w_cut: float = 7.0):
    """Weighted x-slab split (host only): list of nparts+1 plane indices."""
    L = load()
    pb, keep = _marshal(prob)
    out = np.zeros(nparts + 1, dtype=np.int32)
    _check(L.cutfem_partition_x(ctypes.byref(pb), int(nparts), float(w_cut), out.ctypes.data))
    return [int(x) for x in out]


class LocalProblem:
    """Local problem of one x-slab (host only), built by the C library: owned blocks
    then the ghost planes.  Field names match cutgen.Problem."""

    def __init__(self, prob, x_begin: int, x_end: int):
        L = load()
        pb, keep = _marshal(prob)
        loc = _Local()
        _check(L.cutfem_local_build(ctypes.byref(pb), int(x_begin), int(x_end), ctypes.byref(loc)))
        try:
            q = loc.pb
            na, n_sf = int(q.n_active), int(q.n_sfaces)
            self.active_ijk = _arr(q.active_ijk, 3 * na, ctypes.c_int32, np.int32, (na, 3))
            self.is_cut = _arr(q.is_cut, na, ctypes.c_uint8, np.uint8, (na,))
            nc = int(self.is_cut.sum())
            self.vol_ptr = _arr(q.vol_ptr, nc + 1, ctypes.c_int64, np.int64, (nc + 1,))
            self.srf_ptr = _arr(q.srf_ptr, nc + 1, ctypes.c_int64, np.int64, (nc + 1,))
            self.vol_pts = _arr(q.vol_pts, 4 * int(self.vol_ptr[-1]), ctypes.c_double, np.float64, (-1, 4))
            self.srf_pts = _arr(q.srf_pts, 7 * int(self.srf_ptr[-1]), ctypes.c_double, np.float64, (-1, 7))
            self.sf_cells = _arr(q.sf_cells, 2 * n_sf, ctypes.c_int32, np.int32, (n_sf, 2))
            self.sf_axis = _arr(q.sf_axis, n_sf, ctypes.c_uint8, np.uint8, (n_sf,))
            self.sf_ptr = _arr(q.sf_ptr, n_sf + 1, ctypes.c_int64, np.int64, (n_sf + 1,))
            self.sf_pts = _arr(q.sf_pts, 3 * int(self.sf_ptr[-1]), ctypes.c_double, np.float64, (-1, 3))
            self.n_own, self.n_ghost_lo, self.n_ghost_hi = int(loc.n_own), int(loc.n_ghost_lo), int(loc.n_ghost_hi)
            self.global_begin, self.plane_lo, self.plane_hi = int(loc.global_begin), int(loc.plane_lo), int(loc.plane_hi)
        finally:
            L.cutfem_local_free(ctypes.byref(loc))
        for k in ("n_cells", "lower", "h", "degree", "sipg_gamma", "nitsche_tau", "gp_gamma", "level_set"):
            setattr(self, k, getattr(prob, k))
        self.vol_pts = self.vol_pts.reshape(-1, 4)
        self.srf_pts = self.srf_pts.reshape(-1, 7)
        self.sf_pts = self.sf_pts.reshape(-1, 3)

    @property
    def n_active(self):
        return int(self.active_ijk.shape[0])

    @property
    def n_dofs(self):
        return self.n_active * (self.degree + 1) ** 3


def nccl_unique_id() -> bytes:
    L = load()
    buf = ctypes.create_string_buffer(128)
    _check(L.cutfem_nccl_unique_id(buf, 128))
    return bytes(buf.raw)


class CutFEM:
    """Handle for v = A u on one GPU.  ``prob`` is a cutgen.Problem (or anything
    with the same fields).  Device vectors are torch.float64 CUDA tensors."""

    def __init__(self, prob, device: int = 0, term_mask: int = TERM_ALL, _dist=None):
        L = load()
        pb, keep = _marshal(prob, term_mask)
        h = ctypes.c_void_p()
        if _dist is None:
            _check(L.cutfem_setup(ctypes.byref(pb), int(device), ctypes.byref(h)))
        else:
            x0, x1, rank, nranks, nid = _dist
            idb = ctypes.create_string_buffer(nid, 128) if nid is not None else None
            _check(L.cutfem_setup_dist(ctypes.byref(pb), int(x0), int(x1), int(rank), int(nranks), idb,
                                       int(device), ctypes.byref(h)))
        self._h = h
        self._L = L
        self.device = device
        self.degree = int(prob.degree)
        st = self.stats()
        self.n_dofs = int(st["n_dofs"])          # v length (owned blocks)
        self.n_ext_dofs = int(st["n_ext_dofs"])  # u length (owned + ghost blocks)

    def stats(self) -> dict:
        s = Stats()
        _check(self._L.cutfem_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def apply(self, u, v=None, stream=None):
        """v = A u on the device (torch float64 CUDA tensors), stream-ordered."""
        import torch
        if v is None:
            v = torch.empty(self.n_dofs, dtype=u.dtype, device=u.device)
        assert u.dtype == torch.float64 and v.dtype == torch.float64 and u.is_cuda and v.is_cuda
        assert u.numel() == self.n_ext_dofs and v.numel() == self.n_dofs
        assert u.is_contiguous() and v.is_contiguous()
        _check(self._L.cutfem_apply(self._h, u.data_ptr(), v.data_ptr(), _stream_ptr(stream)))
        return v

    def apply_kernel(self, which: int, u, v, stream=None):
        """Launch only the structured (0) or unstructured (1) kernel (timing attribution)."""
        _check(self._L.cutfem_apply_kernel(self._h, int(which), u.data_ptr(), v.data_ptr(),
                                           _stream_ptr(stream)))
        return v

    def apply_host(self, u: np.ndarray, v: np.ndarray | None = None, stream=0) -> np.ndarray:
        """End-to-end path: host u -> device -> A u -> host v (synchronous)."""
        u = np.ascontiguousarray(u, dtype=np.float64)
        if v is None:
            v = np.empty_like(u)
        assert u.size == self.n_dofs and v.size == self.n_dofs and v.flags.c_contiguous
        _check(self._L.cutfem_apply_host(self._h, u.ctypes.data, v.ctypes.data,
                                         _stream_ptr(stream) if stream else None))
        return v

    def apply_host_batch(self, us, vs, stream=0):
        """Pipelined end-to-end path: vs[k] = A us[k] for a list of host arrays (page-locked
        memory lets the copies overlap the applies); synchronous."""
        assert len(us) == len(vs)
        for a in list(us) + list(vs):
            assert a.dtype == np.float64 and a.size == self.n_dofs and a.flags.c_contiguous
        up = (ctypes.c_void_p * len(us))(*[a.ctypes.data for a in us])
        vp = (ctypes.c_void_p * len(vs))(*[a.ctypes.data for a in vs])
        _check(self._L.cutfem_apply_host_batch(self._h, up, vp, len(us), _stream_ptr(stream) if stream else None))
        return vs

    def rhs_const(self, f: float = 1.0, b=None, stream=None):
        """b = f * int_Omega phi_i (device, owned blocks)."""
        import torch
        if b is None:
            b = torch.empty(self.n_dofs, dtype=torch.float64, device=f"cuda:{self.device}")
        _check(self._L.cutfem_rhs_const(self._h, float(f), b.data_ptr(), _stream_ptr(stream)))
        return b

    def cg(self, b, x=None, iters: int = 50, tol: float = 0.0, stream=None, precond: str = "none"):
        """(Preconditioned) CG on A x = b in the library's kernels; x (in/out) needs
        n_ext_dofs entries; precond "none" | "jacobi".  Returns (x, ||r_k||, k = 0..done)."""
        import torch
        if x is None:
            x = torch.zeros(self.n_ext_dofs, dtype=torch.float64, device=b.device)
        assert x.numel() == self.n_ext_dofs and b.numel() == self.n_dofs
        hist = np.zeros(int(iters) + 1, dtype=np.float64)
        done = ctypes.c_int()
        _check(self._L.cutfem_pcg(self._h, b.data_ptr(), x.data_ptr(), int(iters), float(tol), PRECOND[precond],
                                  hist.ctypes.data, ctypes.byref(done), _stream_ptr(stream)))
        return x, hist[:done.value + 1]

    def diag(self, stream=None):
        """diag(A) (device), probed (include/cutfem.h cutfem_diag)."""
        import torch
        d = torch.empty(self.n_dofs, dtype=torch.float64, device=f"cuda:{self.device}")
        _check(self._L.cutfem_diag(self._h, d.data_ptr(), _stream_ptr(stream)))
        return d

    def csr_assemble(self) -> int:
        nnz = ctypes.c_int64()
        _check(self._L.cutfem_csr_assemble(self._h, ctypes.byref(nnz)))
        return int(nnz.value)

    def csr_setup(self, row_ptr, col, val):
        row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        col = np.ascontiguousarray(col, dtype=np.int32)
        val = np.ascontiguousarray(val, dtype=np.float64)
        _check(self._L.cutfem_csr_setup(self._h, row_ptr.size - 1, row_ptr.ctypes.data,
                                        col.ctypes.data, val.ctypes.data))

    def csr_apply(self, u, v=None, stream=None):
        import torch
        if v is None:
            v = torch.empty_like(u)
        _check(self._L.cutfem_csr_apply(self._h, u.data_ptr(), v.data_ptr(), _stream_ptr(stream)))
        return v

    def csr_download(self):
        nnz = int(self._L.cutfem_csr_nnz(self._h))
        rp = np.zeros(self.n_dofs + 1, dtype=np.int64)
        col = np.zeros(nnz, dtype=np.int32)
        val = np.zeros(nnz, dtype=np.float64)
        _check(self._L.cutfem_csr_download(self._h, rp.ctypes.data, col.ctypes.data, val.ctypes.data))
        return rp, col, val

    def close(self):
        if getattr(self, "_h", None):
            self._L.cutfem_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class CutFEMH1:
    """The H^1-conforming (continuous Galerkin) operator v = A_CG u on one GPU
    (include/cutfem.h cutfem_h1_*); vectors hold the n_dofs global lattice nodes."""

    def __init__(self, prob, device: int = 0, term_mask: int = TERM_ALL):
        L = load()
        pb, keep = _marshal(prob, term_mask)
        h = ctypes.c_void_p()
        _check(L.cutfem_h1_setup(ctypes.byref(pb), int(device), ctypes.byref(h)))
        self._h, self._L, self.device = h, L, device
        n = ctypes.c_int64()
        _check(L.cutfem_h1_ndofs(h, ctypes.byref(n)))
        self.n_dofs = int(n.value)
        self.n_blk = int(prob.active_ijk.shape[0]) * (int(prob.degree) + 1) ** 3

    def stats(self) -> dict:
        s = Stats()
        _check(self._L.cutfem_h1_stats(self._h, ctypes.byref(s)))
        return s.as_dict()

    def map(self) -> np.ndarray:
        m = np.zeros(self.n_blk, dtype=np.int32)
        _check(self._L.cutfem_h1_map(self._h, m.ctypes.data if m.size else None))
        return m

    def apply(self, u, v=None, stream=None):
        import torch
        if v is None:
            v = torch.empty(self.n_dofs, dtype=torch.float64, device=u.device)
        assert u.dtype == torch.float64 and u.is_cuda and u.numel() == self.n_dofs and v.numel() == self.n_dofs
        _check(self._L.cutfem_h1_apply(self._h, u.data_ptr(), v.data_ptr(), _stream_ptr(stream)))
        return v

    def rhs_const(self, f: float = 1.0, b=None, stream=None):
        import torch
        if b is None:
            b = torch.empty(self.n_dofs, dtype=torch.float64, device=f"cuda:{self.device}")
        _check(self._L.cutfem_h1_rhs_const(self._h, float(f), b.data_ptr(), _stream_ptr(stream)))
        return b

    def cg(self, b, x=None, iters: int = 50, tol: float = 0.0, stream=None, precond: str = "none"):
        import torch
        if x is None:
            x = torch.zeros(self.n_dofs, dtype=torch.float64, device=b.device)
        hist = np.zeros(int(iters) + 1, dtype=np.float64)
        done = ctypes.c_int()
        _check(self._L.cutfem_h1_pcg(self._h, b.data_ptr(), x.data_ptr(), int(iters), float(tol), PRECOND[precond],
                                     hist.ctypes.data, ctypes.byref(done), _stream_ptr(stream)))
        return x, hist[:done.value + 1]

    def diag(self, stream=None):
        import torch
        d = torch.empty(self.n_dofs, dtype=torch.float64, device=f"cuda:{self.device}")
        _check(self._L.cutfem_h1_diag(self._h, d.data_ptr(), _stream_ptr(stream)))
        return d

    def close(self):
        if getattr(self, "_h", None):
            self._L.cutfem_h1_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class CutFEMDist(CutFEM):
    """One rank's x-slab [x_begin, x_end) of the global problem.  apply(u_ext, v):
    u_ext holds n_ext_dofs values (owned blocks first; the ghost tail is filled by
    the NCCL halo exchange inside the apply), v receives the n_dofs owned values."""

    def __init__(self, prob, x_begin, x_end, rank=0, nranks=1, nccl_id=None, device=0, term_mask=TERM_ALL):
        super().__init__(prob, device=device, term_mask=term_mask,
                         _dist=(x_begin, x_end, rank, nranks, nccl_id))
        n_own, g_lo, g_hi = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _check(self._L.cutfem_dist_info(self._h, ctypes.byref(n_own), ctypes.byref(g_lo), ctypes.byref(g_hi)))
        self.n_own_blocks, self.n_ghost_lo, self.n_ghost_hi = n_own.value, g_lo.value, g_hi.value

    def debug_loopback(self, src_lo, src_hi):
        """Test only: 1-rank NCCL loopback; the halo exchange receives src_lo / src_hi
        (device tensors, the neighbours' boundary planes) into the ghost slots."""
        self._keep = (src_lo, src_hi)
        tp = lambda t: t.data_ptr() if t is not None and t.numel() else None  # noqa: E731
        _check(self._L.cutfem_debug_loopback(self._h, tp(src_lo), tp(src_hi)))


class CutFEMMG:
    """Chebyshev-smoothed polynomial multigrid over DG handles of one mesh
    (include/cutfem.h cutfem_mg_*).  ``levels``: CutFEM handles, coarsest first,
    degrees increasing.  One level = Chebyshev-preconditioned CG."""

    def __init__(self, levels, inner: str = "block", smooth_degree: int = 3, smooth_range: float = 15.0,
                 coarse_degree: int = 16, coarse_range: float = 40.0, eig_iters: int = 20, eig_safety: float = 1.1,
                 stream=None):
        L = load()
        self._L = L
        self.levels = list(levels)  # keeps the handles alive
        prm = MGParams(INNER[inner], int(smooth_degree), float(smooth_range), int(coarse_degree),
                       float(coarse_range), int(eig_iters), float(eig_safety))
        arr = (ctypes.c_void_p * len(self.levels))(*[lv._h for lv in self.levels])
        h = ctypes.c_void_p()
        _check(L.cutfem_mg_setup(arr, len(self.levels), ctypes.byref(prm), _stream_ptr(stream), ctypes.byref(h)))
        self._h = h
        self.device = self.levels[-1].device
        self.n_dofs = self.levels[-1].n_dofs

    def lambdas(self) -> np.ndarray:
        out = np.zeros(len(self.levels))
        _check(self._L.cutfem_mg_lambda(self._h, out.ctypes.data))
        return out

    def set_lambdas(self, lam):
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        assert lam.size == len(self.levels)
        _check(self._L.cutfem_mg_set_lambda(self._h, lam.ctypes.data))

    def vcycle(self, r, z=None, stream=None):
        import torch
        if z is None:
            z = torch.empty_like(r)
        _check(self._L.cutfem_mg_vcycle(self._h, r.data_ptr(), z.data_ptr(), _stream_ptr(stream)))
        return z

    def pcg(self, b, x=None, iters: int = 50, tol: float = 0.0, stream=None):
        """CG on A x = b (finest handle) preconditioned by one V-cycle per iteration.
        Returns (x, ||r_k||, k = 0..done)."""
        import torch
        if x is None:
            x = torch.zeros_like(b)
        hist = np.zeros(int(iters) + 1, dtype=np.float64)
        done = ctypes.c_int()
        _check(self._L.cutfem_mg_pcg(self._h, b.data_ptr(), x.data_ptr(), int(iters), float(tol), hist.ctypes.data,
                                     ctypes.byref(done), _stream_ptr(stream)))
        return x, hist[:done.value + 1]

    def smooth(self, level: int, r, x, degree: int, lam_max: float, lam_min: float, x0_given: bool = False,
               stream=None):
        _check(self._L.cutfem_mg_smooth(self._h, int(level), r.data_ptr(), x.data_ptr(), int(degree),
                                        float(lam_max), float(lam_min), int(bool(x0_given)), _stream_ptr(stream)))
        return x

    def transfer(self, level: int, direction: str, src, dst, stream=None):
        """direction "prolong": dst (level) = P src (level-1); "restrict": dst (level-1) = P^T src (level)."""
        _check(self._L.cutfem_mg_transfer(self._h, int(level), {"prolong": 0, "restrict": 1}[direction],
                                          src.data_ptr(), dst.data_ptr(), _stream_ptr(stream)))
        return dst

    def close(self):
        if getattr(self, "_h", None):
            self._L.cutfem_mg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
