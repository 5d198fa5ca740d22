"""Algorithmic work model of one operator apply (roofline numerators).

F_alg counts the floating-point operations the method must execute (FMA = 2),
each face counted once (not the element-centric duplicate), no padding, no
avoided dense work (SURVEY §8(d) "Algorithmic work definitions").  B_alg counts
the bytes that must cross HBM: read u + write v (16 B/DoF), the quadrature data
(32 B per volume point, 56 B per interface point, 24 B per cut-face point; the
paper's per-point sizes P:907, P:918 plus the normal) and the per-cell
descriptors.  The paper's own closed forms are exposed
for the golden tests.
"""
from __future__ import annotations


def c_eo(n: int) -> int:
    """flops of one even-odd n x n line product."""
    H, HC = n // 2, (n + 1) // 2
    if n % 2 == 0:
        return n * n + 2 * n
    return 2 * H + 2 * (HC * HC + H * H) + 2 * H


def flops_uncut_cell(n: int) -> int:
    """2 x (6 n^2 1-D lines x even-odd cost) + 3 n^3 quadrature scalings
    (interpolate + collocation derivative per direction, then the transposes;
    P:857-861)."""
    return 2 * 6 * n * n * c_eo(n) + 3 * n ** 3


def flops_struct_face(n: int) -> int:
    """SURVEY §8(d), one full face, both sides: normal-derivative trace 2 n^3 per side,
    in-face interpolation of 2 fields (2 sweeps of n lines each), x2 sides, x2 (E + I),
    plus the flux at the n^2 points."""
    return 2 * 2 * (2 * n ** 3 + 2 * 2 * n * c_eo(n)) + 10 * n * n


def flops_gp_face(n: int) -> int:
    """One ghost-penalty face, both sides: n = p+1 normal-derivative traces per
    in-face node projected and back-projected on each side (4 n^4 FMA), in-face mass
    on the n jump fields (2 sweeps of n lines each per field)."""
    return 8 * n ** 4 + 2 * n * n * c_eo(n)


def flops_vol_point(n: int) -> int:
    """SURVEY §8(d) cut-cell point: 2 x 2 (2n^3 + 3n^2 + 4n) (values + gradients,
    P:869-872, evaluate and integrate) + 1-D basis 2 * 3 n (n-1) + 12 point ops."""
    return 4 * (2 * n ** 3 + 3 * n * n + 4 * n) + 6 * n * (n - 1) + 12


def flops_srf_point(n: int) -> int:
    """an interface point: a volume point + 12 Nitsche point ops."""
    return flops_vol_point(n) + 12


def flops_cut_face(n: int, n_pts: int) -> int:
    """SURVEY §8(d) cut face, both sides: 2 (FMA) x 2 (E + I) x 2 (sides) x the paper's
    unstructured face count k^3 + n_q (3k^2 + 4k) (= 3k^4 + 5k^3 at
    n_q = k^2), with the face's actual point count n_q."""
    return 8 * (n ** 3 + n_pts * (3 * n * n + 4 * n))


def face_classes(prob, owned=None) -> dict:
    """Face sides by kind from the problem arrays (the ones cutfem_setup takes):
    every face between two active cells is a full SIPG face unless listed in sf_*
    (then a cut face, or no SIPG when its point range is empty); it is a ghost-
    penalty face when a side is cut.  Each face's work is split in halves between
    its two sides; a side belongs to the cut-cell kernel when its cell is cut.
    ``owned``: optional bool mask of the blocks whose sides are counted."""
    import numpy as np
    ijk = np.asarray(prob.active_ijk, dtype=np.int64)
    cut = np.asarray(prob.is_cut).astype(bool)
    nb = ijk.shape[0]
    own = np.ones(nb, bool) if owned is None else np.asarray(owned, bool)
    out = {"sipg_side_cut": 0, "sipg_side_uncut": 0, "gp_side_cut": 0, "gp_side_uncut": 0,
           "cutface_side": 0, "cutface_pts_side": 0}
    if nb == 0:
        return out
    lo = ijk.min(0)
    dims = ijk.max(0) - lo + 2
    key = ((ijk[:, 0] - lo[0]) * dims[1] + (ijk[:, 1] - lo[1])) * dims[2] + (ijk[:, 2] - lo[2])
    order = np.argsort(key)
    skey = key[order]
    listed = {}
    sfc, sfa, sfp = np.asarray(prob.sf_cells), np.asarray(prob.sf_axis), np.asarray(prob.sf_ptr)
    for f in range(sfc.shape[0]):
        listed[(int(sfc[f, 0]), int(sfa[f]))] = int(sfp[f + 1] - sfp[f])
    for d in range(3):
        step = (dims[1] * dims[2], dims[2], 1)[d]
        pos = np.searchsorted(skey, key + step)
        hit = (pos < nb) & (skey[np.minimum(pos, nb - 1)] == key + step)
        m = np.where(hit)[0]
        pl = order[pos[hit]]
        for a, b in zip(m.tolist(), pl.tolist()):
            npt = listed.get((a, d), -1)
            gp = cut[a] or cut[b]
            for side in (a, b):
                if not own[side]:
                    continue
                c = "cut" if cut[side] else "uncut"
                if gp:
                    out["gp_side_" + c] += 1
                if npt < 0:
                    out["sipg_side_" + c] += 1
                elif npt > 0:
                    out["cutface_side"] += 1
                    out["cutface_pts_side"] += npt
    return out


def apply_work(stats: dict, classes: dict) -> dict:
    """F_alg / B_alg of one apply, in total and per kernel family, from the
    cutfem_stats() counters and face_classes().  Per-unit counts: SURVEY §8(d)
    (functions above).  Attribution follows the kernels: the cut-cell kernel
    (k_cutp at p <= 3, k_cut at p >= 4) computes the volume / interface points,
    the cut faces and the cut cells' halves of the full-face SIPG and ghost-penalty
    faces; the structured family (k_tile2 + k_gpw, k_cell, k_uncw, k_uncut)
    computes the uncut cells and their face halves.  Bytes: 8 B read u + 8 B write v
    per DoF, 32 / 56 / 24 B per volume / interface / cut-face point, 8 B per cell and
    12 B per special (ghost-penalty or cut) face side of metadata."""
    n = stats["degree"] + 1
    n3 = n ** 3
    nu, nc = stats["n_uncut"], stats["n_cut"]
    c = classes
    half_s, half_g = flops_struct_face(n) / 2, flops_gp_face(n) / 2
    F_unc = nu * flops_uncut_cell(n) + c["sipg_side_uncut"] * half_s + c["gp_side_uncut"] * half_g
    # cut faces: half of flops_cut_face per side (a listed face has two cut sides)
    F_cut = (stats["n_vol_pts"] * flops_vol_point(n) + stats["n_srf_pts"] * flops_srf_point(n)
             + 4 * (c["cutface_side"] * n ** 3 + c["cutface_pts_side"] * (3 * n * n + 4 * n))
             + c["sipg_side_cut"] * half_s + c["gp_side_cut"] * half_g)
    B_unc = 16 * nu * n3 + 8 * nu + 12 * c["gp_side_uncut"]
    B_cut = (16 * nc * n3 + 8 * nc + 32 * stats["n_vol_pts"] + 56 * stats["n_srf_pts"]
             + 24 * stats["n_face_pts"] + 12 * (c["gp_side_cut"] + c["cutface_side"]))
    return {"F_uncut": F_unc, "F_cut": F_cut, "F_total": F_unc + F_cut,
            "B_uncut": B_unc, "B_cut": B_cut, "B_total": B_unc + B_cut, "B_vectors": 16 * stats["n_dofs"]}


# ------------------------------------------------ the paper's closed forms (k = p+1)
def paper_structured_cell_fma(k: int) -> int:
    return 6 * k ** 4


def paper_structured_face_fma(k: int) -> int:
    return 7 * k ** 3


def paper_unstructured_cell_fma(k: int) -> int:    # P:869-872 at n_q = k^3
    return 2 * k ** 6 + 3 * k ** 5 + 4 * k ** 4


def paper_unstructured_face_fma(k: int) -> int:    # P:880-883 at n_q = k^2
    return 3 * k ** 4 + 5 * k ** 3


def paper_sparse_dg_bytes_per_dof(p: int, d: int = 3) -> int:
    return 12 * (2 * d + 1) * (p + 1) ** d


def paper_sparse_dg_flops_per_dof(p: int, d: int = 3) -> int:
    return 2 * (2 * d + 1) * (p + 1) ** d


def paper_sparse_cg_bytes_per_dof(p: int, d: int = 3) -> int:
    return 12 * (p + 2) ** d


def paper_sparse_cg_flops_per_dof(p: int, d: int = 3) -> int:
    return 2 * (p + 2) ** d


# ------------------------------------------------------------------- peaks
B200_SMS = 148
B200_FP64_FMA_PER_SM_CLK = 64     # FP64 lanes per SM (4 SMSPs x 16)
B200_SM_MAX_MHZ = 1965.0


def fp64_peak_tflops(sm_mhz: float = B200_SM_MAX_MHZ) -> float:
    """Derived FP64 peak: SMs x FP64 FMA lanes x 2 flops x clock."""
    return B200_SMS * B200_FP64_FMA_PER_SM_CLK * 2 * sm_mhz * 1e6 / 1e12
