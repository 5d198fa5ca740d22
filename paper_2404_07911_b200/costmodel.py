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
    # 3 S sweeps + 3 K_c sweeps (collocation derivative, weight, transpose) + 3 S^T sweeps
    return 9 * n * n * c_eo(n) + 5 * n ** 3


def flops_struct_face(n: int) -> int:
    # normal-derivative traces both sides, flux, in-face mass on 2 fields, spread to both sides
    return 8 * n ** 3 + 4 * n * c_eo(n) + 10 * n * n


def flops_gp_face(n: int) -> int:
    # p+1 = n normal-derivative jumps per in-face node, in-face mass on the n jump fields,
    # back-projection onto both sides
    return 8 * n ** 4 + 2 * n * n * c_eo(n)


def flops_vol_point(n: int) -> int:
    # values+gradients evaluate and integrate (x2 for E and I), 1-D basis
    return 4 * (2 * n ** 3 + 3 * n * n + 4 * n) + 6 * n * (n - 1) + 12


def flops_srf_point(n: int) -> int:
    return flops_vol_point(n) + 12


def flops_cut_face(n: int, n_pts: int) -> int:
    return 8 * n ** 3 + n_pts * (8 * n * n + 8 * n + 8)


def apply_work(stats: dict) -> dict:
    """F_alg / B_alg per kernel family and in total from cutfem_stats() counters.
    Attribution follows the p <= 3 pipeline: the structured family (k_tile* +
    k_gpw) owns the uncut cells, the full-face SIPG faces and the ghost-penalty
    faces; the unstructured kernel (k_cutp) owns the volume / interface points
    and the cut faces."""
    n = stats["degree"] + 1
    n3 = n ** 3
    nu, nc = stats["n_uncut"], stats["n_cut"]
    f_struct = stats["n_faces_struct"] * flops_struct_face(n)
    f_gp = stats["n_faces_gp"] * flops_gp_face(n)
    f_uncut = nu * flops_uncut_cell(n)
    f_cut = (stats["n_vol_pts"] * flops_vol_point(n) + stats["n_srf_pts"] * flops_srf_point(n)
             + stats["n_faces_cut"] * 8 * n ** 3 + stats["n_face_pts"] * (8 * n * n + 8 * n + 8))
    F_unc = f_uncut + f_struct + f_gp
    F_cut = f_cut
    b_vec = 16 * stats["n_dofs"]
    B_unc = 16 * nu * n3 + 32 * nu
    B_cut = (16 * nc * n3 + 64 * nc + 32 * stats["n_vol_pts"] + 56 * stats["n_srf_pts"]
             + 24 * stats["n_face_pts"])
    return {"F_uncut": F_unc, "F_cut": F_cut, "F_total": F_unc + F_cut,
            "B_uncut": B_unc, "B_cut": B_cut, "B_total": B_unc + B_cut, "B_vectors": b_vec}


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
