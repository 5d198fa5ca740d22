"""Oracle of the CONTINUOUS Galerkin (H^1-conforming) CutFEM operator (SURVEY §8(f)
f2) -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md eq:bilinear_cg: on the continuous Q_p space of the active cells
(nodal Lagrange basis in the GLL points, which coincide on shared faces,
edges and vertices),

  a_CG(v,u) = int_{Omega} grad v . grad u
            - int_Gamma (d_n v) u - int_Gamma v (d_n u - tau_D/h u)        (Nitsche)
            + face ghost penalty: sum_{F touching a cut cell} sum_{j=0..p}
              g_j h^(2j-1) int_F [d_n^j v][d_n^j u]                       (BASELINE configs[0], SM1)

(no SIPG: [u] = 0; the j = 0 jump of a continuous function vanishes, DESIGN
reading A22).  Plain definition: the global basis function of lattice node i is
the sum of the cell basis functions that sit on that node, so the matrix is the
standard finite-element assembly  A_CG = sum_K P_K^T A_K P_K + sum_F P_F^T A_F P_F
with the local matrices of the DG oracle (volume + Nitsche per cell, GP per face:
the same integrals) and P_K the 0/1 gather from the global numbering.

Global numbering: lattice node (p i + a, p j + b, p k + c) of cell (i, j, k),
local index (a, b, c); nodes of active cells only, numbered in lexicographic
order (x slowest), the order the C ABI's cutfem_h1_map also uses.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .operator import TERM_CELL, TERM_GP, TERM_NITSCHE, Oracle

TERM_H1 = TERM_CELL | TERM_NITSCHE | TERM_GP


def h1_numbering(prob):
    """(n_h1, map) with map[K, l] = global H1 DoF of local node l of block K."""
    p = prob.degree
    n = p + 1
    ijk = np.asarray(prob.active_ijk, dtype=np.int64)
    a = np.arange(n)
    C, B, A = np.meshgrid(a, a, a, indexing="ij")  # l = a + n b + n^2 c
    loc = np.stack([A.ravel(), B.ravel(), C.ravel()], 1)
    lat = p * ijk[:, None, :] + loc[None]  # (K, l, 3)
    dims = lat.reshape(-1, 3).max(0) + 1 if len(ijk) else np.ones(3, np.int64)
    key = (lat[..., 0] * dims[1] + lat[..., 1]) * dims[2] + lat[..., 2]
    uniq, inv = np.unique(key.ravel(), return_inverse=True)
    return int(uniq.size), inv.reshape(key.shape)


class OracleH1:
    def __init__(self, prob, term_mask: int = TERM_H1):
        self.P = prob
        self.dg = Oracle(prob, term_mask=term_mask & TERM_H1)
        self.n_h1, self.map = h1_numbering(prob)
        self.nd = (prob.degree + 1) ** 3

    def gather_matrix(self):
        """P: (n_blocks * n^3) x n_h1, the 0/1 gather u_K = P_K u."""
        nb = self.map.shape[0]
        rows = np.arange(nb * self.nd)
        return sp.csr_matrix((np.ones(rows.size), (rows, self.map.ravel())), shape=(nb * self.nd, self.n_h1))

    def assemble_csr(self):
        """A_CG = P^T A P with A the DG oracle's local matrices without SIPG."""
        Pm = self.gather_matrix()
        A = self.dg.assemble_csr()
        M = (Pm.T @ A @ Pm).tocsr()
        M.sum_duplicates()
        M.sort_indices()
        return M

    def apply(self, u):
        """v = A_CG u, blockwise: gather, local matrices, scatter-add."""
        u = np.asarray(u, dtype=np.float64)
        ub = u[self.map]  # (K, n^3)
        vb = self.dg.apply(ub.reshape(-1)).reshape(ub.shape)
        v = np.zeros(self.n_h1)
        np.add.at(v, self.map.ravel(), vb.ravel())
        return v

    def rhs(self, f):
        """b_i = int_Omega f phi_i."""
        bb = self.dg.rhs(f).reshape(-1, self.nd)
        b = np.zeros(self.n_h1)
        np.add.at(b, self.map.ravel(), bb.ravel())
        return b

    def l2_error(self, uh, uex, extra: int = 2):
        return self.dg.l2_error(np.asarray(uh)[self.map].reshape(-1), uex, extra)
