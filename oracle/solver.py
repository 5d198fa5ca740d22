"""CPU ORACLE for the preconditioners around the operator — TEST INFRASTRUCTURE ONLY
(see oracle/__init__.py for who may import it).

PAPER §3.5 "Iterative solution": a preconditioned conjugate gradient
iteration; for high-order DG a polynomial (p-)multigrid preconditioner with
Chebyshev smoothers on the levels.  SURVEY §8(f) f4 ("Jacobi/Chebyshev on the
matrix-free operator, then p-multigrid").  What is written out here (DESIGN.md
§5.12, readings A26-A29):

* ``chebyshev``: the Chebyshev iteration with an inner preconditioner D^-1
  (``jacobi``: 1/diag(A); ``block_jacobi``: the inverse n^3 x n^3 cell blocks of A,
  the paper's additive Schwarz smoother on the cells) on the interval [lam_min, lam_max] of D^-1 A (the three-term recurrence of
  Chebyshev acceleration, Saad, Iterative Methods, Alg. 12.1), ``degree`` steps.
  Its error propagation is e_k = T_k((theta - D^-1 A)/delta) / T_k(theta/delta) e_0
  (pinned in tests/test_oracle_mg.py against numpy's Chebyshev polynomials on a
  diagonal matrix).
* ``prolongation_1d`` / ``prolongate`` / ``restrict``: the p-transfer between DG
  spaces of degrees p_c < p_f on the same mesh: the coarse cell
  polynomial interpolated at the fine GLL nodes, I[a, b] = l^c_b(x^f_a), applied
  as I (x) I (x) I per cell; restriction = the transpose.  Cells are matched by
  their (i, j, k) index; a fine cell with no coarse counterpart gets 0.
* ``vcycle``: one V-cycle, levels[0] coarsest: pre-smoothing (Chebyshev from
  0), residual, restriction, the coarser level (recursively; on the coarsest a
  Chebyshev iteration of ``coarse_degree`` from 0), prolongation of the
  correction, post-smoothing (Chebyshev started from the current iterate).  With
  the same polynomial before and after, the V-cycle is a symmetric linear map
  (pinned: u.Bv = v.Bu, SPD).
* ``pcg``: conjugate gradients with any linear preconditioner z = B r.
* ``dense_lambda_max``: the largest eigenvalue of D^-1 A by a dense symmetric
  eigensolver, what the library's Lanczos estimate (largest Ritz value from the
  Jacobi-PCG coefficients) is checked against.
"""
from __future__ import annotations

import numpy as np

from .basis import Basis1D


def chebyshev(apply, minv, r, degree: int, lam_max: float, lam_min: float, x0=None):
    """x ~ A^-1 r by ``degree`` Chebyshev steps with the inner preconditioner
    D^-1 = ``minv`` (a callable: point Jacobi, or the inverse cell blocks).
    [lam_min, lam_max] bounds the spectrum of D^-1 A that is damped.

    theta = (lam_max + lam_min)/2, delta = (lam_max - lam_min)/2, sigma = theta/delta;
    d_0 = D^-1 (r - A x_0) / theta, x_1 = x_0 + d_0;
    rho_0 = 1/sigma, rho_j = 1/(2 sigma - rho_{j-1}),
    d_j = rho_j rho_{j-1} d_{j-1} + (2 rho_j / delta) D^-1 (r - A x_j), x_{j+1} = x_j + d_j.
    A zero start needs no product for the first step (degree - 1 products)."""
    if degree < 1:
        raise ValueError("degree >= 1")
    theta = 0.5 * (lam_max + lam_min)
    delta = 0.5 * (lam_max - lam_min)
    sigma = theta / delta
    if x0 is None:
        x = np.zeros_like(r)
        res = r.copy()
    else:
        x = x0.copy()
        res = r - apply(x)
    d = minv(res) / theta
    x = x + d
    rho = 1.0 / sigma
    for _ in range(1, degree):
        rho_new = 1.0 / (2.0 * sigma - rho)
        res = r - apply(x)
        d = rho_new * rho * d + (2.0 * rho_new / delta) * minv(res)
        x = x + d
        rho = rho_new
    return x


def prolongation_1d(p_c: int, p_f: int) -> np.ndarray:
    """I[a, b] = l^c_b(x^f_a): the degree-p_c GLL Lagrange basis at the degree-p_f GLL nodes."""
    bf, bc = Basis1D(p_f), Basis1D(p_c)
    return bc.values(bf.nodes)


def block_map(ijk_f: np.ndarray, ijk_c: np.ndarray) -> np.ndarray:
    """cmap[K] = the coarse block with the same cell index as fine block K, else -1."""
    where = {tuple(int(v) for v in c): i for i, c in enumerate(ijk_c)}
    return np.array([where.get(tuple(int(v) for v in c), -1) for c in ijk_f], dtype=np.int64)


def prolongate(uc, p_c: int, p_f: int, cmap: np.ndarray) -> np.ndarray:
    """u_f|_K = (I (x) I (x) I) u_c|_{cmap[K]} (l = a + n b + n^2 c, numpy kron order z, y, x)."""
    I = prolongation_1d(p_c, p_f)
    P3 = np.kron(I, np.kron(I, I))
    nc, nf = (p_c + 1) ** 3, (p_f + 1) ** 3
    ub = np.asarray(uc).reshape(-1, nc)
    out = np.zeros((len(cmap), nf))
    for K, c in enumerate(cmap):
        if c >= 0:
            out[K] = P3 @ ub[c]
    return out.reshape(-1)


def restrict(rf, p_c: int, p_f: int, cmap: np.ndarray, n_coarse: int) -> np.ndarray:
    """The transpose of ``prolongate``."""
    I = prolongation_1d(p_c, p_f)
    P3 = np.kron(I, np.kron(I, I))
    nc, nf = (p_c + 1) ** 3, (p_f + 1) ** 3
    rb = np.asarray(rf).reshape(-1, nf)
    out = np.zeros((n_coarse, nc))
    for K, c in enumerate(cmap):
        if c >= 0:
            out[c] += P3.T @ rb[K]
    return out.reshape(-1)


class Level:
    """One multigrid level: the operator apply, the inner preconditioner D^-1 (callable),
    lam_max of D^-1 A, the degree and the cell indices of its blocks."""

    def __init__(self, apply, minv, lam_max: float, degree: int, ijk: np.ndarray):
        self.apply, self.minv, self.lam_max, self.degree, self.ijk = apply, minv, lam_max, degree, ijk
        self.n = len(ijk) * (degree + 1) ** 3


def vcycle(levels, r, smooth_degree: int, smooth_range: float, coarse_degree: int, coarse_range: float):
    """z = B r, one V-cycle (levels[0] coarsest, levels[-1] finest)."""
    def cycle(li, rl):
        L = levels[li]
        if li == 0:
            return chebyshev(L.apply, L.minv, rl, coarse_degree, L.lam_max, L.lam_max / coarse_range)
        lmin = L.lam_max / smooth_range
        x = chebyshev(L.apply, L.minv, rl, smooth_degree, L.lam_max, lmin)
        res = rl - L.apply(x)
        C = levels[li - 1]
        cmap = block_map(L.ijk, C.ijk)
        xc = cycle(li - 1, restrict(res, C.degree, L.degree, cmap, len(C.ijk)))
        x = x + prolongate(xc, C.degree, L.degree, cmap)
        return chebyshev(L.apply, L.minv, rl, smooth_degree, L.lam_max, lmin, x0=x)
    return cycle(len(levels) - 1, np.asarray(r, dtype=np.float64))


def pcg(apply, b, prec, iters: int, x0=None):
    """Conjugate gradients with the linear preconditioner z = prec(r), a fixed number
    of iterations; returns x and the residual norms |r_k| (k = 0..iters)."""
    x = np.zeros_like(b) if x0 is None else x0.copy()
    r = b - apply(x)
    z = prec(r)
    p = z.copy()
    rz = r @ z
    hist = [float(np.linalg.norm(r))]
    for _ in range(iters):
        q = apply(p)
        alpha = rz / (p @ q)
        x = x + alpha * p
        r = r - alpha * q
        hist.append(float(np.linalg.norm(r)))
        z = prec(r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, np.array(hist)


def jacobi(A):
    """Point Jacobi D^-1 = 1 / diag(A) (``.D``: the matrix D)."""
    dg = A.diagonal()
    dinv = 1.0 / dg

    def minv(r):
        return dinv * r
    minv.D = np.diag(dg)
    return minv


def block_jacobi(A, nd: int):
    """Cell-block Jacobi (additive Schwarz on the cells): D = the n^3 x n^3
    diagonal blocks A_KK, D^-1 r applied through their Cholesky factors (``.D``: D)."""
    Ad = A.tocsr()
    blocks = [Ad[i:i + nd, i:i + nd].toarray() for i in range(0, A.shape[0], nd)]
    facs = [np.linalg.cholesky(B) for B in blocks]

    def minv(r):
        rb = np.asarray(r).reshape(-1, nd)
        out = np.empty_like(rb)
        for K, L in enumerate(facs):
            out[K] = np.linalg.solve(L.T, np.linalg.solve(L, rb[K]))
        return out.reshape(-1)
    D = np.zeros(A.shape)
    for K, B in enumerate(blocks):
        D[K * nd:(K + 1) * nd, K * nd:(K + 1) * nd] = B
    minv.D = D
    return minv


def dense_lambda_max(A, minv) -> float:
    """The largest eigenvalue of D^-1 A: the largest of the generalized symmetric
    problem A x = lam D x (D = ``minv.D``, SPD), dense."""
    import scipy.linalg as sl
    Ad = A.toarray() if hasattr(A, "toarray") else np.asarray(A)
    n = Ad.shape[0]
    return float(sl.eigh(Ad, minv.D, eigvals_only=True, subset_by_index=[n - 1, n - 1])[0])
