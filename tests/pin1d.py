"""Independent 1-D route for the oracle pins (TEST HELPER, not the oracle).

Everything here is computed by a different algorithm than oracle/basis.py:

* GLL nodes: mpmath.polyroots of the explicit coefficients of P_p'
  (P_p(x) = 2^-p sum_k (-1)^k C(p,k) C(2p-2k,p) x^(p-2k)); the oracle runs Newton
  on the three-term recurrence.
* derivative traces l_a^(j)(0), l_a^(j)(1): rows 0 / p of D^j, D the barycentric
  nodal differentiation matrix in mpmath (exact because the end points are
  nodes); the oracle differentiates monomial coefficients.
* values at arbitrary points: the barycentric formula (second form); derivatives
  as L(x) @ D (the derivative of a degree-p polynomial interpolated at the
  nodes); the oracle uses product forms.
* integrals over [0, s]: numpy's Gauss-Legendre with 30 points (exact for the
  degree <= 16 integrands here).
"""
from __future__ import annotations

import functools

import mpmath
import numpy as np
import numpy.polynomial.legendre as npleg

_DPS = 40


@functools.lru_cache(maxsize=None)
def gll_mp(p: int):
    with mpmath.workdps(_DPS):
        if p == 1:
            return (mpmath.mpf(0), mpmath.mpf(1))
        # coefficients of P_p, ascending
        c = [mpmath.mpf(0)] * (p + 1)
        for k in range(p // 2 + 1):
            c[p - 2 * k] = (-1) ** k * mpmath.binomial(p, k) * mpmath.binomial(2 * p - 2 * k, p) / mpmath.mpf(2) ** p
        dc = [k * c[k] for k in range(1, p + 1)]  # P_p', ascending
        roots = mpmath.polyroots(dc[::-1], maxsteps=400, extraprec=400)
        inner = sorted((mpmath.re(r) + 1) / 2 for r in roots)
        return tuple([mpmath.mpf(0)] + inner + [mpmath.mpf(1)])


@functools.lru_cache(maxsize=None)
def bary_weights_mp(p: int):
    x = gll_mp(p)
    with mpmath.workdps(_DPS):
        return tuple(1 / mpmath.fprod(x[a] - x[m] for m in range(p + 1) if m != a) for a in range(p + 1))


@functools.lru_cache(maxsize=None)
def diff_matrix_mp(p: int):
    x, w = gll_mp(p), bary_weights_mp(p)
    n = p + 1
    with mpmath.workdps(_DPS):
        D = mpmath.zeros(n, n)
        for i in range(n):
            for j in range(n):
                if i != j:
                    D[i, j] = (w[j] / w[i]) / (x[i] - x[j])
            D[i, i] = -mpmath.fsum(D[i, j] for j in range(n) if j != i)
        return D


def nodes(p: int) -> np.ndarray:
    return np.array([float(v) for v in gll_mp(p)])


def diff_matrix(p: int) -> np.ndarray:
    D = diff_matrix_mp(p)
    return np.array([[float(D[i, j]) for j in range(p + 1)] for i in range(p + 1)])


@functools.lru_cache(maxsize=None)
def _traces(p: int):
    D = diff_matrix_mp(p)
    n = p + 1
    out = np.zeros((p + 1, 2, n))
    with mpmath.workdps(_DPS):
        Dj = mpmath.eye(n)
        for j in range(p + 1):
            for a in range(n):
                out[j, 0, a] = float(Dj[0, a])
                out[j, 1, a] = float(Dj[p, a])
            Dj = Dj * D
    return out


def trace(p: int, j: int, side: int) -> np.ndarray:
    """l_a^(j)(side), side 0 -> xi = 0, 1 -> xi = 1 (reference derivatives)."""
    return _traces(p)[j, side].copy()


def values(p: int, x) -> np.ndarray:
    """l_a(x) for all a (barycentric, second form): (len(x), p+1)."""
    xn = nodes(p)
    w = np.array([float(v) for v in bary_weights_mp(p)])
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    out = np.zeros((x.size, p + 1))
    for q, xq in enumerate(x):
        hit = np.where(xq == xn)[0]
        if hit.size:
            out[q, hit[0]] = 1.0
            continue
        t = w / (xq - xn)
        out[q] = t / t.sum()
    return out


def derivs(p: int, x) -> np.ndarray:
    return values(p, x) @ diff_matrix(p)


def mass_stiff(p: int, s: float = 1.0):
    """M[a,b] = int_0^s l_a l_b, K[a,b] = int_0^s l_a' l_b' (reference)."""
    gx, gw = npleg.leggauss(30)
    x, w = s * (gx + 1) / 2, s * gw / 2
    L, D = values(p, x), derivs(p, x)
    return L.T @ (w[:, None] * L), D.T @ (w[:, None] * D)
