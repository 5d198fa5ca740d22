"""1-D tables for the oracle (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

- Nodal basis: Lagrange polynomials on the p+1 Gauss-Lobatto (GLL) nodes of
  [0,1] ("nodal Lagrangian elements defined in the
  Gauss-Lobatto nodes").
- Structured rule: n = p+1 point Gauss-Legendre on [0,1] ("we choose the
  1D number of quadrature points as k = p+1").
Nodes/weights are computed in mpmath at 50 digits and rounded to double
(SURVEY §8(c) step 1).  Basis values/derivatives at arbitrary points use the
product form l_a(x) = prod_{m!=a} (x-x_m)/(x_a-x_m) (never monomials);
derivative traces l_a^(j)(0), l_a^(j)(1) for the ghost penalty are formed in
mpmath and rounded.
"""
from __future__ import annotations

import functools

import mpmath
import numpy as np

_DPS = 50


def _legendre_and_deriv(n, z):
    """P_n(z), P_n'(z) by the three-term recurrence (mpmath scalars)."""
    p0, p1 = mpmath.mpf(1), mpmath.mpf(0)
    for j in range(1, n + 1):
        p0, p1 = ((2 * j - 1) * z * p0 - (j - 1) * p1) / j, p0
    dp = n * (z * p0 - p1) / (z * z - 1)
    return p0, dp


@functools.lru_cache(maxsize=None)
def gauss_mp(n: int):
    """n-point Gauss-Legendre on [0,1] in mpmath: (nodes, weights) ascending."""
    with mpmath.workdps(_DPS):
        xs, ws = [], []
        for i in range(n):
            z = mpmath.cos(mpmath.pi * (i + mpmath.mpf(3) / 4) / (n + mpmath.mpf(1) / 2))
            for _ in range(200):
                pn, dp = _legendre_and_deriv(n, z)
                dz = pn / dp
                z -= dz
                if abs(dz) < mpmath.mpf(10) ** (-_DPS + 5):
                    break
            pn, dp = _legendre_and_deriv(n, z)
            xs.append((z + 1) / 2)
            ws.append(1 / ((1 - z * z) * dp * dp))  # 2/((1-z^2)P'^2) scaled by 1/2
        order = sorted(range(n), key=lambda k: xs[k])
        return [xs[k] for k in order], [ws[k] for k in order]


@functools.lru_cache(maxsize=None)
def gll_mp(p: int):
    """p+1 Gauss-Lobatto nodes on [0,1] in mpmath: 0, roots of P_p'(2x-1), 1."""
    with mpmath.workdps(_DPS):
        if p == 1:
            return [mpmath.mpf(0), mpmath.mpf(1)]
        inner = []
        for i in range(1, p):
            z = -mpmath.cos(mpmath.pi * i / p)  # Chebyshev-Lobatto initial guess
            for _ in range(200):
                # f = P_p'(z); f' = P_p''(z) from the Legendre ODE
                pn, dp = _legendre_and_deriv(p, z)
                d2p = (2 * z * dp - p * (p + 1) * pn) / (1 - z * z)
                dz = dp / d2p
                z -= dz
                if abs(dz) < mpmath.mpf(10) ** (-_DPS + 5):
                    break
            inner.append((z + 1) / 2)
        return [mpmath.mpf(0)] + sorted(inner) + [mpmath.mpf(1)]


@functools.lru_cache(maxsize=None)
def lagrange_deriv_traces_mp(p: int, jmax: int):
    """T[j][side][a] = l_a^(j)(side) for side in {0: xi=0, 1: xi=1}, j = 0..jmax,
    via mpmath polynomial coefficients at 50 digits (rounded to double)."""
    with mpmath.workdps(_DPS):
        x = gll_mp(p)
        n = p + 1
        out = np.zeros((jmax + 1, 2, n))
        for a in range(n):
            # coefficients of l_a (ascending powers) in mp precision
            coef = [mpmath.mpf(1)]
            den = mpmath.mpf(1)
            for m in range(n):
                if m == a:
                    continue
                den *= x[a] - x[m]
                new = [mpmath.mpf(0)] * (len(coef) + 1)
                for k, c in enumerate(coef):
                    new[k] += -x[m] * c
                    new[k + 1] += c
                coef = new
            coef = [c / den for c in coef]
            for j in range(jmax + 1):
                # j-th derivative coefficients
                dcoef = coef[:]
                for _ in range(j):
                    dcoef = [k * dcoef[k] for k in range(1, len(dcoef))] or [mpmath.mpf(0)]
                v0 = dcoef[0] if dcoef else mpmath.mpf(0)
                v1 = mpmath.fsum(dcoef)
                out[j, 0, a] = float(v0)
                out[j, 1, a] = float(v1)
        return out


class Basis1D:
    """Degree-p GLL Lagrange basis on [0,1] with the (p+1)-point Gauss rule."""

    def __init__(self, p: int):
        if not 1 <= p <= 8:
            raise ValueError("degree must be in 1..8")
        self.p = p
        self.n = p + 1
        self.nodes = np.array([float(v) for v in gll_mp(p)])
        gx, gw = gauss_mp(self.n)
        self.gauss_x = np.array([float(v) for v in gx])
        self.gauss_w = np.array([float(v) for v in gw])
        self.traces = lagrange_deriv_traces_mp(p, p)  # [j][side][a]

    def values(self, x):
        """l_a(x) for all a: array (len(x), n), product form."""
        x = np.asarray(x, dtype=np.float64).reshape(-1)
        xn = self.nodes
        out = np.ones((x.size, self.n))
        for a in range(self.n):
            for m in range(self.n):
                if m != a:
                    out[:, a] *= (x - xn[m]) / (xn[a] - xn[m])
        return out

    def derivs(self, x):
        """l_a'(x) = sum_{k!=a} 1/(x_a-x_k) prod_{m!=a,k} (x-x_m)/(x_a-x_m)."""
        x = np.asarray(x, dtype=np.float64).reshape(-1)
        xn = self.nodes
        out = np.zeros((x.size, self.n))
        for a in range(self.n):
            for k in range(self.n):
                if k == a:
                    continue
                term = np.full(x.size, 1.0 / (xn[a] - xn[k]))
                for m in range(self.n):
                    if m != a and m != k:
                        term = term * (x - xn[m]) / (xn[a] - xn[m])
                out[:, a] += term
        return out

    def trace(self, j: int, side: int):
        """l_a^(j)(side) for side in {0,1} (reference derivative)."""
        return self.traces[j, side].copy()
