"""Pins of the H^1 (continuous Galerkin) oracle, oracle/h1.py.

* level set misses the mesh: the standard continuous Q_p Laplacian of the box =
  Kronecker sum of continuity-assembled 1-D stiffness / mass (independent 1-D route,
  tests/pin1d.py); A 1 = 0;
* axis-aligned plane: every term (volume, Nitsche, GP) = sum of Kronecker products
  of continuity-assembled 1-D factors (truncated in the cut layer);
* continuity: P^T A_DG P with the SIPG terms INCLUDED equals A_CG (every SIPG term
  carries a jump, which vanishes for continuous fields) -- fails for a wrong numbering;
* symmetry, SPD; convergence order of the solve on the manufactured solution.
"""
import math

import numpy as np
import pytest

import pin1d
from oracle import Oracle
from oracle.h1 import OracleH1, h1_numbering
from oracle.operator import TERM_ALL, TERM_CELL, TERM_GP, TERM_NITSCHE
from test_oracle_plane import _gp_pt, _place

FAR = {"type": "sphere", "center": [0.0, 0.0, 0.0], "radius": 10.0}


def _p1(ncell, p):
    """1-D continuity gather: (ncell*(p+1)) x (ncell*p+1)."""
    G = np.zeros((ncell * (p + 1), ncell * p + 1))
    for i in range(ncell):
        for a in range(p + 1):
            G[i * (p + 1) + a, i * p + a] = 1.0
    return G


def _kron3(f):
    return np.kron(f[0], np.kron(f[1], f[2]))


@pytest.mark.parametrize("p,N", [(1, 3), (2, 3), (3, 2), (4, 2)])
def test_h1_level_set_misses_mesh(cutgen_mod, p, N):
    P = cutgen_mod.generate(FAR, N, -1.0, 1.0, p)
    O = OracleH1(P)
    assert O.n_h1 == (N * p + 1) ** 3
    M = O.assemble_csr().toarray()
    h = P.h
    M1, K1 = pin1d.mass_stiff(p)
    G = _p1(N, p)
    Mc = G.T @ np.kron(np.eye(N), h * M1) @ G
    Kc = G.T @ np.kron(np.eye(N), K1 / h) @ G
    ref = _kron3([Kc, Mc, Mc]) + _kron3([Mc, Kc, Mc]) + _kron3([Mc, Mc, Kc])
    assert np.abs(M - ref).max() <= 1e-12 * np.abs(ref).max()
    assert np.abs(M @ np.ones(M.shape[0])).max() <= 1e-12 * np.abs(M).max()


def _plane_h1_parts(p, d, h, ncut, s, nfull, tau, gpg):
    n = p + 1
    M1, K1 = pin1d.mass_stiff(p)
    Ms, Ks = pin1d.mass_stiff(p, s)
    L = ncut - 1
    Md = np.zeros((ncut * n, ncut * n))
    Kd, Nd, Gd, EL = (np.zeros_like(Md) for _ in range(4))
    for i in range(ncut):
        sl = slice(i * n, (i + 1) * n)
        Md[sl, sl] = h * (Ms if i == L else M1)
        Kd[sl, sl] = (Ks if i == L else K1) / h
    EL[L * n:, L * n:] = h * M1
    phi = pin1d.values(p, [s])[0]
    dphi = pin1d.derivs(p, [s])[0] / h
    Nd[L * n:, L * n:] = tau / h * np.outer(phi, phi) - np.outer(dphi, phi) - np.outer(phi, dphi)
    if ncut >= 2:
        _place(Gd, _gp_pt(p, h, gpg), L - 1)
    Me = np.kron(np.eye(nfull), h * M1)
    Ke = np.kron(np.eye(nfull), K1 / h)
    Ge = np.zeros_like(Ke)
    for i in range(nfull - 1):
        _place(Ge, _gp_pt(p, h, gpg), i)
    Gc, Gf = _p1(ncut, p), _p1(nfull, p)
    c = lambda A, G: G.T @ A @ G  # noqa: E731

    def along(e, fe, fd):
        f = [c(Me, Gf)] * 3
        f = list(f)
        f[d] = c(fd, Gc)
        f[e] = c(fe, Gc if e == d else Gf)
        return _kron3(f)

    parts = {"cell": 0, "nitsche": along(d, Nd, Md), "gp": along(d, Gd, Md)}
    for e in range(3):
        parts["cell"] = parts["cell"] + along(e, Kd if e == d else Ke, Md)
        if e != d:
            parts["gp"] = parts["gp"] + along(e, Ge, EL)
    return parts


@pytest.mark.parametrize("d", [0, 1, 2])
@pytest.mark.parametrize("p", [1, 2, 3])
def test_h1_axis_aligned_plane(cutgen_mod, p, d):
    nfull, ncut, h, c = 3, 2, 1.0 / 3.0, 0.45
    s = (c - (ncut - 1) * h) / h
    nrm = [0.0, 0.0, 0.0]
    nrm[d] = 1.0
    P = cutgen_mod.generate({"type": "plane", "normal": nrm, "offset": c}, nfull, 0.0, 1.0, p)
    cnt = [nfull * p + 1] * 3
    cnt[d] = ncut * p + 1
    n_h1, _ = h1_numbering(P)
    assert n_h1 == cnt[0] * cnt[1] * cnt[2]  # the active lattice is a full box: numbering = Kronecker order
    parts = _plane_h1_parts(p, d, h, ncut, s, nfull, P.nitsche_tau, P.gp_gamma)
    R = parts["cell"] + parts["nitsche"] + parts["gp"]
    M = OracleH1(P).assemble_csr().toarray()
    assert np.abs(M - R).max() <= 1e-12 * np.abs(R).max()
    for mask, key in ((TERM_CELL, "cell"), (TERM_NITSCHE, "nitsche"), (TERM_GP, "gp")):
        Mm = OracleH1(P, term_mask=mask).assemble_csr().toarray()
        assert np.abs(Mm - parts[key]).max() <= 1e-12 * np.abs(R).max(), key


@pytest.mark.parametrize("p", [1, 2, 3])
def test_h1_continuity_kills_sipg_and_spd(cutgen_mod, p):
    P = cutgen_mod.generate(cutgen_mod.SPHERE, 6, -1.0, 1.0, p)
    O = OracleH1(P)
    A = O.assemble_csr()
    G = O.gather_matrix()
    Aall = (G.T @ Oracle(P, term_mask=TERM_ALL).assemble_csr() @ G).toarray()
    D = A.toarray()
    assert np.abs(Aall - D).max() <= 1e-11 * np.abs(D).max()
    assert np.abs(D - D.T).max() <= 1e-13 * np.abs(D).max()
    np.linalg.cholesky(D)
    u = np.random.default_rng(1).uniform(-1, 1, O.n_h1)
    assert np.abs(O.apply(u) - A @ u).max() <= 1e-13 * np.abs(A @ u).max()
    # a wrong numbering (two nodes of an interior cell swapped) makes the gathered field
    # discontinuous: the SIPG terms no longer vanish
    bad = OracleH1(P)
    bad.map = bad.map.copy()
    K = int(np.argmin(np.abs(P.active_ijk - 2.5).sum(1)))  # an interior cell: every face shared
    bad.map[K, [0, 1]] = bad.map[K, [1, 0]]
    Gb = bad.gather_matrix()
    Ab = (Gb.T @ Oracle(P, term_mask=TERM_ALL).assemble_csr() @ Gb).toarray()
    Ab2 = (Gb.T @ Oracle(P, term_mask=bad.dg.mask).assemble_csr() @ Gb).toarray()
    assert np.abs(Ab - Ab2).max() > 1e-6 * np.abs(D).max()


def _solve_h1(cutgen_mod, N, p):
    R, om = 0.7, math.pi
    c = np.array(cutgen_mod.SPHERE["center"])
    P = cutgen_mod.generate(cutgen_mod.SPHERE, N, -1.0, 1.0, p)
    O = OracleH1(P)
    A = O.assemble_csr()
    rr = lambda x: np.linalg.norm(x - c, axis=-1)  # noqa: E731
    f = lambda x: -om ** 2 * (np.cos(om * rr(x)) + 2 * np.sinc(om * rr(x) / math.pi))  # noqa: E731
    uex = lambda x: math.cos(om * R) - np.cos(om * rr(x))  # noqa: E731
    b = O.rhs(f)
    import scipy.sparse.linalg as spl
    x = spl.spsolve(A.tocsc(), b)
    assert np.linalg.norm(A @ x - b) <= 1e-8 * np.linalg.norm(b)
    return O.l2_error(x, uex)


@pytest.mark.parametrize("p,meshes", [(1, (8, 16, 32)), (2, (8, 16)), (3, (6, 8))])
def test_h1_convergence_order(cutgen_mod, p, meshes):
    """CG (H^1) solve of the manufactured problem: L2 EOC >= p + 0.7 (slope p+1)."""
    errs = [_solve_h1(cutgen_mod, N, p) for N in meshes]
    for k in range(len(meshes) - 1):
        rate = math.log(errs[k] / errs[k + 1]) / math.log(meshes[k + 1] / meshes[k])
        assert rate >= p + 0.7, (p, meshes, errs, rate)
