"""Oracle pins Q5 (axis-aligned plane, semi-analytic) and Q10 (tensor rule fed as a
cut rule), SURVEY §8(c).  -m "not gpu".

Q5.  Omega = {x_d < c} on a box of cubic cells, c inside cell layer L of axis d
(reference coordinate s = (c - x_L)/h in (0,1)).  Every quadrature rule is then a
tensor rule ([0,s] in d, [0,1] in the others) that integrates its integrand
exactly, so the operator is a SUM OF KRONECKER PRODUCTS of 1-D matrices, built here
from the independent 1-D route of tests/pin1d.py:

  cut axis d (layers 0..L):   M_d = blockdiag(h M1, .., h M(s)),  K_d = blockdiag(K1/h, .., K(s)/h)
                              + 1-D SIPG at the interior points (all inside Omega)
                              + 1-D Nitsche at x = c (normal +e_d; PAPER eq:bilinear_cg P:72-76)
                              + 1-D face ghost penalty between layers L-1 and L
  full axes e (cells 0..N-1): M_e = blockdiag(h M1), K_e = blockdiag(K1/h) + 1-D SIPG,
                              G_e = 1-D ghost penalty at every interior point
  A = sum_e K_e (x) M_others             (volume + SIPG + Nitsche + GP of the cut axis)
    + sum_{e != d} G_e (x) E_L (x) M_e'   (ghost penalty on the faces inside layer L,
                                          full-face rule: E_L = the full mass of layer L only)

The SIPG on the faces of axis e != d inside layer L runs over F cap Omega =
[0,s] x [0,1] (eq:unstructured_face): its d-factor is the
TRUNCATED mass inside M_d.  With d = 0 the truncated coordinate is the face's s
(lower in-face axis) for y- and z-faces; with d = 2 it is t for x- and y-faces;
with d = 1 it is t on x-faces and s on z-faces -- so a swapped (s,t) mapping of the
cut-face points fails this pin.  Q10: the oracle with every cell and face forced
through the unstructured arrays (tensor rules as "cut" rules, full faces listed as
cut faces; PAPER P:850's unstructured-with-structured-quadrature benchmark) equals
the oracle on the structured problem.
"""
import numpy as np
import pytest

import pin1d
from oracle import Oracle
from oracle.operator import TERM_CELL, TERM_GP, TERM_NITSCHE, TERM_SIPG

FAR = {"type": "sphere", "center": [0.0, 0.0, 0.0], "radius": 10.0}


def _sipg_pt(p, h, gamma):
    """1-D SIPG at an interior point on [v^-; v^+] x [u^-; u^+]."""
    J = np.concatenate([pin1d.trace(p, 0, 1), -pin1d.trace(p, 0, 0)])
    Av = 0.5 * np.concatenate([pin1d.trace(p, 1, 1), pin1d.trace(p, 1, 0)]) / h
    sigma = gamma / h
    return sigma * np.outer(J, J) - np.outer(Av, J) - np.outer(J, Av)


def _gp_pt(p, h, gpg):
    """1-D face ghost penalty: sum_j g_j h^(2j-1) D_j D_j^T, D_j physical jumps."""
    G = np.zeros((2 * (p + 1), 2 * (p + 1)))
    for j in range(p + 1):
        D = np.concatenate([pin1d.trace(p, j, 1), -pin1d.trace(p, j, 0)]) * h ** (-j)
        G += gpg[j] * h ** (2 * j - 1) * np.outer(D, D)
    return G


def _place(A, blk, i):
    n = blk.shape[0] // 2
    A[i * n:(i + 2) * n, i * n:(i + 2) * n] += blk


def plane_parts(p, d, h, ncut, s, nfull, gamma, tau, gpg):
    """The plane operator split by term, each a sum of Kronecker products of 1-D
    factors (tensor index: X slowest, Z fastest)."""
    n = p + 1
    M1, K1 = pin1d.mass_stiff(p)
    Ms, Ks = pin1d.mass_stiff(p, s)
    L = ncut - 1  # cut layer
    # cut axis d: layer masses (truncated in layer L), volume + SIPG, Nitsche, GP
    Md = np.zeros((ncut * n, ncut * n))
    Kd = np.zeros_like(Md)
    Nd = np.zeros_like(Md)
    Gd = np.zeros_like(Md)
    EL = np.zeros_like(Md)
    for i in range(ncut):
        sl = slice(i * n, (i + 1) * n)
        Md[sl, sl] = h * (Ms if i == L else M1)
        Kd[sl, sl] = (Ks if i == L else K1) / h
    EL[L * n:, L * n:] = h * M1
    for i in range(ncut - 1):
        _place(Kd, _sipg_pt(p, h, gamma), i)
    phi = pin1d.values(p, [s])[0]
    dphi = pin1d.derivs(p, [s])[0] / h  # n = +e_d
    Nd[L * n:, L * n:] = tau / h * np.outer(phi, phi) - np.outer(dphi, phi) - np.outer(phi, dphi)
    if ncut >= 2:
        _place(Gd, _gp_pt(p, h, gpg), L - 1)
    # full axes
    Me = np.kron(np.eye(nfull), h * M1)
    Ke = np.kron(np.eye(nfull), K1 / h)
    Ge = np.zeros_like(Ke)
    for i in range(nfull - 1):
        _place(Ke, _sipg_pt(p, h, gamma), i)
        _place(Ge, _gp_pt(p, h, gpg), i)

    def kron3(f):
        return np.kron(f[0], np.kron(f[1], f[2]))

    def along(e, fe, fd=None):
        f = [Me, Me, Me]
        f[d] = Md if fd is None else fd
        f[e] = fe
        return kron3(f)

    parts = {"cell_sipg": 0, "nitsche": along(d, Nd), "gp": along(d, Gd)}
    for e in range(3):
        parts["cell_sipg"] = parts["cell_sipg"] + along(e, Kd if e == d else Ke)
        if e != d:
            parts["gp"] = parts["gp"] + along(e, Ge, fd=EL)
    return parts


def plane_operator(p, d, h, ncut, s, nfull, gamma, tau, gpg):
    parts = plane_parts(p, d, h, ncut, s, nfull, gamma, tau, gpg)
    return parts["cell_sipg"] + parts["nitsche"] + parts["gp"]


def _perm(P, d, ncut, nfull):
    """oracle DoF index -> tensor index of plane_operator."""
    n = P.degree + 1
    cnt = [nfull, nfull, nfull]
    cnt[d] = ncut
    perm = np.zeros(P.n_dofs, dtype=np.int64)
    for K, (i, j, k) in enumerate(P.active_ijk.tolist()):
        for c in range(n):
            for b in range(n):
                for a in range(n):
                    X, Y, Z = i * n + a, j * n + b, k * n + c
                    perm[K * n ** 3 + a + n * b + n * n * c] = (X * cnt[1] * n + Y) * cnt[2] * n + Z
    return perm


@pytest.mark.parametrize("d", [0, 1, 2])
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_q5_axis_aligned_plane(cutgen_mod, p, d):
    nfull, ncut, h = 3, 2, 1.0 / 3.0
    c = 0.45  # in layer 1: s = (0.45 - 1/3) * 3 = 0.35
    s = (c - (ncut - 1) * h) / h
    nrm = [0.0, 0.0, 0.0]
    nrm[d] = 1.0
    P = cutgen_mod.generate({"type": "plane", "normal": nrm, "offset": c}, nfull, 0.0, 1.0, p)
    assert P.n_active == ncut * nfull * nfull and P.n_cut == nfull * nfull
    assert P.sf_cells.shape[0] == 2 * nfull * (nfull - 1)  # the in-layer faces of the two other axes
    # the faces' truncated coordinate really is s resp. t where the docstring says
    for f in range(P.sf_cells.shape[0]):
        ax = int(P.sf_axis[f])
        inface = [a for a in range(3) if a != ax]
        pts = P.sf_pts[P.sf_ptr[f]:P.sf_ptr[f + 1]]
        col = inface.index(d)
        assert pts[:, col].max() < s and abs(pts[:, 2].sum() - s * h * h) < 1e-14
    A = plane_operator(p, d, h, ncut, s, nfull, P.sipg_gamma, P.nitsche_tau, P.gp_gamma)
    perm = _perm(P, d, ncut, nfull)
    R = A[np.ix_(perm, perm)]
    O = Oracle(P)
    M = O.assemble_csr().toarray()
    assert np.abs(M - R).max() <= 1e-12 * np.abs(R).max(), np.abs(M - R).max() / np.abs(R).max()
    # term by term: a wrong sign / dropped term in one term cannot hide in another
    parts = plane_parts(p, d, h, ncut, s, nfull, P.sipg_gamma, P.nitsche_tau, P.gp_gamma)
    for mask, key in ((TERM_CELL | TERM_SIPG, "cell_sipg"), (TERM_NITSCHE, "nitsche"), (TERM_GP, "gp")):
        Mm = Oracle(P, term_mask=mask).assemble_csr().toarray()
        Rm = parts[key][np.ix_(perm, perm)]
        assert np.abs(Mm - Rm).max() <= 1e-12 * np.abs(R).max(), (key, np.abs(Mm - Rm).max())


def test_q5_swapped_face_coordinates_are_caught(cutgen_mod):
    """Fault injection: swapping (s,t) of the cut-face points changes the operator."""
    p, d, nfull, ncut, h, c = 2, 0, 3, 2, 1.0 / 3.0, 0.45
    P = cutgen_mod.generate({"type": "plane", "normal": [1, 0, 0], "offset": c}, nfull, 0.0, 1.0, p)
    s = (c - (ncut - 1) * h) / h
    R = plane_operator(p, d, h, ncut, s, nfull, P.sipg_gamma, P.nitsche_tau, P.gp_gamma)
    perm = _perm(P, d, ncut, nfull)
    R = R[np.ix_(perm, perm)]
    P.sf_pts = P.sf_pts.copy()
    P.sf_pts[:, [0, 1]] = P.sf_pts[:, [1, 0]]
    M = Oracle(P).assemble_csr().toarray()
    assert np.abs(M - R).max() > 1e-3 * np.abs(R).max()


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_q10_oracle_tensor_rule_as_cut_rule(cutgen_mod, p):
    """The oracle fed every cell's tensor rule as its cut rule (and every full face
    as a listed cut face) equals the oracle on the structured problem (masks 1|2|4;
    the ghost penalty differs because every cell then counts as cut)."""
    Ps = cutgen_mod.generate(FAR, 3, -1.0, 1.0, p)
    Pu = cutgen_mod.generate(FAR, 3, -1.0, 1.0, p, force_cut_cells=True, force_cut_faces=True)
    assert Pu.n_cut == Pu.n_active and Pu.sf_cells.shape[0] == 3 * 3 * 3 * 2
    m = TERM_CELL | TERM_SIPG | TERM_NITSCHE
    As = Oracle(Ps, term_mask=m).assemble_csr()
    Au = Oracle(Pu, term_mask=m).assemble_csr()
    assert abs(As - Au).max() <= 1e-12 * abs(As).max()
    # and the GP of the forced problem is the GP on every interior face (Q3 per face)
    Ag = Oracle(Pu, term_mask=TERM_GP).assemble_csr()
    u = np.ones(Pu.n_dofs)
    assert np.abs(Ag @ u).max() <= 1e-12 * abs(Ag).max()
