"""Pins of the oracle's VOLUME ghost penalty (PAPER eq:volume_based_gp P:96-108,
stable-neighbour patches; SPEC ghost_penalty_face_term examples).

* closed form on a 2-cell patch: tau_v h [G (x) M (x) M] with G = int_patch of the
  extended 1-D bases (independent route: tests/pin1d.py barycentric values outside
  [0,1]);
* unit jump: u = 1 on E1, 0 on E2  ->  u^T A u = tau_v / h^2 (|E1| + |E2|) = 2 tau_v h;
* extension exactness: A_P q = 0 for every global polynomial of degree <= p;
* axis-aligned plane: every cut cell picks its uncut lower neighbour (volume fraction
  1), and the GP term equals the 1-D patch matrix (x) full masses;
* SPD and L2 convergence order with tau_v = 1.
"""
import math

import numpy as np
import numpy.polynomial.legendre as npleg
import pytest

import pin1d
from oracle import Oracle
from oracle.operator import TERM_GP
from test_oracle_plane import _perm

FAR = {"type": "sphere", "center": [0.0, 0.0, 0.0], "radius": 10.0}


def vgp_1d(p):
    """G = int_0^2 [l(x); -l(x-1)] [l(x); -l(x-1)]^T dx (E1 coordinates), 2n x 2n."""
    gx, gw = npleg.leggauss(20)
    G = np.zeros((2 * (p + 1), 2 * (p + 1)))
    for lo in (0.0, 1.0):
        x, w = lo + (gx + 1) / 2, gw / 2
        J = np.hstack([pin1d.values(p, x), -pin1d.values(p, x - 1.0)])
        G += J.T @ (w[:, None] * J)
    return G


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_vgp_two_cell_closed_form_and_special_cases(cutgen_mod, p):
    h, tau = 0.25, 0.7
    P = cutgen_mod.generate(FAR, [2, 1, 1], [0, 0, 0], [2 * h, h, h], p, force_cut_cells=True,
                            gp_kind=1, tau_v=tau)
    O = Oracle(P)
    assert O.patches == {(0, 1, 0)}
    (m, pl, d, sf), = O.faces
    A = O.face_matrix(m, pl, d, sf, TERM_GP)
    nn, nd = p + 1, (p + 1) ** 3
    M1, _ = pin1d.mass_stiff(p)
    G = tau * h * vgp_1d(p)
    for si in range(2):
        for sj in range(2):
            ref = np.kron(M1, np.kron(M1, G[si * nn:(si + 1) * nn, sj * nn:(sj + 1) * nn]))
            blk = A[si * nd:(si + 1) * nd, sj * nd:(sj + 1) * nd]
            assert np.abs(blk - ref).max() <= 1e-12 * np.abs(G).max()
    u = np.concatenate([np.ones(nd), np.zeros(nd)])
    assert abs(u @ A @ u - 2 * tau * h) <= 1e-13 * (u @ np.abs(A) @ u)
    nodes = pin1d.nodes(p)
    rng = np.random.default_rng(p)
    c = rng.standard_normal(4)
    q = lambda x, y, z: c[0] + c[1] * x ** p + c[2] * (x * y) ** min(p, 2) + c[3] * z * x ** (p - 1)  # noqa: E731
    vals = []
    for cell in range(2):
        Z, Y, X = np.meshgrid(nodes * h, nodes * h, (nodes + cell) * h, indexing="ij")
        vals.append(q(X, Y, Z).ravel())
    qq = np.concatenate(vals)
    assert np.abs(A @ qq).max() <= 1e-11 * np.abs(A).max() * np.abs(qq).max()


@pytest.mark.parametrize("d", [0, 1, 2])
@pytest.mark.parametrize("p", [1, 2, 3])
def test_vgp_plane_patches_and_kronecker(cutgen_mod, p, d):
    nfull, ncut, h, c, tau = 3, 2, 1.0 / 3.0, 0.45, 1.0
    nrm = [0.0, 0.0, 0.0]
    nrm[d] = 1.0
    P = cutgen_mod.generate({"type": "plane", "normal": nrm, "offset": c}, nfull, 0.0, 1.0, p,
                            gp_kind=1, tau_v=tau)
    O = Oracle(P)
    # every cut cell (layer 1) pairs with its uncut lower neighbour (layer 0) along d
    lookup = {tuple(r): k for k, r in enumerate(P.active_ijk.tolist())}
    want = set()
    for K in np.where(P.is_cut.astype(bool))[0]:
        nb = list(P.active_ijk[K])
        nb[d] -= 1
        want.add((lookup[tuple(nb)], int(K), d))
    assert O.patches == want
    n = p + 1
    M1, _ = pin1d.mass_stiff(p)
    Gd = np.zeros((ncut * n, ncut * n))
    Gd[:2 * n, :2 * n] = (tau / h) * vgp_1d(p)  # layers 0, 1
    Me = np.kron(np.eye(nfull), h * M1)
    f = [Me, Me, Me]
    f[d] = Gd
    R = np.kron(f[0], np.kron(f[1], f[2]))
    perm = _perm(P, d, ncut, nfull)
    R = R[np.ix_(perm, perm)]
    M = Oracle(P, term_mask=TERM_GP).assemble_csr().toarray()
    assert np.abs(M - R).max() <= 1e-12 * np.abs(R).max()


def test_vgp_spd(cutgen_mod):
    P = cutgen_mod.generate(cutgen_mod.SPHERE, 6, -1.0, 1.0, 2, gp_kind=1, tau_v=1.0)
    D = Oracle(P).assemble_csr().toarray()
    assert np.abs(D - D.T).max() <= 1e-13 * np.abs(D).max()
    np.linalg.cholesky(D)


def _solve(cutgen_mod, N, p):
    import scipy.sparse.linalg as spl
    R, om = 0.7, math.pi
    c = np.array(cutgen_mod.SPHERE["center"])
    P = cutgen_mod.generate(cutgen_mod.SPHERE, N, -1.0, 1.0, p, gp_kind=1, tau_v=1.0)
    O = Oracle(P)
    A = O.assemble_csr()
    rr = lambda x: np.linalg.norm(x - c, axis=-1)  # noqa: E731
    f = lambda x: -om ** 2 * (np.cos(om * rr(x)) + 2 * np.sinc(om * rr(x) / math.pi))  # noqa: E731
    uex = lambda x: math.cos(om * R) - np.cos(om * rr(x))  # noqa: E731
    x = spl.spsolve(A.tocsc(), O.rhs(f))
    return O.l2_error(x, uex)


@pytest.mark.parametrize("p,meshes", [(1, (8, 16)), (2, (8, 12))])
def test_vgp_convergence_order(cutgen_mod, p, meshes):
    """DG with the volume ghost penalty (tau_v = 1): L2 EOC >= p + 0.7."""
    e1, e2 = (_solve(cutgen_mod, N, p) for N in meshes)
    assert math.log(e1 / e2) / math.log(meshes[1] / meshes[0]) >= p + 0.7, (e1, e2)
