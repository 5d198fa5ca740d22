"""Pins of the CPU oracle against what the paper and the mathematics fix.

Every pin here computes its expected value by a route independent of oracle/:
numpy's Legendre routines (GLL nodes as roots of P_p', high-order Gauss rules),
textbook closed forms, exact identities for global polynomials, invariants, and
the paper's printed convergence data (tests/golden/).
"""
import math

import numpy as np
import numpy.polynomial.legendre as npleg
import pytest
from numpy.polynomial import Polynomial

import pin1d
from oracle import Oracle
from oracle.operator import TERM_CELL, TERM_GP, TERM_NITSCHE, TERM_SIPG, cg

FAR = {"type": "sphere", "center": [0.0, 0.0, 0.0], "radius": 10.0}


# ------------------------------------------------------- independent 1-D route
def gll_np(p):
    """GLL nodes on [0,1] from numpy: 0, roots of P_p', 1."""
    if p == 1:
        return np.array([0.0, 1.0])
    r = np.sort(npleg.Legendre.basis(p).deriv().roots().real)
    return np.concatenate([[0.0], (r + 1) / 2, [1.0]])


def lag_np(x, nodes):
    x = np.atleast_1d(x)
    out = np.ones((x.size, nodes.size))
    for a in range(nodes.size):
        for m in range(nodes.size):
            if m != a:
                out[:, a] *= (x - nodes[m]) / (nodes[a] - nodes[m])
    return out


def dlag_np(x, nodes, eps=None):
    """Derivative via the polynomial class (independent of oracle's product-rule sum)."""
    x = np.atleast_1d(x)
    out = np.zeros((x.size, nodes.size))
    for a in range(nodes.size):
        others = np.delete(nodes, a)
        poly = Polynomial.fromroots(others) / np.prod(nodes[a] - others)
        out[:, a] = poly.deriv()(x)
    return out


def mass_stiff_np(p):
    nodes = gll_np(p)
    gx, gw = npleg.leggauss(30)
    x, w = (gx + 1) / 2, gw / 2
    L, D = lag_np(x, nodes), dlag_np(x, nodes)
    return L.T @ (w[:, None] * L), D.T @ (w[:, None] * D)


def traces_np(p, j, side):
    nodes = gll_np(p)
    out = np.zeros(p + 1)
    for a in range(p + 1):
        others = np.delete(nodes, a)
        poly = Polynomial.fromroots(others) / np.prod(nodes[a] - others)
        out[a] = poly.deriv(j)(float(side)) if j else poly(float(side))
    return out


def far_problem(cutgen_mod, N, p, **kw):
    return cutgen_mod.generate(FAR, N, -1.0, 1.0, p, **kw)


# --------------------------------------------------------------------- Q1
def test_q1_textbook_p1_p2():
    M1, K1 = mass_stiff_np(1)
    assert np.allclose(M1, [[1 / 3, 1 / 6], [1 / 6, 1 / 3]], atol=1e-15)
    assert np.allclose(K1, [[1, -1], [-1, 1]], atol=1e-14)
    M2, K2 = mass_stiff_np(2)
    assert np.allclose(M2, np.array([[4, 2, -1], [2, 16, 2], [-1, 2, 4]]) / 30, atol=1e-15)
    assert np.allclose(K2, np.array([[7, -8, 1], [-8, 16, -8], [1, -8, 7]]) / 3, atol=1e-13)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_q1_uncut_cell_matrix_is_kronecker_sum(cutgen_mod, p):
    P = far_problem(cutgen_mod, 2, p)
    O = Oracle(P)
    A = O.cell_matrix(0, TERM_CELL)
    M1, K1 = mass_stiff_np(p)
    h = P.h
    ref = h * (np.kron(M1, np.kron(M1, K1)) + np.kron(M1, np.kron(K1, M1)) + np.kron(K1, np.kron(M1, M1)))
    assert np.abs(A - ref).max() <= 1e-12 * np.abs(ref).max()
    assert abs(M1.sum() - 1.0) < 1e-13


# --------------------------------------------------------------------- Q2
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("d", [0, 1, 2])
def test_q2_uncut_face_matrix_closed_form(cutgen_mod, p, d):
    n = [1, 1, 1]
    n[d] = 2
    h = 0.5
    P = cutgen_mod.generate(FAR, n, [0, 0, 0], [h * v for v in n], p)
    O = Oracle(P)
    (m, pl, dd, sf), = O.faces
    assert dd == d and sf == -1
    A = O.face_matrix(m, pl, d, sf, TERM_SIPG)
    # independent 1-D route (tests/pin1d.py: barycentric D, mpmath GLL roots)
    M1, _ = pin1d.mass_stiff(p)
    sigma = P.sipg_gamma / h
    J = np.concatenate([pin1d.trace(p, 0, 1), -pin1d.trace(p, 0, 0)])
    Av = 0.5 * np.concatenate([pin1d.trace(p, 1, 1), pin1d.trace(p, 1, 0)]) / h
    if p <= 4:  # a second route (numpy polynomials) for the traces where it is well conditioned
        assert np.allclose(J, np.concatenate([traces_np(p, 0, 1), -traces_np(p, 0, 0)]), atol=1e-13)
        assert np.allclose(Av * h, 0.5 * np.concatenate([traces_np(p, 1, 1), traces_np(p, 1, 0)]), atol=1e-11)
    S = sigma * np.outer(J, J) - np.outer(Av, J) - np.outer(J, Av)
    nn = p + 1
    for si in range(2):
        for sj in range(2):
            Sij = S[si * nn:(si + 1) * nn, sj * nn:(sj + 1) * nn]
            mats = [M1, M1, M1]
            mats[d] = Sij
            ref = h * h * np.kron(mats[2], np.kron(mats[1], mats[0]))
            blk = A[si * nn ** 3:(si + 1) * nn ** 3, sj * nn ** 3:(sj + 1) * nn ** 3]
            assert np.abs(blk - ref).max() <= 1e-12 * np.abs(S).max() * h * h


# --------------------------------------------------------------------- Q3
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_q3_gp_closed_form_and_special_cases(cutgen_mod, p):
    h = 0.25
    P = cutgen_mod.generate(FAR, [2, 1, 1], [0, 0, 0], [2 * h, h, h], p, force_cut_cells=True)
    O = Oracle(P)
    (m, pl, d, sf), = O.faces
    A = O.face_matrix(m, pl, d, sf, TERM_GP)
    nn, nd = p + 1, (p + 1) ** 3
    # u = 1 on K-, 0 on K+: only j = 0 survives -> 0.1 h * |F|/h^2 ... = 0.1 h
    u = np.concatenate([np.ones(nd), np.zeros(nd)])
    assert abs(u @ A @ u - 0.1 * h) <= 1e-14 * (u @ np.abs(A) @ u)
    # closed form [sum_j 0.1 h D_j D_j^T] (x) (M (x) M), checked order by order
    # (j-th term alone via a GP weight vector e_j: the high orders cannot mask a
    # wrong low-order trace), traces from the independent D^j route (pin1d)
    M1, _ = pin1d.mass_stiff(p)
    G = np.zeros((2 * nn, 2 * nn))
    for j in range(p + 1):
        Dj = np.concatenate([pin1d.trace(p, j, 1), -pin1d.trace(p, j, 0)])
        Gj = 0.1 * h * np.outer(Dj, Dj)
        G += Gj
        gj = np.zeros(p + 1)
        gj[j] = 0.1
        Pj = cutgen_mod.generate(FAR, [2, 1, 1], [0, 0, 0], [2 * h, h, h], p, force_cut_cells=True, gp_gamma=gj)
        Oj = Oracle(Pj)
        Aj = Oj.face_matrix(m, pl, d, sf, TERM_GP)
        for si in range(2):
            for sj in range(2):
                ref = np.kron(M1, np.kron(M1, Gj[si * nn:(si + 1) * nn, sj * nn:(sj + 1) * nn]))
                blk = Aj[si * nd:(si + 1) * nd, sj * nd:(sj + 1) * nd]
                assert np.abs(blk - ref).max() <= 1e-11 * np.abs(Gj).max(), (j, np.abs(blk - ref).max())
    for si in range(2):
        for sj in range(2):
            ref = np.kron(M1, np.kron(M1, G[si * nn:(si + 1) * nn, sj * nn:(sj + 1) * nn]))
            blk = A[si * nd:(si + 1) * nd, sj * nd:(sj + 1) * nd]
            assert np.abs(blk - ref).max() <= 1e-11 * np.abs(G).max()
    # A_GP q = 0 for a global polynomial of degree <= p per direction
    nodes = gll_np(p)
    rng = np.random.default_rng(0)
    c = rng.standard_normal(4)
    q = lambda x, y, z: c[0] + c[1] * x ** p + c[2] * (x * y) ** min(p, 2) + c[3] * z * x ** (p - 1)
    vals = []
    for cell in range(2):
        Z, Y, X = np.meshgrid(nodes * h, nodes * h, (nodes + cell) * h, indexing="ij")
        vals.append(q(X, Y, Z).ravel())
    r = A @ np.concatenate(vals)
    assert np.abs(r).max() <= 1e-10 * np.abs(A).max() * np.abs(np.concatenate(vals)).max()


# --------------------------------------------------------------------- Q4
def sipg_1d(N, p, h, gamma):
    """Standard 1-D SIPG (natural BC) on N cells, independent construction."""
    nn = p + 1
    M1, K1 = mass_stiff_np(p)
    A = np.zeros((N * nn, N * nn))
    Mh = np.zeros_like(A)
    for i in range(N):
        A[i * nn:(i + 1) * nn, i * nn:(i + 1) * nn] += K1 / h
        Mh[i * nn:(i + 1) * nn, i * nn:(i + 1) * nn] = h * M1
    sigma = gamma / h
    J = np.concatenate([traces_np(p, 0, 1), -traces_np(p, 0, 0)])
    Av = 0.5 * np.concatenate([traces_np(p, 1, 1), traces_np(p, 1, 0)]) / h
    S = sigma * np.outer(J, J) - np.outer(Av, J) - np.outer(J, Av)
    for i in range(N - 1):
        A[i * nn:(i + 2) * nn, i * nn:(i + 2) * nn] += S
    return A, Mh


@pytest.mark.parametrize("p,N", [(1, 3), (2, 3), (3, 2), (4, 2)])
def test_q4_level_set_misses_mesh_equals_standard_sipg(cutgen_mod, p, N):
    P = far_problem(cutgen_mod, N, p)
    assert P.n_cut == 0 and P.n_active == N ** 3
    O = Oracle(P)
    M = O.assemble_csr().toarray()
    A1, Mh = sipg_1d(N, p, P.h, P.sipg_gamma)
    ref = np.kron(A1, np.kron(Mh, Mh)) + np.kron(Mh, np.kron(A1, Mh)) + np.kron(Mh, np.kron(Mh, A1))
    nn = p + 1
    # oracle index: ((i*N + j)*N + k)*nn^3 + c*nn^2 + b*nn + a ; kron index: (i,a),(j,b),(k,c)
    perm = np.zeros(M.shape[0], dtype=np.int64)
    for i in range(N):
        for j in range(N):
            for k in range(N):
                for c in range(nn):
                    for b in range(nn):
                        for a in range(nn):
                            o = ((i * N + j) * N + k) * nn ** 3 + c * nn * nn + b * nn + a
                            kr = ((i * nn + a) * N * nn + (j * nn + b)) * N * nn + (k * nn + c)
                            perm[o] = kr
    R = ref[np.ix_(perm, perm)]
    assert np.abs(M - R).max() <= 1e-12 * np.abs(R).max()
    assert np.abs(M @ np.ones(M.shape[0])).max() <= 1e-12 * np.abs(M).max()


# --------------------------------------------------------------------- Q6
def _poly_identity_problem(cutgen_mod, p):
    return cutgen_mod.generate(cutgen_mod.SPHERE, 10, -1.0, 1.0, p)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_q6_exact_identities(cutgen_mod, p):
    P = _poly_identity_problem(cutgen_mod, p)
    O = Oracle(P)
    nd = (p + 1) ** 3
    nodes = gll_np(p)
    lower, h = np.asarray(P.lower), P.h
    # (A 1)_K = 0 on every cell without interface points
    v1 = O.apply(np.ones(P.n_dofs)).reshape(-1, nd)
    has_srf = np.zeros(P.n_active, bool)
    cut_ids = np.where(P.is_cut)[0]
    has_srf[cut_ids] = np.diff(P.srf_ptr) > 0
    scale = O.apply(np.ones(P.n_dofs), absolute=True).reshape(-1, nd)
    assert np.abs(v1[~has_srf]).max() <= 1e-12 * scale.max()

    # 1^T A q = sum_srf W (tau/h q - grad q . n) for a global polynomial q
    rng = np.random.default_rng(3)
    cc = rng.standard_normal(4)
    e = min(p, 2)

    def q(x):
        return cc[0] + cc[1] * x[..., 0] + cc[2] * x[..., 1] ** e * x[..., 2] + cc[3] * x[..., 0] ** p

    def gq(x):
        g = np.zeros(x.shape)
        g[..., 0] = cc[1] + cc[3] * p * x[..., 0] ** (p - 1)
        g[..., 1] = cc[2] * e * x[..., 1] ** (e - 1) * x[..., 2]
        g[..., 2] = cc[2] * x[..., 1] ** e
        return g

    Z, Y, X = np.meshgrid(nodes, nodes, nodes, indexing="ij")
    loc = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1)
    xs = lower + h * (P.active_ijk[:, None, :] + loc[None])
    qv = q(xs).reshape(-1)
    lhs = O.apply(qv).sum()
    xsrf = []
    for c, K in enumerate(cut_ids):
        s = P.srf_pts[P.srf_ptr[c]:P.srf_ptr[c + 1]]
        xsrf.append(np.concatenate([lower + h * (P.active_ijk[K] + s[:, :3]), s[:, 3:]], 1))
    xsrf = np.concatenate(xsrf)
    tau = P.nitsche_tau / h
    rhs = np.sum(xsrf[:, 6] * (tau * q(xsrf[:, :3]) - np.sum(gq(xsrf[:, :3]) * xsrf[:, 3:6], 1)))
    assert abs(lhs - rhs) <= 1e-11 * np.sum(np.abs(xsrf[:, 6]) * (tau * np.abs(q(xsrf[:, :3])) + 10))

    # deep interior cells: (A q)_K = -M_K Δq; harmonic q -> 0; q = x^2 -> -2 ∫φ
    lookup = {tuple(r): k for k, r in enumerate(P.active_ijk.tolist())}
    deep = []
    for K, r in enumerate(P.active_ijk.tolist()):
        if P.is_cut[K]:
            continue
        ok = True
        for d in range(3):
            for s in (-1, 1):
                nb = list(r)
                nb[d] += s
                L = lookup.get(tuple(nb))
                if L is None or P.is_cut[L]:
                    ok = False
        if ok:
            deep.append(K)
    assert deep
    if p >= 2:
        qh = (xs[..., 0] ** 2 - xs[..., 1] ** 2).reshape(-1)
        vh = O.apply(qh, blocks=deep)
        gx, gw = npleg.leggauss(20)
        intl = lag_np((gx + 1) / 2, nodes).T @ (gw / 2)
        phi_int = h ** 3 * np.einsum("c,b,a->cba", intl, intl, intl).ravel()
        q2 = (xs[..., 0] ** 2).reshape(-1)
        v2 = O.apply(q2, blocks=deep)
        for K in deep:
            assert np.abs(vh[K]).max() <= 1e-12 * h
            assert np.abs(v2[K] - (-2.0) * phi_int).max() <= 1e-12 * h
    qh = (xs[..., 0] * xs[..., 1] * xs[..., 2]).reshape(-1)
    vh = O.apply(qh, blocks=deep)
    for K in deep:
        assert np.abs(vh[K]).max() <= 1e-12 * h


# ------------------------------------------------------------------ Q7, Q8, Q12
@pytest.mark.parametrize("p", [1, 2, 3])
def test_q7_q8_q12_symmetry_spd_csr(cutgen_mod, p):
    P = cutgen_mod.config("C1", degree=p) if p == 2 else cutgen_mod.generate(
        cutgen_mod.SPHERE, 8, -1.0, 1.0, p)
    O = Oracle(P)
    M = O.assemble_csr()
    u, w = P.seeded_u(1), P.seeded_u(2)
    Au, Aw = O.apply(u), O.apply(w)
    nrmA = np.abs(M).sum(axis=1).max()
    assert abs(u @ Aw - w @ Au) <= 1e-12 * np.linalg.norm(u) * np.linalg.norm(w) * nrmA
    assert np.abs(M @ u - Au).max() <= 1e-13 * np.abs(Au).max()
    D = M.toarray()
    assert np.abs(D - D.T).max() <= 1e-13 * np.abs(D).max()
    np.linalg.cholesky(D)


def test_q8_flipped_penalty_sign_is_caught(cutgen_mod):
    """Fault injection: a negative SIPG penalty must break SPD."""
    P = cutgen_mod.generate(cutgen_mod.SPHERE, 6, -1.0, 1.0, 1, sipg_gamma=-10.0)
    D = Oracle(P).assemble_csr().toarray()
    with pytest.raises(np.linalg.LinAlgError):
        np.linalg.cholesky(D)


# --------------------------------------------------------------------- Q9
def test_q9_quadrature_moments(cutgen_mod):
    V = 4.0 / 3.0 * math.pi * 0.7 ** 3
    Aex = 4.0 * math.pi * 0.7 ** 2
    c = np.array(cutgen_mod.SPHERE["center"])
    errs = []
    for N in (8, 16, 32):
        P = cutgen_mod.generate(cutgen_mod.SPHERE, N, -1.0, 1.0, 3)
        vol = P.vol_pts[:, 3].sum() + (P.n_active - P.n_cut) * P.h ** 3
        area = P.srf_pts[:, 6].sum()
        cut_ids = np.where(P.is_cut)[0]
        K = np.repeat(cut_ids, np.diff(P.srf_ptr))
        x = np.asarray(P.lower) + P.h * (P.active_ijk[K] + P.srf_pts[:, :3])
        W, nrm = P.srf_pts[:, 6], P.srf_pts[:, 3:6]
        en = np.abs((W[:, None] * nrm).sum(0)).max()
        ex = abs(np.sum(W * np.sum(x * nrm, 1)) - 3 * V)
        assert en < 1e-5 and ex < 1e-4
        assert np.all(P.vol_pts[:, 3] > 0) and np.all(W > 0)
        assert np.all((P.vol_pts[:, :3] >= 0) & (P.vol_pts[:, :3] <= 1))
        # points on the interface
        assert np.abs(np.linalg.norm(x - c, axis=1) - 0.7).max() < 1e-12
        assert np.abs(np.linalg.norm(nrm, axis=1) - 1).max() < 1e-14
        errs.append((abs(vol - V), abs(area - Aex), en, ex))
    assert errs[-1][0] < 1e-9 and errs[-1][1] < 1e-8 and errs[-1][2] < 1e-8 and errs[-1][3] < 1e-8
    for k in range(4):
        assert errs[2][k] < errs[0][k]


def test_q9_plane_half_cell(cutgen_mod):
    P = cutgen_mod.generate({"type": "plane", "normal": [1, 0, 0], "offset": 0.5}, 1, 0.0, 1.0, 2)
    assert P.n_cut == 1
    assert abs(P.vol_pts[:, 3].sum() - 0.5) < 1e-14
    assert abs(P.srf_pts[:, 6].sum() - 1.0) < 1e-14
    assert np.allclose(P.srf_pts[:, 3:6], [1, 0, 0])


def test_q9_cut_face_area_divergence(cutgen_mod):
    """Per cut cell: sum_srf W n + sum over its 6 faces of ±|F∩Ω| e_d = 0."""
    P = cutgen_mod.generate(cutgen_mod.SPHERE, 8, -1.0, 1.0, 3, force_cut_faces=True)
    h = P.h
    lookup = {tuple(r): k for k, r in enumerate(P.active_ijk.tolist())}
    face_area = {}
    for f in range(P.sf_cells.shape[0]):
        face_area[(int(P.sf_cells[f, 0]), int(P.sf_axis[f]))] = P.sf_pts[P.sf_ptr[f]:P.sf_ptr[f + 1], 2].sum()
    import itertools
    # brute-force face areas for faces not between two active cells are unknown -> only
    # check cells whose 6 neighbours are all active
    cut_ids = np.where(P.is_cut)[0]
    checked = 0
    for c, K in enumerate(cut_ids):
        r = P.active_ijk[K].tolist()
        flux = (P.srf_pts[P.srf_ptr[c]:P.srf_ptr[c + 1], 6:7] * P.srf_pts[P.srf_ptr[c]:P.srf_ptr[c + 1], 3:6]).sum(0)
        ok = True
        for d in range(3):
            up = list(r)
            up[d] += 1
            dn = list(r)
            dn[d] -= 1
            Lu, Ld = lookup.get(tuple(up)), lookup.get(tuple(dn))
            if Lu is None or Ld is None:
                ok = False
                break
            au = face_area.get((K, d), None)
            ad = face_area.get((Ld, d), None)
            if au is None:
                au = h * h  # structured face: fully inside
            if ad is None:
                ad = h * h
            flux[d] += au - ad
        if ok:
            checked += 1
            assert np.abs(flux).max() < 1e-4 * h * h  # quadrature error only; a wrong face/sign is O(h^2)
    assert checked > 0


# -------------------------------------------------------------------- Q11
def eoc(e_coarse, e_fine):
    return math.log2(e_coarse / e_fine)


def test_eoc_helper_against_paper_golden():
    rows = [l.split() for l in open(__file__.replace("test_oracle_pins.py", "golden/paper_dg_convergence.txt"))
            if l.strip() and not l.startswith("#")]
    data = {}
    for p, hh, e in rows:
        data.setdefault(int(p), []).append((float(hh), float(e)))
    # the paper's DG slopes p=2: 3.52, 3.22, 3.20 ; p=3: 4.27, 4.17
    s2 = [eoc(data[2][i][1], data[2][i + 1][1]) for i in range(3)]
    s3 = [eoc(data[3][i][1], data[3][i + 1][1]) for i in range(2)]
    assert np.allclose(s2, [3.52, 3.22, 3.20], atol=0.01)
    assert np.allclose(s3, [4.27, 4.17], atol=0.01)
    s1 = [eoc(data[1][i][1], data[1][i + 1][1]) for i in range(4)]
    assert min(s1) > 1.9


def _solve_manufactured(cutgen_mod, N, p):
    """Solve A x = b (oracle CSR, oracle RHS) for the manufactured solution
    u = cos(om R) - cos(om r) (-Laplace u = f, u = 0 on the sphere) and
    return the oracle's relative L2 error.  The solver is test-side: CG with a
    cell-block Jacobi preconditioner (inverse of each n^3 x n^3 diagonal block),
    started from the nodal interpolant of u, stopped at ||r|| <= 1e-7 ||r0|| --
    far below the discretisation error it measures (checked: 1e-10 changes the
    8^3 p=3 error in the 7th digit)."""
    R, om = 0.7, math.pi
    c = np.array(cutgen_mod.SPHERE["center"])
    P = cutgen_mod.generate(cutgen_mod.SPHERE, N, -1.0, 1.0, p)
    O = Oracle(P)
    M = O.assemble_csr()

    def rr(x):
        return np.linalg.norm(x - c, axis=-1)

    def f(x):
        r = rr(x)
        return -om ** 2 * (np.cos(om * r) + 2 * np.sinc(om * r / math.pi))

    def uex(x):
        return math.cos(om * R) - np.cos(om * rr(x))

    b = O.rhs(f)
    nd, nb = (p + 1) ** 3, P.n_active
    Binv = np.empty((nb, nd, nd))
    for K in range(nb):
        Binv[K] = np.linalg.inv(M[K * nd:(K + 1) * nd, K * nd:(K + 1) * nd].toarray())

    def prec(r):
        return np.einsum("kij,kj->ki", Binv, r.reshape(nb, nd)).reshape(-1)

    nodes = gll_np(p)
    Z, Y, X = np.meshgrid(nodes, nodes, nodes, indexing="ij")
    loc = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1)
    x = uex(np.asarray(P.lower) + P.h * (P.active_ijk[:, None, :] + loc[None])).reshape(-1)
    r = b - M @ x
    z = prec(r)
    pv = z.copy()
    rz, r0 = r @ z, np.linalg.norm(r)
    for _ in range(20000):
        if np.linalg.norm(r) <= 1e-7 * r0:
            break
        Ap = M @ pv
        alpha = rz / (pv @ Ap)
        x += alpha * pv
        r -= alpha * Ap
        z = prec(r)
        rzn = r @ z
        pv = z + (rzn / rz) * pv
        rz = rzn
    assert np.linalg.norm(r) <= 1e-7 * r0
    return O.l2_error(x, uex)


@pytest.mark.parametrize("p,meshes", [(1, (8, 16, 32)), (2, (8, 16, 32)), (3, (8, 12, 16))])
def test_q11_convergence_order(cutgen_mod, p, meshes):
    """L2 EOC >= p + 0.7 on three meshes (the paper's slope p+1,
    P:716).  p = 3 uses 8/12/16 (a 32^3 p = 3 CSR has ~1.9e8 non-zeros: minutes on the
    CPU; tools/q11_full.py runs 8/16/32 at p = 3 and its output is in profiles/)."""
    errs = [_solve_manufactured(cutgen_mod, N, p) for N in meshes]
    for k in range(len(meshes) - 1):
        rate = math.log(errs[k] / errs[k + 1]) / math.log(meshes[k + 1] / meshes[k])
        assert rate >= p + 0.7, (p, meshes, errs, rate)


# ------------------------------------------------------------- cost formulas
def test_paper_cost_formula_golden():
    """The product's closed forms (paper_2404_07911_b200/costmodel.py) against the
    values of the paper's formulas (tests/golden/paper_cost_formulas.txt)."""
    from paper_2404_07911_b200 import costmodel as cm
    rows = [l.split() for l in open(__file__.replace("test_oracle_pins.py", "golden/paper_cost_formulas.txt"))
            if l.strip() and not l.startswith("#")]
    f = {
        "structured_cell_fma": cm.paper_structured_cell_fma,
        "structured_face_fma": cm.paper_structured_face_fma,
        "unstructured_cell_fma": cm.paper_unstructured_cell_fma,
        "unstructured_face_fma": cm.paper_unstructured_face_fma,
        # the sparse rows are keyed by k = p+1
        "sparse_dg_bytes_per_dof": lambda k: cm.paper_sparse_dg_bytes_per_dof(k - 1),
        "sparse_dg_flops_per_dof": lambda k: cm.paper_sparse_dg_flops_per_dof(k - 1),
        "sparse_cg_bytes_per_dof": lambda k: cm.paper_sparse_cg_bytes_per_dof(k - 1),
        "sparse_cg_flops_per_dof": lambda k: cm.paper_sparse_cg_flops_per_dof(k - 1),
    }
    assert len(rows) == len(f)
    for name, k, val, *_ in rows:
        assert f[name](int(k)) == int(val), (name, f[name](int(k)), val)
    # the cut-face count at n_q = k^2 is the paper's 3k^4 + 5k^3 (x 8: FLOPs, E+I, sides)
    for k in range(2, 10):
        assert cm.flops_cut_face(k, k * k) == 8 * cm.paper_unstructured_face_fma(k)


class _Prob:
    def __init__(self, ijk, cut, sf_cells=(), sf_axis=(), sf_npts=()):
        self.active_ijk = np.asarray(ijk, dtype=np.int32)
        self.is_cut = np.asarray(cut, dtype=np.uint8)
        self.sf_cells = np.asarray(sf_cells, dtype=np.int32).reshape(-1, 2)
        self.sf_axis = np.asarray(sf_axis, dtype=np.uint8)
        self.sf_ptr = np.concatenate([[0], np.cumsum(sf_npts)]).astype(np.int64)


def test_cost_model_hand_counted():
    """apply_work on 2 x 1 x 1 meshes, counted by hand from SURVEY §8(d) at p = 1
    (n = 2, even-odd line cost c_eo = n^2 + 2n = 8):
      uncut cell   2*6*n^2*8 + 3n^3            = 384 + 24         = 408
      full face    2*2*(2n^3 + 2*2*n*8) + 10n^2 = 4*(16 + 64) + 40 = 360
      GP face      8n^4 + 2n^2*8               = 128 + 64         = 192
      volume pt    4(2n^3+3n^2+4n) + 6n(n-1) + 12 = 144 + 12 + 12 = 168
      interface pt volume pt + 12                                 = 180
      cut face     8 (n^3 + n_q (3n^2 + 4n)), n_q = 5: 8 (8 + 100) = 864
    bytes: 16 B per DoF (8 DoFs per cell), 8 B per cell, 12 B per special face side,
    32 / 56 / 24 B per volume / interface / cut-face point."""
    from paper_2404_07911_b200 import costmodel as cm
    # uncut cell 0 | cut cell 1: one full face (SIPG) that is also a GP face
    P = _Prob([[0, 0, 0], [1, 0, 0]], [0, 1])
    c = cm.face_classes(P)
    assert c == {"sipg_side_cut": 1, "sipg_side_uncut": 1, "gp_side_cut": 1, "gp_side_uncut": 1,
                 "cutface_side": 0, "cutface_pts_side": 0}
    st = {"degree": 1, "n_uncut": 1, "n_cut": 1, "n_vol_pts": 10, "n_srf_pts": 4, "n_face_pts": 0, "n_dofs": 16}
    w = cm.apply_work(st, c)
    assert w["F_uncut"] == 408 + 360 / 2 + 192 / 2
    assert w["F_cut"] == 10 * 168 + 4 * 180 + 360 / 2 + 192 / 2
    assert w["B_uncut"] == 16 * 8 + 8 + 12
    assert w["B_cut"] == 16 * 8 + 8 + 10 * 32 + 4 * 56 + 12
    # two cut cells sharing a listed cut face with 5 points (GP too), along y
    P = _Prob([[0, 0, 0], [0, 1, 0]], [1, 1], [[0, 1]], [1], [5])
    c = cm.face_classes(P)
    assert c == {"sipg_side_cut": 0, "sipg_side_uncut": 0, "gp_side_cut": 2, "gp_side_uncut": 0,
                 "cutface_side": 2, "cutface_pts_side": 10}
    st = {"degree": 1, "n_uncut": 0, "n_cut": 2, "n_vol_pts": 0, "n_srf_pts": 0, "n_face_pts": 5, "n_dofs": 16}
    w = cm.apply_work(st, c)
    assert w["F_uncut"] == 0 and w["F_cut"] == 864 + 192
    assert w["B_cut"] == 2 * (16 * 8 + 8) + 5 * 24 + 12 * 4
    # a listed face with no points carries no SIPG (reading A13) but still the GP
    P = _Prob([[0, 0, 0], [0, 0, 1]], [1, 0], [[0, 1]], [2], [0])
    assert cm.face_classes(P)["sipg_side_cut"] == 0 and cm.face_classes(P)["gp_side_uncut"] == 1


def test_cost_model_face_classes_match_oracle_faces(cutgen_mod):
    """face_classes enumerates the same faces as the oracle (C1 and a gyroid box)."""
    from paper_2404_07911_b200 import costmodel as cm
    for P in (cutgen_mod.config("C1"), cutgen_mod.generate(cutgen_mod.GYROID, 6, 0.0, 1.0, 1)):
        O = Oracle(P)
        cut = P.is_cut.astype(bool)
        ref = {"sipg_side_cut": 0, "sipg_side_uncut": 0, "gp_side_cut": 0, "gp_side_uncut": 0,
               "cutface_side": 0, "cutface_pts_side": 0}
        for (m, pl, d, sf) in O.faces:
            npt = -1 if sf < 0 else int(P.sf_ptr[sf + 1] - P.sf_ptr[sf])
            for s in (m, pl):
                k = "cut" if cut[s] else "uncut"
                if cut[m] or cut[pl]:
                    ref["gp_side_" + k] += 1
                if npt < 0:
                    ref["sipg_side_" + k] += 1
                elif npt > 0:
                    ref["cutface_side"] += 1
                    ref["cutface_pts_side"] += npt
        assert cm.face_classes(P) == ref


def test_oracle_cg_solves_spd_system():
    """oracle.operator.cg (used by the GPU CG parity test) against a direct solve."""
    rng = np.random.default_rng(4)
    B = rng.standard_normal((40, 40))
    A = B @ B.T + 40 * np.eye(40)
    b = rng.standard_normal(40)
    x, it = cg(lambda y: A @ y, b, tol=1e-14, maxiter=500)
    assert np.abs(x - np.linalg.solve(A, b)).max() <= 1e-12 * np.abs(x).max()
    x, it = cg(lambda y: A @ y, b, tol=0.0, maxiter=3)
    assert it == 3


def test_oracle_spmv_c_matches_scipy(cutgen_mod):
    """oracle/csrc/spmv.c (the host-core sparse baseline) = scipy's CSR product on the
    oracle-assembled C1 matrix, for 1 and several threads."""
    from oracle import spmv
    P = cutgen_mod.config("C1")
    M = Oracle(P).assemble_csr()
    u = P.seeded_u(2)
    ref = M @ u
    for nt in (1, 3):
        y, _ = spmv.spmv(M, u, nthreads=nt)
        assert np.abs(y - ref).max() <= 1e-13 * np.abs(ref).max()


# -------------------------------------------------------------------- Q13
def _ball_moment(e, R, surface):
    """Integral of X^a Y^b Z^c over the sphere |X| = R (surface) or the ball |X| <= R:
    2 G((a+1)/2) G((b+1)/2) G((c+1)/2) / G((a+b+c+3)/2) R^(a+b+c+2) for even exponents
    (0 otherwise); the ball integral is the radial integral of that, R / (a+b+c+3) times it."""
    if any(k % 2 for k in e):
        return 0.0
    s = sum(e)
    m = 2.0 * math.gamma((e[0] + 1) / 2) * math.gamma((e[1] + 1) / 2) * math.gamma((e[2] + 1) / 2) \
        / math.gamma((s + 3) / 2) * R ** (s + 2)
    return m if surface else m * R / (s + 3)


def _pmul(f, g):
    out = {}
    for ea, ca in f.items():
        for eb, cb in g.items():
            k = (ea[0] + eb[0], ea[1] + eb[1], ea[2] + eb[2])
            out[k] = out.get(k, 0.0) + ca * cb
    return out


def _pdiff(f, d):
    out = {}
    for e, c in f.items():
        if e[d] > 0:
            k = tuple(e[i] - (i == d) for i in range(3))
            out[k] = out.get(k, 0.0) + c * e[d]
    return out


def _padd(f, g, s=1.0):
    out = dict(f)
    for e, c in g.items():
        out[e] = out.get(e, 0.0) + s * c
    return out


def _pint(f, R, surface):
    return sum(c * _ball_moment(e, R, surface) for e, c in f.items())


def _peval(f, X):
    return sum(c * X[..., 0] ** e[0] * X[..., 1] ** e[1] * X[..., 2] ** e[2] for e, c in f.items())


@pytest.mark.parametrize("p", [1, 2, 3])
def test_q13_curved_interface_closed_form(cutgen_mod, p):
    """The absolute value of the curved-interface terms (cut-cell volume + Nitsche on a
    sphere) against a closed form: for GLOBAL polynomials q, r of degree <= p every jump
    vanishes (SIPG, ghost penalty: 0) and eq:bilinear_dg reduces to
        a(q, r) = int_B grad q . grad r - int_S (d_n q r + q d_n r) + tau/h int_S q r
    over the ball B and sphere S, whose monomial moments are Gamma-function closed forms
    (n = X / R on S).  The only error is the generated quadrature's, which Q9 bounds and
    which falls with h; a wrong sign, a dropped tau/h, a flipped normal or a missing weight
    in the oracle's cut-cell volume or Nitsche code is O(1)."""
    R = 0.7
    c = np.array(cutgen_mod.SPHERE["center"])
    rng = np.random.default_rng(13)
    mons = [(a, b, d) for a in range(p + 1) for b in range(p + 1) for d in range(p + 1) if a + b + d <= p]
    q = {e: float(rng.standard_normal()) for e in mons}
    r = {e: float(rng.standard_normal()) for e in mons}
    Xn = {(1, 0, 0): 1.0 / R}, {(0, 1, 0): 1.0 / R}, {(0, 0, 1): 1.0 / R}  # the normal's components on S
    grad = lambda f: [_pdiff(f, d) for d in range(3)]  # noqa: E731
    gq, gr = grad(q), grad(r)
    vol = {}
    dnq, dnr = {}, {}
    for d in range(3):
        vol = _padd(vol, _pmul(gq[d], gr[d]))
        dnq = _padd(dnq, _pmul(gq[d], Xn[d]))
        dnr = _padd(dnr, _pmul(gr[d], Xn[d]))
    nodes = gll_np(p)
    Z, Y, X = np.meshgrid(nodes, nodes, nodes, indexing="ij")
    loc = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1)
    errs = []
    for N in (8, 16):
        P = cutgen_mod.generate(cutgen_mod.SPHERE, N, -1.0, 1.0, p)
        tau = P.nitsche_tau / P.h
        exact = _pint(vol, R, False) - _pint(_padd(_pmul(dnq, r), _pmul(q, dnr)), R, True) \
            + tau * _pint(_pmul(q, r), R, True)
        scale = abs(_pint(vol, R, False)) + tau * abs(_pint(_pmul(q, q), R, True))
        xs = np.asarray(P.lower) + P.h * (P.active_ijk[:, None, :] + loc[None]) - c
        O = Oracle(P)
        got = float(_peval(r, xs).reshape(-1) @ O.apply(_peval(q, xs).reshape(-1)))
        errs.append(abs(got - exact) / scale)
        if N == 8:  # fault injection: flipped interface normals (the consistency terms change sign)
            P.srf_pts[:, 3:6] *= -1.0
            bad = float(_peval(r, xs).reshape(-1) @ Oracle(P).apply(_peval(q, xs).reshape(-1)))
            cons = _pint(_padd(_pmul(dnq, r), _pmul(q, dnr)), R, True)
            assert abs((bad - got) - 2.0 * cons) <= 5e-3 * abs(cons) and abs(cons) > 1e-3 * scale / tau
    # measured: p = 1 6.7e-5 -> 7.9e-6 (the (p+1)-point rules: ~h^3), p = 2 1.9e-6 -> 3.4e-8, p = 3 7.0e-7 -> 2.4e-9
    assert errs[1] <= (2e-5 if p == 1 else 1e-7) and errs[1] <= errs[0] / 4, errs


# -------------------------------------------------------------------- Q14
def _ang(b, c):
    """Integral of cos^b sin^c over [0, 2 pi] (0 unless b, c are even)."""
    if b % 2 or c % 2:
        return 0.0
    return 2.0 * math.gamma((b + 1) / 2) * math.gamma((c + 1) / 2) / math.gamma((b + c + 2) / 2)


def _slab_int(a, m, X0, R):
    """int_{X0}^{R} x^a (R^2 - x^2)^m dx, integer m >= 0 (a 1-D polynomial integral)."""
    from numpy.polynomial import polynomial as npp
    pol = npp.polypow([R * R, 0.0, -1.0], m) if m else np.array([1.0])
    pol = npp.polymul(pol, [0.0] * a + [1.0])
    ip = npp.polyint(pol)
    return float(npp.polyval(R, ip) - npp.polyval(X0, ip))


def _cap_int(f, X0, R, kind):
    """Integral of the polynomial f(X, Y, Z) over the part X > X0 of the ball ("cap": slices
    are disks of radius rho = sqrt(R^2 - X^2), disk moment = ang rho^(b+c+2) / (b+c+2)), of
    the sphere ("scap": dS = R dX dphi, Archimedes) or over the disk X = X0 ("disk")."""
    tot = 0.0
    for (a, b, c), co in f.items():
        g = _ang(b, c)
        if g == 0.0:
            continue
        m = (b + c) // 2
        if kind == "cap":
            tot += co * g / (b + c + 2) * _slab_int(a, m + 1, X0, R)
        elif kind == "scap":
            tot += co * g * R * _slab_int(a, m, X0, R)
        else:
            tot += co * g / (b + c + 2) * X0 ** a * (R * R - X0 * X0) ** (m + 1)
    return tot


@pytest.mark.parametrize("p", [1, 2, 3])
def test_q14_curved_cut_faces_broken_polynomial(cutgen_mod, p):
    """Cut-face SIPG next to a CURVED interface, absolute value: u = q + H J, r = s + H K
    with global polynomials q, s, J, K (degree <= p) and H the indicator of the half space
    X > X0 behind a MESH plane (so u, r are in the DG space and jump only on that plane).
    The faces in the plane, cut by the sphere or not, tile the disk D = plane n ball, so
    with n = e_x from the minus to the plus side, [u] = u- - u+ = -J, {d_n u} = d_x q + d_x J / 2,
        a(u, r) = a(q, s)                                               (Q13, ball / sphere)
                + int_cap (grad q.grad K + grad J.grad s + grad J.grad K)
                - int_scap (d_n q K + d_n J s + d_n J K + q d_n K + J d_n s + J d_n K)
                + tau/h int_scap (q K + J s + J K)
                + int_D ((d_x q + d_x J / 2) K + (d_x s + d_x K / 2) J) + sigma/h int_D J K
    (eq:bilinear_dg P:83-92 with eq:unstructured_face P:489-496, terms 1|2|4; the ghost
    penalty integrates over whole faces and is masked out), all of them 1-D polynomial
    integrals.  Swapped in-face coordinates, a wrong side or sign of the averages, or cut
    faces that do not tile the disk are O(1) errors."""
    R = 0.7
    c = np.array(cutgen_mod.SPHERE["center"])
    rng = np.random.default_rng(14)
    mons = [(a, b, d) for a in range(p + 1) for b in range(p + 1) for d in range(p + 1) if a + b + d <= p]
    q, s, J, K = ({e: float(rng.standard_normal()) for e in mons} for _ in range(4))
    Xn = {(1, 0, 0): 1.0 / R}, {(0, 1, 0): 1.0 / R}, {(0, 0, 1): 1.0 / R}

    def gdot(f, g):
        out = {}
        for d in range(3):
            out = _padd(out, _pmul(_pdiff(f, d), _pdiff(g, d)))
        return out

    def dn(f):
        out = {}
        for d in range(3):
            out = _padd(out, _pmul(_pdiff(f, d), Xn[d]))
        return out

    def psum(*fs):
        out = {}
        for f in fs:
            out = _padd(out, f)
        return out

    half = lambda f: {e: 0.5 * v for e, v in f.items()}  # noqa: E731
    nodes = gll_np(p)
    Z, Y, X = np.meshgrid(nodes, nodes, nodes, indexing="ij")
    loc = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1)
    errs = []
    for N in (8, 16):
        P = cutgen_mod.generate(cutgen_mod.SPHERE, N, -1.0, 1.0, p)
        h = P.h
        i0 = 5 * N // 8  # the mesh plane x = 0.25
        X0 = -1.0 + i0 * h - c[0]
        tau, sig = P.nitsche_tau / h, P.sipg_gamma / h
        exact = (_pint(gdot(q, s), R, False) - _pint(psum(_pmul(dn(q), s), _pmul(q, dn(s))), R, True)
                 + tau * _pint(_pmul(q, s), R, True)
                 + _cap_int(psum(gdot(q, K), gdot(J, s), gdot(J, K)), X0, R, "cap")
                 - _cap_int(psum(_pmul(dn(q), K), _pmul(dn(J), s), _pmul(dn(J), K),
                                 _pmul(q, dn(K)), _pmul(J, dn(s)), _pmul(J, dn(K))), X0, R, "scap")
                 + tau * _cap_int(psum(_pmul(q, K), _pmul(J, s), _pmul(J, K)), X0, R, "scap")
                 + _cap_int(psum(_pmul(psum(_pdiff(q, 0), half(_pdiff(J, 0))), K),
                                 _pmul(psum(_pdiff(s, 0), half(_pdiff(K, 0))), J)), X0, R, "disk")
                 + sig * _cap_int(_pmul(J, K), X0, R, "disk"))
        face_part = abs(sig * _cap_int(_pmul(J, K), X0, R, "disk"))
        xs = np.asarray(P.lower) + h * (P.active_ijk[:, None, :] + loc[None]) - c
        Hc = (P.active_ijk[:, 0] >= i0)[:, None]
        uv = (_peval(q, xs) + Hc * _peval(J, xs)).reshape(-1)
        rv = (_peval(s, xs) + Hc * _peval(K, xs)).reshape(-1)
        got = float(rv @ Oracle(P, term_mask=1 | 2 | 4).apply(uv))
        errs.append(abs(got - exact) / face_part)  # relative to the face penalty term alone
        if N == 8:  # fault injection: the cut faces' in-face coordinates swapped
            P.sf_pts[:, [0, 1]] = P.sf_pts[:, [1, 0]]
            bad = float(rv @ Oracle(P, term_mask=1 | 2 | 4).apply(uv))
            assert abs(bad - exact) / face_part >= 20 * errs[0]  # measured 4.0 / 8.7e-3 / 2.8 (p = 1, 2, 3)
    # measured (relative to the face penalty term; the error is the generated quadrature's, most of
    # it from the volume / interface terms, Q13): p = 1 4.3e-2 -> 2.2e-3, p = 2 8.6e-5 -> 1.6e-6,
    # p = 3 5.6e-4 -> 7.3e-7
    assert errs[1] <= (5e-3 if p == 1 else 5e-6) and errs[1] <= errs[0] / 4, errs
