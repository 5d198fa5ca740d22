"""Pins of the preconditioner oracle (oracle/solver.py).

* Chebyshev iteration: on a diagonal operator the error after k steps is the
  textbook e_k = T_k((theta - lam)/delta) / T_k(theta/delta) e_0 per eigenvalue
  (numpy's Chebyshev polynomials, not the recurrence), degrees 1..8, zero and
  non-zero start; on the DG operator the A-norm error obeys the Chebyshev bound
  1 / T_k(theta/delta) when the interval holds the spectrum (dense eigenvalues).
* p-transfer: a coarse cell polynomial is reproduced exactly at arbitrary points
  (barycentric route of tests/pin1d.py), transfers compose (1 -> 2 -> 4 = 1 -> 4),
  equal degrees give the identity, restriction is the adjoint.
* V-cycle: one level is the coarse Chebyshev iteration; the V-cycle is symmetric
  and positive definite (same polynomial before and after), its error
  propagation I - BA contracts in the A-norm, and PCG with it needs fewer
  iterations than Jacobi-PCG for the same residual reduction.
"""
import numpy as np
import pytest
from numpy.polynomial import chebyshev as npcheb

import pin1d
from oracle import Oracle
from oracle import solver as S


def cheb_T(k, x):
    return npcheb.chebval(x, [0.0] * k + [1.0])


@pytest.mark.parametrize("degree", range(1, 9))
@pytest.mark.parametrize("start", ["zero", "x0"])
def test_chebyshev_closed_form_diagonal(degree, start):
    rng = np.random.default_rng(degree)
    n = 40
    alpha = rng.uniform(0.5, 30.0, n)      # A = diag(alpha)
    dinv = rng.uniform(0.2, 2.0, n)        # D^-1
    lam = dinv * alpha                      # eigenvalues of D^-1 A
    lmax, lmin = lam.max() * 1.05, lam.min() * 0.7
    theta, delta = (lmax + lmin) / 2, (lmax - lmin) / 2
    r = rng.uniform(-1, 1, n)
    xs = r / alpha
    x0 = None if start == "zero" else rng.uniform(-1, 1, n)
    x = S.chebyshev(lambda y: alpha * y, lambda y: dinv * y, r, degree, lmax, lmin, x0=x0)
    e0 = xs - (0.0 if x0 is None else x0)
    ek = cheb_T(degree, (theta - lam) / delta) / cheb_T(degree, theta / delta) * e0
    assert np.abs((xs - x) - ek).max() <= 1e-12 * np.abs(e0).max()


def test_chebyshev_bound_on_operator(cutgen_mod):
    P = cutgen_mod.generate(cutgen_mod.SPHERE, 5, -1.0, 1.0, 1)
    A = Oracle(P).assemble_csr()
    Ad = A.toarray()
    dinv = 1.0 / A.diagonal()
    s = np.sqrt(dinv)
    ev = np.linalg.eigvalsh(s[:, None] * Ad * s[None, :])
    lmin, lmax = ev[0], ev[-1]
    theta, delta = (lmax + lmin) / 2, (lmax - lmin) / 2
    rng = np.random.default_rng(3)
    xs = rng.uniform(-1, 1, A.shape[0])
    b = Ad @ xs
    anorm = lambda e: float(np.sqrt(e @ (Ad @ e)))  # noqa: E731
    for k in (2, 5, 9):
        x = S.chebyshev(lambda y: A @ y, lambda y: dinv * y, b, k, lmax, lmin)
        assert anorm(xs - x) <= anorm(xs) / cheb_T(k, theta / delta) * (1 + 1e-8)


@pytest.mark.parametrize("pc,pf", [(1, 2), (1, 3), (2, 4), (2, 5), (4, 8), (3, 3)])
def test_prolongation_reproduces_coarse_polynomial(pc, pf):
    rng = np.random.default_rng(pc * 10 + pf)
    ncell = 3
    uc = rng.uniform(-1, 1, ncell * (pc + 1) ** 3)
    cmap = np.array([2, 0, -1, 1])           # a fine cell without a coarse counterpart
    uf = S.prolongate(uc, pc, pf, cmap).reshape(len(cmap), -1)
    ucb = uc.reshape(ncell, -1)
    pts = rng.uniform(0, 1, (20, 3))

    def field(coef, p):
        Lx, Ly, Lz = (pin1d.values(p, pts[:, d]) for d in range(3))
        n = p + 1
        c = coef.reshape(n, n, n)  # [c][b][a]
        return np.einsum("qa,qb,qc,cba->q", Lx, Ly, Lz, c)

    for K, c in enumerate(cmap):
        if c < 0:
            assert np.all(uf[K] == 0.0)
        else:
            assert np.abs(field(uf[K], pf) - field(ucb[c], pc)).max() <= 1e-12
    if pc == pf:
        assert np.allclose(S.prolongation_1d(pc, pf), np.eye(pc + 1), atol=1e-14)


def test_transfer_composition_and_adjoint():
    I12, I24, I14 = S.prolongation_1d(1, 2), S.prolongation_1d(2, 4), S.prolongation_1d(1, 4)
    assert np.abs(I24 @ I12 - I14).max() <= 1e-13
    rng = np.random.default_rng(0)
    cmap = np.array([1, -1, 0, 2])
    uc, rf = rng.uniform(-1, 1, 3 * 8), rng.uniform(-1, 1, 4 * 125)
    lhs = S.prolongate(uc, 1, 4, cmap) @ rf
    rhs = uc @ S.restrict(rf, 1, 4, cmap, 3)
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)


def _levels(cutgen_mod, degrees, N=5, lam_scale=1.1, inner="jacobi"):
    # every level takes the finest level's penalties (reading A27: then A_c = P^T A P on
    # the uncut cells and faces)
    pf = degrees[-1]
    levels = []
    for p in degrees:
        P = cutgen_mod.generate(cutgen_mod.SPHERE, N, -1.0, 1.0, p, sipg_gamma=10.0 * pf ** 2,
                                nitsche_tau=10.0 * pf ** 2)
        A = Oracle(P).assemble_csr()
        minv = S.jacobi(A) if inner == "jacobi" else S.block_jacobi(A, (p + 1) ** 3)
        lam = S.dense_lambda_max(A, minv) * lam_scale
        levels.append((S.Level(lambda y, A=A: A @ y, minv, lam, p, P.active_ijk), A, P))
    return levels


def test_vcycle_one_level_is_chebyshev(cutgen_mod):
    (L, A, P), = _levels(cutgen_mod, [2])
    r = np.random.default_rng(1).uniform(-1, 1, L.n)
    z = S.vcycle([L], r, 3, 15.0, 6, 40.0)
    z2 = S.chebyshev(L.apply, L.minv, r, 6, L.lam_max, L.lam_max / 40.0)
    assert np.array_equal(z, z2)


@pytest.mark.parametrize("inner", ["jacobi", "block"])
def test_vcycle_symmetric_spd_and_contracts(cutgen_mod, inner):
    lv = _levels(cutgen_mod, [1, 3], inner=inner)
    levels = [x[0] for x in lv]
    A = lv[-1][1].toarray()
    n = levels[-1].n
    B = lambda r: S.vcycle(levels, r, 3, 15.0, 8, 40.0)  # noqa: E731
    rng = np.random.default_rng(7)
    for _ in range(3):
        u, v = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        bu, bv = B(u), B(v)
        assert abs(u @ bv - v @ bu) <= 1e-11 * np.linalg.norm(u) * np.linalg.norm(bv)
        assert u @ bu > 0 and v @ bv > 0
    # error propagation E = I - B A contracts in the A-norm (power iteration)
    e = rng.uniform(-1, 1, n)
    anorm = lambda x: float(np.sqrt(x @ (A @ x)))  # noqa: E731
    for _ in range(6):
        e1 = e - B(A @ e)
        rho = anorm(e1) / anorm(e)
        e = e1 / anorm(e1)
    assert rho < 0.9, rho


@pytest.mark.parametrize("inner", ["jacobi", "block"])
def test_pmg_pcg_beats_one_level(cutgen_mod, inner):
    lv = _levels(cutgen_mod, [1, 2], N=6, inner=inner)
    levels = [x[0] for x in lv]
    A, P = lv[-1][1], lv[-1][2]
    b = Oracle(P).rhs(lambda x: np.ones(len(x)))
    _, hm = S.pcg(lambda y: A @ y, b, lambda r: S.vcycle(levels, r, 3, 15.0, 8, 40.0), 25)
    _, hj = S.pcg(lambda y: A @ y, b, levels[-1].minv, 25)
    assert hm[-1] < 1e-2 * hj[-1], (hm[-1], hj[-1])
    assert hm[-1] <= 1e-4 * hm[0]


def test_block_jacobi_is_the_block_inverse(cutgen_mod):
    P = cutgen_mod.generate(cutgen_mod.SPHERE, 4, -1.0, 1.0, 2)
    A = Oracle(P).assemble_csr().toarray()
    nd = 27
    r = np.random.default_rng(2).uniform(-1, 1, A.shape[0])
    z = S.block_jacobi(Oracle(P).assemble_csr(), nd)(r)
    for K in range(A.shape[0] // nd):
        sl = slice(K * nd, (K + 1) * nd)
        assert np.abs(A[sl, sl] @ z[sl] - r[sl]).max() <= 1e-10 * np.abs(r[sl]).max()
