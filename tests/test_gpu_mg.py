"""GPU parity of the Chebyshev / p-multigrid preconditioner (include/cutfem.h cutfem_mg_*,
csrc/mg.inl) against oracle/solver.py.

Every oracle input is the oracle's own (its CSR operator, its diagonal / cell blocks,
its dense lam_max); the library is given the same lam_max per level so both sides run
the same polynomial.  Compared: the p-transfers, a Chebyshev iteration with point and
cell-block Jacobi (zero and non-zero start), one V-cycle (2 and 3 levels), the PCG
iterates; the library's Lanczos lam_max is checked against the dense eigenvalue; the
V-cycle PCG converges where Jacobi PCG stalls.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import Oracle  # noqa: E402
from oracle import solver as S  # noqa: E402


@pytest.fixture(scope="module")
def cf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_07911_b200 as m
    m.load()
    return m


def problems(cutgen_mod, degrees, N, geom="sphere"):
    """Level problems of one mesh; every level takes the finest level's penalties (A27)."""
    pf = degrees[-1]
    kw = dict(sipg_gamma=10.0 * pf ** 2, nitsche_tau=10.0 * pf ** 2)
    if geom == "sphere":
        return [cutgen_mod.generate(cutgen_mod.SPHERE, N, -1.0, 1.0, p, **kw) for p in degrees]
    return [cutgen_mod.generate(cutgen_mod.GYROID, N, 0.0, 1.0, p, **kw) for p in degrees]


def oracle_levels(probs, inner):
    out = []
    for P in probs:
        A = Oracle(P).assemble_csr()
        minv = S.jacobi(A) if inner == "jacobi" else S.block_jacobi(A, (P.degree + 1) ** 3)
        lam = 1.1 * S.dense_lambda_max(A, minv)
        out.append(S.Level(lambda y, A=A: A @ y, minv, lam, P.degree, P.active_ijk))
    return out


def block_kappa(probs):
    """max condition number of the cell blocks A_KK over the levels: the GPU inverts them
    by a Gauss-Jordan sweep, the oracle solves with their Cholesky factors, so the two
    inner preconditioners differ by ~kappa * eps relative (the derived tolerance)."""
    k = 1.0
    for P in probs:
        A = Oracle(P).assemble_csr().tocsr()
        nd = (P.degree + 1) ** 3
        k = max(k, max(np.linalg.cond(A[i:i + nd, i:i + nd].toarray()) for i in range(0, A.shape[0], nd)))
    return k


EPS = np.finfo(np.float64).eps


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def relerr(a, b):
    return np.abs(a - b).max() / np.abs(b).max()


@pytest.mark.parametrize("degrees,N", [((1, 3), 6), ((2, 5), 4), ((4, 8), 3)])
def test_transfers_match_oracle(cf, cutgen_mod, degrees, N):
    probs = problems(cutgen_mod, degrees, N)
    ops = [cf.CutFEM(P) for P in probs]
    mg = cf.CutFEMMG(ops, inner="jacobi", eig_iters=0)
    mg.set_lambdas([1.0, 1.0])
    pc, pf = degrees
    cmap = S.block_map(probs[1].active_ijk, probs[0].active_ijk)
    rng = np.random.default_rng(5)
    uc, rf = rng.uniform(-1, 1, probs[0].n_dofs), rng.uniform(-1, 1, probs[1].n_dofs)
    uf = mg.transfer(1, "prolong", dev(uc), torch.empty(probs[1].n_dofs, dtype=torch.float64, device="cuda"))
    rc = mg.transfer(1, "restrict", dev(rf), torch.empty(probs[0].n_dofs, dtype=torch.float64, device="cuda"))
    assert relerr(uf.cpu().numpy(), S.prolongate(uc, pc, pf, cmap)) <= 1e-13
    assert relerr(rc.cpu().numpy(), S.restrict(rf, pc, pf, cmap, probs[0].n_active)) <= 1e-13


@pytest.mark.parametrize("inner", ["jacobi", "block"])
@pytest.mark.parametrize("p,N", [(1, 6), (2, 5), (3, 4)])
def test_chebyshev_matches_oracle(cf, cutgen_mod, inner, p, N):
    P, = problems(cutgen_mod, [p], N)
    L, = oracle_levels([P], inner)
    op = cf.CutFEM(P)
    mg = cf.CutFEMMG([op], inner=inner, eig_iters=0)
    mg.set_lambdas([L.lam_max])
    tol = max(1e-10, 20 * block_kappa([P]) * EPS) if inner == "block" else 1e-10
    rng = np.random.default_rng(11)
    r, x0 = rng.uniform(-1, 1, P.n_dofs), rng.uniform(-1, 1, P.n_dofs)
    for k in (1, 2, 5):
        lmin = L.lam_max / 15.0
        xo = S.chebyshev(L.apply, L.minv, r, k, L.lam_max, lmin)
        xg = mg.smooth(0, dev(r), torch.empty(P.n_dofs, dtype=torch.float64, device="cuda"), k, L.lam_max, lmin)
        assert relerr(xg.cpu().numpy(), xo) <= tol, k
        xo = S.chebyshev(L.apply, L.minv, r, k, L.lam_max, lmin, x0=x0)
        xg = mg.smooth(0, dev(r), dev(x0.copy()), k, L.lam_max, lmin, x0_given=True)
        assert relerr(xg.cpu().numpy(), xo) <= tol, k


@pytest.mark.parametrize("inner", ["jacobi", "block"])
@pytest.mark.parametrize("degrees,N,geom", [((1, 3), 5, "sphere"), ((1, 2, 4), 4, "sphere"), ((1, 2), 5, "gyroid")])
def test_vcycle_and_pcg_match_oracle(cf, cutgen_mod, inner, degrees, N, geom):
    probs = problems(cutgen_mod, degrees, N, geom)
    levels = oracle_levels(probs, inner)
    ops = [cf.CutFEM(P) for P in probs]
    mg = cf.CutFEMMG(ops, inner=inner, smooth_degree=3, smooth_range=15.0, coarse_degree=6, coarse_range=40.0,
                     eig_iters=0)
    mg.set_lambdas([L.lam_max for L in levels])
    kap = block_kappa(probs) if inner == "block" else 1.0
    r = np.random.default_rng(3).uniform(-1, 1, probs[-1].n_dofs)
    zo = S.vcycle(levels, r, 3, 15.0, 6, 40.0)
    zg = mg.vcycle(dev(r)).cpu().numpy()
    assert relerr(zg, zo) <= max(1e-9, 20 * kap * EPS), (relerr(zg, zo), kap)
    b = Oracle(probs[-1]).rhs(lambda x: np.ones(len(x)))
    xo, ho = S.pcg(levels[-1].apply, b, lambda y: S.vcycle(levels, y, 3, 15.0, 6, 40.0), 8)
    xg, hg = mg.pcg(dev(b), iters=8)
    assert len(hg) == 9
    assert relerr(xg.cpu().numpy(), xo) <= max(1e-7, 2000 * kap * EPS)
    assert np.abs(hg - ho).max() <= max(1e-7, 2000 * kap * EPS) * ho[0]


@pytest.mark.parametrize("inner", ["jacobi", "block"])
def test_lanczos_lambda_max(cf, cutgen_mod, inner):
    P, = problems(cutgen_mod, [2], 5)
    L, = oracle_levels([P], inner)
    lam_true = L.lam_max / 1.1
    mg = cf.CutFEMMG([cf.CutFEM(P)], inner=inner, eig_iters=40, eig_safety=1.0)
    lam = mg.lambdas()[0]
    assert 0.95 * lam_true <= lam <= lam_true * (1 + 1e-8), (lam, lam_true)


def test_pmg_pcg_converges_where_jacobi_stalls(cf, cutgen_mod):
    probs = problems(cutgen_mod, [1, 3], 12)
    ops = [cf.CutFEM(P) for P in probs]
    mg = cf.CutFEMMG(ops, inner="block", smooth_degree=4, eig_iters=20)
    b = ops[-1].rhs_const(1.0)
    x, h = mg.pcg(b, iters=200, tol=1e-8)
    assert h[-1] <= 1e-8 * float(b.norm()) and len(h) < 120, len(h)
    r = b - ops[-1].apply(x)
    assert float(r.norm()) <= 2e-8 * float(b.norm())
    _, hj = ops[-1].cg(b, iters=len(h) - 1, precond="jacobi")
    assert hj[-1] > 100 * h[-1]
