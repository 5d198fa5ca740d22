"""GPU checks of the preconditioned solve (Jacobi-PCG around the
matrix-free operator, DG and H1) against the oracle.

* the probed diagonal equals the oracle CSR's diagonal (DG: checkerboard probing;
  H1: lattice mod (2p+1) probing);
* PCG iterates equal the oracle's PCG (oracle.operator.cg with M = 1/diag) up to
  rounding growth;
* after the same number of iterations the Jacobi residual is below the plain one
  (the point of a preconditioner) and the reported residual is the true one;
* the H1 solve of the manufactured problem reaches the oracle's direct-solve error.
"""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import Oracle  # noqa: E402
from oracle.h1 import OracleH1  # noqa: E402
from oracle.operator import cg as oracle_cg  # noqa: E402


@pytest.fixture(scope="module")
def cf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_07911_b200 as m
    m.load()
    return m


@pytest.mark.parametrize("p", [1, 2, 3, 5])
def test_dg_diag_matches_oracle(cf, cutgen_mod, p):
    P = cutgen_mod.generate(cutgen_mod.SPHERE, {1: 8, 2: 7, 3: 6, 5: 4}[p], -1.0, 1.0, p)
    d = cf.CutFEM(P).diag().cpu().numpy()
    do = Oracle(P).assemble_csr().diagonal()
    assert np.abs(d - do).max() <= 1e-11 * np.abs(do).max()


@pytest.mark.parametrize("p", [1, 2, 3])
def test_h1_diag_matches_oracle(cf, cutgen_mod, p):
    P = cutgen_mod.generate(cutgen_mod.SPHERE, {1: 8, 2: 7, 3: 6}[p], -1.0, 1.0, p)
    d = cf.CutFEMH1(P).diag().cpu().numpy()
    do = OracleH1(P).assemble_csr().diagonal()
    assert np.abs(d - do).max() <= 1e-11 * np.abs(do).max()


def test_dg_jacobi_pcg_matches_oracle(cf, cutgen_mod):
    P = cutgen_mod.config("C1")
    op = cf.CutFEM(P)
    O = Oracle(P)
    bo = O.rhs(lambda x: np.ones(len(x)))  # the oracle's RHS feeds both sides
    b = torch.from_numpy(bo).cuda()
    x, hist = op.cg(b, iters=30, precond="jacobi")
    M = O.assemble_csr()
    xo, it = oracle_cg(lambda y: M @ y, bo, tol=0.0, maxiter=30, M=1.0 / M.diagonal())
    assert it == 30 and len(hist) == 31
    assert np.abs(x.cpu().numpy() - xo).max() <= 1e-8 * np.abs(xo).max()
    r = b - op.apply(x)
    assert abs(float(r.norm()) - hist[-1]) <= 1e-8 * hist[0]


def test_dg_jacobi_reduces_residual_faster(cf, cutgen_mod):
    """After the same number of iterations the Jacobi-preconditioned residual is
    smaller than the plain one (C1 and a 12^3 p = 3 sphere)."""
    for P in (cutgen_mod.config("C1"), cutgen_mod.generate(cutgen_mod.SPHERE, 12, -1.0, 1.0, 3)):
        op = cf.CutFEM(P)
        b = op.rhs_const(1.0)
        _, h0 = op.cg(b, iters=300)
        x1, h1 = op.cg(b, iters=300, precond="jacobi")
        assert h1[-1] < h0[-1], (h1[-1], h0[-1])
        assert abs(float((b - op.apply(x1)).norm()) - h1[-1]) <= 1e-8 * h1[0]


def test_h1_pcg_matches_oracle_and_converges(cf, cutgen_mod):
    P = cutgen_mod.config("C1")
    op = cf.CutFEMH1(P)
    O = OracleH1(P)
    bo = O.rhs(lambda x: np.ones(len(x)))  # the oracle's RHS feeds both sides
    b = torch.from_numpy(bo).cuda()
    x, hist = op.cg(b, iters=25, precond="jacobi")
    M = O.assemble_csr()
    xo, _ = oracle_cg(lambda y: M @ y, bo, tol=0.0, maxiter=25, M=1.0 / M.diagonal())
    assert np.abs(x.cpu().numpy() - xo).max() <= 1e-8 * np.abs(xo).max()
    x2, h2 = op.cg(b, iters=3000, tol=1e-10, precond="jacobi")
    assert h2[-1] <= 1e-10 * float(b.norm())


def test_h1_manufactured_solution(cf, cutgen_mod):
    """H1 p = 2 on 12^3: the GPU Jacobi-PCG solution has the oracle's direct-solve
    L2 error (same discrete problem), and the RHS is the oracle's."""
    import scipy.sparse.linalg as spl
    R, om, p, N = 0.7, math.pi, 2, 12
    c = np.array(cutgen_mod.SPHERE["center"])
    P = cutgen_mod.generate(cutgen_mod.SPHERE, N, -1.0, 1.0, p)
    O = OracleH1(P)
    rr = lambda x: np.linalg.norm(x - c, axis=-1)  # noqa: E731
    f = lambda x: -om ** 2 * (np.cos(om * rr(x)) + 2 * np.sinc(om * rr(x) / math.pi))  # noqa: E731
    uex = lambda x: math.cos(om * R) - np.cos(om * rr(x))  # noqa: E731
    b = O.rhs(f)
    xo = spl.spsolve(O.assemble_csr().tocsc(), b)
    op = cf.CutFEMH1(P)
    x, hist = op.cg(torch.from_numpy(b).cuda(), iters=5000, tol=1e-11, precond="jacobi")
    e_gpu, e_orc = O.l2_error(x.cpu().numpy(), uex), O.l2_error(xo, uex)
    assert abs(e_gpu - e_orc) <= 1e-6 * e_orc, (e_gpu, e_orc)
