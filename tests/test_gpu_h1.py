"""GPU parity of the H^1 (continuous Galerkin) operator (cutfem_h1_*) against
oracle/h1.py.  Tolerance: max-norm <= 1e-10 ||v||_inf and, per node, <= 1e-10
(|A||u|)_g (the A18 reading, with |A| from the oracle's absolute local matrices)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import Oracle  # noqa: E402
from oracle.h1 import TERM_H1, OracleH1, h1_numbering  # noqa: E402

TOL = 1e-10


@pytest.fixture(scope="module")
def cf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_07911_b200 as m
    m.load()
    return m


def h1_check(P, vg, u, mask=TERM_H1):
    O = OracleH1(P, term_mask=mask)
    vo = O.apply(u)
    ub = np.abs(u)[O.map]
    sb = O.dg.apply(ub.reshape(-1), absolute=True).reshape(ub.shape)
    scale = np.zeros(O.n_h1)
    np.add.at(scale, O.map.ravel(), sb.ravel())
    err = np.abs(vg - vo)
    assert err.max() <= TOL * np.abs(vo).max(), (err.max(), np.abs(vo).max())
    assert np.all(err <= TOL * np.maximum(scale, 1e-300)), (err / np.maximum(scale, 1e-300)).max()


def test_h1_numbering_matches_oracle(cf, cutgen_mod):
    for P in (cutgen_mod.config("C1"), cutgen_mod.generate(cutgen_mod.GYROID, 6, 0.0, 1.0, 3)):
        op = cf.CutFEMH1(P)
        n, m = h1_numbering(P)
        assert op.n_dofs == n and np.array_equal(op.map(), m.reshape(-1).astype(np.int32))


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_h1_sphere_all_degrees(cf, cutgen_mod, p):
    N = {1: 8, 2: 7, 3: 6, 4: 5, 5: 4, 6: 3, 7: 3, 8: 3}[p]
    P = cutgen_mod.generate(cutgen_mod.SPHERE, N, -1.0, 1.0, p)
    op = cf.CutFEMH1(P)
    u = np.random.default_rng(p).uniform(-1, 1, op.n_dofs)
    v = op.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    h1_check(P, v, u)


@pytest.mark.parametrize("mask", [1, 4, 8])
def test_h1_per_term(cf, cutgen_mod, mask):
    P = cutgen_mod.config("C1")
    op = cf.CutFEMH1(P, term_mask=mask)
    u = np.random.default_rng(mask).uniform(-1, 1, op.n_dofs)
    v = op.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    h1_check(P, v, u, mask)


def test_h1_gyroid_plane_and_sphere16(cf, cutgen_mod):
    for P in (cutgen_mod.generate(cutgen_mod.GYROID, 8, 0.0, 1.0, 2),
              cutgen_mod.generate({"type": "plane", "normal": [1, 0.3, 0.1], "offset": 0.13}, [5, 3, 2],
                                  [0, 0, 0], [1.0, 0.6, 0.4], 3),
              cutgen_mod.generate(cutgen_mod.SPHERE, 16, -1.0, 1.0, 3)):
        op = cf.CutFEMH1(P)
        u = np.random.default_rng(3).uniform(-1, 1, op.n_dofs)
        v = op.apply(torch.from_numpy(u).cuda()).cpu().numpy()
        h1_check(P, v, u)


def test_h1_rhs_symmetry_and_constants(cf, cutgen_mod):
    P = cutgen_mod.config("C1")
    op = cf.CutFEMH1(P)
    b = op.rhs_const(2.5).cpu().numpy()
    bo = OracleH1(P).rhs(lambda x: 2.5 * np.ones(len(x)))
    assert np.abs(b - bo).max() <= 1e-13 * np.abs(bo).max()
    u = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, op.n_dofs)).cuda()
    w = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, op.n_dofs)).cuda()
    a, c = float(w @ op.apply(u)), float(u @ op.apply(w))
    assert abs(a - c) <= 1e-12 * abs(a) * 10
    # away from the interface a continuous constant is in the kernel of A_CG
    P2 = cutgen_mod.generate({"type": "sphere", "center": [0, 0, 0], "radius": 10.0}, 4, -1.0, 1.0, 3)
    op2 = cf.CutFEMH1(P2)
    v1 = op2.apply(torch.ones(op2.n_dofs, dtype=torch.float64, device="cuda")).cpu().numpy()
    assert np.abs(v1).max() <= 1e-12


@pytest.mark.parametrize("cfg", ["C2"])
def test_h1_full_size_sampled(cf, cutgen_mod, cfg):
    """BASELINE configs[1] with the H1 space: sampled nodes against the oracle (the
    blocks around each sampled node, per node tolerance)."""
    P = cutgen_mod.config(cfg)
    op = cf.CutFEMH1(P)
    u = np.random.default_rng(5).uniform(-1, 1, op.n_dofs)
    v = op.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    m = op.map().reshape(P.n_active, -1)
    rng = np.random.default_rng(0)
    cut_blocks = np.where(P.is_cut.astype(bool))[0]
    nodes = set(rng.choice(op.n_dofs, 12, replace=False).tolist())
    nodes |= set(m[rng.choice(cut_blocks, 12, replace=False), 0].tolist())
    O = Oracle(P, term_mask=TERM_H1)
    for g in sorted(nodes):
        Ks, ls = np.where(m == g)
        blocks = sorted(set(Ks.tolist()))
        ub = u[m]
        vo = O.apply(ub.reshape(-1), blocks=blocks)
        so = O.apply(np.abs(ub).reshape(-1), blocks=blocks, absolute=True)
        ref = sum(vo[K][l] for K, l in zip(Ks, ls))
        sc = sum(so[K][l] for K, l in zip(Ks, ls))
        assert abs(v[g] - ref) <= TOL * sc, (g, v[g], ref, sc)
