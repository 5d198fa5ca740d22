"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Tolerance (BASELINE north_star): max-norm error <= 1e-10 * ||v||_inf, and per
block ||v_K^gpu - v_K^orc||_inf <= 1e-10 * ||(|A||u|)_K||_inf,
where |A||u| is formed by the oracle from the absolute values of its blocks.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import Oracle  # noqa: E402

FAR = {"type": "sphere", "center": [0.0, 0.0, 0.0], "radius": 10.0}
TOL = 1e-10


@pytest.fixture(scope="module")
def cf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_07911_b200 as m
    m.load()
    return m


def gpu_apply(cf, P, u, mask=15):
    op = cf.CutFEM(P, term_mask=mask)
    ud = torch.from_numpy(u).cuda()
    v = op.apply(ud)
    torch.cuda.synchronize()
    return v.cpu().numpy(), op


def check(P, v_gpu, u, mask=15, blocks=None):
    O = Oracle(P, term_mask=mask)
    nd = (P.degree + 1) ** 3
    if blocks is None:
        v_orc = O.apply(u)
        scale = O.apply(u, absolute=True).reshape(-1, nd)
        err = np.abs(v_gpu - v_orc)
        assert err.max() <= TOL * max(np.abs(v_orc).max(), 1e-300), (err.max(), np.abs(v_orc).max())
        eb = err.reshape(-1, nd).max(1)
        sb = scale.max(1)
        assert np.all(eb <= TOL * np.maximum(sb, 1e-300)), (eb / np.maximum(sb, 1e-300)).max()
        return err.max() / np.abs(v_orc).max()
    vo = O.apply(u, blocks=blocks)
    so = O.apply(u, blocks=blocks, absolute=True)
    vg = v_gpu.reshape(-1, nd)
    worst = 0.0
    for K in blocks:
        e = np.abs(vg[K] - vo[K]).max()
        assert e <= TOL * so[K].max(), (K, e, so[K].max())
        worst = max(worst, e / so[K].max())
    return worst


def test_c1_full_operator(cf, cutgen_mod):
    P = cutgen_mod.config("C1")
    for seed in (1, 2, 3):
        u = P.seeded_u(seed)
        v, _ = gpu_apply(cf, P, u)
        check(P, v, u)


@pytest.mark.parametrize("mask", [1, 2, 4, 8, 3, 12])
def test_c1_per_term(cf, cutgen_mod, mask):
    P = cutgen_mod.config("C1")
    u = P.seeded_u(1)
    v, _ = gpu_apply(cf, P, u, mask)
    check(P, v, u, mask)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_sphere_all_degrees(cf, cutgen_mod, p):
    N = {1: 8, 2: 7, 3: 6, 4: 5, 5: 5, 6: 5, 7: 5, 8: 5}[p]
    P = cutgen_mod.generate(cutgen_mod.SPHERE, N, -1.0, 1.0, p)
    assert P.n_cut > 0 and P.n_active > P.n_cut
    u = P.seeded_u(p)
    v, _ = gpu_apply(cf, P, u)
    check(P, v, u)
    for mask in ((1, 2, 4, 8) if p <= 5 else ()):
        v, _ = gpu_apply(cf, P, u, mask)
        check(P, v, u, mask)


@pytest.mark.parametrize("p", [1, 3, 5, 8])
def test_level_set_misses_mesh(cf, cutgen_mod, p):
    P = cutgen_mod.generate(FAR, 3 if p < 6 else 2, -1.0, 1.0, p)
    u = P.seeded_u(7)
    v, _ = gpu_apply(cf, P, u)
    check(P, v, u)
    # A 1 = 0 (standard SIPG annihilates constants)
    v1, _ = gpu_apply(cf, P, np.ones(P.n_dofs))
    assert np.abs(v1).max() <= 1e-12 * np.abs(v).max()


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_q10_tensor_rule_as_cut_rule(cf, cutgen_mod, p):
    """Every cell through the unstructured path with its tensor rule (and full
    faces as listed cut faces) equals the structured path (P:850 benchmark)."""
    Ps = cutgen_mod.generate(FAR, 3, -1.0, 1.0, p)
    Pu = cutgen_mod.generate(FAR, 3, -1.0, 1.0, p, force_cut_cells=True, force_cut_faces=True)
    assert Pu.n_cut == Pu.n_active and Pu.sf_cells.shape[0] > 0
    u = Ps.seeded_u(5)
    vs, _ = gpu_apply(cf, Ps, u, mask=1 | 2 | 4)
    vu, _ = gpu_apply(cf, Pu, u, mask=1 | 2 | 4)  # GP differs (all cells "cut"): excluded
    assert np.abs(vs - vu).max() <= 1e-11 * np.abs(vs).max()
    check(Pu, vu, u, mask=1 | 2 | 4)
    vall, _ = gpu_apply(cf, Pu, u)
    check(Pu, vall, u)


def test_gyroid_small(cf, cutgen_mod):
    P = cutgen_mod.generate(cutgen_mod.GYROID, 10, 0.0, 1.0, 2)
    assert P.n_cut > 0
    u = P.seeded_u(11)
    v, _ = gpu_apply(cf, P, u)
    check(P, v, u)


def test_plane_and_ragged(cf, cutgen_mod):
    P = cutgen_mod.generate({"type": "plane", "normal": [1, 0.3, 0.1], "offset": 0.13}, [5, 3, 2],
                            [0, 0, 0], [1.0, 0.6, 0.4], 3)
    u = P.seeded_u(2)
    v, _ = gpu_apply(cf, P, u)
    check(P, v, u)


def test_single_cell_and_empty(cf, cutgen_mod):
    P = cutgen_mod.generate(FAR, 1, 0.0, 1.0, 2)
    u = P.seeded_u(1)
    v, _ = gpu_apply(cf, P, u)
    check(P, v, u)
    E = cutgen_mod.generate({"type": "sphere", "center": [5, 5, 5], "radius": 0.1}, 2, 0.0, 1.0, 2)
    assert E.n_active == 0
    op = cf.CutFEM(E)
    assert op.stats()["n_dofs"] == 0
    op.apply(torch.zeros(0, dtype=torch.float64, device="cuda"), torch.zeros(0, dtype=torch.float64, device="cuda"))


def test_apply_host_matches_device(cf, cutgen_mod):
    P = cutgen_mod.config("C1")
    u = P.seeded_u(3)
    vd, op = gpu_apply(cf, P, u)
    vh = op.apply_host(u)
    assert np.array_equal(vd, vh)


def test_deterministic(cf, cutgen_mod):
    P = cutgen_mod.config("C1", degree=3)
    u = P.seeded_u(1)
    v1, op = gpu_apply(cf, P, u)
    v2 = op.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    assert np.array_equal(v1, v2)


def test_symmetry_gpu(cf, cutgen_mod):
    P = cutgen_mod.config("C1")
    op = cf.CutFEM(P)
    u = torch.from_numpy(P.seeded_u(1)).cuda()
    w = torch.from_numpy(P.seeded_u(2)).cuda()
    a = float(w @ op.apply(u))
    b = float(u @ op.apply(w))
    assert abs(a - b) <= 1e-12 * abs(a) * 10


def test_csr_assemble_matches_oracle(cf, cutgen_mod):
    P = cutgen_mod.config("C1")
    op = cf.CutFEM(P)
    nnz = op.csr_assemble()
    u = P.seeded_u(4)
    ud = torch.from_numpy(u).cuda()
    vc = op.csr_apply(ud).cpu().numpy()
    vm = op.apply(ud).cpu().numpy()
    O = Oracle(P)
    M = O.assemble_csr()
    vo = M @ u
    assert np.abs(vc - vo).max() <= 1e-10 * np.abs(vo).max()
    assert np.abs(vc - vm).max() <= 1e-12 * np.abs(vm).max()
    rp, col, val = op.csr_download()
    G = __import__("scipy.sparse", fromlist=["csr_matrix"]).csr_matrix((val, col, rp), shape=M.shape)
    assert abs(G - M).max() <= 1e-10 * abs(M).max()
    assert nnz >= M.nnz


def test_csr_setup_from_oracle(cf, cutgen_mod):
    P = cutgen_mod.config("C1")
    op = cf.CutFEM(P)
    M = Oracle(P).assemble_csr()
    op.csr_setup(M.indptr.astype(np.int64), M.indices, M.data)
    u = P.seeded_u(8)
    vc = op.csr_apply(torch.from_numpy(u).cuda()).cpu().numpy()
    assert np.abs(vc - M @ u).max() <= 1e-13 * np.abs(M @ u).max()


def test_invalid_inputs(cf, cutgen_mod):
    P = cutgen_mod.config("C1")
    bad = cutgen_mod.config("C1")
    bad.vol_pts = bad.vol_pts.copy()
    bad.vol_pts[0, 0] = 1.5
    with pytest.raises(RuntimeError, match="outside"):
        cf.CutFEM(bad)
    bad = cutgen_mod.config("C1")
    bad.degree = 9
    with pytest.raises(RuntimeError):
        cf.CutFEM(bad)
    op = cf.CutFEM(P)
    u = torch.zeros(P.n_dofs, dtype=torch.float64, device="cuda")
    with pytest.raises(RuntimeError, match="alias"):
        op.apply(u, u)


@pytest.mark.parametrize("cfg", ["C2"])
def test_full_size_sampled_blocks(cf, cutgen_mod, cfg):
    """BASELINE configs[1] at full size: sampled output blocks vs the oracle."""
    P = cutgen_mod.config(cfg)
    u = P.seeded_u(1)
    v, _ = gpu_apply(cf, P, u)
    rng = np.random.default_rng(0)
    cut = np.where(P.is_cut)[0]
    unc = np.where(~P.is_cut.astype(bool))[0]
    blocks = list(rng.choice(cut, 24, replace=False)) + list(rng.choice(unc, 24, replace=False))
    check(P, v, u, blocks=blocks)
    # a property at any size: symmetry
    op = cf.CutFEM(P)
    ud = torch.from_numpy(u).cuda()
    wd = torch.from_numpy(P.seeded_u(2)).cuda()
    a, b = float(wd @ op.apply(ud)), float(ud @ op.apply(wd))
    assert abs(a - b) <= 1e-11 * abs(a)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_sphere16_tiles(cf, cutgen_mod, p):
    """A mesh with many warp-tiles (full and partial bricks, plain cells, ghost-
    penalty cells, cut cells with structured faces): whole operator and the
    face terms alone."""
    P = cutgen_mod.generate(cutgen_mod.SPHERE, 16, -1.0, 1.0, p)
    u = P.seeded_u(10 + p)
    v, op = gpu_apply(cf, P, u)
    assert op.stats()["n_uncut"] > 400
    check(P, v, u)
    for mask in (2, 8):
        v, _ = gpu_apply(cf, P, u, mask)
        check(P, v, u, mask)


@pytest.mark.parametrize("p", [2, 3])
def test_gyroid_box_boundary(cf, cutgen_mod, p):
    """Gyroid in [0,1]^3: uncut cells on the box boundary (missing faces)."""
    P = cutgen_mod.generate(cutgen_mod.GYROID, 8, 0.0, 1.0, p)
    u = P.seeded_u(21)
    v, _ = gpu_apply(cf, P, u)
    check(P, v, u)


@pytest.mark.parametrize("cfg", ["C1", "gyroid"])
def test_rhs_const_matches_oracle(cf, cutgen_mod, cfg):
    """b = f int_Omega phi_i vs the oracle's quadrature sum."""
    P = cutgen_mod.config("C1") if cfg == "C1" else cutgen_mod.generate(cutgen_mod.GYROID, 8, 0.0, 1.0, 3)
    op = cf.CutFEM(P)
    b = op.rhs_const(2.5).cpu().numpy()
    bo = Oracle(P).rhs(lambda x: 2.5 * np.ones(len(x)))
    assert np.abs(b - bo).max() <= 1e-13 * np.abs(bo).max()
    # sum of b = f |Omega| (partition of unity); cross-check with the volume weights
    vol = P.vol_pts[:, 3].sum() + P.h ** 3 * (P.n_active - P.n_cut)
    assert abs(b.sum() - 2.5 * vol) <= 1e-12 * 2.5 * vol


def test_cg_matches_oracle_cg(cf, cutgen_mod):
    """30 unpreconditioned CG iterations in the library's kernels vs the oracle's
    CG on its own operator: the same iterates up to rounding growth."""
    from oracle.operator import cg as oracle_cg
    P = cutgen_mod.config("C1")
    op = cf.CutFEM(P)
    O = Oracle(P)
    bo = O.rhs(lambda x: np.ones(len(x)))  # the oracle's RHS feeds both sides
    b = torch.from_numpy(bo).cuda()
    x, hist = op.cg(b, iters=30)
    xo, it = oracle_cg(O.apply, bo, tol=0.0, maxiter=30)
    assert len(hist) == 31 and it == 30
    xg = x.cpu().numpy()
    assert np.abs(xg - xo).max() <= 1e-8 * np.abs(xo).max()
    r = b - op.apply(x)
    assert abs(float(r.norm()) - hist[-1]) <= 1e-8 * hist[0]


def test_cg_tolerance_stop(cf, cutgen_mod):
    P = cutgen_mod.config("C1")
    op = cf.CutFEM(P)
    b = op.rhs_const(1.0)
    x, hist = op.cg(b, iters=2000, tol=1e-9)
    assert hist[-1] <= 1e-9 * float(b.norm()) and len(hist) < 2001
    assert float((b - op.apply(x)).norm()) <= 1e-8 * float(b.norm())


@pytest.mark.parametrize("p,N", [(4, 10), (5, 9), (6, 8)])
def test_sphere_high_degree_tiles(cf, cutgen_mod, p, N):
    """k_uncw (p = 4, 5) and k_uncut (p = 6): several tiles of uncut cells, plain and
    next to cut cells."""
    P = cutgen_mod.generate(cutgen_mod.SPHERE, N, -1.0, 1.0, p)
    u = P.seeded_u(30 + p)
    v, op = gpu_apply(cf, P, u)
    assert op.stats()["n_uncut"] > 30
    check(P, v, u)
    v, _ = gpu_apply(cf, P, u, 8)
    check(P, v, u, 8)
