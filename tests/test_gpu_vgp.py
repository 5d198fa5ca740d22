"""GPU parity of the volume ghost penalty (gp_kind = 1, stable-neighbour patches;
PAPER eq:volume_based_gp P:96-108) through every kernel family, DG and H1."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from test_gpu_h1 import h1_check  # noqa: E402
from test_gpu_parity import check, gpu_apply  # noqa: E402


@pytest.fixture(scope="module")
def cf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_07911_b200 as m
    m.load()
    return m


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_vgp_sphere_all_degrees(cf, cutgen_mod, p):
    N = {1: 8, 2: 7, 3: 6, 4: 5, 5: 5, 6: 4, 7: 4, 8: 4}[p]
    P = cutgen_mod.generate(cutgen_mod.SPHERE, N, -1.0, 1.0, p, gp_kind=1, tau_v=1.0)
    u = P.seeded_u(60 + p)
    v, _ = gpu_apply(cf, P, u)
    check(P, v, u)
    v, _ = gpu_apply(cf, P, u, 8)
    check(P, v, u, 8)


@pytest.mark.parametrize("p", [2, 3])
def test_vgp_multi_tile_and_gyroid(cf, cutgen_mod, p):
    for P in (cutgen_mod.generate(cutgen_mod.SPHERE, 16, -1.0, 1.0, p, gp_kind=1, tau_v=0.5),
              cutgen_mod.generate(cutgen_mod.GYROID, 8, 0.0, 1.0, p, gp_kind=1, tau_v=1.0)):
        u = P.seeded_u(70 + p)
        v, _ = gpu_apply(cf, P, u)
        check(P, v, u)


def test_vgp_h1(cf, cutgen_mod):
    P = cutgen_mod.generate(cutgen_mod.SPHERE, 7, -1.0, 1.0, 2, gp_kind=1, tau_v=1.0)
    op = cf.CutFEMH1(P)
    u = np.random.default_rng(9).uniform(-1, 1, op.n_dofs)
    v = op.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    h1_check(P, v, u)


def test_vgp_c2_sampled(cf, cutgen_mod):
    P = cutgen_mod.config("C2", gp_kind=1, tau_v=1.0)
    u = P.seeded_u(1)
    v, _ = gpu_apply(cf, P, u)
    rng = np.random.default_rng(3)
    cut = np.where(P.is_cut.astype(bool))[0]
    unc = np.where(~P.is_cut.astype(bool))[0]
    check(P, v, u, blocks=sorted(set(rng.choice(cut, 16, replace=False).tolist())
                                  | set(rng.choice(unc, 16, replace=False).tolist())))


def test_vgp_rejected_on_distributed_handle(cf, cutgen_mod):
    P = cutgen_mod.generate(cutgen_mod.SPHERE, 10, -1.0, 1.0, 2, gp_kind=1)
    xs = cf.partition_x(P, 2, 7.0)
    with pytest.raises(RuntimeError, match="distributed"):
        cf.CutFEMDist(P, xs[0], xs[1])
