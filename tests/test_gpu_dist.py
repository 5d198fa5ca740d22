"""GPU checks of the x-slab distributed handle (one GPU: no rank waits on another).

- a single slab covering the mesh equals the plain apply bit for bit;
- two slabs, each its own handle (nranks = 1), with the ghost planes filled from
  the global vector as the NCCL halo would, reproduce the global apply exactly
  (every cell's arithmetic is the same) -- this exercises the interior/boundary
  launch split and the ghost indexing on the device.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cf():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2404_07911_b200 as m
    m.load()
    return m


@pytest.mark.parametrize("p", [2, 3])
def test_single_slab_equals_plain(cf, cutgen_mod, p):
    P = cutgen_mod.generate(cutgen_mod.SPHERE, 10, -1.0, 1.0, p)
    u = torch.from_numpy(P.seeded_u(1)).cuda()
    v0 = cf.CutFEM(P).apply(u)
    d = cf.CutFEMDist(P, 0, P.n_cells[0])
    assert d.n_ghost_lo == 0 and d.n_ghost_hi == 0
    v1 = d.apply(u)
    torch.cuda.synchronize()
    assert torch.equal(v0, v1)


@pytest.mark.parametrize("p,nparts", [(2, 2), (3, 3), (1, 4), (5, 2), (7, 2)])
def test_slabs_with_emulated_halo(cf, cutgen_mod, p, nparts):
    P = cutgen_mod.generate(cutgen_mod.SPHERE, 12, -1.0, 1.0, p)
    nd = (p + 1) ** 3
    ug = P.seeded_u(2).reshape(-1, nd)
    vg = cf.CutFEM(P).apply(torch.from_numpy(ug.reshape(-1)).cuda()).cpu().numpy().reshape(-1, nd)
    xs = cf.partition_x(P, nparts, 7.0)
    out = np.zeros_like(vg)
    for r in range(nparts):
        L = cf.LocalProblem(P, xs[r], xs[r + 1])
        d = cf.CutFEMDist(P, xs[r], xs[r + 1])
        ue = np.zeros((L.n_active, nd))
        ue[:L.n_own] = ug[L.global_begin:L.global_begin + L.n_own]
        lo0 = L.global_begin - L.n_ghost_lo
        ue[L.n_own:L.n_own + L.n_ghost_lo] = ug[lo0:L.global_begin]
        hi0 = L.global_begin + L.n_own
        ue[L.n_own + L.n_ghost_lo:] = ug[hi0:hi0 + L.n_ghost_hi]
        v = d.apply(torch.from_numpy(ue.reshape(-1)).cuda()).cpu().numpy().reshape(-1, nd)
        out[L.global_begin:L.global_begin + L.n_own] = v
    assert np.array_equal(out, vg)
