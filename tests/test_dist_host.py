"""x-slab partition and halo logic of the distributed path (host side, CPU only).

The local problems come from the C library's host builder (cutfem_local_build,
the same code cutfem_setup_dist uses); the ghost planes are exchanged exactly as
the NCCL halo does (owned first plane -> rank-1's ghost_hi, owned last plane ->
rank+1's ghost_lo), here over gloo with world_size 2; each rank applies the CPU
oracle to its local problem and the owned rows must equal the global apply.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import cutgen
from oracle import Oracle


def _lib():
    import paper_2404_07911_b200 as m
    m.build()
    return m


def test_partition_covers_and_balances():
    m = _lib()
    P = cutgen.config("C1", degree=2)
    for parts in (1, 2, 3, 4):
        xs = m.partition_x(P, parts, 7.0)
        assert xs[0] == 0 and xs[-1] == P.n_cells[0] and all(a < b for a, b in zip(xs, xs[1:]))
    P = cutgen.generate(cutgen.SPHERE, 32, -1.0, 1.0, 1)
    xs = m.partition_x(P, 4, 7.0)
    w = np.zeros(32)
    np.add.at(w, P.active_ijk[:, 0], np.where(P.is_cut, 7.0, 1.0))
    parts = [w[a:b].sum() for a, b in zip(xs, xs[1:])]
    assert max(parts) <= 1.25 * sum(parts) / 4


def test_local_problem_structure():
    m = _lib()
    P = cutgen.config("C1", degree=2)
    xs = m.partition_x(P, 3, 7.0)
    owned = 0
    for r in range(3):
        L = m.LocalProblem(P, xs[r], xs[r + 1])
        owned += L.n_own
        assert np.array_equal(L.active_ijk[:L.n_own], P.active_ijk[L.global_begin:L.global_begin + L.n_own])
        assert np.all(L.active_ijk[L.n_own:L.n_own + L.n_ghost_lo, 0] == xs[r] - 1)
        assert np.all(L.active_ijk[L.n_own + L.n_ghost_lo:, 0] == xs[r + 1])
        if r > 0:
            prev = m.LocalProblem(P, xs[r - 1], xs[r])
            assert prev.plane_hi == L.n_ghost_lo
            assert L.plane_lo == prev.n_ghost_hi
    assert owned == P.n_active


def _worker(rank, world, port, xs, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = _lib()
        P = cutgen.config("C1", degree=2)
        L = m.LocalProblem(P, xs[rank], xs[rank + 1])
        nd = (P.degree + 1) ** 3
        u = P.seeded_u(3).reshape(-1, nd)
        ue = np.zeros((L.n_active, nd))
        ue[:L.n_own] = u[L.global_begin:L.global_begin + L.n_own]
        # the halo, in the order of the NCCL exchange
        reqs = []
        if rank > 0:
            reqs.append(dist.isend(torch.from_numpy(ue[:L.plane_lo].copy()), rank - 1))
            lo = torch.zeros(L.n_ghost_lo, nd, dtype=torch.float64)
            dist.recv(lo, rank - 1)
            ue[L.n_own:L.n_own + L.n_ghost_lo] = lo.numpy()
        if rank < world - 1:
            reqs.append(dist.isend(torch.from_numpy(ue[L.n_own - L.plane_hi:L.n_own].copy()), rank + 1))
            hi = torch.zeros(L.n_ghost_hi, nd, dtype=torch.float64)
            dist.recv(hi, rank + 1)
            ue[L.n_own + L.n_ghost_lo:] = hi.numpy()
        for r in reqs:
            r.wait()
        v = Oracle(L).apply(ue.reshape(-1)).reshape(-1, nd)[:L.n_own]
        q.put((rank, L.global_begin, v))
    finally:
        dist.destroy_process_group()


def test_two_rank_halo_matches_global_apply():
    m = _lib()
    P = cutgen.config("C1", degree=2)
    xs = m.partition_x(P, 2, 7.0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, xs, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    nd = (P.degree + 1) ** 3
    v = np.zeros((P.n_active, nd))
    for rank, g0, vr in res:
        v[g0:g0 + vr.shape[0]] = vr
    vg = Oracle(P).apply(P.seeded_u(3)).reshape(-1, nd)
    assert np.abs(v - vg).max() <= 1e-12 * np.abs(vg).max()
