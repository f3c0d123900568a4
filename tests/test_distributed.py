"""Multi-rank host logic, world_size 2 over gloo on CPU (no GPU needed).

The device path shards subdomains over ranks (one process per GPU) and does
per PCG iteration: a p-halo exchange (grouped NCCL send/recv), all-reduces of
the dot products and an all-reduce of the coarse residual r0, then solves K0
redundantly (paper_2512_19536_b200/csrc/cuda/comm.cu). These tests check the
host-side plan every rank computes independently (cell ranges, halo lists,
local rows, K0 partial sums) and run the same distributed PCG algorithm with
gloo collectives and exact local solves, against the single-process oracle.
"""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spl
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2
CFG = dict(cells=1024, lloyd=5, degree=2, subdomains=16, coarse=-1, chi_m=1.0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _local_problem(rank, world):
    from paper_2512_19536_b200.simulation import Problem, SimulationConfig
    return Problem(SimulationConfig(**CFG, rank=rank, world=world))


def _halo(P, peer):
    import ctypes as C
    from paper_2512_19536_b200 import _lib
    cnt = (C.c_int * 2)()
    _lib.lib().pdg_problem_halo(P._h, peer, None, None, cnt)
    s = np.zeros(cnt[0], np.int32)
    r = np.zeros(cnt[1], np.int32)
    _lib.lib().pdg_problem_halo(P._h, peer, _lib.iptr(s), _lib.iptr(r), cnt)
    return s, r


def _starts(P, world):
    from paper_2512_19536_b200 import _lib
    st = np.zeros(world + 1, np.int32)
    _lib.lib().pdg_problem_rank_cells(P._h, _lib.iptr(st))
    return st


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    os.environ.setdefault("POLYDG_THREADS", "2")
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        P = _local_problem(rank, world)
        st = _starts(P, world)
        perm = P.perm()
        b, N = P.n_local, P.n_cells
        lo, hi = st[rank], st[rank + 1]
        res["range"] = (int(lo), int(hi), int(P.cell_begin), int(P.cell_end))
        # halo lists (global internal cell ids)
        halo = {}
        for peer in range(world):
            if peer == rank:
                continue
            s, r = _halo(P, peer)
            halo[peer] = (s + lo, r)
        gathered = [None] * world
        dist.all_gather_object(gathered, {k: (v[0].tolist(), v[1].tolist()) for k, v in halo.items()})
        ok = True
        for peer in range(world):
            if peer == rank:
                continue
            # what I receive from peer == what peer sends to me
            ok &= gathered[peer][rank][0] == halo[peer][1].tolist()
        res["halo_consistent"] = bool(ok)
        # local rows of K, in reference dof order
        K_loc = P.export("K")
        my_dofs = (perm[lo:hi, None] * b + np.arange(b)).ravel()
        rows_present = np.unique(K_loc.nonzero()[0])
        res["rows_are_mine"] = bool(np.array_equal(np.sort(rows_present), np.sort(my_dofs)))
        # K0 partials summed over ranks
        K0p = P.export("K0").toarray()
        import torch
        t = torch.from_numpy(K0p.copy())
        dist.all_reduce(t)
        K0 = t.numpy()
        res["K0"] = K0 if rank == 0 else None
        # ---- distributed PCG (same algorithm as the NCCL path) ----
        E_loc = P.export("E")                   # local rows of E (n x coarse)
        sub = P.owner("subdomain")
        my_cells = perm[lo:hi]
        rng = np.random.default_rng(7)
        bvec = rng.uniform(-1, 1, N * b)         # every rank draws the same RHS
        n = N * b
        mask = np.zeros(n, bool)
        mask[my_dofs] = True

        def exchange(v_local_full):
            """v has my dofs filled; pull halo dofs from peers (send/recv)."""
            v = v_local_full.copy()
            for peer in range(world):
                if peer == rank:
                    continue
                send_cells, recv_cells = halo[peer]
                sd = (perm[send_cells][:, None] * b + np.arange(b)).ravel()
                rd = (perm[recv_cells][:, None] * b + np.arange(b)).ravel()
                sbuf = torch.from_numpy(v[sd].copy())
                rbuf = torch.zeros(len(rd), dtype=torch.float64)
                reqs = [dist.isend(sbuf, peer), dist.irecv(rbuf, peer)]
                for q in reqs:
                    q.wait()
                v[rd] = rbuf.numpy()
            return v

        def allsum(x):
            t = torch.tensor([x], dtype=torch.float64)
            dist.all_reduce(t)
            return float(t.item())

        K0f = sp.csc_matrix(K0)
        locals_ = {}
        for s in np.unique(sub[my_cells]):
            cells = np.nonzero(sub == s)[0]
            d = (cells[:, None] * b + np.arange(b)).ravel()
            locals_[s] = (d, spl.splu(K_loc[d][:, d].tocsc()))

        def precond(r):
            z = np.zeros(n)
            for d, lu in locals_.values():
                z[d] = lu.solve(r[d])
            r0 = torch.from_numpy(E_loc.T @ r)
            dist.all_reduce(r0)
            z += E_loc @ spl.spsolve(K0f, r0.numpy())
            z[~mask] = 0.0
            return z

        x = np.zeros(n)
        r = np.where(mask, bvec, 0.0)
        denom = np.sqrt(allsum(r @ r))
        z = precond(r)
        p = z.copy()
        rho = allsum(r @ z)
        it = 0
        for it in range(1, 500):
            q = np.where(mask, K_loc @ exchange(p), 0.0)
            alpha = rho / allsum(p @ q)
            x += alpha * p
            r -= alpha * q
            if np.sqrt(allsum(r @ r)) / denom < 1e-10:
                break
            z = precond(r)
            rho_new = allsum(r @ z)
            p = z + (rho_new / rho) * p
            rho = rho_new
        xs = torch.from_numpy(x)
        dist.all_reduce(xs)
        res["pcg"] = (it, xs.numpy() if rank == 0 else None)
        out[rank] = res
    finally:
        dist.destroy_process_group()


@pytest.fixture(scope="module")
def results():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(WORLD, port, out), nprocs=WORLD, join=True)
    return dict(out)


def test_rank_ranges_partition_cells(results):
    ranges = sorted(results[r]["range"] for r in range(WORLD))
    assert ranges[0][0] == 0 and ranges[-1][1] == CFG["cells"]
    for a, b2 in zip(ranges, ranges[1:]):
        assert a[1] == b2[0]
    for r in range(WORLD):
        lo, hi, cb, ce = results[r]["range"]
        assert (lo, hi) == (cb, ce)


def test_halo_lists_agree_between_ranks(results):
    assert all(results[r]["halo_consistent"] for r in range(WORLD))


def test_each_rank_assembles_only_its_rows(results):
    assert all(results[r]["rows_are_mine"] for r in range(WORLD))


def test_k0_partials_sum_to_single_rank_k0(results):
    from paper_2512_19536_b200.simulation import Problem, SimulationConfig
    K0 = Problem(SimulationConfig(**CFG)).export("K0").toarray()
    assert np.abs(results[0]["K0"] - K0).max() <= 1e-12 * np.abs(K0).max()


def test_distributed_pcg_matches_oracle(results):
    from paper_2512_19536_b200.simulation import SimulationConfig
    from tests.oracle_binding import oracle_for
    orc, _ = oracle_for(SimulationConfig(**CFG))
    bvec = np.random.default_rng(7).uniform(-1, 1, orc.dimension)
    xo, ro = orc.pcg_solve(bvec, 1e-10)
    it, x = results[0]["pcg"]
    assert abs(it - ro["iterations"]) <= 1
    assert np.linalg.norm(x - xo) <= 1e-9 * np.linalg.norm(xo)
