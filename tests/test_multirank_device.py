"""The multi-rank device data path on ONE GPU, through the in-process
loopback transport (pdg_loopback_create / pdg_sim_attach_loopback).

Two ranks (rank 0 and 1 of world 2, both on cuda:0) each build their half of
the problem (whole subdomains per rank), attach to one loopback group and are
driven from two threads, exactly as two processes would drive NCCL: per PCG
iteration the halo pack kernel + exchange into the halo tail, the p.q
all-reduce, the combined [r0 ; ||r||^2] all-reduce behind the speculative
restriction, the finish kernels, the redundant coarse solve and r.z
(paper_2512_19536_b200/csrc/cuda/comm.cu, sim.cu record_iteration). Checked
against world = 1 on the same device and against the CPU oracle: iterations
+-1, states within 1e-10 (north star; the rank partial sums only reorder
rounding).
"""
import threading

import numpy as np
import pytest

from tests.conftest import gpu_available

pytestmark = pytest.mark.gpu

CFG = dict(cells=2048, lloyd=5, degree=2, subdomains=16, coarse=-1, dt=0.01, T=0.05, tol=1e-8,
           sigma_white_l=1.0, sigma_white_n=0.2, sigma_grey_l=0.5, sigma_grey_n=0.5, fiber_random=True,
           stimulus=("strip", 2.0e4, 0.1, 1.0), initial=("constant", -85.0))


def _ranks(world, **kw):
    from paper_2512_19536_b200.simulation import LoopbackGroup, Simulation, SimulationConfig
    sims = [Simulation(SimulationConfig(**{**CFG, **kw}, rank=r, world=world, device=0)) for r in range(world)]
    g = LoopbackGroup(world)
    errs = []

    def attach(s):
        try:
            g.attach(s)
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)

    _parallel([lambda s=s: attach(s) for s in sims])
    assert not errs, errs
    return sims, g


def _parallel(fns):
    out = [None] * len(fns)
    errs = []

    def run(i):
        try:
            out[i] = fns[i]()
        except Exception as e:
            errs.append(e)

    th = [threading.Thread(target=run, args=(i,)) for i in range(len(fns))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.skipif(not gpu_available(), reason="needs a GPU")
@pytest.mark.parametrize("world", [2, 3])
def test_loopback_steps_match_single_rank_and_oracle(world):
    from paper_2512_19536_b200.simulation import Simulation, SimulationConfig
    from tests.oracle_binding import oracle_for
    sims, g = _ranks(world)
    one = Simulation(SimulationConfig(**CFG))
    orc, _ = oracle_for(SimulationConfig(**CFG))
    for _ in range(5):
        st = _parallel([s.step for s in sims])
        s1, so = one.step(), orc.step()
        its = {x.iterations for x in st}
        assert len(its) == 1, "all ranks stop after the same iteration"
        assert abs(st[0].iterations - so["iterations"]) <= 1
        assert abs(st[0].iterations - s1.iterations) <= 1
    parts = [s.state() for s in sims]
    U = sum(p[2] for p in parts)       # each rank fills its own cells, zeros elsewhere
    Y = sum(p[4] for p in parts)
    _, _, U1, _, Y1, _ = one.state()
    _, _, Uo, _, Yo, _ = orc.state()
    assert _rel(U, Uo) <= 1e-10 and _rel(Y[0], Yo[0]) <= 1e-10
    assert _rel(U, U1) <= 1e-10


@pytest.mark.skipif(not gpu_available(), reason="needs a GPU")
def test_loopback_operators_and_solve():
    from paper_2512_19536_b200 import _lib
    from paper_2512_19536_b200.simulation import Simulation, SimulationConfig
    sims, g = _ranks(2)
    one = Simulation(SimulationConfig(**CFG))
    n = one.dimension
    b = _lib.uniform_rhs(42, n)
    y = sum(_parallel([lambda s=s: s.apply_K(b) for s in sims]))
    assert _rel(y, one.apply_K(b)) <= 1e-13
    z = sum(_parallel([lambda s=s: s.apply_precond(b) for s in sims]))
    assert _rel(z, one.apply_precond(b)) <= 1e-12
    res = _parallel([lambda s=s: s.pcg_solve(b, 1e-10) for s in sims])
    x = sum(r[0] for r in res)
    x1, r1 = one.pcg_solve(b, 1e-10)
    assert res[0][1].iterations == res[1][1].iterations
    assert abs(res[0][1].iterations - r1.iterations) <= 1 and res[0][1].converged
    assert _rel(x, x1) <= 1e-10


@pytest.mark.skipif(not gpu_available(), reason="needs a GPU")
def test_loopback_attach_guards():
    from paper_2512_19536_b200._lib import PdgError
    from paper_2512_19536_b200.simulation import LoopbackGroup
    sims, g = _ranks(2)
    with pytest.raises(PdgError):  # a second transport would scale K0 by world again
        LoopbackGroup(2).attach(sims[0])
