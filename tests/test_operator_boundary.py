"""The reference's operator-level construction from caller data.

SparseOperator(K) (krylov.hpp:22-30), SchwarzPreconditioner(K, space,
partition_S, coarse) (schwarz.hpp:51-53), build_coarse_embedding (schwarz.hpp:38-39)
and pcg_solve (krylov.hpp:49-51) with K, the subdomain partition and E handed
over by the caller (pdg_sim_create_from_operator). The GPU tests build K, the
partitions and E with the CPU oracle and check the device operators and PCG
against the oracle's on the same inputs; the preconditioner uses the product's
own graph-only ordering, so z agrees to rounding (1e-10), iterations +-1.
"""
import ctypes as C

import numpy as np
import pytest

from tests.conftest import gpu_available


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_operator_entry_points_exported():
    from paper_2512_19536_b200 import _lib
    L = _lib.lib()
    for name in ("pdg_sim_create_from_operator", "pdg_mesh_coarse_embedding"):
        assert hasattr(L, name)


def test_coarse_embedding_matches_problem_E():
    """build_coarse_embedding on the mesh == the E the simulation setup forms."""
    from paper_2512_19536_b200.mesh import Mesh
    from paper_2512_19536_b200.simulation import Problem, SimulationConfig
    m = Mesh(256, lloyd=5)
    own, cnt, _ = m.agglomerate(8)
    E = m.coarse_embedding(2, own, cnt, 2)
    P = Problem(SimulationConfig(cells=256, lloyd=5, degree=2, subdomains=8, coarse=-1))
    assert abs(E - P.export("E")).max() == 0.0
    from paper_2512_19536_b200._lib import PdgError
    with pytest.raises(PdgError, match="q must lie"):
        m.coarse_embedding(2, own, cnt, 3)


@pytest.mark.skipif(gpu_available(), reason="checks the no-device failure")
def test_operator_solver_fails_loudly_without_gpu():
    import scipy.sparse as sp
    from paper_2512_19536_b200._lib import PdgError
    from paper_2512_19536_b200.simulation import Simulation
    with pytest.raises(PdgError, match="CudaError"):
        Simulation.from_operator(sp.identity(6, format="csr"), 3, precond="none")


def _oracle_inputs(cells, degree, subdomains):
    from paper_2512_19536_b200.simulation import SimulationConfig
    from tests.oracle_binding import oracle_for
    cfg = SimulationConfig(cells=cells, lloyd=5, degree=degree, subdomains=subdomains, coarse=-1,
                           fiber_random=True)
    orc, extra = oracle_for(cfg)
    return cfg, orc


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a GPU")
@pytest.mark.parametrize("cells,degree,subdomains", [(256, 2, 8), (1024, 3, 16)])
def test_operator_solver_matches_oracle(cells, degree, subdomains):
    from paper_2512_19536_b200.mesh import Mesh
    from paper_2512_19536_b200.simulation import Simulation
    cfg, orc = _oracle_inputs(cells, degree, subdomains)
    K = orc.export("K")
    m = Mesh(cells, lloyd=5)
    own, cnt, _ = m.agglomerate(subdomains)
    b = (degree + 1) * (degree + 2) // 2
    E = m.coarse_embedding(degree, own, cnt, degree)
    sim = Simulation.from_operator(K, b, "two-level", partition=(own, cnt), coarse=(E, cnt, b))
    assert sim.dimension == K.shape[0]
    x = np.random.default_rng(1).uniform(-1, 1, sim.dimension)
    assert _rel(sim.apply_K(x), K @ x) <= 1e-12
    assert _rel(sim.apply_precond(x), orc.apply_precond(x)) <= 1e-10
    xs, rep = sim.pcg_solve(x, 1e-10)
    xo, ro = orc.pcg_solve(x, 1e-10)
    assert rep.converged and abs(rep.iterations - ro["iterations"]) <= 1
    assert _rel(xs, xo) <= 1e-10
    # no time stepper on an operator-built solver (ConfigError, not a crash)
    from paper_2512_19536_b200._lib import PdgError
    with pytest.raises(PdgError, match="ConfigError"):
        sim.step()


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a GPU")
def test_operator_solver_one_level_and_plain_cg():
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl
    from paper_2512_19536_b200.mesh import Mesh
    from paper_2512_19536_b200.simulation import Simulation
    cfg, orc = _oracle_inputs(256, 1, 8)
    K = orc.export("K")
    own, cnt, _ = Mesh(256, lloyd=5).agglomerate(8)
    r = np.random.default_rng(2).uniform(-1, 1, K.shape[0])
    # one-level Schwarz: z = sum_i R_i^T K_i^{-1} R_i r (schwarz.cpp:152-164)
    sim = Simulation.from_operator(K, 3, "block-jacobi", partition=(own, cnt))
    z = np.zeros_like(r)
    for s in range(cnt):
        d = (np.nonzero(own == s)[0][:, None] * 3 + np.arange(3)).ravel()
        z[d] = spl.spsolve(sp.csc_matrix(K[d][:, d]), r[d])
    assert _rel(sim.apply_precond(r), z) <= 1e-10
    # element block Jacobi (no partition) and plain CG (no preconditioner)
    bj = Simulation.from_operator(K, 3, "block-jacobi")
    assert bj.pcg_solve(r, 1e-8)[1].converged
    cg = Simulation.from_operator(K, 3, "none")
    x, rep = cg.pcg_solve(r, 1e-10, use_precond=False)
    assert rep.converged and _rel(K @ x, r) <= 1e-8
    with pytest.raises(Exception, match="dimension mismatch"):
        cg.apply_K(r[:-1])
