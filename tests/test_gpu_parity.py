"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bars (north star): identical PCG iteration counts +-1 per step; U and every
Y_l within 1e-10 relative L2 after the full run; operator applications within
1e-12 relative (FP64 rounding of different summation orders).
"""
import numpy as np
import pytest

from paper_2512_19536_b200 import configs
from paper_2512_19536_b200._lib import PdgError
from paper_2512_19536_b200.simulation import Simulation, SimulationConfig
from tests.conftest import gpu_available
from tests.oracle_binding import OracleError, oracle_for

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

APPLY_TOL = 1e-12
STATE_TOL = 1e-10

SMALL = [
    dict(cells=64, degree=1),                                             # reference default: identity + hierarchy
    dict(cells=256, degree=2, subdomains=8, coarse=-1, fiber_random=True),
    dict(cells=512, degree=1, precond="block-jacobi"),
    dict(cells=300, degree=3, subdomains=6, coarse=4, q=2),
    dict(cells=700, degree=4, subdomains=12, coarse=-1, q=4),
    dict(cells=400, degree=2, precond="none"),
]


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module", params=SMALL, ids=lambda k: "-".join(f"{a}{b}" for a, b in k.items()))
def pair(request):
    cfg = SimulationConfig(**request.param)
    sim = Simulation(cfg)
    orc, mesh = oracle_for(cfg)
    yield cfg, sim, orc
    sim.close()


def test_operator_and_preconditioner_apply(pair):
    cfg, sim, orc = pair
    rng = np.random.default_rng(3)
    for _ in range(3):
        x = rng.uniform(-1, 1, sim.dimension)
        y, yo = sim.apply_K(x), orc.apply_K(x)
        assert np.abs(y - yo).max() <= APPLY_TOL * np.abs(yo).max()
        z, zo = sim.apply_precond(x), orc.apply_precond(x)
        assert np.abs(z - zo).max() <= 1e-10 * np.abs(zo).max()
        assert rel(z, zo) <= 1e-11


def test_pcg_solve_matches_oracle(pair):
    cfg, sim, orc = pair
    b = np.random.default_rng(5).uniform(-1, 1, sim.dimension)   # acceptance.cpp:285-286 pattern
    x, rep = sim.pcg_solve(b, 1e-10)
    xo, ro = orc.pcg_solve(b, 1e-10)
    assert rep.converged and ro["converged"]
    assert abs(rep.iterations - ro["iterations"]) <= 1
    assert rel(x, xo) <= STATE_TOL
    k = min(rep.iterations, ro["iterations"])
    # early step lengths agree to rounding (later ones drift as rounding propagates)
    np.testing.assert_allclose(rep.alphas[:5], ro["alphas"][:5], rtol=1e-9)
    assert all(a > 0 for a in rep.alphas) and all(bb >= 0 for bb in rep.betas)
    if rep.condition_estimate is not None and ro["condition_estimate"] is not None:
        assert abs(rep.condition_estimate - ro["condition_estimate"]) <= 1e-6 * ro["condition_estimate"]


def test_time_steps_match_oracle(pair):
    cfg, sim, orc = pair
    sim.set_state(0, orc.state()[2], orc.state()[3], orc.state()[4], orc.state()[5])
    for _ in range(5):
        s, so = sim.step(), orc.step()
        assert abs(s.iterations - so["iterations"]) <= 1
    _, _, U, _, Y, _ = sim.state()
    _, _, Uo, _, Yo, _ = orc.state()
    assert rel(U, Uo) <= STATE_TOL
    for l in range(Y.shape[0]):
        assert rel(Y[l], Yo[l]) <= STATE_TOL


def test_initial_projection_matches_oracle():
    cfg = SimulationConfig(cells=512, degree=2)  # default disc-imbalance initial data
    sim = Simulation(cfg)
    orc, _ = oracle_for(cfg)
    assert rel(sim.state()[2], orc.state()[2]) <= 1e-13


def test_config1_full_run():
    """BASELINE config 1 end to end (100 CN steps), FHN standing in for the unpinned BC kinetics."""
    cfg = configs.config1()
    sim = Simulation(cfg)
    orc, _ = oracle_for(cfg)
    its, its_o = [], []
    for _ in range(cfg.n_steps()):
        its.append(sim.step().iterations)
        its_o.append(orc.step()["iterations"])
    assert max(abs(a - b) for a, b in zip(its, its_o)) <= 1
    _, _, U, _, Y, _ = sim.state()
    _, _, Uo, _, Yo, _ = orc.state()
    assert rel(U, Uo) <= STATE_TOL and rel(Y[0], Yo[0]) <= STATE_TOL
    assert U.max() > -84.0  # the strip stimulus depolarised something


def test_config2_mesh_partial_run():
    """BASELINE config 2 (16,384 cells, p = 3, 64 subdomains): the first 20 CN
    steps against the oracle (all 200 steps: scripts/parity_full.py, profiles/)."""
    cfg = configs.config2()
    sim = Simulation(cfg)
    orc, _ = oracle_for(cfg)
    for _ in range(20):
        s, so = sim.step(), orc.step()
        assert abs(s.iterations - so["iterations"]) <= 1
    assert rel(sim.state()[2], orc.state()[2]) <= STATE_TOL
    assert rel(sim.state()[4][0], orc.state()[4][0]) <= STATE_TOL


def test_determinism_bitwise():
    cfg = SimulationConfig(cells=512, degree=2, subdomains=8, coarse=-1)
    a, b = Simulation(cfg), Simulation(cfg)
    ia = [a.step().iterations for _ in range(10)]
    ib = [b.step().iterations for _ in range(10)]
    assert ia == ib
    assert np.array_equal(a.state()[2], b.state()[2])


def test_repeated_sweeps_are_bitwise_identical():
    """The sweep's counters are monotone across launches (sweep number, no
    memsets): hundreds of preconditioner applies on the same input must give
    the same bits, including applies after solves and steps."""
    cfg = SimulationConfig(cells=2048, degree=3, lloyd=5, subdomains=16, coarse=-1)
    sim = Simulation(cfg)
    r = np.random.default_rng(21).uniform(-1, 1, sim.dimension)
    z0 = sim.apply_precond(r)
    for _ in range(200):
        z = sim.apply_precond(r)
    assert np.array_equal(z, z0)
    sim.step()
    sim.pcg_solve(r, 1e-10)
    assert np.array_equal(sim.apply_precond(r), z0)


def test_pcg_edge_cases():
    sim = Simulation(SimulationConfig(cells=128, degree=1))
    n = sim.dimension
    x, rep = sim.pcg_solve(np.zeros(n), 1e-12)                      # krylov test :73-79
    assert rep.converged and rep.iterations == 0 and rep.condition_estimate is None
    assert rep.residual_history == [0.0]
    b = np.random.default_rng(16).uniform(-1, 1, n)
    x, rep = sim.pcg_solve(b, 1e-14, maxit=3)                       # :89-94
    assert not rep.converged and rep.iterations == 3 and len(rep.betas) == 3
    bad = b.copy()
    bad[7] = np.nan
    with pytest.raises(PdgError) as e:                               # :96-100
        sim.pcg_solve(bad, 1e-10)
    assert e.value.kind == "SolverError"
    with pytest.raises(PdgError) as e:                               # :102-104
        sim.pcg_solve(b, 2.0)
    assert e.value.kind == "SolverError"
    x1, r1 = sim.pcg_solve(b, 1e-10, use_precond=False)              # plain CG
    orc, _ = oracle_for(SimulationConfig(cells=128, degree=1))
    xo, ro = orc.pcg_solve(b, 1e-10, use_precond=False)
    assert abs(r1.iterations - ro["iterations"]) <= 1 and rel(x1, xo) <= STATE_TOL
    x2, r2 = sim.pcg_solve(b, 1e-10)                                 # two-level beats CG
    assert r2.iterations < r1.iterations and r2.condition_estimate < r1.condition_estimate


def test_solver_failure_carries_step_index_and_keeps_state():
    cfg = SimulationConfig(cells=64, seed=1, degree=1, chi_m=1.0, precond="none", maxit=2, tol=1e-12,
                           initial=("cosine", 1.0, 0.0), T=2.5e-3)
    sim = Simulation(cfg)
    U0 = sim.state()[2]
    with pytest.raises(PdgError) as e:                               # test_timestepper.cpp:203-221
        sim.step()
    assert e.value.kind == "SolverError" and "step 1" in str(e.value)
    assert np.array_equal(sim.state()[2], U0) and sim.state()[0] == 0


def test_equilibrium_fixed_point():
    cfg = SimulationConfig(cells=24, seed=3, degree=1, q=1, initial=("constant", -85.0), T=0.25)
    sim = Simulation(cfg)
    u0 = sim.state()[2]
    res = sim.run(100)                                               # test_timestepper.cpp:73-90
    assert res.converged_all and np.abs(sim.state()[2] - u0).max() <= 1e-8


@pytest.mark.parametrize("p,S", [(1, 256), (2, 64)])
def test_config3_solve_property(p, S):
    """Full-size config-3 operator: B r and one rtol-1e-10 solve against the
    CPU oracle on the same seeded right-hand side (mt19937_64, acceptance.cpp:
    285-286), plus the residual through apply_K and the symmetry of B."""
    from paper_2512_19536_b200 import _lib
    from tests import oracle_binding as ob
    cfg = configs.config3(p, S)
    sim = Simulation(cfg)
    b = _lib.uniform_rhs(42, sim.dimension)
    orc, _ = oracle_for(cfg)
    assert np.array_equal(b, ob.uniform_rhs(42, sim.dimension))
    assert rel(sim.apply_precond(b), orc.apply_precond(b)) <= 1e-10
    x, rep = sim.pcg_solve(b, 1e-10)
    xo, ro = orc.pcg_solve(b, 1e-10)
    assert rep.converged and abs(rep.iterations - ro["iterations"]) <= 1 and rel(x, xo) <= 1e-10
    del orc
    r = b - sim.apply_K(x)
    assert np.linalg.norm(r) <= 1.5e-10 * np.linalg.norm(b)
    # z = B r is linear and symmetric: <u, B v> == <v, B u>
    rng = np.random.default_rng(1)
    u, v = rng.uniform(-1, 1, sim.dimension), rng.uniform(-1, 1, sim.dimension)
    assert abs(u @ sim.apply_precond(v) - v @ sim.apply_precond(u)) <= 1e-10 * abs(u @ sim.apply_precond(v))


def test_device_factor_matches_host_factor(monkeypatch):
    """The subdomain Cholesky computed on the device (cuda/factor.cu) and on
    the host (host/factor.cpp, PDG_HOST_FACTOR=1) give the same preconditioner
    to rounding, and the same PCG iteration counts."""
    cfg = SimulationConfig(cells=2048, degree=3, lloyd=5, subdomains=16, coarse=-1, fiber_random=True)
    dev = Simulation(cfg)
    monkeypatch.setenv("PDG_HOST_FACTOR", "1")
    host = Simulation(cfg)
    r = np.random.default_rng(8).uniform(-1, 1, dev.dimension)
    zd, zh = dev.apply_precond(r), host.apply_precond(r)
    assert rel(zd, zh) <= 1e-12
    xd, rd = dev.pcg_solve(r, 1e-10)
    xh, rh = host.pcg_solve(r, 1e-10)
    assert rd.iterations == rh.iterations and rel(xd, xh) <= 1e-11
