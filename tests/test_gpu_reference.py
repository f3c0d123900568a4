"""The device path against the REFERENCE's own numeric code.

Golden outputs come from the reference's proj/src numeric sources compiled in
this repository's oracle/_ref with the Eigen API stand-in
(tests/golden/reference_numeric.json, scripts/make_reference_golden.py):
acceptance criteria 2, 3, 7, 8, 9 (proj/tests/acceptance.cpp:138-203,
339-400), BASELINE config 1 over all 100 CN steps, and the reference's default
Simulation (identity subdomains, H/h = 2 hierarchy coarse space). Bars: PCG
iterations +-1 per step, states within 1e-10 relative L2 (north star), the
acceptance criteria's own thresholds, and manufactured-solution errors equal
to the reference's to 1e-6 relative.
"""
import numpy as np
import pytest

from tests.conftest import gpu_available
from tests.test_reference_numeric import GOLD, _rel, check_convergence_criteria, check_iteration_criteria
from tests.reference_configs import config1, default_sim

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a GPU")]


def _run(cfg):
    from paper_2512_19536_b200.simulation import Simulation
    sim = Simulation(cfg)
    its = [sim.step().iterations for _ in range(cfg.n_steps())]
    return sim, its


@pytest.mark.parametrize("name,make", [("config1", config1), ("default_sim", default_sim)])
def test_gpu_full_run_matches_reference_build(name, make):
    sim, its = _run(make())
    g = GOLD[name]
    assert max(abs(a - b) for a, b in zip(its, g["iterations"])) <= 1
    _, _, U, _, Y, _ = sim.state()
    assert _rel(U, g["U"]) <= 1e-10 and _rel(Y[0], g["Y"]) <= 1e-10


def test_gpu_acceptance_iteration_criteria():
    avg = check_iteration_criteria(lambda cfg: _run(cfg)[1])
    assert avg["c7_two_level"] > 0


def test_gpu_acceptance_convergence_criteria():
    from tests.oracle_binding import oracle_for

    def final_state(cfg, want_mass=False):
        sim, _ = _run(cfg)
        return sim.state()[2], (sim.problem.export("M") if want_mass else None)

    def l2(cfg, U):  # l2_error (dg_space.cpp:94-115) evaluated by the oracle on the device's U
        return oracle_for(cfg)[0].l2_error_cosine(U, 1.0, 1.0, cfg.T)

    check_convergence_criteria(final_state, l2)
