"""Device assembly (cuda/assemble.cu) against the host
assembly that is pinned bitwise to the oracle and to the reference build
(tests/test_host_setup.py, tests/test_reference_numeric.py): K, M, E and K0
exported from a device Simulation equal the host Problem's bit for bit, and the
projected initial state U0 / Y0 equals the host-assembled simulation's
(PDG_HOST_ASSEMBLY=1). The cosine initial condition goes through the device
cos, which may differ from glibc's in the last bit: 1e-15 there. Setups that
factor on the host (one element per subdomain, PDG_HOST_FACTOR=1) keep the
host assembly (checked last)."""
import numpy as np
import pytest

from tests.conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a GPU")]

CASES = {
    "p1_two_level": dict(cells=512, lloyd=5, degree=1, subdomains=8, coarse=-1),
    "p3_fibres_strip": dict(cells=1024, lloyd=5, degree=3, subdomains=16, coarse=-1, fiber_random=True,
                            sigma_white_l=1.0, sigma_white_n=0.2, sigma_grey_l=0.5, sigma_grey_n=0.5,
                            stimulus=("strip", 2e4, 0.1, 1.0)),
    "p2_hierarchy_disc": dict(cells=256, lloyd=5, degree=2, subdomains=16),
    "p2_plain_cg": dict(cells=256, lloyd=5, degree=2, precond="none"),
    "p4_block_jacobi": dict(cells=256, lloyd=5, degree=4, subdomains=8, precond="block-jacobi"),
    "p2_bc_model": dict(cells=256, lloyd=5, degree=2, subdomains=8, coarse=-1, ionic_model="barreto-cressman"),
    "p2_cosine": dict(cells=256, lloyd=5, degree=2, subdomains=8, coarse=-1, initial=("cosine", 1.0, 0.0)),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_device_assembly_matches_host(name, monkeypatch):
    from paper_2512_19536_b200.simulation import Problem, Simulation, SimulationConfig
    cfg = SimulationConfig(**CASES[name])
    sim = Simulation(cfg)
    assert sim.problem.flags()["device_assembly"]
    host = Problem(cfg)
    assert not host.flags()["device_assembly"]
    kinds = ["K", "M"] + (["E", "K0"] if cfg.precond == "two-level" else [])
    for w in kinds:
        d, h = sim.problem.export(w), host.export(w)
        assert d.shape == h.shape and (d != h).nnz == 0, w
    monkeypatch.setenv("PDG_HOST_ASSEMBLY", "1")
    ref = Simulation(cfg)
    assert not ref.problem.flags()["device_assembly"]
    tol = 1e-15 if name == "p2_cosine" else 0.0
    for a, b in zip(sim.state()[2:], ref.state()[2:]):
        a, b = np.asarray(a), np.asarray(b)
        assert np.abs(a - b).max() <= tol * max(1.0, np.abs(b).max())
    # and the solver on top takes the same path
    s1, s2 = sim.step(), ref.step()
    assert s1.iterations == s2.iterations


def test_host_factor_setups_keep_host_assembly(monkeypatch):
    from paper_2512_19536_b200.simulation import Simulation, SimulationConfig
    assert not Simulation(SimulationConfig(cells=64, degree=2)).problem.flags()["device_assembly"]
    monkeypatch.setenv("PDG_HOST_FACTOR", "1")
    sim = Simulation(SimulationConfig(cells=256, degree=2, subdomains=8, coarse=-1))
    assert sim.problem.flags() == {"device_assembly": False, "device_factor": False}
