"""Barreto-Cressman kinetics (ext; BASELINE config 1 names the model).

The reference registers the model name but ships no kinetics
(/root/reference/proj/src/ionics.cpp:52-57, test_ionics.cpp:70 expects a
ConfigError), so parity is UNPINNED against the reference: the oracle's C++
restatement (oracle/src/discretization.cpp) is checked here against a third,
independent numpy restatement of Cressman et al. 2009, and the GPU path is
checked against the oracle (tests marked gpu).
"""
import math

import numpy as np
import pytest

from paper_2512_19536_b200 import configs
from paper_2512_19536_b200._lib import PdgError, default_config
from paper_2512_19536_b200.simulation import SimulationConfig, ionic_rest
from tests import oracle_binding as ob
from tests.conftest import gpu_available

P = list(default_config().bc)


def np_bc(u, y, p=P):
    """Independent restatement (parameter order: PDG_BC_* in include/polydg_b200.h)."""
    gna, gk, gnal, gkl, gcll, phi, rho, gglia, eps, kbath, gamma, beta, tau, rtf, cli, clo, nai0, ki0, nao0, amp = p
    n, h, ko, nai = y
    xe = lambda x: 1.0 if x == 0 else x / (1 - math.exp(-x))
    am, bm = xe(0.1 * (u + 30)), 4 * math.exp(-(u + 55) / 18)
    an, bn = 0.1 * xe(0.1 * (u + 34)), 0.125 * math.exp(-(u + 44) / 80)
    ah, bh = 0.07 * math.exp(-(u + 44) / 20), 1 / (1 + math.exp(-0.1 * (u + 14)))
    minf = am / (am + bm)
    ki, nao = ki0 + (nai0 - nai), nao0 - beta * (nai - nai0)
    ena, ek, ecl = rtf * math.log(nao / nai), rtf * math.log(ko / ki), rtf * math.log(cli / clo)
    ina = gna * minf ** 3 * h * (u - ena) + gnal * (u - ena)
    ik = gk * n ** 4 * (u - ek) + gkl * (u - ek)
    icl = gcll * (u - ecl)
    pump = rho / (1 + math.exp((25 - nai) / 3)) / (1 + math.exp(5.5 - ko))
    glia = gglia / (1 + math.exp((18 - ko) / 2.5))
    diff = eps * (ko - kbath)
    dy = [phi * (an * (1 - n) - bn * n), phi * (ah * (1 - h) - bh * h),
          (gamma * beta * ik - 2 * beta * pump - glia - diff) / tau, (-gamma * ina - 3 * pump) / tau]
    return amp * (ina + ik + icl), -np.array(dy)


def test_pointwise_matches_independent_restatement():
    rng = np.random.default_rng(7)
    for _ in range(200):
        u = rng.uniform(-100, 50)
        y = [rng.uniform(0, 1), rng.uniform(0, 1), rng.uniform(2, 12), rng.uniform(10, 30)]
        f, m = ob.barreto_cressman(u, y)
        fr, mr = np_bc(u, y)
        assert abs(f - fr) <= 1e-12 * max(1.0, abs(fr))
        assert np.allclose(m, mr, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("u", [-30.0, -34.0])
def test_removable_singularities(u):
    """alpha_m at u = -30 and alpha_n at u = -34 are 0/0 in the closed form."""
    y = [0.3, 0.6, 4.0, 18.0]
    f0, m0 = ob.barreto_cressman(u, y)
    f1, m1 = ob.barreto_cressman(u + 1e-7, y)
    assert np.isfinite(f0) and np.all(np.isfinite(m0))
    assert abs(f0 - f1) <= 1e-4 and np.allclose(m0, m1, atol=1e-6)


def test_resting_state_is_a_fixed_point_and_product_agrees():
    cfg = SimulationConfig(ionic_model="barreto-cressman")
    nc, u, y = ionic_rest(cfg)
    nco, uo, yo = ob.ionic_rest(cfg)
    assert nc == nco == 4
    assert abs(u - uo) <= 1e-12 and np.allclose(y, yo, rtol=1e-12)
    f, m = np_bc(u, y)
    assert abs(f) <= 1e-11 and np.abs(m).max() <= 1e-13
    assert -75 < u < -60 and 0 < y[0] < 1 and 0 < y[1] < 1   # physiological rest
    assert ionic_rest(SimulationConfig())[:2] == (1, -85.0)   # FHN: u_min, w = 0 (ionics.hpp:56-57)


def test_action_potential_in_zero_dimensions():
    """Forward-Euler point model from rest with a 1 ms, 20 uA/cm^2 pulse fires a spike."""
    _, u, y = ionic_rest(SimulationConfig(ionic_model="barreto-cressman"))
    y = np.array(y)
    peak = u
    for k in range(2000):
        f, m = ob.barreto_cressman(u, y)
        u += 0.01 * (-f + (20.0 if k < 100 else 0.0))
        y = y - 0.01 * m
        peak = max(peak, u)
    assert peak > 20.0 and u < -60.0


def test_errors():
    with pytest.raises(ob.OracleError, match="non-finite"):
        ob.barreto_cressman(float("nan"), [0.1, 0.9, 4.0, 18.0])
    with pytest.raises(ob.OracleError, match="non-finite"):
        ob.barreto_cressman(-60.0, [0.1, 0.9, -1.0, 18.0])   # log of a negative concentration
    with pytest.raises(PdgError, match="unknown barreto-cressman parameter"):
        SimulationConfig(ionic_model="barreto-cressman", ionic_params={"a": 1.0}).to_c()
    with pytest.raises(PdgError, match="barreto-cressman"):
        ionic_rest(SimulationConfig(ionic_model="barreto-cressman", ionic_params={"tau": 0.0}))


def test_config1_bc_starts_from_rest():
    cfg = configs.config1_bc()
    assert cfg.ionic_model == "barreto-cressman" and cfg.initial[0] == "constant"
    assert abs(cfg.initial[1] - ionic_rest(cfg)[1]) == 0.0


def test_oracle_short_run_from_rest_stays_at_rest():
    cfg = SimulationConfig(cells=48, seed=3, degree=1, ionic_model="barreto-cressman", dt=0.01, T=0.05)
    cfg.initial = ("constant", ionic_rest(cfg)[1])
    orc, _ = ob.oracle_for(cfg)
    _, _, U0, _, Y0, _ = orc.state()
    for _ in range(5):
        assert orc.step()["converged"]
    _, _, U, _, Y, _ = orc.state()
    assert np.abs(U - U0).max() <= 1e-8 * np.abs(U0).max()
    assert np.abs(Y - Y0).max() <= 1e-8 * np.abs(Y0).max()




def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
@pytest.mark.parametrize("kw", [dict(cells=256, degree=2, subdomains=8, coarse=-1, fiber_random=True),
                                dict(cells=300, degree=3, subdomains=6, coarse=4, q=2)],
                         ids=["p2", "p3"])
def test_gpu_bc_steps_match_oracle(kw):
    """Stimulated BC steps: iterations +-1 per step, U and every Y component within 1e-10."""
    from paper_2512_19536_b200.simulation import Simulation
    cfg = SimulationConfig(ionic_model="barreto-cressman", dt=0.01, T=0.2, tol=1e-10,
                           stimulus=("strip", 2.0e4, 0.3, 1.0), **kw)
    cfg.initial = ("constant", ionic_rest(cfg)[1])
    sim = Simulation(cfg)
    orc, _ = ob.oracle_for(cfg)
    assert sim.n_comp == 4
    for _ in range(20):
        s, so = sim.step(), orc.step()
        assert s.converged and abs(s.iterations - so["iterations"]) <= 1
    _, _, U, Up, Y, _ = sim.state()
    _, _, Uo, Upo, Yo, _ = orc.state()
    assert rel(U, Uo) <= 1e-10 and rel(Up, Upo) <= 1e-10
    for l in range(4):
        assert rel(Y[l], Yo[l]) <= 1e-10, l
    assert U.max() > ionic_rest(cfg)[1] + 1.0   # the stimulus depolarised the strip
    sim.close()


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_gpu_config1_bc_full_run():
    """BASELINE config 1 with Barreto-Cressman, all 100 CN steps against the oracle."""
    from paper_2512_19536_b200.simulation import Simulation
    cfg = configs.config1_bc()
    sim = Simulation(cfg)
    orc, _ = ob.oracle_for(cfg)
    its, its_o = [], []
    for _ in range(cfg.n_steps()):
        its.append(sim.step().iterations)
        its_o.append(orc.step()["iterations"])
    assert max(abs(a - b) for a, b in zip(its, its_o)) <= 1
    _, _, U, _, Y, _ = sim.state()
    _, _, Uo, _, Yo, _ = orc.state()
    assert rel(U, Uo) <= 1e-10
    for l in range(4):
        assert rel(Y[l], Yo[l]) <= 1e-10, l
    sim.close()


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_gpu_bc_rest_is_a_fixed_point():
    from paper_2512_19536_b200.simulation import Simulation
    cfg = SimulationConfig(cells=64, seed=3, degree=2, ionic_model="barreto-cressman", dt=0.01, T=0.5)
    cfg.initial = ("constant", ionic_rest(cfg)[1])
    sim = Simulation(cfg)
    _, _, U0, _, Y0, _ = sim.state()
    res = sim.run(50)
    _, _, U, _, Y, _ = sim.state()
    assert res.converged_all
    assert np.abs(U - U0).max() <= 1e-8 * np.abs(U0).max()
    assert np.abs(Y - Y0).max() <= 1e-8 * np.abs(Y0).max()
    sim.close()
