"""The reference's acceptance / default configurations as SimulationConfig
(shared by the golden generator, the oracle tests and the GPU tests).

paper(), manufactured(): proj/tests/acceptance.cpp:52-95 (paper_config,
manufactured_config); default_sim(): SimulationConfig defaults
(timestepper.hpp:21-80) on a small mesh and a short run; config1(): BASELINE
config 1 (paper_2512_19536_b200.configs).
"""
import math

from paper_2512_19536_b200 import configs
from paper_2512_19536_b200.simulation import SimulationConfig


def paper(cells, p, ratio, kind):
    # acceptance.cpp:52-67: chi_m = 1, dt = 2.5e-3, T = 0.25 (100 steps), tol 1e-9, maxit 20000, q = 1
    return SimulationConfig(cells=cells, seed=42, degree=p, chi_m=1.0, C_m=1.0, dt=2.5e-3, T=0.25, tol=1e-9,
                            maxit=20000, precond=kind, h_ratio=ratio, q=1)


def manufactured(cells, p, dt, T):
    # acceptance.cpp:69-95: heat problem with exact solution cos(pi x) cos(pi y) e^{-t}
    return SimulationConfig(cells=cells, seed=42, degree=p, chi_m=1.0, C_m=1.0, sigma_grey_l=1.0, sigma_grey_n=1.0,
                            sigma_white_l=1.0, sigma_white_n=1.0, dt=dt, T=T, ionic_model="none", tol=1e-12,
                            maxit=20000, precond="two-level", h_ratio=2, q=1, initial=("cosine", 1.0, 0.0),
                            stimulus=("cosine", 2 * math.pi ** 2 - 1.0, 1.0))


def default_sim():
    # the reference's defaults (identity subdomains, H/h = 2 hierarchy, disc
    # initial condition, FHN) on 256 cells at p = 2, 20 steps
    return SimulationConfig(cells=256, degree=2, T=0.05)


def config1():
    return configs.config1()
