"""The C-ABI library loads and exports every symbol include/polydg_b200.h declares."""
import ctypes
import re

from tests.conftest import ROOT

from paper_2512_19536_b200 import _lib


def declared_symbols():
    text = (ROOT / "include" / "polydg_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pdg_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    L = ctypes.CDLL(str(_lib.LIB_PATH))
    names = declared_symbols()
    assert len(names) > 30
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, f"declared but not exported: {missing}"


def test_default_config_matches_reference_defaults():
    # SimulationConfig defaults, /root/reference/proj/include/polydg/timestepper.hpp:21-80
    c = _lib.default_config()
    assert (c.mesh_cells, c.mesh_seed, c.mesh_lloyd) == (512, 42, 20)
    assert (c.degree, c.eta0, c.chi_m, c.C_m, c.dt, c.T) == (1, 10.0, 1000.0, 1.0, 2.5e-3, 10.0)
    assert (c.sigma_grey_l, c.sigma_grey_n, c.sigma_white_l, c.sigma_white_n) == (6.3, 6.3, 6.9, 25.71)
    assert (c.tol, c.maxit, c.warm_start) == (1e-9, 0, 1)
    assert (c.precond_kind, c.h_ratio, c.q) == (_lib.PRECOND_TWO_LEVEL, 2, 0)
    assert list(c.fhn) == [0.13, 0.013, 0.26, 0.1, 1.0, -85.0, 20.0, 1.0]
    assert (c.u_rest, c.u_patch, c.omega0_r2) == (-67.0, -50.0, 0.016)


def test_default_max_iterations():
    # krylov.cpp:12-15: min(20 sqrt(n), n)
    L = _lib.lib()
    assert L.pdg_default_max_iterations(4) == 4
    assert L.pdg_default_max_iterations(10000) == 2000
    assert L.pdg_default_max_iterations(163840) == int(20 * 163840 ** 0.5)


def test_no_device_fails_loudly_without_gpu():
    from tests.conftest import gpu_available
    if gpu_available():
        return
    from paper_2512_19536_b200.simulation import Simulation, SimulationConfig
    try:
        Simulation(SimulationConfig(cells=16))
    except _lib.PdgError as e:
        assert e.kind == "CudaError"
    else:
        raise AssertionError("a simulation was created without a GPU")
