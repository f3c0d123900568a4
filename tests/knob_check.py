"""Runs one small device solve + 3 CN steps against the CPU oracle under the
current PDG_* environment (tests/test_tuning_knobs.py sets it per case).
Exit status 0 = parity holds: B r within 1e-10, PCG iterations +-1 and x within
1e-10, per-step iterations +-1 and U within 1e-10."""
import sys

import numpy as np

sys.path.insert(0, __import__("pathlib").Path(__file__).resolve().parents[1].as_posix())
from paper_2512_19536_b200.simulation import Simulation, SimulationConfig  # noqa: E402
from tests.oracle_binding import oracle_for  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def main():
    cfg = SimulationConfig(cells=2048, lloyd=5, degree=2, subdomains=16, coarse=-1, fiber_random=True,
                           dt=0.01, T=0.03, tol=1e-8, stimulus=("strip", 2e4, 0.1, 1.0))
    sim = Simulation(cfg)
    orc, _ = oracle_for(cfg)
    r = np.random.default_rng(3).uniform(-1, 1, sim.dimension)
    e_pc = rel(sim.apply_precond(r), orc.apply_precond(r))
    x, rep = sim.pcg_solve(r, 1e-10)
    xo, ro = orc.pcg_solve(r, 1e-10)
    its = [(sim.step().iterations, orc.step()["iterations"]) for _ in range(3)]
    e_u = rel(sim.state()[2], orc.state()[2])
    ok = (e_pc <= 1e-10 and abs(rep.iterations - ro["iterations"]) <= 1 and rel(x, xo) <= 1e-10
          and all(abs(a - b) <= 1 for a, b in its) and e_u <= 1e-10)
    print(f"precond {e_pc:.2e} pcg {rep.iterations}/{ro['iterations']} x {rel(x, xo):.2e} steps {its} U {e_u:.2e}")
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
