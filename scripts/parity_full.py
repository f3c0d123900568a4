"""Full-run parity of a BASELINE config: the device path against the CPU oracle
for every CN step (north star: PCG iterations equal +-1 per step; U and every
Y_l within 1e-10 relative L2 after the full run, Euclidean and M-weighted as in
test_timestepper.cpp:129). Writes one JSON summary line.

    python scripts/parity_full.py [config2] [steps]
"""
import json
import pathlib
import sys
import time

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2512_19536_b200 import configs  # noqa: E402
from paper_2512_19536_b200.simulation import Simulation  # noqa: E402
from tests.oracle_binding import oracle_for  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config2"
cfg = getattr(configs, name)()
steps = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n_steps()
sim = Simulation(cfg)
orc, _ = oracle_for(cfg)
M = sim.problem.export("M")
its, its_o, t0 = [], [], time.time()
for k in range(steps):
    its.append(sim.step().iterations)
    its_o.append(orc.step()["iterations"])
_, _, U, _, Y, _ = sim.state()
_, _, Uo, _, Yo, _ = orc.state()
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
relM = lambda a, b: float(np.sqrt((a - b) @ (M @ (a - b)) / (b @ (M @ b))))
d = [a - b for a, b in zip(its, its_o)]
out = {"config": name, "steps": steps, "dofs": sim.dimension, "iterations_gpu_total": sum(its),
       "iterations_oracle_total": sum(its_o), "max_abs_iteration_diff": max(abs(x) for x in d),
       "steps_with_diff": sum(1 for x in d if x), "U_rel_l2": rel(U, Uo), "U_rel_M": relM(U, Uo),
       "Y_rel_l2": rel(Y[0], Yo[0]), "Y_rel_M": relM(Y[0], Yo[0]), "U_max": float(U.max()),
       "wall_s": round(time.time() - t0, 1),
       "pass": max(abs(x) for x in d) <= 1 and rel(U, Uo) <= 1e-10 and rel(Y[0], Yo[0]) <= 1e-10}
print(json.dumps(out), flush=True)
