"""Short driver for ncu: builds a BASELINE workload and runs a few CN steps.

    python scripts/profile_step.py [config2] [steps]
"""
import sys
import pathlib

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))

from paper_2512_19536_b200 import configs  # noqa: E402
from paper_2512_19536_b200.simulation import Simulation  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
sim = Simulation(getattr(configs, name)())
for _ in range(steps):
    s = sim.step()
print(f"{name}: {steps} steps, last {s.iterations} its, {s.step_ms:.3f} ms")
