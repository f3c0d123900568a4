"""BASELINE config 3: robustness sweep on the 65,536-cell seeded Voronoi square.

p = 1..4 x subdomains {64, 256} (coarse agglomerates = subdomains, q = p),
grey/white anisotropy with per-element fibres, 50 CN steps each, FP64.
Reports iterations/step and DOF-iter/s per (p, S) through the study harness
(paper_2512_19536_b200/study.py), plus the reference-style study.csv/.txt.

    python scripts/c3_study.py [out_dir] [steps]
"""
import json
import pathlib
import sys

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2512_19536_b200 import configs  # noqa: E402
from paper_2512_19536_b200.study import StudySpec, run_scaling_study, write_throughput_table  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else None
base = configs.config3(1, 64)
spec = StudySpec(cells=[base.cells], ratios=[2], degrees=[(p, p) for p in (1, 2, 3, 4)], kinds=["two-level"],
                 base=base, subdomains=[64, 256])
rows = run_scaling_study(spec, out_dir=out, steps=steps,
                         log=lambda r: print(json.dumps(r.__dict__) if hasattr(r, "__dict__") else r, flush=True))
with open(pathlib.Path(out) / "throughput.md", "w") as f:
    write_throughput_table(rows, f)
print(open(pathlib.Path(out) / "throughput.md").read())
