"""Golden outputs of the REFERENCE's own numeric code (tests/golden/reference_numeric.json).

Runs the reference's proj/src numeric sources, compiled here by
`make -C oracle refnum` with the Eigen API stand-in (oracle/_ref/
libpolydg_refnum.so, tests/refnum.py), on:
  * acceptance criteria 2, 3, 7, 8, 9 (proj/tests/acceptance.cpp:138-203,
    339-400): manufactured-solution errors and slopes, per-step PCG iterations
    and averages, exactly as the reference's acceptance configs set them up;
  * BASELINE config 1 (isotropic, 16 agglomerated subdomains = coarse
    partition, strip stimulus, FHN from rest), all 100 CN steps: per-step
    iterations and the final U, Y;
  * the reference's default Simulation (identity subdomains, H/h = 2
    hierarchy coarse space, disc initial condition) on 256 cells, p = 2.
The GPU tests (tests/test_gpu_reference.py) compare the device path with
these numbers; tests/test_reference_numeric.py compares the oracle.

    python scripts/make_reference_golden.py   (needs oracle/_ref/libpolydg_refnum.so)
"""
import json
import math
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from tests.refnum import RefSim  # noqa: E402
from tests.reference_configs import config1, default_sim, manufactured, paper  # noqa: E402


def steps(sim, n):
    return [sim.step()["iterations"] for _ in range(n)]


def main():
    out = {"source": "reference proj/src numeric path compiled with oracle/eigen_shim (oracle/_ref/libpolydg_refnum.so)"}
    t0 = time.time()
    # criterion 2: spatial order of the manufactured heat problem
    c2 = {}
    for p in (1, 2):
        hs, errs = [], []
        for cells in (128, 512, 2048):
            cfg = manufactured(cells, p, 1e-4, 0.02)
            s = RefSim(cfg)
            steps(s, cfg.n_steps())
            errs.append(s.l2_error_cosine(s.state()[2], 1.0, 1.0, 0.02))
            hs.append(s.mesh_size())
        c2[str(p)] = {"h": hs, "errors": errs, "slope": float(np.polyfit(np.log(hs), np.log(errs), 1)[0])}
    out["criterion2"] = c2
    # criterion 3: temporal order against a fine-step solution
    cfg = manufactured(64, 1, 1.25e-4, 0.4)
    r = RefSim(cfg)
    steps(r, cfg.n_steps())
    uref = r.state()[2]
    M = r.export("M")
    errs = []
    for dt in (4e-3, 2e-3, 1e-3):
        cfg = manufactured(64, 1, dt, 0.4)
        s = RefSim(cfg)
        steps(s, cfg.n_steps())
        d = s.state()[2] - uref
        errs.append(math.sqrt(d @ (M @ d)))
    out["criterion3"] = {"dts": [4e-3, 2e-3, 1e-3], "errors": errs,
                         "slope": float(np.polyfit(np.log([4e-3, 2e-3, 1e-3]), np.log(errs), 1)[0]),
                         "u_fine": uref.tolist()}
    # criteria 7-9: PCG iteration statistics
    its = {}
    for key, cfg in {"c7_two_level": paper(512, 1, 2, "two-level"), "c7_cg": paper(512, 1, 2, "none"),
                     "c8_128": paper(128, 1, 2, "two-level"), "c8_2048": paper(2048, 1, 2, "two-level"),
                     "c9_4": paper(512, 1, 4, "two-level"), "c9_8": paper(512, 1, 8, "two-level")}.items():
        its[key] = steps(RefSim(cfg), cfg.n_steps())
    out["iterations"] = its
    # BASELINE config 1, full run
    cfg = config1()
    s = RefSim(cfg)
    it1 = steps(s, cfg.n_steps())
    _, _, U, _, Y, _ = s.state()
    out["config1"] = {"iterations": it1, "U": U.tolist(), "Y": Y[0].tolist()}
    # reference default Simulation
    cfg = default_sim()
    s = RefSim(cfg)
    itd = steps(s, cfg.n_steps())
    _, _, U, _, Y, _ = s.state()
    out["default_sim"] = {"iterations": itd, "U": U.tolist(), "Y": Y[0].tolist()}
    out["wall_s"] = round(time.time() - t0, 1)
    path = ROOT / "tests" / "golden" / "reference_numeric.json"
    path.write_text(json.dumps(out))
    print(f"wrote {path} ({path.stat().st_size >> 10} KB) in {out['wall_s']} s")


if __name__ == "__main__":
    main()
