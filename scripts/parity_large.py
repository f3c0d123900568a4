"""Parity of the device path against the CPU oracle on the large BASELINE configs.

North star: identical PCG iteration counts (+-1) per step and U, Y within 1e-10
relative L2 on the same seeded inputs. Two phases so host memory holds one
solver at a time: the device run first (results kept in numpy), then the
oracle (row-parallel CSR products, same bits as serial; lean storage).

    python scripts/parity_large.py c3 P S [steps]   # config 3 row, 50 steps default
    python scripts/parity_large.py c4 [steps]        # config 4, first 3 CN steps default
    python scripts/parity_large.py c5 P              # config 5 one solve, rtol 1e-10, x0 = 0

Besides the steps / solve: K x and B r on the config-5 style random vector
(mt19937_64(42), acceptance.cpp:285-286) against the oracle at 1e-12 / 1e-10.
Prints one JSON line (also appended to $PARITY_OUT when set).
"""
import json
import os
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2512_19536_b200 import _lib, configs  # noqa: E402
from paper_2512_19536_b200.simulation import Simulation  # noqa: E402
from tests import oracle_binding as ob  # noqa: E402

RHS_SEED = 42


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb else float(np.linalg.norm(a))


def main():
    kind = sys.argv[1]
    if kind == "c3":
        p, S = int(sys.argv[2]), int(sys.argv[3])
        cfg = configs.config3(p, S)
        steps = int(sys.argv[4]) if len(sys.argv) > 4 else cfg.n_steps()
        name = f"config3 p={p} S={S}"
    elif kind == "c4":
        cfg = configs.config4()
        steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
        name = "config4"
    elif kind == "c5":
        p = int(sys.argv[2])
        cfg = configs.config5(p)
        steps = 0
        name = f"config5 p={p}"
    else:
        raise SystemExit(__doc__)

    out = {"config": name, "cells": cfg.cells, "degree": cfg.degree, "subdomains": cfg.subdomains}
    # ---- phase 1: device ----
    t0 = time.time()
    sim = Simulation(cfg)
    n = sim.dimension
    out["dofs"] = n
    out["gpu_setup_s"] = round(time.time() - t0, 1)
    b = _lib.uniform_rhs(RHS_SEED, n)
    y_gpu, z_gpu = sim.apply_K(b), sim.apply_precond(b)
    its_gpu, x_gpu, st_gpu = [], None, None
    t0 = time.time()
    if steps:
        for _ in range(steps):
            its_gpu.append(sim.step().iterations)
        st_gpu = sim.state()
        Mdiag = sim.problem.export("M")
    else:
        x_gpu, rep = sim.pcg_solve(b, cfg.tol)
        its_gpu = [rep.iterations]
        out["gpu_converged"] = rep.converged
    out["gpu_run_s"] = round(time.time() - t0, 1)
    sim.close()
    del sim

    # ---- phase 2: oracle ----
    ob.set_parallel(True)
    ob.set_lean(1 if steps else 2)
    t0 = time.time()
    orc, _ = ob.oracle_for(cfg)
    out["oracle_setup_s"] = round(time.time() - t0, 1)
    assert orc.dimension == n
    b_o = ob.uniform_rhs(RHS_SEED, n)
    out["rhs_bitwise_equal"] = bool(np.array_equal(b, b_o))
    out["apply_K_rel"] = rel(y_gpu, orc.apply_K(b))
    out["apply_precond_rel"] = rel(z_gpu, orc.apply_precond(b))
    its_o = []
    t0 = time.time()
    if steps:
        for _ in range(steps):
            its_o.append(orc.step()["iterations"])
        _, _, U, _, Y, _ = st_gpu
        _, _, Uo, _, Yo, _ = orc.state()
        relM = lambda a, c: float(np.sqrt((a - c) @ (Mdiag @ (a - c)) / (c @ (Mdiag @ c))))
        out["U_rel_l2"], out["U_rel_M"] = rel(U, Uo), relM(U, Uo)
        out["Y_rel_l2"] = max(rel(Y[l], Yo[l]) for l in range(len(Y))) if len(Y) else 0.0
        out["Y_rel_M"] = max(relM(Y[l], Yo[l]) for l in range(len(Y))) if len(Y) else 0.0
        errs = [out["U_rel_l2"], out["Y_rel_l2"]]
    else:
        xo, ro = orc.pcg_solve(b, cfg.tol)
        its_o = [ro["iterations"]]
        out["oracle_converged"] = ro["converged"]
        out["x_rel_l2"] = rel(x_gpu, xo)
        errs = [out["x_rel_l2"]]
    out["oracle_run_s"] = round(time.time() - t0, 1)
    out["oracle_threads"] = ob.lib().orc_threads()
    out["oracle_factor_blocks_per_cell"] = round(orc.factor_blocks() / cfg.cells, 3)
    d = [a - c for a, c in zip(its_gpu, its_o)]
    out["steps"] = steps
    out["iterations_gpu"] = its_gpu
    out["iterations_oracle"] = its_o
    out["max_abs_iteration_diff"] = max(abs(x) for x in d)
    out["pass"] = (out["max_abs_iteration_diff"] <= 1 and max(errs) <= 1e-10 and out["apply_K_rel"] <= 1e-12
                   and out["apply_precond_rel"] <= 1e-10 and out["rhs_bitwise_equal"])
    line = json.dumps(out)
    print(line, flush=True)
    if os.environ.get("PARITY_OUT"):
        with open(os.environ["PARITY_OUT"], "a") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
