"""Config 4 (1,048,576 cells, p=3, 512 subdomains) on one GPU: host setup time
and peak memory, device footprint, a few CN steps with live sweep timing.

    python scripts/c4_probe.py [steps] [config4 | config3:P:S | config5:P]
"""
import ctypes as C
import json
import pathlib
import resource
import sys
import time

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2512_19536_b200 import _lib, configs  # noqa: E402
from paper_2512_19536_b200.simulation import Simulation  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
name = sys.argv[2] if len(sys.argv) > 2 else "config4"
if ":" in name:  # e.g. config3:3:64 or config5:2
    parts = name.split(":")
    cfg = getattr(configs, parts[0])(*[int(a) for a in parts[1:]])
else:
    cfg = getattr(configs, name)()
t0 = time.time()
sim = Simulation(cfg)
setup_s = time.time() - t0
L = _lib.lib()
info = (C.c_int64 * 12)()
L.pdg_problem_info(L.pdg_sim_problem(sim._h), info)
free_b, total_b = C.c_size_t(), C.c_size_t()
try:
    import torch
    free_b.value, total_b.value = torch.cuda.mem_get_info()
except Exception:
    pass
out = {"config": name, "setup_s": round(setup_s, 1),
       "host_peak_rss_gb": round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6, 1),
       "cells": info[0], "dofs": info[2], "subdomains": info[3], "coarse_dim": info[5],
       "nnz_blocks": info[6], "factor_gb": round(info[7] * 8 / 1e9, 2), "tasks": info[8],
       "device_used_gb": round((total_b.value - free_b.value) / 1e9, 1)}
print(json.dumps(out), flush=True)
n0, ms0 = C.c_int64(), C.c_double()
L.pdg_sim_sweep_live(sim._h, C.byref(n0), C.byref(ms0))
its, solve_ms = [], 0.0
t1 = time.time()
for k in range(steps):
    s = sim.step()
    its.append(s.iterations)
    solve_ms += s.solve_ms
    print(json.dumps({"step": k, "iterations": s.iterations, "solve_ms": round(s.solve_ms, 2),
                      "step_ms": round(s.step_ms, 2)}), flush=True)
n1, ms1 = C.c_int64(), C.c_double()
L.pdg_sim_sweep_live(sim._h, C.byref(n1), C.byref(ms1))
sweeps = n1.value - n0.value
sweep_ms = (ms1.value - ms0.value) / max(1, sweeps)
fb = info[7] * 8
print(json.dumps({"steps": steps, "iterations": its, "wall_s": round(time.time() - t1, 2),
                  "dof_iter_per_s": info[2] * sum(its) / (solve_ms * 1e-3) if solve_ms else None,
                  "sweep_live_ms": round(sweep_ms, 3), "sweeps": sweeps,
                  "sweep_GBs": round(fb / (sweep_ms * 1e-3) / 1e9, 1) if sweep_ms else None}), flush=True)
