"""Config 5: the config-4 mesh at p (2 or 4), 1,024 subdomains, one PCG solve to
rtol 1e-10 from x0 = 0 with a seeded uniform [-1, 1] right-hand side (the
reference draws it with mt19937_64, acceptance.cpp:285-286; numpy's generator
stands in, same distribution).
Reports the solve and, separately, SpMV, Schwarz apply (sweep incl. the
coarse solve), the other per-iteration kernels, and the coarse solve's share
of one traced sweep.

    python scripts/c5_probe.py [p]
"""
import ctypes as C
import json
import pathlib
import resource
import sys
import time

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2512_19536_b200 import _lib, configs  # noqa: E402
from paper_2512_19536_b200.simulation import Simulation  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = configs.config5(p)
t0 = time.time()
sim = Simulation(cfg)
setup_s = time.time() - t0
L = _lib.lib()
info = (C.c_int64 * 12)()
L.pdg_problem_info(L.pdg_sim_problem(sim._h), info)
print(json.dumps({"config": f"config5 p={p}", "setup_s": round(setup_s, 1),
                  "host_peak_rss_gb": round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6, 1),
                  "dofs": info[2], "subdomains": info[3], "coarse_dim": info[5], "nnz_blocks": info[6],
                  "factor_gb": round(info[7] * 8 / 1e9, 2)}), flush=True)


b = np.random.default_rng(42).uniform(-1.0, 1.0, info[2])  # seeded stand-in for the mt19937_64 draw
n0, ms0 = C.c_int64(), C.c_double()
L.pdg_sim_sweep_live(sim._h, C.byref(n0), C.byref(ms0))
t1 = time.time()
x, rep = sim.pcg_solve(b, 1e-10)
wall = time.time() - t1
n1, ms1 = C.c_int64(), C.c_double()
L.pdg_sim_sweep_live(sim._h, C.byref(n1), C.byref(ms1))
sweeps = n1.value - n0.value
sweep_ms = (ms1.value - ms0.value) / max(1, sweeps)
kms = (C.c_double * 9)()
kby = (C.c_int64 * 9)()
_lib.check(L.pdg_sim_profile(sim._h, 5, kms, kby))
names = ["spmv", "update", "restrict", "sweep", "restrict_combine", "prolong_dot", "pupdate", "ionic", "rhs"]
print(json.dumps({"iterations": rep.iterations, "converged": rep.converged, "solve_wall_s": round(wall, 3),
                  "dof_iter_per_s": info[2] * rep.iterations / wall,
                  "condition_estimate": rep.condition_estimate,
                  "schwarz_apply_live_ms": round(sweep_ms, 3),
                  "schwarz_apply_GBs": round(info[7] * 8 / (sweep_ms * 1e-3) / 1e9, 1),
                  "kernels_isolated_cold_L2": {k: {"ms": round(kms[i], 4), "GB/s": round(kby[i] / (kms[i] * 1e-3) / 1e9, 1)
                                                   if kms[i] else None} for i, k in enumerate(names) if kms[i]}}),
      flush=True)

# The coarse solve separately (the reference times it apart, schwarz.cpp:165-168). Here it runs
# inside the sweep (coarse forward, dense coarse root, coarse backward are ordinary units), so its
# time is read from one traced sweep: the span from the first coarse unit's start to the last
# coarse unit's end, and the CTA time its units took.
L.pdg_sim_trace_sweep.restype = C.c_int
L.pdg_sim_trace_sweep.argtypes = [C.c_void_p, C.POINTER(C.c_longlong), C.c_int]
cap, F = 3000000, 12
buf = np.zeros(cap * F, np.int64)
for _ in range(2):
    n = L.pdg_sim_trace_sweep(sim._h, buf.ctypes.data_as(C.POINTER(C.c_longlong)), cap)
t = buf[:n * F].reshape(n, F).astype(np.float64)
t0_ = t[:, 0].min()
st, done = t[:, 0] - t0_, t[:, 3] - t0_
co = (t[:, 9] > 0) & (t[:, 11] == 1)  # individually scheduled units of coarse tasks
print(json.dumps({"traced_sweep_us": round(done.max() / 1e3, 1), "coarse_units": int(co.sum()),
                  "coarse_solve_span_us": round((done[co].max() - st[co].min()) / 1e3, 1) if co.any() else None,
                  "coarse_first_start_us": round(st[co].min() / 1e3, 1) if co.any() else None,
                  "coarse_last_end_us": round(done[co].max() / 1e3, 1) if co.any() else None,
                  "coarse_cta_time_us": round((done - st)[co].sum() / 1e3, 1) if co.any() else None}), flush=True)
