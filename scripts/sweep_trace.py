"""Traces one Schwarz sweep (globaltimer stamps per work unit) and summarises it.

    python scripts/sweep_trace.py [config2] [--steps 2]
Phases per unit: wait (ticket -> dependencies met), stage (deps met -> panel +
inputs in smem), compute (-> published).
"""
import ctypes as C
import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2512_19536_b200 import _lib, configs  # noqa: E402
from paper_2512_19536_b200.simulation import Simulation  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "config2"
sim = Simulation(getattr(configs, name)())
for _ in range(2):
    sim.step()
L = _lib.lib()
L.pdg_sim_trace_sweep.restype = C.c_int
L.pdg_sim_trace_sweep.argtypes = [C.c_void_p, C.POINTER(C.c_longlong), C.c_int]
cap = 3000000
F = 12
buf = np.zeros(cap * F, np.int64)
for rep in range(3):
    n = L.pdg_sim_trace_sweep(sim._h, buf.ctypes.data_as(C.POINTER(C.c_longlong)), cap)
t = buf[:n * F].reshape(n, F).astype(np.float64)
t0 = t[:, 0].min()
st, dep, stg, done, staged, comp = (t[:, i] - t0 for i in range(6))
task, direc, nbytes, nchunk, height, coarse = (t[:, i] for i in range(6, 12))
span = done.max()
print(f"units {n}: span {span / 1e3:.1f} us; fwd {int((direc == 0).sum())} bwd {int((direc == 1).sum())}")
ready = dep <= st + 300  # dependencies already met when the unit started
print(f"  units whose dependencies were met at start: {int(ready.sum())}")
for lab, v in (("wait", dep - st), ("staging", staged - st), ("deps->gathered", stg - dep),
               ("mat-vec", comp - stg), ("publish", done - comp), ("total", done - st),
               ("total|ready", (done - st)[ready]), ("staging|ready", (staged - st)[ready]),
               ("gather|ready", (stg - dep)[ready]), ("matvec|ready", (comp - stg)[ready]),
               ("publish|ready", (done - comp)[ready])):
    print(f"  {lab:15s} mean {v.mean() / 1e3:6.2f} us  p50 {np.median(v) / 1e3:6.2f}  p90 {np.percentile(v, 90) / 1e3:6.2f}"
          f"  max {v.max() / 1e3:6.2f}")
print(f"  sum unit time / span = mean concurrency {((done - st).sum() / span):.0f}")
print(f"  last forward unit done at {done[direc == 0].max() / 1e3:.1f} us, first backward start {st[direc == 1].min() / 1e3:.1f} us")
edges = np.linspace(0, span, 21)
active = [int(((st <= e) & (done > e)).sum()) for e in edges]
waiting = [int(((st <= e) & (dep > e)).sum()) for e in edges]
print("  time(us) active waiting:")
for e, a_, w_ in zip(edges, active, waiting):
    print(f"    {e / 1e3:7.1f} {a_:6d} {w_:6d}")
print(f"  bytes {nbytes.sum() / 1e6:.1f} MB -> {nbytes.sum() / span:.0f} GB/s over the span")
kb = nbytes / 1024
for lo, hi in ((0, 4), (4, 16), (16, 44), (44, 88), (88, 129)):
    m = (kb >= lo) & (kb < hi)
    print(f"  unit {lo:4.0f}-{hi:4.0f} KB: {int(m.sum()):6d} units, {nbytes[m].sum() / 1e6:6.1f} MB, "
          f"mean time {((done - st)[m].mean() if m.any() else 0) / 1e3:5.2f} us")
ch = nchunk > 1
print(f"  chunked units {int(ch.sum())} ({nbytes[ch].sum() / 1e6:.1f} MB), whole-tile units {int((~ch).sum())}")
ntask = len(np.unique(task))
print(f"  tasks {ntask}, units/task {n / ntask:.1f}")
# the tail of the sweep: which units finish last, and when their dependencies were met
order = np.argsort(done)[::-1][:25]
print("  last units to finish (task, dir, chunks, bytes, start, deps met, staged, done; us):")
for u in order:
    print(f"    task {int(task[u]):5d} dir {int(direc[u])} nch {int(nchunk[u]):2d} {int(nbytes[u]):6d} B  "
          f"{st[u] / 1e3:6.1f} {dep[u] / 1e3:6.1f} {stg[u] / 1e3:6.1f} {done[u] / 1e3:6.1f}")
