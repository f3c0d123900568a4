"""Traces one Schwarz sweep and summarises level-chunk units against the individually scheduled ones.

    python scripts/chunk_trace.py config4
"""
import ctypes as C
import pathlib
import sys

import numpy as np

sys.path.insert(0, str(pathlib.Path(__file__).resolve().parents[1]))
from paper_2512_19536_b200 import _lib, configs  # noqa: E402
from paper_2512_19536_b200.simulation import Simulation  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config4"
sim = Simulation(getattr(configs, name)())
sim.step()
L = _lib.lib()
L.pdg_sim_trace_sweep.restype = C.c_int
L.pdg_sim_trace_sweep.argtypes = [C.c_void_p, C.POINTER(C.c_longlong), C.c_int]
cap = 3000000
F = 12
buf = np.zeros(cap * F, np.int64)
for rep in range(2):
    n = L.pdg_sim_trace_sweep(sim._h, buf.ctypes.data_as(C.POINTER(C.c_longlong)), cap)
t = buf[:n * F].reshape(n, F).astype(np.float64)
t0 = t[:, 0].min()
st, dep, stg, done, staged, comp = (t[:, i] - t0 for i in range(6))
task, direc, nbytes, nchunk, height, coarse = (t[:, i] for i in range(6, 12))
span = done.max()
print(f"units {n}: span {span / 1e3:.1f} us, {nbytes.sum() / 1e9:.2f} GB -> {nbytes.sum() / span:.0f} GB/s")
for lab, m in (("chunk fwd", (nchunk == 0) & (direc == 0)), ("chunk bwd", (nchunk == 0) & (direc == 1)),
               ("regular fwd", (nchunk > 0) & (direc == 0)), ("regular bwd", (nchunk > 0) & (direc == 1))):
    if not m.any():
        continue
    tot = (done - st)[m]
    print(f"{lab}: {int(m.sum())} units, {nbytes[m].sum() / 1e9:.2f} GB, mean {nbytes[m].mean() / 1024:.1f} KB; "
          f"CTA time {tot.sum() / 1e6:.1f} ms total -> {nbytes[m].sum() / tot.sum():.2f} GB/s per CTA")
    ck = lab.startswith("chunk")
    # chunk stamps: [0] start, [1] waits done, [4] record in smem, [2] inputs gathered, [5] tiles done, [3] published
    phases = ((("wait", (dep - st)[m]), ("record", (staged - st)[m]), ("gather", (stg - np.maximum(dep, staged))[m]),
               ("tiles", (comp - stg)[m]), ("publish", (done - comp)[m]), ("total", tot),
               ("first tile", height[m]), ("tiles/chunk", coarse[m] * 1e3)) if ck else
              (("wait", (dep - st)[m]), ("stage", (staged - dep)[m]), ("work", (comp - staged)[m]),
               ("publish", (done - comp)[m]), ("total", tot)))
    for ph, v in phases:
        print(f"   {ph:13s} mean {v.mean() / 1e3:6.2f} us  p50 {np.median(v) / 1e3:6.2f}  p90 {np.percentile(v, 90) / 1e3:6.2f}")
edges = np.linspace(0, span, 21)
print("time(us) active chunk-active:")
for e in edges:
    a_ = (st <= e) & (done > e)
    print(f"  {e / 1e3:7.1f} {int(a_.sum()):6d} {int((a_ & (nchunk == 0)).sum()):6d}")
