#!/usr/bin/env python
"""Benchmark of the per-time-step solve (BASELINE.json metric) on B200.

A "step" is one Crank-Nicolson step of the PolyDG monodomain system
(Simulation::step, /root/reference/proj/src/timestepper.cpp:144-200): ionic
terms at quadrature nodes, CN right-hand side, two-level-Schwarz PCG to rtol
1e-8, explicit ionic-state update. Workload: BASELINE config 2 (16,384
Voronoi cells, p = 3, 64 subdomains = 64 coarse agglomerates, grey/white
anisotropy), synthetic seeded mesh and data.

    value  = PCG DOF-iterations/s = n_dofs * sum(PCG iterations) / device time,
             whole job over all ranks (max-over-ranks device time)
    e2e    = the same metric through the public C-ABI with the state held on
             the host: every step set_state (H2D from pinned memory) -> step ->
             get_state (D2H)
    --impl reference: the reference's CPU path (the Eigen-free restatement in
             oracle/, since the reference itself cannot be built here) on the
             same workload with all host threads.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Multi-GPU: python -m torch.distributed.run --nproc-per-node N bench.py --gpus N
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import pathlib
import statistics
import subprocess
import sys
import time

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "PCG DOF-iterations/s and solve time per CN step; % of HBM roofline, 1/2/4/8 GPU"
UNIT = "DOF-iter/s"
KERNELS = ["spmv", "update", "restrict", "sweep", "restrict_combine", "prolong_dot", "pupdate", "ionic", "rhs"]
REF_BUDGET_S = 150.0


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def workload_config(name, rank=0, world=1, device=0, scaling="weak"):
    """The BASELINE workload. Weak scaling (default) keeps the per-GPU problem
    at the config's size: N GPUs solve one coupled mesh of N x cells with
    N x subdomains (one halo exchange + all-reduces per PCG iteration);
    strong scaling shards the config's own mesh over the N GPUs."""
    from paper_2512_19536_b200 import configs
    cfg = getattr(configs, name)()
    if scaling == "weak" and world > 1:
        cfg.cells *= world
        cfg.subdomains *= world
    cfg.rank, cfg.world, cfg.device = rank, world, device
    return cfg


def workload_desc(cfg):
    return (f"{cfg.cells} seeded Voronoi cells (lloyd {cfg.lloyd}), p={cfg.degree}, "
            f"{cfg.subdomains} subdomains = {cfg.subdomains} coarse agglomerates (q=p), grey/white "
            f"anisotropy with per-element fibres, FHN ionics, dt={cfg.dt} ms, rtol {cfg.tol}")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = pathlib.Path(f"/tmp/pdg_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.device)], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for line in self.path.read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7 and parts[0].isdigit():
                rows.append(parts)
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(float(r[0]) for r in rows), "sm_max_mhz": float(rows[0][1]),
                "reasons": reasons, "samples": len(rows)}


def cpu_baseline(cfg, budget_s=20.0, min_steps=1):
    """Times the oracle port (reference algorithm, reference threading) on the workload."""
    from tests.oracle_binding import lib as orc_lib, oracle_for
    t0 = time.perf_counter()
    orc, _ = oracle_for(cfg)
    setup = time.perf_counter() - t0
    n = orc.dimension
    its, steps, t0 = 0, 0, time.perf_counter()
    while True:
        its += orc.step()["iterations"]
        steps += 1
        el = time.perf_counter() - t0
        if steps >= min_steps and el >= budget_s:
            break
        if el + el / steps > budget_s * 1.5 and steps >= min_steps:
            break
    return {"value": n * its / el, "unit": UNIT, "cores": orc_lib().orc_threads(), "kind": "port",
            "sample": f"{steps} CN steps of the workload ({its} PCG iterations, {el:.1f} s) after {setup:.1f} s "
                      f"untimed setup; oracle/ restatement (reference cannot be built: Eigen3 absent)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # the arm's own workload (weak scaling: N x the config's mesh), solved by
    # the single-process CPU oracle
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    cfg = workload_config(args.config, 0, world, 0, args.scaling)
    cfg.rank, cfg.world = 0, 1
    from tests.oracle_binding import lib as orc_lib, oracle_for
    orc, _ = oracle_for(cfg)
    n = orc.dimension
    for _ in range(args.warmup):
        orc.step()
    its, done, t0 = 0, 0, time.perf_counter()
    for _ in range(args.steps):
        its += orc.step()["iterations"]
        done += 1
        if time.perf_counter() - t0 > REF_BUDGET_S:
            break
    el = time.perf_counter() - t0
    value = n * its / el
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * el / done, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{args.config}: " + workload_desc(cfg), "dofs": n},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": orc_lib().orc_threads(), "kind": "port",
                             "sample": f"{done} of {args.steps} requested CN steps timed "
                                       f"(budget {REF_BUDGET_S:.0f} s), {its} PCG iterations"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="config2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")

    from paper_2512_19536_b200 import _lib
    from paper_2512_19536_b200.simulation import Simulation
    L = _lib.lib()
    cfg = workload_config(args.config, rank, world, local, args.scaling)
    sim = Simulation(cfg)
    if world > 1:
        nb = L.pdg_nccl_unique_id_bytes()
        uid = (C.c_char * nb)()
        if rank == 0:
            _lib.check(L.pdg_nccl_get_unique_id(uid))
        t = torch.tensor(list(bytearray(uid.raw)), dtype=torch.uint8)
        dist.broadcast(t, 0)
        uid = (C.c_char * nb).from_buffer_copy(bytes(t.tolist()))
        _lib.check(L.pdg_sim_attach_comm(sim._h, uid, rank, world))
    n_global = sim.dimension

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t)
        return float(t.item())

    for _ in range(args.warmup):
        sim.step()
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    launches0 = L.pdg_sim_kernel_launches(sim._h)
    live_n0, live_ms0 = C.c_int64(), C.c_double()
    _lib.check(L.pdg_sim_sweep_live(sim._h, C.byref(live_n0), C.byref(live_ms0)))
    ms = C.c_double()
    barrier()
    _lib.check(L.pdg_sim_timer(sim._h, 0, None))
    its, solve_ms = 0, 0.0
    for _ in range(args.steps):
        s = sim.step()
        its += s.iterations
        solve_ms += s.solve_ms
    _lib.check(L.pdg_sim_timer(sim._h, 1, C.byref(ms)))
    barrier()
    clk = clocks.stop()
    launches = L.pdg_sim_kernel_launches(sim._h) - launches0
    live_n1, live_ms1 = C.c_int64(), C.c_double()
    _lib.check(L.pdg_sim_sweep_live(sim._h, C.byref(live_n1), C.byref(live_ms1)))
    # the sweep's average launch duration inside the timed region (device
    # globaltimer, first CTA start -> last CTA end), max over ranks
    sweep_live_ms = max_over_ranks((live_ms1.value - live_ms0.value) / max(1, live_n1.value - live_n0.value))
    sweep_live_launches = live_n1.value - live_n0.value
    elapsed_ms = max_over_ranks(ms.value)
    value = n_global * its / (elapsed_ms * 1e-3)

    # ---- e2e: state on the host, round-tripped through the C-ABI every step ----
    n, nc = sim.dimension, sim.n_comp
    pin = lambda m: torch.empty(m, dtype=torch.float64, pin_memory=True).numpy()
    hU, hUp, hY, hYp = pin(n), pin(n), pin(max(nc, 1) * n), pin(max(nc, 1) * n)
    k0, _, U, Up, Y, Yp = sim.state()
    hU[:], hUp[:] = U, Up
    hY[:nc * n], hYp[:nc * n] = Y.ravel(), Yp.ravel()
    d = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
    kk = C.c_int()
    t_ = C.c_double()
    e2e_its = 0
    e2e_steps = max(1, min(args.steps, 50))
    barrier()
    _lib.check(L.pdg_sim_timer(sim._h, 0, None))
    st = _lib.StepStats()
    for i in range(e2e_steps):
        # inputs of this step (host-owned state) -> device
        _lib.check(L.pdg_sim_set_state(sim._h, k0 + i, d(hU), d(hUp), d(hY), d(hYp)))
        _lib.check(L.pdg_sim_step(sim._h, C.byref(st)))
        e2e_its += st.iterations
        # result -> host (the new state the host integrator keeps)
        hUp[:] = hU
        hYp[:] = hY
        _lib.check(L.pdg_sim_get_state(sim._h, C.byref(kk), C.byref(t_), d(hU), None, d(hY), None))
    e2e_ms = C.c_double()
    _lib.check(L.pdg_sim_timer(sim._h, 1, C.byref(e2e_ms)))
    barrier()
    e2e_value = n_global * sum_over_ranks(e2e_its) / world / (max_over_ranks(e2e_ms.value) * 1e-3)
    h2d = (2 + 2 * nc) * n * 8
    d2h = (1 + nc) * n * 8

    # ---- per-kernel device times for the roofline ----
    kms = (C.c_double * 9)()
    kby = (C.c_int64 * 9)()
    _lib.check(L.pdg_sim_profile(sim._h, 20, kms, kby))
    per_step = {"spmv": its / args.steps, "update": its / args.steps}
    for k in ("restrict", "sweep", "restrict_combine", "prolong_dot", "pupdate"):
        per_step[k] = its / args.steps + 1
    per_step["rhs"] = 1
    per_step["ionic"] = 1
    # the sweep's duration as measured live inside the timed region replaces
    # its isolated (cold-L2) profile time
    iso_sweep_ms = kms[KERNELS.index("sweep")]
    if sweep_live_launches > 0:
        kms[KERNELS.index("sweep")] = sweep_live_ms
    shares = {k: kms[i] * per_step.get(k, 0) / (elapsed_ms / args.steps) for i, k in enumerate(KERNELS)}
    dom = max(shares, key=shares.get)
    di = KERNELS.index(dom)
    peak, peak_kind = peaks()
    achieved = kby[di] / (kms[di] * 1e-3) / 1e9
    timing = ("live: device globaltimer per launch inside the timed region, "
              f"{sweep_live_launches} launches" if dom == "sweep" and sweep_live_launches > 0
              else "isolated launches, L2 flushed before each")
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get(args.config, {}).get(dom)
    # bytes of one whole PCG iteration vs its device time (all kernels of the body)
    iter_bytes = sum(kby[KERNELS.index(k)] for k in ("spmv", "update", "restrict", "sweep", "restrict_combine",
                                                      "prolong_dot", "pupdate"))
    iter_ms = sum(kms[KERNELS.index(k)] for k in ("spmv", "update", "restrict", "sweep", "restrict_combine",
                                                   "prolong_dot", "pupdate"))

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(workload_config(args.config))
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "port", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: " + workload_desc(cfg), "dofs": n_global,
                       "steps_timed": args.steps, "pcg_iterations": its,
                       "avg_iterations_per_step": its / args.steps,
                       "solve_ms_per_step": solve_ms / args.steps,
                       "l2": "operands (K 91 MB + Schwarz panels 408 MB) exceed the 126 MB L2; "
                             "per-kernel profile times flush L2 before each launch",
                       "parallelism": f"subdomains sharded over {world} GPU(s)" + (
                           f" ({args.config} per GPU: {cfg.cells} cells, {cfg.subdomains} subdomains in total)"
                           if args.scaling == "weak" and world > 1 else "")},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "algorithmic_bytes_per_launch": int(kby[di]),
                         "launch_ms": kms[di], "launch_timing": timing, "share_of_step": shares[dom],
                         "sweep_isolated_ms": iso_sweep_ms,
                         "pcg_iteration": {"bytes": int(iter_bytes), "kernel_ms": iter_ms,
                                           "GB/s": iter_bytes / (iter_ms * 1e-3) / 1e9 if iter_ms else None},
                         "kernels": {k: {"ms": kms[i], "bytes": int(kby[i]),
                                         "GB/s": (kby[i] / (kms[i] * 1e-3) / 1e9) if kms[i] else None,
                                         "share": shares[k]} for i, k in enumerate(KERNELS)}},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "steps": e2e_steps},
            "gpu_launches": int(sum_over_ranks(launches)),
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
