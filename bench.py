#!/usr/bin/env python
"""Benchmark of the per-time-step solve (BASELINE.json metric) on B200.

A "step" is one Crank-Nicolson step of the PolyDG monodomain system
(Simulation::step, /root/reference/proj/src/timestepper.cpp:144-200): ionic
terms at quadrature nodes, CN right-hand side, two-level-Schwarz PCG to rtol
1e-8, explicit ionic-state update. Default workload: BASELINE config 4 (the
config the metric's 1/2/4/8-GPU figures are quoted on): 1,048,576 seeded
Voronoi cells, p = 3 (10.5 M dofs), 512 subdomains = 512 coarse agglomerates,
grey/white anisotropy with per-element fibres, strip stimulus, FHN.

    value  = PCG DOF-iterations/s = n_dofs * sum(PCG iterations) / device time
             of the timed steps (whole job, max over ranks)
    e2e    = the same metric through the public C-ABI with the state held on
             the host: every step set_state (H2D from pinned memory) -> step ->
             get_state (D2H)
    roofline: the Schwarz sweep (dominant kernel) against the measured HBM
             peak, bytes per SURVEY §8(d): 2 * 8 * nnz(L) (structural, local +
             coarse factors) + r read / z write; stored panel bytes separately
    --impl reference: the reference's CPU path (oracle/ restatement; the
             reference's numeric sources need Eigen, which is absent) on the
             same config, mesh and partitions from the reference's own
             compiled mesh code (oracle/_ref), no product library loaded.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
       [--config config4|config2|...] [--scaling strong|weak]
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
L2_BYTES = 126 * 2**20
REF_BUDGET_S = 75.0        # timed CPU work of the reference arm (bounded sample)
REF_ITERS_PER_STEP = 2     # PCG iterations per reference-arm step
CPU_BASELINE_S = 20.0


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def workload_config(name, rank=0, world=1, device=0, scaling="strong"):
    """The BASELINE workload. Strong scaling (default) shards the config's own
    mesh over the N GPUs (whole subdomains per rank); weak scaling solves one
    coupled mesh of N x cells with N x subdomains."""
    from paper_2512_19536_b200 import configs
    cfg = getattr(configs, name)()
    if scaling == "weak" and world > 1:
        cfg.cells *= world
        cfg.subdomains *= world
    cfg.rank, cfg.world, cfg.device = rank, world, device
    return cfg


def config_json(name, cfg, world, scaling):
    """The `config` object both arms print (computed without any library)."""
    b = (cfg.degree + 1) * (cfg.degree + 2) // 2
    q = cfg.q if cfg.q > 0 else cfg.degree
    aniso = cfg.sigma_white_l != cfg.sigma_white_n or cfg.sigma_grey_l != cfg.sigma_grey_n
    stim = "none"
    if cfg.stimulus and cfg.stimulus[0] == "strip":
        stim = f"strip x<{cfg.stimulus[2]} for t<{cfg.stimulus[3]} ms, {cfg.stimulus[1]:g} uA/cm^3"
    return {
        "workload": name,
        "mesh": f"{cfg.cells} seeded Voronoi cells (seed {cfg.seed}, lloyd {cfg.lloyd}), unit square",
        "degree": cfg.degree, "dofs": cfg.cells * b,
        "subdomains": cfg.subdomains, "coarse_agglomerates": cfg.subdomains if cfg.coarse == -1 else cfg.coarse,
        "coarse_degree": q,
        "conductivity": ("grey/white anisotropic, per-element fibres" if aniso and cfg.fiber_random
                         else "anisotropic" if aniso else "isotropic"),
        "ionic": cfg.ionic_model, "stimulus": stim, "dt_ms": cfg.dt, "rtol": cfg.tol,
        "l2": f"no flush needed: the operands streamed by one PCG iteration (K ~{8 * cfg.cells * 7 * b * b / 1e9:.2f} GB "
              f"plus Schwarz factors > {2 * 8 * cfg.cells * 10 * b * b / 1e9:.2f} GB) exceed the {L2_BYTES >> 20} MB L2",
        "parallelism": f"{world} GPU(s), whole subdomains per rank, {scaling} scaling",
    }


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


def time_oracle_iterations(orc, budget_s, iters_per_sample, max_samples=None, warmup=1):
    """Times bounded samples of PCG iterations on the oracle: each sample is
    `iters_per_sample` iterations (SpMV, Schwarz local + coarse apply, vector
    updates; tol 1e-300 so the sample never stops early) from the warm start
    U^k on a seeded right-hand side. Returns (samples, iterations, seconds)."""
    from tests import oracle_binding as ob
    n = orc.dimension
    b = ob.uniform_rhs(42, n)
    x0 = orc.state()[2]
    for _ in range(warmup):
        orc.pcg_solve(b, 1e-300, maxit=iters_per_sample, x0=x0)
    samples, its, t0 = 0, 0, time.perf_counter()
    while True:
        _, rep = orc.pcg_solve(b, 1e-300, maxit=iters_per_sample, x0=x0)
        its += rep["iterations"]
        samples += 1
        el = time.perf_counter() - t0
        if max_samples is not None and samples >= max_samples:
            break
        if el >= budget_s or el + el / samples > 1.5 * budget_s:
            break
    return samples, its, time.perf_counter() - t0


def cpu_baseline(cfg, budget_s=CPU_BASELINE_S):
    """The oracle port (reference algorithm and threading) on the workload."""
    from tests import oracle_binding as ob
    ob.set_parallel(False)   # the reference's single-threaded SpMV / vector ops
    ob.set_lean(1)
    t0 = time.perf_counter()
    orc, _ = ob.oracle_for(cfg)
    setup = time.perf_counter() - t0
    n = orc.dimension
    samples, its, el = time_oracle_iterations(orc, budget_s, REF_ITERS_PER_STEP)
    return {"value": n * its / el, "unit": UNIT, "cores": ob.lib().orc_threads(), "kind": "port",
            "sample": f"{its} PCG iterations ({samples} x {REF_ITERS_PER_STEP}) of the workload's system in "
                      f"{el:.1f} s after {setup:.0f} s untimed setup; oracle/ restatement with the reference's "
                      f"threading (parallel_for local solves, serial SpMV/vector ops); the reference's numeric "
                      f"sources build here only against an Eigen API stand-in without Eigen's SIMD kernels "
                      f"(oracle/eigen_shim, a parity oracle), so the restatement is the timed baseline"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    from paper_2512_19536_b200 import configs  # dataclasses only; no library is loaded
    cfg = getattr(configs, args.config)()
    if args.scaling == "weak" and world > 1:
        cfg.cells *= world
        cfg.subdomains *= world
    from tests import oracle_binding as ob
    ob.set_parallel(False)
    ob.set_lean(1)
    t0 = time.perf_counter()
    orc, _ = ob.oracle_for(cfg, reference_mesh=True)
    setup = time.perf_counter() - t0
    n = orc.dimension
    for _ in range(min(args.warmup, 1)):
        orc.pcg_solve(ob.uniform_rhs(42, n), 1e-300, maxit=REF_ITERS_PER_STEP, x0=orc.state()[2])
    samples, its, el = time_oracle_iterations(orc, REF_BUDGET_S, REF_ITERS_PER_STEP, max_samples=args.steps,
                                              warmup=0)
    value = n * its / el
    loaded = sorted({p for p in _loaded_libs() if str(ROOT) in p})
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * el / samples, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_json(args.config, cfg, world, args.scaling),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": ob.lib().orc_threads(), "kind": "port",
                             "sample": f"{samples} of {args.steps} requested steps timed, each step = "
                                       f"{REF_ITERS_PER_STEP} PCG iterations of the workload's CN system "
                                       f"({its} iterations, {el:.1f} s, budget {REF_BUDGET_S:.0f} s) after "
                                       f"{setup:.0f} s untimed setup (mesh and partitions by the reference's own "
                                       f"compiled mesh code, oracle/_ref); ms_per_step is per sampled step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "native_libs": loaded}
    print(json.dumps(line), flush=True)


def _loaded_libs():
    try:
        return [l.split()[-1] for l in open("/proc/self/maps") if l.rstrip().endswith(".so")]
    except OSError:
        return []


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="config4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--scaling", default="strong", choices=["weak", "strong"])
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
    t_setup = time.perf_counter()
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
    setup_s = time.perf_counter() - t_setup
    n_global = sim.dimension

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    def reduce(x, op):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=op)
        return float(t.item())

    max_over_ranks = lambda x: reduce(x, dist.ReduceOp.MAX if dist else None)
    sum_over_ranks = lambda x: reduce(x, dist.ReduceOp.SUM if dist else None)

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
    its, solve_ms, per_step_its = 0, 0.0, []
    for _ in range(args.steps):
        s = sim.step()
        its += s.iterations
        per_step_its.append(s.iterations)
        solve_ms += s.solve_ms
    _lib.check(L.pdg_sim_timer(sim._h, 1, C.byref(ms)))
    barrier()
    clk = clocks.stop()
    launches = L.pdg_sim_kernel_launches(sim._h) - launches0
    live_n1, live_ms1 = C.c_int64(), C.c_double()
    _lib.check(L.pdg_sim_sweep_live(sim._h, C.byref(live_n1), C.byref(live_ms1)))
    # the sweep's average launch duration inside the timed region (device
    # globaltimer, first CTA start -> last CTA end), max over ranks
    sweep_live_launches = live_n1.value - live_n0.value
    sweep_live_ms = max_over_ranks((live_ms1.value - live_ms0.value) / max(1, sweep_live_launches))
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
    kk, t_ = C.c_int(), C.c_double()
    e2e_its = 0
    e2e_steps = max(1, min(args.steps, 5))
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

    # ---- per-kernel device times; the sweep's live time replaces its cold one ----
    kms = (C.c_double * 9)()
    kby = (C.c_int64 * 9)()
    _lib.check(L.pdg_sim_profile(sim._h, 10, kms, kby))
    stats = sim.problem.factor_stats()
    per_step = {"spmv": its / args.steps, "update": its / args.steps}
    for k in ("restrict", "sweep", "restrict_combine", "prolong_dot", "pupdate"):
        per_step[k] = its / args.steps + 1
    per_step["rhs"] = per_step["ionic"] = 1
    iso_sweep_ms = kms[KERNELS.index("sweep")]
    if sweep_live_launches > 0:
        kms[KERNELS.index("sweep")] = sweep_live_ms
    step_ms = elapsed_ms / args.steps
    shares = {k: kms[i] * per_step.get(k, 0) / step_ms for i, k in enumerate(KERNELS)}
    dom = "sweep"
    di = KERNELS.index(dom)
    peak, peak_kind = peaks()
    # SURVEY §8(d) algorithmic bytes of one Schwarz apply (this rank): forward +
    # backward over the structural local factors and the coarse factor, r in, z out
    N_local = sim.problem.cell_end - sim.problem.cell_begin
    n_local = N_local * sim.problem.n_local
    sweep_alg = 2 * 8 * (stats["l_struct"] + stats["l0_struct"]) + 16 * n_local
    sweep_stored = int(kby[di])
    achieved = sweep_alg / (kms[di] * 1e-3) / 1e9
    traffic = None
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    if tfile.exists():
        traffic = json.loads(tfile.read_text()).get(args.config, {}).get(dom)
    # whole PCG iteration by §8(d): K + row structure, factors, E^T and E, 12 vectors
    qd = cfg.q if cfg.q > 0 else cfg.degree
    b, bq = sim.problem.n_local, (qd + 1) * (qd + 2) // 2
    iter_alg = (8 * stats["k_blocks"] * b * b + 4 * stats["k_blocks"] + 4 * (N_local + 1)
                + 2 * 8 * (stats["l_struct"] + stats["l0_struct"]) + 2 * 8 * N_local * b * bq + 12 * 8 * n_local)
    iter_ms = solve_ms / its if its else None
    iter_frac = max_over_ranks(iter_alg / (iter_ms * 1e-3) / 1e9) / peak if iter_ms else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(workload_config(args.config))
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": UNIT, "cores": None, "kind": "port", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_json(args.config, cfg, world, args.scaling),
            "stats": {"pcg_iterations": its, "iterations_per_step": per_step_its,
                      "solve_ms_per_step": solve_ms / args.steps, "setup_s": round(setup_s, 1)},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "algorithmic_bytes_per_launch": sweep_alg,
                         "algorithmic_bytes": "SURVEY 8(d): 2*8*(nnz(L_loc)+nnz(L_0)) structural (this "
                                              "implementation's ordering) + 16 n (r in, z out)",
                         "nnz_L_loc": stats["l_struct"], "nnz_L0": stats["l0_struct"],
                         "stored_panel_bytes_per_launch": sweep_stored,
                         "stored_GB/s": sweep_stored / (kms[di] * 1e-3) / 1e9,
                         "launch_ms": kms[di],
                         "launch_timing": f"live: device globaltimer per launch inside the timed region, "
                                          f"{sweep_live_launches} launches",
                         "share_of_step": shares[dom], "sweep_isolated_ms": iso_sweep_ms,
                         "pcg_iteration": {"algorithmic_bytes": iter_alg, "ms": iter_ms, "frac": iter_frac,
                                           "note": "SpMV + Schwarz apply + E/E^T + 12 vectors per SURVEY 8(d) "
                                                   "over the device time of the solves / iterations"},
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
