"""Scaling-study harness on the device path (mirrors polydg/study.hpp, study.cpp).

`run_scaling_study` runs every (mesh size, degree pair, coarse ratio,
preconditioner) combination of a `StudySpec` through the device `Simulation`
(study.cpp:20-74); a failing combination becomes a non-converged row instead
of aborting the study. `write_study_csv` / `write_study_table` reproduce the
reference's CSV header and paper-style table (study.cpp:76-176).

Beyond the reference's columns each row also carries the device throughput
(`dofs`, `total_iterations`, `solve_s`, `dof_iter_per_s`), which is what the
BASELINE config-3 robustness sweep reports per (p, subdomain count); the
`subdomains` / `coarse` extensions of `SimulationConfig` select the
multi-cell partitions of that sweep.
"""
from __future__ import annotations

import dataclasses
import io
import os
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

from ._lib import PdgError
from .simulation import Simulation, SimulationConfig


@dataclass
class StudySpec:
    """StudySpec (config.hpp:17-23)."""
    cells: Sequence[int]
    ratios: Sequence[int] = (2,)
    degrees: Sequence[Tuple[int, int]] = ((1, 1),)
    kinds: Sequence[str] = ("two-level",)
    base: SimulationConfig = field(default_factory=SimulationConfig)
    # ext (config 3): subdomain counts swept per combination; 0 = the reference's
    # one cell per subdomain with the h_ratio coarse hierarchy
    subdomains: Sequence[int] = (0,)


@dataclass
class StudyRow:
    """StudyRow (study.hpp:14-28) + device throughput columns."""
    N_h: int = 0
    h: float = 0.0
    ratio: int = 0
    N_H: int = 0
    p: int = 0
    q: int = 0
    precond: str = "none"
    avg_iters: float = 0.0
    cond_est: Optional[float] = None
    cond_mean: Optional[float] = None
    wall_s: float = 0.0
    converged: bool = True
    subdomains: int = 0
    dofs: int = 0
    total_iterations: int = 0
    solve_s: float = 0.0
    dof_iter_per_s: float = 0.0


def run_scaling_study(spec: StudySpec, out_dir: Optional[str] = None, steps: Optional[int] = None,
                      log=None) -> List[StudyRow]:
    """study.cpp:20-74 (and :165-176 when out_dir is given)."""
    rows: List[StudyRow] = []
    for n_h in spec.cells:
        h = 0.0
        for p, q in spec.degrees:
            for ratio in spec.ratios:
                for kind in spec.kinds:
                    for S in spec.subdomains:
                        row = StudyRow(N_h=n_h, ratio=ratio, p=p, q=q, precond=kind, subdomains=S)
                        t0 = time.perf_counter()
                        try:
                            cfg = dataclasses.replace(spec.base, cells=n_h, degree=p, precond=kind,
                                                      h_ratio=ratio, q=q, subdomains=S,
                                                      coarse=-1 if S > 0 else 0)
                            sim = Simulation(cfg)
                            mesh = sim.problem.mesh().data()
                            h = float(mesh.cell_geo[:, 3].max())
                            row.h = h
                            row.dofs = sim.dimension
                            if kind == "two-level":
                                row.N_H = sim.problem.coarse_dim // ((q + 1) * (q + 2) // 2)
                            res = sim.run(steps)
                            row.avg_iters = res.avg_iterations
                            row.cond_est = res.cond_at_max_iter_step
                            row.cond_mean = res.cond_mean
                            row.converged = res.converged_all
                            row.total_iterations = sum(s.iterations for s in res.steps)
                            row.solve_s = sum(s.solve_ms for s in res.steps) * 1e-3
                            if row.solve_s > 0:
                                row.dof_iter_per_s = row.dofs * row.total_iterations / row.solve_s
                            sim.close()
                        except PdgError as e:
                            if log:
                                log(f"study: combination N_h={n_h} p={p} ratio={ratio} precond={kind} "
                                    f"failed: {e}")
                            row.h = h
                            row.converged = False
                        row.wall_s = time.perf_counter() - t0
                        rows.append(row)
                        if log:
                            log(row)
    if out_dir is not None:
        os.makedirs(out_dir, exist_ok=True)
        write_study_csv(rows, os.path.join(out_dir, "study.csv"))
        with open(os.path.join(out_dir, "study.txt"), "w") as f:
            write_study_table(rows, f)
    return rows


def _g17(x: float) -> str:
    return "%.17g" % x


def write_study_csv(rows: Sequence[StudyRow], path: str) -> None:
    """study.cpp:76-89: fixed header, 17 significant digits; device columns appended."""
    try:
        with open(path, "w") as out:
            out.write("N_h,h,ratio,N_H,p,q,precond,avg_iters,cond_est,wall_s,converged,"
                      "subdomains,dofs,total_iterations,solve_s,dof_iter_per_s\n")
            for r in rows:
                out.write(f"{r.N_h},{_g17(r.h)},{r.ratio},{r.N_H},{r.p},{r.q},{r.precond},"
                          f"{_g17(r.avg_iters)},{_g17(r.cond_est or 0.0)},{_g17(r.wall_s)},"
                          f"{1 if r.converged else 0},{r.subdomains},{r.dofs},{r.total_iterations},"
                          f"{_g17(r.solve_s)},{_g17(r.dof_iter_per_s)}\n")
    except OSError as e:
        raise PdgError(5, f"cannot open study csv for writing: {path}") from e


def _cell_text(r: StudyRow) -> str:
    if not r.converged:
        return "failed"
    if r.cond_est is not None and r.cond_mean is not None:
        return "%.4g/%.4g (%.4g)" % (r.cond_est, r.cond_mean, r.avg_iters)
    return "- (%.4g)" % r.avg_iters


def write_study_table(rows: Sequence[StudyRow], out: io.TextIOBase) -> None:
    """study.cpp:104-163: one block per (p, q); rows = coarse ratios, then BJ / CG."""
    degree_pairs = sorted({(r.p, r.q) for r in rows})
    meshes = sorted({r.N_h for r in rows})
    ratios = sorted({r.ratio for r in rows if r.precond == "two-level"})

    def find(p, q, n_h, kind, ratio):
        for r in rows:
            if r.p == p and r.q == q and r.N_h == n_h and r.precond == kind and \
                    (kind != "two-level" or r.ratio == ratio):
                return r
        return None

    out.write("condition estimate max-step/mean (average PCG iterations per step)\n")
    for p, q in degree_pairs:
        out.write(f"\np = {p}, q = {q}\n")
        h_of = {r.N_h: r.h for r in rows if r.p == p and r.h > 0.0}
        out.write("      ")
        for n_h in meshes:
            out.write("| " + "h=%-7.3g N=%-6d" % (h_of.get(n_h, 0.0), n_h))
        out.write("\n")
        for ratio in ratios:
            out.write("%4dh " % ratio)
            for n_h in meshes:
                r = find(p, q, n_h, "two-level", ratio)
                out.write("| %-22s" % (_cell_text(r) if r else "-"))
            out.write("\n")
        for kind in ("block-jacobi", "none"):
            if not any(r.p == p and r.q == q and r.precond == kind for r in rows):
                continue
            out.write("%5s " % ("CG" if kind == "none" else "BJ"))
            for n_h in meshes:
                r = find(p, q, n_h, kind, 0)
                out.write("| %-22s" % (_cell_text(r) if r else "-"))
            out.write("\n")


def write_throughput_table(rows: Sequence[StudyRow], out: io.TextIOBase) -> None:
    """Config-3 view: iterations/step and DOF-iter/s per (p, subdomains)."""
    out.write("| p | subdomains | dofs | avg iterations/step | DOF-iter/s | solve s | converged |\n")
    out.write("|---|---|---|---|---|---|---|\n")
    for r in rows:
        out.write(f"| {r.p} | {r.subdomains} | {r.dofs:,} | {r.avg_iters:.2f} | {r.dof_iter_per_s:.3g} | "
                  f"{r.solve_s:.3f} | {int(r.converged)} |\n")
