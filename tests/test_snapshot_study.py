"""Snapshot (cell means) and scaling-study harness on the device path.

Reference behaviour: snapshot.cpp:13-75 (cell_means, vtk-legacy /
csv-cellmeans writers, unknown format -> ConfigError) and study.cpp:20-176
(one row per combination, CSV header, paper-style table).
"""
import io

import numpy as np
import pytest

from paper_2512_19536_b200._lib import PdgError
from paper_2512_19536_b200.simulation import Simulation, SimulationConfig
from paper_2512_19536_b200.study import (StudyRow, StudySpec, run_scaling_study, write_study_csv,
                                          write_study_table)
from tests.conftest import gpu_available
from tests.oracle_binding import oracle_for

gpu = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def test_study_writers_follow_reference_layout(tmp_path):
    rows = [StudyRow(N_h=64, h=0.25, ratio=2, N_H=16, p=1, q=1, precond="two-level", avg_iters=7.5,
                     cond_est=12.0, cond_mean=11.0, wall_s=0.5),
            StudyRow(N_h=64, h=0.25, ratio=0, p=1, q=1, precond="none", avg_iters=30.0, converged=False)]
    write_study_csv(rows, str(tmp_path / "s.csv"))
    lines = (tmp_path / "s.csv").read_text().splitlines()
    assert lines[0].startswith("N_h,h,ratio,N_H,p,q,precond,avg_iters,cond_est,wall_s,converged")
    assert lines[1].split(",")[:11] == ["64", "0.25", "2", "16", "1", "1", "two-level", "7.5", "12",
                                        "0.5", "1"]
    buf = io.StringIO()
    write_study_table(rows, buf)
    txt = buf.getvalue()
    assert txt.startswith("condition estimate max-step/mean (average PCG iterations per step)\n")
    assert "p = 1, q = 1" in txt and "12/11 (7.5)" in txt
    assert "   CG | failed" in txt


@pytest.mark.parametrize("kw", [dict(cells=256, degree=2, subdomains=8, coarse=-1, fiber_random=True),
                                dict(cells=300, degree=3, initial=("cosine", 10.0, -60.0))])
@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_cell_means_match_oracle(kw):
    cfg = SimulationConfig(dt=0.01, T=0.03, tol=1e-8, **kw)
    sim = Simulation(cfg)
    orc, _ = oracle_for(cfg)
    for _ in range(2):
        sim.step()
    U = sim.state()[2]
    m, mo = sim.cell_means(), orc.cell_means(U)
    assert m.shape == mo.shape
    assert np.abs(m - mo).max() <= 1e-12 * np.abs(mo).max()


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_export_snapshot_formats(tmp_path):
    cfg = SimulationConfig(cells=64, degree=1, initial=("bilinear", -60.0, 5.0, 2.0, 0.0), dt=0.01, T=0.01)
    sim = Simulation(cfg)
    means = sim.cell_means()
    mesh = sim.problem.mesh().data()
    # a bilinear field without cross term is affine: the mean is its centroid value
    ctr = mesh.cell_geo[:, 1:3]
    assert np.allclose(means, -60.0 + 5.0 * ctr[:, 0] + 2.0 * ctr[:, 1], rtol=0, atol=1e-9)
    sim.export_snapshot(str(tmp_path / "u.csv"), "csv-cellmeans")
    lines = (tmp_path / "u.csv").read_text().splitlines()
    assert lines[0] == "cell_id,centroid_x,centroid_y,u_mean" and len(lines) == 65
    c, cx, cy, u = lines[5].split(",")
    assert int(c) == 4 and float(u) == means[4] and float(cx) == ctr[4, 0]
    sim.export_snapshot(str(tmp_path / "u.vtk"), "vtk-legacy")
    vtk = (tmp_path / "u.vtk").read_text().splitlines()
    assert vtk[0] == "# vtk DataFile Version 3.0" and vtk[1].startswith("polydg transmembrane potential t=0 ms")
    assert vtk[4] == f"POINTS {len(mesh.vertices)} double"
    assert f"CELL_DATA 64" in vtk and float(vtk[-1]) == means[-1]
    with pytest.raises(PdgError) as e:
        sim.export_snapshot(str(tmp_path / "u.x"), "png")
    assert e.value.status == 2 and "unknown snapshot format 'png'" in str(e.value)
    with pytest.raises(PdgError) as e:
        sim.export_snapshot(str(tmp_path / "missing" / "u.csv"), "csv-cellmeans")
    assert e.value.status == 5


@pytest.mark.gpu
@pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")
def test_study_rows_match_oracle_iterations(tmp_path):
    base = SimulationConfig(dt=0.01, T=0.03, tol=1e-8, initial=("disc",))
    spec = StudySpec(cells=[128], ratios=[2, 4], degrees=[(1, 1), (2, 1)], kinds=["two-level", "none"], base=base)
    rows = run_scaling_study(spec, out_dir=str(tmp_path))
    assert len(rows) == 8 and all(r.converged for r in rows)
    assert (tmp_path / "study.csv").exists() and (tmp_path / "study.txt").exists()
    for r in rows:
        import dataclasses
        cfg = dataclasses.replace(base, cells=r.N_h, degree=r.p, precond=r.precond, h_ratio=r.ratio, q=r.q)
        orc, _ = oracle_for(cfg)
        its = [orc.step()["iterations"] for _ in range(cfg.n_steps())]
        assert abs(r.avg_iters - np.mean(its)) <= 1.0, (r, its)
        assert r.dof_iter_per_s > 0
