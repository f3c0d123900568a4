"""Generates tests/golden/mesh_golden.json from the REFERENCE's own mesh code.

Run here (where /root/reference exists): `make -C oracle ref && python scripts/make_golden.py`.
For every case it records SHA-256 digests of the reference generator's vertex
coordinates (raw float64 bytes), cell loops, regions, interior/boundary faces,
per-cell geometry and agglomeration owner maps, plus a few plain numbers. The
product's mesh/agglomeration code is then checked against these digests on any
machine (tests/test_mesh_golden.py), so the bit-exact claim does not depend on
/root/reference at test time.
"""
from __future__ import annotations

import hashlib
import json
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from tests.refmesh import RefMesh  # noqa: E402

# (cells, lloyd, seed, split_y, agglomeration targets, hierarchy levels)
CASES = [
    (1, 0, 123, None, [], []),
    (12, 3, 77, None, [3], []),
    (24, 10, 4, 0.5, [6], [1]),
    (64, 20, 42, 0.5, [16], [1]),
    (512, 20, 42, 0.5, [128, 16], [1, 2, 3]),
    (1024, 5, 42, 0.5, [16, 256], [1]),           # BASELINE config 1 (S = 16)
    (2048, 20, 42, 0.5, [512], [1]),
    (16384, 5, 42, 0.5, [64], []),                # BASELINE config 2 (S = 64)
    (65536, 5, 42, 0.5, [64, 256], []),           # BASELINE config 3 (S = 64 / 256)
]
SLOW_CASES = [
    (1048576, 5, 42, 0.5, [512, 1024], []),       # BASELINE configs 4/5
]


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def mesh_record(d) -> dict:
    return {
        "n_cells": int(d.n_cells), "n_vertices": int(len(d.vertices)),
        "n_interior": int(len(d.interior_cells)), "n_boundary": int(len(d.boundary_cells)),
        "vertices": digest(d.vertices), "cell_off": digest(d.cell_off), "cell_vtx": digest(d.cell_vtx),
        "regions": digest(d.regions), "interior_cells": digest(d.interior_cells),
        "interior_geo": digest(d.interior_geo), "boundary_cells": digest(d.boundary_cells),
        "boundary_geo": digest(d.boundary_geo), "cell_geo": digest(d.cell_geo),
        "h": float(d.cell_geo[:, 3].max()),
    }


def main(slow: bool = False):
    out = {}
    for cells, lloyd, seed, split, targets, levels in CASES + (SLOW_CASES if slow else []):
        t0 = time.time()
        m = RefMesh(cells, seed=seed, lloyd=lloyd, split_y=split)
        rec = mesh_record(m.data())
        rec["agglomerate"] = {}
        for t in targets:
            owner, cnt, H = m.agglomerate(t)
            rec["agglomerate"][str(t)] = {"count": int(cnt), "owner": digest(owner), "H": digest(H),
                                          "sizes_min_max": [int(np.bincount(owner).min()),
                                                            int(np.bincount(owner).max())]}
        rec["hierarchy"] = {}
        for lv in levels:
            owner, cnt = m.agglomerate_hierarchy(lv)
            rec["hierarchy"][str(lv)] = {"count": int(cnt), "owner": digest(owner)}
        key = f"{cells}_{lloyd}_{seed}_{split}"
        out[key] = rec
        print(key, f"{time.time() - t0:.1f}s", rec["n_interior"], flush=True)
    dst = ROOT / "tests" / "golden" / "mesh_golden.json"
    old = json.loads(dst.read_text()) if dst.exists() else {}
    old.update(out)
    dst.write_text(json.dumps(old, indent=1, sort_keys=True))


if __name__ == "__main__":
    main(slow="--slow" in sys.argv)
