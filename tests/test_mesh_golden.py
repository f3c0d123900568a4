"""Bit-exact mesh / face / region / agglomeration index maps (north star).

Pinned two ways: against tests/golden/mesh_golden.json (digests produced by
the reference's own compiled mesh sources, scripts/make_golden.py) and, when
oracle/_ref is built, directly against the reference library.
"""
import json

import numpy as np
import pytest

from tests.conftest import ROOT
from paper_2512_19536_b200.mesh import Mesh
from scripts.make_golden import CASES, SLOW_CASES, mesh_record

from tests import refmesh

GOLD = json.loads((ROOT / "tests" / "golden" / "mesh_golden.json").read_text())


def _cases(slow=False):
    for c in CASES + (SLOW_CASES if slow else []):
        key = f"{c[0]}_{c[1]}_{c[2]}_{c[3]}"
        if key in GOLD:
            yield pytest.param(c, id=key, marks=[pytest.mark.slow] if c in SLOW_CASES else [])


@pytest.mark.parametrize("case", list(_cases(slow=True)))
def test_product_mesh_matches_reference_digests(case):
    cells, lloyd, seed, split, targets, levels = case
    gold = GOLD[f"{cells}_{lloyd}_{seed}_{split}"]
    m = Mesh(cells, seed=seed, lloyd=lloyd, split_y=split)
    rec = mesh_record(m.data())
    for k, v in rec.items():
        assert v == gold[k], f"{k} differs from the reference generator"
    for t in targets:
        owner, cnt, H = m.agglomerate(t)
        g = gold["agglomerate"][str(t)]
        assert cnt == g["count"]
        from scripts.make_golden import digest
        assert digest(owner) == g["owner"], f"agglomerate({t}) owner map differs"
        assert digest(H) == g["H"]
    for lv in levels:
        owner, cnt = m.agglomerate_hierarchy(lv)
        from scripts.make_golden import digest
        assert cnt == gold["hierarchy"][str(lv)]["count"]
        assert digest(owner) == gold["hierarchy"][str(lv)]["owner"]


@pytest.mark.skipif(not refmesh.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("cells,lloyd,seed,split", [(1, 0, 2, None), (4, 3, 5, None), (48, 5, 21, 0.5),
                                                   (300, 7, 9, 0.3), (777, 2, 1234, 0.61)])
def test_product_mesh_equals_reference_library(cells, lloyd, seed, split):
    a = Mesh(cells, seed=seed, lloyd=lloyd, split_y=split).data()
    r = refmesh.RefMesh(cells, seed=seed, lloyd=lloyd, split_y=split).data()
    for f in a.__dataclass_fields__:
        assert np.array_equal(getattr(a, f), getattr(r, f)), f


@pytest.mark.skipif(not refmesh.available(), reason="oracle/_ref not built")
def test_agglomeration_equals_reference_library():
    m = Mesh(700, seed=17, lloyd=6, split_y=0.45)
    r = refmesh.RefMesh(700, seed=17, lloyd=6, split_y=0.45)
    for t in (1, 2, 7, 100, 699):
        o1, c1, H1 = m.agglomerate(t)
        o2, c2, H2 = r.agglomerate(t)
        assert c1 == c2 and np.array_equal(o1, o2) and np.array_equal(H1, H2)


def test_mesh_invariants():
    # test_mesh.cpp:82-124 — single seed, congruent quarter cells, 512-cell resolution
    d = Mesh(1, seed=123, lloyd=0, split_y=None).data()
    assert d.n_cells == 1 and abs(d.cell_geo[0, 0] - 1.0) <= 1e-14
    assert len(d.interior_cells) == 0 and len(d.boundary_cells) == 4
    d = Mesh(512, seed=42, lloyd=20, split_y=None).data()
    h = d.cell_geo[:, 3].max()
    assert 0.087 * 0.7 < h < 0.087 * 1.3
    assert abs(d.cell_geo[:, 0].sum() - 1.0) <= 1e-10
    faces = 2 * d.interior_geo[:, 6].sum() + d.boundary_geo[:, 6].sum()
    per = sum(np.linalg.norm(np.roll(d.cell_points(c), -1, 0) - d.cell_points(c), axis=1).sum()
              for c in range(d.n_cells))
    assert abs(faces - per) <= 1e-10 * per
    assert np.all(np.abs(np.linalg.norm(d.interior_geo[:, 4:6], axis=1) - 1.0) <= 1e-14)


def test_partition_invariants():
    # test_mesh.cpp:37-78: region purity, face-connectivity, labels in range
    m = Mesh(2048, seed=42, lloyd=5, split_y=0.5)
    d = m.data()
    owner, cnt, _ = m.agglomerate(64)
    assert cnt == 64 and owner.min() == 0 and owner.max() == 63
    for a in range(cnt):
        assert len(set(d.regions[owner == a])) == 1
    import scipy.sparse as sp
    import scipy.sparse.csgraph as cg
    ic = d.interior_cells
    same = owner[ic[:, 0]] == owner[ic[:, 1]]
    G = sp.coo_matrix((np.ones(same.sum()), (ic[same, 0], ic[same, 1])), shape=(d.n_cells,) * 2)
    ncomp, lab = cg.connected_components(G, directed=False)
    assert ncomp == cnt


def test_quadrature_rules_match_reference():
    from tests.oracle_binding import polygon_quadrature as oq
    from paper_2512_19536_b200.mesh import polygon_quadrature as pq
    d = Mesh(24, seed=4, lloyd=10, split_y=None).data()
    for c in range(d.n_cells):
        poly = d.cell_points(c)
        for order in (3, 4, 6, 8, 10):
            p1, w1 = pq(poly, order)
            p2, w2 = oq(poly, order)
            assert np.array_equal(p1, p2) and np.array_equal(w1, w2)
            if refmesh.available():
                p3, w3 = refmesh.ref_polygon_quadrature(poly, order)
                assert np.array_equal(p1, p3) and np.array_equal(w1, w3)
    # exactness on monomials up to the order (quadrature.hpp:28-31)
    tri = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]])
    p, w = pq(tri, 4)
    assert abs(w.sum() - 0.5) <= 1e-15
    assert abs((w * p[:, 0] ** 2 * p[:, 1] ** 2).sum() - 1.0 / 180.0) <= 1e-15
