"""Host mesh API (mirrors /root/reference/proj/include/polydg/mesh.hpp:15-130).

Thin NumPy views over the C-ABI; the generator and agglomerator run in the
native library and are bit-exact with the reference (tests/test_mesh_golden.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import check, dptr, iptr, lib

UNIT = (0.0, 0.0, 1.0, 1.0)


@dataclass
class MeshData:
    vertices: np.ndarray      # (nv, 2)
    cell_off: np.ndarray      # (nc+1,)
    cell_vtx: np.ndarray      # (corners,)
    regions: np.ndarray       # (nc,) uint8, 0 = Grey, 1 = White
    interior_cells: np.ndarray  # (nf, 2) cell_in, cell_out
    interior_geo: np.ndarray    # (nf, 7) a.x a.y b.x b.y n.x n.y length
    boundary_cells: np.ndarray
    boundary_geo: np.ndarray
    cell_geo: np.ndarray        # (nc, 4) area cx cy diameter

    @property
    def n_cells(self) -> int:
        return len(self.regions)

    def cell_points(self, c: int) -> np.ndarray:
        return self.vertices[self.cell_vtx[self.cell_off[c]:self.cell_off[c + 1]]]


class Mesh:
    """Owning handle of a native pdg_mesh."""

    def __init__(self, n_cells: int, domain=UNIT, seed: int = 42, lloyd: int = 20,
                 split_y: float | None = 0.5):
        L = lib()
        self._h = C.c_void_p()
        d = (C.c_double * 4)(*domain)
        split = -1e300 if split_y is None else float(split_y)
        check(L.pdg_mesh_generate(int(n_cells), d, C.c_uint64(seed), int(lloyd), split, C.byref(self._h)))

    @classmethod
    def _adopt(cls, handle):
        obj = cls.__new__(cls)
        obj._h = handle
        return obj

    def __del__(self):
        if getattr(self, "_h", None):
            lib().pdg_mesh_free(self._h)
            self._h = None

    def data(self) -> MeshData:
        return _read_mesh(lib(), self._h, "pdg_")

    def agglomerate(self, target: int) -> tuple[np.ndarray, int, np.ndarray]:
        nc = self.data().n_cells if not hasattr(self, "_nc") else self._nc
        owner = np.zeros(nc, np.int32)
        H = np.zeros(nc, np.float64)
        cnt = lib().pdg_mesh_agglomerate(self._h, int(target), iptr(owner), dptr(H))
        if cnt < 0:
            check(3 if b"target" not in lib().pdg_last_error() else 2)
        return owner, cnt, H[:cnt]

    def coarse_embedding(self, p: int, owner: np.ndarray, count: int, q: int):
        """build_coarse_embedding(space, partition, q) (schwarz.hpp:38-39): E as a
        scipy CSR matrix (n_cells*b x count*bq), one b x bq block per element."""
        import scipy.sparse as sp
        nc = self.data().n_cells
        b, bq = (p + 1) * (p + 2) // 2, (q + 1) * (q + 2) // 2
        own = np.ascontiguousarray(owner, np.int32)
        blocks = np.zeros(nc * b * bq)
        check(lib().pdg_mesh_coarse_embedding(self._h, int(p), iptr(own), int(count), int(q), dptr(blocks)))
        blocks = blocks.reshape(nc, bq, b)  # column-major b x bq per element
        rows = (np.arange(nc)[:, None, None] * b + np.arange(b)[None, None, :]).repeat(bq, 1)
        cols = (own[:, None, None] * bq + np.arange(bq)[None, :, None]).repeat(b, 2)
        return sp.csr_matrix((blocks.ravel(), (rows.ravel(), cols.ravel())), shape=(nc * b, count * bq))

    def agglomerate_hierarchy(self, levels: int) -> tuple[np.ndarray, int]:
        nc = self.data().n_cells
        owner = np.zeros(nc, np.int32)
        cnt = lib().pdg_mesh_agglomerate_hierarchy(self._h, int(levels), iptr(owner))
        if cnt < 0:
            check(2)
        return owner, cnt


def _read_mesh(L, h, prefix: str) -> MeshData:
    counts = (C.c_int * 5)()
    getattr(L, prefix + "mesh_counts")(h, counts)
    nc, nv, ncorner, nint, nbnd = list(counts)
    verts = np.zeros((nv, 2))
    off = np.zeros(nc + 1, np.int32)
    idx = np.zeros(ncorner, np.int32)
    reg = np.zeros(nc, np.uint8)
    getattr(L, prefix + "mesh_arrays")(h, dptr(verts), iptr(off), iptr(idx),
                                       reg.ctypes.data_as(C.POINTER(C.c_uint8)))
    ic = np.zeros((nint, 2), np.int32)
    ig = np.zeros((nint, 7))
    bc = np.zeros((nbnd, 2), np.int32)
    bg = np.zeros((nbnd, 7))
    getattr(L, prefix + "mesh_faces")(h, 1, iptr(ic), dptr(ig))
    getattr(L, prefix + "mesh_faces")(h, 0, iptr(bc), dptr(bg))
    cg = np.zeros((nc, 4))
    getattr(L, prefix + "mesh_cell_geometry")(h, dptr(cg))
    return MeshData(verts, off, idx, reg, ic, ig, bc, bg, cg)


def polygon_quadrature(poly: np.ndarray, order: int) -> tuple[np.ndarray, np.ndarray]:
    poly = np.ascontiguousarray(poly, dtype=np.float64)
    cap = 4096
    pts = np.zeros((cap, 2))
    w = np.zeros(cap)
    n = lib().pdg_polygon_quadrature(dptr(poly), len(poly), int(order), dptr(pts), dptr(w), cap)
    if n < 0:
        check(4)
    return pts[:n].copy(), w[:n].copy()
