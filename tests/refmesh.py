"""TEST INFRASTRUCTURE: ctypes binding of oracle/_ref/libpolydg_ref.so, the
reference's own mesh/agglomeration sources compiled by oracle/Makefile.

Only tests (and scripts generating tests/golden) import this module.
"""
from __future__ import annotations

import ctypes as C
import pathlib

import numpy as np

from paper_2512_19536_b200.mesh import MeshData, _read_mesh

ROOT = pathlib.Path(__file__).resolve().parents[1]
REF_LIB = ROOT / "oracle" / "_ref" / "libpolydg_ref.so"

_ref = None


def available() -> bool:
    return REF_LIB.exists()


def ref():
    global _ref
    if _ref is None:
        L = C.CDLL(str(REF_LIB))
        vp, i32, dbl = C.c_void_p, C.c_int, C.c_double
        P = C.POINTER
        L.ref_mesh_generate.restype = vp
        L.ref_mesh_generate.argtypes = [i32, dbl, dbl, dbl, dbl, C.c_uint64, i32, dbl]
        L.ref_mesh_free.argtypes = [vp]
        L.ref_mesh_counts.argtypes = [vp, P(i32)]
        L.ref_mesh_arrays.argtypes = [vp, P(dbl), P(i32), P(i32), P(C.c_uint8)]
        L.ref_mesh_faces.argtypes = [vp, i32, P(i32), P(dbl)]
        L.ref_mesh_cell_geometry.argtypes = [vp, P(dbl)]
        L.ref_agglomerate.restype = i32
        L.ref_agglomerate.argtypes = [vp, i32, P(i32), P(dbl)]
        L.ref_agglomerate_hierarchy.restype = i32
        L.ref_agglomerate_hierarchy.argtypes = [vp, i32, P(i32)]
        L.ref_polygon_quadrature.restype = i32
        L.ref_polygon_quadrature.argtypes = [P(dbl), i32, i32, P(dbl), P(dbl), i32]
        L.ref_gauss_legendre.restype = i32
        L.ref_gauss_legendre.argtypes = [i32, P(dbl), P(dbl)]
        L.ref_last_error.restype = C.c_char_p
        _ref = L
    return _ref


class RefMesh:
    def __init__(self, n, domain=(0.0, 0.0, 1.0, 1.0), seed=42, lloyd=20, split_y=0.5):
        L = ref()
        split = -1e300 if split_y is None else split_y
        self._h = L.ref_mesh_generate(n, *domain, C.c_uint64(seed), lloyd, split)
        if not self._h:
            raise RuntimeError(L.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "_h", None):
            ref().ref_mesh_free(self._h)

    def data(self) -> MeshData:
        if getattr(self, "_data", None) is not None:
            return self._data
        L = ref()
        # the ref shim uses the same argument layout as the product's mesh readers
        class _Shim:
            mesh_counts = L.ref_mesh_counts
            mesh_arrays = L.ref_mesh_arrays
            mesh_faces = L.ref_mesh_faces
            mesh_cell_geometry = L.ref_mesh_cell_geometry
        self._data = _read_mesh(_Shim, self._h, "")
        return self._data

    def agglomerate(self, target):
        nc = self.data().n_cells
        owner = np.zeros(nc, np.int32)
        H = np.zeros(nc)
        cnt = ref().ref_agglomerate(self._h, target, owner.ctypes.data_as(C.POINTER(C.c_int)),
                                    H.ctypes.data_as(C.POINTER(C.c_double)))
        if cnt < 0:
            raise RuntimeError(ref().ref_last_error().decode())
        return owner, cnt, H[:cnt]

    def agglomerate_hierarchy(self, levels):
        nc = self.data().n_cells
        owner = np.zeros(nc, np.int32)
        cnt = ref().ref_agglomerate_hierarchy(self._h, levels, owner.ctypes.data_as(C.POINTER(C.c_int)))
        return owner, cnt


def ref_polygon_quadrature(poly, order):
    poly = np.ascontiguousarray(poly, dtype=np.float64)
    cap = 4096
    pts = np.zeros((cap, 2))
    w = np.zeros(cap)
    n = ref().ref_polygon_quadrature(poly.ctypes.data_as(C.POINTER(C.c_double)), len(poly), order,
                                     pts.ctypes.data_as(C.POINTER(C.c_double)),
                                     w.ctypes.data_as(C.POINTER(C.c_double)), cap)
    return pts[:n].copy(), w[:n].copy()
