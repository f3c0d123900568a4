"""ctypes binding of the C-ABI declared in include/polydg_b200.h.

The shared library is built in-tree (``make -C paper_2512_19536_b200/csrc``)
and is the ONLY compute path: there is no Python/NumPy fallback. Loading fails
loudly if the library is missing.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

import numpy as np

_HERE = pathlib.Path(__file__).resolve().parent
LIB_PATH = _HERE / "libpolydg_b200.so"

PDG_OK = 0
STATUS_NAMES = {2: "ConfigError", 3: "SolverError", 4: "MeshError", 5: "IoError",
                6: "CudaError", 7: "InternalError"}

PRECOND_NONE, PRECOND_BLOCK_JACOBI, PRECOND_TWO_LEVEL = 0, 1, 2
IONIC_NONE, IONIC_FHN, IONIC_BC = 0, 1, 2
INIT_DISC, INIT_CONSTANT, INIT_COSINE, INIT_BILINEAR = 0, 1, 2, 3
STIM_NONE, STIM_STRIP, STIM_COSINE = 0, 1, 2


class PdgConfig(C.Structure):
    _fields_ = [
        ("mesh_cells", C.c_int), ("mesh_seed", C.c_uint64), ("mesh_lloyd", C.c_int),
        ("domain", C.c_double * 4), ("split_y", C.c_double),
        ("degree", C.c_int), ("eta0", C.c_double), ("chi_m", C.c_double), ("C_m", C.c_double),
        ("dt", C.c_double), ("T", C.c_double),
        ("sigma_grey_l", C.c_double), ("sigma_grey_n", C.c_double),
        ("sigma_white_l", C.c_double), ("sigma_white_n", C.c_double),
        ("fiber_grey", C.c_double * 2), ("fiber_white", C.c_double * 2),
        ("fiber_random", C.c_int), ("fiber_seed", C.c_uint64),
        ("ionic_model", C.c_int), ("fhn", C.c_double * 8),
        ("init_kind", C.c_int), ("u_rest", C.c_double), ("u_patch", C.c_double),
        ("omega0", C.c_double * 2), ("omega0_r2", C.c_double), ("init_params", C.c_double * 4),
        ("stim_kind", C.c_int), ("stim_params", C.c_double * 4),
        ("tol", C.c_double), ("maxit", C.c_int), ("warm_start", C.c_int),
        ("precond_kind", C.c_int), ("h_ratio", C.c_int), ("q", C.c_int),
        ("subdomains", C.c_int), ("coarse_count", C.c_int),
        ("rank", C.c_int), ("world", C.c_int), ("device", C.c_int),
        ("bc", C.c_double * 20),
    ]


class StepStats(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("final_residual", C.c_double),
                ("has_condition", C.c_int), ("condition_estimate", C.c_double),
                ("solve_ms", C.c_double), ("step_ms", C.c_double)]


class PcgReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("has_condition", C.c_int),
                ("condition_estimate", C.c_double), ("capacity", C.c_int),
                ("residual_history", C.POINTER(C.c_double)), ("alphas", C.POINTER(C.c_double)),
                ("betas", C.POINTER(C.c_double))]


class OperatorDesc(C.Structure):
    """pdg_operator_desc: K, partition_S and the coarse embedding from the caller."""
    _fields_ = [("n_cells", C.c_int), ("block", C.c_int),
                ("row_ptr", C.POINTER(C.c_int64)), ("col", C.POINTER(C.c_int)), ("val", C.POINTER(C.c_double)),
                ("precond_kind", C.c_int), ("sub_owner", C.POINTER(C.c_int)), ("n_sub", C.c_int),
                ("n_coarse", C.c_int), ("coarse_block", C.c_int),
                ("e_row_ptr", C.POINTER(C.c_int64)), ("e_col", C.POINTER(C.c_int)), ("e_val", C.POINTER(C.c_double)),
                ("maxit", C.c_int), ("device", C.c_int)]


class PdgError(RuntimeError):
    """Raised for a non-OK pdg_status; ``kind`` is the reference exception name."""

    def __init__(self, status: int, message: str):
        self.status = status
        self.kind = STATUS_NAMES.get(status, f"status{status}")
        super().__init__(f"{self.kind}: {message}")


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: build it with "
                              "`make -C paper_2512_19536_b200/csrc` (no CPU fallback exists)")
        L = C.CDLL(str(LIB_PATH))
        vp, i32, i64, dbl = C.c_void_p, C.c_int, C.c_int64, C.c_double
        P = C.POINTER
        sig = {
            "pdg_config_default": (None, [P(PdgConfig)]),
            "pdg_last_error": (C.c_char_p, []),
            "pdg_ionic_rest": (i32, [P(PdgConfig), P(i32), P(dbl), P(dbl)]),
            "pdg_mesh_generate": (i32, [i32, P(dbl), C.c_uint64, i32, dbl, P(vp)]),
            "pdg_mesh_free": (None, [vp]),
            "pdg_mesh_counts": (None, [vp, P(i32)]),
            "pdg_mesh_arrays": (None, [vp, P(dbl), P(i32), P(i32), P(C.c_uint8)]),
            "pdg_mesh_faces": (None, [vp, i32, P(i32), P(dbl)]),
            "pdg_mesh_cell_geometry": (None, [vp, P(dbl)]),
            "pdg_mesh_agglomerate": (i32, [vp, i32, P(i32), P(dbl)]),
            "pdg_mesh_agglomerate_hierarchy": (i32, [vp, i32, P(i32)]),
            "pdg_mesh_coarse_embedding": (i32, [vp, i32, P(i32), i32, i32, P(dbl)]),
            "pdg_polygon_quadrature": (i32, [P(dbl), i32, i32, P(dbl), P(dbl), i32]),
            "pdg_problem_create": (i32, [P(PdgConfig), P(vp)]),
            "pdg_problem_free": (None, [vp]),
            "pdg_problem_info": (None, [vp, P(i64)]),
            "pdg_problem_export": (i64, [vp, i32, P(i64), P(i64), P(dbl)]),
            "pdg_problem_owner": (None, [vp, i32, P(i32)]),
            "pdg_problem_perm": (None, [vp, P(i32)]),
            "pdg_problem_rank_cells": (None, [vp, P(i32)]),
            "pdg_problem_halo": (None, [vp, i32, P(i32), P(i32), P(i32)]),
            "pdg_problem_mesh": (i32, [vp, P(vp)]),
            "pdg_default_max_iterations": (i32, [i64]),
            "pdg_uniform_rhs": (None, [C.c_uint64, i64, P(C.c_double)]),
            "pdg_problem_factor_stats": (None, [vp, P(i64)]),
            "pdg_problem_sweep_stats": (None, [vp, P(i64)]),
            "pdg_problem_flags": (i32, [vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _bind_device(L)
        _lib = L
    return _lib


def _bind_device(L):
    vp, i32, i64, dbl = C.c_void_p, C.c_int, C.c_int64, C.c_double
    P = C.POINTER
    sig = {
        "pdg_sim_create": (i32, [P(PdgConfig), P(vp)]),
        "pdg_sim_create_from_operator": (i32, [P(OperatorDesc), P(vp)]),
        "pdg_sim_free": (None, [vp]),
        "pdg_sim_problem": (vp, [vp]),
        "pdg_sim_dimension": (i64, [vp]),
        "pdg_sim_step": (i32, [vp, P(StepStats)]),
        "pdg_sim_get_state": (i32, [vp, P(i32), P(dbl), P(dbl), P(dbl), P(dbl), P(dbl)]),
        "pdg_sim_set_state": (i32, [vp, i32, P(dbl), P(dbl), P(dbl), P(dbl)]),
        "pdg_sim_apply_K": (i32, [vp, P(dbl), P(dbl)]),
        "pdg_sim_apply_precond": (i32, [vp, P(dbl), P(dbl)]),
        "pdg_sim_cell_means": (i32, [vp, P(dbl)]),
        "pdg_sim_export_snapshot": (i32, [vp, C.c_char_p, C.c_char_p]),
        "pdg_sim_pcg": (i32, [vp, P(dbl), P(dbl), dbl, i32, i32, P(dbl), P(PcgReport)]),
        "pdg_sim_pcg_device": (i32, [vp, vp, vp, dbl, i32, vp, P(PcgReport)]),
        "pdg_condition_estimate": (i32, [P(dbl), P(dbl), i32, P(dbl)]),
        "pdg_nccl_unique_id_bytes": (i32, []),
        "pdg_nccl_get_unique_id": (i32, [vp]),
        "pdg_sim_attach_comm": (i32, [vp, vp, i32, i32]),
        "pdg_loopback_create": (i32, [i32, P(vp)]),
        "pdg_loopback_free": (None, [vp]),
        "pdg_sim_attach_loopback": (i32, [vp, vp, i32, i32]),
        "pdg_sim_timer": (i32, [vp, i32, P(dbl)]),
        "pdg_sim_kernel_launches": (i64, [vp]),
        "pdg_sim_profile": (i32, [vp, i32, P(dbl), P(i64)]),
        "pdg_sim_sweep_live": (i32, [vp, P(i64), P(dbl)]),
        "pdg_sim_trace_sweep": (i32, [vp, P(i64), i32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name, None)
        if f is None:
            continue
        f.restype = res
        f.argtypes = args


def check(status: int) -> None:
    if status != PDG_OK:
        msg = lib().pdg_last_error()
        raise PdgError(status, msg.decode() if msg else "")


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def iptr(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_int))


def lptr(a: np.ndarray):
    assert a.dtype == np.int64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_int64))


def uniform_rhs(seed: int, n: int):
    """BASELINE config-5 right-hand side: 2 (rng()>>11) 2^-53 - 1, mt19937_64(seed)
    (proj/tests/acceptance.cpp:285-286)."""
    import numpy as np
    out = np.zeros(int(n))
    lib().pdg_uniform_rhs(C.c_uint64(seed), int(n), out.ctypes.data_as(C.POINTER(C.c_double)))
    return out


def default_config(**kw) -> PdgConfig:
    cfg = PdgConfig()
    lib().pdg_config_default(C.byref(cfg))
    for k, v in kw.items():
        if not hasattr(cfg, k):
            raise KeyError(f"unknown config key {k!r}")
        cur = getattr(cfg, k)
        if isinstance(cur, C.Array):
            for i, x in enumerate(v):
                cur[i] = x
        else:
            setattr(cfg, k, v)
    return cfg


def env_threads() -> int:
    return int(os.environ.get("POLYDG_THREADS", os.cpu_count() or 1))
