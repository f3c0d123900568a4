"""TEST INFRASTRUCTURE: ctypes binding of oracle/_ref/libpolydg_refnum.so, the
reference's OWN numeric sources (proj/src/{dg_space,assembly,ionics,krylov,
schwarz,timestepper,snapshot}.cpp) compiled where they lie with the Eigen API
stand-in oracle/eigen_shim (oracle/Makefile target `refnum`).

It exists only where /root/reference was present at build time (this
container); GPU-box tests that need it skip when it is absent.
"""
from __future__ import annotations

import ctypes as C
import pathlib

import numpy as np

from paper_2512_19536_b200._lib import PdgConfig

ROOT = pathlib.Path(__file__).resolve().parents[1]
LIB = ROOT / "oracle" / "_ref" / "libpolydg_refnum.so"
_L = None


def available() -> bool:
    return LIB.exists()


class RefReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("has_condition", C.c_int),
                ("condition_estimate", C.c_double), ("capacity", C.c_int),
                ("residual_history", C.POINTER(C.c_double)), ("alphas", C.POINTER(C.c_double)),
                ("betas", C.POINTER(C.c_double)), ("n_resid", C.c_int), ("n_alpha", C.c_int),
                ("n_beta", C.c_int)]


class RefError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        self.kind = {2: "ConfigError", 3: "SolverError"}.get(status, "Error")
        super().__init__(f"{self.kind}: {msg}")


def lib():
    global _L
    if _L is None:
        L = C.CDLL(str(LIB))
        vp, i32, i64, dbl, P = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.POINTER
        sigs = {
            "refn_last_error": (C.c_char_p, []),
            "refn_config_size": (i32, []),
            "refn_sim_create": (i32, [P(PdgConfig), P(vp)]),
            "refn_sim_free": (None, [vp]),
            "refn_sim_dimension": (i64, [vp]),
            "refn_sim_n_comp": (i32, [vp]),
            "refn_sim_step": (i32, [vp, P(i32), P(i32), P(dbl), P(i32), P(dbl)]),
            "refn_sim_state": (i32, [vp, P(i32), P(dbl), P(dbl), P(dbl), P(dbl), P(dbl)]),
            "refn_sim_export": (i64, [vp, i32, P(i64), P(i64), P(dbl)]),
            "refn_sim_apply_K": (i32, [vp, P(dbl), P(dbl)]),
            "refn_sim_apply_precond": (i32, [vp, P(dbl), P(dbl)]),
            "refn_sim_pcg": (i32, [vp, P(dbl), P(dbl), dbl, i32, i32, P(dbl), P(RefReport)]),
            "refn_l2_error_cosine": (i32, [vp, P(dbl), dbl, dbl, dbl, P(dbl)]),
            "refn_mesh_size": (dbl, [vp]),
            "refn_cell_means": (i32, [vp, P(dbl), P(dbl)]),
        }
        for k, (r, a) in sigs.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        assert L.refn_config_size() == C.sizeof(PdgConfig)
        _L = L
    return _L


def _d(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def _check(st):
    if st != 0:
        raise RefError(st, lib().refn_last_error().decode())


class RefSim:
    """The reference's polydg::Simulation (agglomerated subdomains swapped in
    through its own SchwarzPreconditioner when config.subdomains > 0)."""

    def __init__(self, config):
        from tests.oracle_binding import oracle_config
        cfg = oracle_config(config)
        self._h = C.c_void_p()
        _check(lib().refn_sim_create(C.byref(cfg), C.byref(self._h)))
        self.dimension = lib().refn_sim_dimension(self._h)
        self.n_comp = lib().refn_sim_n_comp(self._h)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().refn_sim_free(self._h)
            self._h = None

    def step(self):
        it, cv, hc = C.c_int(), C.c_int(), C.c_int()
        fr, cond = C.c_double(), C.c_double()
        _check(lib().refn_sim_step(self._h, C.byref(it), C.byref(cv), C.byref(fr), C.byref(hc), C.byref(cond)))
        return dict(iterations=it.value, converged=bool(cv.value), final_residual=fr.value,
                    condition_estimate=cond.value if hc.value else None)

    def state(self):
        n, nc = self.dimension, self.n_comp
        U, Up = np.zeros(n), np.zeros(n)
        Y, Yp = np.zeros(max(nc, 1) * n), np.zeros(max(nc, 1) * n)
        k, t = C.c_int(), C.c_double()
        _check(lib().refn_sim_state(self._h, C.byref(k), C.byref(t), _d(U), _d(Up), _d(Y), _d(Yp)))
        return k.value, t.value, U, Up, Y[:nc * n].reshape(nc, n), Yp[:nc * n].reshape(nc, n)

    def export(self, which):
        import scipy.sparse as sp
        w = {"K": 0, "M": 1, "A": 2, "E": 3, "K0": 4}[which]
        nnz = lib().refn_sim_export(self._h, w, None, None, None)
        if nnz < 0:
            raise ValueError(which)
        r, c, v = np.zeros(nnz, np.int64), np.zeros(nnz, np.int64), np.zeros(nnz)
        lib().refn_sim_export(self._h, w, r.ctypes.data_as(C.POINTER(C.c_int64)),
                              c.ctypes.data_as(C.POINTER(C.c_int64)), _d(v))
        shape = (int(r.max()) + 1, int(c.max()) + 1)
        if which in ("K", "M", "A"):
            shape = (self.dimension, self.dimension)
        return sp.csr_matrix((v, (r, c)), shape=shape)

    def apply_K(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.dimension)
        _check(lib().refn_sim_apply_K(self._h, _d(x), _d(y)))
        return y

    def apply_precond(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.zeros(self.dimension)
        _check(lib().refn_sim_apply_precond(self._h, _d(r), _d(z)))
        return z

    def pcg_solve(self, b, tol, maxit=0, x0=None, use_precond=True):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x0a = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
        x = np.zeros(self.dimension)
        cap = (maxit if maxit > 0 else 20 * int(np.sqrt(self.dimension)) + 1) + 2
        hist = [np.zeros(cap) for _ in range(3)]
        rep = RefReport()
        rep.capacity = cap
        rep.residual_history, rep.alphas, rep.betas = (_d(h) for h in hist)
        _check(lib().refn_sim_pcg(self._h, _d(b), _d(x0a), tol, maxit, int(use_precond), _d(x), C.byref(rep)))
        return x, dict(iterations=rep.iterations, converged=bool(rep.converged),
                       residual_history=hist[0][:rep.n_resid].copy(), alphas=hist[1][:rep.n_alpha].copy(),
                       betas=hist[2][:rep.n_beta].copy(),
                       condition_estimate=rep.condition_estimate if rep.has_condition else None)

    def l2_error_cosine(self, U, c0, c1, t):
        e = C.c_double()
        _check(lib().refn_l2_error_cosine(self._h, _d(np.ascontiguousarray(U, dtype=np.float64)), c0, c1, t,
                                          C.byref(e)))
        return e.value

    def mesh_size(self):
        return lib().refn_mesh_size(self._h)
