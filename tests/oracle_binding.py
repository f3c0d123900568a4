"""TEST INFRASTRUCTURE: ctypes binding of the CPU oracle (oracle/build/libpdg_oracle.so).

The oracle is an Eigen-free restatement of the reference's numeric path
(oracle/src/*.cpp). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg use it; the product never does.
"""
from __future__ import annotations

import ctypes as C
import pathlib
import subprocess

import numpy as np

from paper_2512_19536_b200._lib import PdgConfig
from paper_2512_19536_b200.simulation import SimulationConfig

ROOT = pathlib.Path(__file__).resolve().parents[1]
ORACLE_LIB = ROOT / "oracle" / "build" / "libpdg_oracle.so"

_L = None


class OrcReport(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("has_condition", C.c_int),
                ("condition_estimate", C.c_double), ("capacity", C.c_int),
                ("residual_history", C.POINTER(C.c_double)), ("alphas", C.POINTER(C.c_double)),
                ("betas", C.POINTER(C.c_double)), ("n_resid", C.c_int), ("n_alpha", C.c_int),
                ("n_beta", C.c_int)]


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        self.status = status
        self.kind = {2: "ConfigError", 3: "SolverError"}.get(status, "Error")
        super().__init__(f"{self.kind}: {msg}")


def lib():
    global _L
    if _L is None:
        if not ORACLE_LIB.exists():
            subprocess.run(["make", "-C", str(ROOT / "oracle"), "oracle"], check=True,
                           capture_output=True)
        L = C.CDLL(str(ORACLE_LIB))
        vp, i32, i64, dbl, P = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.POINTER
        sigs = {
            "orc_last_error": (C.c_char_p, []),
            "orc_config_size": (i32, []),
            "orc_threads": (i32, []),
            "orc_sim_create": (i32, [P(PdgConfig), P(dbl), i32, P(i32), P(i32), i32, P(C.c_uint8),
                                     P(i32), i32, P(i32), i32, P(vp)]),
            "orc_sim_free": (None, [vp]),
            "orc_sim_step": (i32, [vp, P(i32), P(i32), P(dbl), P(i32), P(dbl)]),
            "orc_sim_state": (i32, [vp, P(i32), P(dbl), P(dbl), P(dbl), P(dbl), P(dbl)]),
            "orc_sim_set_state": (i32, [vp, i32, P(dbl), P(dbl), P(dbl), P(dbl)]),
            "orc_sim_dimension": (i64, [vp]),
            "orc_sim_apply_K": (i32, [vp, P(dbl), P(dbl)]),
            "orc_sim_apply_precond": (i32, [vp, P(dbl), P(dbl)]),
            "orc_sim_pcg": (i32, [vp, P(dbl), P(dbl), dbl, i32, i32, P(dbl), P(OrcReport)]),
            "orc_sim_export": (i64, [vp, i32, P(i64), P(i64), P(dbl)]),
            "orc_sim_ionic_terms": (i32, [vp, P(dbl), P(dbl), P(dbl), P(dbl)]),
            "orc_sim_cell_means": (i32, [vp, P(dbl), P(dbl)]),
            "orc_pcg_dense": (i32, [i32, P(dbl), P(dbl), P(dbl), dbl, i32, P(dbl), P(dbl), P(OrcReport)]),
            "orc_condition_estimate": (i32, [P(dbl), P(dbl), i32, P(dbl)]),
            "orc_fhn": (i32, [P(dbl), dbl, dbl, P(dbl), P(dbl)]),
            "orc_bc": (i32, [P(dbl), dbl, P(dbl), P(dbl), P(dbl)]),
            "orc_ionic_rest": (i32, [P(PdgConfig), P(i32), P(dbl), P(dbl)]),
            "orc_polygon_quadrature": (i32, [P(dbl), i32, i32, P(dbl), P(dbl), i32]),
            "orc_set_parallel": (None, [i32]),
            "orc_set_lean": (None, [i32]),
            "orc_config_default": (None, [P(PdgConfig)]),
            "orc_uniform_rhs": (None, [C.c_uint64, i64, P(dbl)]),
            "orc_sim_factor_blocks": (i64, [vp, i32]),
            "orc_l2_error_cosine": (i32, [vp, P(dbl), dbl, dbl, dbl, P(dbl)]),
            "orc_mesh_size": (dbl, [vp]),
        }
        for k, (r, a) in sigs.items():
            f = getattr(L, k)
            f.restype, f.argtypes = r, a
        assert L.orc_config_size() == C.sizeof(PdgConfig), "oracle/product config layouts differ"
        _L = L
    return _L


def oracle_config(config: SimulationConfig) -> PdgConfig:
    """config.to_c() on the oracle's own defaults (does not load the product library)."""
    base = PdgConfig()
    lib().orc_config_default(C.byref(base))
    return config.to_c(base)


def set_parallel(on: bool) -> None:
    """Row-parallel CSR products in the oracle (same bits; large parity runs only)."""
    lib().orc_set_parallel(int(on))


def set_lean(level: int) -> None:
    """1: drop M, A after setup; 2: also skip K_rhs (single-solve workloads)."""
    lib().orc_set_lean(int(level))


def uniform_rhs(seed: int, n: int) -> np.ndarray:
    """b_i = 2 (rng()>>11) 2^-53 - 1, mt19937_64(seed) (acceptance.cpp:285-286)."""
    out = np.zeros(int(n))
    lib().orc_uniform_rhs(C.c_uint64(seed), int(n), _d(out))
    return out


def _d(a):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))


def _i(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _check(st):
    if st != 0:
        raise OracleError(st, lib().orc_last_error().decode())


def _report(cap):
    hist = [np.zeros(cap) for _ in range(3)]
    rep = OrcReport()
    rep.capacity = cap
    rep.residual_history, rep.alphas, rep.betas = (_d(h) for h in hist)
    return rep, hist


def _unpack(rep, hist):
    return dict(iterations=rep.iterations, converged=bool(rep.converged),
                residual_history=hist[0][:rep.n_resid].copy(), alphas=hist[1][:rep.n_alpha].copy(),
                betas=hist[2][:rep.n_beta].copy(),
                condition_estimate=rep.condition_estimate if rep.has_condition else None)


def pcg_dense(A, b, P=None, tol=1e-10, maxit=0, x0=None):
    A = np.ascontiguousarray(A, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    n = len(b)
    Pm = None if P is None else np.ascontiguousarray(P, dtype=np.float64)
    x0a = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
    x = np.zeros(n)
    rep, hist = _report((maxit if maxit > 0 else n) + 2 + 20 * int(np.sqrt(n)))
    _check(lib().orc_pcg_dense(n, _d(A), _d(b), _d(Pm), tol, maxit, _d(x0a), _d(x), C.byref(rep)))
    return x, _unpack(rep, hist)


def condition_estimate(alphas, betas):
    a = np.ascontiguousarray(alphas, dtype=np.float64)
    b = np.ascontiguousarray(betas if len(betas) else [0.0], dtype=np.float64)
    k = C.c_double()
    return k.value if lib().orc_condition_estimate(_d(a), _d(b), len(a), C.byref(k)) else None


def fhn(u, w, params=None):
    prm = np.array(params if params is not None else [0.13, 0.013, 0.26, 0.1, 1.0, -85.0, 20.0, 1.0])
    f, m = C.c_double(), C.c_double()
    _check(lib().orc_fhn(_d(prm), u, w, C.byref(f), C.byref(m)))
    return f.value, m.value


def barreto_cressman(u, y, params=None):
    """Pointwise (current, rates) of the oracle's Barreto-Cressman restatement."""
    from paper_2512_19536_b200._lib import default_config
    prm = np.array(params if params is not None else list(default_config().bc))
    ya = np.ascontiguousarray(y, dtype=np.float64)
    f, m = C.c_double(), np.zeros(4)
    _check(lib().orc_bc(_d(prm), u, _d(ya), C.byref(f), _d(m)))
    return f.value, m


def ionic_rest(config):
    cfg = config.to_c()
    nc, u, y = C.c_int(), C.c_double(), np.zeros(4)
    _check(lib().orc_ionic_rest(C.byref(cfg), C.byref(nc), C.byref(u), _d(y)))
    return nc.value, u.value, list(y[:nc.value])


def polygon_quadrature(poly, order):
    poly = np.ascontiguousarray(poly, dtype=np.float64)
    pts, w = np.zeros((4096, 2)), np.zeros(4096)
    n = lib().orc_polygon_quadrature(_d(poly), len(poly), order, _d(pts), _d(w), 4096)
    return pts[:n].copy(), w[:n].copy()


class OracleSim:
    """CPU restatement of polydg::Simulation on a given mesh + partitions."""

    def __init__(self, config: SimulationConfig, mesh, sub_owner, n_sub, coarse_owner=None, n_coarse=0):
        self.config = config
        cfg = oracle_config(config)
        verts = np.ascontiguousarray(mesh.vertices, dtype=np.float64)
        off = np.ascontiguousarray(mesh.cell_off, dtype=np.int32)
        idx = np.ascontiguousarray(mesh.cell_vtx, dtype=np.int32)
        reg = np.ascontiguousarray(mesh.regions, dtype=np.uint8)
        so = np.ascontiguousarray(sub_owner, dtype=np.int32)
        co = None if coarse_owner is None else np.ascontiguousarray(coarse_owner, dtype=np.int32)
        self._h = C.c_void_p()
        _check(lib().orc_sim_create(C.byref(cfg), _d(verts), len(verts), _i(off), _i(idx), len(reg),
                                    reg.ctypes.data_as(C.POINTER(C.c_uint8)), _i(so), int(n_sub),
                                    None if co is None else _i(co), int(n_coarse), C.byref(self._h)))
        self.dimension = lib().orc_sim_dimension(self._h)
        self.n_comp = {"fhn": 1, "barreto-cressman": 4}.get(config.ionic_model, 0)
        self.regions = reg

    def __del__(self):
        if getattr(self, "_h", None):
            lib().orc_sim_free(self._h)
            self._h = None

    def step(self):
        it, cv, hc = C.c_int(), C.c_int(), C.c_int()
        fr, cond = C.c_double(), C.c_double()
        _check(lib().orc_sim_step(self._h, C.byref(it), C.byref(cv), C.byref(fr), C.byref(hc), C.byref(cond)))
        return dict(iterations=it.value, converged=bool(cv.value), final_residual=fr.value,
                    condition_estimate=cond.value if hc.value else None)

    def state(self):
        n, nc = self.dimension, self.n_comp
        U, Up = np.zeros(n), np.zeros(n)
        Y, Yp = np.zeros(max(nc, 1) * n), np.zeros(max(nc, 1) * n)
        k, t = C.c_int(), C.c_double()
        _check(lib().orc_sim_state(self._h, C.byref(k), C.byref(t), _d(U), _d(Up), _d(Y), _d(Yp)))
        return k.value, t.value, U, Up, Y[:nc * n].reshape(nc, n), Yp[:nc * n].reshape(nc, n)

    def set_state(self, k, U, Up=None, Y=None, Yp=None):
        c = lambda a: None if a is None else np.ascontiguousarray(a, dtype=np.float64).ravel()
        arrs = [c(a) for a in (U, Up, Y, Yp)]
        _check(lib().orc_sim_set_state(self._h, int(k), *[_d(a) for a in arrs]))

    def apply_K(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.dimension)
        _check(lib().orc_sim_apply_K(self._h, _d(x), _d(y)))
        return y

    def apply_precond(self, r):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.zeros(self.dimension)
        _check(lib().orc_sim_apply_precond(self._h, _d(r), _d(z)))
        return z

    def pcg_solve(self, b, tol, maxit=0, x0=None, use_precond=True):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x0a = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
        x = np.zeros(self.dimension)
        rep, hist = _report((maxit if maxit > 0 else 20 * int(np.sqrt(self.dimension)) + 1) + 2)
        _check(lib().orc_sim_pcg(self._h, _d(b), _d(x0a), tol, maxit, int(use_precond), _d(x), C.byref(rep)))
        return x, _unpack(rep, hist)

    def export(self, which):
        import scipy.sparse as sp
        w = {"K": 0, "M": 1, "A": 2, "E": 3, "K0": 4, "Krhs": 5}[which]
        nnz = lib().orc_sim_export(self._h, w, None, None, None)
        if nnz < 0:
            raise ValueError(which)
        r, c, v = np.zeros(nnz, np.int64), np.zeros(nnz, np.int64), np.zeros(nnz)
        lib().orc_sim_export(self._h, w, r.ctypes.data_as(C.POINTER(C.c_int64)),
                             c.ctypes.data_as(C.POINTER(C.c_int64)), _d(v))
        shape = (int(r.max()) + 1 if nnz else 0, int(c.max()) + 1 if nnz else 0)
        if which in ("K", "M", "A", "Krhs"):
            shape = (self.dimension, self.dimension)
        return sp.csr_matrix((v, (r, c)), shape=shape)

    def l2_error_cosine(self, U, c0, c1, t):
        """l2_error (dg_space.cpp:94-115) of U against c0 cos(pi x) cos(pi y) e^{-c1 t}."""
        e = C.c_double()
        _check(lib().orc_l2_error_cosine(self._h, _d(np.ascontiguousarray(U, dtype=np.float64)), c0, c1, t,
                                         C.byref(e)))
        return e.value

    def mesh_size(self):
        return lib().orc_mesh_size(self._h)

    def factor_blocks(self, coarse=False):
        """Stored b x b blocks of the oracle's local (or coarse) factors."""
        return lib().orc_sim_factor_blocks(self._h, int(coarse))

    def ionic_terms(self, U, Y):
        U = np.ascontiguousarray(U, dtype=np.float64)
        Y = np.ascontiguousarray(Y, dtype=np.float64)
        I, G = np.zeros(self.dimension), np.zeros(max(self.n_comp, 1) * self.dimension)
        _check(lib().orc_sim_ionic_terms(self._h, _d(U), _d(Y), _d(I), _d(G)))
        return I, (G if self.n_comp <= 1 else G.reshape(self.n_comp, self.dimension))

    def cell_means(self, U):
        U = np.ascontiguousarray(U, dtype=np.float64)
        nc = len(self.regions)
        m = np.zeros(nc)
        _check(lib().orc_sim_cell_means(self._h, _d(U), _d(m)))
        return m


def oracle_for(config: SimulationConfig, mesh=None, reference_mesh=False):
    """Builds the oracle on the bit-exact mesh/partitions for `config`.

    reference_mesh=False: the product's mesh code (bit-exact against the
    reference, tests/test_mesh_golden.py); True: the reference's own mesh and
    agglomeration sources compiled in oracle/_ref (no product library loaded).
    Partitions follow the reference recipe: identity subdomains unless
    config.subdomains > 0 (agglomerate), coarse = hierarchy / explicit count.
    """
    split = config.split_y if config.domain[1] < config.split_y < config.domain[3] else None
    if reference_mesh:
        from tests.refmesh import RefMesh
        m = RefMesh(config.cells, config.domain, config.seed, config.lloyd, split)
    else:
        from paper_2512_19536_b200.mesh import Mesh
        m = Mesh(config.cells, config.domain, config.seed, config.lloyd, split)
    data = m.data()
    nc = data.n_cells
    if config.subdomains > 0:
        sub, ns, _ = m.agglomerate(config.subdomains)
    else:
        sub, ns = np.arange(nc, dtype=np.int32), nc
    co, nco = None, 0
    if config.precond == "two-level":
        if config.coarse == -1 or (config.coarse > 0 and config.coarse == config.subdomains):
            co, nco = sub, ns
        elif config.coarse > 0:
            co, nco, _ = m.agglomerate(config.coarse)
        else:
            levels = int(round(np.log2(config.h_ratio)))
            co, nco = m.agglomerate_hierarchy(levels)
    return OracleSim(config, data, sub, ns, co, nco), data
