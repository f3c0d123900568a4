"""Host-facing API mirroring the reference's solver interfaces.

    SimulationConfig  ~ polydg::SimulationConfig   (timestepper.hpp:53-80)
    Simulation        ~ polydg::Simulation          (timestepper.hpp:109-152)
    PCGReport         ~ polydg::PCGReport           (krylov.hpp:32-39)
    StepStats         ~ polydg::StepStats           (timestepper.hpp:94-99)
    SimulationResult  ~ polydg::SimulationResult    (timestepper.hpp:101-110)
    Problem           ~ the setup half of Simulation (mesh, partitions, K, M, E, K0)

Everything computes in the native library (CUDA for the Simulation); errors
surface as PdgError whose ``kind`` is the reference exception name
(ConfigError / SolverError / MeshError / IoError).
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import PcgReport as _PcgReport, StepStats as _StepStats, check, dptr, lib

PRECOND = {"none": _lib.PRECOND_NONE, "block-jacobi": _lib.PRECOND_BLOCK_JACOBI,
           "two-level": _lib.PRECOND_TWO_LEVEL}
IONIC = {"none": _lib.IONIC_NONE, "fhn": _lib.IONIC_FHN, "barreto-cressman": _lib.IONIC_BC}
FHN_KEYS = ["a", "b", "c1", "c2", "d", "u_min", "u_max", "amp"]
# Barreto-Cressman (ext; PDG_BC_* in include/polydg_b200.h)
BC_KEYS = ["g_na", "g_k", "g_nal", "g_kl", "g_cll", "phi", "rho", "g_glia", "eps", "k_bath",
           "gamma", "beta", "tau", "rtf", "cl_i", "cl_o", "na_i0", "k_i0", "na_o0", "amp"]


@dataclass
class SimulationConfig:
    """Field names follow SimulationConfig; closed forms replace std::function hooks."""
    cells: int = 512
    seed: int = 42
    lloyd: int = 20
    domain: tuple = (0.0, 0.0, 1.0, 1.0)
    split_y: float = 0.5
    degree: int = 1
    eta0: float = 10.0
    chi_m: float = 1000.0
    C_m: float = 1.0
    dt: float = 2.5e-3
    T: float = 10.0
    sigma_grey_l: float = 6.3
    sigma_grey_n: float = 6.3
    sigma_white_l: float = 6.9
    sigma_white_n: float = 25.71
    fiber_grey: tuple = (0.0, 1.0)
    fiber_white: tuple = (0.0, 1.0)
    fiber_random: bool = False
    fiber_seed: int = 42
    ionic_model: str = "fhn"
    ionic_params: dict = field(default_factory=dict)
    # initial potential: ("disc",) default InitialSpec, ("constant", v),
    # ("cosine", amp, offset), ("bilinear", c0, cx, cy, cxy)
    initial: tuple = ("disc",)
    u_rest: float = -67.0
    u_patch: float = -50.0
    omega0_center: tuple = (0.5, 1.0)
    omega0_r2: float = 0.016
    # external current: None, ("strip", amp, x_max, t_end), ("cosine", amp, decay)
    stimulus: Optional[tuple] = None
    tol: float = 1e-9
    maxit: int = 0
    warm_start: bool = True
    precond: str = "two-level"
    h_ratio: int = 2
    q: int = 0
    subdomains: int = 0
    coarse: int = 0
    rank: int = 0
    world: int = 1
    device: int = 0

    def n_steps(self) -> int:
        # std::llround (timestepper.cpp:37): halves round away from zero
        return max(1, int(math.floor(self.T / self.dt + 0.5)))

    def to_c(self, base: Optional[_lib.PdgConfig] = None) -> _lib.PdgConfig:
        """The C struct; `base` supplies the defaults of fields this dataclass
        does not carry (default: pdg_config_default of the library)."""
        c = base if base is not None else _lib.default_config()
        c.mesh_cells, c.mesh_seed, c.mesh_lloyd = self.cells, self.seed, self.lloyd
        for i, v in enumerate(self.domain):
            c.domain[i] = v
        c.split_y = self.split_y
        c.degree, c.eta0, c.chi_m, c.C_m, c.dt, c.T = (self.degree, self.eta0, self.chi_m,
                                                       self.C_m, self.dt, self.T)
        c.sigma_grey_l, c.sigma_grey_n = self.sigma_grey_l, self.sigma_grey_n
        c.sigma_white_l, c.sigma_white_n = self.sigma_white_l, self.sigma_white_n
        c.fiber_grey[0], c.fiber_grey[1] = self.fiber_grey
        c.fiber_white[0], c.fiber_white[1] = self.fiber_white
        c.fiber_random, c.fiber_seed = int(self.fiber_random), self.fiber_seed
        if self.ionic_model not in IONIC:
            raise _lib.PdgError(2, f"unknown ionic model '{self.ionic_model}'")
        c.ionic_model = IONIC[self.ionic_model]
        bc = self.ionic_model == "barreto-cressman"
        keys, arr = (BC_KEYS, c.bc) if bc else (FHN_KEYS, c.fhn)
        for k, v in self.ionic_params.items():
            if k not in keys:
                name = "barreto-cressman" if bc else "fhn"
                raise _lib.PdgError(2, f"unknown {name} parameter 'ionic.params.{k}'")
            arr[keys.index(k)] = v
        kind = self.initial[0]
        kinds = {"disc": _lib.INIT_DISC, "constant": _lib.INIT_CONSTANT,
                 "cosine": _lib.INIT_COSINE, "bilinear": _lib.INIT_BILINEAR}
        c.init_kind = kinds[kind]
        for i, v in enumerate(self.initial[1:]):
            c.init_params[i] = v
        c.u_rest, c.u_patch = self.u_rest, self.u_patch
        c.omega0[0], c.omega0[1] = self.omega0_center
        c.omega0_r2 = self.omega0_r2
        if self.stimulus is None:
            c.stim_kind = _lib.STIM_NONE
        else:
            c.stim_kind = {"strip": _lib.STIM_STRIP, "cosine": _lib.STIM_COSINE}[self.stimulus[0]]
            for i, v in enumerate(self.stimulus[1:]):
                c.stim_params[i] = v
        c.tol, c.maxit, c.warm_start = self.tol, self.maxit, int(self.warm_start)
        c.precond_kind = PRECOND[self.precond]
        c.h_ratio, c.q, c.subdomains, c.coarse_count = self.h_ratio, self.q, self.subdomains, self.coarse
        c.rank, c.world, c.device = self.rank, self.world, self.device
        return c


def ionic_rest(config: "SimulationConfig"):
    """IonicModel::state_dim / resting_potential / resting_state (ionics.hpp:25-31)
    of config.ionic_model: (n_comp, u_rest, [y_rest...])."""
    c = config.to_c()
    nc, u, y = C.c_int(), C.c_double(), (C.c_double * 4)()
    check(lib().pdg_ionic_rest(C.byref(c), C.byref(nc), C.byref(u), y))
    return nc.value, u.value, list(y[:nc.value])


@dataclass
class PCGReport:
    iterations: int = 0
    converged: bool = False
    residual_history: list = field(default_factory=list)
    alphas: list = field(default_factory=list)
    betas: list = field(default_factory=list)
    condition_estimate: Optional[float] = None


@dataclass
class StepStats:
    iterations: int
    final_residual: float
    converged: bool
    condition_estimate: Optional[float]
    solve_ms: float = 0.0
    step_ms: float = 0.0


@dataclass
class SimulationResult:
    steps: list = field(default_factory=list)
    wall_seconds: float = 0.0
    avg_iterations: float = 0.0
    cond_at_max_iter_step: Optional[float] = None
    cond_mean: Optional[float] = None
    converged_all: bool = True

    def finalize_stats(self):  # timestepper.cpp:46-65
        total, max_it, csum, cn = 0.0, -1, 0.0, 0
        for s in self.steps:
            total += s.iterations
            self.converged_all = self.converged_all and s.converged
            if s.condition_estimate is not None:
                csum += s.condition_estimate
                cn += 1
            if s.iterations > max_it:
                max_it = s.iterations
                self.cond_at_max_iter_step = s.condition_estimate
        if self.steps:
            self.avg_iterations = total / len(self.steps)
        if cn:
            self.cond_mean = csum / cn


def default_max_iterations(n: int) -> int:
    return lib().pdg_default_max_iterations(int(n))


def condition_estimate(alphas, betas) -> Optional[float]:
    a = np.ascontiguousarray(alphas, dtype=np.float64)
    b = np.ascontiguousarray(betas if len(betas) else [0.0], dtype=np.float64)
    k = C.c_double()
    ok = lib().pdg_condition_estimate(dptr(a), dptr(b), len(a), C.byref(k))
    return k.value if ok else None


class Problem:
    """Host setup only (no device): mesh, partitions, ordering, K/M/A/E/K0."""

    def __init__(self, config: SimulationConfig):
        self.config = config
        self._h = C.c_void_p()
        self._cfg = config.to_c()
        check(lib().pdg_problem_create(C.byref(self._cfg), C.byref(self._h)))
        self._owned = True
        self._read_info()

    @classmethod
    def _view(cls, handle, config, owner):
        # non-owning view of the Problem held by `owner` (a Simulation): keep
        # the owner alive as long as the view is reachable
        obj = cls.__new__(cls)
        obj.config, obj._h, obj._owned, obj._owner = config, C.c_void_p(handle), False, owner
        obj._read_info()
        return obj

    def _handle(self):
        if getattr(self, "_owner", None) is not None:
            self._owner._handle()
        if not self._h:
            raise _lib.PdgError(2, "problem: handle is closed")
        return self._h

    def _read_info(self):
        info = (C.c_int64 * 12)()
        lib().pdg_problem_info(self._h, info)
        (self.n_cells, self.n_local, self.dimension, self.n_subdomains, self.n_coarse,
         self.coarse_dim, self.nnz_blocks, self.factor_values, self.n_tasks, self.n_comp,
         self.cell_begin, self.cell_end) = list(info)

    def __del__(self):
        if getattr(self, "_owned", False) and self._h:
            lib().pdg_problem_free(self._h)
            self._h = None

    def export(self, which: str):
        """scipy.sparse.csr_matrix of K, M, A, E (n x coarse_dim) or K0 (reference order)."""
        import scipy.sparse as sp
        w = {"K": 0, "M": 1, "A": 2, "E": 3, "K0": 4}[which]
        nnz = lib().pdg_problem_export(self._handle(), w, None, None, None)
        if nnz < 0:
            raise ValueError(f"{which} not available")
        r = np.zeros(nnz, np.int64)
        c = np.zeros(nnz, np.int64)
        v = np.zeros(nnz)
        lib().pdg_problem_export(self._handle(), w, _lib.lptr(r), _lib.lptr(c), dptr(v))
        shape = {"E": (self.dimension, self.coarse_dim), "K0": (self.coarse_dim, self.coarse_dim)}.get(
            which, (self.dimension, self.dimension))
        return sp.csr_matrix((v, (r, c)), shape=shape)

    def factor_stats(self) -> dict:
        """Sizes for the SURVEY §8(d) byte model (pdg_problem_factor_stats)."""
        st = (C.c_int64 * 6)()
        lib().pdg_problem_factor_stats(self._handle(), st)
        keys = ["l_struct", "l0_struct", "fwd_panel_doubles", "bwd_panel_doubles", "k_blocks", "e_doubles"]
        return dict(zip(keys, list(st)))

    def sweep_stats(self) -> dict:
        """The sweep's work plan: supernodes, bottom levels and level chunks (pdg_problem_sweep_stats)."""
        st = (C.c_int64 * 8)()
        lib().pdg_problem_sweep_stats(self._handle(), st)
        keys = ["supernodes", "bottom_supernodes", "bottom_levels", "fwd_chunks", "bwd_chunks",
                "fwd_chunk_supernodes", "bwd_chunk_supernodes", "plan_ok"]
        return dict(zip(keys, list(st)))

    def flags(self) -> dict:
        """Where setup ran (pdg_problem_flags)."""
        f = lib().pdg_problem_flags(self._handle())
        return {"device_assembly": bool(f & 1), "device_factor": bool(f & 2)}

    def owner(self, which: str = "subdomain") -> np.ndarray:
        o = np.zeros(self.n_cells, np.int32)
        lib().pdg_problem_owner(self._handle(), 0 if which == "subdomain" else 1, _lib.iptr(o))
        return o

    def mesh(self):
        """The problem's mesh (reference cell order) as an owning mesh.Mesh."""
        from .mesh import Mesh
        h = C.c_void_p()
        check(lib().pdg_problem_mesh(self._handle(), C.byref(h)))
        return Mesh._adopt(h)

    def perm(self) -> np.ndarray:
        p = np.zeros(self.n_cells, np.int32)
        lib().pdg_problem_perm(self._handle(), _lib.iptr(p))
        return p


class Simulation:
    """Device-resident CN PolyDG monodomain solver (one rank)."""

    def __init__(self, config: SimulationConfig):
        self.config = config
        self._cfg = config.to_c()
        self._h = C.c_void_p()
        check(lib().pdg_sim_create(C.byref(self._cfg), C.byref(self._h)))
        self.problem = Problem._view(lib().pdg_sim_problem(self._h), config, self)
        self.dimension = self.problem.dimension
        self.n_comp = self.problem.n_comp

    @classmethod
    def from_operator(cls, K, block: int, precond: str = "two-level", partition=None, coarse=None,
                      maxit: int = 0, device: int = 0) -> "Simulation":
        """SparseOperator(K) + SchwarzPreconditioner(K, space, partition_S, coarse)
        (schwarz.hpp:51-53) from caller data, for apply_K / apply_precond /
        pcg_solve (no time stepper). K: scipy sparse (n x n, symmetric, element-major
        blocks of `block` dofs). partition: (owner, count) or None (one element
        per subdomain). coarse: (E, n_coarse, coarse_block) with E scipy sparse
        n x n_coarse*coarse_block, one block per element row (CoarseEmbedding::E),
        required for "two-level"."""
        import scipy.sparse as sp
        kind = {"none": _lib.PRECOND_NONE, "block-jacobi": _lib.PRECOND_BLOCK_JACOBI,
                "two-level": _lib.PRECOND_TWO_LEVEL}[precond]
        Kc = sp.csr_matrix(K)
        n = Kc.shape[0]
        if Kc.shape != (n, n) or n % block:
            raise _lib.PdgError(2, "operator: K must be square with a multiple of block rows")
        keep = []  # arrays referenced by the descriptor until the call returns
        d = _lib.OperatorDesc()
        d.n_cells, d.block = n // block, block
        rp = np.ascontiguousarray(Kc.indptr, np.int64)
        ci = np.ascontiguousarray(Kc.indices, np.int32)
        va = np.ascontiguousarray(Kc.data, np.float64)
        keep += [rp, ci, va]
        d.row_ptr, d.col, d.val = _lib.lptr(rp), _lib.iptr(ci), dptr(va)
        d.precond_kind = kind
        if partition is not None:
            own = np.ascontiguousarray(partition[0], np.int32)
            keep.append(own)
            d.sub_owner, d.n_sub = _lib.iptr(own), int(partition[1])
        if coarse is not None:
            E, nco, bq = coarse
            Ec = sp.csr_matrix(E)
            erp = np.ascontiguousarray(Ec.indptr, np.int64)
            eci = np.ascontiguousarray(Ec.indices, np.int32)
            eva = np.ascontiguousarray(Ec.data, np.float64)
            keep += [erp, eci, eva]
            d.n_coarse, d.coarse_block = int(nco), int(bq)
            d.e_row_ptr, d.e_col, d.e_val = _lib.lptr(erp), _lib.iptr(eci), dptr(eva)
        d.maxit, d.device = maxit, device
        obj = cls.__new__(cls)
        obj.config = None
        obj._h = C.c_void_p()
        check(lib().pdg_sim_create_from_operator(C.byref(d), C.byref(obj._h)))
        obj.problem = Problem._view(lib().pdg_sim_problem(obj._h), None, obj)
        obj.dimension = obj.problem.dimension
        obj.n_comp = 0
        return obj

    def close(self):
        if getattr(self, "_h", None):
            lib().pdg_sim_free(self._h)
            self._h = None

    def _handle(self):
        if not getattr(self, "_h", None):
            raise _lib.PdgError(2, "simulation: handle is closed")
        return self._h

    def _vec(self, a, what, rows=1):
        """float64 contiguous copy of `a`, checked against the dimension the
        C-ABI reads (krylov.cpp:22-23 throws SolverError on a mismatch)."""
        a = np.ascontiguousarray(a, dtype=np.float64).ravel()
        if a.size != rows * self.dimension:
            raise _lib.PdgError(3, f"{what}: vector dimension mismatch")
        return a

    def __del__(self):
        self.close()

    # --- timestepper.hpp:122-152 ---
    def step(self) -> StepStats:
        s = _StepStats()
        check(lib().pdg_sim_step(self._handle(), C.byref(s)))
        return StepStats(s.iterations, s.final_residual, bool(s.converged),
                         s.condition_estimate if s.has_condition else None, s.solve_ms, s.step_ms)

    def run(self, n_steps: Optional[int] = None) -> SimulationResult:
        t0 = time.perf_counter()
        res = SimulationResult()
        for _ in range(self.config.n_steps() if n_steps is None else n_steps):
            res.steps.append(self.step())
        res.finalize_stats()
        res.wall_seconds = time.perf_counter() - t0
        return res

    def state(self):
        """(k, t, U_curr, U_prev, Y_curr, Y_prev) in reference order; Y as (n_comp, n)."""
        n, nc = self.dimension, self.n_comp
        U, Up = np.zeros(n), np.zeros(n)
        Y, Yp = np.zeros(max(nc, 1) * n), np.zeros(max(nc, 1) * n)
        k, t = C.c_int(), C.c_double()
        check(lib().pdg_sim_get_state(self._handle(), C.byref(k), C.byref(t), dptr(U), dptr(Up),
                                      dptr(Y), dptr(Yp)))
        return k.value, t.value, U, Up, Y[:nc * n].reshape(nc, n), Yp[:nc * n].reshape(nc, n)

    def set_state(self, k, U_curr, U_prev=None, Y_curr=None, Y_prev=None):
        nc = max(self.n_comp, 1)
        keep = [None if a is None else self._vec(a, "set_state", rows)
                for a, rows in ((U_curr, 1), (U_prev, 1), (Y_curr, nc), (Y_prev, nc))]
        if keep[0] is None:
            raise _lib.PdgError(3, "set_state: U_curr is required")
        check(lib().pdg_sim_set_state(self._handle(), int(k), *[dptr(a) if a is not None else None for a in keep]))

    # --- snapshot.hpp:13-22 (means on the device, file written by the library) ---
    def cell_means(self) -> np.ndarray:
        """Per-cell means of U^k (snapshot.cpp:13-28), reference cell order."""
        m = np.zeros(self.problem.n_cells)
        check(lib().pdg_sim_cell_means(self._handle(), dptr(m)))
        return m

    def export_snapshot(self, path: str, fmt: str = "vtk-legacy") -> None:
        """export_snapshot (snapshot.cpp:30-75) of U^k at the current time."""
        check(lib().pdg_sim_export_snapshot(self._handle(), str(path).encode(), fmt.encode()))

    # --- LinearOperator::apply (krylov.hpp:15-30, schwarz.hpp:47-72) ---
    def apply_K(self, x: np.ndarray) -> np.ndarray:
        x = self._vec(x, "apply_K")
        y = np.zeros(self.dimension)
        check(lib().pdg_sim_apply_K(self._handle(), dptr(x), dptr(y)))
        return y

    def apply_precond(self, r: np.ndarray) -> np.ndarray:
        r = self._vec(r, "schwarz apply")
        z = np.zeros(self.dimension)
        check(lib().pdg_sim_apply_precond(self._handle(), dptr(r), dptr(z)))
        return z

    # --- pcg_solve (krylov.hpp:49-57) ---
    def pcg_solve(self, b, tol, maxit: int = 0, x0=None, use_precond: bool = True):
        b = self._vec(b, "pcg")
        x = np.zeros(self.dimension)
        x0a = None if x0 is None else self._vec(x0, "pcg")
        cap = (maxit if maxit > 0 else default_max_iterations(self.dimension)) + 2
        hist = [np.zeros(cap) for _ in range(3)]
        rep = _PcgReport()
        rep.capacity = cap
        rep.residual_history, rep.alphas, rep.betas = (dptr(h) for h in hist)
        check(lib().pdg_sim_pcg(self._handle(), dptr(b), dptr(x0a) if x0a is not None else None,
                                float(tol), int(maxit), int(use_precond), dptr(x), C.byref(rep)))
        it = rep.iterations
        nres = it if it > 0 else (1 if rep.converged else 0)
        nbeta = it - 1 if rep.converged else it
        out = PCGReport(it, bool(rep.converged), hist[0][:nres].tolist(), hist[1][:it].tolist(),
                        hist[2][:max(nbeta, 0)].tolist(),
                        rep.condition_estimate if rep.has_condition else None)
        return x, out


class LoopbackGroup:
    """In-process transport for `world` ranks (pdg_loopback_create): every
    rank's Simulation lives in this process, typically on one GPU, and is
    driven from its own thread. Exercises the whole multi-rank data path where
    NCCL cannot run (two ranks on one device). Not a fast path."""

    def __init__(self, world: int):
        self._h = C.c_void_p()
        check(lib().pdg_loopback_create(int(world), C.byref(self._h)))
        self.world = world

    def attach(self, sim: "Simulation") -> None:
        check(lib().pdg_sim_attach_loopback(sim._handle(), self._h, sim.config.rank, self.world))
        sim._group = self  # the group outlives its members

    def __del__(self):
        if getattr(self, "_h", None):
            lib().pdg_loopback_free(self._h)
            self._h = None


def run_simulation(config: SimulationConfig) -> SimulationResult:
    return Simulation(config).run()
