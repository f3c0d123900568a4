/*
 * polydg-b200 — C-ABI of the B200-native per-time-step solve of the
 * reference's Crank–Nicolson PolyDG monodomain solver.
 *
 * This is the drop-in boundary: plain pointers and sizes,
 * no torch / CUDA types. Host vectors are always in the REFERENCE layout:
 * element-major blocks of n_local = (p+1)(p+2)/2 modes in cell-index order
 * (/root/reference/proj/include/polydg/dg_space.hpp:15-32). Internally the
 * library permutes to a subdomain-major nested-dissection order.
 *
 * Every entry point returns a pdg_status; on failure pdg_last_error() holds
 * the message. Status codes mirror the reference's exception taxonomy
 * (/root/reference/proj/include/polydg/errors.hpp:13-35) so a C++ shim can
 * rethrow ConfigError / MeshError / SolverError / IoError unchanged.
 * One host thread per handle.
 */
#ifndef POLYDG_B200_H
#define POLYDG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum pdg_status {
  PDG_OK = 0,
  PDG_ERR_CONFIG = 2, /* ConfigError  (CLI exit 2) */
  PDG_ERR_SOLVER = 3, /* SolverError  (CLI exit 3) */
  PDG_ERR_MESH = 4,   /* MeshError */
  PDG_ERR_IO = 5,     /* IoError */
  PDG_ERR_CUDA = 6,   /* device / driver failure (no reference analogue) */
  PDG_ERR_INTERNAL = 7
} pdg_status;

enum { PDG_PRECOND_NONE = 0, PDG_PRECOND_BLOCK_JACOBI = 1, PDG_PRECOND_TWO_LEVEL = 2 };
enum { PDG_IONIC_NONE = 0, PDG_IONIC_FHN = 1, PDG_IONIC_BARRETO_CRESSMAN = 2 };
enum { PDG_INIT_DISC = 0, PDG_INIT_CONSTANT = 1, PDG_INIT_COSINE = 2, PDG_INIT_BILINEAR = 3 };
enum { PDG_STIM_NONE = 0, PDG_STIM_STRIP = 1, PDG_STIM_COSINE = 2 };
/* ext: Barreto-Cressman kinetics (Cressman et al. 2009, J Comput Neurosci 26:159;
 * the reference registers the model name but ships no kinetics, ionics.cpp:52-57).
 * State y = (n, h, [K]o, [Na]i); indices into pdg_config.bc: */
enum {
  PDG_BC_G_NA = 0, PDG_BC_G_K, PDG_BC_G_NAL, PDG_BC_G_KL, PDG_BC_G_CLL, /* mS/cm^2 */
  PDG_BC_PHI,                                                         /* gating time scale, 1/ms */
  PDG_BC_RHO, PDG_BC_G_GLIA, PDG_BC_EPS, PDG_BC_K_BATH,               /* mM/s, mM/s, 1/s, mM */
  PDG_BC_GAMMA, PDG_BC_BETA, PDG_BC_TAU,                              /* mM cm^2/uC, -, ms/s */
  PDG_BC_RTF, PDG_BC_CL_I, PDG_BC_CL_O,                               /* mV, mM, mM */
  PDG_BC_NA_I0, PDG_BC_K_I0, PDG_BC_NA_O0, PDG_BC_AMP,                /* mM, mM, mM, - */
  PDG_BC_NPARAM
};

/*
 * Mirrors polydg::SimulationConfig (/root/reference/proj/include/polydg/
 * timestepper.hpp:21-80) with the std::function hooks replaced by closed
 * forms, plus the BASELINE.json extensions (marked ext).
 */
typedef struct pdg_config {
  /* MeshSpec (timestepper.hpp:21-27) */
  int mesh_cells;
  uint64_t mesh_seed;
  int mesh_lloyd;
  double domain[4]; /* xmin ymin xmax ymax */
  double split_y;
  /* discretisation (timestepper.hpp:53-66) */
  int degree;
  double eta0, chi_m, C_m, dt, T;
  double sigma_grey_l, sigma_grey_n, sigma_white_l, sigma_white_n;
  double fiber_grey[2], fiber_white[2];
  int fiber_random;    /* ext: per-element angle theta ~ U[0,pi) from fiber_seed */
  uint64_t fiber_seed; /*      theta_K = pi*(rng()>>11)*2^-53 in cell order */
  /* ionic model (ionics.hpp:38-61, ionics.cpp:35-59) */
  int ionic_model;
  double fhn[8]; /* a b c1 c2 d u_min u_max amp */
  /* initial data: InitialSpec (timestepper.hpp:28-33) or the test hook
   * initial_potential as a closed form:
   *   DISC:     u_patch inside |x-omega0|^2 < omega0_r2 else u_rest
   *   CONSTANT: init_params[0]
   *   COSINE:   init_params[0]*cos(pi x)cos(pi y) + init_params[1]
   *   BILINEAR: init_params[0] + init_params[1] x + init_params[2] y + init_params[3] x y */
  int init_kind;
  double u_rest, u_patch, omega0[2], omega0_r2;
  double init_params[4];
  /* external current I_ext(x, t), evaluated at t + dt/2 (timestepper.cpp:128-142,159):
   *   STRIP:  stim_params[0] if x < stim_params[1] and t < stim_params[2]   (ext)
   *   COSINE: stim_params[0]*cos(pi x)cos(pi y)*exp(-stim_params[1] t)     (test hook) */
  int stim_kind;
  double stim_params[4];
  /* SolverSpec (timestepper.hpp:35-39) */
  double tol;
  int maxit; /* 0 = min(20 sqrt(n), n) */
  int warm_start;
  /* PrecondSpec (timestepper.hpp:41-45) + ext */
  int precond_kind;
  int h_ratio;      /* coarse = agglomerate_hierarchy(log2 h_ratio) when coarse_count == 0 */
  int q;            /* 0 = degree */
  int subdomains;   /* ext: 0 = one cell per subdomain (reference); S>0 = agglomerate(mesh,S) */
  int coarse_count; /* ext: 0 = hierarchy; -1 = same partition as the subdomains; >0 = agglomerate(mesh,n) */
  /* placement */
  int rank, world, device;
  /* ext: Barreto-Cressman parameters (PDG_BC_* above); appended so the
   * earlier layout is unchanged */
  double bc[PDG_BC_NPARAM];
} pdg_config;

void pdg_config_default(pdg_config* cfg);
/* IonicModel::state_dim / resting_potential / resting_state (ionics.hpp:25-31) of
 * cfg->ionic_model: n_comp = 0 (none), 1 (FHN: u_min, y = 0) or 4 (Barreto-Cressman:
 * the fixed point of the membrane + concentration equations, found by Newton);
 * y_rest holds up to 4 values */
pdg_status pdg_ionic_rest(const pdg_config* cfg, int* n_comp, double* u_rest, double* y_rest);
const char* pdg_last_error(void);

/* ---- mesh level (host setup; bit-exact with the reference generator) ---- */
typedef struct pdg_mesh pdg_mesh;
/* generate_polygonal_mesh + assign_regions (mesh.hpp:104-112); split_y <= ymin skips regions */
pdg_status pdg_mesh_generate(int n_cells, const double domain[4], uint64_t seed, int lloyd,
                             double split_y, pdg_mesh** out);
void pdg_mesh_free(pdg_mesh* m);
/* counts: n_cells, n_vertices, n_corners, n_interior_faces, n_boundary_faces */
void pdg_mesh_counts(const pdg_mesh* m, int counts[5]);
void pdg_mesh_arrays(const pdg_mesh* m, double* verts, int* cell_off, int* cell_vtx,
                     uint8_t* regions);
void pdg_mesh_faces(const pdg_mesh* m, int interior, int* cells, double* geo7);
void pdg_mesh_cell_geometry(const pdg_mesh* m, double* area_cx_cy_h);
/* agglomerate(mesh, target) (mesh.hpp:114-120); returns count or -1 */
int pdg_mesh_agglomerate(const pdg_mesh* m, int target, int* owner, double* H);
int pdg_mesh_agglomerate_hierarchy(const pdg_mesh* m, int levels, int* owner);
/* polygon_quadrature (quadrature.hpp:34): returns #points or -1 */
int pdg_polygon_quadrature(const double* poly, int n, int order, double* pts, double* w, int cap);

/* ---- problem (host setup: partitions, ordering, assembly, factorisation) ---- */
typedef struct pdg_problem pdg_problem;
pdg_status pdg_problem_create(const pdg_config* cfg, pdg_problem** out);
void pdg_problem_free(pdg_problem* p);
/* info: n_cells, n_local, dimension, n_subdomains, n_coarse_aggs, coarse_dim,
 *       nnz_blocks(K), factor_values, n_tasks, n_comp, rank cells begin, end */
void pdg_problem_info(const pdg_problem* p, int64_t info[12]);
/* K (system matrix) as COO triplets in reference dof order; returns nnz when
 * rows == NULL. which: 0 = K, 1 = M, 2 = A, 3 = E (n x coarse_dim), 4 = K0 */
int64_t pdg_problem_export(const pdg_problem* p, int which, int64_t* rows, int64_t* cols,
                           double* vals);
/* factor / operator sizes of this rank for the SURVEY §8(d) byte model:
 * stats[0] structural nnz(L) of the local Schwarz factors (scalar, lower incl.
 * diagonal, this implementation's ordering), [1] the same for the coarse
 * factor, [2] / [3] stored forward / backward sweep panel doubles (explicit
 * zeros and padding included), [4] local K blocks, [5] E doubles held */
void pdg_problem_factor_stats(const pdg_problem* p, int64_t stats[6]);
/* the sweep's work plan on this rank (diagnostic; no reference counterpart):
 * stats[0] sweep supernodes, [1] of which solved in level chunks (the bottom
 * levels of the elimination trees), [2] bottom levels, [3] / [4] forward /
 * backward level chunks, [5] supernodes covered by the forward chunks, [6] by
 * the backward chunks plus the dense roots among [1] (no backward solve),
 * [7] 1 if every chunk's dependency precedes it in the ticket order and every
 * record fits the sweep CTA's shared block */
void pdg_problem_sweep_stats(const pdg_problem* p, int64_t stats[8]);
/* partition maps: which 0 = subdomain owner, 1 = coarse owner; per reference cell */
/* where setup ran: bit 0 = operator assembled on the device (cuda/assemble.cu),
 * bit 1 = local factors computed on the device (cuda/factor.cu) */
int pdg_problem_flags(const pdg_problem* p);
void pdg_problem_owner(const pdg_problem* p, int which, int* owner);
/* internal order: perm[i] = reference cell of internal position i */
void pdg_problem_perm(const pdg_problem* p, int* perm);
/* multi-rank layout: internal cell range per rank (world+1 entries) and the
 * SpMV halo against `peer`: send = this rank's local cells (relative to its
 * first cell), recv = peer's global internal cells; counts = {nsend, nrecv};
 * NULL arrays query the sizes */
void pdg_problem_rank_cells(const pdg_problem* p, int* starts);
/* copy of the problem's mesh (reference cell order) as an owning pdg_mesh */
pdg_status pdg_problem_mesh(const pdg_problem* p, pdg_mesh** out);
void pdg_problem_halo(const pdg_problem* p, int peer, int* send, int* recv, int counts[2]);

/* ---- simulation on the device (Simulation, timestepper.hpp:109-152) ---- */
typedef struct pdg_sim pdg_sim;

typedef struct pdg_step_stats { /* StepStats (timestepper.hpp:94-99) */
  int iterations;
  int converged;
  double final_residual;
  int has_condition;
  double condition_estimate;
  double solve_ms;  /* device time of the PCG solve */
  double step_ms;   /* device time of the whole step */
} pdg_step_stats;

typedef struct pdg_pcg_report { /* PCGReport (krylov.hpp:32-39) */
  int iterations;
  int converged;
  int has_condition;
  double condition_estimate;
  int capacity;             /* caller-allocated length of the arrays below */
  double* residual_history; /* >= iterations (+1 when denom == 0) */
  double* alphas;
  double* betas;
} pdg_pcg_report;

pdg_status pdg_sim_create(const pdg_config* cfg, pdg_sim** out);

/* ---- solver from caller-supplied operator data ----
 * SparseOperator(K) (krylov.hpp:22-30) + SchwarzPreconditioner(K, space,
 * partition_S, coarse) (schwarz.hpp:51-53) + pcg_solve (krylov.hpp:49-51)
 * without the mesh / time stepper: the caller hands over K and the partitions
 * the reference's constructor takes, and gets a pdg_sim whose apply_K,
 * apply_precond and pcg (host or device vectors) work; pdg_sim_step returns
 * PDG_ERR_CONFIG. The context copies everything; vectors are in the caller's
 * (reference) dof order, element-major blocks of `block` dofs. */
typedef struct pdg_operator_desc {
  int n_cells;              /* elements (DGSpace::n_elements); dimension = n_cells * block */
  int block;                /* dofs per element (DGSpace::n_local, assembly.hpp:44-50 block_dim) */
  const int64_t* row_ptr;   /* K as scalar CSR (symmetric, both triangles, Eigen's SparseMatrix */
  const int* col;           /*   arrays; for a symmetric matrix CSR == CSC): n+1 / nnz / nnz */
  const double* val;
  int precond_kind;         /* PDG_PRECOND_NONE / _BLOCK_JACOBI / _TWO_LEVEL */
  const int* sub_owner;     /* partition_S.owner: element -> subdomain (NULL: one element each) */
  int n_sub;                /* partition_S.count */
  /* CoarseEmbedding (schwarz.hpp:29-36), two-level only: E as scalar CSR of
   * n rows x n_coarse*coarse_block columns, one block per element row (the
   * element's agglomerate columns), as build_coarse_embedding forms it */
  int n_coarse;
  int coarse_block;         /* b_q */
  const int64_t* e_row_ptr;
  const int* e_col;
  const double* e_val;
  int maxit;                /* default maxit for pcg (0: min(20 sqrt(n), n)) */
  int device;
} pdg_operator_desc;
pdg_status pdg_sim_create_from_operator(const pdg_operator_desc* desc, pdg_sim** out);
/* build_coarse_embedding(space, partition, q) (schwarz.hpp:38-39) on a
 * generated mesh with degree-p elements: E as the per-element blocks
 * (n_cells x block x coarse_block doubles, column-major blocks) for
 * agglomerate owner[] (count agglomerates). ConfigError if q not in [1, p]. */
pdg_status pdg_mesh_coarse_embedding(const pdg_mesh* m, int p, const int* owner, int count, int q,
                                     double* E_blocks);
void pdg_sim_free(pdg_sim* s);
const pdg_problem* pdg_sim_problem(const pdg_sim* s);
int64_t pdg_sim_dimension(const pdg_sim* s);
/* Simulation::step (timestepper.cpp:144-200). Throws-equivalent:
 * PDG_ERR_SOLVER with "time step k: ..." on non-convergence. */
pdg_status pdg_sim_step(pdg_sim* s, pdg_step_stats* stats);
/* state in reference order; any pointer may be NULL. Y arrays hold n_comp fields. */
pdg_status pdg_sim_get_state(pdg_sim* s, int* k, double* t, double* U_curr, double* U_prev,
                             double* Y_curr, double* Y_prev);
pdg_status pdg_sim_set_state(pdg_sim* s, int k, const double* U_curr, const double* U_prev,
                             const double* Y_curr, const double* Y_prev);
/* LinearOperator::apply of the system matrix (krylov.hpp:22-30) and of the
 * Schwarz preconditioner (schwarz.hpp:47-72); host vectors, reference order. */
pdg_status pdg_sim_apply_K(pdg_sim* s, const double* x, double* y);
pdg_status pdg_sim_apply_precond(pdg_sim* s, const double* r, double* z);
/* pcg_solve(K, b, precond, tol, maxit, x0) (krylov.hpp:49-51); use_precond 0
 * gives plain CG. maxit <= 0 -> default_max_iterations. */
pdg_status pdg_sim_pcg(pdg_sim* s, const double* b, const double* x0, double tol, int maxit,
                       int use_precond, double* x, pdg_pcg_report* rep);
/* cell_means (snapshot.cpp:13-28) of the current potential U^k, computed on
 * the device at the order-2p+2 rule; `means` holds n_cells doubles in
 * reference cell order (cells of other ranks are left 0). */
pdg_status pdg_sim_cell_means(pdg_sim* s, double* means);
/* export_snapshot (snapshot.cpp:30-75) of U^k at the simulation time:
 * format "vtk-legacy" or "csv-cellmeans"; PDG_ERR_CONFIG on an unknown
 * format, PDG_ERR_IO when the file cannot be written. */
pdg_status pdg_sim_export_snapshot(pdg_sim* s, const char* path, const char* format);
/* device-resident variants for benchmarking: vectors already on the device,
 * internal order. */
pdg_status pdg_sim_pcg_device(pdg_sim* s, const double* d_b, const double* d_x0, double tol,
                              int maxit, double* d_x, pdg_pcg_report* rep);
/* ---- measurement (no reference analogue; the reference only times wall
 * clock, timestepper.cpp:203,227-228) ---- */
/* stop = 0 records a start event on the solver stream; stop = 1 records the
 * end event, waits for it and returns the device time between the two */
pdg_status pdg_sim_timer(pdg_sim* s, int stop, double* elapsed_ms);
/* kernels issued by pdg_sim_step so far (graph-replayed launches included) */
int64_t pdg_sim_kernel_launches(const pdg_sim* s);
/* per-kernel device time (ms, averaged over reps) and algorithmic bytes per
 * launch, slots: 0 spmv, 1 update, 2 restrict, 3 sweep_fwd, 4 sweep_bwd,
 * 5 prolong_dot, 6 pupdate, 7 ionic, 8 rhs */
pdg_status pdg_sim_profile(pdg_sim* s, int reps, double* ms9, int64_t* bytes9);
/* live timing of the Schwarz sweep inside the solves run so far: launches and
 * their summed device duration (first CTA start to last CTA end, globaltimer) */
pdg_status pdg_sim_sweep_live(pdg_sim* s, int64_t* launches, double* total_ms);
/* one traced Schwarz sweep: 12 int64 per work unit (globaltimer at start,
 * deps met, inputs gathered, published, staging done, mat-vec done; task,
 * direction, panel bytes, chunks, task height, coarse flag); returns the unit
 * count (scripts/sweep_trace.py) */
int pdg_sim_trace_sweep(pdg_sim* s, long long* out, int cap);

/* BASELINE config-5 input: b_i = 2 (rng()>>11) 2^-53 - 1 drawn from
 * std::mt19937_64(seed) in dof order, the reference's seeded uniform [-1, 1)
 * pattern (proj/tests/acceptance.cpp:285-286) */
void pdg_uniform_rhs(uint64_t seed, int64_t n, double* out);

/* default_max_iterations (krylov.cpp:12-15) and condition_estimate (:85-103) */
int pdg_default_max_iterations(int64_t n);
int pdg_condition_estimate(const double* alphas, const double* betas, int m, double* kappa);

/* ---- multi-GPU (one process per GPU) ---- */
int pdg_nccl_unique_id_bytes(void);
pdg_status pdg_nccl_get_unique_id(void* id128);
pdg_status pdg_sim_attach_comm(pdg_sim* s, const void* id128, int rank, int world);
/* In-process loopback transport: `world` simulations of one process (e.g. on
 * one GPU), each driven by its own host thread, exchange halos and all-reduces
 * through host staging. A test transport for the multi-rank data path where
 * NCCL cannot run (NCCL rejects two ranks on one device); not a fast path. */
typedef struct pdg_loopback pdg_loopback;
pdg_status pdg_loopback_create(int world, pdg_loopback** out);
void pdg_loopback_free(pdg_loopback* g);
pdg_status pdg_sim_attach_loopback(pdg_sim* s, pdg_loopback* g, int rank, int world);

#ifdef __cplusplus
}
#endif
#endif /* POLYDG_B200_H */
