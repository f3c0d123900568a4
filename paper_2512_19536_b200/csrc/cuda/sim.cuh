// DeviceSim: one rank's device-resident state and solver (see sim.cu).
#pragma once

#include <memory>
#include <vector>

#include "../host/problem.hpp"
#include "kernels.cuh"

namespace pdg {

struct PcgResult {
  int iterations = 0;
  int converged = 0;
  int error = 0;
  double denom = 0.0;
  std::vector<double> resid, alpha, beta;
};

struct StepResult {
  int iterations = 0;
  int converged = 0;
  double final_residual = 0.0;
  std::vector<double> alpha, beta;
  double step_ms = 0.0, solve_ms = 0.0;
};

void set_sweep_smem(int bytes);
int sweep_ctas_per_sm(int smem, int threads);  // occupancy of the sweep kernel
int sweep_smem_bytes(int xcap, int threads);   // dynamic shared memory of the sweep
// Extreme-eigenvalue ratio of the Lanczos tridiagonal (krylov.cpp:85-103).
bool lanczos_condition(const double* alpha, const double* beta, int m, double* kappa);

class DeviceSim;
struct LoopbackGroup;

// Exchanges of the multi-rank data path (comm.cu): NCCL between processes, or
// an in-process loopback group (test transport for several ranks on one GPU).
class Transport {
 public:
  virtual ~Transport() = default;
  virtual void allreduce(const double* src, double* dst, long long count, cudaStream_t st) = 0;
  // halo tail of v from the peers' packed d_sendbuf
  virtual void exchange(DeviceSim& s, double* v, cudaStream_t st) = 0;
  virtual const char* name() const = 0;
};

class DeviceSim {
 public:
  explicit DeviceSim(std::unique_ptr<Problem> prob);
  virtual ~DeviceSim();

  std::unique_ptr<Problem> P;
  cudaStream_t st = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
  int b = 0, bq = 0, ncells = 0, n_comp = 0, n_tasks = 0;
  long long n = 0, n_ext = 0;
  int maxit_default = 0;
  int k = 0;
  double t = 0.0;
  std::vector<int> halo_cells;  // global internal cells appended after the local ones

  // operator
  int *d_ptr = nullptr, *d_col = nullptr;
  double *d_kval = nullptr, *d_M = nullptr, *d_Minv = nullptr;
  // state and work vectors (internal order)
  double* d_U[2] = {nullptr, nullptr};  // curr, prev
  double* d_Y[3] = {nullptr, nullptr, nullptr};  // curr, prev, next
  double *d_x = nullptr, *d_p = nullptr, *d_r = nullptr, *d_z = nullptr, *d_q = nullptr;
  double *d_rhs = nullptr, *d_ion = nullptr, *d_tmp = nullptr, *d_tmp2 = nullptr, *d_scratch = nullptr;
  // coarse
  double *d_E = nullptr, *d_r0 = nullptr, *d_y0 = nullptr;
  int *d_cell_agg = nullptr, *d_agg_ptr = nullptr, *d_agg_cells = nullptr;
  int n_chunks = 0, max_chunk_cells = 0;
  bool chunks_contiguous = false;
  int *d_chunk_ptr = nullptr, *d_node_chunk_ptr = nullptr;
  double* d_r0part = nullptr;
  // sweep
  DevTask* d_tasks = nullptr;
  int *d_nunit = nullptr, *d_task_child = nullptr, *d_in_ptr = nullptr;
  int* d_bmeta = nullptr;                       // level chunk records (host/problem.hpp LevelChunk)
  int2 *d_broots = nullptr, *d_bdeps = nullptr;  // their forward publish / backward wait lists
  DevUnit *d_fwd_units = nullptr, *d_bwd_units = nullptr;
  int n_units_f = 0, n_units_b = 0, n_tile_ctrs = 0;
  double* d_part = nullptr;
  double *d_fmat = nullptr, *d_hmat = nullptr, *d_ubuf = nullptr, *d_yfwd = nullptr;
  DevTile *d_ftiles = nullptr, *d_htiles = nullptr;
  long long *d_row_dof = nullptr, *d_in_idx = nullptr;
  int* d_flags = nullptr;
  unsigned int* d_ticket = nullptr;
  int smem_fwd = 0, smem_bwd = 0, sweep_xcap = 0;
  int sweep_threads = 128;  // sweep CTA size (64 or 128, chosen in upload_tasks)
  unsigned long long* d_live = nullptr;  // live sweep timing (sweep.cu)
  long long panel_values = 0;            // F + H doubles on the device
  // ionic
  double *d_bbox = nullptr, *d_tri = nullptr;
  int *d_tri_ptr = nullptr, *d_ionflags = nullptr;
  double *d_area = nullptr, *d_means = nullptr;  // cell means (snapshot.cpp:13-28), lazy
  // pcg bookkeeping
  Reducer red{};
  PcgScalars* d_S = nullptr;
  PcgScalars* h_S = nullptr;
  double* d_hist = nullptr;
  int hist_cap = 0;
  PcgHist H{};
  int* d_perm = nullptr;

  struct Graph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    ~Graph();
    void reset();
  };
  Graph graphs[2];
  bool plain_cg = false;  // run pcg_solve with precond = nullptr
  bool use_pc() const { return P->has_precond && !plain_cg; }

  PcgResult pcg(const double* d_b, const double* d_x0, double* d_xout, double tol, int maxit);
  void apply_K(const double* x, double* y);
  void apply_precond(const double* r, double* z);
  StepResult step();
  // per-cell means of the current potential, this rank's cells, internal order
  void cell_means(std::vector<double>& out);

  // multi-rank hooks (no-ops on one GPU)
  virtual void halo_exchange(double* v);
  virtual void coarse_reduce_hook();
  virtual void dot_reduce_hook(int finish);

  // ---- multi-rank state (comm.cu) ----
  int rank = 0, world = 1;
  std::unique_ptr<Transport> transport;
  struct HaloPeer {
    int peer;
    int send_off, send_count;  // cells in d_send_cells / d_sendbuf
    int recv_off, recv_count;  // halo slots (after the local cells)
  };
  std::vector<HaloPeer> halo_peers;
  int* d_send_cells = nullptr;
  double* d_sendbuf = nullptr;
  double *d_dot_local = nullptr, *d_dot_global = nullptr;
  void attach_comm(const void* id128, int rank, int world);
  void attach_loopback(const std::shared_ptr<LoopbackGroup>& g, int rank, int world);
  void connect(std::unique_ptr<Transport> t);
  void comm_allreduce(const double* src, double* dst, long long count);
  void comm_exchange(double* v, cudaStream_t on);
  // multi-rank SpMV with the halo in flight: interior rows, then the rows
  // that read the halo (row lists built at connect)
  void spmv_overlapped(double* v, double* y);
  cudaStream_t st_comm = nullptr;
  cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
  int *d_rows_int = nullptr, *d_rows_bnd = nullptr;
  int n_rows_int = 0, n_rows_bnd = 0;
  void release_tasks();
  void comm_destroy();

  // ---- measurement ----
  long long launches = 0;  // kernels issued by step()
  cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;
  double* d_stage = nullptr;  // host<->device staging (reference order)
  long long stage_len = 0;
  int precond_launches() const;
  int body_launches() const;
  void timer(int stop, double* ms);
  void profile(int reps, double* ms, long long* bytes);
  // one traced preconditioner sweep: 8 int64 per unit (4 globaltimer stamps,
  // task, direction, staged bytes, chunks); returns the unit count
  long long* d_trace = nullptr;
  std::vector<DevUnit> h_units;
  int trace_sweep(long long* out, int cap);
  double* stage(long long len);

 protected:
  ReduceCtx red_for(int finish);
  void after_reduce(int finish, bool honor);
  void upload_tasks();
  void build_panels();  // panels.cu
  void device_factor(double* d_lval);  // factor.cu: numeric subdomain factors into d_lval
  void alloc_history(int cap);
  void assemble_on_device();
  ReduceCtx rctx(int finish, double* out = nullptr);
  SweepArgs sweep_args(bool fwd, const double* r, double* z, const PcgScalars* S);
  void precond_apply(const double* r, double* z, int finish, bool honor, bool restricted = false);
  IonicArgs ionic_args(bool has_prev) const;
  double* z_of(double* r);
  void record_iteration();
  void record_solve_tail();
  void build_solve_graph(Graph& g);
  void reset_scalars(double tol, int maxit);
  void run_solve(int maxit, PcgResult& res);
};

}  // namespace pdg
