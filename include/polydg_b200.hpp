// polydg-b200 C++ shim: the reference's solver interfaces over the C-ABI.
//
// Header-only. Mirrors /root/reference/proj/include/polydg/{krylov,schwarz,
// timestepper,errors}.hpp so a caller of the reference's per-step path can
// switch by changing includes and namespace:
//   polydg::LinearOperator          -> polydg_b200::LinearOperator    (krylov.hpp:15-20)
//   polydg::SparseOperator          -> polydg_b200::SparseOperator(K) / SystemOperator (krylov.hpp:22-30)
//   polydg::SchwarzPreconditioner   -> polydg_b200::SchwarzPreconditioner (schwarz.hpp:47-72):
//                                      (K, partition_S, coarse) from caller data, or a Simulation's
//   polydg::build_coarse_embedding  -> polydg_b200::build_coarse_embedding (schwarz.hpp:38-39)
//   polydg::pcg_solve / PCGReport   -> polydg_b200::pcg_solve / PCGReport (krylov.hpp:32-57)
//   polydg::condition_estimate      -> polydg_b200::condition_estimate (krylov.hpp:59-63)
//   polydg::Simulation / StepStats  -> polydg_b200::Simulation / StepStats (timestepper.hpp:94-155)
//   ConfigError / MeshError / SolverError / IoError               (errors.hpp:13-35)
// Differences: Eigen::VectorXd becomes std::vector<double> (Eigen is not a
// dependency), SimulationConfig is the C struct pdg_config (closed forms
// instead of std::function hooks), and pcg_solve runs on the device, so its
// operators must be device operators: a Simulation's, or SparseOperator(K) with
// SchwarzPreconditioner(K, partition_S, coarse) built from the same caller
// matrix (dimension mismatch, tol outside (0, 1) and breakdown throw
// SolverError exactly as krylov.cpp:22-24,46-68).
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "polydg_b200.h"

namespace polydg_b200 {

struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct MeshError : std::runtime_error { using std::runtime_error::runtime_error; };
struct SolverError : std::runtime_error { using std::runtime_error::runtime_error; };
struct IoError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DeviceError : std::runtime_error { using std::runtime_error::runtime_error; };

inline void check(pdg_status s) {
  if (s == PDG_OK) return;
  const std::string msg = pdg_last_error();
  switch (s) {
    case PDG_ERR_CONFIG: throw ConfigError(msg);
    case PDG_ERR_SOLVER: throw SolverError(msg);
    case PDG_ERR_MESH: throw MeshError(msg);
    case PDG_ERR_IO: throw IoError(msg);
    default: throw DeviceError(msg);
  }
}

using Vector = std::vector<double>;
using SimulationConfig = pdg_config;

inline SimulationConfig default_config() {
  SimulationConfig c;
  pdg_config_default(&c);
  return c;
}

struct PCGReport {
  int iterations = 0;
  bool converged = false;
  std::vector<double> residual_history;
  std::vector<double> alphas;
  std::vector<double> betas;
  std::optional<double> condition_estimate;
};

struct StepStats {
  int iterations = 0;
  double final_residual = 0.0;
  bool converged = false;
  std::optional<double> condition_estimate;
};

struct SimulationResult {
  std::vector<StepStats> steps;
  double avg_iterations = 0.0;
  std::optional<double> cond_at_max_iter_step;
  std::optional<double> cond_mean;
  bool converged_all = true;
  void finalize_stats() {  // timestepper.cpp:46-65
    double sum = 0.0, cs = 0.0;
    int max_it = -1, cn = 0;
    for (const StepStats& s : steps) {
      sum += s.iterations;
      converged_all = converged_all && s.converged;
      if (s.condition_estimate) {
        cs += *s.condition_estimate;
        ++cn;
      }
      if (s.iterations > max_it) {
        max_it = s.iterations;
        cond_at_max_iter_step = s.condition_estimate;
      }
    }
    if (!steps.empty()) avg_iterations = sum / static_cast<double>(steps.size());
    if (cn > 0) cond_mean = cs / cn;
  }
};

inline int default_max_iterations(std::int64_t n) { return pdg_default_max_iterations(n); }

inline std::optional<double> condition_estimate(const PCGReport& r) {
  double k = 0.0;
  if (r.alphas.size() < 2) return std::nullopt;
  if (!pdg_condition_estimate(r.alphas.data(), r.betas.data(), static_cast<int>(r.alphas.size()), &k))
    return std::nullopt;
  return k;
}

class Simulation;

// Eigen::SparseMatrix<double> stand-in: scalar CSR arrays (for the symmetric
// matrices of this path CSR == CSC). SparseSymMatrix adds the element block
// size (assembly.hpp:44-50 block_dim).
struct SparseMatrix {
  std::int64_t rows = 0, cols = 0;
  std::vector<std::int64_t> row_ptr{0};
  std::vector<int> col;
  std::vector<double> val;
};
struct SparseSymMatrix : SparseMatrix {
  int block_dim = 0;
};
// AgglomeratedPartition (mesh.hpp): element -> agglomerate
struct AgglomeratedPartition {
  std::vector<int> owner;
  int count = 0;
};
// CoarseEmbedding (schwarz.hpp:29-36): E (n x count*n_local), degree q, n_local = b_q
struct CoarseEmbedding {
  SparseMatrix E;
  int q = 0;
  int n_local = 0;
  int count = 0;
};

namespace detail {
struct SimFree {
  void operator()(pdg_sim* s) const { pdg_sim_free(s); }
};
using Context = std::shared_ptr<pdg_sim>;
inline Context make_operator_context(const SparseSymMatrix& K, int kind, const AgglomeratedPartition* S,
                                     const CoarseEmbedding* coarse) {
  if (K.block_dim <= 0 || K.rows != K.cols || K.rows % K.block_dim != 0)
    throw ConfigError("operator: K must be square with block_dim > 0 dividing its size");
  pdg_operator_desc d{};
  d.n_cells = static_cast<int>(K.rows / K.block_dim);
  d.block = K.block_dim;
  d.row_ptr = K.row_ptr.data();
  d.col = K.col.data();
  d.val = K.val.data();
  d.precond_kind = kind;
  if (S) {
    d.sub_owner = S->owner.data();
    d.n_sub = S->count;
  }
  if (coarse) {
    d.n_coarse = coarse->count;
    d.coarse_block = coarse->n_local;
    d.e_row_ptr = coarse->E.row_ptr.data();
    d.e_col = coarse->E.col.data();
    d.e_val = coarse->E.val.data();
  }
  pdg_sim* h = nullptr;
  check(pdg_sim_create_from_operator(&d, &h));
  return Context(h, SimFree{});
}
}  // namespace detail

class LinearOperator {
 public:
  virtual ~LinearOperator() = default;
  virtual std::int64_t dimension() const = 0;
  virtual void apply(const Vector& x, Vector& y) const = 0;
  // the device context that holds this operator, and the caller matrix it was
  // built from (pcg_solve pairs a SparseOperator with a SchwarzPreconditioner
  // built from the same matrix)
  virtual pdg_sim* device_context() const { return nullptr; }
  virtual const void* source_matrix() const { return nullptr; }
};

// y = K x with the device system matrix of a Simulation (SparseOperator role)
class SystemOperator final : public LinearOperator {
 public:
  explicit SystemOperator(const Simulation* s) : sim_(s) {}
  std::int64_t dimension() const override;
  void apply(const Vector& x, Vector& y) const override;
  pdg_sim* device_context() const override;

 private:
  const Simulation* sim_;
};

// SparseOperator(K) (krylov.hpp:22-30) over a caller matrix: K lives on the device
class SparseOperator final : public LinearOperator {
 public:
  explicit SparseOperator(const SparseSymMatrix& K)
      : K_(&K), ctx_(detail::make_operator_context(K, PDG_PRECOND_NONE, nullptr, nullptr)) {}
  std::int64_t dimension() const override { return pdg_sim_dimension(ctx_.get()); }
  void apply(const Vector& x, Vector& y) const override {
    if (static_cast<std::int64_t>(x.size()) != dimension()) throw SolverError("apply: vector dimension mismatch");
    y.resize(x.size());
    check(pdg_sim_apply_K(ctx_.get(), x.data(), y.data()));
  }
  pdg_sim* device_context() const override { return ctx_.get(); }
  const void* source_matrix() const override { return K_; }

 private:
  const SparseSymMatrix* K_;
  detail::Context ctx_;
};

// z = B r with the device Schwarz preconditioner: a Simulation's, or built like
// the reference's SchwarzPreconditioner(K, space, partition_S, coarse)
// (schwarz.hpp:51-53; the block size comes from K.block_dim, coarse may be
// null for the one-level method). Immutable after construction.
class SchwarzPreconditioner final : public LinearOperator {
 public:
  explicit SchwarzPreconditioner(const Simulation* s) : sim_(s) {}
  SchwarzPreconditioner(const SparseSymMatrix& K, const AgglomeratedPartition& partition_S,
                        const CoarseEmbedding* coarse)
      : sim_(nullptr),
        K_(&K),
        ctx_(detail::make_operator_context(K, coarse ? PDG_PRECOND_TWO_LEVEL : PDG_PRECOND_BLOCK_JACOBI,
                                           &partition_S, coarse)) {}
  std::int64_t dimension() const override;
  void apply(const Vector& r, Vector& z) const override;
  pdg_sim* device_context() const override;
  const void* source_matrix() const override { return K_; }

 private:
  const Simulation* sim_;
  const SparseSymMatrix* K_ = nullptr;
  detail::Context ctx_;
};

class Simulation {
 public:
  explicit Simulation(const SimulationConfig& cfg) : cfg_(cfg), K_(this), B_(this) {
    pdg_sim* s = nullptr;
    check(pdg_sim_create(&cfg_, &s));
    h_.reset(s);
  }
  StepStats step() {
    pdg_step_stats st{};
    check(pdg_sim_step(h_.get(), &st));
    StepStats out;
    out.iterations = st.iterations;
    out.final_residual = st.final_residual;
    out.converged = st.converged != 0;
    if (st.has_condition) out.condition_estimate = st.condition_estimate;
    return out;
  }
  SimulationResult run() {
    SimulationResult r;
    const int n = std::max(1, static_cast<int>(cfg_.T / cfg_.dt + 0.5));
    for (int k = 0; k < n; ++k) r.steps.push_back(step());
    r.finalize_stats();
    return r;
  }
  std::int64_t dimension() const { return pdg_sim_dimension(h_.get()); }
  const LinearOperator& system_operator() const { return K_; }
  const SchwarzPreconditioner* preconditioner() const {
    return cfg_.precond_kind == PDG_PRECOND_NONE ? nullptr : &B_;
  }
  const SimulationConfig& config() const { return cfg_; }
  // TimeStepState (timestepper.hpp:82-87): U_curr, U_prev and n_comp Y fields
  void state(int* k, double* t, Vector* U_curr, Vector* U_prev, Vector* Y_curr, Vector* Y_prev) const {
    const std::size_t n = static_cast<std::size_t>(dimension());
    int nc = 0;  // IonicModel::state_dim (ionics.hpp:25): 1 FHN, 4 Barreto-Cressman
    check(pdg_ionic_rest(&cfg_, &nc, nullptr, nullptr));
    if (U_curr) U_curr->resize(n);
    if (U_prev) U_prev->resize(n);
    if (Y_curr) Y_curr->resize(n * nc);
    if (Y_prev) Y_prev->resize(n * nc);
    check(pdg_sim_get_state(h_.get(), k, t, U_curr ? U_curr->data() : nullptr, U_prev ? U_prev->data() : nullptr,
                            Y_curr && nc ? Y_curr->data() : nullptr, Y_prev && nc ? Y_prev->data() : nullptr));
  }
  // cell_means (snapshot.cpp:13-28), computed on the device: n_cells means of
  // U^k in reference cell order
  Vector cell_means() const {
    const pdg_problem* p = pdg_sim_problem(h_.get());
    std::int64_t info[12];
    pdg_problem_info(p, info);
    Vector m(static_cast<std::size_t>(info[0]));
    check(pdg_sim_cell_means(h_.get(), m.data()));
    return m;
  }
  // export_snapshot (snapshot.cpp:30-75): "vtk-legacy" or "csv-cellmeans";
  // ConfigError on an unknown format, IoError when the file cannot be written
  void export_snapshot(const std::string& path, const std::string& format) const {
    check(pdg_sim_export_snapshot(h_.get(), path.c_str(), format.c_str()));
  }
  pdg_sim* handle() const { return h_.get(); }

 private:
  struct Free {
    void operator()(pdg_sim* s) const { pdg_sim_free(s); }
  };
  SimulationConfig cfg_;
  std::unique_ptr<pdg_sim, Free> h_;
  SystemOperator K_;
  SchwarzPreconditioner B_;
};

inline std::int64_t SystemOperator::dimension() const { return sim_->dimension(); }
inline pdg_sim* SystemOperator::device_context() const { return sim_->handle(); }
inline void SystemOperator::apply(const Vector& x, Vector& y) const {
  if (static_cast<std::int64_t>(x.size()) != dimension()) throw SolverError("apply: vector dimension mismatch");
  y.resize(x.size());
  check(pdg_sim_apply_K(sim_->handle(), x.data(), y.data()));
}
inline pdg_sim* SchwarzPreconditioner::device_context() const { return sim_ ? sim_->handle() : ctx_.get(); }
inline std::int64_t SchwarzPreconditioner::dimension() const { return pdg_sim_dimension(device_context()); }
inline void SchwarzPreconditioner::apply(const Vector& r, Vector& z) const {
  if (static_cast<std::int64_t>(r.size()) != dimension()) throw SolverError("apply: vector dimension mismatch");
  z.resize(r.size());
  check(pdg_sim_apply_precond(device_context(), r.data(), z.data()));
}

// build_coarse_embedding(space, partition, q) (schwarz.hpp:38-39) on a
// generated mesh with degree-p elements; ConfigError if q is not in [1, p]
inline CoarseEmbedding build_coarse_embedding(const pdg_mesh* mesh, int p, const AgglomeratedPartition& part, int q) {
  const int b = (p + 1) * (p + 2) / 2, bq = (q + 1) * (q + 2) / 2;
  const std::int64_t nc = static_cast<std::int64_t>(part.owner.size());
  std::vector<double> blocks(static_cast<std::size_t>(nc) * b * bq);
  check(pdg_mesh_coarse_embedding(mesh, p, part.owner.data(), part.count, q, blocks.data()));
  CoarseEmbedding ce;
  ce.q = q;
  ce.n_local = bq;
  ce.count = part.count;
  ce.E.rows = nc * b;
  ce.E.cols = static_cast<std::int64_t>(part.count) * bq;
  ce.E.row_ptr.assign(1, 0);
  for (std::int64_t c = 0; c < nc; ++c)
    for (int r = 0; r < b; ++r) {
      for (int m = 0; m < bq; ++m) {
        ce.E.col.push_back(part.owner[c] * bq + m);
        ce.E.val.push_back(blocks[static_cast<std::size_t>(c) * b * bq + static_cast<std::size_t>(m) * b + r]);
      }
      ce.E.row_ptr.push_back(static_cast<std::int64_t>(ce.E.col.size()));
    }
  return ce;
}

// pcg_solve(K, b, precond, tol, maxit, x0) (krylov.hpp:49-51), device-resident loop
inline std::pair<Vector, PCGReport> pcg_solve(const LinearOperator& K, const Vector& b,
                                              const LinearOperator* precond, double tol, int maxit,
                                              const Vector& x0) {
  // the device context that holds both operators: a Simulation's K and B, or
  // a SparseOperator and a SchwarzPreconditioner built from the same matrix
  pdg_sim* ctx = K.device_context();
  if (precond && precond->device_context() != ctx) {
    if (precond->source_matrix() && precond->source_matrix() == K.source_matrix()) ctx = precond->device_context();
    else ctx = nullptr;
  }
  if (!ctx) throw ConfigError("pcg_solve: K and the preconditioner must be device operators of the same matrix");
  if (static_cast<std::int64_t>(b.size()) != K.dimension() || x0.size() != b.size())
    throw SolverError("pcg: vector dimension mismatch");
  const int cap = (maxit > 0 ? maxit : default_max_iterations(K.dimension())) + 2;
  PCGReport rep;
  rep.residual_history.resize(cap);
  rep.alphas.resize(cap);
  rep.betas.resize(cap);
  pdg_pcg_report c{};
  c.capacity = cap;
  c.residual_history = rep.residual_history.data();
  c.alphas = rep.alphas.data();
  c.betas = rep.betas.data();
  Vector x(b.size());
  check(pdg_sim_pcg(ctx, b.data(), x0.data(), tol, maxit, precond != nullptr, x.data(), &c));
  rep.iterations = c.iterations;
  rep.converged = c.converged != 0;
  rep.residual_history.resize(c.iterations > 0 ? c.iterations : (c.converged ? 1 : 0));
  rep.alphas.resize(c.iterations);
  rep.betas.resize(c.converged ? std::max(0, c.iterations - 1) : c.iterations);
  if (c.has_condition) rep.condition_estimate = c.condition_estimate;
  return {std::move(x), std::move(rep)};
}

// convenience overload: x0 = 0, default maxit (krylov.hpp:53-57)
inline std::pair<Vector, PCGReport> pcg_solve(const LinearOperator& K, const Vector& b,
                                              const LinearOperator* precond, double tol) {
  return pcg_solve(K, b, precond, tol, 0, Vector(b.size(), 0.0));
}

inline SimulationResult run_simulation(const SimulationConfig& cfg) { return Simulation(cfg).run(); }

}  // namespace polydg_b200
