// polydg-b200 C++ shim: the reference's solver interfaces over the C-ABI.
//
// Header-only. Mirrors /root/reference/proj/include/polydg/{krylov,schwarz,
// timestepper,errors}.hpp so a caller of the reference's per-step path can
// switch by changing includes and namespace:
//   polydg::LinearOperator          -> polydg_b200::LinearOperator    (krylov.hpp:15-20)
//   polydg::SparseOperator          -> polydg_b200::SystemOperator    (krylov.hpp:22-30)
//   polydg::SchwarzPreconditioner   -> polydg_b200::SchwarzPreconditioner (schwarz.hpp:47-72)
//   polydg::pcg_solve / PCGReport   -> polydg_b200::pcg_solve / PCGReport (krylov.hpp:32-57)
//   polydg::condition_estimate      -> polydg_b200::condition_estimate (krylov.hpp:59-63)
//   polydg::Simulation / StepStats  -> polydg_b200::Simulation / StepStats (timestepper.hpp:94-155)
//   ConfigError / MeshError / SolverError / IoError               (errors.hpp:13-35)
// Differences: Eigen::VectorXd becomes std::vector<double> (Eigen is not a
// dependency), SimulationConfig is the C struct pdg_config (closed forms
// instead of std::function hooks), and pcg_solve runs on the device, so its
// operators must be the ones of a Simulation (dimension mismatch, tol outside
// (0, 1) and breakdown throw SolverError exactly as krylov.cpp:22-24,46-68).
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

class LinearOperator {
 public:
  virtual ~LinearOperator() = default;
  virtual std::int64_t dimension() const = 0;
  virtual void apply(const Vector& x, Vector& y) const = 0;
  virtual const Simulation* device_owner() const { return nullptr; }
};

// y = K x with the device system matrix
class SystemOperator final : public LinearOperator {
 public:
  explicit SystemOperator(const Simulation* s) : sim_(s) {}
  std::int64_t dimension() const override;
  void apply(const Vector& x, Vector& y) const override;
  const Simulation* device_owner() const override { return sim_; }

 private:
  const Simulation* sim_;
};

// z = B r with the device two-level Schwarz preconditioner
class SchwarzPreconditioner final : public LinearOperator {
 public:
  explicit SchwarzPreconditioner(const Simulation* s) : sim_(s) {}
  std::int64_t dimension() const override;
  void apply(const Vector& r, Vector& z) const override;
  const Simulation* device_owner() const override { return sim_; }

 private:
  const Simulation* sim_;
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
inline void SystemOperator::apply(const Vector& x, Vector& y) const {
  y.resize(x.size());
  check(pdg_sim_apply_K(sim_->handle(), x.data(), y.data()));
}
inline std::int64_t SchwarzPreconditioner::dimension() const { return sim_->dimension(); }
inline void SchwarzPreconditioner::apply(const Vector& r, Vector& z) const {
  z.resize(r.size());
  check(pdg_sim_apply_precond(sim_->handle(), r.data(), z.data()));
}

// pcg_solve(K, b, precond, tol, maxit, x0) (krylov.hpp:49-51), device-resident loop
inline std::pair<Vector, PCGReport> pcg_solve(const LinearOperator& K, const Vector& b,
                                              const LinearOperator* precond, double tol, int maxit,
                                              const Vector& x0) {
  const Simulation* sim = K.device_owner();
  if (!sim || (precond && precond->device_owner() != sim))
    throw ConfigError("pcg_solve: operators must belong to the same device Simulation");
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
  check(pdg_sim_pcg(sim->handle(), b.data(), x0.data(), tol, maxit, precond != nullptr, x.data(), &c));
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
