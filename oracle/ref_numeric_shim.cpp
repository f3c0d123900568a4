// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI over the reference's OWN numeric path, compiled by oracle/Makefile
// (target `refnum`) straight from /root/reference/proj/src/{dg_space,assembly,
// ionics,krylov,schwarz,timestepper,snapshot,...}.cpp with the Eigen API
// stand-in of oracle/eigen_shim (Eigen3 is not installed here) into
// oracle/_ref/libpolydg_refnum.so. It is a second oracle: the reference's
// Simulation::step, pcg_solve, SchwarzPreconditioner, assembly and ionic
// terms run unmodified; tests compare it with the restated oracle (oracle/src)
// and with the device path. No reference source is copied into this repo.
//
// The reference's Simulation hard-codes identity subdomains and a hierarchy
// coarse space (timestepper.cpp:91-104). The BASELINE configs use
// agglomerated subdomains with S_H = S (SURVEY §8(d) ext), which the
// reference's SchwarzPreconditioner accepts (schwarz.hpp:51-53): after
// construction the shim swaps in SchwarzPreconditioner(K, space,
// agglomerate(mesh, S), &build_coarse_embedding(space, agglomerate(mesh, S_H), q))
// built by the reference's own functions, then steps with the reference's step().
#include <cstring>
#include <functional>
#include <memory>
#include <string>

// the preconditioner swap above needs Simulation's members
#define private public
#include "polydg/timestepper.hpp"
#undef private
#include "polydg/errors.hpp"
#include "polydg/krylov.hpp"
#include "polydg/snapshot.hpp"

using namespace polydg;

extern "C" {
// same C layout as include/polydg_b200.h pdg_config / oracle/src/capi.cpp orc_config
typedef struct refn_config {
  int mesh_cells;
  uint64_t mesh_seed;
  int mesh_lloyd;
  double domain[4];
  double split_y;
  int degree;
  double eta0, chi_m, C_m, dt, T;
  double sigma_grey_l, sigma_grey_n, sigma_white_l, sigma_white_n;
  double fiber_grey[2], fiber_white[2];
  int fiber_random;
  uint64_t fiber_seed;
  int ionic_model;
  double fhn[8];
  int init_kind;
  double u_rest, u_patch, omega0[2], omega0_r2;
  double init_params[4];
  int stim_kind;
  double stim_params[4];
  double tol;
  int maxit;
  int warm_start;
  int precond_kind;
  int h_ratio;
  int q;
  int subdomains;
  int coarse_count;
  int rank, world, device;
  double bc[20];
} refn_config;

typedef struct refn_report {
  int iterations, converged, has_condition;
  double condition_estimate;
  int capacity;
  double *residual_history, *alphas, *betas;
  int n_resid, n_alpha, n_beta;
} refn_report;
}

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const SolverError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 7;
  }
}

struct RefSim {
  std::unique_ptr<Simulation> sim;
  std::unique_ptr<AgglomeratedPartition> sub, coarse_part;
};

SimulationConfig convert(const refn_config& c) {
  SimulationConfig s;
  s.mesh.cells = c.mesh_cells;
  s.mesh.seed = c.mesh_seed;
  s.mesh.lloyd = c.mesh_lloyd;
  s.mesh.domain = Rect{c.domain[0], c.domain[1], c.domain[2], c.domain[3]};
  s.mesh.split_y = c.split_y;
  s.degree = c.degree;
  s.eta0 = c.eta0;
  s.chi_m = c.chi_m;
  s.C_m = c.C_m;
  s.dt = c.dt;
  s.T = c.T;
  s.sigma_grey_l = c.sigma_grey_l;
  s.sigma_grey_n = c.sigma_grey_n;
  s.sigma_white_l = c.sigma_white_l;
  s.sigma_white_n = c.sigma_white_n;
  s.fiber_grey = {c.fiber_grey[0], c.fiber_grey[1]};
  s.fiber_white = {c.fiber_white[0], c.fiber_white[1]};
  if (c.fiber_random) throw ConfigError("refnum: per-element fibres are an extension the reference does not have");
  static const char* fhn_keys[8] = {"a", "b", "c1", "c2", "d", "u_min", "u_max", "amp"};
  if (c.ionic_model == 0) {
    s.ionic_model = "none";
  } else if (c.ionic_model == 1) {
    s.ionic_model = "fhn";
    for (int i = 0; i < 8; ++i) s.ionic_params[fhn_keys[i]] = c.fhn[i];
  } else {
    s.ionic_model = "barreto-cressman";  // the reference throws ConfigError (ionics.cpp:52-57)
  }
  s.init.u_rest = c.u_rest;
  s.init.u_patch = c.u_patch;
  s.init.omega0_center = {c.omega0[0], c.omega0[1]};
  s.init.omega0_r2 = c.omega0_r2;
  const double* ip = c.init_params;
  const double a0 = ip[0], a1 = ip[1], a2 = ip[2], a3 = ip[3];
  switch (c.init_kind) {
    case 0: break;  // InitialSpec disc (timestepper.cpp:108-114)
    case 1: s.initial_potential = [a0](const Point2&) { return a0; }; break;
    case 2:
      s.initial_potential = [a0, a1](const Point2& p) { return a0 * std::cos(M_PI * p.x) * std::cos(M_PI * p.y) + a1; };
      break;
    case 3:
      s.initial_potential = [a0, a1, a2, a3](const Point2& p) { return a0 + a1 * p.x + a2 * p.y + a3 * p.x * p.y; };
      break;
    default: throw ConfigError("refnum: unknown initial condition");
  }
  const double s0 = c.stim_params[0], s1 = c.stim_params[1], s2 = c.stim_params[2];
  if (c.stim_kind == 1)
    s.I_ext = [s0, s1, s2](const Point2& p, double t) { return (p.x < s1 && t < s2) ? s0 : 0.0; };
  else if (c.stim_kind == 2)
    s.I_ext = [s0, s1](const Point2& p, double t) {
      return s0 * std::cos(M_PI * p.x) * std::cos(M_PI * p.y) * std::exp(-s1 * t);
    };
  s.solver.tol = c.tol;
  s.solver.maxit = c.maxit;
  s.solver.warm_start = c.warm_start != 0;
  s.precond.kind = c.precond_kind == 0 ? PrecondKind::None
                   : c.precond_kind == 1 ? PrecondKind::BlockJacobi
                                         : PrecondKind::TwoLevel;
  s.precond.h_ratio = c.h_ratio;
  s.precond.q = c.q;
  return s;
}

RefSim& R(void* h) { return *static_cast<RefSim*>(h); }

void fill(const PCGReport& r, refn_report* o) {
  if (!o) return;
  o->iterations = r.iterations;
  o->converged = r.converged;
  o->has_condition = r.condition_estimate.has_value();
  o->condition_estimate = r.condition_estimate.value_or(0.0);
  o->n_resid = static_cast<int>(r.residual_history.size());
  o->n_alpha = static_cast<int>(r.alphas.size());
  o->n_beta = static_cast<int>(r.betas.size());
  auto cp = [o](const std::vector<double>& v, double* d) {
    if (d)
      for (int i = 0; i < static_cast<int>(v.size()) && i < o->capacity; ++i) d[i] = v[i];
  };
  cp(r.residual_history, o->residual_history);
  cp(r.alphas, o->alphas);
  cp(r.betas, o->betas);
}

Eigen::VectorXd vec(const double* p, Eigen::Index n) {
  Eigen::VectorXd v(n);
  for (Eigen::Index i = 0; i < n; ++i) v(i) = p[i];
  return v;
}
void out(const Eigen::VectorXd& v, double* p) {
  for (Eigen::Index i = 0; i < v.size(); ++i) p[i] = v(i);
}
}  // namespace

extern "C" {

const char* refn_last_error() { return g_err.c_str(); }
int refn_config_size() { return static_cast<int>(sizeof(refn_config)); }

int refn_sim_create(const refn_config* cfg, void** h) {
  return guarded([&] {
    auto r = std::make_unique<RefSim>();
    r->sim = std::make_unique<Simulation>(convert(*cfg));
    Simulation& s = *r->sim;
    if (cfg->subdomains > 0 && cfg->precond_kind != 0) {
      // agglomerated subdomains, coarse partition S_H (-1: the same)
      r->sub = std::make_unique<AgglomeratedPartition>(agglomerate(*s.mesh_, cfg->subdomains));
      s.precond_.reset();
      s.coarse_.reset();
      if (cfg->precond_kind == 2) {
        const int nH = cfg->coarse_count > 0 ? cfg->coarse_count : cfg->subdomains;
        r->coarse_part = std::make_unique<AgglomeratedPartition>(
            cfg->coarse_count > 0 && cfg->coarse_count != cfg->subdomains ? agglomerate(*s.mesh_, nH) : *r->sub);
        r->coarse_part->parent = s.mesh_.get();
        s.coarse_ = std::make_unique<CoarseEmbedding>(
            build_coarse_embedding(*s.space_, *r->coarse_part, s.config_.coarse_degree()));
      }
      s.precond_ = std::make_unique<SchwarzPreconditioner>(s.K_, *s.space_, *r->sub, s.coarse_.get());
    }
    *h = r.release();
  });
}

void refn_sim_free(void* h) { delete static_cast<RefSim*>(h); }

int64_t refn_sim_dimension(void* h) { return R(h).sim->space().dimension(); }
int refn_sim_n_comp(void* h) { return R(h).sim->model_ ? R(h).sim->model_->state_dim() : 0; }

int refn_sim_step(void* h, int* iterations, int* converged, double* final_residual, int* has_cond, double* cond) {
  return guarded([&] {
    const StepStats s = R(h).sim->step();
    *iterations = s.iterations;
    *converged = s.converged;
    *final_residual = s.final_residual;
    *has_cond = s.condition_estimate.has_value();
    *cond = s.condition_estimate.value_or(0.0);
  });
}

int refn_sim_state(void* h, int* k, double* t, double* U, double* Up, double* Y, double* Yp) {
  return guarded([&] {
    const TimeStepState& st = R(h).sim->state();
    if (k) *k = st.k;
    if (t) *t = st.t;
    const Eigen::Index n = st.U_curr.size();
    if (U) out(st.U_curr, U);
    if (Up) out(st.U_prev, Up);
    for (std::size_t l = 0; l < st.Y_curr.Y.size(); ++l) {
      if (Y) out(st.Y_curr.Y[l], Y + l * n);
      if (Yp) out(st.Y_prev.Y[l], Yp + l * n);
    }
  });
}

// which: 0 K, 1 M, 2 A, 3 E, 4 K0; COO of the CSC matrix; returns nnz (rows == NULL: count only)
int64_t refn_sim_export(void* h, int which, int64_t* rows, int64_t* cols, double* vals) {
  Simulation& s = *R(h).sim;
  const Eigen::SparseMatrix<double>* m = nullptr;
  if (which == 0) m = &s.K_.mat;
  else if (which == 1) m = &s.M_.mat;
  else if (which == 2) m = &s.A_.mat;
  else if (which == 3 && s.coarse_) m = &s.coarse_->E;
  else if (which == 4 && s.precond_ && s.precond_->has_coarse()) m = &s.precond_->coarse_matrix();
  if (!m) return -1;
  int64_t k = 0;
  for (Eigen::Index c = 0; c < m->outerSize(); ++c)
    for (Eigen::SparseMatrix<double>::InnerIterator it(*m, c); it; ++it, ++k)
      if (rows) {
        rows[k] = it.row();
        cols[k] = it.col();
        vals[k] = it.value();
      }
  return k;
}

int refn_sim_apply_K(void* h, const double* x, double* y) {
  return guarded([&] {
    Simulation& s = *R(h).sim;
    Eigen::VectorXd yv;
    s.K_op_->apply(vec(x, s.K_.dimension()), yv);
    out(yv, y);
  });
}

int refn_sim_apply_precond(void* h, const double* r, double* z) {
  return guarded([&] {
    Simulation& s = *R(h).sim;
    if (!s.precond_) throw ConfigError("refnum: no preconditioner");
    Eigen::VectorXd zv;
    s.precond_->apply(vec(r, s.K_.dimension()), zv);
    out(zv, z);
  });
}

int refn_sim_pcg(void* h, const double* b, const double* x0, double tol, int maxit, int use_precond, double* x,
                 refn_report* rep) {
  return guarded([&] {
    Simulation& s = *R(h).sim;
    const Eigen::Index n = s.K_.dimension();
    const LinearOperator* P = use_precond ? s.precond_.get() : nullptr;
    auto res = maxit > 0 || x0 ? pcg_solve(*s.K_op_, vec(b, n), P, tol, maxit > 0 ? maxit : default_max_iterations(n),
                                           x0 ? vec(x0, n) : Eigen::VectorXd::Zero(n))
                               : pcg_solve(*s.K_op_, vec(b, n), P, tol);
    out(res.first, x);
    fill(res.second, rep);
  });
}

// l2_error (dg_space.cpp:94-115) of U against c0 cos(pi x) cos(pi y) e^{-c1 t}
int refn_l2_error_cosine(void* h, const double* U, double c0, double c1, double t, double* err) {
  return guarded([&] {
    Simulation& s = *R(h).sim;
    *err = l2_error(s.space(), vec(U, s.space().dimension()), [=](const Point2& p) {
      return c0 * std::cos(M_PI * p.x) * std::cos(M_PI * p.y) * std::exp(-c1 * t);
    });
  });
}

double refn_mesh_size(void* h) { return R(h).sim->mesh().mesh_size(); }

int refn_cell_means(void* h, const double* U, double* means) {
  return guarded([&] {
    Simulation& s = *R(h).sim;
    const std::vector<double> m = cell_means(s.space(), vec(U, s.space().dimension()));
    std::memcpy(means, m.data(), m.size() * sizeof(double));
  });
}

}  // extern "C"
