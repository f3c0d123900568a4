// TEST INFRASTRUCTURE ONLY: C-ABI of the CPU oracle (oracle/build/libpdg_oracle.so).
// The config struct has the same C layout as include/polydg_b200.h's
// pdg_config so tests can pass one ctypes structure to both; it is redeclared
// here so the oracle does not compile against product headers.
#include <cstring>
#include <memory>
#include <random>
#include <string>

#include "oracle.hpp"

extern "C" {
typedef struct orc_config {
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
} orc_config;

typedef struct orc_report {
  int iterations, converged, has_condition;
  double condition_estimate;
  int capacity;
  double *residual_history, *alphas, *betas;
  int n_resid, n_alpha, n_beta;
} orc_report;
}

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const orc::ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const orc::SolverError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 7;
  }
}

orc::Config convert(const orc_config& c) {
  orc::Config o;
  o.degree = c.degree;
  o.eta0 = c.eta0;
  o.chi_m = c.chi_m;
  o.C_m = c.C_m;
  o.dt = c.dt;
  o.T = c.T;
  o.sgl = c.sigma_grey_l;
  o.sgn = c.sigma_grey_n;
  o.swl = c.sigma_white_l;
  o.swn = c.sigma_white_n;
  o.fiber_grey = {c.fiber_grey[0], c.fiber_grey[1]};
  o.fiber_white = {c.fiber_white[0], c.fiber_white[1]};
  o.fiber_random = c.fiber_random;
  o.fiber_seed = c.fiber_seed;
  o.ionic = c.ionic_model;
  if (o.ionic > 2) throw orc::ConfigError("oracle: unknown ionic model");
  std::memcpy(o.fhn, c.fhn, sizeof o.fhn);
  std::memcpy(o.bc, c.bc, sizeof o.bc);
  o.init_kind = c.init_kind;
  o.u_rest = c.u_rest;
  o.u_patch = c.u_patch;
  o.omega0 = {c.omega0[0], c.omega0[1]};
  o.omega0_r2 = c.omega0_r2;
  std::memcpy(o.init_params, c.init_params, sizeof o.init_params);
  o.stim_kind = c.stim_kind;
  std::memcpy(o.stim_params, c.stim_params, sizeof o.stim_params);
  o.tol = c.tol;
  o.maxit = c.maxit;
  o.warm_start = c.warm_start;
  o.precond = c.precond_kind;
  o.q = c.q;
  return o;
}

void fill(const orc::PcgReport& r, orc_report* o) {
  if (!o) return;
  o->iterations = r.iterations;
  o->converged = r.converged;
  o->has_condition = r.has_cond;
  o->condition_estimate = r.cond;
  o->n_resid = static_cast<int>(r.resid.size());
  o->n_alpha = static_cast<int>(r.alpha.size());
  o->n_beta = static_cast<int>(r.beta.size());
  auto cp = [o](const orc::Vec& v, double* d) {
    if (d)
      for (int i = 0; i < static_cast<int>(v.size()) && i < o->capacity; ++i) d[i] = v[i];
  };
  cp(r.resid, o->residual_history);
  cp(r.alpha, o->alphas);
  cp(r.beta, o->betas);
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }
int orc_config_size() { return static_cast<int>(sizeof(orc_config)); }
int orc_threads() { return orc::thread_count(); }
void orc_set_parallel(int on) { orc::set_parallel_ops(on != 0); }
void orc_set_lean(int level) { orc::set_lean(level); }

// SimulationConfig defaults (timestepper.hpp:21-80, ionics.hpp:42-51), so the
// oracle can be configured without loading the product library
void orc_config_default(orc_config* c) {
  std::memset(c, 0, sizeof *c);
  const orc::Config d;
  c->mesh_cells = 512;
  c->mesh_seed = 42;
  c->mesh_lloyd = 20;
  c->domain[2] = c->domain[3] = 1.0;
  c->split_y = 0.5;
  c->degree = d.degree;
  c->eta0 = d.eta0;
  c->chi_m = d.chi_m;
  c->C_m = d.C_m;
  c->dt = d.dt;
  c->T = d.T;
  c->sigma_grey_l = d.sgl;
  c->sigma_grey_n = d.sgn;
  c->sigma_white_l = d.swl;
  c->sigma_white_n = d.swn;
  c->fiber_grey[1] = c->fiber_white[1] = 1.0;
  c->fiber_seed = 42;
  c->ionic_model = 1;
  std::memcpy(c->fhn, d.fhn, sizeof d.fhn);
  std::memcpy(c->bc, d.bc, sizeof d.bc);
  c->init_kind = 0;
  c->u_rest = d.u_rest;
  c->u_patch = d.u_patch;
  c->omega0[0] = d.omega0.x;
  c->omega0[1] = d.omega0.y;
  c->omega0_r2 = d.omega0_r2;
  c->tol = d.tol;
  c->warm_start = 1;
  c->precond_kind = 2;
  c->h_ratio = 2;
  c->world = 1;
}

// b_i = 2 (rng()>>11) 2^-53 - 1 with mt19937_64(seed) (acceptance.cpp:285-286)
void orc_uniform_rhs(uint64_t seed, int64_t n, double* out) {
  std::mt19937_64 rng(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = 2.0 * (static_cast<double>(rng() >> 11) * 0x1.0p-53) - 1.0;
}

// stored blocks of the local factors (sum over subdomains) and of the coarse factor
int64_t orc_sim_factor_blocks(void* h, int which) {
  const auto& s = *static_cast<orc::Simulation*>(h);
  if (which == 1) return s.S.coarse.blocks();
  int64_t t = 0;
  for (const auto& f : s.S.local) t += f.blocks();
  return t;
}

int orc_sim_create(const orc_config* cfg, const double* verts, int nv, const int* off, const int* idx,
                   int nc, const uint8_t* regions, const int* sub_owner, int n_sub,
                   const int* coarse_owner, int n_coarse, void** out) {
  return guarded([&] {
    orc::MeshView m;
    m.verts.resize(nv);
    for (int i = 0; i < nv; ++i) m.verts[i] = {verts[2 * i], verts[2 * i + 1]};
    m.off.assign(off, off + nc + 1);
    m.idx.assign(idx, idx + off[nc]);
    m.region.assign(regions, regions + nc);
    auto s = std::make_unique<orc::Simulation>();
    s->build(convert(*cfg), std::move(m), std::vector<int>(sub_owner, sub_owner + nc), n_sub,
             coarse_owner ? std::vector<int>(coarse_owner, coarse_owner + nc) : std::vector<int>(),
             coarse_owner ? n_coarse : 0);
    *out = s.release();
  });
}

void orc_sim_free(void* h) { delete static_cast<orc::Simulation*>(h); }

int orc_sim_step(void* h, int* iterations, int* converged, double* final_residual, int* has_cond,
                 double* cond) {
  return guarded([&] {
    const orc::StepStats s = static_cast<orc::Simulation*>(h)->step();
    *iterations = s.iterations;
    *converged = s.converged;
    *final_residual = s.final_residual;
    *has_cond = s.has_cond;
    *cond = s.cond;
  });
}

int orc_sim_state(void* h, int* k, double* t, double* U, double* Up, double* Y, double* Yp) {
  return guarded([&] {
    auto& s = *static_cast<orc::Simulation*>(h);
    if (k) *k = s.k;
    if (t) *t = s.t;
    const std::size_t n = s.U.size();
    if (U) std::memcpy(U, s.U.data(), n * sizeof(double));
    if (Up) std::memcpy(Up, s.Up.data(), n * sizeof(double));
    for (std::size_t l = 0; l < s.Y.size(); ++l) {
      if (Y) std::memcpy(Y + l * n, s.Y[l].data(), n * sizeof(double));
      if (Yp) std::memcpy(Yp + l * n, s.Yp[l].data(), n * sizeof(double));
    }
  });
}

int orc_sim_set_state(void* h, int k, const double* U, const double* Up, const double* Y, const double* Yp) {
  return guarded([&] {
    auto& s = *static_cast<orc::Simulation*>(h);
    s.k = k;
    s.t = k * s.cfg.dt;
    const std::size_t n = s.U.size();
    if (U) s.U.assign(U, U + n);
    if (Up) s.Up.assign(Up, Up + n);
    for (std::size_t l = 0; l < s.Y.size(); ++l) {
      if (Y) s.Y[l].assign(Y + l * n, Y + (l + 1) * n);
      if (Yp) s.Yp[l].assign(Yp + l * n, Yp + (l + 1) * n);
    }
  });
}

int64_t orc_sim_dimension(void* h) { return static_cast<int64_t>(static_cast<orc::Simulation*>(h)->U.size()); }

int orc_sim_apply_K(void* h, const double* x, double* y) {
  return guarded([&] {
    auto& s = *static_cast<orc::Simulation*>(h);
    orc::Vec xv(x, x + s.U.size()), yv;
    s.D.K.apply(xv, yv);
    std::memcpy(y, yv.data(), yv.size() * sizeof(double));
  });
}

int orc_sim_apply_precond(void* h, const double* r, double* z) {
  return guarded([&] {
    auto& s = *static_cast<orc::Simulation*>(h);
    orc::Vec rv(r, r + s.U.size()), zv;
    if (s.has_precond) s.S.apply(rv, zv);
    else zv = rv;
    std::memcpy(z, zv.data(), zv.size() * sizeof(double));
  });
}

int orc_sim_pcg(void* h, const double* b, const double* x0, double tol, int maxit, int use_precond,
                double* x, orc_report* rep) {
  return guarded([&] {
    auto& s = *static_cast<orc::Simulation*>(h);
    const int64_t n = static_cast<int64_t>(s.U.size());
    orc::Operator K{n, [&s](const orc::Vec& a, orc::Vec& o) { s.D.K.apply(a, o); }};
    orc::Operator P{n, [&s](const orc::Vec& a, orc::Vec& o) { s.S.apply(a, o); }};
    orc::PcgReport r;
    const orc::Vec xv = orc::pcg(K, orc::Vec(b, b + n), (use_precond && s.has_precond) ? &P : nullptr, tol,
                                 maxit > 0 ? maxit : orc::default_max_iterations(n),
                                 x0 ? orc::Vec(x0, x0 + n) : orc::Vec(n, 0.0), r);
    std::memcpy(x, xv.data(), n * sizeof(double));
    fill(r, rep);
  });
}

// which: 0 K, 1 M, 2 A, 3 E, 4 K0, 5 K_rhs
int64_t orc_sim_export(void* h, int which, int64_t* rows, int64_t* cols, double* vals) {
  auto& s = *static_cast<orc::Simulation*>(h);
  const orc::Csr* A = nullptr;
  switch (which) {
    case 0: A = &s.D.K; break;
    case 1: A = &s.D.M; break;
    case 2: A = &s.D.A; break;
    case 3: A = s.S.two_level ? &s.S.E : nullptr; break;
    case 4: A = s.S.two_level ? &s.S.K0 : nullptr; break;
    case 5: A = &s.D.Krhs; break;
  }
  if (!A) return -1;
  if (rows)
    for (int64_t r = 0; r < A->rows; ++r)
      for (int64_t k = A->ptr[r]; k < A->ptr[r + 1]; ++k) {
        rows[k] = r;
        cols[k] = A->idx[k];
        vals[k] = A->val[k];
      }
  return static_cast<int64_t>(A->val.size());
}

int orc_sim_ionic_terms(void* h, const double* U, const double* Y, double* I, double* G) {
  return guarded([&] {
    auto& s = *static_cast<orc::Simulation*>(h);
    const std::size_t n = s.U.size();
    std::vector<orc::Vec> yv;
    for (std::size_t l = 0; l < s.Y.size(); ++l) yv.emplace_back(Y + l * n, Y + (l + 1) * n);
    const orc::IonicTerms t = orc::ionic_terms(s.D, orc::Vec(U, U + n), yv, s.cfg, nullptr);
    std::memcpy(I, t.I.data(), n * sizeof(double));
    for (std::size_t l = 0; l < t.G.size(); ++l) std::memcpy(G + l * n, t.G[l].data(), n * sizeof(double));
  });
}

int orc_sim_cell_means(void* h, const double* U, double* means) {
  return guarded([&] {
    auto& s = *static_cast<orc::Simulation*>(h);
    const orc::Vec m = orc::cell_means(s.D, orc::Vec(U, U + s.U.size()));
    std::memcpy(means, m.data(), m.size() * sizeof(double));
  });
}

// l2_error against c0 cos(pi x) cos(pi y) e^{-c1 t} (acceptance.cpp:147-150)
int orc_l2_error_cosine(void* h, const double* U, double c0, double c1, double t, double* err) {
  return guarded([&] {
    auto& s = *static_cast<orc::Simulation*>(h);
    *err = orc::l2_error(s.D, orc::Vec(U, U + s.U.size()), [=](orc::P2 p) {
      return c0 * std::cos(M_PI * p.x) * std::cos(M_PI * p.y) * std::exp(-c1 * t);
    });
  });
}

double orc_mesh_size(void* h) { return static_cast<orc::Simulation*>(h)->mesh.mesh_size(); }

int orc_pcg_dense(int n, const double* A, const double* b, const double* Pm, double tol, int maxit,
                  const double* x0, double* x, orc_report* rep) {
  return guarded([&] {
    orc::Operator K{n, [A, n](const orc::Vec& a, orc::Vec& o) {
                      o.assign(n, 0.0);
                      for (int i = 0; i < n; ++i) {
                        double s = 0.0;
                        for (int j = 0; j < n; ++j) s += A[static_cast<int64_t>(i) * n + j] * a[j];
                        o[i] = s;
                      }
                    }};
    orc::Operator P{n, [Pm, n](const orc::Vec& a, orc::Vec& o) {
                      o.assign(n, 0.0);
                      for (int i = 0; i < n; ++i) {
                        double s = 0.0;
                        for (int j = 0; j < n; ++j) s += Pm[static_cast<int64_t>(i) * n + j] * a[j];
                        o[i] = s;
                      }
                    }};
    orc::PcgReport r;
    const orc::Vec xv = orc::pcg(K, orc::Vec(b, b + n), Pm ? &P : nullptr, tol,
                                 maxit > 0 ? maxit : orc::default_max_iterations(n),
                                 x0 ? orc::Vec(x0, x0 + n) : orc::Vec(n, 0.0), r);
    std::memcpy(x, xv.data(), n * sizeof(double));
    fill(r, rep);
  });
}

int orc_condition_estimate(const double* alpha, const double* beta, int m, double* kappa) {
  return orc::condition_estimate(orc::Vec(alpha, alpha + m), orc::Vec(beta, beta + (m > 0 ? m - 1 : 0)), kappa)
             ? 1
             : 0;
}

int orc_fhn(const double* prm, double u, double w, double* f, double* m) {
  return guarded([&] {
    *f = orc::fhn_current(prm, u, w);
    *m = orc::fhn_rate(prm, u, w);
  });
}

int orc_bc(const double* prm, double u, const double* y, double* f, double* m) {
  return guarded([&] {
    *f = orc::bc_current(prm, u, y);
    orc::bc_rates(prm, u, y, m);
  });
}

int orc_ionic_rest(const orc_config* c, int* n_comp, double* u, double* y) {
  return guarded([&] { *n_comp = orc::model_rest(convert(*c), u, y); });
}

int orc_polygon_quadrature(const double* poly, int n, int order, double* pts, double* w, int cap) {
  std::vector<orc::P2> p(n);
  for (int i = 0; i < n; ++i) p[i] = {poly[2 * i], poly[2 * i + 1]};
  const orc::Rule r = orc::polygon_rule(p, order);
  for (int i = 0; i < static_cast<int>(r.w.size()) && i < cap; ++i) {
    pts[2 * i] = r.pts[i].x;
    pts[2 * i + 1] = r.pts[i].y;
    w[i] = r.w[i];
  }
  return static_cast<int>(r.w.size());
}

}  // extern "C"
