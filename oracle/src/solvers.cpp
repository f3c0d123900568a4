// TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// Restates krylov.cpp:12-103 (PCG, Lanczos estimate), schwarz.cpp:13-169
// (coarse embedding, two-level additive Schwarz) and timestepper.cpp:36-200
// (Simulation::step) of /root/reference/proj/src.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <numeric>

#include "oracle.hpp"

namespace orc {

// ---------------- PCG (krylov.cpp:12-76) ----------------
int default_max_iterations(int64_t n) {
  const double cap = 20.0 * std::sqrt(static_cast<double>(n));
  return static_cast<int>(std::min(cap, static_cast<double>(n)));
}

static double dotv(const Vec& a, const Vec& b) {
  double s = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

Vec pcg(const Operator& K, const Vec& b, const Operator* P, double tol, int maxit, const Vec& x0,
        PcgReport& rep) {
  const int64_t n = K.n;
  if (static_cast<int64_t>(b.size()) != n || static_cast<int64_t>(x0.size()) != n)
    throw SolverError("pcg: vector dimension mismatch");
  if (!(tol > 0.0 && tol < 1.0)) throw SolverError("pcg: tol must lie in (0, 1)");
  rep = PcgReport();
  Vec x = x0, r(n), z(n), p(n), q(n);
  K.apply(x, r);
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  const double denom = std::sqrt(dotv(r, r));
  if (denom == 0.0) {
    rep.converged = true;
    rep.resid.push_back(0.0);
    return x;
  }
  auto precond = [&](const Vec& in, Vec& out) {
    if (P) P->apply(in, out);
    else out = in;
  };
  precond(r, z);
  p = z;
  double rho = dotv(r, z);
  if (!std::isfinite(rho)) throw SolverError("pcg: non-finite preconditioned product");
  if (rho <= 0.0) throw SolverError("pcg: preconditioner is not positive definite");
  for (int it = 0; it < maxit; ++it) {
    K.apply(p, q);
    const double pq = dotv(p, q);
    if (!std::isfinite(pq)) throw SolverError("pcg: non-finite operator product");
    if (pq <= 0.0) throw SolverError("pcg: operator is not positive definite");
    const double alpha = rho / pq;
    rep.alpha.push_back(alpha);
    for (int64_t i = 0; i < n; ++i) {
      x[i] += alpha * p[i];
      r[i] -= alpha * q[i];
    }
    const double rel = std::sqrt(dotv(r, r)) / denom;
    rep.resid.push_back(rel);
    ++rep.iterations;
    if (rel < tol) {
      rep.converged = true;
      break;
    }
    precond(r, z);
    const double rho_next = dotv(r, z);
    if (!std::isfinite(rho_next)) throw SolverError("pcg: non-finite scalar");
    if (rho_next <= 0.0) throw SolverError("pcg: preconditioner is not positive definite");
    const double beta = rho_next / rho;
    rep.beta.push_back(beta);
    for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    rho = rho_next;
  }
  rep.has_cond = condition_estimate(rep.alpha, rep.beta, &rep.cond);
  return x;
}

// Lanczos tridiagonal (krylov.cpp:85-103), eigenvalues by implicit QL.
bool condition_estimate(const Vec& alpha, const Vec& beta, double* kappa) {
  const int m = static_cast<int>(alpha.size());
  if (m < 2) return false;
  Vec d(m), e(m, 0.0);
  d[0] = 1.0 / alpha[0];
  for (int k = 1; k < m; ++k) d[k] = 1.0 / alpha[k] + beta[k - 1] / alpha[k - 1];
  for (int k = 0; k + 1 < m; ++k) e[k] = std::sqrt(beta[k]) / alpha[k];
  // implicit QL with Wilkinson-type shifts on (d, e), e[i] couples i and i+1
  for (int l = 0; l < m; ++l) {
    int iter = 0;
    for (;;) {
      int mm = l;
      for (; mm < m - 1; ++mm) {
        const double dd = std::abs(d[mm]) + std::abs(d[mm + 1]);
        if (std::abs(e[mm]) <= 1e-16 * dd) break;
      }
      if (mm == l) break;
      if (++iter > 200) return false;
      double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
      double r = std::hypot(g, 1.0);
      g = d[mm] - d[l] + e[l] / (g + (g >= 0 ? r : -r));
      double s = 1.0, c = 1.0, pp = 0.0;
      int i = mm - 1;
      for (; i >= l; --i) {
        double f = s * e[i];
        const double b = c * e[i];
        r = std::hypot(f, g);
        e[i + 1] = r;
        if (r == 0.0) {
          d[i + 1] -= pp;
          e[mm] = 0.0;
          break;
        }
        s = f / r;
        c = g / r;
        g = d[i + 1] - pp;
        r = (d[i] - g) * s + 2.0 * c * b;
        pp = s * r;
        d[i + 1] = g + pp;
        g = c * r - b;
        (void)f;
      }
      if (r == 0.0 && i >= l) continue;
      d[l] -= pp;
      e[l] = g;
      e[mm] = 0.0;
    }
  }
  const double lo = *std::min_element(d.begin(), d.end());
  const double hi = *std::max_element(d.begin(), d.end());
  if (!(lo > 0.0)) return false;
  *kappa = hi / lo;
  return true;
}

// ---------------- coarse embedding (schwarz.cpp:13-77) ----------------
Csr coarse_embedding(const Discretization& D, const std::vector<int>& owner, int count, int q) {
  const int p = D.p;
  if (q < 1 || q > p) throw ConfigError("coarse embedding: requires 1 <= q <= p");
  const MeshView& m = *D.mesh;
  const int nq = n_modes(q), nl = D.nloc;
  std::vector<Box> box(count);
  std::vector<char> seen(count, 0);
  for (int c = 0; c < m.n_cells(); ++c) {
    const int a = owner[c];
    const Box& cb = m.bbox[c];
    if (!seen[a]) {
      box[a] = cb;
      seen[a] = 1;
    } else {
      box[a].x0 = std::min(box[a].x0, cb.x0);
      box[a].x1 = std::max(box[a].x1, cb.x1);
      box[a].y0 = std::min(box[a].y0, cb.y0);
      box[a].y1 = std::max(box[a].y1, cb.y1);
    }
  }
  // one nl x nq coefficient block per cell, computed in parallel; E's rows
  // (cell-major dofs) hold exactly that block at columns agg*nq.., so the CSR
  // is written directly (no duplicates to sum)
  const int nc = m.n_cells();
  Vec coef(static_cast<std::size_t>(nc) * nl * nq);
  parallel_for(static_cast<std::size_t>(nc), [&](std::size_t ci) {
    const int c = static_cast<int>(ci);
    Vec fv, cv;
    const int a = owner[c];
    const Rule r = polygon_rule(m.cell(c), 2 * p + 2);
    eval_basis(m.bbox[c], p, r.pts, fv, nullptr, nullptr);
    eval_basis(box[a], q, r.pts, cv, nullptr, nullptr);
    Vec mass(nl * nl, 0.0), rhs(nl * nq, 0.0);
    for (std::size_t k = 0; k < r.w.size(); ++k)
      for (int i = 0; i < nl; ++i) {
        for (int j = 0; j < nl; ++j) mass[i * nl + j] += r.w[k] * fv[k * nl + i] * fv[k * nl + j];
        for (int mm = 0; mm < nq; ++mm) rhs[i * nq + mm] += r.w[k] * fv[k * nl + i] * cv[k * nq + mm];
      }
    // dense Cholesky solve mass * coeff = rhs
    Vec Lm(nl * nl, 0.0);
    for (int j = 0; j < nl; ++j) {
      double d = mass[j * nl + j];
      for (int k = 0; k < j; ++k) d -= Lm[j * nl + k] * Lm[j * nl + k];
      Lm[j * nl + j] = std::sqrt(d);
      for (int i = j + 1; i < nl; ++i) {
        double s = mass[i * nl + j];
        for (int k = 0; k < j; ++k) s -= Lm[i * nl + k] * Lm[j * nl + k];
        Lm[i * nl + j] = s / Lm[j * nl + j];
      }
    }
    double* out = &coef[ci * nl * nq];
    for (int mm = 0; mm < nq; ++mm) {
      Vec x(nl);
      for (int i = 0; i < nl; ++i) x[i] = rhs[i * nq + mm];
      for (int i = 0; i < nl; ++i) {
        double s = x[i];
        for (int k = 0; k < i; ++k) s -= Lm[i * nl + k] * x[k];
        x[i] = s / Lm[i * nl + i];
      }
      for (int i = nl - 1; i >= 0; --i) {
        double s = x[i];
        for (int k = i + 1; k < nl; ++k) s -= Lm[k * nl + i] * x[k];
        x[i] = s / Lm[i * nl + i];
      }
      for (int i = 0; i < nl; ++i) out[i * nq + mm] = x[i];
    }
  });
  Csr E;
  E.rows = static_cast<int64_t>(nc) * nl;
  E.cols = static_cast<int64_t>(count) * nq;
  E.ptr.resize(E.rows + 1);
  for (int64_t r = 0; r <= E.rows; ++r) E.ptr[r] = r * nq;
  E.idx.resize(E.rows * nq);
  E.val.assign(coef.begin(), coef.end());
  for (int64_t r = 0; r < E.rows; ++r)
    for (int mm = 0; mm < nq; ++mm) E.idx[r * nq + mm] = static_cast<int64_t>(owner[r / nl]) * nq + mm;
  return E;
}

// ---------------- Schwarz (schwarz.cpp:79-169) ----------------
void Schwarz::build(const Csr& K, const Discretization& D, const std::vector<int>& sub_owner, int n_sub,
                    const std::vector<int>& coarse_owner, int n_coarse, int q) {
  n = K.rows;
  const int nl = D.nloc;
  dofs.assign(n_sub, {});
  for (int c = 0; c < D.mesh->n_cells(); ++c)
    for (int i = 0; i < nl; ++i) dofs[sub_owner[c]].push_back(static_cast<int64_t>(c) * nl + i);
  local.assign(n_sub, BlockChol());
  std::vector<std::string> err(n_sub);
  parallel_for(n_sub, [&](std::size_t s) {
    const auto& d = dofs[s];
    std::vector<int64_t> g2l;
    std::vector<Triplet> t;
    // principal submatrix: dofs are sorted, so binary search maps global -> local
    for (std::size_t j = 0; j < d.size(); ++j)
      for (int64_t k = K.ptr[d[j]]; k < K.ptr[d[j] + 1]; ++k) {
        const auto it = std::lower_bound(d.begin(), d.end(), K.idx[k]);
        if (it != d.end() && *it == K.idx[k]) t.push_back({static_cast<int64_t>(j), it - d.begin(), K.val[k]});
      }
    const Csr Ki = from_triplets(static_cast<int64_t>(d.size()), static_cast<int64_t>(d.size()), t);
    try {
      local[s].factor(Ki, nl);
    } catch (const SolverError&) {
      err[s] = "schwarz: subdomain " + std::to_string(s) + " factorization failed (not positive definite)";
    }
  });
  for (const auto& e : err)
    if (!e.empty()) throw SolverError(e);
  two_level = n_coarse > 0;
  if (std::getenv("ORC_TIMES")) std::fprintf(stderr, "oracle setup: local factors done\n");
  const auto tE = std::chrono::steady_clock::now();
  if (two_level) {
    E = coarse_embedding(D, coarse_owner, n_coarse, q);
    Et = transpose(E);
    K0 = multiply(Et, multiply(K, E));
    if (std::getenv("ORC_TIMES"))
      std::fprintf(stderr, "oracle setup: E, K0 %.2f s\n",
                   std::chrono::duration<double>(std::chrono::steady_clock::now() - tE).count());
    try {
      coarse.factor(K0, n_modes(q));
    } catch (const SolverError&) {
      throw SolverError("schwarz: coarse operator factorization failed");
    }
  }
}

void Schwarz::apply(const Vec& r, Vec& z) const {
  if (static_cast<int64_t>(r.size()) != n) throw SolverError("schwarz apply: dimension mismatch");
  z.assign(n, 0.0);
  parallel_for(dofs.size(), [&](std::size_t s) {
    const auto& d = dofs[s];
    Vec loc(d.size());
    for (std::size_t i = 0; i < d.size(); ++i) loc[i] = r[d[i]];
    local[s].solve(loc);
    for (std::size_t i = 0; i < d.size(); ++i) z[d[i]] = loc[i];
  });
  if (two_level) {
    Vec r0, corr;
    Et.apply(r, r0);
    coarse.solve(r0);
    E.apply(r0, corr);
    for (int64_t i = 0; i < n; ++i) z[i] += corr[i];
  }
}

// ---------------- Simulation (timestepper.cpp:67-200) ----------------
double Simulation::initial(P2 x) const {
  switch (cfg.init_kind) {
    case 0: {
      const double dx = x.x - cfg.omega0.x, dy = x.y - cfg.omega0.y;
      return dx * dx + dy * dy < cfg.omega0_r2 ? cfg.u_patch : cfg.u_rest;
    }
    case 1: return cfg.init_params[0];
    case 2: return cfg.init_params[0] * std::cos(M_PI * x.x) * std::cos(M_PI * x.y) + cfg.init_params[1];
    case 3:
      return cfg.init_params[0] + cfg.init_params[1] * x.x + cfg.init_params[2] * x.y +
             cfg.init_params[3] * x.x * x.y;
  }
  throw ConfigError("unknown initial condition");
}

void Simulation::build(const Config& c, MeshView m, const std::vector<int>& sub_owner, int n_sub,
                       const std::vector<int>& coarse_owner, int n_coarse) {
  cfg = c;
  if (!(c.dt > 0.0)) throw ConfigError("time.dt must be positive");
  if (!(c.tol > 0.0 && c.tol < 1.0)) throw ConfigError("solver.tol must lie in (0, 1)");
  static const bool times = std::getenv("ORC_TIMES") != nullptr;
  auto t0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!times) return;
    const auto t1 = std::chrono::steady_clock::now();
    std::fprintf(stderr, "oracle setup: %s %.2f s\n", what, std::chrono::duration<double>(t1 - t0).count());
    t0 = t1;
  };
  mesh = std::move(m);
  mesh.build();
  lap("mesh topology");
  D.build(mesh, cfg);
  lap("assembly");
  has_precond = cfg.precond != 0;
  if (has_precond) {
    const int q = cfg.q > 0 ? cfg.q : cfg.degree;
    S.build(D.K, D, sub_owner, n_sub, coarse_owner, cfg.precond == 2 ? n_coarse : 0, q);
    lap("schwarz");
  }
  U = D.l2_project([this](P2 x) { return initial(x); });
  Up = U;
  Y.clear();
  double u_rest = 0.0, y_rest[4] = {0.0, 0.0, 0.0, 0.0};
  const int ncomp = model_rest(cfg, &u_rest, y_rest);
  for (int l = 0; l < ncomp; ++l) {  // timestepper.cpp:116-123
    const double v = y_rest[l];
    Y.push_back(D.l2_project([v](P2) { return v; }));
  }
  Yp = Y;
  k = 0;
  t = 0.0;
}

Vec Simulation::external_term(double t_mid) const {
  Vec F(U.size(), 0.0), val;
  const int nl = D.nloc;
  for (int e = 0; e < mesh.n_cells(); ++e) {
    const Rule r = polygon_rule(mesh.cell(e), 2 * D.p + 2);
    eval_basis(mesh.bbox[e], D.p, r.pts, val, nullptr, nullptr);
    for (std::size_t q = 0; q < r.w.size(); ++q) {
      const P2 x = r.pts[q];
      double g = 0.0;
      if (cfg.stim_kind == 1)
        g = (x.x < cfg.stim_params[1] && t_mid < cfg.stim_params[2]) ? cfg.stim_params[0] : 0.0;
      else if (cfg.stim_kind == 2)
        g = cfg.stim_params[0] * std::cos(M_PI * x.x) * std::cos(M_PI * x.y) * std::exp(-cfg.stim_params[1] * t_mid);
      for (int i = 0; i < nl; ++i) F[static_cast<int64_t>(e) * nl + i] += r.w[q] * g * val[q * nl + i];
    }
  }
  return F;
}

StepStats Simulation::step() {
  const bool has_prev = k > 0;
  const double dt = cfg.dt;
  const int64_t n = static_cast<int64_t>(U.size());
  Vec rhs;
  D.Krhs.apply(U, rhs);
  if (cfg.ionic != 0) {
    Vec us = U;
    std::vector<Vec> ys = Y;
    if (has_prev) {
      for (int64_t i = 0; i < n; ++i) us[i] = 2.0 * U[i] - Up[i];
      for (std::size_t l = 0; l < Y.size(); ++l)
        for (int64_t i = 0; i < n; ++i) ys[l][i] = 2.0 * Y[l][i] - Yp[l][i];
    }
    bool oob = false;
    const IonicTerms at_star = ionic_terms(D, us, ys, cfg, &oob);
    if (oob) std::fprintf(stderr, "oracle: warning: membrane potential left the admissible range\n");
    for (int64_t i = 0; i < n; ++i) rhs[i] -= (cfg.chi_m * dt) * at_star.I[i];
  }
  if (cfg.stim_kind != 0) {
    const Vec F = external_term(t + 0.5 * dt);
    for (int64_t i = 0; i < n; ++i) rhs[i] += dt * F[i];
  }
  const int maxit = cfg.maxit > 0 ? cfg.maxit : default_max_iterations(n);
  const Vec x0 = cfg.warm_start ? U : Vec(n, 0.0);
  Operator Kop{n, [this](const Vec& x, Vec& y) { D.K.apply(x, y); }};
  Operator Pop{n, [this](const Vec& x, Vec& y) { S.apply(x, y); }};
  PcgReport rep;
  Vec u_next = pcg(Kop, rhs, has_precond ? &Pop : nullptr, cfg.tol, maxit, x0, rep);
  if (!rep.converged) {
    char buf[256];
    std::snprintf(buf, sizeof buf, "time step %d: PCG did not converge within %d iterations (residual %f)",
                  k + 1, maxit, rep.resid.empty() ? 1.0 : rep.resid.back());
    throw SolverError(buf);
  }
  if (cfg.ionic != 0 && !Y.empty()) {
    const IonicTerms at_curr = ionic_terms(D, U, Y, cfg, nullptr);
    std::vector<Vec> ynext = Y;
    for (std::size_t l = 0; l < ynext.size(); ++l) {
      const Vec s = D.mass_solve(at_curr.G[l]);
      for (int64_t i = 0; i < n; ++i) ynext[l][i] -= dt * s[i];
    }
    Yp = std::move(Y);
    Y = std::move(ynext);
  }
  Up = std::move(U);
  U = std::move(u_next);
  k += 1;
  t = k * dt;
  StepStats st;
  st.iterations = rep.iterations;
  st.final_residual = rep.resid.empty() ? 0.0 : rep.resid.back();
  st.converged = rep.converged;
  st.has_cond = rep.has_cond;
  st.cond = rep.cond;
  return st;
}

}  // namespace orc
