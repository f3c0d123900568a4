// Problem setup (see problem.hpp). Reference anchors:
//   config validation          timestepper.cpp:15-34
//   conductivity tensors       assembly.cpp:13-32, penalty :38-47
//   mass / SIPG stiffness      assembly.cpp:89-183 (volume first, then faces)
//   K = C_m chi_m M + dt/2 A    assembly.cpp:185-202
//   mass block solver          assembly.cpp:204-226
//   L2 projection              assembly.cpp:228-242
//   coarse embedding E         schwarz.cpp:13-77, K0 = E^T K E :138-146
//   subdomain factors          schwarz.cpp:99-136
#include <chrono>
#include <cstdio>
#include "problem.hpp"
#include "bc_model.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <functional>
#include <map>
#include <numeric>
#include <random>
#include <string>

#include "ordering.hpp"
#include "parallel.hpp"
#include "quadrature.hpp"

namespace pdg {

namespace {

struct Tensor {
  double t00, t01, t10, t11;
};

Tensor make_tensor(double sl, double sn, double fx, double fy) {
  const double len = std::hypot(fx, fy);
  if (!(len > 0.0)) throw ConfigError("conductivity: zero fiber direction");
  const double nx = -fy / len, ny = fx / len;
  Tensor t{sl, 0.0, 0.0, sl};
  t.t00 += (sn - sl) * nx * nx;
  t.t01 += (sn - sl) * nx * ny;
  t.t10 += (sn - sl) * ny * nx;
  t.t11 += (sn - sl) * ny * ny;
  return t;
}

bool is_pow2(int r) { return r >= 2 && (r & (r - 1)) == 0; }

std::uint32_t morton(double x, double y, const Box& d) {
  auto q = [](double v) {
    v = std::clamp(v, 0.0, 1.0);
    return static_cast<std::uint32_t>(v * 65535.0);
  };
  auto spread = [](std::uint32_t v) {
    v &= 0xffff;
    v = (v | (v << 8)) & 0x00ff00ff;
    v = (v | (v << 4)) & 0x0f0f0f0f;
    v = (v | (v << 2)) & 0x33333333;
    v = (v | (v << 1)) & 0x55555555;
    return v;
  };
  return spread(q((x - d.xmin) / d.width())) | (spread(q((y - d.ymin) / d.height())) << 1);
}

// In-place inverse of a small SPD block (column-major) through Cholesky.
void spd_inverse(int n, const double* a, double* inv) {
  std::vector<double> L(static_cast<std::size_t>(n) * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double d = a[j * n + j];
    for (int k = 0; k < j; ++k) d -= L[k * n + j] * L[k * n + j];
    if (!(d > 0.0)) throw SolverError("mass block is not positive definite");
    d = std::sqrt(d);
    L[j * n + j] = d;
    for (int i = j + 1; i < n; ++i) {
      double s = a[j * n + i];
      for (int k = 0; k < j; ++k) s -= L[k * n + i] * L[k * n + j];
      L[j * n + i] = s / d;
    }
  }
  // inv = L^-T L^-1 column by column
  std::vector<double> x(n);
  for (int c = 0; c < n; ++c) {
    std::fill(x.begin(), x.end(), 0.0);
    x[c] = 1.0;
    for (int i = 0; i < n; ++i) {
      double s = x[i];
      for (int k = 0; k < i; ++k) s -= L[k * n + i] * x[k];
      x[i] = s / L[i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = x[i];
      for (int k = i + 1; k < n; ++k) s -= L[i * n + k] * x[k];
      x[i] = s / L[i * n + i];
    }
    for (int i = 0; i < n; ++i) inv[c * n + i] = x[i];
  }
}

// Solve SPD (n x n, column-major) X = R (n x m) via Cholesky.
void spd_solve(int n, int m, const double* a, double* r) {
  std::vector<double> inv(static_cast<std::size_t>(n) * n);
  std::vector<double> L(static_cast<std::size_t>(n) * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double d = a[j * n + j];
    for (int k = 0; k < j; ++k) d -= L[k * n + j] * L[k * n + j];
    if (!(d > 0.0)) throw SolverError("coarse embedding: cell mass not positive definite");
    d = std::sqrt(d);
    L[j * n + j] = d;
    for (int i = j + 1; i < n; ++i) {
      double s = a[j * n + i];
      for (int k = 0; k < j; ++k) s -= L[k * n + i] * L[k * n + j];
      L[j * n + i] = s / d;
    }
  }
  for (int c = 0; c < m; ++c) {
    double* x = r + static_cast<std::size_t>(c) * n;
    for (int i = 0; i < n; ++i) {
      double s = x[i];
      for (int k = 0; k < i; ++k) s -= L[k * n + i] * x[k];
      x[i] = s / L[i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = x[i];
      for (int k = i + 1; k < n; ++k) s -= L[i * n + k] * x[k];
      x[i] = s / L[i * n + i];
    }
  }
}

double init_value(const pdg_config& c, Pt x) {
  switch (c.init_kind) {
    case PDG_INIT_DISC: {
      const double dx = x.x - c.omega0[0], dy = x.y - c.omega0[1];
      return dx * dx + dy * dy < c.omega0_r2 ? c.u_patch : c.u_rest;
    }
    case PDG_INIT_CONSTANT:
      return c.init_params[0];
    case PDG_INIT_COSINE:
      return c.init_params[0] * std::cos(M_PI * x.x) * std::cos(M_PI * x.y) + c.init_params[1];
    case PDG_INIT_BILINEAR:
      return c.init_params[0] + c.init_params[1] * x.x + c.init_params[2] * x.y +
             c.init_params[3] * x.x * x.y;
  }
  throw ConfigError("unknown initial condition kind");
}

}  // namespace

int ionic_rest(const pdg_config& c, double& u, double* y) {
  if (c.ionic_model == PDG_IONIC_FHN) {  // ionics.hpp:56-57
    u = c.fhn[5];
    y[0] = 0.0;
    return 1;
  }
  if (c.ionic_model != PDG_IONIC_BARRETO_CRESSMAN) {
    u = c.u_rest;
    return 0;
  }
  // Barreto-Cressman rest: gates at their steady state n_inf(u), h_inf(u) and
  // (u, [K]o, [Na]i) solving I = 0, d[K]o/dt = 0, d[Na]i/dt = 0 (Newton with a
  // forward-difference Jacobian from u = -68 mV, [K]o = k_bath, [Na]i = Na_i0)
  const double* P = c.bc;
  auto full = [&](const double* z, double* yy) {
    double an, bn, ah, bh;
    bc::gating_rates(z[0], an, bn, ah, bh);
    yy[0] = an / (an + bn);
    yy[1] = ah / (ah + bh);
    yy[2] = z[1];
    yy[3] = z[2];
  };
  auto resid = [&](const double* z, double* f) {
    double yy[4], m[4];
    full(z, yy);
    bc::rates(P, z[0], yy, m);
    f[0] = bc::current(P, z[0], yy);
    f[1] = m[2] * P[PDG_BC_TAU];
    f[2] = m[3] * P[PDG_BC_TAU];
  };
  double z[3] = {-68.0, P[PDG_BC_K_BATH], P[PDG_BC_NA_I0]};
  bool ok = false;
  for (int it = 0; it < 100 && !ok; ++it) {
    double f[3], J[3][3];
    resid(z, f);
    for (int j = 0; j < 3; ++j) {
      double zz[3] = {z[0], z[1], z[2]}, g[3];
      const double h = 1e-7 * std::max(1.0, std::fabs(z[j]));
      zz[j] += h;
      resid(zz, g);
      for (int i = 0; i < 3; ++i) J[i][j] = (g[i] - f[i]) / h;
    }
    // Cramer's rule on the 3x3 system J dz = -f
    auto det3 = [](double a[3][3]) {
      return a[0][0] * (a[1][1] * a[2][2] - a[1][2] * a[2][1]) - a[0][1] * (a[1][0] * a[2][2] - a[1][2] * a[2][0]) +
             a[0][2] * (a[1][0] * a[2][1] - a[1][1] * a[2][0]);
    };
    const double d = det3(J);
    if (!std::isfinite(d) || d == 0.0) break;
    double step = 0.0;
    for (int j = 0; j < 3; ++j) {
      double a[3][3];
      for (int r = 0; r < 3; ++r)
        for (int k = 0; k < 3; ++k) a[r][k] = k == j ? -f[r] : J[r][k];
      const double dz = det3(a) / d;
      z[j] += dz;
      step = std::max(step, std::fabs(dz) / std::max(1.0, std::fabs(z[j])));
    }
    ok = step < 1e-14;
  }
  if (!ok || !(z[1] > 0.0) || !(z[2] > 0.0))
    throw ConfigError("barreto-cressman: no resting state found for these parameters");
  u = z[0];
  full(z, y);
  return 4;
}

void validate_config(const pdg_config& c) {
  if (!(c.dt > 0.0)) throw ConfigError("time.dt must be positive");
  if (!(c.T >= c.dt)) throw ConfigError("time.T must be at least one step");
  if (!(c.tol > 0.0 && c.tol < 1.0)) throw ConfigError("solver.tol must lie in (0, 1)");
  if (c.degree < 1) throw ConfigError("fem.degree must be >= 1");
  if (c.degree > 6) throw ConfigError("fem.degree above 6 is not supported on the device path");
  if (!(c.eta0 > 0.0)) throw ConfigError("fem.eta0 must be positive");
  if (!(c.chi_m > 0.0)) throw ConfigError("membrane.chi must be positive");
  if (!(c.C_m > 0.0)) throw ConfigError("membrane.Cm must be positive");
  if (!(c.sigma_grey_l > 0.0 && c.sigma_grey_n > 0.0 && c.sigma_white_l > 0.0 && c.sigma_white_n > 0.0))
    throw ConfigError("conductivity: all sigma values must be positive");
  if (c.mesh_cells < 1) throw ConfigError("generate_polygonal_mesh: n_cells must be >= 1");
  if (c.precond_kind < 0 || c.precond_kind > 2) throw ConfigError("precond.kind must be none, block-jacobi or two-level");
  if (c.precond_kind == PDG_PRECOND_TWO_LEVEL) {
    if (c.coarse_count == 0 && !is_pow2(c.h_ratio))
      throw ConfigError("precond.H_ratio must be a power of two >= 2");
    const int q = c.q > 0 ? c.q : c.degree;
    if (q > c.degree) throw ConfigError("precond.q must not exceed fem.degree");
    if (c.coarse_count == -1 && c.subdomains <= 0)
      throw ConfigError("precond.coarse = subdomains needs precond.subdomains > 0");
  }
  if (c.subdomains < 0 || c.subdomains > c.mesh_cells)
    throw ConfigError("precond.subdomains must lie in [0, mesh.cells]");
  if (c.coarse_count > c.mesh_cells || c.coarse_count < -1)
    throw ConfigError("precond.coarse must lie in [-1, mesh.cells]");
  if (c.ionic_model == PDG_IONIC_FHN) {
    if (!(c.fhn[6] > c.fhn[5])) throw ConfigError("fhn: u_max must exceed u_min");
    if (!(c.fhn[1] >= 0.0 && c.fhn[2] > 0.0)) throw ConfigError("fhn: invalid rate constants");
  } else if (c.ionic_model == PDG_IONIC_BARRETO_CRESSMAN) {
    for (int k = 0; k < PDG_BC_NPARAM; ++k)
      if (!std::isfinite(c.bc[k]) || c.bc[k] < 0.0)
        throw ConfigError("barreto-cressman: parameters must be finite and non-negative");
    if (!(c.bc[PDG_BC_TAU] > 0.0 && c.bc[PDG_BC_RTF] > 0.0 && c.bc[PDG_BC_CL_I] > 0.0 &&
          c.bc[PDG_BC_CL_O] > 0.0 && c.bc[PDG_BC_NA_I0] > 0.0 && c.bc[PDG_BC_K_I0] > 0.0 &&
          c.bc[PDG_BC_NA_O0] > 0.0))
      throw ConfigError("barreto-cressman: tau, RTF and the reference concentrations must be positive");
  } else if (c.ionic_model != PDG_IONIC_NONE) {
    throw ConfigError("unknown ionic model");
  }
  if (c.world < 1 || c.rank < 0 || c.rank >= c.world) throw ConfigError("invalid rank/world");
}

// Device factorisation plan of one unit (see Problem::FactorSn): tasks
// [base, base + nsn) were just packed from the symbolic factor F.
static void add_factor_plan(Problem& pr, const SupernodalFactor& F, const std::vector<std::vector<int>>& upd,
                            int base, int cell0) {
  const int bs = F.bs;
  for (int s = 0; s < static_cast<int>(F.sn.size()); ++s) {
    const Supernode& S = F.sn[s];
    const TaskDesc& t = pr.tasks[base + s];
    Problem::FactorSn f{};
    f.p_off = pr.fp_len;
    f.cell0 = cell0;
    f.ucells = F.m;
    f.s0 = S.s0;
    f.s1 = S.s1;
    f.w = t.w;
    f.H = t.w + t.nr;
    pr.fp_len += static_cast<std::int64_t>(f.H) * f.w;
    pr.fp_len += pr.fp_len & 1;
    f.rows_off = static_cast<int>(pr.frows.size());
    f.nrows = static_cast<int>(S.rows.size());
    pr.frows.insert(pr.frows.end(), S.rows.begin(), S.rows.end());
    f.upd_off = static_cast<int>(pr.fupd.size());
    f.nupd = static_cast<int>(upd[s].size());
    f.height = t.height;
    for (int d : upd[s]) {
      const Supernode& D = F.sn[d];
      Problem::FactorUpd u{};
      u.d = base + d;
      u.a = static_cast<int>(std::lower_bound(D.rows.begin(), D.rows.end(), S.s0) - D.rows.begin());
      u.ce = static_cast<int>(std::lower_bound(D.rows.begin(), D.rows.end(), S.s1) - D.rows.begin());
      u.nrd = static_cast<int>(D.rows.size());
      u.map_off = static_cast<std::int64_t>(pr.fmap.size());
      for (int k = u.a; k < u.nrd; ++k) {
        const int q = D.rows[k];
        int rc;
        if (q < S.s1) {
          rc = q - S.s0;
        } else {
          const auto it = std::lower_bound(S.rows.begin(), S.rows.end(), q);
          if (it == S.rows.end() || *it != q) throw SolverError("factor plan: descendant row outside the supernode");
          rc = (S.s1 - S.s0) + static_cast<int>(it - S.rows.begin());
        }
        pr.fmap.push_back(rc);
      }
      pr.fupd.push_back(u);
    }
    pr.fsn.push_back(f);
  }
  (void)bs;
}


struct Placement {
  std::vector<std::vector<int>> units;  // reference cells per unit (subdomain)
  std::vector<int> unit_order;          // placement order of the units
  std::vector<int> unit_rank, unit_start;
  std::vector<NdTree> nd;               // per unit: supernode tree of its local factor
  std::vector<std::vector<int>> unit_cells;  // per unit: cells in internal order
  std::vector<int> my_units;            // this rank's units in placement order
  bool multi_sub = false;
};

// Internal order (problem.hpp): units (subdomains) in `unit_order`, split over
// ranks as contiguous cell-balanced ranges; inside each multi-cell unit a
// fill-reducing order of its exact local factor (host/ordering.hpp). `pos`
// (cell centroids) enables geometric nested dissection; without it (an
// operator given by the caller) the order is graph-only minimum degree.
static void place_units(Problem& pr, Placement& pl, const std::vector<std::vector<int>>& nbr,
                        const std::vector<Pt>* pos) {
  const pdg_config& cfg = pr.cfg;
  const int N = static_cast<int>(nbr.size());
  const int b = pr.b;
  const int n_units = static_cast<int>(pl.units.size());
  const auto& units = pl.units;
  const auto& unit_order = pl.unit_order;
  const bool multi_sub = pl.multi_sub;
  // contiguous split of the ordered units over ranks, balanced by cells
  pl.unit_rank.assign(n_units, 0);
  auto& unit_rank = pl.unit_rank;
  pr.rank_cell_start.assign(cfg.world + 1, 0);
  {
    std::int64_t acc = 0;
    int r = 0;
    for (int k = 0; k < n_units; ++k) {
      const int u = unit_order[k];
      while (r < cfg.world - 1 && acc >= static_cast<std::int64_t>(N) * (r + 1) / cfg.world) ++r;
      unit_rank[u] = r;
      acc += static_cast<std::int64_t>(units[u].size());
    }
  }
  // ND inside each multi-cell subdomain
  // Nested-dissection shape. Merging two separator levels per supernode
  // halves the elimination-tree depth (the sweep's critical path) at ~20%
  // more panel bytes; it pays while the sweep is latency bound (config2,
  // config3 p=3: +2-9%) and costs once it streams with wide blocks (config3
  // p=4: -9%, config4: -11%, config5 p=4: -35%). With p <= 2 the unmerged
  // tree of small blocks is latency bound even on the 1M-cell mesh (config5
  // p=2: -9%). Leaf size: dense leaves of ~64 dofs.
  // PDG_ND_MERGE / PDG_ND_LEAF override.
  const bool big = static_cast<std::int64_t>(N) * b > 800000 && b >= 10;
  int nd_merge = big ? 1 : 2;
  if (const char* env = std::getenv("PDG_ND_MERGE")) nd_merge = std::max(1, std::atoi(env));
  int leaf = std::clamp(64 / b, 4, 16);  // config4: 6-cell leaves +3.8% over 4
  if (const char* env = std::getenv("PDG_ND_LEAF")) leaf = std::max(1, std::atoi(env));
  // Ordering family (profiles/r02c-r02e, B200). Minimum degree with relaxed
  // supernodes (host/ordering.hpp: <= 8 cells merged while the merge adds
  // < 50% explicit zeros) stores fewer panel bytes than the ND above on the
  // large meshes and its supernodes are as wide: config4 6.4 vs 7.5 ms per
  // sweep, config5 p=2 2.8 vs 3.2 ms, p=4 12.2 vs 13.3 ms. Below ~2M dofs the
  // sweep is latency bound and the shallower ND tree wins (config2 0.10 vs
  // 0.22 ms, config3 p=3 0.43 vs 0.56 ms). Without cell positions (an
  // operator handed over by the caller) the order is graph-only MD.
  // PDG_ORDER=nd|md and PDG_MD_RELAX override.
  // The size that matters is what one rank holds (config 4 strong-scaled over 8
  // GPUs is a 1.3M-dof problem per rank); every rank orders every subdomain,
  // so the choice depends on (N, b, world) only.
  const std::int64_t dofs_per_rank = static_cast<std::int64_t>(N) * b / std::max(1, cfg.world);
  const bool md_default = dofs_per_rank >= 2000000;
  const char* ord_env = std::getenv("PDG_ORDER");
  const bool md_order = !pos || (ord_env ? std::string(ord_env) == "md" : md_default);
  // With the bottom levels solved in level chunks (host/pack.cpp) the small
  // supernodes cost no per-unit round trips, so no amalgamation: fundamental
  // supernodes store no explicit zeros (config 4: 26.6 GB of panels instead
  // of 35.0 GB; sweep 6.17 -> 5.86 ms, profiles/r02u). Small blocks (b < 10)
  // merge up to 2 cells (config 5 p=2: 2.22 ms vs 2.48 ms fundamental).
  const bool bottom_on = md_order && bottom_level_bytes(dofs_per_rank, b) > 0;
  const int md_relax =
      std::getenv("PDG_MD_RELAX") ? std::max(1, std::atoi(std::getenv("PDG_MD_RELAX"))) : bottom_on ? (b >= 10 ? 1 : 2) : 8;
  pl.nd.assign(n_units, NdTree{});
  auto& nd = pl.nd;
  pl.unit_cells.assign(n_units, {});
  auto& unit_cells = pl.unit_cells;  // cells in internal order
  std::vector<std::int64_t> unit_fill(n_units, 0);
  parallel_for(n_units, [&](int u) {
    const auto& cells = units[u];
    const int m = static_cast<int>(cells.size());
    if (!multi_sub) {
      unit_cells[u] = cells;
      return;
    }
    std::map<int, int> loc;
    for (int i = 0; i < m; ++i) loc[cells[i]] = i;
    std::vector<int> ap{0}, aj;
    std::vector<Pt> lpos(m);
    for (int i = 0; i < m; ++i) {
      for (int nb : nbr[cells[i]]) {
        auto it = loc.find(nb);
        if (it != loc.end()) aj.push_back(it->second);
      }
      ap.push_back(static_cast<int>(aj.size()));
      if (pos) lpos[i] = (*pos)[cells[i]];
    }
    nd[u] = md_order ? md_supernodes(m, ap, aj, md_relax) : nested_dissection(m, ap, aj, lpos, leaf, nd_merge);
    unit_fill[u] = structural_fill(m, ap, aj, nd[u].order).scalar(b);
    unit_cells[u].resize(m);
    for (int i = 0; i < m; ++i) unit_cells[u][i] = cells[nd[u].order[i]];
  });
  pr.perm.clear();
  pl.unit_start.assign(n_units, 0);
  auto& unit_start = pl.unit_start;
  for (int r = 0; r < cfg.world; ++r) {
    pr.rank_cell_start[r] = static_cast<int>(pr.perm.size());
    for (int k = 0; k < n_units; ++k) {
      const int u = unit_order[k];
      if (unit_rank[u] != r) continue;
      unit_start[u] = static_cast<int>(pr.perm.size());
      pr.perm.insert(pr.perm.end(), unit_cells[u].begin(), unit_cells[u].end());
    }
  }
  pr.rank_cell_start[cfg.world] = N;
  for (int u = 0; u < n_units; ++u)
    if (unit_rank[u] == cfg.rank)
      pr.l_struct += multi_sub ? unit_fill[u] : static_cast<std::int64_t>(b) * (b + 1) / 2 * units[u].size();
  pr.iperm.assign(N, -1);
  for (int i = 0; i < N; ++i) pr.iperm[pr.perm[i]] = i;
  pr.cell_begin = pr.rank_cell_start[cfg.rank];
  pr.cell_end = pr.rank_cell_start[cfg.rank + 1];
  for (int k = 0; k < n_units; ++k)
    if (unit_rank[unit_order[k]] == cfg.rank) pl.my_units.push_back(unit_order[k]);
}


// Exact local factors of this rank's subdomains (schwarz.cpp:99-136): the
// symbolic plan (device factorisation) or the host supernodal Cholesky, packed
// into sweep tasks (host/pack.cpp). pr.K must be in internal order.
static void factor_units(Problem& pr, const Placement& pl) {
  const pdg_config& cfg = pr.cfg;
  const int b = pr.b, b2 = b * b;
  const int nloc = pr.cell_end - pr.cell_begin;
  const bool multi_sub = pl.multi_sub;
  const auto& unit_cells = pl.unit_cells;
  const auto& unit_start = pl.unit_start;
  const auto& nd = pl.nd;
  // ---- Schwarz local factors (schwarz.cpp:99-136) ----
  struct UnitFactor {
    int unit;
    SupernodalFactor F;
    std::vector<std::vector<int>> upd;  // device factorisation: left-looking updaters
  };
  // one rank, multi-cell subdomains: the GPU computes the numeric factor
  // (cuda/factor.cu) from a host symbolic plan; PDG_HOST_FACTOR=1 keeps the
  // host supernodal Cholesky
  pr.device_factor = multi_sub && cfg.world == 1 && pr.has_precond &&
                     !(std::getenv("PDG_HOST_FACTOR") && std::getenv("PDG_HOST_FACTOR")[0] == '1');
  const std::vector<int>& my_units = pl.my_units;
  std::vector<UnitFactor> factors;
  pr.in_ptr = {0};
  bool packed = false;
  if (pr.has_precond) {
    if (multi_sub) {
      // factor a batch of subdomains in parallel, pack it (in subdomain
      // order) and free it: only one batch of unpacked factors is alive, so
      // the host peak is the packed panels plus a batch (config 4: ~40 GB of
      // panels instead of twice that)
      const int n_my = static_cast<int>(my_units.size());
      const int batch = std::max(1, 4 * setup_threads());
      for (int b0 = 0; b0 < n_my; b0 += batch) {
      const int b1 = std::min(n_my, b0 + batch);
      factors.assign(b1 - b0, UnitFactor{});
      parallel_for(b1 - b0, [&](int kb) {
        const int k = kb;
        const int u = my_units[b0 + kb];
        const int m = static_cast<int>(unit_cells[u].size());
        const int s0 = unit_start[u];
        BlockMatrix Bm;
        Bm.m = m;
        Bm.bs = b;
        Bm.ptr.assign(m + 1, 0);
        for (int i = 0; i < m; ++i) {
          const int li = s0 + i - pr.cell_begin;
          for (int kk = pr.K.ptr[li]; kk < pr.K.ptr[li + 1]; ++kk) {
            const int j = pr.K.col[kk];
            if (j < s0 || j >= s0 + m) continue;
            Bm.col.push_back(j - s0);
            if (!pr.device_factor)
              Bm.val.insert(Bm.val.end(), pr.K.val.begin() + static_cast<std::size_t>(kk) * b2,
                            pr.K.val.begin() + static_cast<std::size_t>(kk + 1) * b2);
          }
          Bm.ptr[i + 1] = static_cast<int>(Bm.col.size());
        }
        NdTree t;
        t.order.resize(m);
        std::iota(t.order.begin(), t.order.end(), 0);
        t.sn_start = nd[u].sn_start;
        t.parent = nd[u].parent;
        factors[k].unit = u;
        if (pr.device_factor) {
          factors[k].F = symbolic_factor(Bm, t, factors[k].upd);
          return;
        }
        try {
          factors[k].F = supernodal_cholesky(Bm, t);
        } catch (const SolverError&) {
          throw SolverError("schwarz: subdomain " + std::to_string(u) +
                            " factorization failed (not positive definite)");
        }
      });
      for (const UnitFactor& uf : factors) {
        const int base = static_cast<int>(pr.tasks.size());
        pack_unit_tasks(pr, uf.F, 0, static_cast<std::int64_t>(unit_start[uf.unit] - pr.cell_begin) * b);
        if (pr.device_factor) add_factor_plan(pr, uf.F, uf.upd, base, unit_start[uf.unit] - pr.cell_begin);
      }
      factors.clear();
      }
      packed = true;
    } else {
      // one element per subdomain: dense b x b Cholesky (schwarz.cpp:103-112)
      factors.resize(nloc);
      parallel_for(nloc, [&](int i) {
        BlockMatrix Bm;
        Bm.m = 1;
        Bm.bs = b;
        Bm.ptr = {0, 1};
        Bm.col = {0};
        const int k = pr.K.ptr[i] + static_cast<int>(std::lower_bound(pr.K.col.begin() + pr.K.ptr[i],
                                                                 pr.K.col.begin() + pr.K.ptr[i + 1],
                                                                 pr.cell_begin + i) -
                                                  (pr.K.col.begin() + pr.K.ptr[i]));
        Bm.val.assign(pr.K.val.begin() + static_cast<std::size_t>(k) * b2,
                      pr.K.val.begin() + static_cast<std::size_t>(k + 1) * b2);
        NdTree t;
        t.order = {0};
        t.sn_start = {0, 1};
        t.parent = {-1};
        factors[i].unit = pr.sub.owner[pr.perm[pr.cell_begin + i]];
        try {
          factors[i].F = supernodal_cholesky(Bm, t);
        } catch (const SolverError&) {
          throw SolverError("schwarz: subdomain " + std::to_string(factors[i].unit) +
                            " block is not positive definite");
        }
      }, 256);
    }
  }
  // pack fine tasks (host/pack.cpp); the multi-cell subdomains were packed
  // batch by batch above
  if (!packed)
    for (const UnitFactor& uf : factors)
      pack_unit_tasks(pr, uf.F, 0, static_cast<std::int64_t>(&uf - factors.data()) * b);
  pr.n_fine_tasks = static_cast<int>(pr.tasks.size());
  factors.clear();
  finish_bottom_levels(pr);
  if (std::getenv("PDG_SETUP_TIMES")) {
    std::int64_t bt = 0, bb = 0;
    for (const LevelChunk& c : pr.chunks) {
      bb += c.bytes;
      if (c.dir == 0) bt += c.n_task;
    }
    int small16 = 0, small48 = 0, reg = 0;
    for (const TaskDesc& t : pr.tasks) {
      if (t.bottom >= 0) continue;
      ++reg;
      const std::int64_t fb = 8LL * t.w * (t.w + t.nr);
      small16 += fb < 16384;
      small48 += fb < 49152;
    }
    std::fprintf(stderr,
                 "[pdg] sweep tasks %zu: %d scheduled one by one (%d under 16 KB, %d under 48 KB), %lld in %d bottom "
                 "levels, %zu level chunks (%.2f GB of %.2f GB panels)\n",
                 pr.tasks.size(), reg, small16, small48, static_cast<long long>(bt), pr.n_bottom_levels,
                 pr.chunks.size(), bb / 1e9, 8.0 * (pr.fmat_len + pr.hmat_len) / 1e9);
  }
}


// Coarse space from E (one b x bq block per cell, schwarz.cpp:49-75): coarse
// internal order over the agglomerate graph (geometric ND with centres `apos`,
// else minimum degree), per local cell E block and coarse node, coarse node ->
// cells lists, and this rank's partial K0 = E^T K E (schwarz.cpp:141) in the
// coarse internal order. Eall[e_slot[g]] = E block of global internal cell g
// (local cells and the halo cells their rows touch).
static void coarse_space(Problem& pr, std::vector<std::vector<int>>& anbr, const std::vector<Pt>* apos,
                         const std::vector<double>& Eall, const std::vector<int>& e_slot) {
  const int na = pr.coarse.count;
  const int b = pr.b, b2 = b * b, bq = pr.bq;
  const int nloc = pr.cell_end - pr.cell_begin;
  std::vector<int> ap{0}, aj;
  for (int a = 0; a < na; ++a) {
    auto& v = anbr[a];
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
    aj.insert(aj.end(), v.begin(), v.end());
    ap.push_back(static_cast<int>(aj.size()));
  }
  const NdTree cnd = apos ? nested_dissection(na, ap, aj, *apos, std::clamp(64 / pr.bq, 4, 16))
                          : md_supernodes(na, ap, aj, 8);
  pr.l0_struct = structural_fill(na, ap, aj, cnd.order).scalar(pr.bq);
  pr.n_agg = na;
  pr.agg_order = cnd.order;  // position -> label
  pr.coarse_nd = cnd;
  std::vector<int> apos_of(na);
  for (int i = 0; i < na; ++i) apos_of[cnd.order[i]] = i;
  const bool values = !Eall.empty();  // false: E and K0 are formed on the device
  if (values) pr.E.resize(static_cast<std::size_t>(nloc) * b * bq);
  pr.cell_agg.resize(nloc);
  for (int i = 0; i < nloc; ++i) {
    const int g = pr.cell_begin + i;
    if (values)
      std::copy(Eall.begin() + static_cast<std::size_t>(e_slot[g]) * b * bq,
                Eall.begin() + static_cast<std::size_t>(e_slot[g] + 1) * b * bq,
                pr.E.begin() + static_cast<std::size_t>(i) * b * bq);
    pr.cell_agg[i] = apos_of[pr.coarse.owner[pr.perm[g]]];
  }
  // agglomerate -> local cells
  pr.agg_cell_ptr.assign(na + 1, 0);
  for (int i = 0; i < nloc; ++i) ++pr.agg_cell_ptr[pr.cell_agg[i] + 1];
  for (int a = 0; a < na; ++a) pr.agg_cell_ptr[a + 1] += pr.agg_cell_ptr[a];
  pr.agg_cells.resize(nloc);
  {
    std::vector<int> fill(pr.agg_cell_ptr.begin(), pr.agg_cell_ptr.end() - 1);
    for (int i = 0; i < nloc; ++i) pr.agg_cells[fill[pr.cell_agg[i]]++] = i;
  }
  // K0 partial over local rows: K0[a,a'] += E_i^T K_ij E_j, coarse internal order
  Bsr& K0 = pr.K0;
  K0.rows = na;
  K0.b = bq;
  K0.ptr.assign(na + 1, 0);
  for (int i = 0; i < na; ++i) {
    const int a = cnd.order[i];
    std::vector<int> cols{i};
    for (int nb : anbr[a]) cols.push_back(apos_of[nb]);
    std::sort(cols.begin(), cols.end());
    K0.col.insert(K0.col.end(), cols.begin(), cols.end());
    K0.ptr[i + 1] = static_cast<int>(K0.col.size());
  }
  const int bq2 = bq * bq;
  K0.val.assign(static_cast<std::size_t>(K0.col.size()) * bq2, 0.0);
  if (!values) return;
  // one coarse row per task: its cells in increasing local index, which is
  // the order a serial sweep over all local rows would add them (same bits)
  parallel_for(na, [&](int ai) {
  std::vector<double> KE(static_cast<std::size_t>(b) * bq);
  for (int ci = pr.agg_cell_ptr[ai]; ci < pr.agg_cell_ptr[ai + 1]; ++ci) {
    const int i = pr.agg_cells[ci];
    const double* Ei = &pr.E[static_cast<std::size_t>(i) * b * bq];
    for (int k = pr.K.ptr[i]; k < pr.K.ptr[i + 1]; ++k) {
      const int j = pr.K.col[k];
      const int aj2 = apos_of[pr.coarse.owner[pr.perm[j]]];
      const double* Ej = &Eall[static_cast<std::size_t>(e_slot[j]) * b * bq];
      const double* Kb = &pr.K.val[static_cast<std::size_t>(k) * b2];
      // KE = K_ij E_j  (b x bq)
      for (int m = 0; m < bq; ++m)
        for (int r = 0; r < b; ++r) {
          double s = 0.0;
          for (int c = 0; c < b; ++c) s += Kb[c * b + r] * Ej[m * b + c];
          KE[m * b + r] = s;
        }
      const int* c0 = K0.col.data() + K0.ptr[ai];
      const int* c1 = K0.col.data() + K0.ptr[ai + 1];
      const int blk = static_cast<int>(std::lower_bound(c0, c1, aj2) - K0.col.data());
      double* out = &K0.val[static_cast<std::size_t>(blk) * bq2];
      for (int m2 = 0; m2 < bq; ++m2)
        for (int m1 = 0; m1 < bq; ++m1) {
          double s = 0.0;
          for (int r = 0; r < b; ++r) s += Ei[m1 * b + r] * KE[m2 * b + r];
          out[m2 * bq + m1] += s;
        }
    }
  }
  }, 1);
}


// Bounding box of every agglomerate: union of its cells' boxes (schwarz.cpp:26-36).
static std::vector<Box> agglomerate_boxes(const Mesh& mesh, const std::vector<int>& owner, int na) {
  std::vector<Box> abox(na);
  std::vector<bool> seen(na, false);
  for (int c = 0; c < mesh.n_cells(); ++c) {
    const int a = owner[c];
    const std::vector<Pt> pts = mesh.cell_points(c);
    const Box cb = bbox_of(pts.data(), static_cast<int>(pts.size()));
    if (!seen[a]) {
      abox[a] = cb;
      seen[a] = true;
    } else {
      abox[a].xmin = std::min(abox[a].xmin, cb.xmin);
      abox[a].xmax = std::max(abox[a].xmax, cb.xmax);
      abox[a].ymin = std::min(abox[a].ymin, cb.ymin);
      abox[a].ymax = std::max(abox[a].ymax, cb.ymax);
    }
  }
  return abox;
}

// E_K = M_K^{-1} int_K phi psi^T for the listed cells (schwarz.cpp:49-75):
// fine modes on the cell's bbox, degree-q coarse modes on its agglomerate's
// bbox, quadrature order 2p+2 (exact). One b x bq column-major block per cell.
static std::vector<double> coarse_embedding_cells(const Mesh& mesh, int p, const std::vector<int>& owner,
                                                  const std::vector<Box>& abox, int q, const std::vector<int>& cells) {
  const int b = n_modes(p), bq = n_modes(q), order = 2 * p + 2;
  std::vector<double> Eall(cells.size() * static_cast<std::size_t>(b) * bq);
  parallel_for(static_cast<int>(cells.size()), [&](int k) {
    const int c = cells[k];
    const int a = owner[c];
    const std::vector<Pt> poly = mesh.cell_points(c);
    const Box cb = bbox_of(poly.data(), static_cast<int>(poly.size()));
    const Rule rule = polygon_rule(poly, order);
    std::vector<double> mass(static_cast<std::size_t>(b) * b, 0.0), rhs(static_cast<std::size_t>(b) * bq, 0.0);
    std::vector<double> fv(b), cv(bq);
    for (std::size_t qp = 0; qp < rule.size(); ++qp) {
      const double w = rule.w[qp];
      basis_at(cb, p, rule.pts[qp], fv.data());
      basis_at(abox[a], q, rule.pts[qp], cv.data());
      for (int jj = 0; jj < b; ++jj)
        for (int ii = 0; ii < b; ++ii) mass[jj * b + ii] += w * fv[ii] * fv[jj];
      for (int m = 0; m < bq; ++m)
        for (int ii = 0; ii < b; ++ii) rhs[m * b + ii] += w * fv[ii] * cv[m];
    }
    spd_solve(b, bq, mass.data(), rhs.data());
    std::copy(rhs.begin(), rhs.end(), Eall.begin() + static_cast<std::size_t>(k) * b * bq);
  }, 64);
  return Eall;
}

std::vector<double> coarse_embedding(const Mesh& mesh, int p, const std::vector<int>& owner, int count, int q) {
  if (q < 1 || q > p) throw ConfigError("build_coarse_embedding: q must lie in [1, p]");
  if (static_cast<int>(owner.size()) != mesh.n_cells()) throw ConfigError("build_coarse_embedding: owner size");
  for (int o : owner)
    if (o < 0 || o >= count) throw ConfigError("build_coarse_embedding: owner out of range");
  std::vector<int> cells(mesh.n_cells());
  std::iota(cells.begin(), cells.end(), 0);
  return coarse_embedding_cells(mesh, p, owner, agglomerate_boxes(mesh, owner, count), q, cells);
}

std::unique_ptr<Problem> build_problem(const pdg_config& cfg, bool device) {
  validate_config(cfg);
  auto P = std::make_unique<Problem>();
  Problem& pr = *P;
  pr.cfg = cfg;
  // PDG_SETUP_TIMES=1: wall time of each setup phase on stderr
  static const bool times = std::getenv("PDG_SETUP_TIMES") && std::getenv("PDG_SETUP_TIMES")[0] == '1';
  auto t_last = std::chrono::steady_clock::now();
  auto phase = [&](const char* name) {
    if (!times) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "setup %-14s %8.2f s\n", name, std::chrono::duration<double>(now - t_last).count());
    t_last = now;
  };
  const Box dom{cfg.domain[0], cfg.domain[1], cfg.domain[2], cfg.domain[3]};
  {
    Mesh m = generate_mesh(cfg.mesh_cells, dom, cfg.mesh_seed, cfg.mesh_lloyd);
    pr.mesh = (cfg.split_y > dom.ymin && cfg.split_y < dom.ymax) ? assign_regions(m, cfg.split_y) : std::move(m);
  }
  phase("mesh");
  const Mesh& mesh = pr.mesh;
  const int N = mesh.n_cells();
  pr.n_cells_global = N;
  pr.p = cfg.degree;
  pr.b = n_modes(pr.p);
  pr.q = cfg.q > 0 ? cfg.q : cfg.degree;
  pr.bq = n_modes(pr.q);
  pr.has_precond = cfg.precond_kind != PDG_PRECOND_NONE;
  pr.two_level = cfg.precond_kind == PDG_PRECOND_TWO_LEVEL;
  // one rank on the device: M, A, K, M^-1, U0/Y0, E and K0 are assembled by
  // cuda/assemble.cu (same bits) when no host step needs K's values, i.e.
  // the local factors are computed on the device too (multi-cell subdomains,
  // factor_units) or there is no preconditioner; PDG_HOST_ASSEMBLY=1 keeps
  // the host assembly
  auto env_on = [](const char* k) { return std::getenv(k) && std::getenv(k)[0] == '1'; };
  pr.device_assembly = device && cfg.world == 1 && !env_on("PDG_HOST_ASSEMBLY") &&
                       (!pr.has_precond || (cfg.subdomains > 0 && !env_on("PDG_HOST_FACTOR")));
  const bool dev_asm = pr.device_assembly;
  double u_model_rest = 0.0, y_rest[4] = {0.0, 0.0, 0.0, 0.0};
  pr.n_comp = ionic_rest(cfg, u_model_rest, y_rest);
  const int b = pr.b, b2 = b * b;

  // ---- partitions (timestepper.cpp:92-102 + ext) ----
  pr.sub = cfg.subdomains > 0 ? agglomerate(mesh, cfg.subdomains) : identity_partition(mesh);
  if (pr.two_level) {
    if (cfg.coarse_count == -1 || (cfg.coarse_count > 0 && cfg.coarse_count == cfg.subdomains))
      pr.coarse = pr.sub;
    else if (cfg.coarse_count > 0)
      pr.coarse = agglomerate(mesh, cfg.coarse_count);
    else {
      const int levels = static_cast<int>(std::lround(std::log2(static_cast<double>(cfg.h_ratio))));
      pr.coarse = agglomerate_hierarchy(mesh, levels).back();
    }
  }

  phase("partitions");
  // ---- adjacency (reference cell ids) ----
  std::vector<std::vector<int>> nbr(N);
  for (const Face& f : mesh.interior_faces()) {
    nbr[f.cell_in].push_back(f.cell_out);
    nbr[f.cell_out].push_back(f.cell_in);
  }
  for (auto& v : nbr) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }

  // ---- placement units and internal order ----
  std::vector<std::vector<int>> units_in;
  const bool multi_sub = cfg.subdomains > 0;
  if (multi_sub) {
    units_in = pr.sub.members();
  } else if (pr.two_level) {
    units_in = pr.coarse.members();
  } else {
    std::vector<int> cells(N);
    std::iota(cells.begin(), cells.end(), 0);
    std::vector<std::uint32_t> code(N);
    for (int c = 0; c < N; ++c) code[c] = morton(mesh.centroid(c).x, mesh.centroid(c).y, dom);
    std::stable_sort(cells.begin(), cells.end(), [&](int a, int b2_) { return code[a] < code[b2_]; });
    for (int s = 0; s < N; s += 256)
      units_in.emplace_back(cells.begin() + s, cells.begin() + std::min(N, s + 256));
  }
  std::vector<int> unit_order_in(units_in.size());
  std::iota(unit_order_in.begin(), unit_order_in.end(), 0);
  {
    const int n_units = static_cast<int>(units_in.size());
    const auto& units = units_in;
    std::vector<std::uint32_t> code(n_units);
    for (int u = 0; u < n_units; ++u) {
      double sx = 0, sy = 0;
      for (int c : units[u]) {
        sx += mesh.centroid(c).x;
        sy += mesh.centroid(c).y;
      }
      code[u] = morton(sx / units[u].size(), sy / units[u].size(), dom);
    }
    std::stable_sort(unit_order_in.begin(), unit_order_in.end(), [&](int a, int c) { return code[a] < code[c]; });
  }
  Placement pl;
  pl.units = std::move(units_in);
  pl.unit_order = std::move(unit_order_in);
  pl.multi_sub = multi_sub;
  {
    std::vector<Pt> cpos(N);
    for (int c = 0; c < N; ++c) cpos[c] = mesh.centroid(c);
    place_units(pr, pl, nbr, &cpos);
  }
  pr.cell_begin = pr.rank_cell_start[cfg.rank];
  pr.cell_end = pr.rank_cell_start[cfg.rank + 1];
  const int nloc = pr.cell_end - pr.cell_begin;

  phase("ordering");
  // ---- assembly of local rows (assembly.cpp:89-183) ----
  pr.keep_matrices = static_cast<std::int64_t>(N) * b <= 2000000;
  Bsr& A = pr.A;
  A.rows = nloc;
  A.b = b;
  A.ptr.assign(nloc + 1, 0);
  for (int i = 0; i < nloc; ++i) A.ptr[i + 1] = A.ptr[i] + 1 + static_cast<int>(nbr[pr.perm[pr.cell_begin + i]].size());
  A.col.resize(A.ptr[nloc]);
  for (int i = 0; i < nloc; ++i) {
    const int c = pr.perm[pr.cell_begin + i];
    std::vector<int> cols{pr.cell_begin + i};
    for (int nb : nbr[c]) cols.push_back(pr.iperm[nb]);
    std::sort(cols.begin(), cols.end());
    std::copy(cols.begin(), cols.end(), A.col.begin() + A.ptr[i]);
  }
  if (!dev_asm) A.val.assign(static_cast<std::size_t>(A.ptr[nloc]) * b2, 0.0);
  auto find_block = [&](int i_loc, int j_glob) {
    const int* b0 = A.col.data() + A.ptr[i_loc];
    const int* e0 = A.col.data() + A.ptr[i_loc + 1];
    const int* it = std::lower_bound(b0, e0, j_glob);
    return static_cast<int>(it - A.col.data());
  };
  // conductivity per cell
  std::vector<Tensor> sig(N);
  std::vector<double> sig_norm(N);
  {
    std::vector<double> theta;
    if (cfg.fiber_random) {
      std::mt19937_64 rng(cfg.fiber_seed);
      theta.resize(N);
      for (int c = 0; c < N; ++c) theta[c] = M_PI * (static_cast<double>(rng() >> 11) * 0x1.0p-53);
    }
    for (int c = 0; c < N; ++c) {
      const bool grey = mesh.region(c) == kGrey;
      const double sl = grey ? cfg.sigma_grey_l : cfg.sigma_white_l;
      const double sn = grey ? cfg.sigma_grey_n : cfg.sigma_white_n;
      double fx = grey ? cfg.fiber_grey[0] : cfg.fiber_white[0];
      double fy = grey ? cfg.fiber_grey[1] : cfg.fiber_white[1];
      if (cfg.fiber_random) {
        fx = std::cos(theta[c]);
        fy = std::sin(theta[c]);
      }
      sig[c] = make_tensor(sl, sn, fx, fy);
      sig_norm[c] = std::max(sl, sn);
    }
  }
  if (dev_asm) {
    pr.sigma.resize(static_cast<std::size_t>(N) * 4);
    for (int g = 0; g < N; ++g) {
      const Tensor& t = sig[pr.perm[g]];
      pr.sigma[4 * g] = t.t00;
      pr.sigma[4 * g + 1] = t.t01;
      pr.sigma[4 * g + 2] = t.t10;
      pr.sigma[4 * g + 3] = t.t11;
    }
  }
  const int order = 2 * pr.p + 2;
  if (!dev_asm) {
    pr.M.assign(static_cast<std::size_t>(nloc) * b2, 0.0);
    pr.Minv.assign(static_cast<std::size_t>(nloc) * b2, 0.0);
    pr.U0.assign(static_cast<std::size_t>(nloc) * b, 0.0);
    pr.Y0.assign(static_cast<std::size_t>(nloc) * b * pr.n_comp, 0.0);
  }
  for (int l = 0; l < pr.n_comp; ++l) pr.y_rest[l] = y_rest[l];
  pr.bbox.resize(static_cast<std::size_t>(nloc) * 4);
  pr.tri_ptr.assign(nloc + 1, 0);
  std::vector<std::vector<double>> tri_loc(nloc);
  parallel_for(nloc, [&](int i) {
    const int c = pr.perm[pr.cell_begin + i];
    const std::vector<Pt> poly = mesh.cell_points(c);
    const Box bx = bbox_of(poly.data(), static_cast<int>(poly.size()));
    pr.bbox[4 * i] = bx.xmin;
    pr.bbox[4 * i + 1] = bx.ymin;
    pr.bbox[4 * i + 2] = bx.xmax;
    pr.bbox[4 * i + 3] = bx.ymax;
    std::vector<std::array<Pt, 3>> tris;
    cell_triangles(poly, tris);
    for (const auto& t : tris)
      for (const Pt& v : t) {
        tri_loc[i].push_back(v.x);
        tri_loc[i].push_back(v.y);
      }
    if (dev_asm) return;  // the quadrature runs on the device (cuda/assemble.cu)
    const Rule rule = polygon_rule(poly, order);
    const int nq = static_cast<int>(rule.size());
    std::vector<double> val(static_cast<std::size_t>(nq) * b), gx(val.size()), gy(val.size());
    for (int k = 0; k < nq; ++k) basis_at(bx, pr.p, rule.pts[k], &val[k * b], &gx[k * b], &gy[k * b]);
    std::vector<double> mloc(b2, 0.0), aloc(b2, 0.0);
    const Tensor& s = sig[c];
    for (int k = 0; k < nq; ++k) {
      const double w = rule.w[k];
      const double* v = &val[k * b];
      for (int ii = 0; ii < b; ++ii)
        for (int jj = ii; jj < b; ++jj) mloc[jj * b + ii] += w * v[ii] * v[jj];
    }
    for (int k = 0; k < nq; ++k) {
      const double w = rule.w[k];
      const double* X = &gx[k * b];
      const double* Y = &gy[k * b];
      for (int jj = 0; jj < b; ++jj) {
        const double sx = s.t00 * X[jj] + s.t01 * Y[jj];
        const double sy = s.t10 * X[jj] + s.t11 * Y[jj];
        for (int ii = 0; ii <= jj; ++ii) aloc[jj * b + ii] += w * (X[ii] * sx + Y[ii] * sy);
      }
    }
    double* Mb = &pr.M[static_cast<std::size_t>(i) * b2];
    double* Ab = &A.val[static_cast<std::size_t>(find_block(i, pr.cell_begin + i)) * b2];
    for (int jj = 0; jj < b; ++jj)
      for (int ii = 0; ii <= jj; ++ii) {
        Mb[jj * b + ii] = Mb[ii * b + jj] = mloc[jj * b + ii];
        Ab[jj * b + ii] = Ab[ii * b + jj] = aloc[jj * b + ii];
      }
    spd_inverse(b, Mb, &pr.Minv[static_cast<std::size_t>(i) * b2]);
    // initial data: l2 projection (assembly.cpp:228-242), Y at the model rest state (0 for FHN)
    std::vector<double> rhs(b, 0.0);
    for (int k = 0; k < nq; ++k) {
      const double g = init_value(cfg, rule.pts[k]);
      for (int ii = 0; ii < b; ++ii) rhs[ii] += rule.w[k] * g * val[k * b + ii];
    }
    const double* Mi = &pr.Minv[static_cast<std::size_t>(i) * b2];
    for (int ii = 0; ii < b; ++ii) {
      double acc = 0.0;
      for (int jj = 0; jj < b; ++jj) acc += Mi[jj * b + ii] * rhs[jj];
      pr.U0[static_cast<std::size_t>(i) * b + ii] = acc;
    }
    // Y: l2 projection of the model's constant resting state (timestepper.cpp:116-123)
    for (int l = 0; l < pr.n_comp; ++l) {
      if (y_rest[l] == 0.0) continue;
      std::vector<double> ry(b, 0.0);
      for (int k = 0; k < nq; ++k)
        for (int ii = 0; ii < b; ++ii) ry[ii] += rule.w[k] * y_rest[l] * val[k * b + ii];
      for (int ii = 0; ii < b; ++ii) {
        double acc = 0.0;
        for (int jj = 0; jj < b; ++jj) acc += Mi[jj * b + ii] * ry[jj];
        pr.Y0[static_cast<std::size_t>(l) * nloc * b + static_cast<std::size_t>(i) * b + ii] = acc;
      }
    }
  }, 16);
  for (int i = 0; i < nloc; ++i) pr.tri_ptr[i + 1] = pr.tri_ptr[i] + static_cast<int>(tri_loc[i].size() / 6);
  pr.tri.reserve(static_cast<std::size_t>(pr.tri_ptr[nloc]) * 6);
  for (auto& t : tri_loc) pr.tri.insert(pr.tri.end(), t.begin(), t.end());
  gauss_legendre((order + 3) / 2, pr.gl_x, pr.gl_w);
  gauss_legendre((order + 2) / 2, pr.gs_x, pr.gs_w);

  if (dev_asm) {
    // face records for the device: cells, midpoint, half direction, half
    // length, normal, penalty (host/quadrature.cpp segment_rule, assembly.cpp:40-46)
    const auto& faces = mesh.interior_faces();
    const int nf = static_cast<int>(faces.size());
    pr.fcell.resize(2 * static_cast<std::size_t>(nf));
    pr.fgeo.resize(8 * static_cast<std::size_t>(nf));
    pr.fptr.assign(nloc + 1, 0);
    parallel_for(nf, [&](int f) {
      const Face& fc = faces[f];
      const int K = fc.cell_in, L = fc.cell_out;
      pr.fcell[2 * f] = pr.iperm[K];
      pr.fcell[2 * f + 1] = pr.iperm[L];
      const double hk = mesh.diameter(K), hl = mesh.diameter(L);
      const Pt mid = (fc.a + fc.b) * 0.5, dir = (fc.b - fc.a) * 0.5;
      double* g = &pr.fgeo[8 * static_cast<std::size_t>(f)];
      g[0] = mid.x;
      g[1] = mid.y;
      g[2] = dir.x;
      g[3] = dir.y;
      g[4] = 0.5 * dist(fc.a, fc.b);
      g[5] = fc.normal.x;
      g[6] = fc.normal.y;
      g[7] = cfg.eta0 * (0.5 * (sig_norm[K] + sig_norm[L])) * pr.p * pr.p / (2.0 * hk * hl / (hk + hl));
    }, 4096);
    for (int f = 0; f < nf; ++f) {
      ++pr.fptr[pr.fcell[2 * f] + 1];
      ++pr.fptr[pr.fcell[2 * f + 1] + 1];
    }
    for (int i = 0; i < nloc; ++i) pr.fptr[i + 1] += pr.fptr[i];
    pr.fent.resize(pr.fptr[nloc]);
    std::vector<int> fill(pr.fptr.begin(), pr.fptr.end() - 1);
    for (int f = 0; f < nf; ++f) {  // entry = 2 f + side, faces in face order per cell
      pr.fent[fill[pr.fcell[2 * f]]++] = 2 * f;
      pr.fent[fill[pr.fcell[2 * f + 1]]++] = 2 * f + 1;
    }
  } else {
  // interior faces (sequential in face order so the diagonal sums keep the reference order)
  {
    const auto& faces = mesh.interior_faces();
    const int nf = static_cast<int>(faces.size());
    std::vector<int> touched;
    for (int f = 0; f < nf; ++f) {
      const int iK = pr.iperm[faces[f].cell_in], iL = pr.iperm[faces[f].cell_out];
      const bool lk = iK >= pr.cell_begin && iK < pr.cell_end;
      const bool ll = iL >= pr.cell_begin && iL < pr.cell_end;
      if (lk || ll) touched.push_back(f);
    }
    const int nt = static_cast<int>(touched.size());
    std::vector<double> blocks(static_cast<std::size_t>(nt) * 3 * b2);
    parallel_for(nt, [&](int t) {
      const Face& f = faces[touched[t]];
      const int K = f.cell_in, L = f.cell_out;
      const double nk = sig_norm[K], nl = sig_norm[L];
      const double hk = mesh.diameter(K), hl = mesh.diameter(L);
      const double eta = cfg.eta0 * (0.5 * (nk + nl)) * pr.p * pr.p / (2.0 * hk * hl / (hk + hl));
      const Tensor& sk = sig[K];
      const Tensor& sl = sig[L];
      const std::vector<Pt> pk = mesh.cell_points(K), pl = mesh.cell_points(L);
      const Box bk = bbox_of(pk.data(), static_cast<int>(pk.size()));
      const Box bl = bbox_of(pl.data(), static_cast<int>(pl.size()));
      const Rule rule = segment_rule(f.a, f.b, order);
      double* kk = &blocks[static_cast<std::size_t>(t) * 3 * b2];
      double* lL = kk + b2;
      double* kl = lL + b2;
      std::vector<double> vk(b), vl(b), gxk(b), gyk(b), gxl(b), gyl(b), ak(b), al(b);
      for (std::size_t k = 0; k < rule.size(); ++k) {
        const double w = rule.w[k];
        basis_at(bk, pr.p, rule.pts[k], vk.data(), gxk.data(), gyk.data());
        basis_at(bl, pr.p, rule.pts[k], vl.data(), gxl.data(), gyl.data());
        for (int m = 0; m < b; ++m) {
          ak[m] = (sk.t00 * gxk[m] + sk.t01 * gyk[m]) * f.normal.x + (sk.t10 * gxk[m] + sk.t11 * gyk[m]) * f.normal.y;
          al[m] = (sl.t00 * gxl[m] + sl.t01 * gyl[m]) * f.normal.x + (sl.t10 * gxl[m] + sl.t11 * gyl[m]) * f.normal.y;
        }
        for (int ii = 0; ii < b; ++ii) {
          const double vki = vk[ii], vli = vl[ii];
          for (int jj = ii; jj < b; ++jj) {
            kk[jj * b + ii] += w * (-0.5 * (ak[jj] * vki + ak[ii] * vk[jj]) + eta * vk[jj] * vki);
            lL[jj * b + ii] += w * (0.5 * (al[jj] * vli + al[ii] * vl[jj]) + eta * vl[jj] * vli);
          }
          for (int jj = 0; jj < b; ++jj)
            kl[jj * b + ii] += w * (-0.5 * al[jj] * vki + 0.5 * ak[ii] * vl[jj] - eta * vl[jj] * vki);
        }
      }
    }, 64);
    // scatter per local cell, its faces in face order: each diagonal block
    // sums its face terms in the serial order and every off-diagonal block
    // has one face, so the parallel scatter gives the serial bits
    std::vector<int> tptr(nloc + 1, 0), tent;
    for (int t = 0; t < nt; ++t) {
      const Face& f = faces[touched[t]];
      const int iK = pr.iperm[f.cell_in], iL = pr.iperm[f.cell_out];
      if (iK >= pr.cell_begin && iK < pr.cell_end) ++tptr[iK - pr.cell_begin + 1];
      if (iL >= pr.cell_begin && iL < pr.cell_end) ++tptr[iL - pr.cell_begin + 1];
    }
    for (int i = 0; i < nloc; ++i) tptr[i + 1] += tptr[i];
    tent.resize(tptr[nloc]);
    {
      std::vector<int> fill(tptr.begin(), tptr.end() - 1);
      for (int t = 0; t < nt; ++t) {  // entry = 2 t + side (0: cell_in, 1: cell_out)
        const Face& f = faces[touched[t]];
        const int iK = pr.iperm[f.cell_in], iL = pr.iperm[f.cell_out];
        if (iK >= pr.cell_begin && iK < pr.cell_end) tent[fill[iK - pr.cell_begin]++] = 2 * t;
        if (iL >= pr.cell_begin && iL < pr.cell_end) tent[fill[iL - pr.cell_begin]++] = 2 * t + 1;
      }
    }
    parallel_for(nloc, [&](int li) {
      for (int e = tptr[li]; e < tptr[li + 1]; ++e) {
        const int t = tent[e] >> 1, side = tent[e] & 1;
        const Face& f = faces[touched[t]];
        const int iK = pr.iperm[f.cell_in], iL = pr.iperm[f.cell_out];
        const double* kk = &blocks[static_cast<std::size_t>(t) * 3 * b2];
        const double* lL = kk + b2;
        const double* kl = lL + b2;
        const double* dd = side == 0 ? kk : lL;
        const int self = side == 0 ? iK : iL, other = side == 0 ? iL : iK;
        double* D = &A.val[static_cast<std::size_t>(find_block(li, self)) * b2];
        for (int jj = 0; jj < b; ++jj)
          for (int ii = 0; ii <= jj; ++ii) {
            D[jj * b + ii] += dd[jj * b + ii];
            if (ii != jj) D[ii * b + jj] += dd[jj * b + ii];
          }
        double* O = &A.val[static_cast<std::size_t>(find_block(li, other)) * b2];
        if (side == 0) {
          for (int k = 0; k < b2; ++k) O[k] += kl[k];
        } else {
          for (int jj = 0; jj < b; ++jj)
            for (int ii = 0; ii < b; ++ii) O[jj * b + ii] += kl[ii * b + jj];
        }
      }
    }, 256);
  }
  }  // host faces
  // K = C_m chi_m M + dt/2 A (assembly.cpp:197-202)
  pr.K.rows = nloc;
  pr.K.b = b;
  pr.K.ptr = A.ptr;
  pr.K.col = A.col;
  if (!dev_asm) {
    const double a = cfg.C_m * cfg.chi_m, hb = 0.5 * cfg.dt;
    pr.K.val.resize(A.val.size());
    parallel_for(nloc, [&](int i) {
      for (int k = A.ptr[i]; k < A.ptr[i + 1]; ++k) {
        const bool diag = A.col[k] == pr.cell_begin + i;
        const double* a_ = &A.val[static_cast<std::size_t>(k) * b2];
        double* kv = &pr.K.val[static_cast<std::size_t>(k) * b2];
        const double* m_ = &pr.M[static_cast<std::size_t>(i) * b2];
        for (int e = 0; e < b2; ++e) kv[e] = diag ? a * m_[e] + hb * a_[e] : hb * a_[e];
      }
    }, 256);
    if (!pr.keep_matrices) {
      A.val.clear();
      A.val.shrink_to_fit();
    }
  }

  phase("assembly");
  factor_units(pr, pl);
  phase("factor+pack");
  // ---- coarse embedding E (schwarz.cpp:13-77) and local K0 contribution ----
  if (pr.two_level) {
    const int na = pr.coarse.count;
    const std::vector<Box> abox = agglomerate_boxes(mesh, pr.coarse.owner, na);
    // coarse internal order: ND over the agglomerate graph
    std::vector<std::vector<int>> anbr(na);
    for (const Face& f : mesh.interior_faces()) {
      const int a = pr.coarse.owner[f.cell_in], c2 = pr.coarse.owner[f.cell_out];
      if (a != c2) {
        anbr[a].push_back(c2);
        anbr[c2].push_back(a);
      }
    }
    std::vector<Pt> apos(na);
    for (int a = 0; a < na; ++a) apos[a] = {0.5 * (abox[a].xmin + abox[a].xmax), 0.5 * (abox[a].ymin + abox[a].ymax)};
    // E for local cells and for the halo cells their rows touch
    std::vector<int> need;  // global internal cells needing E
    {
      std::vector<char> mark(N, 0);
      for (int i = 0; i < nloc; ++i)
        for (int k = pr.K.ptr[i]; k < pr.K.ptr[i + 1]; ++k) mark[pr.K.col[k]] = 1;
      for (int g = 0; g < N; ++g)
        if (mark[g]) need.push_back(g);
    }
    std::vector<int> e_slot(N, -1);
    for (std::size_t k = 0; k < need.size(); ++k) e_slot[need[k]] = static_cast<int>(k);
    std::vector<int> need_ref(need.size());
    for (std::size_t k = 0; k < need.size(); ++k) need_ref[k] = pr.perm[need[k]];
    std::vector<double> Eall;
    if (dev_asm) {  // E and K0 on the device: coarse boxes and labels only
      pr.abox.resize(4 * static_cast<std::size_t>(na));
      for (int a = 0; a < na; ++a) {
        pr.abox[4 * a] = abox[a].xmin;
        pr.abox[4 * a + 1] = abox[a].ymin;
        pr.abox[4 * a + 2] = abox[a].xmax;
        pr.abox[4 * a + 3] = abox[a].ymax;
      }
      pr.cell_label.resize(nloc);
      for (int i = 0; i < nloc; ++i) pr.cell_label[i] = pr.coarse.owner[pr.perm[pr.cell_begin + i]];
    } else {
      Eall = coarse_embedding_cells(mesh, pr.p, pr.coarse.owner, abox, pr.q, need_ref);
    }
    coarse_space(pr, anbr, &apos, Eall, e_slot);
    phase("coarse E,K0");
    if (cfg.world == 1 && !dev_asm) finish_coarse(pr);
    phase("coarse factor");
  }
  return P;
}


std::unique_ptr<Problem> build_problem_from_operator(const pdg_operator_desc& d) {
  const int N = d.n_cells, b = d.block;
  if (N <= 0 || b <= 0) throw ConfigError("operator: n_cells and block must be positive");
  if (!d.row_ptr || !d.col || !d.val) throw ConfigError("operator: K arrays are required");
  if (d.precond_kind != PDG_PRECOND_NONE && d.precond_kind != PDG_PRECOND_BLOCK_JACOBI &&
      d.precond_kind != PDG_PRECOND_TWO_LEVEL)
    throw ConfigError("operator: unknown preconditioner kind");
  auto P = std::make_unique<Problem>();
  Problem& pr = *P;
  pdg_config_default(&pr.cfg);
  pr.cfg.device = d.device;
  pr.cfg.maxit = d.maxit;
  pr.cfg.precond_kind = d.precond_kind;
  pr.cfg.subdomains = d.sub_owner ? d.n_sub : 0;
  pr.cfg.ionic_model = PDG_IONIC_NONE;
  pr.cfg.rank = 0;
  pr.cfg.world = 1;
  pr.from_operator = true;
  pr.n_cells_global = N;
  pr.b = b;
  pr.p = 0;
  while (n_modes(pr.p + 1) <= b) ++pr.p;  // P^p with (p+1)(p+2)/2 = b when b is triangular
  pr.has_precond = d.precond_kind != PDG_PRECOND_NONE;
  pr.two_level = d.precond_kind == PDG_PRECOND_TWO_LEVEL;
  pr.n_comp = 0;
  const std::int64_t n = static_cast<std::int64_t>(N) * b;
  const int b2 = b * b;
  // ---- K: scalar CSR -> element blocks (cell adjacency = nonzero blocks) ----
  std::vector<std::vector<int>> nbr(N);
  for (std::int64_t i = 0; i < n; ++i) {
    if (d.row_ptr[i + 1] < d.row_ptr[i]) throw ConfigError("operator: row_ptr must be non-decreasing");
    for (std::int64_t k = d.row_ptr[i]; k < d.row_ptr[i + 1]; ++k) {
      const int j = d.col[k];
      if (j < 0 || j >= n) throw ConfigError("operator: column index out of range");
      const int ci = static_cast<int>(i / b), cj = j / b;
      if (ci != cj) {
        nbr[ci].push_back(cj);
        nbr[cj].push_back(ci);  // symmetric pattern even if an entry is missing
      }
    }
  }
  parallel_for(N, [&](int c) {
    auto& v = nbr[c];
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }, 1024);
  // ---- partitions ----
  auto check_owner = [&](const int* o, int count, const char* what) {
    if (count <= 0) throw ConfigError(std::string("operator: ") + what + " count must be positive");
    for (int c = 0; c < N; ++c)
      if (o[c] < 0 || o[c] >= count) throw ConfigError(std::string("operator: ") + what + " owner out of range");
  };
  if (d.sub_owner) {
    check_owner(d.sub_owner, d.n_sub, "subdomain");
    pr.sub.owner.assign(d.sub_owner, d.sub_owner + N);
    pr.sub.count = d.n_sub;
  } else {
    pr.sub.owner.resize(N);
    std::iota(pr.sub.owner.begin(), pr.sub.owner.end(), 0);
    pr.sub.count = N;
  }
  // coarse embedding: agglomerate of each element row block from E's columns
  std::vector<double> Eblk;
  if (pr.two_level) {
    if (!d.e_row_ptr || !d.e_col || !d.e_val || d.n_coarse <= 0 || d.coarse_block <= 0)
      throw ConfigError("operator: two-level preconditioner needs the coarse embedding E");
    const int bq = d.coarse_block;
    pr.bq = bq;
    pr.q = 0;
    while (n_modes(pr.q + 1) <= bq) ++pr.q;
    pr.coarse.owner.assign(N, -1);
    pr.coarse.count = d.n_coarse;
    Eblk.assign(static_cast<std::size_t>(N) * b * bq, 0.0);
    for (std::int64_t i = 0; i < n; ++i)
      for (std::int64_t k = d.e_row_ptr[i]; k < d.e_row_ptr[i + 1]; ++k) {
        const int j = d.e_col[k];
        if (j < 0 || j >= d.n_coarse * bq) throw ConfigError("operator: E column out of range");
        const int c = static_cast<int>(i / b), a = j / bq;
        if (pr.coarse.owner[c] < 0) pr.coarse.owner[c] = a;
        if (pr.coarse.owner[c] != a) throw ConfigError("operator: E must hold one agglomerate block per element");
        Eblk[static_cast<std::size_t>(c) * b * bq + static_cast<std::size_t>(j % bq) * b + i % b] = d.e_val[k];
      }
    for (int c = 0; c < N; ++c)
      if (pr.coarse.owner[c] < 0) throw ConfigError("operator: E has an empty element row block");
  }
  // ---- placement units: subdomains (label order), else 256-cell runs ----
  Placement pl;
  pl.multi_sub = d.sub_owner != nullptr;
  if (pl.multi_sub) {
    pl.units = pr.sub.members();
  } else if (pr.two_level) {
    pl.units = pr.coarse.members();
  } else {
    for (int s = 0; s < N; s += 256) {
      pl.units.emplace_back();
      for (int c = s; c < std::min(N, s + 256); ++c) pl.units.back().push_back(c);
    }
  }
  pl.unit_order.resize(pl.units.size());
  std::iota(pl.unit_order.begin(), pl.unit_order.end(), 0);
  place_units(pr, pl, nbr, nullptr);
  // ---- K in internal order ----
  Bsr& K = pr.K;
  K.rows = N;
  K.b = b;
  K.ptr.assign(N + 1, 0);
  for (int i = 0; i < N; ++i) K.ptr[i + 1] = K.ptr[i] + 1 + static_cast<int>(nbr[pr.perm[i]].size());
  K.col.resize(K.ptr[N]);
  K.val.assign(static_cast<std::size_t>(K.ptr[N]) * b2, 0.0);
  parallel_for(N, [&](int i) {
    const int c = pr.perm[i];
    std::vector<int> cols{i};
    for (int nb : nbr[c]) cols.push_back(pr.iperm[nb]);
    std::sort(cols.begin(), cols.end());
    std::copy(cols.begin(), cols.end(), K.col.begin() + K.ptr[i]);
    for (int r = 0; r < b; ++r) {
      const std::int64_t row = static_cast<std::int64_t>(c) * b + r;
      for (std::int64_t k = d.row_ptr[row]; k < d.row_ptr[row + 1]; ++k) {
        const int j = d.col[k], gj = pr.iperm[j / b];
        const int blk = static_cast<int>(std::lower_bound(cols.begin(), cols.end(), gj) - cols.begin());
        K.val[static_cast<std::size_t>(K.ptr[i] + blk) * b2 + static_cast<std::size_t>(j % b) * b + r] += d.val[k];
      }
    }
  }, 256);
  pr.keep_matrices = false;
  pr.U0.assign(static_cast<std::size_t>(n), 0.0);
  factor_units(pr, pl);
  // ---- coarse space from the caller's E ----
  if (pr.two_level) {
    const int na = pr.coarse.count, bq = pr.bq;
    std::vector<std::vector<int>> anbr(na);
    for (int c = 0; c < N; ++c)
      for (int nb : nbr[c]) {
        const int a = pr.coarse.owner[c], a2 = pr.coarse.owner[nb];
        if (a != a2) anbr[a].push_back(a2);
      }
    std::vector<double> Eall(static_cast<std::size_t>(N) * b * bq);
    std::vector<int> e_slot(N);
    for (int g = 0; g < N; ++g) {
      e_slot[g] = g;
      std::copy(Eblk.begin() + static_cast<std::size_t>(pr.perm[g]) * b * bq,
                Eblk.begin() + static_cast<std::size_t>(pr.perm[g] + 1) * b * bq,
                Eall.begin() + static_cast<std::size_t>(g) * b * bq);
    }
    coarse_space(pr, anbr, nullptr, Eall, e_slot);
    finish_coarse(pr);
  }
  return P;
}

void finish_coarse(Problem& pr) {
  if (!pr.two_level) return;
  // the coarse unit is replicated on every rank; K0 is already in the coarse
  // nested-dissection position order, so the tree applies directly
  BlockMatrix Pm;
  Pm.m = pr.K0.rows;
  Pm.bs = pr.K0.b;
  Pm.ptr = pr.K0.ptr;
  Pm.col = pr.K0.col;
  Pm.val = pr.K0.val;
  NdTree tid = pr.coarse_nd;
  std::iota(tid.order.begin(), tid.order.end(), 0);
  SupernodalFactor F;
  try {
    F = supernodal_cholesky(Pm, tid);
  } catch (const SolverError&) {
    throw SolverError("schwarz: coarse operator factorization failed");
  }
  // coarse tasks use vector set 1 (r0 -> y0) and follow the fine ones
  pack_unit_tasks(pr, F, 1, 0);
}

}  // namespace pdg
