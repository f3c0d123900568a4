// C-ABI entry points for host setup (mesh, partitions, problem export).
// Declared in include/polydg_b200.h; each maps reference exceptions to
// pdg_status codes (errors.hpp:13-35 -> PDG_ERR_*).
#include <cmath>
#include <cstring>
#include <random>
#include <string>

#include "../../include/polydg_b200.h"
#include "capi_internal.hpp"
#include "host/problem.hpp"
#include "host/quadrature.hpp"

struct pdg_mesh {
  pdg::Mesh m;
};
struct pdg_problem {
  std::unique_ptr<pdg::Problem> p;
};

namespace pdg {
thread_local std::string g_last_error;
void set_error(const std::string& s) { g_last_error = s; }
}  // namespace pdg

extern "C" {

const char* pdg_last_error(void) { return pdg::g_last_error.c_str(); }

void pdg_config_default(pdg_config* c) {
  std::memset(c, 0, sizeof *c);
  // SimulationConfig defaults (timestepper.hpp:21-80)
  c->mesh_cells = 512;
  c->mesh_seed = 42;
  c->mesh_lloyd = 20;
  c->domain[0] = 0.0;
  c->domain[1] = 0.0;
  c->domain[2] = 1.0;
  c->domain[3] = 1.0;
  c->split_y = 0.5;
  c->degree = 1;
  c->eta0 = 10.0;
  c->chi_m = 1000.0;
  c->C_m = 1.0;
  c->dt = 2.5e-3;
  c->T = 10.0;
  c->sigma_grey_l = 6.3;
  c->sigma_grey_n = 6.3;
  c->sigma_white_l = 6.9;
  c->sigma_white_n = 25.71;
  c->fiber_grey[1] = 1.0;
  c->fiber_white[1] = 1.0;
  c->fiber_seed = 42;
  c->ionic_model = PDG_IONIC_FHN;
  const double fhn[8] = {0.13, 0.013, 0.26, 0.1, 1.0, -85.0, 20.0, 1.0};  // ionics.hpp:42-51
  std::memcpy(c->fhn, fhn, sizeof fhn);
  c->init_kind = PDG_INIT_DISC;
  c->u_rest = -67.0;
  c->u_patch = -50.0;
  c->omega0[0] = 0.5;
  c->omega0[1] = 1.0;
  c->omega0_r2 = 0.016;
  c->stim_kind = PDG_STIM_NONE;
  c->tol = 1e-9;
  c->maxit = 0;
  c->warm_start = 1;
  c->precond_kind = PDG_PRECOND_TWO_LEVEL;
  c->h_ratio = 2;
  c->q = 0;
  c->subdomains = 0;
  c->coarse_count = 0;
  c->rank = 0;
  c->world = 1;
  c->device = 0;
  // Barreto-Cressman (ext): Cressman et al. 2009 values, k_bath = 4 mM
  const double bc[PDG_BC_NPARAM] = {100.0, 40.0, 0.0175, 0.05, 0.05,  // g_Na g_K g_NaL g_KL g_ClL
                                    3.0,                             // phi
                                    1.25, 66.0, 1.2, 4.0,            // rho G_glia eps k_bath
                                    0.0445, 7.0, 1000.0,             // gamma beta tau
                                    26.64, 6.0, 130.0,               // RT/F, [Cl]i, [Cl]o
                                    18.0, 140.0, 144.0, 1.0};        // Na_i0 K_i0 Na_o0 amp
  std::memcpy(c->bc, bc, sizeof bc);
}

pdg_status pdg_ionic_rest(const pdg_config* cfg, int* n_comp, double* u_rest, double* y_rest) {
  return pdg::guarded([&] {
    pdg::validate_config(*cfg);
    double u = 0.0, y[4] = {0.0, 0.0, 0.0, 0.0};
    const int nc = pdg::ionic_rest(*cfg, u, y);
    if (n_comp) *n_comp = nc;
    if (u_rest) *u_rest = u;
    if (y_rest)
      for (int l = 0; l < nc; ++l) y_rest[l] = y[l];
  });
}

void pdg_uniform_rhs(uint64_t seed, int64_t n, double* out) {
  std::mt19937_64 rng(seed);
  for (int64_t i = 0; i < n; ++i) out[i] = 2.0 * (static_cast<double>(rng() >> 11) * 0x1.0p-53) - 1.0;
}

int pdg_default_max_iterations(int64_t n) {
  // krylov.cpp:12-15
  const double cap = 20.0 * std::sqrt(static_cast<double>(n));
  return static_cast<int>(std::min(cap, static_cast<double>(n)));
}

pdg_status pdg_mesh_generate(int n, const double d[4], uint64_t seed, int lloyd, double split_y,
                             pdg_mesh** out) {
  return pdg::guarded([&] {
    pdg::Mesh m = pdg::generate_mesh(n, pdg::Box{d[0], d[1], d[2], d[3]}, seed, lloyd);
    if (split_y > d[1]) m = pdg::assign_regions(m, split_y);
    *out = new pdg_mesh{std::move(m)};
  });
}

void pdg_mesh_free(pdg_mesh* m) { delete m; }

void pdg_mesh_counts(const pdg_mesh* h, int counts[5]) {
  const auto& m = h->m;
  counts[0] = m.n_cells();
  counts[1] = m.n_vertices();
  counts[2] = static_cast<int>(m.cell_vertex_ids().size());
  counts[3] = static_cast<int>(m.interior_faces().size());
  counts[4] = static_cast<int>(m.boundary_faces().size());
}

void pdg_mesh_arrays(const pdg_mesh* h, double* verts, int* off, int* idx, uint8_t* regions) {
  const auto& m = h->m;
  for (int v = 0; v < m.n_vertices(); ++v) {
    verts[2 * v] = m.vertices()[v].x;
    verts[2 * v + 1] = m.vertices()[v].y;
  }
  std::memcpy(off, m.cell_offsets().data(), sizeof(int) * m.cell_offsets().size());
  std::memcpy(idx, m.cell_vertex_ids().data(), sizeof(int) * m.cell_vertex_ids().size());
  std::memcpy(regions, m.regions().data(), m.regions().size());
}

void pdg_mesh_faces(const pdg_mesh* h, int interior, int* cells, double* geo) {
  const auto& fs = interior ? h->m.interior_faces() : h->m.boundary_faces();
  for (std::size_t i = 0; i < fs.size(); ++i) {
    const pdg::Face& f = fs[i];
    cells[2 * i] = f.cell_in;
    cells[2 * i + 1] = f.cell_out;
    const double g[7] = {f.a.x, f.a.y, f.b.x, f.b.y, f.normal.x, f.normal.y, f.length};
    std::memcpy(geo + 7 * i, g, sizeof g);
  }
}

void pdg_mesh_cell_geometry(const pdg_mesh* h, double* out) {
  const auto& m = h->m;
  for (int c = 0; c < m.n_cells(); ++c) {
    out[4 * c] = m.area(c);
    out[4 * c + 1] = m.centroid(c).x;
    out[4 * c + 2] = m.centroid(c).y;
    out[4 * c + 3] = m.diameter(c);
  }
}

pdg_status pdg_mesh_coarse_embedding(const pdg_mesh* h, int p, const int* owner, int count, int q,
                                     double* E_blocks) {
  return pdg::guarded([&] {
    if (p < 1) throw pdg::ConfigError("build_coarse_embedding: degree must be >= 1");
    const std::vector<int> own(owner, owner + h->m.n_cells());
    const std::vector<double> E = pdg::coarse_embedding(h->m, p, own, count, q);
    std::memcpy(E_blocks, E.data(), sizeof(double) * E.size());
  });
}

int pdg_mesh_agglomerate(const pdg_mesh* h, int target, int* owner, double* H) {
  int count = -1;
  const pdg_status st = pdg::guarded([&] {
    const pdg::Partition p = pdg::agglomerate(h->m, target);
    std::memcpy(owner, p.owner.data(), sizeof(int) * p.owner.size());
    if (H) std::memcpy(H, p.H.data(), sizeof(double) * p.H.size());
    count = p.count;
  });
  return st == PDG_OK ? count : -1;
}

int pdg_mesh_agglomerate_hierarchy(const pdg_mesh* h, int levels, int* owner) {
  int count = -1;
  const pdg_status st = pdg::guarded([&] {
    const auto hier = pdg::agglomerate_hierarchy(h->m, levels);
    std::memcpy(owner, hier.back().owner.data(), sizeof(int) * hier.back().owner.size());
    count = hier.back().count;
  });
  return st == PDG_OK ? count : -1;
}

int pdg_polygon_quadrature(const double* poly, int n, int order, double* pts, double* w, int cap) {
  int np = -1;
  const pdg_status st = pdg::guarded([&] {
    std::vector<pdg::Pt> p(n);
    for (int i = 0; i < n; ++i) p[i] = {poly[2 * i], poly[2 * i + 1]};
    const pdg::Rule r = pdg::polygon_rule(p, order);
    np = static_cast<int>(r.size());
    for (int i = 0; i < np && i < cap; ++i) {
      pts[2 * i] = r.pts[i].x;
      pts[2 * i + 1] = r.pts[i].y;
      w[i] = r.w[i];
    }
  });
  return st == PDG_OK ? np : -1;
}

pdg_status pdg_problem_create(const pdg_config* cfg, pdg_problem** out) {
  return pdg::guarded([&] { *out = new pdg_problem{pdg::build_problem(*cfg)}; });
}

void pdg_problem_free(pdg_problem* p) { delete p; }

void pdg_problem_info(const pdg_problem* h, int64_t info[12]) {
  pdg::problem_info(*h->p, info);
}

int pdg_problem_flags(const pdg_problem* h) {
  return (h->p->device_assembly ? 1 : 0) | (h->p->device_factor ? 2 : 0);
}

int64_t pdg_problem_export(const pdg_problem* h, int which, int64_t* rows, int64_t* cols,
                           double* vals) {
  return pdg::problem_export(*h->p, which, rows, cols, vals);
}

void pdg_problem_owner(const pdg_problem* h, int which, int* owner) {
  const auto& pr = *h->p;
  const auto& src = which == 0 ? pr.sub.owner : pr.coarse.owner;
  for (std::size_t c = 0; c < src.size(); ++c) owner[c] = src[c];
}

void pdg_problem_factor_stats(const pdg_problem* h, int64_t stats[6]) {
  const auto& pr = *h->p;
  int64_t nnzb_local = 0;
  for (std::size_t i = 0; i + 1 < pr.K.ptr.size(); ++i) nnzb_local += pr.K.ptr[i + 1] - pr.K.ptr[i];
  stats[0] = pr.l_struct;
  stats[1] = pr.l0_struct;
  stats[2] = pr.fmat_len;
  stats[3] = pr.hmat_len;
  stats[4] = nnzb_local;
  stats[5] = static_cast<int64_t>(pr.E.size());
}

void pdg_problem_sweep_stats(const pdg_problem* h, int64_t stats[8]) {
  const auto& pr = *h->p;
  for (int i = 0; i < 8; ++i) stats[i] = 0;
  stats[0] = static_cast<int64_t>(pr.tasks.size());
  int64_t dense_bottom = 0;
  for (const auto& t : pr.tasks)
    if (t.bottom >= 0) {
      ++stats[1];
      dense_bottom += t.root_dense;
    }
  stats[2] = pr.n_bottom_levels;
  // chunks are stored in ticket order per direction: a chunk's dependency slot must already hold chunks
  bool ok = true;
  std::vector<int> seen[2];
  seen[0].assign(pr.level_chunks[0].size(), 0);
  seen[1].assign(pr.level_chunks[1].size(), 0);
  int64_t covered_b = 0;
  for (const auto& c : pr.chunks) {
    ++stats[3 + c.dir];
    if (c.dir == 0) stats[5] += c.n_task;
    else covered_b += c.n_task;
    ok = ok && c.meta_n <= pdg::kChunkMetaInts && c.xneed <= 4096;
    if (c.dep_slot >= 0)
      ok = ok && (c.dep_dir < c.dir || seen[c.dep_dir][c.dep_slot] == pr.level_chunks[c.dep_dir][c.dep_slot]) &&
           pr.level_chunks[c.dep_dir][c.dep_slot] > 0;
    if (c.slot >= 0) ++seen[c.dir][c.slot];
    ++seen[c.dir][c.gslot];
  }
  stats[6] = covered_b;  // backward chunks list every bottom supernode too (dense roots carry no tiles)
  (void)dense_bottom;
  stats[7] = ok ? 1 : 0;
}

void pdg_problem_perm(const pdg_problem* h, int* perm) {
  std::memcpy(perm, h->p->perm.data(), sizeof(int) * h->p->perm.size());
}

}  // extern "C"

namespace pdg {

void problem_info(const Problem& pr, int64_t info[12]) {
  info[0] = pr.n_cells_global;
  info[1] = pr.b;
  info[2] = pr.n_global_dofs();
  info[3] = pr.sub.count;
  info[4] = pr.two_level ? pr.n_agg : 0;
  info[5] = pr.two_level ? static_cast<int64_t>(pr.n_agg) * pr.bq : 0;
  info[6] = static_cast<int64_t>(pr.K.col.size());
  info[7] = pr.factor_values;
  info[8] = static_cast<int64_t>(pr.tasks.size());
  info[9] = pr.n_comp;
  info[10] = pr.cell_begin;
  info[11] = pr.cell_end;
}

int64_t problem_export(const Problem& pr, int which, int64_t* rows, int64_t* cols, double* vals) {
  const int b = pr.b, b2 = b * b;
  int64_t n = 0;
  auto emit = [&](int64_t r, int64_t c, double v) {
    if (rows) {
      rows[n] = r;
      cols[n] = c;
      vals[n] = v;
    }
    ++n;
  };
  const auto ref_dof = [&](int internal_cell, int r) {
    return static_cast<int64_t>(pr.perm[internal_cell]) * b + r;
  };
  if (which == 0 || which == 2) {
    const Bsr& X = which == 0 ? pr.K : pr.A;
    if (X.val.empty()) return -1;
    for (int i = 0; i < X.rows; ++i)
      for (int k = X.ptr[i]; k < X.ptr[i + 1]; ++k)
        for (int c = 0; c < b; ++c)
          for (int r = 0; r < b; ++r)
            emit(ref_dof(pr.cell_begin + i, r), ref_dof(X.col[k], c), X.val[static_cast<size_t>(k) * b2 + c * b + r]);
  } else if (which == 1) {
    for (int i = 0; i < pr.cell_end - pr.cell_begin; ++i)
      for (int c = 0; c < b; ++c)
        for (int r = 0; r < b; ++r)
          emit(ref_dof(pr.cell_begin + i, r), ref_dof(pr.cell_begin + i, c), pr.M[static_cast<size_t>(i) * b2 + c * b + r]);
  } else if (which == 3) {
    if (!pr.two_level) return -1;
    const int bq = pr.bq;
    for (int i = 0; i < pr.cell_end - pr.cell_begin; ++i) {
      const int label = pr.agg_order[pr.cell_agg[i]];
      for (int m = 0; m < bq; ++m)
        for (int r = 0; r < b; ++r)
          emit(ref_dof(pr.cell_begin + i, r), static_cast<int64_t>(label) * bq + m,
               pr.E[static_cast<size_t>(i) * b * bq + m * b + r]);
    }
  } else if (which == 4) {
    if (!pr.two_level) return -1;
    const int bq = pr.bq, bq2 = bq * bq;
    for (int i = 0; i < pr.K0.rows; ++i)
      for (int k = pr.K0.ptr[i]; k < pr.K0.ptr[i + 1]; ++k)
        for (int c = 0; c < bq; ++c)
          for (int r = 0; r < bq; ++r)
            emit(static_cast<int64_t>(pr.agg_order[i]) * bq + r,
                 static_cast<int64_t>(pr.agg_order[pr.K0.col[k]]) * bq + c,
                 pr.K0.val[static_cast<size_t>(k) * bq2 + c * bq + r]);
  } else {
    return -1;
  }
  return n;
}

}  // namespace pdg

extern "C" {

// SpMV halo of this rank against `peer` (host/pack.cpp halo_plan): send = local
// internal cells (relative to the rank's first cell), recv = global internal
// cells; counts[0..1] = sizes. Arrays may be NULL to query the sizes.
pdg_status pdg_problem_mesh(const pdg_problem* h, pdg_mesh** out) {
  return pdg::guarded([&] { *out = new pdg_mesh{h->p->mesh}; });
}

void pdg_problem_halo(const pdg_problem* h, int peer, int* send, int* recv, int counts[2]) {
  std::vector<std::vector<int>> s, r;
  pdg::halo_plan(*h->p, s, r);
  counts[0] = static_cast<int>(s[peer].size());
  counts[1] = static_cast<int>(r[peer].size());
  if (send) std::copy(s[peer].begin(), s[peer].end(), send);
  if (recv) std::copy(r[peer].begin(), r[peer].end(), recv);
}

// internal cell range of every rank: world+1 entries
void pdg_problem_rank_cells(const pdg_problem* h, int* starts) {
  std::copy(h->p->rank_cell_start.begin(), h->p->rank_cell_start.end(), starts);
}

}  // extern "C"
