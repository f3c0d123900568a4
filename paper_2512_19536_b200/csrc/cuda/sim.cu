// Device-resident solver: uploads the host setup once (K_h is constant in
// time, timestepper.hpp:113-115) and runs Simulation::step / pcg_solve on the
// GPU. The PCG loop is one CUDA graph whose body is a conditional WHILE node,
// so an entire solve is a single launch and the iteration count, convergence
// test (krylov.cpp:58-64) and breakdown checks (:46-53, :66-68) are decided on
// the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <queue>
#include <vector>

#include "../host/problem.hpp"
#include "kernels.cuh"
#include "../host/bc_model.hpp"
#include "sim.cuh"

namespace pdg {

template <class T>
static T* dalloc(std::size_t n) {
  T* p = nullptr;
  if (n == 0) n = 1;
  PDG_CUDA(cudaMalloc(&p, n * sizeof(T)));
  return p;
}

template <class T>
static T* dupload(const std::vector<T>& v, cudaStream_t st) {
  T* p = dalloc<T>(v.size());
  if (!v.empty()) PDG_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
  return p;
}

static const char* pcg_error_message(int e) {
  switch (e) {
    case kPcgRhoNonFinite0: return "pcg: non-finite preconditioned product";
    case kPcgRhoNonPos0: return "pcg: preconditioner is not positive definite";
    case kPcgPqNonFinite: return "pcg: non-finite operator product";
    case kPcgPqNonPos: return "pcg: operator is not positive definite";
    case kPcgRhoNonFinite: return "pcg: non-finite scalar";
    case kPcgRhoNonPos: return "pcg: preconditioner is not positive definite";
  }
  return "pcg: unknown breakdown";
}

__global__ void set_condition_kernel(cudaGraphConditionalHandle h, const PcgScalars* S) {
  pdl_wait();
  cudaGraphSetConditional(h, S->stop ? 0u : 1u);
}

DeviceSim::DeviceSim(std::unique_ptr<Problem> prob) : P(std::move(prob)) {
  const Problem& pr = *P;
  PDG_CUDA(cudaSetDevice(pr.cfg.device));
  PDG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  PDG_CUDA(cudaEventCreate(&ev0));
  PDG_CUDA(cudaEventCreate(&ev1));
  PDG_CUDA(cudaEventCreate(&ev2));
  PDG_CUDA(cudaEventCreate(&ev_t0));
  PDG_CUDA(cudaEventCreate(&ev_t1));
  b = pr.b;
  bq = pr.two_level ? pr.bq : 0;
  ncells = pr.cell_end - pr.cell_begin;
  n = static_cast<long long>(ncells) * b;
  n_comp = pr.n_comp;
  rank = pr.cfg.rank;
  world = pr.cfg.world;
  maxit_default = pr.cfg.maxit > 0 ? pr.cfg.maxit : pdg_default_max_iterations(pr.n_global_dofs());

  // ---- operator: columns remapped to local positions (halo appended, multi-rank) ----
  // Halo cells sorted by global internal index: ranks own contiguous ranges,
  // so the halo is grouped by source rank, in the order the sender packs it.
  std::vector<int> col(pr.K.col.size());
  halo_cells.clear();
  {
    for (int g : pr.K.col)
      if (g < pr.cell_begin || g >= pr.cell_end) halo_cells.push_back(g);
    std::sort(halo_cells.begin(), halo_cells.end());
    halo_cells.erase(std::unique(halo_cells.begin(), halo_cells.end()), halo_cells.end());
    for (std::size_t k = 0; k < pr.K.col.size(); ++k) {
      const int g = pr.K.col[k];
      col[k] = (g >= pr.cell_begin && g < pr.cell_end)
                   ? g - pr.cell_begin
                   : ncells + static_cast<int>(std::lower_bound(halo_cells.begin(), halo_cells.end(), g) -
                                               halo_cells.begin());
    }
  }
  n_ext = n + static_cast<long long>(halo_cells.size()) * b;
  d_ptr = dupload(pr.K.ptr, st);
  d_col = dupload(col, st);
  if (pr.device_assembly) {  // values formed by cuda/assemble.cu below
    const std::size_t nkv = static_cast<std::size_t>(pr.K.ptr[ncells]) * b * b;
    d_kval = dalloc<double>(nkv);
    PDG_CUDA(cudaMemsetAsync(d_kval, 0, nkv * sizeof(double), st));
    d_M = dalloc<double>(static_cast<std::size_t>(ncells) * b * b);
    d_Minv = dalloc<double>(static_cast<std::size_t>(ncells) * b * b);
  } else {
    d_kval = dupload(pr.K.val, st);
    d_M = dupload(pr.M, st);
    d_Minv = dupload(pr.Minv, st);
  }

  for (auto& v : d_U) v = dalloc<double>(n_ext);
  d_x = dalloc<double>(n_ext);
  d_p = dalloc<double>(n_ext);
  d_r = dalloc<double>(n);
  d_z = dalloc<double>(n);
  d_q = dalloc<double>(n);
  d_rhs = dalloc<double>(n);
  d_ion = dalloc<double>(n);
  d_tmp = dalloc<double>(n_ext);
  d_tmp2 = dalloc<double>(n_ext);
  d_scratch = dalloc<double>(8);
  for (auto& v : d_Y) v = dalloc<double>(std::max<long long>(n * n_comp, 1));
  PDG_CUDA(cudaMemsetAsync(d_p, 0, n_ext * sizeof(double), st));
  PDG_CUDA(cudaMemsetAsync(d_x, 0, n_ext * sizeof(double), st));
  for (auto& v : d_U) PDG_CUDA(cudaMemsetAsync(v, 0, n_ext * sizeof(double), st));

  // ---- coarse space ----
  if (pr.two_level) {
    d_E = pr.device_assembly ? dalloc<double>(static_cast<std::size_t>(ncells) * b * pr.bq) : dupload(pr.E, st);
    d_cell_agg = dupload(pr.cell_agg, st);
    d_agg_ptr = dupload(pr.agg_cell_ptr, st);
    d_agg_cells = dupload(pr.agg_cells, st);
    // + 1: the multi-rank loop all-reduces [r0 ; ||r||^2 partial] in one call
    d_r0 = dalloc<double>(static_cast<std::size_t>(pr.n_agg) * pr.bq + 1);
    d_y0 = dalloc<double>(static_cast<std::size_t>(pr.n_agg) * pr.bq);
    // restriction chunks: <= kChunk cells of one agglomerate per CTA;
    // small chunks keep the fused update + restriction spread over all SMs
    constexpr int kChunk = 32;
    std::vector<int> cptr{0}, nptr{0};
    for (int a = 0; a < pr.n_agg; ++a) {
      for (int k = pr.agg_cell_ptr[a]; k < pr.agg_cell_ptr[a + 1]; k += kChunk)
        cptr.push_back(std::min(k + kChunk, pr.agg_cell_ptr[a + 1]));
      nptr.push_back(static_cast<int>(cptr.size()) - 1);
    }
    n_chunks = static_cast<int>(cptr.size()) - 1;
    // chunks of consecutive cells -> the coarse kernels stage E by bulk copy
    chunks_contiguous = true;
    max_chunk_cells = 1;
    for (int c = 0; c < n_chunks; ++c) {
      max_chunk_cells = std::max(max_chunk_cells, cptr[c + 1] - cptr[c]);
      for (int k = cptr[c]; k < cptr[c + 1]; ++k)
        if (pr.agg_cells[k] != pr.agg_cells[cptr[c]] + (k - cptr[c])) chunks_contiguous = false;
    }
    d_chunk_ptr = dupload(cptr, st);
    d_node_chunk_ptr = dupload(nptr, st);
    d_r0part = dalloc<double>(static_cast<std::size_t>(std::max(n_chunks, 1)) * pr.bq);
  }
  // ---- ionic geometry (also the device assembly's) ----
  d_bbox = dupload(pr.bbox, st);
  d_tri_ptr = dupload(pr.tri_ptr, st);
  d_tri = dupload(pr.tri, st);
  if (pr.device_assembly) assemble_on_device();
  upload_tasks();

  if (!pr.gl_x.empty()) set_gauss_nodes(pr.gl_x.data(), pr.gl_w.data(), static_cast<int>(pr.gl_x.size()));
  d_ionflags = dalloc<int>(1);
  PDG_CUDA(cudaMemsetAsync(d_ionflags, 0, sizeof(int), st));

  // ---- reductions / scalars / history ----
  const long long max_grid = std::max<long long>(ncells + 1, 4096) + 4096;
  red.partial = dalloc<double>(max_grid);
  red.counter = dalloc<unsigned int>(4);
  PDG_CUDA(cudaMemsetAsync(red.counter, 0, 4 * sizeof(unsigned int), st));
  d_S = dalloc<PcgScalars>(1);
  PDG_CUDA(cudaMallocHost(&h_S, sizeof(PcgScalars)));
  hist_cap = std::max(maxit_default, 16) + 2;
  alloc_history(hist_cap);
  d_perm = dupload(std::vector<int>(pr.perm.begin() + pr.cell_begin, pr.perm.begin() + pr.cell_end), st);

  // ---- state ----
  if (pr.device_assembly) {  // U0 / Y0 were projected into slot 0 on the device
    PDG_CUDA(cudaMemcpyAsync(d_U[1], d_U[0], n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    if (n_comp > 0)
      PDG_CUDA(cudaMemcpyAsync(d_Y[1], d_Y[0], n * n_comp * sizeof(double), cudaMemcpyDeviceToDevice, st));
  } else {
    PDG_CUDA(cudaMemcpyAsync(d_U[0], pr.U0.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
    PDG_CUDA(cudaMemcpyAsync(d_U[1], pr.U0.data(), n * sizeof(double), cudaMemcpyHostToDevice, st));
    if (n_comp > 0) {
      PDG_CUDA(cudaMemcpyAsync(d_Y[0], pr.Y0.data(), n * n_comp * sizeof(double), cudaMemcpyHostToDevice, st));
      PDG_CUDA(cudaMemcpyAsync(d_Y[1], pr.Y0.data(), n * n_comp * sizeof(double), cudaMemcpyHostToDevice, st));
    }
  }
  PDG_CUDA(cudaStreamSynchronize(st));
}

// M, A, K, M^-1, U0/Y0, E and this rank's K0 on the device (cuda/assemble.cu,
// same bits as the host assembly), then the coarse factorisation on the host
// (K0 is small) and the host copies the exports read (M, E; K when kept).
void DeviceSim::assemble_on_device() {
  Problem& pr = *P;
  const pdg_config& c = pr.cfg;
  std::vector<void*> tmp;
  auto up = [&](const auto& v) {
    auto* d = dupload(v, st);
    tmp.push_back(d);
    return d;
  };
  AsmArgs a{};
  a.ncells = ncells;
  a.cell0 = pr.cell_begin;
  a.b = b;
  a.p = pr.p;
  a.q = pr.q;
  a.bq = pr.two_level ? pr.bq : 0;
  a.n_comp = n_comp;
  a.ngl = static_cast<int>(pr.gl_x.size());
  a.ngs = static_cast<int>(pr.gs_x.size());
  a.init_kind = c.init_kind;
  a.two_level = pr.two_level ? 1 : 0;
  a.bbox = d_bbox;
  a.tri_ptr = d_tri_ptr;
  a.tri = d_tri;
  a.glx = up(pr.gl_x);
  a.glw = up(pr.gl_w);
  a.gsx = up(pr.gs_x);
  a.gsw = up(pr.gs_w);
  a.sigma = up(pr.sigma);
  a.fptr = up(pr.fptr);
  a.fent = up(pr.fent);
  a.fcell = up(pr.fcell);
  a.fgeo = up(pr.fgeo);
  a.kptr = d_ptr;
  a.kcol = d_col;
  a.kval = d_kval;
  a.M = d_M;
  a.Minv = d_Minv;
  a.U0 = d_U[0];
  a.Y0 = d_Y[0];
  a.am = c.C_m * c.chi_m;
  a.hb = 0.5 * c.dt;
  a.u_rest = c.u_rest;
  a.u_patch = c.u_patch;
  a.omega0[0] = c.omega0[0];
  a.omega0[1] = c.omega0[1];
  a.omega0_r2 = c.omega0_r2;
  for (int k = 0; k < 4; ++k) {
    a.ip[k] = c.init_params[k];
    a.y_rest[k] = pr.y_rest[k];
  }
  int* d_err = dalloc<int>(1);
  tmp.push_back(d_err);
  PDG_CUDA(cudaMemsetAsync(d_err, 0, sizeof(int), st));
  a.err = d_err;
  double* d_k0 = nullptr;
  if (pr.two_level) {
    a.abox = up(pr.abox);
    a.cell_label = up(pr.cell_label);
    a.cell_agg = d_cell_agg;
    a.agg_ptr = d_agg_ptr;
    a.agg_cells = d_agg_cells;
    a.E = d_E;
    a.k0ptr = up(pr.K0.ptr);
    a.k0col = up(pr.K0.col);
    d_k0 = dalloc<double>(pr.K0.val.size());
    tmp.push_back(d_k0);
    PDG_CUDA(cudaMemsetAsync(d_k0, 0, pr.K0.val.size() * sizeof(double), st));
    a.k0val = d_k0;
  }
  launch_assembly(a, st);
  int err = 0;
  PDG_CUDA(cudaMemcpyAsync(&err, d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
  PDG_CUDA(cudaStreamSynchronize(st));
  if (err & 1) throw SolverError("mass block is not positive definite");
  if (err & 2) throw SolverError("coarse embedding: cell mass not positive definite");
  const std::size_t b2 = static_cast<std::size_t>(b) * b;
  pr.M.resize(static_cast<std::size_t>(ncells) * b2);
  PDG_CUDA(cudaMemcpyAsync(pr.M.data(), d_M, pr.M.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (pr.keep_matrices) {
    pr.K.val.resize(static_cast<std::size_t>(pr.K.ptr[ncells]) * b2);
    PDG_CUDA(cudaMemcpyAsync(pr.K.val.data(), d_kval, pr.K.val.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  if (pr.two_level) {
    launch_k0(a, pr.n_agg, st);
    pr.E.resize(static_cast<std::size_t>(ncells) * b * pr.bq);
    PDG_CUDA(cudaMemcpyAsync(pr.E.data(), d_E, pr.E.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaMemcpyAsync(pr.K0.val.data(), d_k0, pr.K0.val.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
  }
  PDG_CUDA(cudaStreamSynchronize(st));
  for (void* p : tmp) cudaFree(p);
  if (pr.two_level && world == 1) finish_coarse(pr);
}

void DeviceSim::alloc_history(int cap) {
  if (d_hist) cudaFree(d_hist);
  d_hist = dalloc<double>(static_cast<std::size_t>(cap) * 3);
  hist_cap = cap;
  H.resid = d_hist;
  H.alpha = d_hist + cap;
  H.beta = d_hist + 2 * cap;
  for (auto& g : graphs) g.reset();
}

void DeviceSim::release_tasks() {
  void* ptrs[] = {d_tasks, d_fwd_units, d_bwd_units, d_nunit, d_part, d_task_child, d_fmat, d_hmat, d_ftiles, d_htiles,
                  d_row_dof, d_in_ptr, d_in_idx, d_ubuf, d_flags, d_ticket, d_yfwd, d_bmeta, d_broots, d_bdeps};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  d_yfwd = nullptr;
  d_bmeta = nullptr;
  d_broots = d_bdeps = nullptr;
  d_tasks = nullptr;
  d_nunit = d_task_child = d_in_ptr = d_flags = nullptr;
  d_fwd_units = d_bwd_units = nullptr;
  d_fmat = d_hmat = d_ubuf = d_part = nullptr;
  d_ftiles = d_htiles = nullptr;
  d_row_dof = d_in_idx = nullptr;
  d_ticket = nullptr;
}

namespace {

// Orders the sweep's work units by a simulated list schedule on `slots`
// resident CTAs: a unit is released when its task-level dependencies finish
// (forward: all children forward; backward: parent backward and own forward),
// the free CTA takes the released unit with the longest path to the end of
// the sweep, and tickets follow the simulated start times. A unit's
// dependencies start strictly earlier, so the ticket order stays topological
// (the persistent sweep's deadlock-freedom argument, sweep.cu).
std::vector<int> list_schedule(const Problem& pr, const std::vector<DevUnit>& units, int slots) {
  // cost model of the simulated schedule (ns); calibrating it to the traced
  // unit times (7 us fixed, 10 GB/s per CTA) changed nothing measurable
  // (profiles/r02l sched_*)
  constexpr double kFixed = 1500.0, kPerByte = 1.0 / 25.0, kPublish = 700.0;
  // only the individually scheduled supernodes take part: the bottom levels
  // (TaskDesc::bottom >= 0) run before (forward) and after (backward) them
  const int nt = static_cast<int>(pr.tasks.size());
  const int nn = nt, nu = static_cast<int>(units.size());
  auto node_of_unit = [&](const DevUnit& u) { return u.task; };
  auto cost = [&](const DevUnit& u) { return kFixed + kPerByte * u.bytes; };
  std::vector<std::vector<int>> pars(nn), kids(nn);
  std::vector<char> dense_root(nn, 0);
  for (int s = 0; s < nt; ++s) {
    const TaskDesc& t = pr.tasks[s];
    if (t.bottom >= 0) continue;
    dense_root[s] = static_cast<char>(t.root_dense);
    if (t.parent >= 0) {
      pars[s].push_back(t.parent);
      kids[t.parent].push_back(s);
    }
  }
  std::vector<double> cmax_f(nn, 0.0), cmax_b(nn, 0.0);
  std::vector<int> left_f(nn, 0), left_b(nn, 0);
  std::vector<std::vector<int>> units_f(nn), units_b(nn);
  for (int i = 0; i < nu; ++i) {
    const DevUnit& u = units[i];
    const int n = node_of_unit(u);
    if (u.dir == 0) {
      cmax_f[n] = std::max(cmax_f[n], cost(u));
      units_f[n].push_back(i);
    } else {
      cmax_b[n] = std::max(cmax_b[n], cost(u));
      units_b[n].push_back(i);
    }
  }
  // longest remaining path (bottom level) per node and direction; children
  // precede parents in task order
  std::vector<int> topo;
  topo.reserve(nn);
  for (int s = 0; s < nt; ++s)
    if (pr.tasks[s].bottom < 0) topo.push_back(s);
  std::vector<double> Lb(nn, 0.0), Lf(nn, 0.0);
  for (int n : topo) {
    double kid = 0.0;
    for (int c : kids[n]) kid = std::max(kid, Lb[c]);
    Lb[n] = cmax_b[n] + kPublish + kid;
  }
  for (auto it = topo.rbegin(); it != topo.rend(); ++it) {
    const int n = *it;
    double up = Lb[n];
    for (int p : pars[n]) up = std::max(up, Lf[p]);
    Lf[n] = cmax_f[n] + kPublish + up;
  }
  std::vector<double> prio(nu);
  for (int i = 0; i < nu; ++i) {
    const DevUnit& u = units[i];
    const int n = node_of_unit(u);
    prio[i] = u.dir == 0 ? Lf[n] - cmax_f[n] + cost(u) : Lb[n] - cmax_b[n] + cost(u);
  }
  // pending dependency counts per node and direction
  std::vector<int> dep_f(nn, 0), dep_b(nn, 0);
  for (int n : topo) {
    dep_f[n] = static_cast<int>(kids[n].size());
    dep_b[n] = 1 + static_cast<int>(pars[n].size());
    left_f[n] = static_cast<int>(units_f[n].size());
    left_b[n] = static_cast<int>(units_b[n].size());
  }
  using TI = std::pair<double, int>;
  std::priority_queue<TI, std::vector<TI>, std::greater<TI>> release, finish, cta;
  std::priority_queue<TI> ready;  // by priority
  std::vector<double> done_f(nn, 0.0), done_b(nn, 0.0), start(nu, 0.0);
  auto release_dir = [&](int n, bool fwd, double t) {
    for (int i : fwd ? units_f[n] : units_b[n]) release.push({t, i});
  };
  for (int n : topo)
    if (dep_f[n] == 0) release_dir(n, true, 0.0);
  for (int c = 0; c < slots; ++c) cta.push({0.0, c});
  std::function<void(int, double)> release_children_bwd = [&](int n, double r) {
    for (int c : kids[n])
      if (--dep_b[c] == 0) {
        release_dir(c, false, r);
        // a node without backward units (nothing to do) passes the release on
        if (units_b[c].empty()) release_children_bwd(c, r);
      }
  };
  auto complete = [&](int i, double t) {
    const DevUnit& u = units[i];
    const int n = node_of_unit(u);
    if (u.dir == 0) {
      done_f[n] = std::max(done_f[n], t);
      if (--left_f[n] > 0) return;
      const double r = done_f[n] + kPublish;
      for (int p : pars[n])
        if (--dep_f[p] == 0) release_dir(p, true, r);
      if (dense_root[n]) release_children_bwd(n, r);  // x_S is final after the forward
      else if (--dep_b[n] == 0) {
        release_dir(n, false, r);
        if (units_b[n].empty()) release_children_bwd(n, r);
      }
    } else {
      done_b[n] = std::max(done_b[n], t);
      if (--left_b[n] > 0) return;
      release_children_bwd(n, done_b[n] + kPublish);
    }
  };
  int placed = 0;
  std::vector<int> order;
  order.reserve(nu);
  while (placed < nu) {
    auto [t, c] = cta.top();
    cta.pop();
    while (!finish.empty() && finish.top().first <= t) {
      complete(finish.top().second, finish.top().first);
      finish.pop();
    }
    while (!release.empty() && release.top().first <= t) {
      ready.push({prio[release.top().second], release.top().second});
      release.pop();
    }
    if (ready.empty()) {
      // idle until the next completion or release
      double nxt = 1e300;
      if (!finish.empty()) nxt = std::min(nxt, finish.top().first);
      if (!release.empty()) nxt = std::min(nxt, release.top().first);
      if (nxt >= 1e300) throw SolverError("schwarz: sweep schedule has a dependency cycle");
      cta.push({std::max(nxt, t), c});
      continue;
    }
    const int i = ready.top().second;
    ready.pop();
    start[i] = t;
    order.push_back(i);
    ++placed;
    const double f = t + cost(units[i]);
    finish.push({f, i});
    cta.push({f, c});
  }
  return order;
}

}  // namespace

void DeviceSim::upload_tasks() {
  release_tasks();
  const Problem& pr = *P;
  n_tasks = static_cast<int>(pr.tasks.size());
  std::vector<DevTask> t(n_tasks);
  int wmax = 0, nrmax = 0;
  for (int i = 0; i < n_tasks; ++i) {
    const TaskDesc& s = pr.tasks[i];
    t[i] = DevTask{s.coarse, s.bs, s.w, s.nr, s.dof0, s.ubuf_off, s.f_tile0, s.f_ntile, s.h_tile0,
                   s.h_ntile, s.rows_off, s.in_off, s.parent, s.child_off, s.n_child, s.root_dense};
    wmax = std::max(wmax, s.w);
    nrmax = std::max(nrmax, s.nr);
  }
  // topological ticket orders: forward by height (children first), backward
  // by depth (parents first); larger supernodes first within a level
  std::vector<int> fo(n_tasks), bo(n_tasks);
  for (int i = 0; i < n_tasks; ++i) fo[i] = bo[i] = i;
  std::stable_sort(fo.begin(), fo.end(), [&](int a, int c) {
    const auto &A = pr.tasks[a], &C = pr.tasks[c];
    if (A.height != C.height) return A.height < C.height;
    return A.w * (A.w + A.nr) > C.w * (C.w + C.nr);
  });
  std::stable_sort(bo.begin(), bo.end(), [&](int a, int c) {
    const auto &A = pr.tasks[a], &C = pr.tasks[c];
    if (A.depth != C.depth) return A.depth < C.depth;
    return A.w * (A.w + A.nr) > C.w * (C.w + C.nr);
  });
  (void)wmax;
  (void)nrmax;
  d_tasks = dupload(t, st);
  // Work units of <= kUnitBytes of panel: runs of whole tiles, or column
  // chunks of one wide tile (partials reduced by the last chunk, sweep.cu).
  // unit size (panel bytes per CTA visit): a unit's fixed cost (~5 us of
  // dependent round trips) dominates below ~32 KB, while the separators near
  // the roots are the critical path; leaves (height 0) and the rest can use
  // different sizes. PDG_UNIT_KB / PDG_LEAF_KB override.
  auto env_kb = [](const char* k, int d) {
    const char* e = std::getenv(k);
    return 1024LL * (e ? std::max(2, std::atoi(e)) : d);
  };
  // Default: ~20 units per resident CTA per sweep, clamped to [44, 128] KB.
  // Small problems (config2: 351 KB of panel per CTA) are critical-path
  // bound and want small units (44 KB was the best of a 16-96 KB scan);
  // large ones (config3 p=3: 1.9 MB per CTA) are bandwidth bound and want
  // the per-unit round trips amortised over more bytes (88 KB: +8.5%).
  long long panel_bytes = 0;
  for (const auto& tl : pr.ftiles) panel_bytes += 8LL * tl.ncol * tl.stride;
  for (const auto& tl : pr.htiles) panel_bytes += 8LL * tl.ncol * tl.stride;
  int sms_u = 148, dev_u = 0;
  PDG_CUDA(cudaGetDevice(&dev_u));
  PDG_CUDA(cudaDeviceGetAttribute(&sms_u, cudaDevAttrMultiProcessorCount, dev_u));
  // up to 128 KB: config4 sweep 6.33 ms vs 6.51 ms at 88 KB (profiles/r02e)
  const int max_kb = std::getenv("PDG_UNIT_MAX_KB") ? std::max(44, std::atoi(std::getenv("PDG_UNIT_MAX_KB"))) : 128;
  const int auto_kb = static_cast<int>(std::clamp<long long>(panel_bytes / (20LL * sms_u * 8) / 1024, 44, max_kb));
  const long long kUnitBytes = env_kb("PDG_UNIT_KB", auto_kb);
  const long long kLeafBytes = env_kb("PDG_LEAF_KB", static_cast<int>(kUnitBytes / 1024));
  int n_parts = 0, n_tile_ctr = 0;
  long long max_panel = 0, max_in = 0;
  // dependency counters a unit waits on (sweep.cu): forward = children's
  // forward tiles, backward = parent's backward tiles (roots: own forward)
  const int nt_flag = std::max(n_tasks, 1);
  auto set_deps = [&](DevUnit& u, int tk, bool fwd) {
    const TaskDesc& s = pr.tasks[tk];
    u.own_fwd = -1;
    u.own_need = 0;
    if (fwd) {
      u.n_dep = s.n_child;
      for (int k = 0; k < s.n_child && k < 2; ++k) {
        const int c = pr.task_child[s.child_off + k];
        u.dep[k] = c;
        u.need[k] = pr.tasks[c].f_ntile;
      }
    } else if (s.parent >= 0) {
      // the parent's x_S: its backward tiles, or a dense root's forward ones
      const TaskDesc& ps = pr.tasks[s.parent];
      u.n_dep = 1;
      u.dep[0] = ps.root_dense ? s.parent : nt_flag + s.parent;
      u.need[0] = ps.root_dense ? ps.f_ntile : ps.h_ntile;
      u.own_fwd = tk;
      u.own_need = s.f_ntile;
    } else {
      u.n_dep = 1;
      u.dep[0] = tk;
      u.need[0] = s.f_ntile;
    }
  };
  auto make_units = [&](const std::vector<int>& order, bool fwd, std::vector<DevUnit>& units) {
    for (int tk : order) {
      const TaskDesc& s = pr.tasks[tk];
      if (s.bottom >= 0) continue;  // a bottom-level supernode: solved in level chunks (below)
      const int t0 = fwd ? s.f_tile0 : s.h_tile0, nt = fwd ? s.f_ntile : s.h_ntile;
      const auto& tiles = fwd ? pr.ftiles : pr.htiles;
      auto tbytes = [&](int r) { return 8LL * tiles[t0 + r].ncol * tiles[t0 + r].stride; };
      const long long kUnit = s.height == 0 ? kLeafBytes : kUnitBytes;
      // input column range and (forward) its incoming-update list, so the
      // kernel stages without dependent metadata loads
      auto set_cols = [&](DevUnit& u, int lo, int hi) {
        u.col_lo = lo;
        u.col_hi = hi;
        u.in_e0 = u.in_n = 0;
        if (fwd) {
          const int c_lo = lo / s.bs, c_hi = (hi + s.bs - 1) / s.bs;
          u.in_e0 = pr.in_ptr[s.in_off + c_lo];
          u.in_n = pr.in_ptr[s.in_off + c_hi] - u.in_e0;
        }
      };
      int b0 = 0;
      while (b0 < nt) {
        const auto& tb = tiles[t0 + b0];
        if (tbytes(b0) > kUnit) {
          // balanced column chunks of an even number of columns (no small
          // remainder chunk paying a whole unit's fixed cost)
          const long long max_cols = std::max<long long>(2, (kUnit / (8LL * tb.stride)) & ~1LL);
          const int nch0 = static_cast<int>((tb.ncol + max_cols - 1) / max_cols);
          long long cols = (tb.ncol + nch0 - 1) / nch0;
          cols = std::max<long long>(2, (cols + 1) & ~1LL);
          const int nch = static_cast<int>((tb.ncol + cols - 1) / cols);
          for (int c = 0; c < nch; ++c) {
            const int c0 = static_cast<int>(c * cols), c1 = std::min<int>(tb.ncol, static_cast<int>((c + 1) * cols));
            DevUnit u{};
            u.task = tk;
            u.tile_begin = b0;
            u.tile_end = b0 + 1;
            u.c0 = c0;
            u.c1 = c1;
            u.chunk = c;
            u.nchunk = nch;
            u.part_base = n_parts;
            u.tile_ctr = n_tile_ctr;
            u.dir = fwd ? 0 : 1;
            u.src_off = tb.off + static_cast<long long>(c0) * tb.stride;
            u.bytes = static_cast<int>(8LL * (c1 - c0) * tb.stride);
            max_panel = std::max<long long>(max_panel, u.bytes);
            max_in = std::max<long long>(max_in, c1 - c0);
            set_cols(u, tb.col0 + c0, tb.col0 + c1);
            set_deps(u, tk, fwd);
            units.push_back(u);
          }
          n_parts += nch;
          ++n_tile_ctr;
          ++b0;
          continue;
        }
        long long bytes = 0;
        int e = b0;
        while (e < nt && tbytes(e) <= kUnit && (e == b0 || bytes + tbytes(e) <= kUnit)) {
          bytes += tbytes(e);
          ++e;
        }
        DevUnit u{};
        u.task = tk;
        u.tile_begin = b0;
        u.tile_end = e;
        u.nchunk = 1;
        u.dir = fwd ? 0 : 1;
        u.src_off = tb.off;
        u.bytes = static_cast<int>(bytes);
        int lo = tiles[t0 + b0].col0, hi = 0;
        for (int r = b0; r < e; ++r) hi = std::max(hi, tiles[t0 + r].col0 + tiles[t0 + r].ncol);
        max_panel = std::max(max_panel, bytes);
        max_in = std::max<long long>(max_in, hi - lo);
        set_cols(u, lo, hi);
        set_deps(u, tk, fwd);
        units.push_back(u);
        b0 = e;
      }
    }
  };
  std::vector<DevUnit> fu, bu;
  make_units(fo, true, fu);
  make_units(bo, false, bu);
  // bottom levels: one unit per level chunk (sweep.cu run_chunk). A level
  // waits for the previous one through one counter per level and direction
  // (after the task counters in d_flags); forward chunks also publish the
  // counters of their supernodes that have an individually scheduled parent,
  // backward chunks wait for the distinct such parents (their backward tiles,
  // or a dense root's forward ones). The first backward level waits for the
  // last forward one (a whole tree inside the bottom levels has no such parent).
  std::vector<int2> broots, bdeps;
  std::vector<DevUnit> cfu, cbu;
  const int nslots = static_cast<int>(pr.level_chunks[0].size());  // (group, level) counters per direction
  const int lev_flag0 = 2 * nt_flag;
  for (std::size_t ci = 0; ci < pr.chunks.size(); ++ci) {
    const LevelChunk& C = pr.chunks[ci];
    DevUnit u{};
    u.task = C.first_task;
    u.tile_begin = static_cast<int>(ci);
    u.nchunk = 0;
    u.dir = C.dir;
    u.src_off = C.src_off;
    u.bytes = C.bytes;
    u.in_e0 = C.meta_off;
    u.in_n = C.meta_n;
    // the counters this chunk adds to: its global level's and (grouped levels) its group's
    u.own_fwd = lev_flag0 + C.dir * nslots + C.gslot;
    u.chunk = C.slot >= 0 ? lev_flag0 + C.dir * nslots + C.slot : -1;
    if (C.dep_slot >= 0) {
      u.n_dep = 1;
      u.dep[0] = lev_flag0 + C.dep_dir * nslots + C.dep_slot;
      u.need[0] = pr.level_chunks[C.dep_dir][C.dep_slot];
    }
    if (C.dir == 0) {
      u.part_base = static_cast<int>(broots.size());
      u.tile_ctr = C.n_root;
      for (int k = 0; k < C.n_root; ++k) {
        const int r = pr.chunk_roots[C.root_off + k];
        broots.push_back(make_int2(r, pr.tasks[r].f_ntile));
      }
    } else {
      u.c0 = static_cast<int>(bdeps.size());
      u.c1 = C.n_par;
      for (int k = 0; k < C.n_par; ++k) {
        const int p = pr.chunk_parents[C.par_off + k];
        const TaskDesc& ps = pr.tasks[p];
        bdeps.push_back(ps.root_dense ? make_int2(p, ps.f_ntile) : make_int2(nt_flag + p, ps.h_ntile));
      }
    }
    max_in = std::max<long long>(max_in, C.xneed);
    (C.dir ? cbu : cfu).push_back(u);
  }
  d_bmeta = dupload(pr.bmeta, st);
  d_broots = dupload(broots, st);
  d_bdeps = dupload(bdeps, st);
  // one ticket space (sweep.cu): forward and backward units in the order of a
  // simulated list schedule (critical path first)
  n_units_f = static_cast<int>(fu.size());
  n_units_b = static_cast<int>(bu.size());
  fu.insert(fu.end(), bu.begin(), bu.end());
  // panels stream from L2 (bulk-prefetched); smem holds partial sums + inputs
  // partial sums + the unit's input buffer (sweep.cu)
  sweep_xcap = static_cast<int>(max_in) + 2;
  // 64-thread CTAs (twice as many resident) for large problems with small
  // blocks (b <= 6): config5 p=2 sweep 2.32 vs 2.64 ms; 128 everywhere else
  // (config4 6.35 vs 7.16 ms, config2 0.098 vs 0.129 ms; profiles/r02l)
  // With bottom levels (level chunks: one warp per tile) 128 again: config5
  // p=2 2.22 ms vs 3.29 ms at 64 (profiles/r02aa).
  sweep_threads = (pr.b <= 6 && pr.n_global_dofs() / std::max(1, pr.cfg.world) >= 2000000 && pr.chunks.empty()) ? 64 : 128;
  if (const char* e = std::getenv("PDG_SWEEP_THREADS")) sweep_threads = std::atoi(e) == 64 ? 64 : 128;
  smem_fwd = smem_bwd = sweep_smem_bytes(sweep_xcap, sweep_threads);
  if (smem_fwd > 220 * 1024) throw SolverError("schwarz: sweep unit does not fit in shared memory");
  if (smem_fwd > 48 * 1024) set_sweep_smem(smem_fwd);
  {
    int sms = 148, dev = 0;
    PDG_CUDA(cudaGetDevice(&dev));
    PDG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const std::vector<int> perm = list_schedule(pr, fu, sms * sweep_ctas_per_sm(smem_fwd, sweep_threads));
    // tickets: forward bottom levels, the scheduled supernodes, backward bottom levels
    std::vector<DevUnit> o;
    o.reserve(fu.size() + cfu.size() + cbu.size());
    o.insert(o.end(), cfu.begin(), cfu.end());
    for (std::size_t i = 0; i < perm.size(); ++i) o.push_back(fu[perm[i]]);
    o.insert(o.end(), cbu.begin(), cbu.end());
    fu.swap(o);
    n_units_f += static_cast<int>(cfu.size());
    n_units_b += static_cast<int>(cbu.size());
  }
  h_units = fu;
  d_fwd_units = dupload(fu, st);
  n_tile_ctrs = std::max(n_tile_ctr, 1);
  // chunk counters of split tiles; like the task counters they are monotone
  // across sweeps (sweep.cu), so they are zeroed once here
  d_nunit = dalloc<int>(n_tile_ctrs);
  PDG_CUDA(cudaMemsetAsync(d_nunit, 0, n_tile_ctrs * sizeof(int), st));
  d_part = dalloc<double>(static_cast<std::size_t>(std::max(n_parts, 1)) * 32);
  (void)max_panel;
  d_task_child = dupload(pr.task_child, st);
  std::vector<DevTile> ft(pr.ftiles.size()), ht(pr.htiles.size());
  for (std::size_t i = 0; i < ft.size(); ++i)
    ft[i] = DevTile{pr.ftiles[i].off, pr.ftiles[i].ncol, pr.ftiles[i].col0, pr.ftiles[i].rows, pr.ftiles[i].stride};
  for (std::size_t i = 0; i < ht.size(); ++i)
    ht[i] = DevTile{pr.htiles[i].off, pr.htiles[i].ncol, pr.htiles[i].col0, pr.htiles[i].rows, pr.htiles[i].stride};
  d_ftiles = dupload(ft, st);
  d_htiles = dupload(ht, st);
  build_panels();  // F and H from the factor values (panels.cu)
  std::vector<long long> rd(pr.row_dof.begin(), pr.row_dof.end());
  d_row_dof = dupload(rd, st);
  d_in_ptr = dupload(pr.in_ptr, st);
  std::vector<long long> ii(pr.in_idx.begin(), pr.in_idx.end());
  d_in_idx = dupload(ii, st);
  d_ubuf = dalloc<double>(std::max<std::int64_t>(pr.ubuf_size, 1));
  d_yfwd = dalloc<double>(n + static_cast<std::size_t>(pr.two_level ? pr.n_agg * pr.bq : 0));
  // tile counters per task and direction, then one counter per bottom level and direction
  const std::size_t n_flags = 2 * static_cast<std::size_t>(std::max(n_tasks, 1)) + 2 * pr.level_chunks[0].size();
  d_flags = dalloc<int>(n_flags);
  PDG_CUDA(cudaMemsetAsync(d_flags, 0, n_flags * sizeof(int), st));
  // [0] next ticket, [1] sweep number, [2] CTAs finished (sweep.cu)
  d_ticket = dalloc<unsigned int>(4);
  PDG_CUDA(cudaMemsetAsync(d_ticket, 0, 4 * sizeof(unsigned int), st));
  if (!d_live) {
    d_live = dalloc<unsigned long long>(3);
    PDG_CUDA(cudaMemsetAsync(d_live, 0, 3 * sizeof(unsigned long long), st));
  }
  PDG_CUDA(cudaStreamSynchronize(st));
  panel_values = static_cast<long long>(pr.fmat_len + pr.hmat_len);
  // one rank: the panels live on the device from now on (config 4: ~20 GB of
  // factor values back to the host); several ranks re-pack after the coarse
  // all-reduce
  if (pr.cfg.world == 1) {
    Problem& mp = *P;
    std::vector<double>().swap(mp.lval);
    std::vector<Problem::FactorSn>().swap(mp.fsn);
    std::vector<Problem::FactorUpd>().swap(mp.fupd);
    std::vector<int>().swap(mp.frows);
    std::vector<int>().swap(mp.fmap);
  }
}

DeviceSim::~DeviceSim() {
  for (auto& g : graphs) g.reset();
  void* ptrs[] = {d_ptr, d_col, d_kval, d_M, d_Minv, d_U[0], d_U[1], d_x, d_p, d_r, d_z, d_q,
                  d_rhs, d_ion, d_tmp, d_tmp2, d_Y[0], d_Y[1], d_E, d_cell_agg, d_agg_ptr,
                  d_agg_cells, d_r0, d_y0, d_tasks, d_fwd_units, d_bwd_units, d_nunit, d_task_child,
                  d_fmat, d_hmat, d_ftiles, d_htiles, d_row_dof, d_in_ptr, d_in_idx, d_ubuf, d_flags, d_ticket, d_bmeta, d_broots, d_bdeps, d_bbox,
                  d_tri_ptr, d_tri, d_ionflags, red.partial, red.counter, d_S, d_hist, d_perm,
                  d_Y[2], d_scratch, d_send_cells, d_sendbuf, d_dot_local, d_dot_global, d_stage, d_chunk_ptr, d_node_chunk_ptr, d_r0part,
                  d_live, d_area, d_means, d_rows_int, d_rows_bnd};
  cudaEventDestroy(ev_t0);
  cudaEventDestroy(ev_t1);
  comm_destroy();
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (h_S) cudaFreeHost(h_S);
  if (st) cudaStreamDestroy(st);
  if (st_comm) cudaStreamDestroy(st_comm);
  if (ev_pack) cudaEventDestroy(ev_pack);
  if (ev_halo) cudaEventDestroy(ev_halo);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  cudaEventDestroy(ev2);
}

ReduceCtx DeviceSim::rctx(int finish, double* out) {
  if (!out) out = d_scratch;
  ReduceCtx rc;
  rc.red = red;
  rc.S = d_S;
  rc.H = H;
  rc.out = out;
  rc.finish = finish;
  return rc;
}

SweepArgs DeviceSim::sweep_args(bool, const double* r, double* z, const PcgScalars* S) {
  SweepArgs a;
  static const char* pf = std::getenv("PDG_SWEEP_PREFETCH");
  a.prefetch = pf ? std::atoi(pf) : 3;  // bit 0: L2 bulk prefetch, bit 1: evict-first panel loads
  a.threads = sweep_threads;
  a.tasks = d_tasks;
  a.units = d_fwd_units;
  a.n_units_f = n_units_f;
  a.n_units = n_units_f + n_units_b;
  a.tile_ctr = d_nunit;
  a.part = d_part;
  a.n_tasks = std::max(n_tasks, 1);
  a.ticket = d_ticket;
  a.flags = d_flags;
  a.task_child = d_task_child;
  a.bmeta = d_bmeta;
  a.broots = d_broots;
  a.bdeps = d_bdeps;
  a.fmat = d_fmat;
  a.hmat = d_hmat;
  a.ftiles = d_ftiles;
  a.htiles = d_htiles;
  a.row_dof = d_row_dof;
  a.in_ptr = d_in_ptr;
  a.in_idx = d_in_idx;
  a.ubuf = d_ubuf;
  a.r = r;
  a.z = z;
  a.r0 = d_r0;
  a.y0 = d_y0;
  a.yf = d_yfwd;
  a.yc = d_yfwd + n;
  // one rank: the coarse forward sums r0 from the restriction chunks itself;
  // several ranks: r0 is combined and all-reduced first
  a.r0part = (world == 1 && P->two_level) ? d_r0part : nullptr;
  a.node_chunk_ptr = d_node_chunk_ptr;
  a.S = S;
  a.epoch = reinterpret_cast<int*>(d_ticket) + 1;
  a.xcap = sweep_xcap;
  a.live = d_live;
  a.trace = d_trace;
  // diagnostics for traced sweeps only (results become wrong): bit 4 = level
  // chunks skip their scattered gather loads, bit 5 = skip their stores
  if (d_trace)
    if (const char* dbg = std::getenv("PDG_CHUNK_DEBUG")) a.prefetch |= std::atoi(dbg) << 4;
  return a;
}

// z = B r with the r.z reduction finished as `finish`. `S_honor` makes every
// kernel a no-op once the solve has stopped.
void DeviceSim::precond_apply(const double* r, double* z, int finish, bool honor, bool restricted) {
  const Problem& pr = *P;
  const PcgScalars* Sh = honor ? d_S : nullptr;
  if (!use_pc()) {
    // plain CG: z aliases r (krylov.cpp:39-42: out = in)
    launch_prolong_dot(b, 0, ncells, nullptr, nullptr, nullptr, r, const_cast<double*>(r), red_for(finish), st);
    after_reduce(finish, honor);
    return;
  }
  if (pr.two_level && !restricted) {
    // restricted: r0 is already in place (single rank: the chunk partials of
    // the fused update; several ranks: combined and all-reduced with ||r||^2)
    launch_restrict(b, bq, n_chunks, d_chunk_ptr, d_agg_cells, d_E, r, d_r0part, Sh, st);
    if (world > 1) {
      launch_restrict_combine(bq, pr.n_agg, d_node_chunk_ptr, d_r0part, d_r0, Sh, st);
      coarse_reduce_hook();
    }
  }
  launch_sweep(sweep_args(true, r, z, Sh), smem_fwd, st);
  if (pr.two_level && chunks_contiguous)
    launch_prolong_dot_tma(b, bq, n_chunks, max_chunk_cells, d_chunk_ptr, d_agg_cells, d_cell_agg, d_E, d_y0, r, z,
                           red_for(finish), st);
  else
    launch_prolong_dot(b, bq, ncells, d_E, d_cell_agg, d_y0, r, z, red_for(finish), st);
  after_reduce(finish, honor);
}

double* DeviceSim::z_of(double* r) { return use_pc() ? d_z : r; }

ReduceCtx DeviceSim::red_for(int finish) {
  if (world == 1 || finish == kFinNone || finish == kFinStore) return rctx(finish);
  return rctx(kFinStore, d_dot_local);
}

// Multi-rank: sum the per-rank partial over NCCL, then apply the finish on
// every rank (identical inputs, so every rank takes identical decisions).
void DeviceSim::after_reduce(int finish, bool honor) {
  if (world == 1 || finish == kFinNone || finish == kFinStore) return;
  comm_allreduce(d_dot_local, d_dot_global, 1);
  launch_finish(rctx(finish), d_dot_global, honor, st);
}

// p-halo for the SpMV: pack the cells each peer needs, grouped send/recv
// straight into the halo tail of v.
void DeviceSim::halo_exchange(double* v) {
  if (world == 1 || halo_peers.empty()) return;
  for (const HaloPeer& h : halo_peers)
    launch_pack(v, d_send_cells + h.send_off, h.send_count, b, d_sendbuf + static_cast<long long>(h.send_off) * b, st);
  comm_exchange(v, st);
}

// every rank solves the coarse problem redundantly on the summed r0 (C3)
void DeviceSim::coarse_reduce_hook() {
  if (world == 1) return;
  comm_allreduce(d_r0, d_r0, static_cast<long long>(P->n_agg) * P->bq);
}
void DeviceSim::dot_reduce_hook(int) {}

// The body of one PCG iteration (krylov.cpp:49-73), every kernel gated on S->stop.
void DeviceSim::record_iteration() {
  double* p = d_p;
  if (world > 1 && !halo_peers.empty()) {
    spmv_overlapped(d_p, d_q);  // p.q partial -> d_dot_local, all-reduced below
  } else {
    halo_exchange(d_p);
    launch_spmv(b, ncells, d_ptr, d_col, d_kval, d_p, d_q, d_p, red_for(kFinPq), true, st);
  }
  after_reduce(kFinPq, true);
  if (world > 1) {
    // Several ranks: the update stores this rank's ||r||^2 partial behind r0,
    // the restriction runs speculatively (gated kernels, before the
    // convergence test), and ONE all-reduce carries [r0 ; ||r||^2]. Per
    // iteration: the p halo + three all-reduces (p.q, [r0 ; r.r], r.z).
    const bool coarse = use_pc() && P->two_level;
    const long long nr0 = coarse ? static_cast<long long>(P->n_agg) * P->bq : 0;
    double* rr = coarse ? d_r0 + nr0 : d_dot_local;
    launch_update(n, d_x, d_r, p, d_q, rctx(kFinStore, rr), st);
    if (coarse) {
      launch_restrict(b, bq, n_chunks, d_chunk_ptr, d_agg_cells, d_E, d_r, d_r0part, d_S, st);
      launch_restrict_combine(bq, P->n_agg, d_node_chunk_ptr, d_r0part, d_r0, d_S, st);
      comm_allreduce(d_r0, d_r0, nr0 + 1);
      launch_finish(rctx(kFinRr), rr, true, st);
    } else {
      comm_allreduce(d_dot_local, d_dot_global, 1);
      launch_finish(rctx(kFinRr), d_dot_global, true, st);
    }
    precond_apply(d_r, z_of(d_r), kFinRz, true, coarse);
    launch_pupdate(n, d_p, z_of(d_r), d_S, false, st);
    return;
  }
  const bool fuse = use_pc() && P->two_level && world == 1;
  if (fuse && chunks_contiguous)
    launch_update_restrict_tma(b, bq, n_chunks, max_chunk_cells, d_chunk_ptr, d_agg_cells, d_E, d_x, d_r, p, d_q,
                               d_r0part, red_for(kFinRr), st);
  else if (fuse)
    launch_update_restrict(b, bq, n_chunks, d_chunk_ptr, d_agg_cells, d_E, d_x, d_r, p, d_q, d_r0part,
                           red_for(kFinRr), st);
  else
    launch_update(n, d_x, d_r, p, d_q, red_for(kFinRr), st);
  after_reduce(kFinRr, true);
  precond_apply(d_r, z_of(d_r), kFinRz, true, fuse);
  launch_pupdate(n, d_p, z_of(d_r), d_S, false, st);
}

// PCG after r = b - K x0 and denom are in place: z = B r, rho, p = z, then
// the while loop.
void DeviceSim::record_solve_tail() {
  precond_apply(d_r, z_of(d_r), kFinRzInit, true);
  launch_pupdate(n, d_p, z_of(d_r), d_S, true, st);
}

DeviceSim::Graph::~Graph() { reset(); }
void DeviceSim::Graph::reset() {
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  exec = nullptr;
  graph = nullptr;
}

void DeviceSim::build_solve_graph(Graph& g) {
  g.reset();
  PDG_CUDA(cudaGraphCreate(&g.graph, 0));
  // tail (z, rho, p) captured into the outer graph
  cudaGraph_t tail = nullptr;
  PDG_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  record_solve_tail();
  PDG_CUDA(cudaStreamEndCapture(st, &tail));
  cudaGraphNode_t tail_node;
  PDG_CUDA(cudaGraphAddChildGraphNode(&tail_node, g.graph, nullptr, 0, tail));
  cudaGraphDestroy(tail);

  cudaGraphConditionalHandle handle;
  PDG_CUDA(cudaGraphConditionalHandleCreate(&handle, g.graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cond_node;
  PDG_CUDA(cudaGraphAddNode(&cond_node, g.graph, &tail_node, 1, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  PDG_CUDA(cudaStreamBeginCaptureToGraph(st, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  record_iteration();
  launch_pdl(set_condition_kernel, 1, 1, 0, st, handle, d_S);
  PDG_CUDA(cudaStreamEndCapture(st, &body));
  PDG_CUDA(cudaGraphInstantiate(&g.exec, g.graph, 0));
}

void DeviceSim::reset_scalars(double tol, int maxit) {
  std::memset(h_S, 0, sizeof(PcgScalars));
  h_S->tol = tol;
  h_S->maxit = maxit;
  PDG_CUDA(cudaMemcpyAsync(d_S, h_S, sizeof(PcgScalars), cudaMemcpyHostToDevice, st));
}

// Runs the device loop on (d_r, d_x) prepared by the caller; fills rep.
void DeviceSim::run_solve(int maxit, PcgResult& res) {
  if (maxit + 2 > hist_cap) alloc_history(maxit + 2);
  // PDG_NO_GRAPH=1 runs the host-driven loop (kernels inside conditional
  // graphs are invisible to ncu)
  static const bool no_graph = std::getenv("PDG_NO_GRAPH") && std::getenv("PDG_NO_GRAPH")[0] == '1';
  if (world == 1 && !no_graph) {
    Graph& g = graphs[use_pc() ? 1 : 0];
    if (!g.exec) build_solve_graph(g);
    PDG_CUDA(cudaGraphLaunch(g.exec, st));
    PDG_CUDA(cudaMemcpyAsync(h_S, d_S, sizeof(PcgScalars), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
  } else {
    // multi-rank: host-driven loop (NCCL calls stay outside conditional
    // graphs); every rank sees the same all-reduced scalars, so all ranks
    // stop after the same iteration and issue the same collectives.
    if (world > 1 && !transport) throw SolverError("multi-rank simulation: call pdg_sim_attach_comm first");
    record_solve_tail();
    constexpr int kPoll = 4;
    for (int it = 0; it < maxit;) {
      for (int j = 0; j < kPoll && it < maxit; ++j, ++it) record_iteration();
      PDG_CUDA(cudaMemcpyAsync(h_S, d_S, sizeof(PcgScalars), cudaMemcpyDeviceToHost, st));
      PDG_CUDA(cudaStreamSynchronize(st));
      if (h_S->stop) break;
    }
  }
  res.iterations = h_S->iter;
  res.converged = h_S->converged;
  res.error = h_S->error;
  res.denom = h_S->denom;
  const int m = h_S->iter;
  res.resid.resize(std::max(m, 1));
  res.alpha.resize(m);
  res.beta.resize(m);
  if (h_S->denom == 0.0 && h_S->error == 0) {
    res.resid.assign(1, 0.0);
    res.alpha.clear();
    res.beta.clear();
    return;
  }
  if (m > 0) {
    PDG_CUDA(cudaMemcpyAsync(res.resid.data(), H.resid, m * sizeof(double), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaMemcpyAsync(res.alpha.data(), H.alpha, m * sizeof(double), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaMemcpyAsync(res.beta.data(), H.beta, m * sizeof(double), cudaMemcpyDeviceToHost, st));
    PDG_CUDA(cudaStreamSynchronize(st));
  } else {
    res.resid.clear();
  }
  // betas recorded so far: one per completed precond apply after an iteration
  int nb = m;
  if (res.converged) nb = m - 1;
  if (res.error != 0) nb = std::max(0, m - 1);
  res.beta.resize(std::max(nb, 0));
  if (res.error) throw SolverError(pcg_error_message(res.error));
}

// pcg_solve(K, b, precond, tol, maxit, x0) on internal-order device vectors.
PcgResult DeviceSim::pcg(const double* d_b, const double* d_x0, double* d_xout, double tol, int maxit) {
  if (!(tol > 0.0 && tol < 1.0)) throw SolverError("pcg: tol must lie in (0, 1)");
  if (maxit <= 0) maxit = maxit_default;
  PcgResult res;
  reset_scalars(tol, maxit);
  if (d_x0 != d_x) PDG_CUDA(cudaMemcpyAsync(d_x, d_x0, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  halo_exchange(d_x);
  launch_residual(b, ncells, d_ptr, d_col, d_kval, d_x, d_b, d_r, red_for(kFinDenom), st);
  after_reduce(kFinDenom, false);
  run_solve(maxit, res);
  if (d_xout != d_x) PDG_CUDA(cudaMemcpyAsync(d_xout, d_x, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  PDG_CUDA(cudaStreamSynchronize(st));
  return res;
}

void DeviceSim::apply_K(const double* x, double* y) {
  PDG_CUDA(cudaMemcpyAsync(d_tmp, x, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  halo_exchange(d_tmp);
  launch_spmv(b, ncells, d_ptr, d_col, d_kval, d_tmp, y, nullptr, rctx(kFinNone), false, st);
  PDG_CUDA(cudaStreamSynchronize(st));
}

void DeviceSim::apply_precond(const double* r, double* z) {
  reset_scalars(0.5, 1);
  // r.z is computed into scratch; z may not alias r
  PDG_CUDA(cudaMemsetAsync(z, 0, n * sizeof(double), st));
  if (!use_pc()) {
    PDG_CUDA(cudaMemcpyAsync(z, r, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  } else {
    precond_apply(r, z, kFinStore, false);  // r.z -> scratch
  }
  PDG_CUDA(cudaStreamSynchronize(st));
}

// Simulation::step (timestepper.cpp:144-200)
// ionic terms, stimulus and Y update of one step (ionics.cpp:61-113,
// timestepper.cpp:128-186) on the current state
IonicArgs DeviceSim::ionic_args(bool has_prev) const {
  const Problem& pr = *P;
  const pdg_config& c = pr.cfg;
  IonicArgs a{};
  a.b = b;
  a.p = pr.p;
  a.ncells = ncells;
  a.n_comp = pr.n_comp;
  a.ngl = static_cast<int>(pr.gl_x.size());
  a.has_prev = has_prev ? 1 : 0;
  a.model = c.ionic_model;
  a.stim = c.stim_kind;
  a.bbox = d_bbox;
  a.tri_ptr = d_tri_ptr;
  a.tri = d_tri;
  a.U = d_U[0];
  a.Up = d_U[1];
  a.Y = d_Y[0];
  a.Yp = d_Y[1];
  a.Ynext = d_Y[2];
  a.Minv = d_Minv;
  a.ion = d_ion;
  a.n = n;
  a.chi = c.chi_m;
  a.dt = c.dt;
  a.t_mid = t + 0.5 * c.dt;
  std::memcpy(a.fhn, c.fhn, sizeof a.fhn);
  std::memcpy(a.bc, c.bc, sizeof a.bc);
  if (c.ionic_model == PDG_IONIC_BARRETO_CRESSMAN) {
    a.ubounds[0] = bc::kUMin;
    a.ubounds[1] = bc::kUMax;
  } else {
    a.ubounds[0] = c.fhn[5];
    a.ubounds[1] = c.fhn[6];
  }
  std::memcpy(a.stim_p, c.stim_params, sizeof a.stim_p);
  a.flags = d_ionflags;
  return a;
}

// cell_means (snapshot.cpp:13-28) of U^k on the device
void DeviceSim::cell_means(std::vector<double>& out) {
  const Problem& pr = *P;
  if (!d_area) {
    std::vector<double> area(ncells);
    for (int i = 0; i < ncells; ++i) area[i] = pr.mesh.area(pr.perm[pr.cell_begin + i]);
    d_area = dupload(area, st);
    d_means = dalloc<double>(ncells);
  }
  launch_cell_means(pr.p, ncells, static_cast<int>(pr.gl_x.size()), d_bbox, d_tri_ptr, d_tri, d_U[0], d_area,
                    d_means, st);
  PDG_CUDA(cudaGetLastError());
  out.resize(ncells);
  PDG_CUDA(cudaMemcpyAsync(out.data(), d_means, sizeof(double) * ncells, cudaMemcpyDeviceToHost, st));
  PDG_CUDA(cudaStreamSynchronize(st));
}

StepResult DeviceSim::step() {
  const Problem& pr = *P;
  if (pr.from_operator) throw ConfigError("step: this solver was built from an operator (no time stepper)");
  const pdg_config& c = pr.cfg;
  const bool has_prev = k > 0;
  StepResult out;
  const int maxit = maxit_default;
  PDG_CUDA(cudaEventRecord(ev0, st));
  double* U = d_U[0];
  double* Up = d_U[1];
  const bool ionic = pr.n_comp > 0 || c.stim_kind != PDG_STIM_NONE;
  if (ionic) {
    launch_ionic(ionic_args(has_prev), st);
  }
  reset_scalars(c.tol, maxit);
  halo_exchange(U);
  launch_rhs(b, ncells, d_ptr, d_col, d_kval, d_M, 2.0 * c.C_m * c.chi_m, U, ionic ? d_ion : nullptr,
             c.warm_start, d_rhs, d_x, d_r, red_for(kFinDenom), st);
  after_reduce(kFinDenom, false);
  PDG_CUDA(cudaEventRecord(ev1, st));
  // the ionic flags are read and cleared whatever the solve does, and a
  // non-finite ionic state is reported in preference to the PCG breakdown it
  // causes (the reference throws from the ionic assembly before solving,
  // ionics.cpp:22-23, timestepper.cpp:156)
  auto take_ionflags = [&]() {
    int f = 0;
    if (ionic) {
      PDG_CUDA(cudaMemcpyAsync(&f, d_ionflags, sizeof(int), cudaMemcpyDeviceToHost, st));
      PDG_CUDA(cudaMemsetAsync(d_ionflags, 0, sizeof(int), st));
    }
    PDG_CUDA(cudaStreamSynchronize(st));
    return f;
  };
  auto ionic_error = [&]() {
    return SolverError(c.ionic_model == PDG_IONIC_BARRETO_CRESSMAN
                           ? "barreto-cressman: non-finite state in current evaluation"
                           : "fhn: non-finite state in current evaluation");
  };
  PcgResult res;
  try {
    run_solve(maxit, res);
  } catch (const SolverError&) {
    if (take_ionflags() & 2) throw ionic_error();
    throw;
  }
  PDG_CUDA(cudaEventRecord(ev2, st));
  const int ionflags = take_ionflags();
  if (ionflags & 2) throw ionic_error();
  if (ionflags & 1)
    std::fprintf(stderr,
                 "polydg: warning: membrane potential left the admissible range by more than 10x "
                 "the model span\n");
  if (!res.converged) {
    char buf[256];
    std::snprintf(buf, sizeof buf, "time step %d: PCG did not converge within %d iterations (residual %f)",
                  k + 1, maxit, res.resid.empty() ? 1.0 : res.resid.back());
    throw SolverError(buf);
  }
  // shift: U_prev <- U_curr, U_curr <- x ; Y_prev <- Y_curr, Y_curr <- Y_next
  std::swap(d_U[0], d_U[1]);
  PDG_CUDA(cudaMemcpyAsync(d_U[0], d_x, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  if (pr.n_comp > 0) {
    double* old_prev = d_Y[1];
    d_Y[1] = d_Y[0];
    d_Y[0] = d_Y[2];
    d_Y[2] = old_prev;
  }
  k += 1;
  t = k * c.dt;
  launches += (ionic ? 1 : 0) + 1 + precond_launches() + 1 + body_launches() * static_cast<long long>(res.iterations);
  float ms_all = 0.f, ms_solve = 0.f;
  cudaEventElapsedTime(&ms_all, ev0, ev2);
  cudaEventElapsedTime(&ms_solve, ev1, ev2);
  out.iterations = res.iterations;
  out.converged = res.converged;
  out.final_residual = res.resid.empty() ? 0.0 : res.resid.back();
  out.alpha = std::move(res.alpha);
  out.beta = std::move(res.beta);
  out.step_ms = ms_all;
  out.solve_ms = ms_solve;
  return out;
}

}  // namespace pdg

namespace pdg {

// kernels issued by one stand-alone precond apply: restrict (+ combine on
// several ranks), the sweep, prolong+dot
int DeviceSim::precond_launches() const {
  if (!use_pc()) return 1;
  return (P->two_level ? (world > 1 ? 2 : 1) : 0) + (n_tasks > 0 ? 1 : 0) + 1;
}

// kernels per PCG iteration: spmv, update, precond, pupdate, loop condition
// (+ finish kernels and halo packs on multi-rank runs); on one rank the
// restriction is fused into the update
int DeviceSim::body_launches() const {
  const int fused = (use_pc() && P->two_level && world == 1) ? 1 : 0;
  // spmv, update, preconditioner, pupdate, set_condition
  int k = 1 + 1 + precond_launches() - fused + 1 + (world == 1 ? 1 : 0);
  if (world > 1) k += 3 + static_cast<int>(halo_peers.size());  // finish kernels + halo packs
  return k;
}

double* DeviceSim::stage(long long len) {
  if (len > stage_len) {
    if (d_stage) cudaFree(d_stage);
    d_stage = dalloc<double>(len);
    stage_len = len;
  }
  return d_stage;
}

void DeviceSim::timer(int stop, double* ms) {
  if (!stop) {
    PDG_CUDA(cudaEventRecord(ev_t0, st));
    return;
  }
  PDG_CUDA(cudaEventRecord(ev_t1, st));
  PDG_CUDA(cudaEventSynchronize(ev_t1));
  float f = 0.f;
  PDG_CUDA(cudaEventElapsedTime(&f, ev_t0, ev_t1));
  if (ms) *ms = f;
}

// Times each kernel class in isolation on the live operands (device events on
// the solver stream) and returns its algorithmic bytes per launch:
//   0 spmv   8 nnz + 4 nnzb + 4 (rows+1) + 8 n (x) + 8 n (y) + 8 n (dot weight)
//   1 update 8 n * 5 (x, r, p, q read; x, r written: 6 passes, p/q read once)
//   2 restrict 8 N b bq (E) + 8 n (r) + 4 N
//   3 sweep_fwd / 4 sweep_bwd: 8 factor values + 16 n + index arrays
//   5 prolong_dot 8 N b bq + 24 n + 4 N ; 6 pupdate 24 n ; 7 ionic ; 8 rhs
void DeviceSim::profile(int reps, double* ms, long long* bytes) {
  const Problem& pr = *P;
  reset_scalars(0.5, 1 << 30);
  h_S->rho = 1e-30;
  h_S->pq = 1.0;
  PDG_CUDA(cudaMemcpyAsync(d_S, h_S, sizeof(PcgScalars), cudaMemcpyHostToDevice, st));
  PDG_CUDA(cudaMemcpyAsync(d_p, d_U[0], n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  PDG_CUDA(cudaMemcpyAsync(d_r, d_U[0], n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  const ReduceCtx rs = rctx(kFinStore);
  cudaEvent_t a, z;
  PDG_CUDA(cudaEventCreate(&a));
  PDG_CUDA(cudaEventCreate(&z));
  const long long N = ncells, nnzb = static_cast<long long>(pr.K.col.size());
  // cold L2 for every timed launch, as inside a PCG iteration (the sweep
  // streams > 400 MB between two SpMVs): a 256 MB buffer is written between
  // launches and only the launch itself is timed
  int l2 = 0, dev = 0;
  PDG_CUDA(cudaGetDevice(&dev));
  PDG_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  const std::size_t flush_bytes = std::max<std::size_t>(2 * static_cast<std::size_t>(l2), 64u << 20);
  void* flush = nullptr;
  PDG_CUDA(cudaMalloc(&flush, flush_bytes));
  auto timeit = [&](int slot, long long by, const std::function<void()>& f) {
    f();
    double total = 0.0;
    for (int i = 0; i < reps; ++i) {
      PDG_CUDA(cudaMemsetAsync(flush, i & 0xff, flush_bytes, st));
      PDG_CUDA(cudaEventRecord(a, st));
      f();
      PDG_CUDA(cudaEventRecord(z, st));
      PDG_CUDA(cudaEventSynchronize(z));
      float t = 0.f;
      PDG_CUDA(cudaEventElapsedTime(&t, a, z));
      total += t;
    }
    ms[slot] = total / reps;
    bytes[slot] = by;
  };
  for (int i = 0; i < 9; ++i) {
    ms[i] = 0.0;
    bytes[i] = 0;
  }
  timeit(0, 8 * nnzb * b * b + 4 * nnzb + 4 * (N + 1) + 24 * n,
         [&] { launch_spmv(b, ncells, d_ptr, d_col, d_kval, d_p, d_q, d_p, rs, false, st); });
  const bool fused = use_pc() && pr.two_level && world == 1;
  if (fused)  // slot 1 = the update fused with the restriction (slots 2, 4 stay 0)
    timeit(1, 48 * n + 8 * N * b * bq + 4 * N + 8LL * n_chunks * bq, [&] {
      if (chunks_contiguous)
        launch_update_restrict_tma(b, bq, n_chunks, max_chunk_cells, d_chunk_ptr, d_agg_cells, d_E, d_x, d_r, d_p,
                                   d_q, d_r0part, rs, st);
      else
        launch_update_restrict(b, bq, n_chunks, d_chunk_ptr, d_agg_cells, d_E, d_x, d_r, d_p, d_q, d_r0part, rs, st);
    });
  else
    timeit(1, 48 * n, [&] { launch_update(n, d_x, d_r, d_p, d_q, rs, st); });
  const long long fvf = panel_values, fvh = 0;  // F + H values (host copies released after upload)
  const long long tile_bytes = 24LL * static_cast<long long>(pr.ftiles.size());
  const long long idx_bytes = 8 * static_cast<long long>(pr.row_dof.size() + pr.in_idx.size()) +
                              4 * static_cast<long long>(pr.in_ptr.size()) + 64LL * n_tasks;
  if (use_pc()) {
    if (pr.two_level && !fused) {
      timeit(2, 8 * N * b * bq + 8 * n + 4 * N + 8LL * n_chunks * bq,
             [&] { launch_restrict(b, bq, n_chunks, d_chunk_ptr, d_agg_cells, d_E, d_r, d_r0part, nullptr, st); });
      timeit(4, 16LL * n_chunks * bq + 8LL * pr.n_agg * bq,
             [&] { launch_restrict_combine(bq, pr.n_agg, d_node_chunk_ptr, d_r0part, d_r0, nullptr, st); });
    }
    // slot 3: the fused forward + backward sweep (panels F and H once each)
    timeit(3, 8 * (fvf + fvh) + 32 * n + 2 * (idx_bytes + tile_bytes),
           [&] { launch_sweep(sweep_args(true, d_r, d_z, nullptr), smem_fwd, st); });
    timeit(5, 8 * N * b * bq + 24 * n + 4 * N,
           [&] {
             if (pr.two_level && chunks_contiguous)
               launch_prolong_dot_tma(b, bq, n_chunks, max_chunk_cells, d_chunk_ptr, d_agg_cells, d_cell_agg, d_E,
                                      d_y0, d_r, d_z, rs, st);
             else
               launch_prolong_dot(b, bq, ncells, d_E, d_cell_agg, d_y0, d_r, d_z, rs, st);
           });
  }
  timeit(6, 24 * n, [&] { launch_pupdate(n, d_tmp, d_z, d_S, false, st); });
  timeit(8, 8 * nnzb * b * b + 4 * nnzb + 4 * (N + 1) + 8 * N * b * b + 56 * n, [&] {
    launch_rhs(b, ncells, d_ptr, d_col, d_kval, d_M, 2.0, d_U[0], nullptr, 1, d_tmp, d_tmp2, d_q, rs, st);
  });
  // slot 7: ionic terms (FP64-FMA bound: the basis is evaluated at every
  // quadrature point); bytes = states in, ion + Y_next out, M^-1 blocks, geometry
  if (pr.n_comp > 0 || pr.cfg.stim_kind != PDG_STIM_NONE)
    timeit(7, 8 * (6 * n + N * b * b + 4 * N) + 48 * static_cast<long long>(pr.tri.size() / 6),
           [&] { launch_ionic(ionic_args(k > 0), st); });
  cudaFree(flush);
  cudaEventDestroy(a);
  cudaEventDestroy(z);
  PDG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace pdg
