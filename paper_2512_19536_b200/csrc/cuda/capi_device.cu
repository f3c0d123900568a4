// C-ABI entry points of the device simulation (include/polydg_b200.h).
// Host vectors are in the reference layout and are permuted to the internal
// subdomain-major order on the device (gather/scatter kernels).
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <string>
#include <vector>
#include <algorithm>

#include "../capi_internal.hpp"
#include "../host/snapshot.hpp"
#include "sim.cuh"

struct pdg_problem {
  std::unique_ptr<pdg::Problem> p;
};

struct pdg_sim {
  std::unique_ptr<pdg::DeviceSim> d;
  pdg_problem view;  // non-owning alias for pdg_sim_problem
};

namespace {

pdg::DeviceSim& S(pdg_sim* s) { return *s->d; }

// host (reference order) -> device (internal order) for this rank's cells
void to_device(pdg::DeviceSim& d, const double* h, double* dst, int nfields = 1) {
  const auto& pr = *d.P;
  const long long N = pr.n_global_dofs();
  double* stage = d.stage(N * nfields);
  PDG_CUDA(cudaMemcpyAsync(stage, h, sizeof(double) * N * nfields, cudaMemcpyHostToDevice, d.st));
  pdg::launch_gather_perm(stage, dst, d.d_perm, d.ncells, d.b, nfields, N, d.n, d.st);
}

void to_host(pdg::DeviceSim& d, const double* src, double* h, int nfields = 1) {
  const auto& pr = *d.P;
  const long long N = pr.n_global_dofs();
  double* stage = d.stage(N * nfields);
  if (d.world > 1) PDG_CUDA(cudaMemsetAsync(stage, 0, sizeof(double) * N * nfields, d.st));
  pdg::launch_scatter_perm(src, stage, d.d_perm, d.ncells, d.b, nfields, d.n, N, d.st);
  PDG_CUDA(cudaMemcpyAsync(h, stage, sizeof(double) * N * nfields, cudaMemcpyDeviceToHost, d.st));
  PDG_CUDA(cudaStreamSynchronize(d.st));
}

void fill_report(const pdg::PcgResult& r, pdg_pcg_report* rep) {
  if (!rep) return;
  rep->iterations = r.iterations;
  rep->converged = r.converged;
  double kappa = 0.0;
  rep->has_condition = pdg::lanczos_condition(r.alpha.data(), r.beta.data(),
                                              static_cast<int>(r.alpha.size()), &kappa)
                           ? 1
                           : 0;
  // condition_estimate is attached only after a completed loop (krylov.cpp:74)
  if (r.denom == 0.0) rep->has_condition = 0;
  rep->condition_estimate = kappa;
  const int cap = rep->capacity;
  auto cp = [cap](const std::vector<double>& v, double* dst) {
    if (!dst) return;
    for (int i = 0; i < static_cast<int>(v.size()) && i < cap; ++i) dst[i] = v[i];
  };
  cp(r.resid, rep->residual_history);
  cp(r.alpha, rep->alphas);
  cp(r.beta, rep->betas);
}

// device cell means scattered to reference cell order (other ranks' cells 0)
void cell_means_ref(pdg::DeviceSim& d, double* means) {
  const pdg::Problem& pr = *d.P;
  if (pr.from_operator) throw pdg::ConfigError("cell_means: this solver was built from an operator (no mesh)");
  std::vector<double> local;
  d.cell_means(local);
  std::fill(means, means + pr.n_cells_global, 0.0);
  for (int i = 0; i < d.ncells; ++i) means[pr.perm[pr.cell_begin + i]] = local[i];
}

}  // namespace

extern "C" {

pdg_status pdg_sim_create(const pdg_config* cfg, pdg_sim** out) {
  return pdg::guarded([&] {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw pdg::CudaError("no CUDA device available (the solver has no CPU fallback)");
    auto prob = pdg::build_problem(*cfg, true);
    auto* s = new pdg_sim;
    try {
      s->d = std::make_unique<pdg::DeviceSim>(std::move(prob));
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

pdg_status pdg_sim_create_from_operator(const pdg_operator_desc* desc, pdg_sim** out) {
  return pdg::guarded([&] {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw pdg::CudaError("no CUDA device available (the solver has no CPU fallback)");
    if (!desc) throw pdg::ConfigError("operator: null descriptor");
    auto prob = pdg::build_problem_from_operator(*desc);
    auto* s = new pdg_sim;
    try {
      s->d = std::make_unique<pdg::DeviceSim>(std::move(prob));
    } catch (...) {
      delete s;
      throw;
    }
    *out = s;
  });
}

void pdg_sim_free(pdg_sim* s) {
  if (!s) return;
  s->view.p.release();
  delete s;
}

const pdg_problem* pdg_sim_problem(const pdg_sim* s) {
  auto* m = const_cast<pdg_sim*>(s);
  if (!m->view.p) m->view.p.reset(m->d->P.get());
  return &m->view;
}

int64_t pdg_sim_dimension(const pdg_sim* s) { return s->d->P->n_global_dofs(); }

pdg_status pdg_sim_step(pdg_sim* s, pdg_step_stats* stats) {
  return pdg::guarded([&] {
    const pdg::StepResult r = S(s).step();
    if (stats) {
      stats->iterations = r.iterations;
      stats->converged = r.converged;
      stats->final_residual = r.final_residual;
      double kappa = 0.0;
      stats->has_condition = pdg::lanczos_condition(r.alpha.data(), r.beta.data(),
                                                    static_cast<int>(r.alpha.size()), &kappa)
                                 ? 1
                                 : 0;
      stats->condition_estimate = kappa;
      stats->solve_ms = r.solve_ms;
      stats->step_ms = r.step_ms;
    }
  });
}

pdg_status pdg_sim_cell_means(pdg_sim* s, double* means) {
  return pdg::guarded([&] { cell_means_ref(S(s), means); });
}

pdg_status pdg_sim_export_snapshot(pdg_sim* s, const char* path, const char* format) {
  return pdg::guarded([&] {
    pdg::DeviceSim& d = S(s);
    const pdg::Problem& pr = *d.P;
    if (std::string(format) != "vtk-legacy" && std::string(format) != "csv-cellmeans")
      throw pdg::ConfigError("unknown snapshot format '" + std::string(format) + "'");
    std::vector<double> means(pr.n_cells_global);
    cell_means_ref(d, means.data());
    pdg::write_snapshot(pr.mesh, means, d.t, path, format);
  });
}

pdg_status pdg_sim_get_state(pdg_sim* s, int* k, double* t, double* U_curr, double* U_prev,
                             double* Y_curr, double* Y_prev) {
  return pdg::guarded([&] {
    auto& d = S(s);
    if (k) *k = d.k;
    if (t) *t = d.t;
    if (U_curr) to_host(d, d.d_U[0], U_curr);
    if (U_prev) to_host(d, d.d_U[1], U_prev);
    if (d.n_comp > 0) {
      if (Y_curr) to_host(d, d.d_Y[0], Y_curr, d.n_comp);
      if (Y_prev) to_host(d, d.d_Y[1], Y_prev, d.n_comp);
    }
  });
}

pdg_status pdg_sim_set_state(pdg_sim* s, int k, const double* U_curr, const double* U_prev,
                             const double* Y_curr, const double* Y_prev) {
  return pdg::guarded([&] {
    auto& d = S(s);
    d.k = k;
    d.t = k * d.P->cfg.dt;
    if (U_curr) to_device(d, U_curr, d.d_U[0]);
    if (U_prev) to_device(d, U_prev, d.d_U[1]);
    if (d.n_comp > 0) {
      if (Y_curr) to_device(d, Y_curr, d.d_Y[0], d.n_comp);
      if (Y_prev) to_device(d, Y_prev, d.d_Y[1], d.n_comp);
    }
  });
}

pdg_status pdg_sim_apply_K(pdg_sim* s, const double* x, double* y) {
  return pdg::guarded([&] {
    auto& d = S(s);
    to_device(d, x, d.d_tmp2);
    d.apply_K(d.d_tmp2, d.d_q);
    to_host(d, d.d_q, y);
  });
}

pdg_status pdg_sim_apply_precond(pdg_sim* s, const double* r, double* z) {
  return pdg::guarded([&] {
    auto& d = S(s);
    to_device(d, r, d.d_tmp2);
    d.apply_precond(d.d_tmp2, d.d_z);
    to_host(d, d.d_z, z);
  });
}

pdg_status pdg_sim_pcg(pdg_sim* s, const double* b, const double* x0, double tol, int maxit,
                       int use_precond, double* x, pdg_pcg_report* rep) {
  return pdg::guarded([&] {
    auto& d = S(s);
    to_device(d, b, d.d_rhs);
    if (x0) to_device(d, x0, d.d_x);
    else PDG_CUDA(cudaMemsetAsync(d.d_x, 0, d.n * sizeof(double), d.st));
    struct Restore {
      pdg::DeviceSim& d;
      ~Restore() { d.plain_cg = false; }
    } restore{d};
    d.plain_cg = !use_precond;
    const pdg::PcgResult r = d.pcg(d.d_rhs, d.d_x, d.d_x, tol, maxit);
    to_host(d, d.d_x, x);
    fill_report(r, rep);
  });
}

pdg_status pdg_sim_timer(pdg_sim* s, int stop, double* elapsed_ms) {
  return pdg::guarded([&] { S(s).timer(stop, elapsed_ms); });
}

int64_t pdg_sim_kernel_launches(const pdg_sim* s) { return s->d->launches; }

pdg_status pdg_sim_profile(pdg_sim* s, int reps, double* ms9, int64_t* bytes9) {
  return pdg::guarded([&] {
    long long b[9];
    S(s).profile(reps, ms9, b);
    for (int i = 0; i < 9; ++i) bytes9[i] = b[i];
  });
}

pdg_status pdg_sim_sweep_live(pdg_sim* s, int64_t* launches, double* total_ms) {
  return pdg::guarded([&] {
    auto& d = S(s);
    unsigned long long v[3] = {0, 0, 0};
    PDG_CUDA(cudaStreamSynchronize(d.st));
    if (d.d_live) PDG_CUDA(cudaMemcpy(v, d.d_live, sizeof v, cudaMemcpyDeviceToHost));
    if (launches) *launches = static_cast<int64_t>(v[2]);
    if (total_ms) *total_ms = static_cast<double>(v[1]) * 1e-6;
  });
}

pdg_status pdg_sim_attach_comm(pdg_sim* s, const void* id128, int rank, int world) {
  return pdg::guarded([&] { S(s).attach_comm(id128, rank, world); });
}

pdg_status pdg_sim_attach_loopback(pdg_sim* s, pdg_loopback* g, int rank, int world) {
  return pdg::guarded([&] {
    S(s).attach_loopback(*reinterpret_cast<std::shared_ptr<pdg::LoopbackGroup>*>(g), rank, world);
  });
}

pdg_status pdg_sim_pcg_device(pdg_sim* s, const double* d_b, const double* d_x0, double tol, int maxit,
                              double* d_x, pdg_pcg_report* rep) {
  return pdg::guarded([&] {
    auto& d = S(s);
    const pdg::PcgResult r = d.pcg(d_b, d_x0, d_x, tol, maxit);
    fill_report(r, rep);
  });
}

}  // extern "C"

namespace pdg {

int DeviceSim::trace_sweep(long long* out, int cap) {
  const int nu = n_units_f + n_units_b;
  if (!d_trace) PDG_CUDA(cudaMalloc(&d_trace, sizeof(long long) * 8 * std::max(nu, 1)));
  PDG_CUDA(cudaMemsetAsync(d_trace, 0, sizeof(long long) * 8 * std::max(nu, 1), st));
  PDG_CUDA(cudaMemcpyAsync(d_tmp2, d_r, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  apply_precond(d_tmp2, d_z);
  std::vector<long long> tr(8 * static_cast<std::size_t>(nu));
  PDG_CUDA(cudaMemcpy(tr.data(), d_trace, tr.size() * sizeof(long long), cudaMemcpyDeviceToHost));
  cudaFree(d_trace);
  d_trace = nullptr;
  for (int u = 0; u < nu && u < cap; ++u) {
    long long* o = out + 12LL * u;
    for (int k = 0; k < 6; ++k) o[k] = tr[8 * u + k];
    o[6] = h_units[u].task;
    o[7] = h_units[u].dir;
    o[8] = h_units[u].bytes;
    o[9] = h_units[u].nchunk;
    o[10] = P->tasks[h_units[u].task].height;
    o[11] = P->tasks[h_units[u].task].coarse;
    if (h_units[u].nchunk == 0) {  // level chunk: first tile's round trip (ns) and tile count
      o[10] = tr[8 * u + 6];
      o[11] = tr[8 * u + 7];
    }
  }
  return nu;
}

}  // namespace pdg

extern "C" int pdg_sim_trace_sweep(pdg_sim* s, long long* out, int cap) {
  int n = -1;
  pdg::guarded([&] { n = S(s).trace_sweep(out, cap); });
  return n;
}
