// Reference-style caller of the C++ shim (include/polydg_b200.hpp): the same
// calls a user of polydg::Simulation / pcg_solve makes. Built and run by
// tests/test_cpp_shim.py (compile on CPU, run on the GPU box).
#include <algorithm>
#include <cmath>
#include <cstdio>

#include "polydg_b200.hpp"

int main() {
  using namespace polydg_b200;
  SimulationConfig cfg = default_config();
  cfg.mesh_cells = 256;
  cfg.degree = 2;
  cfg.subdomains = 8;
  cfg.coarse_count = -1;
  cfg.T = 10 * cfg.dt;
  Simulation sim(cfg);
  const SimulationResult res = sim.run();
  std::printf("steps %zu avg_iterations %.2f converged %d\n", res.steps.size(), res.avg_iterations,
              res.converged_all ? 1 : 0);
  Vector b(static_cast<std::size_t>(sim.dimension()));
  for (std::size_t i = 0; i < b.size(); ++i) b[i] = std::sin(0.1 * static_cast<double>(i));
  auto [x, rep] = pcg_solve(sim.system_operator(), b, sim.preconditioner(), 1e-10);
  Vector Kx;
  sim.system_operator().apply(x, Kx);
  double rr = 0.0, bb = 0.0;
  for (std::size_t i = 0; i < b.size(); ++i) {
    rr += (Kx[i] - b[i]) * (Kx[i] - b[i]);
    bb += b[i] * b[i];
  }
  std::printf("pcg iterations %d converged %d rel_residual %.3e kappa %.3f\n", rep.iterations,
              rep.converged ? 1 : 0, std::sqrt(rr / bb), rep.condition_estimate.value_or(-1.0));
  try {
    pcg_solve(sim.system_operator(), b, sim.preconditioner(), 2.0);
    return 1;
  } catch (const SolverError&) {
  }
  // snapshot.hpp: device cell means + the reference's writers and errors
  const Vector means = sim.cell_means();
  std::printf("cell_means %zu first %.6f\n", means.size(), means.empty() ? 0.0 : means[0]);
  sim.export_snapshot("/tmp/pdg_shim_snapshot.csv", "csv-cellmeans");
  try {
    sim.export_snapshot("/tmp/pdg_shim_snapshot.x", "png");
    return 3;
  } catch (const ConfigError&) {
  }
  if (means.size() != 256) return 4;

  // the reference's operator-level construction (krylov.hpp:22-30,
  // schwarz.hpp:38-39,51-53) from caller data: K from the simulation's setup,
  // partition_S = agglomerate(mesh, 8), coarse = build_coarse_embedding(q = p)
  const pdg_problem* prob = pdg_sim_problem(sim.handle());
  const std::int64_t nnz = pdg_problem_export(prob, 0, nullptr, nullptr, nullptr);
  std::vector<std::int64_t> ri(nnz), ci(nnz);
  std::vector<double> vi(nnz);
  pdg_problem_export(prob, 0, ri.data(), ci.data(), vi.data());
  SparseSymMatrix K;
  K.rows = K.cols = sim.dimension();
  K.block_dim = 6;
  {
    std::vector<std::vector<std::pair<int, double>>> rows(static_cast<std::size_t>(K.rows));
    for (std::int64_t k = 0; k < nnz; ++k) rows[ri[k]].push_back({static_cast<int>(ci[k]), vi[k]});
    for (auto& r : rows) {
      std::sort(r.begin(), r.end());
      for (auto& [c, v] : r) {
        K.col.push_back(c);
        K.val.push_back(v);
      }
      K.row_ptr.push_back(static_cast<std::int64_t>(K.col.size()));
    }
  }
  pdg_mesh* mesh = nullptr;
  check(pdg_problem_mesh(prob, &mesh));
  AgglomeratedPartition part;
  part.owner.resize(256);
  part.count = pdg_mesh_agglomerate(mesh, 8, part.owner.data(), nullptr);
  const CoarseEmbedding coarse = build_coarse_embedding(mesh, 2, part, 2);
  pdg_mesh_free(mesh);
  const SparseOperator Kop(K);
  const SchwarzPreconditioner B(K, part, &coarse);
  auto [x2, rep2] = pcg_solve(Kop, b, &B, 1e-10);
  double dx = 0.0, xx = 0.0;
  for (std::size_t i = 0; i < b.size(); ++i) {
    dx += (x2[i] - x[i]) * (x2[i] - x[i]);
    xx += x[i] * x[i];
  }
  std::printf("operator pcg iterations %d (simulation %d) rel_diff %.3e\n", rep2.iterations, rep.iterations,
              std::sqrt(dx / xx));
  if (!rep2.converged || std::abs(rep2.iterations - rep.iterations) > 1 || std::sqrt(dx / xx) > 1e-9) return 5;
  try {  // a preconditioner of another matrix is rejected
    SparseSymMatrix K2 = K;
    const SparseOperator other(K2);
    pcg_solve(other, b, &B, 1e-10);
    return 6;
  } catch (const ConfigError&) {
  }
  return (res.converged_all && rep.converged && std::sqrt(rr / bb) < 1e-9) ? 0 : 2;
}
