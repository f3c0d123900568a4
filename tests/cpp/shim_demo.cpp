// Reference-style caller of the C++ shim (include/polydg_b200.hpp): the same
// calls a user of polydg::Simulation / pcg_solve makes. Built and run by
// tests/test_cpp_shim.py (compile on CPU, run on the GPU box).
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
  return (res.converged_all && rep.converged && std::sqrt(rr / bb) < 1e-9) ? 0 : 2;
}
