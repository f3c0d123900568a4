// Shared helpers for the C-ABI translation units.
#pragma once

#include <cstdint>
#include <exception>
#include <string>

#include "../../include/polydg_b200.h"
#include "host/core.hpp"

namespace pdg {

struct Problem;
struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};

void set_error(const std::string& s);
void problem_info(const Problem& pr, int64_t info[12]);
int64_t problem_export(const Problem& pr, int which, int64_t* rows, int64_t* cols, double* vals);

// Runs fn, mapping the reference's exception taxonomy to status codes.
template <class F>
pdg_status guarded(F&& fn) {
  try {
    fn();
    return PDG_OK;
  } catch (const ConfigError& e) {
    set_error(e.what());
    return PDG_ERR_CONFIG;
  } catch (const SolverError& e) {
    set_error(e.what());
    return PDG_ERR_SOLVER;
  } catch (const MeshError& e) {
    set_error(e.what());
    return PDG_ERR_MESH;
  } catch (const IoError& e) {
    set_error(e.what());
    return PDG_ERR_IO;
  } catch (const CudaError& e) {
    set_error(e.what());
    return PDG_ERR_CUDA;
  } catch (const std::exception& e) {
    set_error(e.what());
    return PDG_ERR_INTERNAL;
  }
}

}  // namespace pdg
