// Device-side shared definitions for the sm_100a solver kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "../capi_internal.hpp"

#define PDG_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t _e = (call);                                                             \
    if (_e != cudaSuccess)                                                               \
      throw ::pdg::CudaError(std::string(#call) + ": " + cudaGetErrorString(_e));        \
  } while (0)

namespace pdg {

// One supernode of the Schwarz sweep (see host/problem.hpp TaskDesc).
struct DevTask {
  int coarse, bs, w, nr;
  long long dof0, ubuf_off;
  int f_tile0, f_ntile, h_tile0, h_ntile;
  int rows_off, in_off, parent, child_off, n_child, pad;  // pad = 1: dense root (TaskDesc::root_dense)
};

// A CTA's share of one supernode in one sweep direction: row tiles
// [tile_begin, tile_end) of the task's panel. Big separators are split into
// many units so the critical path of the elimination tree streams at
// multi-SM bandwidth.
// Two kinds: whole tiles [tile_begin, tile_end) (nchunk == 1), or one column
// chunk [c0, c1) of a single wide tile (nchunk > 1) whose partial sums land in
// part slot part_base + chunk; the last chunk to finish (tile counter) reduces
// them in chunk order.
// A third kind, nchunk == 0: a level chunk of bottom supernodes
// (host/problem.hpp LevelChunk), tile_begin = chunk id, src_off / bytes = its
// contiguous panels, [in_e0, in_e0 + in_n) = its record in bmeta, dep[0] /
// need[0] = the level counter it waits for (n_dep), own_fwd / chunk = the global
// and (>= 0) group level counters it adds to, part_base / tile_ctr = first entry / count of its forward
// publish list, c0 / c1 = first entry / count of its backward wait list.
struct DevUnit {
  int task, tile_begin, tile_end, c0, c1, chunk, nchunk, part_base, tile_ctr, dir;
  int n_dep;          // flags to wait on (> 2: walk the task's children)
  int dep[2], need[2];
  int own_fwd;        // backward: own forward counter index (its y_S), -1 for forward units
  long long src_off;  // first panel double staged by TMA
  int bytes;          // staged bytes (multiple of 16)
  int own_need;
  int col_lo, col_hi;  // input columns [col_lo, col_hi) of the task's panel this unit reads
  int in_e0, in_n;     // forward: its incoming-update list in_idx[in_e0, in_e0 + in_n)
};

// One 32-row tile of a supernode panel (host/problem.hpp Problem::Tile).
struct DevTile {
  long long off;
  int ncol, col0, rows, stride;
};

// Scalars of one PCG solve, resident in device memory. The iteration index,
// convergence and breakdown are decided on the device so the host only polls.
struct PcgScalars {
  double rho;      // r.z of the current iterate
  double denom;    // ||b - K x0||
  double tol;
  double pq;
  double rr;
  double alpha, beta;
  int iter;        // completed iterations
  int maxit;
  int stop;        // 1 = no more work this solve
  int converged;
  int error;       // PcgError
  int pad;
};

enum PcgError : int {
  kPcgOk = 0,
  kPcgRhoNonFinite0 = 1,  // "non-finite preconditioned product"
  kPcgRhoNonPos0 = 2,     // "preconditioner is not positive definite"
  kPcgPqNonFinite = 3,    // "non-finite operator product"
  kPcgPqNonPos = 4,       // "operator is not positive definite"
  kPcgRhoNonFinite = 5,   // "non-finite scalar"
  kPcgRhoNonPos = 6,      // "preconditioner is not positive definite"
};

// Reduction scratch: per-CTA partials + arrival counter (last block finalises).
struct Reducer {
  double* partial;
  unsigned int* counter;
};

constexpr int kSweepThreads = 128;  // default sweep CTA size (sweep.cu also instantiates 64)
constexpr int kVecThreads = 256;

// Programmatic dependent launch: the PCG body kernels are launched so that a
// kernel's CTAs can be scheduled while its predecessor in the stream drains;
// every such kernel calls pdl_wait() before touching anything the predecessor
// wrote (a no-op for ordinary launches). PDG_PDL=0 turns it off.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  PDG_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

}  // namespace pdg
