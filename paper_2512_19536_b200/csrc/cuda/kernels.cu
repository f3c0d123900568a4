// sm_100a kernels of the per-step solve. Reference hot loops replaced
// (SURVEY.md §2.1):
//   K1/K2 SpMV + fused dot / CN rhs      krylov.hpp:26, timestepper.cpp:148
//   K3/K4 PCG vector updates             krylov.cpp:54-71
//   K5    Schwarz local solves           schwarz.cpp:155-164
//   K6/K8 coarse restriction/prolong.    schwarz.cpp:166-167
//   K7    coarse solve (same sweep)      schwarz.cpp:167
//   K9-11 ionic terms, stimulus, Y update ionics.cpp:61-113, timestepper.cpp:128-186
// Reductions are deterministic: fixed per-CTA trees, partials summed in index
// order by the last CTA to arrive, so reruns are bit-identical (the
// reference's determinism contract, parallel.hpp:14-16).
#include <cmath>
#include <cstdlib>

#include "kernels.cuh"
#include "../host/bc_model.hpp"

#ifndef PDG_SPMV_UNROLL
#define PDG_SPMV_UNROLL 2
#endif

namespace pdg {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;  // lane 0
}

// blockDim.x must be a multiple of 32; result valid in thread 0.
__device__ double block_sum(double v) {
  __shared__ double sh[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double r = 0.0;
  if (wid == 0) {
    r = lane < static_cast<int>(blockDim.x >> 5) ? sh[lane] : 0.0;
    r = warp_sum(r);
  }
  return r;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ void apply_finish(const ReduceCtx& rc, double s) {
  PcgScalars* S = rc.S;
  auto fail = [&](int e) {
    S->error = e;
    S->stop = 1;
  };
  switch (rc.finish) {
    case kFinPq:
      S->pq = s;
      break;
    case kFinDenom: {
      const double d = sqrt(s);
      S->denom = d;
      if (d == 0.0) {
        S->converged = 1;
        S->stop = 1;
        rc.H.resid[0] = 0.0;
      }
      break;
    }
    case kFinRr: {
      const int it = S->iter;
      const double rel = sqrt(s) / S->denom;
      rc.H.resid[it] = rel;
      S->rr = s;
      S->iter = it + 1;
      if (rel < S->tol) {
        S->converged = 1;
        S->stop = 1;
      }
      break;
    }
    case kFinRzInit:
      if (!isfinite(s)) fail(kPcgRhoNonFinite0);
      else if (s <= 0.0) fail(kPcgRhoNonPos0);
      else S->rho = s;
      if (S->maxit <= 0) S->stop = 1;
      break;
    case kFinRz:
      if (!isfinite(s)) {
        fail(kPcgRhoNonFinite);
      } else if (s <= 0.0) {
        fail(kPcgRhoNonPos);
      } else {
        const double beta = s / S->rho;
        rc.H.beta[S->iter - 1] = beta;
        S->beta = beta;
        S->rho = s;
        if (S->iter >= S->maxit) S->stop = 1;
      }
      break;
    case kFinStore:
      *rc.out = s;
      break;
    case kFinAccum:
      *rc.out += s;
      break;
    default:
      break;
  }
}

// Publishes this CTA's partial; the last CTA sums all partials in index order.
__device__ void grid_finish(double block_total, const ReduceCtx& rc) {
  __shared__ int is_last;
  if (threadIdx.x == 0) {
    rc.red.partial[blockIdx.x] = block_total;
    __threadfence();
    const unsigned t = atomicAdd(rc.red.counter, 1u);
    is_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  // each thread sums partials t, t + blockDim, ... in that order; the loads
  // go out eight at a time (same sums, an eighth of the dependent round trips
  // in this serial tail: grids of 30-40K CTAs at config 4)
  double s = 0.0;
  const int n = static_cast<int>(gridDim.x), st = blockDim.x;
  int i = threadIdx.x;
  for (; i + 7 * st < n; i += 8 * st) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = __ldcg(rc.red.partial + i + u * st);
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; i < n; i += st) s += __ldcg(rc.red.partial + i);
  s = block_sum(s);
  if (threadIdx.x == 0) {
    *rc.red.counter = 0u;
    apply_finish(rc, s);
  }
}

template <int B>
struct RowGeom {
  static constexpr int kRows = 256 / B;
  static constexpr int kThreads = ((kRows * B + 31) / 32) * 32;
};

// One thread per scalar row r of block-row `row`; blocks column-major so the
// B threads of a block-row read B consecutive doubles per column step.
template <int B>
__device__ __forceinline__ double bsr_row_dot(int row, int r, const int* __restrict__ ptr,
                                              const int* __restrict__ col,
                                              const double* __restrict__ val,
                                              const double* __restrict__ x) {
  // all 2B loads of a block are issued before its FMAs, and the next block's
  // column index is loaded one block ahead (memory-level parallelism)
  double acc0 = 0.0, acc1 = 0.0;
  const int k0 = __ldg(ptr + row), k1 = __ldg(ptr + row + 1);
  int c = k0 < k1 ? __ldg(col + k0) : 0;
  for (int k = k0; k < k1; ++k) {
    const int cn = k + 1 < k1 ? __ldg(col + k + 1) : 0;
    const double* blk = val + static_cast<long long>(k) * (B * B) + r;
    const double* xb = x + static_cast<long long>(c) * B;
    double v[B], xv[B];
#pragma unroll
    for (int cc = 0; cc < B; ++cc) {
      v[cc] = __ldg(blk + cc * B);
      xv[cc] = __ldg(xb + cc);
    }
#pragma unroll
    for (int cc = 0; cc < B; cc += 2) {
      acc0 = fma(v[cc], xv[cc], acc0);
      if (cc + 1 < B) acc1 = fma(v[cc + 1], xv[cc + 1], acc1);
    }
    c = cn;
  }
  return acc0 + acc1;
}

template <int B>
__global__ void __launch_bounds__(RowGeom<B>::kThreads)
    spmv_kernel(int rows, const int* __restrict__ ptr, const int* __restrict__ col,
                const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y,
                const double* __restrict__ dotw, ReduceCtx rc, int honor_stop,
                const int* __restrict__ rowlist) {
  pdl_wait();
  if (honor_stop && rc.S->stop) return;
  const int lr = threadIdx.x / B, r = threadIdx.x - lr * B;
  const int groups = (rows + RowGeom<B>::kRows - 1) / RowGeom<B>::kRows;
  double contrib = 0.0;
  for (int gi = blockIdx.x; gi < groups; gi += gridDim.x) {  // persistent: groups blockIdx.x + k gridDim.x
    const int slot = gi * RowGeom<B>::kRows + lr;
    if (lr < RowGeom<B>::kRows && slot < rows) {
      const int row = rowlist ? __ldg(rowlist + slot) : slot;
      const double acc = bsr_row_dot<B>(row, r, ptr, col, val, x);
      const long long i = static_cast<long long>(row) * B + r;
      y[i] = acc;
      if (dotw) contrib += dotw[i] * acc;
    }
  }
  if (rc.finish != kFinNone) grid_finish(block_sum(contrib), rc);
}

// Warp per block-row SpMV for even B (p = 2, 3): the row's blocks are
// contiguous in `val`, so lane l streams double2 j = l + 32t of every block
// (fully used sectors, 2 blocks in flight per iteration). With B even a
// double2 never straddles a column, so lane l always accumulates the fixed
// row pair r = (2l + 64t) % B of column (2j)/B; lanes l = k (mod B/2) share a
// pair and are summed by a shuffle tree in a fixed order (deterministic).

template <int B>
__global__ void __launch_bounds__(256)
    spmv_warp_kernel(int rows, const int* __restrict__ ptr, const int* __restrict__ col,
                     const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y,
                     const double* __restrict__ dotw, ReduceCtx rc, int honor_stop,
                     const int* __restrict__ rowlist) {
  static_assert(B % 2 == 0, "even block size");
  constexpr int H = B * B / 2, NT = (H + 31) / 32, S = B / 2;
  pdl_wait();
  if (honor_stop && rc.S->stop) return;
  auto operand = [&](long long idx) { return __ldg(x + idx); };
  __shared__ double ys[8][B];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int slot = blockIdx.x * 8 + wl;
  double contrib = 0.0;
  if (slot < rows) {
    const int row = rowlist ? __ldg(rowlist + slot) : slot;
    const double2* __restrict__ v2 = reinterpret_cast<const double2*>(val);
    double2 acc[NT];
    int cj[NT];
    bool on[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int j = lane + 32 * t;
      on[t] = j < H;
      cj[t] = (2 * j) / B;
      acc[t] = make_double2(0.0, 0.0);
    }
    const int k0 = __ldg(ptr + row), k1 = __ldg(ptr + row + 1);
    int k = k0;
    // PDG_SPMV_UNROLL blocks in flight per iteration; the accumulation order
    // is block order whatever the unroll, so results do not depend on it
    constexpr int U = PDG_SPMV_UNROLL;
    for (; k + U - 1 < k1; k += U) {
      int cu[U];
#pragma unroll
      for (int u = 0; u < U; ++u) cu[u] = __ldg(col + k + u);
      double2 va[U][NT];
      double xa[U][NT];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          if (on[t]) {
            va[u][t] = __ldg(v2 + static_cast<long long>(k + u) * H + lane + 32 * t);
            xa[u][t] = operand(static_cast<long long>(cu[u]) * B + cj[t]);
          }
        }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          if (on[t]) {
            acc[t].x = fma(va[u][t].x, xa[u][t], acc[t].x);
            acc[t].y = fma(va[u][t].y, xa[u][t], acc[t].y);
          }
        }
    }
    for (; k < k1; ++k) {
      const int ca = __ldg(col + k);
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        if (on[t]) {
          const double2 va = __ldg(v2 + static_cast<long long>(k) * H + lane + 32 * t);
          const double xa = operand(static_cast<long long>(ca) * B + cj[t]);
          acc[t].x = fma(va.x, xa, acc[t].x);
          acc[t].y = fma(va.y, xa, acc[t].y);
        }
      }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
#pragma unroll
      for (int off = S; off < 32; off *= 2) {
        const double sx = __shfl_down_sync(0xffffffffu, acc[t].x, off);
        const double sy = __shfl_down_sync(0xffffffffu, acc[t].y, off);
        if (lane + off < 32) {
          acc[t].x += sx;
          acc[t].y += sy;
        }
      }
      if (lane < S) {
        const int r = (2 * lane + 64 * t) % B;
        if (t == 0) {
          ys[wl][r] = acc[t].x;
          ys[wl][r + 1] = acc[t].y;
        } else {
          ys[wl][r] += acc[t].x;
          ys[wl][r + 1] += acc[t].y;
        }
      }
      __syncwarp();
    }
    if (lane < B) {
      const double yv = ys[wl][lane];
      const long long i = static_cast<long long>(row) * B + lane;
      y[i] = yv;
      if (dotw) contrib = dotw[i] * yv;
    }
  }
  if (rc.finish != kFinNone) grid_finish(block_sum(contrib), rc);
}

template <int B>
__global__ void __launch_bounds__(RowGeom<B>::kThreads)
    residual_kernel(int rows, const int* __restrict__ ptr, const int* __restrict__ col,
                    const double* __restrict__ val, const double* __restrict__ x,
                    const double* __restrict__ bvec, double* __restrict__ rvec, ReduceCtx rc) {
  const int lr = threadIdx.x / B, r = threadIdx.x - lr * B;
  const int row = blockIdx.x * RowGeom<B>::kRows + lr;
  double contrib = 0.0;
  if (lr < RowGeom<B>::kRows && row < rows) {
    const double acc = bsr_row_dot<B>(row, r, ptr, col, val, x);
    const long long i = static_cast<long long>(row) * B + r;
    const double v = bvec[i] - acc;
    rvec[i] = v;
    contrib = v * v;
  }
  grid_finish(block_sum(contrib), rc);
}

template <int B>
__global__ void __launch_bounds__(RowGeom<B>::kThreads)
    rhs_kernel(int rows, const int* __restrict__ ptr, const int* __restrict__ col,
               const double* __restrict__ val, const double* __restrict__ M, double two_a,
               const double* __restrict__ U, const double* __restrict__ ion, int warm,
               double* __restrict__ rhs, double* __restrict__ x, double* __restrict__ rvec,
               ReduceCtx rc) {
  const int lr = threadIdx.x / B, r = threadIdx.x - lr * B;
  const int row = blockIdx.x * RowGeom<B>::kRows + lr;
  double contrib = 0.0;
  if (lr < RowGeom<B>::kRows && row < rows) {
    const double ku = bsr_row_dot<B>(row, r, ptr, col, val, U);
    const double* mb = M + static_cast<long long>(row) * (B * B) + r;
    const double* ub = U + static_cast<long long>(row) * B;
    double mu = 0.0;
#pragma unroll
    for (int cc = 0; cc < B; ++cc) mu = fma(__ldg(mb + cc * B), __ldg(ub + cc), mu);
    const long long i = static_cast<long long>(row) * B + r;
    double b = two_a * mu - ku;
    if (ion) b += ion[i];
    rhs[i] = b;
    const double rv = warm ? b - ku : b;
    x[i] = warm ? ub[r] : 0.0;
    rvec[i] = rv;
    contrib = rv * rv;
  }
  grid_finish(block_sum(contrib), rc);
}

__global__ void update_kernel(long long n, double* __restrict__ x, double* __restrict__ r,
                              const double* __restrict__ p, const double* __restrict__ q,
                              ReduceCtx rc) {
  pdl_wait();
  PcgScalars* S = rc.S;
  if (S->stop) return;
  const double pq = S->pq;
  const int it = S->iter;
  if (!isfinite(pq) || pq <= 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      S->error = !isfinite(pq) ? kPcgPqNonFinite : kPcgPqNonPos;
      S->stop = 1;
    }
    return;
  }
  const double alpha = S->rho / pq;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    rc.H.alpha[it] = alpha;
    S->alpha = alpha;
  }
  double contrib = 0.0;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    x[i] += alpha * p[i];
    const double rv = r[i] - alpha * q[i];
    r[i] = rv;
    contrib += rv * rv;
  }
  grid_finish(block_sum(contrib), rc);
}

__global__ void pupdate_kernel(long long n, double* __restrict__ p, const double* __restrict__ z,
                               PcgScalars* S, int first) {
  pdl_wait();
  if (!first && S->stop) return;
  const double beta = first ? 0.0 : S->beta;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride)
    p[i] = first ? z[i] : fma(beta, p[i], z[i]);
  // p = z also for a following direction-fused SpMV, which forms fma(beta, p, z)
  if (first && blockIdx.x == 0 && threadIdx.x == 0) S->beta = 0.0;
}

template <int B, int BQ>
__global__ void prolong_dot_kernel(int ncells, const double* __restrict__ E,
                                   const int* __restrict__ cell_agg, const double* __restrict__ y0,
                                   const double* __restrict__ r, double* __restrict__ z,
                                   ReduceCtx rc) {
  pdl_wait();
  if (rc.S->stop) return;
  const long long n = static_cast<long long>(ncells) * B;
  double contrib = 0.0;
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n; i += stride) {
    double zi = z[i];
    if constexpr (BQ > 0) {
      const long long c = i / B;
      const int rr = static_cast<int>(i - c * B);
      const double* e = E + c * (B * BQ) + rr;
      const double* y = y0 + static_cast<long long>(__ldg(cell_agg + c)) * BQ;
      double acc = 0.0;
#pragma unroll
      for (int m = 0; m < BQ; ++m) acc = fma(__ldg(e + m * B), __ldg(y + m), acc);
      zi += acc;
      z[i] = zi;
    }
    contrib += r[i] * zi;
  }
  grid_finish(block_sum(contrib), rc);
}

template <int B, int BQ>
__global__ void restrict_kernel(const int* __restrict__ agg_ptr, const int* __restrict__ agg_cells,
                                const double* __restrict__ E, const double* __restrict__ r,
                                double* __restrict__ r0, const PcgScalars* S) {
  pdl_wait();
  if (S && S->stop) return;
  const int a = blockIdx.x;
  const int c0 = agg_ptr[a], c1 = agg_ptr[a + 1];
  double acc[BQ];
#pragma unroll
  for (int m = 0; m < BQ; ++m) acc[m] = 0.0;
  for (int k = c0 + threadIdx.x; k < c1; k += blockDim.x) {
    const long long c = agg_cells[k];
    const double* e = E + c * (B * BQ);
    const double* rc = r + c * B;
    double rl[B];
#pragma unroll
    for (int i = 0; i < B; ++i) rl[i] = rc[i];
#pragma unroll
    for (int m = 0; m < BQ; ++m) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < B; ++i) s = fma(__ldg(e + m * B + i), rl[i], s);
      acc[m] += s;
    }
  }
#pragma unroll
  for (int m = 0; m < BQ; ++m) {
    const double s = block_sum(acc[m]);
    if (threadIdx.x == 0) r0[static_cast<long long>(a) * BQ + m] = s;
  }
}

// PCG update fused with the coarse restriction (krylov.cpp:54-58 then
// schwarz.cpp:166): one CTA per restriction chunk (<= 64 cells of one
// agglomerate) updates x and r for its cells, keeps the new r in shared
// memory and writes the chunk's E^T r partial (coalesced over the E blocks);
// ||r||^2 is finished grid-wide as in update_kernel. Deterministic.
template <int B, int BQ>
__global__ void __launch_bounds__(256) update_restrict_kernel(const int* __restrict__ chunk_ptr,
                                                              const int* __restrict__ cells,
                                                              const double* __restrict__ E, double* __restrict__ x,
                                                              double* __restrict__ r, const double* __restrict__ p,
                                                              const double* __restrict__ q,
                                                              double* __restrict__ r0part, ReduceCtx rc) {
  pdl_wait();
  PcgScalars* S = rc.S;
  if (S->stop) return;
  const double pq = S->pq;
  const int it = S->iter;
  if (!isfinite(pq) || pq <= 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      S->error = !isfinite(pq) ? kPcgPqNonFinite : kPcgPqNonPos;
      S->stop = 1;
    }
    return;
  }
  const double alpha = S->rho / pq;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    rc.H.alpha[it] = alpha;
    S->alpha = alpha;
  }
  constexpr int kCells = 64;
  __shared__ double rs[kCells * B];
  __shared__ int cl[kCells];
  __shared__ double wsum[8][BQ];
  const int c0 = chunk_ptr[blockIdx.x], nc = chunk_ptr[blockIdx.x + 1] - c0;
  for (int k = threadIdx.x; k < nc; k += blockDim.x) cl[k] = cells[c0 + k];
  __syncthreads();
  double contrib = 0.0;
  for (int e = threadIdx.x; e < nc * B; e += blockDim.x) {
    const int k = e / B, i = e - k * B;
    const long long d = static_cast<long long>(cl[k]) * B + i;
    x[d] += alpha * p[d];
    const double rv = r[d] - alpha * q[d];
    r[d] = rv;
    rs[e] = rv;
    contrib += rv * rv;
  }
  __syncthreads();
  double acc[BQ];
#pragma unroll
  for (int m = 0; m < BQ; ++m) acc[m] = 0.0;
  // 8 E loads in flight per thread before any is consumed
  const int total = nc * B * BQ;
  constexpr int kU = 8;
  for (int e0 = threadIdx.x; e0 < total; e0 += kU * blockDim.x) {
    double ev[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * blockDim.x;
      ev[u] = 0.0;
      if (e < total) {
        const int k = e / (B * BQ), f = e - k * (B * BQ);
        ev[u] = __ldg(E + static_cast<long long>(cl[k]) * (B * BQ) + f);
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int e = e0 + u * blockDim.x;
      if (e >= total) break;
      const int k = e / (B * BQ), f = e - k * (B * BQ), m = f / B, i = f - m * B;
      const double v = ev[u] * rs[k * B + i];
#pragma unroll
      for (int mm = 0; mm < BQ; ++mm)
        if (mm == m) acc[mm] += v;
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int m = 0; m < BQ; ++m) {
    const double v = warp_sum(acc[m]);
    if (lane == 0) wsum[wid][m] = v;
  }
  __syncthreads();
  if (threadIdx.x < BQ) {
    double s = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) s += wsum[w][threadIdx.x];
    r0part[static_cast<long long>(blockIdx.x) * BQ + threadIdx.x] = s;
  }
  grid_finish(block_sum(contrib), rc);
}

// ---- coarse-space kernels with the chunk's E blocks staged by TMA ----
// When every restriction chunk is a run of consecutive cells (the coarse
// partition is the subdomain partition, so agglomerates are contiguous in the
// internal order), a chunk's E blocks are one contiguous byte range: one bulk
// copy (cp.async.bulk + mbarrier) brings it into shared memory while the CTA
// does its vector work, instead of strided per-thread E loads.

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Thread 0 starts the copy of the (16-byte widened) range [lo, hi) into dst;
// returns the offset of lo inside dst. Call __syncthreads() before waiting.
__device__ __forceinline__ int stage_bytes(const void* lo, const void* hi, unsigned char* dst, uint64_t* bar) {
  const unsigned long long a = reinterpret_cast<unsigned long long>(lo), b = reinterpret_cast<unsigned long long>(hi);
  const unsigned long long alo = a & ~15ull, ahi = (b + 15) & ~15ull;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(static_cast<unsigned>(ahi - alo))
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(alo), "r"(static_cast<unsigned>(ahi - alo)), "r"(smem_addr(bar))
        : "memory");
  }
  return static_cast<int>(a - alo);
}

__device__ __forceinline__ void wait_bytes(uint64_t* bar) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_addr(bar))
        : "memory");
  }
}

template <int B, int BQ>
__global__ void __launch_bounds__(256) update_restrict_tma_kernel(const int* __restrict__ chunk_ptr,
                                                                  const int* __restrict__ cells,
                                                                  const double* __restrict__ E,
                                                                  double* __restrict__ x, double* __restrict__ r,
                                                                  const double* __restrict__ p,
                                                                  const double* __restrict__ q,
                                                                  double* __restrict__ r0part, ReduceCtx rc,
                                                                  int n_chunks) {
  pdl_wait();
  PcgScalars* S = rc.S;
  if (S->stop) return;
  const double pq = S->pq;
  const int it = S->iter;
  if (!isfinite(pq) || pq <= 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      S->error = !isfinite(pq) ? kPcgPqNonFinite : kPcgPqNonPos;
      S->stop = 1;
    }
    return;
  }
  const double alpha = S->rho / pq;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    rc.H.alpha[it] = alpha;
    S->alpha = alpha;
  }
  extern __shared__ __align__(128) unsigned char dyn[];
  __shared__ uint64_t bar;
  __shared__ double rs[64 * B];
  __shared__ double red[B * BQ];
  // chunks blockIdx.x, + gridDim.x, ...: one grid reduction per CTA for all
  // of its chunks (a grid of resident CTAs instead of one CTA per chunk)
  double contrib = 0.0;
  for (int ch = blockIdx.x; ch < n_chunks; ch += gridDim.x) {
    __syncthreads();  // smem and the barrier of the previous chunk are free
    const int c0 = chunk_ptr[ch], nc = chunk_ptr[ch + 1] - c0;
    const long long cell0 = cells[c0];
    const double* Eg = E + cell0 * (B * BQ);
    const int off = stage_bytes(Eg, Eg + static_cast<long long>(nc) * (B * BQ), dyn, &bar);
    const double* Es = reinterpret_cast<const double*>(dyn + off);
    // the x / r update overlaps the copy (consecutive dofs: coalesced)
    const long long d0 = cell0 * B;
    for (int e = threadIdx.x; e < nc * B; e += blockDim.x) {
      const long long d = d0 + e;
      x[d] += alpha * p[d];
      const double rv = r[d] - alpha * q[d];
      r[d] = rv;
      rs[e] = rv;
      contrib += rv * rv;
    }
    __syncthreads();
    wait_bytes(&bar);
    // r0part[m] = sum_i sum_k E_k(i, m) r_k(i): thread f = (m, i) sums over cells
    for (int f = threadIdx.x; f < B * BQ; f += blockDim.x) {
      const int i = f % B;
      double acc = 0.0;
      for (int k = 0; k < nc; ++k) acc = fma(Es[k * (B * BQ) + f], rs[k * B + i], acc);
      red[f] = acc;
    }
    __syncthreads();
    if (threadIdx.x < BQ) {
      double s = 0.0;
      for (int i = 0; i < B; ++i) s += red[threadIdx.x * B + i];
      r0part[static_cast<long long>(ch) * BQ + threadIdx.x] = s;
    }
  }
  grid_finish(block_sum(contrib), rc);
}

// z += E y0 for one chunk (all its cells share the agglomerate) and r.z
template <int B, int BQ>
__global__ void __launch_bounds__(256) prolong_dot_tma_kernel(const int* __restrict__ chunk_ptr,
                                                              const int* __restrict__ cells,
                                                              const int* __restrict__ cell_agg,
                                                              const double* __restrict__ E,
                                                              const double* __restrict__ y0,
                                                              const double* __restrict__ r, double* __restrict__ z,
                                                              ReduceCtx rc, int n_chunks) {
  pdl_wait();
  if (rc.S->stop) return;
  extern __shared__ __align__(128) unsigned char dyn[];
  __shared__ uint64_t bar;
  __shared__ double ys[BQ];
  double contrib = 0.0;
  for (int ch = blockIdx.x; ch < n_chunks; ch += gridDim.x) {
  __syncthreads();  // smem and the barrier of the previous chunk are free
  const int c0 = chunk_ptr[ch], nc = chunk_ptr[ch + 1] - c0;
  const long long cell0 = cells[c0];
  const double* Eg = E + cell0 * (B * BQ);
  const int off = stage_bytes(Eg, Eg + static_cast<long long>(nc) * (B * BQ), dyn, &bar);
  const double* Es = reinterpret_cast<const double*>(dyn + off);
  if (threadIdx.x < BQ) ys[threadIdx.x] = y0[static_cast<long long>(cell_agg[cell0]) * BQ + threadIdx.x];
  // r and z of the chunk are loaded while the E copy is in flight (chunks
  // hold <= 32 cells: at most kPer elements per thread)
  constexpr int kPer = (32 * B + 255) / 256;
  const long long d0 = cell0 * B;
  double rv[kPer], zv[kPer];
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int e = threadIdx.x + j * 256;
    if (e < nc * B) {
      rv[j] = r[d0 + e];
      zv[j] = z[d0 + e];
    }
  }
  __syncthreads();
  wait_bytes(&bar);
#pragma unroll
  for (int j = 0; j < kPer; ++j) {
    const int e = threadIdx.x + j * 256;
    if (e >= nc * B) continue;
    const int k = e / B, i = e - k * B;
    const double* ek = Es + k * (B * BQ) + i;
    double acc = 0.0;
#pragma unroll
    for (int m = 0; m < BQ; ++m) acc = fma(ek[m * B], ys[m], acc);
    const double zi = zv[j] + acc;
    z[d0 + e] = zi;
    contrib += rv[j] * zi;
  }
  }
  grid_finish(block_sum(contrib), rc);
}

// Schwarz supernode sweeps: see sweep.cu

// ---------------- ionic terms at quadrature nodes ----------------

__constant__ double c_glx[16];
__constant__ double c_glw[16];

template <int P>
__device__ __forceinline__ void basis_eval(double xi, double eta, double inv, double* phi) {
  double px[P + 1], py[P + 1];
  px[0] = 1.0;
  py[0] = 1.0;
  px[1] = xi;
  py[1] = eta;
#pragma unroll
  for (int k = 1; k < P; ++k) {
    px[k + 1] = ((2 * k + 1) * xi * px[k] - k * px[k - 1]) / (k + 1);
    py[k + 1] = ((2 * k + 1) * eta * py[k] - k * py[k - 1]) / (k + 1);
  }
  int m = 0;
#pragma unroll
  for (int d = 0; d <= P; ++d)
#pragma unroll
    for (int ax = d; ax >= 0; --ax, ++m) {
      const int ay = d - ax;
      phi[m] = inv * (sqrt(2.0 * ax + 1.0) * px[ax]) * (sqrt(2.0 * ay + 1.0) * py[ay]);
    }
}

// NC = state components of the model: 1 (FHN, or no model with a stimulus), 4 (Barreto-Cressman)
template <int P, int NC>
__global__ void __launch_bounds__(256) ionic_kernel(IonicArgs a) {
  constexpr int B = (P + 1) * (P + 2) / 2;
  __shared__ double sc[8][(2 + 2 * NC) * B];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int c = blockIdx.x * 8 + wl;
  if (c >= a.ncells) return;
  const long long o = static_cast<long long>(c) * B;
  double* Us = sc[wl];                // extrapolated U*
  double* Uc = sc[wl] + B;            // current U
  double* Ys = sc[wl] + 2 * B;        // extrapolated Y*, NC fields
  double* Yc = sc[wl] + (2 + NC) * B; // current Y, NC fields
  const bool model = a.model != 0 && a.n_comp > 0;
  for (int k = lane; k < B; k += 32) {
    const double u = a.U[o + k];
    Uc[k] = u;
    Us[k] = a.has_prev ? 2.0 * u - a.Up[o + k] : u;
    if (model) {
#pragma unroll
      for (int l = 0; l < NC; ++l) {
        const double y = a.Y[l * a.n + o + k];
        Yc[l * B + k] = y;
        Ys[l * B + k] = a.has_prev ? 2.0 * y - a.Yp[l * a.n + o + k] : y;
      }
    }
  }
  __syncwarp();
  const double bx0 = a.bbox[4 * c], by0 = a.bbox[4 * c + 1], bx1 = a.bbox[4 * c + 2], by1 = a.bbox[4 * c + 3];
  const double wx = bx1 - bx0, wy = by1 - by0;
  const double inv = 1.0 / sqrt(wx * wy);
  const int t0 = a.tri_ptr[c], t1 = a.tri_ptr[c + 1];
  const int ng = a.ngl, npt = (t1 - t0) * ng * ng;
  double accI[B], accF[B], accG[NC][B];
#pragma unroll
  for (int k = 0; k < B; ++k) {
    accI[k] = accF[k] = 0.0;
#pragma unroll
    for (int l = 0; l < NC; ++l) accG[l][k] = 0.0;
  }
  const double span = a.ubounds[1] - a.ubounds[0];
  int flag = 0;
  for (int pidx = lane; pidx < npt; pidx += 32) {
    const int tri = pidx / (ng * ng), rem = pidx - tri * ng * ng;
    const int i = rem / ng, j = rem - i * ng;
    const double* T = a.tri + static_cast<long long>(t0 + tri) * 6;
    const double ax = T[0], ay = T[1], bxx = T[2], byy = T[3], cx = T[4], cy = T[5];
    const double s = 0.5 * (c_glx[i] + 1.0), tt = 0.5 * (c_glx[j] + 1.0);
    const double eta = tt * (1.0 - s);
    const double area2 = (bxx - ax) * (cy - ay) - (byy - ay) * (cx - ax);
    const double px = ax + (bxx - ax) * s + (cx - ax) * eta;
    const double py = ay + (byy - ay) * s + (cy - ay) * eta;
    const double w = c_glw[i] * c_glw[j] * 0.25 * (1.0 - s) * area2;
    double phi[B];
    basis_eval<P>((2.0 * px - bx0 - bx1) / wx, (2.0 * py - by0 - by1) / wy, inv, phi);
    if (model) {
      double us = 0.0, uc = 0.0, ys[NC], yc[NC];
#pragma unroll
      for (int l = 0; l < NC; ++l) ys[l] = yc[l] = 0.0;
#pragma unroll
      for (int k = 0; k < B; ++k) {
        us = fma(Us[k], phi[k], us);
        uc = fma(Uc[k], phi[k], uc);
#pragma unroll
        for (int l = 0; l < NC; ++l) {
          ys[l] = fma(Ys[l * B + k], phi[k], ys[l]);
          yc[l] = fma(Yc[l * B + k], phi[k], yc[l]);
        }
      }
      bool finite = isfinite(us) && isfinite(uc);
#pragma unroll
      for (int l = 0; l < NC; ++l) finite = finite && isfinite(ys[l]) && isfinite(yc[l]);
      const double slack = 10.0 * span;
      if (us < a.ubounds[0] - slack || us > a.ubounds[1] + slack || uc < a.ubounds[0] - slack ||
          uc > a.ubounds[1] + slack)
        flag |= 1;
      double f, m[NC];
      if constexpr (NC == 4) {
        // Barreto-Cressman (bc_model.hpp): current at the extrapolated state, rates at the current one
        f = bc::current(a.bc, us, ys);
        bc::rates(a.bc, uc, yc, m);
        finite = finite && isfinite(f);
#pragma unroll
        for (int l = 0; l < NC; ++l) finite = finite && isfinite(m[l]);
      } else {
        // FitzHugh-Nagumo, Rogers-McCulloch form (ionics.cpp:20-33)
        const double v = (us - a.fhn[5]) / span;
        f = a.fhn[7] * (a.fhn[2] * v * (v - a.fhn[0]) * (v - 1.0) + a.fhn[3] * v * ys[0]) * span;
        const double vc = (uc - a.fhn[5]) / span;
        m[0] = -a.fhn[1] * (vc - a.fhn[4] * yc[0]);
      }
      if (!finite) flag |= 2;
      const double wf = w * f;
#pragma unroll
      for (int k = 0; k < B; ++k) accI[k] = fma(wf, phi[k], accI[k]);
#pragma unroll
      for (int l = 0; l < NC; ++l) {
        const double wm = w * m[l];
#pragma unroll
        for (int k = 0; k < B; ++k) accG[l][k] = fma(wm, phi[k], accG[l][k]);
      }
    }
    if (a.stim != 0) {
      double g = 0.0;
      if (a.stim == 1)
        g = (px < a.stim_p[1] && a.t_mid < a.stim_p[2]) ? a.stim_p[0] : 0.0;
      else
        g = a.stim_p[0] * cos(M_PI * px) * cos(M_PI * py) * exp(-a.stim_p[1] * a.t_mid);
      const double wg = w * g;
#pragma unroll
      for (int k = 0; k < B; ++k) accF[k] = fma(wg, phi[k], accF[k]);
    }
  }
  // warp reductions (lane 0 holds the sums), broadcast through shared memory
#pragma unroll
  for (int k = 0; k < B; ++k) {
    accI[k] = warp_sum(accI[k]);
    accF[k] = warp_sum(accF[k]);
#pragma unroll
    for (int l = 0; l < NC; ++l) accG[l][k] = warp_sum(accG[l][k]);
  }
  flag = __reduce_or_sync(0xffffffffu, flag);
  __syncwarp();
  if (lane == 0) {
    if (flag) atomicOr(a.flags, flag);
#pragma unroll
    for (int k = 0; k < B; ++k) a.ion[o + k] = -(a.chi * a.dt) * accI[k] + a.dt * accF[k];
#pragma unroll
    for (int l = 0; l < NC; ++l)
#pragma unroll
      for (int k = 0; k < B; ++k) Ys[l * B + k] = accG[l][k];  // reuse as G
  }
  __syncwarp();
  if (model) {
    const double* Mi = a.Minv + static_cast<long long>(c) * B * B;
    for (int idx = lane; idx < NC * B; idx += 32) {
      const int l = idx / B, k = idx - l * B;
      double acc = 0.0;
#pragma unroll
      for (int jj = 0; jj < B; ++jj) acc = fma(Mi[jj * B + k], Ys[l * B + jj], acc);
      a.Ynext[l * a.n + o + k] = Yc[l * B + k] - a.dt * acc;
    }
  }
}

__global__ void gather_perm_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                   const int* __restrict__ perm, int ncells, int b, int nfields,
                                   long long ss, long long sd) {
  const long long n = static_cast<long long>(ncells) * b;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long c = i / b;
    const int r = static_cast<int>(i - c * b);
    const long long s = static_cast<long long>(perm[c]) * b + r;
    for (int f = 0; f < nfields; ++f) dst[f * sd + i] = src[f * ss + s];
  }
}

__global__ void scatter_perm_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                    const int* __restrict__ perm, int ncells, int b, int nfields,
                                    long long ss, long long sd) {
  const long long n = static_cast<long long>(ncells) * b;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long c = i / b;
    const int r = static_cast<int>(i - c * b);
    const long long d = static_cast<long long>(perm[c]) * b + r;
    for (int f = 0; f < nfields; ++f) dst[f * sd + d] = src[f * ss + i];
  }
}

// r0[node] = sum of the node's chunk partials, fixed order
__global__ void restrict_combine_kernel(int bq, int n_agg, const int* __restrict__ node_chunk_ptr,
                                        const double* __restrict__ part, double* __restrict__ r0,
                                        const PcgScalars* S) {
  pdl_wait();
  if (S && S->stop) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_agg * bq) return;
  const int a = i / bq, m = i - a * bq;
  double s = 0.0;
  for (int ch = node_chunk_ptr[a]; ch < node_chunk_ptr[a + 1]; ++ch) s += part[static_cast<long long>(ch) * bq + m];
  r0[i] = s;
}

// Multi-rank: the producing kernel stored its local sum; after the NCCL
// all-reduce this applies the finish on every rank identically.
__global__ void finish_kernel(ReduceCtx rc, const double* sum, int honor) {
  if (honor && rc.S->stop) return;
  apply_finish(rc, *sum);
}

__global__ void pack_kernel(const double* __restrict__ v, const int* __restrict__ cells, int ncells, int b,
                            double* __restrict__ out) {
  const long long n = static_cast<long long>(ncells) * b;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long k = i / b;
    out[i] = v[static_cast<long long>(cells[k]) * b + (i - k * b)];
  }
}

}  // namespace

bool pdl_enabled() {
  static const bool on = !(std::getenv("PDG_PDL") && std::atoi(std::getenv("PDG_PDL")) == 0);
  return on;
}

namespace {

int vec_grid(long long n) {
  long long g = (n + kVecThreads - 1) / kVecThreads;
  if (g > 148 * 16) g = 148 * 16;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

#define PDG_B_DISPATCH(b, MACRO) \
  switch (b) {                   \
    case 3: MACRO(3); break;     \
    case 6: MACRO(6); break;     \
    case 10: MACRO(10); break;   \
    case 15: MACRO(15); break;   \
    case 21: MACRO(21); break;   \
    case 28: MACRO(28); break;   \
    default: throw CudaError("unsupported block size"); \
  }

// Persistent grids (default): the per-iteration vector kernels run one
// resident grid that strides over their chunks / row groups, so the grid
// reduction's per-CTA fence + atomic and the last CTA's sum happen once per
// resident CTA instead of once per 32-cell chunk (30-40K CTAs at config 4).
// PDG_PERSIST=0: one CTA per chunk / row group.
bool persistent_grids() {
  static const bool on = !(std::getenv("PDG_PERSIST") && std::getenv("PDG_PERSIST")[0] == '0');
  return on;
}

template <class K>
static int resident_ctas(K kernel, int threads, int smem) {
  int per_sm = 0, sms = 0, dev = 0;
  PDG_CUDA(cudaGetDevice(&dev));
  PDG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  PDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
  return std::max(1, per_sm) * sms;
}

void launch_spmv(int b, int rows, const int* ptr, const int* col, const double* val, const double* x,
                 double* y, const double* dotw, ReduceCtx rc, bool honor_stop, cudaStream_t st,
                 const int* rowlist) {
  // even B (p = 2, 3) on small row counts: warp per block row. The
  // thread-per-row kernel fills only ~half the GPU below ~30K block rows
  // (config2: 656 CTAs) but streams better once every SM holds several of its
  // CTAs (config5 p=2: 4.5 vs 2.2 TB/s). PDG_SPMV_WARP=0/1 forces either.
  static const char* wenv = std::getenv("PDG_SPMV_WARP");
  const bool warp_rows = wenv ? wenv[0] == '1' : rows <= 32768;
  if (rows > 0 && warp_rows && (b == 6 || b == 10)) {
    const int g = (rows + 7) / 8;
    if (b == 6)
      launch_pdl(spmv_warp_kernel<6>, g, 256, 0, st, rows, ptr, col, val, x, y, dotw, rc, honor_stop ? 1 : 0,
                 rowlist);
    else
      launch_pdl(spmv_warp_kernel<10>, g, 256, 0, st, rows, ptr, col, val, x, y, dotw, rc, honor_stop ? 1 : 0,
                 rowlist);
    return;
  }
#define L(B)                                                                                  \
  {                                                                                           \
    const int g = (rows + RowGeom<B>::kRows - 1) / RowGeom<B>::kRows;                         \
    static const int res = resident_ctas(spmv_kernel<B>, RowGeom<B>::kThreads, 0);            \
    launch_pdl(spmv_kernel<B>, persistent_grids() ? std::min(g, res) : g, RowGeom<B>::kThreads, 0, st, rows, ptr, \
               col, val, x, y, dotw, rc, honor_stop ? 1 : 0, rowlist);                        \
  }
  if (rows > 0) PDG_B_DISPATCH(b, L)
#undef L
}

void launch_residual(int b, int rows, const int* ptr, const int* col, const double* val,
                     const double* x, const double* bvec, double* r, ReduceCtx rc, cudaStream_t st) {
#define L(B)                                                                                  \
  {                                                                                           \
    const int g = (rows + RowGeom<B>::kRows - 1) / RowGeom<B>::kRows;                         \
    residual_kernel<B><<<g, RowGeom<B>::kThreads, 0, st>>>(rows, ptr, col, val, x, bvec, r, rc); \
  }
  PDG_B_DISPATCH(b, L)
#undef L
}

void launch_rhs(int b, int rows, const int* ptr, const int* col, const double* val, const double* M,
                double two_a, const double* U, const double* ion, int warm, double* rhs, double* x,
                double* r, ReduceCtx rc, cudaStream_t st) {
#define L(B)                                                                                   \
  {                                                                                            \
    const int g = (rows + RowGeom<B>::kRows - 1) / RowGeom<B>::kRows;                          \
    rhs_kernel<B><<<g, RowGeom<B>::kThreads, 0, st>>>(rows, ptr, col, val, M, two_a, U, ion,   \
                                                      warm, rhs, x, r, rc);                    \
  }
  PDG_B_DISPATCH(b, L)
#undef L
}

void launch_update(long long n, double* x, double* r, const double* p, const double* q, ReduceCtx rc,
                   cudaStream_t st) {
  launch_pdl(update_kernel, vec_grid(n), kVecThreads, 0, st, n, x, r, p, q, rc);
}

void launch_pupdate(long long n, double* p, const double* z, PcgScalars* S, bool first,
                    cudaStream_t st) {
  launch_pdl(pupdate_kernel, vec_grid(n), kVecThreads, 0, st, n, p, z, S, first ? 1 : 0);
}

template <int B>
static void prolong_dispatch(int bq, int ncells, const double* E, const int* cell_agg,
                             const double* y0, const double* r, double* z, ReduceCtx rc,
                             cudaStream_t st) {
  const int g = vec_grid(static_cast<long long>(ncells) * B);
  switch (bq) {
    case 0: launch_pdl(prolong_dot_kernel<B, 0>, g, kVecThreads, 0, st, ncells, E, cell_agg, y0, r, z, rc); break;
    case 3: launch_pdl(prolong_dot_kernel<B, 3>, g, kVecThreads, 0, st, ncells, E, cell_agg, y0, r, z, rc); break;
    case 6: if constexpr (B >= 6) { launch_pdl(prolong_dot_kernel<B, 6>, g, kVecThreads, 0, st, ncells, E, cell_agg, y0, r, z, rc); break; }
    [[fallthrough]];
    case 10: if constexpr (B >= 10) { launch_pdl(prolong_dot_kernel<B, 10>, g, kVecThreads, 0, st, ncells, E, cell_agg, y0, r, z, rc); break; }
    [[fallthrough]];
    case 15: if constexpr (B >= 15) { launch_pdl(prolong_dot_kernel<B, 15>, g, kVecThreads, 0, st, ncells, E, cell_agg, y0, r, z, rc); break; }
    [[fallthrough]];
    default: throw CudaError("unsupported coarse block size");
  }
}

void launch_prolong_dot(int b, int bq, int ncells, const double* E, const int* cell_agg,
                        const double* y0, const double* r, double* z, ReduceCtx rc, cudaStream_t st) {
#define L(B) prolong_dispatch<B>(bq, ncells, E, cell_agg, y0, r, z, rc, st)
  PDG_B_DISPATCH(b, L)
#undef L
}

template <int B>
static void restrict_dispatch(int bq, int n_agg, const int* agg_ptr, const int* agg_cells,
                              const double* E, const double* r, double* r0, const PcgScalars* S,
                              cudaStream_t st) {
  switch (bq) {
    case 3: launch_pdl(restrict_kernel<B, 3>, n_agg, 256, 0, st, agg_ptr, agg_cells, E, r, r0, S); break;
    case 6: if constexpr (B >= 6) { launch_pdl(restrict_kernel<B, 6>, n_agg, 256, 0, st, agg_ptr, agg_cells, E, r, r0, S); break; }
    [[fallthrough]];
    case 10: if constexpr (B >= 10) { launch_pdl(restrict_kernel<B, 10>, n_agg, 256, 0, st, agg_ptr, agg_cells, E, r, r0, S); break; }
    [[fallthrough]];
    case 15: if constexpr (B >= 15) { launch_pdl(restrict_kernel<B, 15>, n_agg, 256, 0, st, agg_ptr, agg_cells, E, r, r0, S); break; }
    [[fallthrough]];
    default: throw CudaError("unsupported coarse block size");
  }
}

void launch_restrict(int b, int bq, int n_agg, const int* agg_ptr, const int* agg_cells,
                     const double* E, const double* r, double* r0, const PcgScalars* S, cudaStream_t st) {
#define L(B) restrict_dispatch<B>(bq, n_agg, agg_ptr, agg_cells, E, r, r0, S, st)
  PDG_B_DISPATCH(b, L)
#undef L
}

template <int B>
static void update_restrict_dispatch(int bq, int n_chunks, const int* chunk_ptr, const int* cells, const double* E,
                                     double* x, double* r, const double* p, const double* q, double* r0part,
                                     ReduceCtx rc, cudaStream_t st) {
  switch (bq) {
#define UR(BQ) launch_pdl(update_restrict_kernel<B, BQ>, n_chunks, 256, 0, st, chunk_ptr, cells, E, x, r, p, q, r0part, rc)
    case 3: UR(3); break;
    case 6: if constexpr (B >= 6) { UR(6); break; }
    [[fallthrough]];
    case 10: if constexpr (B >= 10) { UR(10); break; }
    [[fallthrough]];
    case 15: if constexpr (B >= 15) { UR(15); break; }
    [[fallthrough]];
#undef UR
    default: throw CudaError("unsupported coarse block size");
  }
}

void launch_update_restrict(int b, int bq, int n_chunks, const int* chunk_ptr, const int* cells, const double* E,
                            double* x, double* r, const double* p, const double* q, double* r0part, ReduceCtx rc,
                            cudaStream_t st) {
#define L(B) update_restrict_dispatch<B>(bq, n_chunks, chunk_ptr, cells, E, x, r, p, q, r0part, rc, st)
  PDG_B_DISPATCH(b, L)
#undef L
}

template <int B, int BQ>
static void coarse_tma_launch(bool update, int n_chunks, int max_nc, const int* chunk_ptr, const int* cells,
                              const int* cell_agg, const double* E, double* x, double* r, const double* p,
                              const double* q, double* r0part, const double* y0, double* z, ReduceCtx rc,
                              cudaStream_t st) {
  const int smem = max_nc * B * BQ * 8 + 32;  // + widening of the range to 16-byte ends
  static int set_u = 0, set_p = 0, res_u = 0, res_p = 0;
  if (update) {
    if (smem > set_u) {
      PDG_CUDA(cudaFuncSetAttribute(update_restrict_tma_kernel<B, BQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      set_u = smem;
      res_u = resident_ctas(update_restrict_tma_kernel<B, BQ>, 256, smem);
    }
    const int grid = persistent_grids() ? std::min(n_chunks, res_u) : n_chunks;
    launch_pdl(update_restrict_tma_kernel<B, BQ>, grid, 256, smem, st, chunk_ptr, cells, E, x, r, p, q, r0part, rc,
               n_chunks);
  } else {
    if (smem > set_p) {
      PDG_CUDA(cudaFuncSetAttribute(prolong_dot_tma_kernel<B, BQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      set_p = smem;
      res_p = resident_ctas(prolong_dot_tma_kernel<B, BQ>, 256, smem);
    }
    const int grid = persistent_grids() ? std::min(n_chunks, res_p) : n_chunks;
    launch_pdl(prolong_dot_tma_kernel<B, BQ>, grid, 256, smem, st, chunk_ptr, cells, cell_agg, E, y0, r, z, rc,
               n_chunks);
  }
}

template <int B>
static void coarse_tma_dispatch(bool update, int bq, int n_chunks, int max_nc, const int* chunk_ptr,
                                const int* cells, const int* cell_agg, const double* E, double* x, double* r,
                                const double* p, const double* q, double* r0part, const double* y0, double* z,
                                ReduceCtx rc, cudaStream_t st) {
#define CT(BQ) coarse_tma_launch<B, BQ>(update, n_chunks, max_nc, chunk_ptr, cells, cell_agg, E, x, r, p, q, r0part, y0, z, rc, st)
  switch (bq) {
    case 3: CT(3); break;
    case 6: if constexpr (B >= 6) { CT(6); break; }
    [[fallthrough]];
    case 10: if constexpr (B >= 10) { CT(10); break; }
    [[fallthrough]];
    case 15: if constexpr (B >= 15) { CT(15); break; }
    [[fallthrough]];
    default: throw CudaError("unsupported coarse block size");
  }
#undef CT
}

void launch_update_restrict_tma(int b, int bq, int n_chunks, int max_chunk_cells, const int* chunk_ptr,
                                const int* cells, const double* E, double* x, double* r, const double* p,
                                const double* q, double* r0part, ReduceCtx rc, cudaStream_t st) {
#define L(B) coarse_tma_dispatch<B>(true, bq, n_chunks, max_chunk_cells, chunk_ptr, cells, nullptr, E, x, r, p, q, \
                                    r0part, nullptr, nullptr, rc, st)
  PDG_B_DISPATCH(b, L)
#undef L
}

void launch_prolong_dot_tma(int b, int bq, int n_chunks, int max_chunk_cells, const int* chunk_ptr, const int* cells,
                            const int* cell_agg, const double* E, const double* y0, const double* r, double* z,
                            ReduceCtx rc, cudaStream_t st) {
#define L(B) coarse_tma_dispatch<B>(false, bq, n_chunks, max_chunk_cells, chunk_ptr, cells, cell_agg, E, nullptr, \
                                    const_cast<double*>(r), nullptr, nullptr, nullptr, y0, z, rc, st)
  PDG_B_DISPATCH(b, L)
#undef L
}

void launch_restrict_combine(int bq, int n_agg, const int* node_chunk_ptr, const double* part, double* r0,
                             const PcgScalars* S, cudaStream_t st) {
  const int n = n_agg * bq;
  launch_pdl(restrict_combine_kernel, (n + 255) / 256, 256, 0, st, bq, n_agg, node_chunk_ptr, part, r0, S);
}

void launch_finish(ReduceCtx rc, const double* sum, bool honor, cudaStream_t st) {
  finish_kernel<<<1, 1, 0, st>>>(rc, sum, honor ? 1 : 0);
}

void launch_pack(const double* v, const int* cells, int ncells, int b, double* out, cudaStream_t st) {
  if (ncells == 0) return;
  pack_kernel<<<vec_grid(static_cast<long long>(ncells) * b), kVecThreads, 0, st>>>(v, cells, ncells, b, out);
}

// ---------------- per-cell means (snapshot.cpp:13-28) ----------------
// mean_K = (1/|K|) sum_q w_q (Phi U_K)_q over the order-2p+2 rule, one warp
// per cell; the quadrature points are generated exactly like the ionic ones.
template <int P>
__global__ void __launch_bounds__(256) cell_means_kernel(int ncells, int ngl, const double* __restrict__ bbox,
                                                         const int* __restrict__ tri_ptr,
                                                         const double* __restrict__ tri,
                                                         const double* __restrict__ U,
                                                         const double* __restrict__ area,
                                                         double* __restrict__ out) {
  constexpr int B = (P + 1) * (P + 2) / 2;
  const int lane = threadIdx.x & 31;
  const int c = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (c >= ncells) return;
  const long long o = static_cast<long long>(c) * B;
  double Uc[B];
#pragma unroll
  for (int k = 0; k < B; ++k) Uc[k] = U[o + k];
  const double bx0 = bbox[4 * c], by0 = bbox[4 * c + 1], bx1 = bbox[4 * c + 2], by1 = bbox[4 * c + 3];
  const double wx = bx1 - bx0, wy = by1 - by0;
  const double inv = 1.0 / sqrt(wx * wy);
  const int t0 = tri_ptr[c], t1 = tri_ptr[c + 1];
  const int npt = (t1 - t0) * ngl * ngl;
  double acc = 0.0;
  for (int pidx = lane; pidx < npt; pidx += 32) {
    const int tr = pidx / (ngl * ngl), rem = pidx - tr * ngl * ngl;
    const int i = rem / ngl, j = rem - i * ngl;
    const double* T = tri + static_cast<long long>(t0 + tr) * 6;
    const double ax = T[0], ay = T[1], bxx = T[2], byy = T[3], cx = T[4], cy = T[5];
    const double s = 0.5 * (c_glx[i] + 1.0), tt = 0.5 * (c_glx[j] + 1.0);
    const double eta = tt * (1.0 - s);
    const double area2 = (bxx - ax) * (cy - ay) - (byy - ay) * (cx - ax);
    const double px = ax + (bxx - ax) * s + (cx - ax) * eta;
    const double py = ay + (byy - ay) * s + (cy - ay) * eta;
    const double w = c_glw[i] * c_glw[j] * 0.25 * (1.0 - s) * area2;
    double phi[B];
    basis_eval<P>((2.0 * px - bx0 - bx1) / wx, (2.0 * py - by0 - by1) / wy, inv, phi);
    double u = 0.0;
#pragma unroll
    for (int k = 0; k < B; ++k) u = fma(phi[k], Uc[k], u);
    acc = fma(w, u, acc);
  }
  acc = warp_sum(acc);
  if (lane == 0) out[c] = acc / area[c];
}

void set_gauss_nodes(const double* x, const double* w, int n) {
  PDG_CUDA(cudaMemcpyToSymbol(c_glx, x, sizeof(double) * n));
  PDG_CUDA(cudaMemcpyToSymbol(c_glw, w, sizeof(double) * n));
}

void launch_ionic(const IonicArgs& a, cudaStream_t st) {
  const int g = (a.ncells + 7) / 8;
  if (a.ncells == 0) return;
  const bool bcm = a.model == PDG_IONIC_BARRETO_CRESSMAN && a.n_comp == 4;
#define PDG_ION(P)                                  \
  (bcm ? ionic_kernel<P, 4><<<g, 256, 0, st>>>(a)   \
       : ionic_kernel<P, 1><<<g, 256, 0, st>>>(a))
  switch (a.p) {
    case 1: PDG_ION(1); break;
    case 2: PDG_ION(2); break;
    case 3: PDG_ION(3); break;
    case 4: PDG_ION(4); break;
    case 5: PDG_ION(5); break;
    case 6: PDG_ION(6); break;
    default: throw CudaError("unsupported degree for the ionic kernel");
  }
#undef PDG_ION
}

void launch_cell_means(int p, int ncells, int ngl, const double* bbox, const int* tri_ptr, const double* tri,
                       const double* U, const double* area, double* out, cudaStream_t st) {
  const int g = (ncells + 7) / 8;
  if (ncells == 0) return;
#define PDG_CM(P) cell_means_kernel<P><<<g, 256, 0, st>>>(ncells, ngl, bbox, tri_ptr, tri, U, area, out)
  switch (p) {
    case 1: PDG_CM(1); break;
    case 2: PDG_CM(2); break;
    case 3: PDG_CM(3); break;
    case 4: PDG_CM(4); break;
    case 5: PDG_CM(5); break;
    case 6: PDG_CM(6); break;
    default: throw CudaError("unsupported degree for the cell-means kernel");
  }
#undef PDG_CM
}

void launch_gather_perm(const double* src, double* dst, const int* perm, int ncells, int b, int nf,
                        long long ss, long long sd, cudaStream_t st) {
  gather_perm_kernel<<<vec_grid(static_cast<long long>(ncells) * b), kVecThreads, 0, st>>>(src, dst, perm, ncells, b, nf, ss, sd);
}
void launch_scatter_perm(const double* src, double* dst, const int* perm, int ncells, int b, int nf,
                         long long ss, long long sd, cudaStream_t st) {
  scatter_perm_kernel<<<vec_grid(static_cast<long long>(ncells) * b), kVecThreads, 0, st>>>(src, dst, perm, ncells, b, nf, ss, sd);
}

}  // namespace pdg
