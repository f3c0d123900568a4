// Schwarz local solves and the coarse solve as one sync-free supernode sweep
// per direction (replaces the parallel_for of LLT / SimplicialLLT solves,
// /root/reference/proj/src/schwarz.cpp:155-167).
//
// Every CTA takes a ticket in topological order (forward: children first;
// backward: parents first), so a CTA only ever waits on tasks whose units all
// hold smaller tickets, i.e. are already running: deadlock-free without a
// grid barrier, and subdomains of very different sizes (1.77x at config 4)
// overlap instead of running in waves.
// Each supernode is ONE dense mat-vec over its row-tiled panel (host/pack.cpp):
//   forward : [y_S ; u_S] = F (r_S - sum of incoming descendant updates u_D)
//   backward: x_S         = H [y_S ; -x_R]
// and is cut into units of row tiles, one CTA each, so the large separators
// on the critical path of the elimination tree stream at multi-SM bandwidth.
// Inside a unit a warp streams a (tile, column-chunk) item: each half-warp
// takes every other input column and each lane a double2 (two rows), with 8
// loads in flight per lane.
// Results of other tasks (update slices, ancestor x) are read with ld.cg so a
// stale L1 line can never be observed; a unit publishes with barrier + fence
// + a release add on the task's completion counter.
#include "kernels.cuh"

namespace pdg {

namespace {

__device__ __forceinline__ int ld_acquire_s(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

constexpr int kWarps = kSweepThreads / 32;
constexpr int kMaxSmemTiles = 32;

template <bool FWD>
__global__ void __launch_bounds__(kSweepThreads) sweep_kernel(SweepArgs a) {
  if (a.S && a.S->stop) return;
  extern __shared__ double sm[];
  __shared__ DevUnit s_unit;
  __shared__ DevTile s_tiles[kMaxSmemTiles];
  if (threadIdx.x == 0) s_unit = a.units[atomicAdd(a.ticket, 1u)];
  __syncthreads();
  const DevUnit U = s_unit;
  const DevTask T = a.tasks[U.task];
  const int ntile = U.tile_end - U.tile_begin;
  const int tile0 = (FWD ? T.f_tile0 : T.h_tile0) + U.tile_begin;
  // tile descriptors do not depend on other tasks: fetch them while waiting
  for (int i = threadIdx.x; i < ntile && i < kMaxSmemTiles; i += blockDim.x) s_tiles[i] = a.tiles[tile0 + i];
  if (threadIdx.x == 0) {
    if (FWD) {
      for (int k = 0; k < T.n_child; ++k) {
        const int c = a.task_child[T.child_off + k];
        const int need = a.task_nunit[c];
        while (ld_acquire_s(a.flags + c) < need) __nanosleep(20);
      }
    } else if (T.parent >= 0) {
      const int need = a.task_nunit[T.parent];
      while (ld_acquire_s(a.flags + T.parent) < need) __nanosleep(20);
    }
  }
  __syncthreads();
  const int w = T.w, nr = T.nr, bs = T.bs, h = w + nr;
  double* outv = T.coarse ? a.y0 : a.z;
  double* xin = sm;                       // FWD: w inputs, BWD: h inputs
  double* part = sm + (FWD ? w : h);      // split-column partials (<= kSweepThreads)
  if (FWD) {
    const double* in = T.coarse ? a.r0 : a.r;
    for (int i = threadIdx.x; i < w; i += blockDim.x) {
      const int cell = i / bs, rr = i - cell * bs;
      double v = in[T.dof0 + i];
      const int k0 = a.in_ptr[T.in_off + cell], k1 = a.in_ptr[T.in_off + cell + 1];
      for (int k = k0; k < k1; ++k) v -= __ldcg(a.ubuf + a.in_idx[k] + rr);
      xin[i] = v;
    }
  } else {
    // only inputs i >= first row of this unit are touched (H is upper triangular in its first w columns)
    const int i0 = U.tile_begin * 32;
    for (int i = i0 + threadIdx.x; i < h; i += blockDim.x) {
      if (i < w) {
        xin[i] = __ldcg(outv + T.dof0 + i);
      } else {
        const int k = i - w, cell = k / bs, rr = k - cell * bs;
        xin[i] = -__ldcg(outv + a.row_dof[T.rows_off + cell] + rr);
      }
    }
  }
  __syncthreads();
  const int split = ntile >= kWarps ? 1 : kWarps / ntile;
  const int items = ntile * split;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int half = lane >> 4, l2 = lane & 15;
  for (int it = warp; it < items; it += kWarps) {
    const int R = it / split, c = it - R * split;
    const DevTile tl = R < kMaxSmemTiles ? s_tiles[R] : a.tiles[tile0 + R];
    const int chunk = (((tl.ncol + split - 1) / split) + 1) & ~1;  // even: halves keep their parity
    const int j0 = c * chunk, j1 = min(tl.ncol, j0 + chunk);
    double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0, acc2 = acc0, acc3 = acc0;
    if (2 * l2 < tl.rows) {
      const double2* m = reinterpret_cast<const double2*>(a.mat + tl.off) + l2;
      const long long cs = tl.stride >> 1;  // double2 per column
      const double* x = xin + tl.col0;
      int j = j0 + half;
      for (; j + 14 < j1; j += 16) {
        double2 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(m + (j + 2 * u) * cs);
        acc0.x = fma(v[0].x, x[j], acc0.x);
        acc0.y = fma(v[0].y, x[j], acc0.y);
        acc1.x = fma(v[1].x, x[j + 2], acc1.x);
        acc1.y = fma(v[1].y, x[j + 2], acc1.y);
        acc2.x = fma(v[2].x, x[j + 4], acc2.x);
        acc2.y = fma(v[2].y, x[j + 4], acc2.y);
        acc3.x = fma(v[3].x, x[j + 6], acc3.x);
        acc3.y = fma(v[3].y, x[j + 6], acc3.y);
        acc0.x = fma(v[4].x, x[j + 8], acc0.x);
        acc0.y = fma(v[4].y, x[j + 8], acc0.y);
        acc1.x = fma(v[5].x, x[j + 10], acc1.x);
        acc1.y = fma(v[5].y, x[j + 10], acc1.y);
        acc2.x = fma(v[6].x, x[j + 12], acc2.x);
        acc2.y = fma(v[6].y, x[j + 12], acc2.y);
        acc3.x = fma(v[7].x, x[j + 14], acc3.x);
        acc3.y = fma(v[7].y, x[j + 14], acc3.y);
      }
      for (; j < j1; j += 2) {
        const double2 v0 = __ldg(m + j * cs);
        acc0.x = fma(v0.x, x[j], acc0.x);
        acc0.y = fma(v0.y, x[j], acc0.y);
      }
    }
    double vx = (acc0.x + acc1.x) + (acc2.x + acc3.x), vy = (acc0.y + acc1.y) + (acc2.y + acc3.y);
    vx += __shfl_down_sync(0xffffffffu, vx, 16);
    vy += __shfl_down_sync(0xffffffffu, vy, 16);
    if (half == 0 && 2 * l2 < tl.rows) {
      if (split == 1) {
        const int o = (U.tile_begin + R) * 32 + 2 * l2;
        if (!FWD || o < w) outv[T.dof0 + o] = vx;
        else a.ubuf[T.ubuf_off + (o - w)] = vx;
        if (2 * l2 + 1 < tl.rows) {
          if (!FWD || o + 1 < w) outv[T.dof0 + o + 1] = vy;
          else a.ubuf[T.ubuf_off + (o + 1 - w)] = vy;
        }
      } else {
        part[it * 32 + 2 * l2] = vx;
        part[it * 32 + 2 * l2 + 1] = vy;
      }
    }
  }
  if (split > 1) {
    __syncthreads();
    for (int q = threadIdx.x; q < ntile * 32; q += blockDim.x) {
      const int R = q >> 5, l = q & 31;
      if (l >= s_tiles[R].rows) continue;
      double v = 0.0;
      for (int c = 0; c < split; ++c) v += part[(R * split + c) * 32 + l];
      const int o = (U.tile_begin + R) * 32 + l;
      if (!FWD || o < w) outv[T.dof0 + o] = v;
      else a.ubuf[T.ubuf_off + (o - w)] = v;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    red_release_add(a.flags + U.task, 1);
  }
}

}  // namespace

void launch_sweep_fwd(const SweepArgs& a, int smem, cudaStream_t st) {
  if (a.n_units == 0) return;
  sweep_kernel<true><<<a.n_units, kSweepThreads, smem, st>>>(a);
}

void launch_sweep_bwd(const SweepArgs& a, int smem, cudaStream_t st) {
  if (a.n_units == 0) return;
  sweep_kernel<false><<<a.n_units, kSweepThreads, smem, st>>>(a);
}

void set_sweep_smem(int bytes) {
  PDG_CUDA(cudaFuncSetAttribute(sweep_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  PDG_CUDA(cudaFuncSetAttribute(sweep_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

}  // namespace pdg
