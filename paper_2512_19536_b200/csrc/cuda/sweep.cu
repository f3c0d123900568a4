// Schwarz local solves and the coarse solve as ONE sync-free supernode sweep
// (forward then backward in a single launch), replacing the parallel_for of
// LLT / SimplicialLLT solves (/root/reference/proj/src/schwarz.cpp:155-167).
//
// Every CTA takes a ticket; tickets enumerate forward units in topological
// order (children first) and then backward units (parents first). A CTA only
// ever waits on units with smaller tickets, which are already running, so the
// sweep is deadlock-free without a grid barrier, subdomains of very different
// sizes (1.77x at config 4) overlap instead of running in waves, and the
// backward sweep of a finished subtree starts while other subtrees are still
// in their forward sweep.
// Each supernode is ONE dense mat-vec over its row-tiled panel (host/pack.cpp):
//   forward : [y_S ; u_S] = F (r_S - sum of incoming descendant updates u_D)
//   backward: x_S         = H [y_S ; -x_R]
// cut into units of row tiles, one CTA each, so the large separators on the
// critical path of the elimination tree stream at multi-SM bandwidth. Inside
// a unit a warp streams a (tile, column-chunk) item: each half-warp takes
// every other input column and each lane a double2 (two rows), 8 loads in
// flight per lane.
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
__device__ __forceinline__ void wait_count(const int* flag, int need) {
  while (ld_acquire_s(flag) < need) __nanosleep(20);
}

constexpr int kWarps = kSweepThreads / 32;
constexpr int kMaxSmemTiles = 32;

template <bool FWD>
__device__ __forceinline__ void run_unit(const SweepArgs& a, const DevUnit& U, double* sm, DevTile* s_tiles) {
  const DevTask T = a.tasks[U.task];
  const int ntile = U.tile_end - U.tile_begin;
  const int tile0 = (FWD ? T.f_tile0 : T.h_tile0) + U.tile_begin;
  const DevTile* tiles = FWD ? a.ftiles : a.htiles;
  const double* mat = FWD ? a.fmat : a.hmat;
  // tile descriptors do not depend on other tasks: fetch them while waiting
  for (int i = threadIdx.x; i < ntile && i < kMaxSmemTiles; i += blockDim.x) s_tiles[i] = tiles[tile0 + i];
  if (threadIdx.x == 0) {
    if (FWD) {
      for (int k = 0; k < T.n_child; ++k) {
        const int c = a.task_child[T.child_off + k];
        wait_count(a.flags + c, a.task_nunit[c]);
      }
    } else if (T.parent >= 0) {
      wait_count(a.flags + a.n_tasks + T.parent, a.task_nunit[a.n_tasks + T.parent]);
    } else {
      // a root's backward needs its own forward result
      wait_count(a.flags + U.task, a.task_nunit[U.task]);
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
    // only inputs i >= first row of this unit are touched (H's first w columns are upper triangular)
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
    const DevTile tl = R < kMaxSmemTiles ? s_tiles[R] : tiles[tile0 + R];
    const int chunk = (((tl.ncol + split - 1) / split) + 1) & ~1;  // even: halves keep their parity
    const int j0 = c * chunk, j1 = min(tl.ncol, j0 + chunk);
    double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0, acc2 = acc0, acc3 = acc0;
    if (2 * l2 < tl.rows) {
      const double2* m = reinterpret_cast<const double2*>(mat + tl.off) + l2;
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
    red_release_add(a.flags + (FWD ? 0 : a.n_tasks) + U.task, 1);
  }
}

__global__ void __launch_bounds__(kSweepThreads) sweep_kernel(SweepArgs a) {
  if (a.S && a.S->stop) return;
  extern __shared__ double sm[];
  __shared__ int s_ticket;
  __shared__ DevUnit s_unit;
  __shared__ DevTile s_tiles[kMaxSmemTiles];
  if (threadIdx.x == 0) {
    const int tk = static_cast<int>(atomicAdd(a.ticket, 1u));
    s_ticket = tk;
    s_unit = a.units[tk];
  }
  __syncthreads();
  const DevUnit U = s_unit;
  if (s_ticket < a.n_units_f) run_unit<true>(a, U, sm, s_tiles);
  else run_unit<false>(a, U, sm, s_tiles);
}

}  // namespace

void launch_sweep(const SweepArgs& a, int smem, cudaStream_t st) {
  if (a.n_units == 0) return;
  sweep_kernel<<<a.n_units, kSweepThreads, smem, st>>>(a);
}

void set_sweep_smem(int bytes) {
  PDG_CUDA(cudaFuncSetAttribute(sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

}  // namespace pdg
