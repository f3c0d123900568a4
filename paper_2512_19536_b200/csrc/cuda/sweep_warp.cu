// The Schwarz sweep with WARP workers (PDG_SWEEP=warp): the same units,
// tickets, panels and counters as sweep.cu, but every warp is an independent
// worker that takes a ticket, waits for the unit's dependencies, gathers its
// inputs, streams the unit's panel tiles and publishes — no CTA barrier on
// the per-unit path. Small supernodes (minimum-degree orderings with little
// amalgamation, ~1-4 cells) then cost one warp's round trips instead of a
// whole CTA's, and an SM keeps ~32 units in flight instead of 8.
//
// Deadlock freedom is the sweep.cu argument per worker: tickets are taken in
// increasing order by each warp and run in that order; a unit's dependencies
// hold smaller tickets (list schedule, sim.cu), so the lowest unfinished
// ticket is always some warp's current unit and its dependencies are done.
//
// Per unit, lane roles: the unit's dependency counters are polled by one lane
// each (in parallel), lane 0 takes the lookahead ticket and lanes 0..23 /
// 0..17 load its descriptor / task record while the current unit runs.
#include <cstdint>

#include "kernels.cuh"

namespace pdg {

namespace {

constexpr int kWW = kSweepThreads / 32;  // workers per CTA
constexpr int kTilesW = 16;              // tile descriptors staged per unit
constexpr int kIdxW = 192;               // gather offsets staged per unit
constexpr int kPtrW = 64;                // in_ptr entries staged per unit

__device__ __forceinline__ int ld_acquire_w(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed_w(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_w(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_acq_rel_w(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ long long gtimer_w() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void wait_w(const int* flag, int need) {
  if (ld_acquire_w(flag) >= need) return;
  const long long t0 = clock64();
  do {
    __nanosleep(32);
    if (clock64() - t0 > (1LL << 33)) __trap();
  } while (ld_relaxed_w(flag) < need);
  (void)ld_acquire_w(flag);
}

__device__ __forceinline__ double2 ldp(const double2* p, unsigned long long pol) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}

// one warp: rows of tile `tl` times input columns [j0, j1) (x indexed by the
// tile's column); lanes 0..15 return the sums of rows (2 l, 2 l + 1)
__device__ __forceinline__ double2 tile_dot_w(const double* m, const DevTile& tl, const double* x, int j0, int j1,
                                              unsigned long long pol) {
  const int lane = threadIdx.x & 31, half = lane >> 4, l2 = lane & 15;
  double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0, acc2 = acc0, acc3 = acc0;
  if (2 * l2 < tl.rows) {
    const double2* mm = reinterpret_cast<const double2*>(m) + l2;
    const long long cs = tl.stride >> 1;
    int j = j0 + half;
    constexpr int D = 8;
    for (; j + 2 * D - 2 < j1; j += 2 * D) {
      double2 v[D];
#pragma unroll
      for (int u = 0; u < D; ++u) v[u] = ldp(mm + (j + 2 * u) * cs, pol);
#pragma unroll
      for (int u = 0; u < D; u += 4) {
        acc0.x = fma(v[u].x, x[j + 2 * u], acc0.x);
        acc0.y = fma(v[u].y, x[j + 2 * u], acc0.y);
        acc1.x = fma(v[u + 1].x, x[j + 2 * u + 2], acc1.x);
        acc1.y = fma(v[u + 1].y, x[j + 2 * u + 2], acc1.y);
        acc2.x = fma(v[u + 2].x, x[j + 2 * u + 4], acc2.x);
        acc2.y = fma(v[u + 2].y, x[j + 2 * u + 4], acc2.y);
        acc3.x = fma(v[u + 3].x, x[j + 2 * u + 6], acc3.x);
        acc3.y = fma(v[u + 3].y, x[j + 2 * u + 6], acc3.y);
      }
    }
    for (; j < j1; j += 2) {
      const double2 v0 = ldp(mm + j * cs, pol);
      acc0.x = fma(v0.x, x[j], acc0.x);
      acc0.y = fma(v0.y, x[j], acc0.y);
    }
  }
  double vx = (acc0.x + acc1.x) + (acc2.x + acc3.x), vy = (acc0.y + acc1.y) + (acc2.y + acc3.y);
  vx += __shfl_down_sync(0xffffffffu, vx, 16);
  vy += __shfl_down_sync(0xffffffffu, vy, 16);
  return make_double2(vx, vy);
}

template <bool FWD>
__device__ __forceinline__ void store_w(const SweepArgs& a, const DevTask& T, double* outv, int o, double v) {
  if (!FWD) outv[T.dof0 + o] = v;
  else if (T.pad) (T.coarse ? a.y0 : a.z)[T.dof0 + o] = v;
  else if (o < T.w) (T.coarse ? a.yc : a.yf)[T.dof0 + o] = v;
  else a.ubuf[T.ubuf_off + (o - T.w)] = v;
}

struct WSlot {
  DevUnit u;
  DevTask t;
  DevTile tiles[kTilesW];
  int iptr[kPtrW];
  long long idx[kIdxW];
};

template <bool FWD>
__device__ __forceinline__ void run_unit_w(const SweepArgs& a, WSlot& S, double* xin, int ep, int tk,
                                           unsigned long long pol) {
  const int lane = threadIdx.x & 31;
  const DevUnit& U = S.u;
  const DevTask& T = S.t;
  long long* tr = a.trace ? a.trace + 8LL * tk : nullptr;
  if (tr && lane == 0) tr[0] = gtimer_w();
  // L2 prefetch of the panel (consumed by evict-first loads below)
  if (lane == 0 && (a.prefetch & 1))
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"((FWD ? a.fmat : a.hmat) + U.src_off),
                 "r"(U.bytes)
                 : "memory");
  const int bs = T.bs, w = T.w;
  const int col_lo = U.col_lo, col_hi = U.col_hi;
  const int cell_lo = col_lo / bs, cell_hi = (col_hi + bs - 1) / bs;
  // ---- staging independent of the awaited units (one round of loads) ----
  const int tile0 = (FWD ? T.f_tile0 : T.h_tile0) + U.tile_begin;
  const int ntile = U.tile_end - U.tile_begin;
  const DevTile* gtiles = (FWD ? a.ftiles : a.htiles) + tile0;
  for (int i = lane; i < ntile && i < kTilesW; i += 32) S.tiles[i] = gtiles[i];
  bool meta = false;
  if (FWD) {
    const int nc = cell_hi - cell_lo;
    meta = nc + 1 <= kPtrW && U.in_n <= kIdxW;
    if (meta) {
      for (int c = lane; c <= nc; c += 32) S.iptr[c] = a.in_ptr[T.in_off + cell_lo + c];
      for (int k = lane; k < U.in_n; k += 32) S.idx[k] = a.in_idx[U.in_e0 + k];
    }
    if (T.coarse && a.r0part) {
      for (int i = col_lo + lane; i < col_hi; i += 32) {
        const int d = static_cast<int>(T.dof0) + i, node = d / bs, mm = d - node * bs;
        double v = 0.0;
        for (int c = a.node_chunk_ptr[node]; c < a.node_chunk_ptr[node + 1]; ++c) v += a.r0part[c * bs + mm];
        xin[i - col_lo] = v;
      }
    } else {
      const double* in = T.coarse ? a.r0 : a.r;
      for (int i = col_lo + lane; i < col_hi; i += 32) xin[i - col_lo] = in[T.dof0 + i];
    }
  } else {
    const int r_lo = max(col_lo, w);
    const int rc0 = (r_lo - w) / bs;
    const int nr_cells = col_hi > w ? (col_hi - w + bs - 1) / bs - rc0 : 0;
    meta = nr_cells <= kIdxW;
    if (meta)
      for (int k = lane; k < nr_cells; k += 32) S.idx[k] = a.row_dof[T.rows_off + rc0 + k];
  }
  // ---- dependencies: one lane per counter ----
  if (U.n_dep <= 2) {
    if (lane < U.n_dep) wait_w(a.flags + U.dep[lane], (ep + 1) * U.need[lane]);
  } else {
    for (int k = lane; k < T.n_child; k += 32) {
      const int c = a.task_child[T.child_off + k];
      wait_w(a.flags + c, (ep + 1) * a.tasks[c].f_ntile);
    }
  }
  if (!FWD && U.own_fwd >= 0 && col_lo < w && lane == 31) wait_w(a.flags + U.own_fwd, (ep + 1) * U.own_need);
  __syncwarp();
  if (tr && lane == 0) tr[1] = gtimer_w();
  // ---- the dependent gather ----
  double* outv = T.coarse ? a.y0 : a.z;
  if (FWD) {
    for (int i = col_lo + lane; i < col_hi; i += 32) {
      const int cell = i / bs, rr = i - cell * bs;
      double v = xin[i - col_lo];
      if (meta) {
        const int e0 = S.iptr[0];
        for (int k = S.iptr[cell - cell_lo]; k < S.iptr[cell - cell_lo + 1]; ++k) v -= __ldcg(a.ubuf + S.idx[k - e0] + rr);
      } else {
        const int k0 = a.in_ptr[T.in_off + cell], k1 = a.in_ptr[T.in_off + cell + 1];
        for (int k = k0; k < k1; ++k) v -= __ldcg(a.ubuf + a.in_idx[k] + rr);
      }
      xin[i - col_lo] = v;
    }
  } else {
    const int rc0 = (max(col_lo, w) - w) / bs;
    for (int i = col_lo + lane; i < col_hi; i += 32) {
      double v;
      if (i < w) {
        v = __ldcg((T.coarse ? a.yc : a.yf) + T.dof0 + i);
      } else {
        const int k = i - w, cell = k / bs, rr = k - cell * bs;
        const long long base = meta ? S.idx[cell - rc0] : a.row_dof[T.rows_off + cell];
        v = -__ldcg(outv + base + rr);
      }
      xin[i - col_lo] = v;
    }
  }
  __syncwarp();
  if (tr && lane == 0) tr[2] = gtimer_w();
  const int l2 = lane & 15;
  const double* panel = FWD ? a.fmat : a.hmat;
  if (U.nchunk > 1) {
    // columns [c0, c1) of one wide tile: 32 partial sums, the last chunk reduces
    const DevTile tl = S.tiles[0];
    const double2 v = tile_dot_w(panel + U.src_off, tl, xin, 0, U.c1 - U.c0, pol);
    double* gp = a.part + static_cast<long long>(U.part_base + U.chunk) * 32;
    if (lane < 16) {
      __stcg(gp + 2 * l2, v.x);
      __stcg(gp + 2 * l2 + 1, v.y);
    }
    __syncwarp();
    int last = 0;
    if (lane == 0) last = atom_acq_rel_w(a.tile_ctr + U.tile_ctr, 1) + 1 == (ep + 1) * U.nchunk;
    last = __shfl_sync(0xffffffffu, last, 0);
    if (last) {
      if (lane < tl.rows) {
        double sum = 0.0;
        const double* base = a.part + static_cast<long long>(U.part_base) * 32 + lane;
        for (int c = 0; c < U.nchunk; ++c) sum += __ldcg(base + c * 32);
        store_w<FWD>(a, T, outv, U.tile_begin * 32 + lane, sum);
      }
      __syncwarp();
      if (lane == 0) red_release_w(a.flags + (FWD ? 0 : a.n_tasks) + U.task, 1);
    }
  } else {
    for (int R = 0; R < ntile; ++R) {
      const DevTile tl = R < kTilesW ? S.tiles[R] : gtiles[R];
      const double2 v = tile_dot_w(panel + tl.off, tl, xin + (tl.col0 - col_lo), 0, tl.ncol, pol);
      if (lane < 16 && 2 * l2 < tl.rows) {
        const int o = (U.tile_begin + R) * 32 + 2 * l2;
        store_w<FWD>(a, T, outv, o, v.x);
        if (2 * l2 + 1 < tl.rows) store_w<FWD>(a, T, outv, o + 1, v.y);
      }
    }
    __syncwarp();
    if (lane == 0) red_release_w(a.flags + (FWD ? 0 : a.n_tasks) + U.task, ntile);
  }
  if (tr && lane == 0) tr[3] = gtimer_w();
}

__device__ __forceinline__ void load_desc(const SweepArgs& a, WSlot& S, int tk) {
  const int lane = threadIdx.x & 31;
  constexpr int nu = sizeof(DevUnit) / 4, nt = sizeof(DevTask) / 4;
  static_assert(nu <= 32 && nt <= 32, "descriptor fits one warp load");
  if (tk < a.n_units && lane < nu) reinterpret_cast<int*>(&S.u)[lane] = reinterpret_cast<const int*>(a.units + tk)[lane];
  __syncwarp();
  if (tk < a.n_units && lane < nt)
    reinterpret_cast<int*>(&S.t)[lane] = reinterpret_cast<const int*>(a.tasks + S.u.task)[lane];
  __syncwarp();
}

__global__ void __launch_bounds__(kSweepThreads) sweep_warp_kernel(SweepArgs a) {
  pdl_wait();
  if (a.S && a.S->stop) return;
  extern __shared__ __align__(128) double smw[];
  __shared__ WSlot slots[kWW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WSlot& S = slots[warp];
  double* xin = smw + warp * a.xcap;
  if (threadIdx.x == 0 && blockIdx.x == 0 && a.live) a.live[0] = static_cast<unsigned long long>(gtimer_w());
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  int ep = 0;
  if (lane == 0) ep = __ldcg(a.epoch);
  ep = __shfl_sync(0xffffffffu, ep, 0);
  int tk = 0;
  if (lane == 0) tk = static_cast<int>(atomicAdd(a.ticket, 1u));
  tk = __shfl_sync(0xffffffffu, tk, 0);
  load_desc(a, S, tk);
  while (tk < a.n_units) {
    // lookahead: the next ticket is taken now and its descriptor loaded after the unit
    int tkn = 0;
    if (lane == 0) tkn = static_cast<int>(atomicAdd(a.ticket, 1u));
    if (S.u.dir == 0) run_unit_w<true>(a, S, xin, ep, tk, pol);
    else run_unit_w<false>(a, S, xin, ep, tk, pol);
    tk = __shfl_sync(0xffffffffu, tkn, 0);
    load_desc(a, S, tk);
  }
  // the last worker of this sweep resets the tickets and advances the epoch
  if (lane == 0) {
    if (atomicAdd(a.epoch + 1, 1) == static_cast<int>(gridDim.x) * kWW - 1) {
      a.epoch[1] = 0;
      *a.ticket = 0u;
      a.epoch[0] = ep + 1;
      if (a.live) {
        a.live[1] += static_cast<unsigned long long>(gtimer_w()) - __ldcg(a.live);
        a.live[2] += 1;
      }
      __threadfence();
    }
  }
}

}  // namespace

void launch_sweep_warp(const SweepArgs& a, int smem, cudaStream_t st) {
  if (a.n_units == 0) return;
  static int cached_smem = -1, resident = 0;
  if (cached_smem != smem) {
    int per_sm = 0, sms = 0, dev = 0;
    PDG_CUDA(cudaGetDevice(&dev));
    PDG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    PDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_warp_kernel, kSweepThreads, smem));
    resident = (per_sm > 0 ? per_sm : 1) * sms;
    cached_smem = smem;
  }
  const int workers = (a.n_units + kWW - 1) / kWW;
  const int grid = workers < resident ? workers : resident;
  launch_pdl(sweep_warp_kernel, grid, kSweepThreads, smem, st, a);
}

int sweep_warp_workers_per_sm(int smem) {
  int per_sm = 0;
  PDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_warp_kernel, kSweepThreads, smem));
  return (per_sm > 0 ? per_sm : 1) * kWW;
}

void set_sweep_warp_smem(int bytes) {
  PDG_CUDA(cudaFuncSetAttribute(sweep_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

}  // namespace pdg
