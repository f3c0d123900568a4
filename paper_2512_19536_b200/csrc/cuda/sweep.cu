// Schwarz local solves and the coarse solve as ONE sync-free supernode sweep
// (forward then backward in a single launch), replacing the parallel_for of
// LLT / SimplicialLLT solves (/root/reference/proj/src/schwarz.cpp:155-167).
//
// Every CTA takes a ticket; tickets enumerate forward units in topological
// order (children first) and then backward units (parents first). A CTA only
// ever waits on units with smaller tickets, which are already running, so the
// sweep is deadlock-free without a grid barrier, subdomains of very different
// sizes overlap instead of running in waves, and the backward sweep of a
// finished subtree starts while other subtrees are still going forward.
// Each supernode is ONE dense mat-vec over its row-tiled panel (host/pack.cpp):
//   forward : [y_S ; u_S] = F (r_S - sum of incoming descendant updates u_D)
//   backward: x_S         = H [y_S ; -x_R]
// cut into units of <= 16 KB of panel: whole 32-row tiles, or column chunks
// of a wide tile. A unit stages its panel bytes into shared memory with one
// TMA bulk copy (cp.async.bulk + mbarrier) issued BEFORE it waits for its
// dependencies, so HBM streaming is taken off the elimination tree's critical
// path; after the wait only the input gather and an smem mat-vec remain.
// Column chunks write 32 partial sums each; the last chunk of a tile to finish
// (counter) reduces them in chunk order, so results are deterministic.
// Results of other tasks are read with ld.cg; a unit publishes with barrier +
// one red.release.gpu (cumulative over the barrier).
#include <cstdint>

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
__device__ __forceinline__ int atom_acq_rel_add(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void wait_count(const int* flag, int need) {
  while (ld_acquire_s(flag) < need) __nanosleep(20);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, int bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, int phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}

constexpr int kWarps = kSweepThreads / 32;
constexpr int kMaxSmemTiles = 32;

// one warp: out rows of tile `tl` restricted to input columns [j0, j1) from the
// staged panel `m` (tile base in smem); returns (row 2*l2, row 2*l2+1) sums in half 0
__device__ __forceinline__ double2 tile_dot(const double* m, const DevTile& tl, const double* x, int j0, int j1) {
  const int lane = threadIdx.x & 31, half = lane >> 4, l2 = lane & 15;
  double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0;
  if (2 * l2 < tl.rows) {
    const double2* mm = reinterpret_cast<const double2*>(m) + l2;
    const int cs = tl.stride >> 1;
    int j = j0 + half;
    for (; j + 2 < j1; j += 4) {
      const double2 v0 = mm[j * cs], v1 = mm[(j + 2) * cs];
      const double x0 = x[j], x1 = x[j + 2];
      acc0.x = fma(v0.x, x0, acc0.x);
      acc0.y = fma(v0.y, x0, acc0.y);
      acc1.x = fma(v1.x, x1, acc1.x);
      acc1.y = fma(v1.y, x1, acc1.y);
    }
    for (; j < j1; j += 2) {
      const double2 v0 = mm[j * cs];
      acc0.x = fma(v0.x, x[j], acc0.x);
      acc0.y = fma(v0.y, x[j], acc0.y);
    }
  }
  double vx = acc0.x + acc1.x, vy = acc0.y + acc1.y;
  vx += __shfl_down_sync(0xffffffffu, vx, 16);
  vy += __shfl_down_sync(0xffffffffu, vy, 16);
  return make_double2(vx, vy);
}

template <bool FWD>
__device__ __forceinline__ void store_row(const SweepArgs& a, const DevTask& T, double* outv, int o, double v) {
  if (!FWD || o < T.w) outv[T.dof0 + o] = v;
  else a.ubuf[T.ubuf_off + (o - T.w)] = v;
}

template <bool FWD>
__device__ __forceinline__ void run_unit(const SweepArgs& a, const DevUnit& U, double* panel, double* xin,
                                         double* part, DevTile* s_tiles, uint64_t* bar) {
  const DevTask T = a.tasks[U.task];
  const int tile0 = (FWD ? T.f_tile0 : T.h_tile0) + U.tile_begin;
  const int ntile = U.tile_end - U.tile_begin;
  const DevTile* tiles = FWD ? a.ftiles : a.htiles;
  const double* mat = FWD ? a.fmat : a.hmat;
  // 1. stage this unit's panel bytes (independent of other tasks) ...
  if (threadIdx.x == 0) tma_load_1d(panel, mat + U.src_off, U.bytes, bar);
  for (int i = threadIdx.x; i < ntile && i < kMaxSmemTiles; i += blockDim.x) s_tiles[i] = tiles[tile0 + i];
  // 2. ... while waiting for the tasks it reads
  if (threadIdx.x == 0) {
    if (FWD) {
      for (int k = 0; k < T.n_child; ++k) {
        const int c = a.task_child[T.child_off + k];
        wait_count(a.flags + c, a.tasks[c].f_ntile);
      }
    } else if (T.parent >= 0) {
      wait_count(a.flags + a.n_tasks + T.parent, a.tasks[T.parent].h_ntile);
    } else {
      wait_count(a.flags + U.task, T.f_ntile);  // a root's backward needs its own forward
    }
  }
  __syncthreads();
  // 3. gather the input columns this unit touches
  const int w = T.w, bs = T.bs;
  double* outv = T.coarse ? a.y0 : a.z;
  const DevTile t0 = s_tiles[0];
  const int col_lo = t0.col0 + (U.nchunk > 1 ? U.c0 : 0);
  int col_hi = t0.col0 + (U.nchunk > 1 ? U.c1 : t0.ncol);
  for (int r = 1; r < ntile && r < kMaxSmemTiles; ++r) col_hi = max(col_hi, s_tiles[r].col0 + s_tiles[r].ncol);
  if (FWD) {
    const double* in = T.coarse ? a.r0 : a.r;
    for (int i = col_lo + threadIdx.x; i < col_hi; i += blockDim.x) {
      const int cell = i / bs, rr = i - cell * bs;
      double v = in[T.dof0 + i];
      const int k0 = a.in_ptr[T.in_off + cell], k1 = a.in_ptr[T.in_off + cell + 1];
      for (int k = k0; k < k1; ++k) v -= __ldcg(a.ubuf + a.in_idx[k] + rr);
      xin[i - col_lo] = v;
    }
  } else {
    for (int i = col_lo + threadIdx.x; i < col_hi; i += blockDim.x) {
      double v;
      if (i < w) {
        v = __ldcg(outv + T.dof0 + i);
      } else {
        const int k = i - w, cell = k / bs, rr = k - cell * bs;
        v = -__ldcg(outv + a.row_dof[T.rows_off + cell] + rr);
      }
      xin[i - col_lo] = v;
    }
  }
  mbar_wait(bar, 0);
  __syncthreads();
  // 4. smem mat-vec
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, l2 = lane & 15;
  if (U.nchunk > 1) {
    // one tile, columns [c0, c1): warps split the columns, partials to global
    const DevTile tl = t0;
    const int nc = U.c1 - U.c0;
    const int per = (((nc + kWarps - 1) / kWarps) + 1) & ~1;
    const int j0 = warp * per, j1 = min(nc, j0 + per);
    const double2 v = tile_dot(panel, tl, xin, j0, j1);
    if (lane < 16) {
      part[warp * 32 + 2 * l2] = v.x;
      part[warp * 32 + 2 * l2 + 1] = v.y;
    }
    __syncthreads();
    double* gp = a.part + static_cast<long long>(U.part_base + U.chunk) * 32;
    if (threadIdx.x < 32) {
      double s = 0.0;
      for (int q = 0; q < kWarps; ++q) s += part[q * 32 + threadIdx.x];
      __stcg(gp + threadIdx.x, s);
    }
    __syncthreads();
    __shared__ int s_last;
    if (threadIdx.x == 0) s_last = atom_acq_rel_add(a.tile_ctr + U.tile_ctr, 1) == U.nchunk - 1;
    __syncthreads();
    if (!s_last) return;
    if (threadIdx.x < tl.rows) {
      double s = 0.0;
      const double* base = a.part + static_cast<long long>(U.part_base) * 32 + threadIdx.x;
      for (int c = 0; c < U.nchunk; ++c) s += __ldcg(base + c * 32);
      store_row<FWD>(a, T, outv, U.tile_begin * 32 + threadIdx.x, s);
    }
    __syncthreads();
    if (threadIdx.x == 0) red_release_add(a.flags + (FWD ? 0 : a.n_tasks) + U.task, 1);
    return;
  }
  // whole tiles: items = (tile, column split) over the warps
  const int split = ntile >= kWarps ? 1 : kWarps / ntile;
  const int items = ntile * split;
  const double* pbase = panel;
  // tile R's smem base = sum of previous tile sizes
  for (int it = warp; it < items; it += kWarps) {
    const int R = it / split, c = it - R * split;
    const DevTile tl = R < kMaxSmemTiles ? s_tiles[R] : tiles[tile0 + R];
    const double* m = pbase + (tl.off - U.src_off);
    const int chunk = (((tl.ncol + split - 1) / split) + 1) & ~1;
    const int j0 = c * chunk, j1 = min(tl.ncol, j0 + chunk);
    const double2 v = tile_dot(m, tl, xin + (tl.col0 - col_lo), j0, j1);
    if (lane < 16 && 2 * l2 < tl.rows) {
      if (split == 1) {
        const int o = (U.tile_begin + R) * 32 + 2 * l2;
        store_row<FWD>(a, T, outv, o, v.x);
        if (2 * l2 + 1 < tl.rows) store_row<FWD>(a, T, outv, o + 1, v.y);
      } else {
        part[it * 32 + 2 * l2] = v.x;
        part[it * 32 + 2 * l2 + 1] = v.y;
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
      store_row<FWD>(a, T, outv, (U.tile_begin + R) * 32 + l, v);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) red_release_add(a.flags + (FWD ? 0 : a.n_tasks) + U.task, ntile);
}

__global__ void __launch_bounds__(kSweepThreads) sweep_kernel(SweepArgs a, int panel_doubles) {
  if (a.S && a.S->stop) return;
  extern __shared__ __align__(128) double sm[];
  __shared__ int s_ticket;
  __shared__ DevUnit s_unit;
  __shared__ DevTile s_tiles[kMaxSmemTiles];
  __shared__ __align__(8) uint64_t s_bar;
  if (threadIdx.x == 0) {
    const int tk = static_cast<int>(atomicAdd(a.ticket, 1u));
    s_ticket = tk;
    s_unit = a.units[tk];
    mbar_init(&s_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const DevUnit U = s_unit;
  double* panel = sm;
  double* part = sm + panel_doubles;          // kSweepThreads doubles
  double* xin = part + kSweepThreads;
  if (s_ticket < a.n_units_f) run_unit<true>(a, U, panel, xin, part, s_tiles, &s_bar);
  else run_unit<false>(a, U, panel, xin, part, s_tiles, &s_bar);
}

}  // namespace

void launch_sweep(const SweepArgs& a, int smem, int panel_doubles, cudaStream_t st) {
  if (a.n_units == 0) return;
  sweep_kernel<<<a.n_units, kSweepThreads, smem, st>>>(a, panel_doubles);
}

void set_sweep_smem(int bytes) {
  PDG_CUDA(cudaFuncSetAttribute(sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

}  // namespace pdg
