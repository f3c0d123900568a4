// Schwarz local solves and the coarse solve as ONE sync-free supernode sweep
// (forward then backward in a single launch), replacing the parallel_for of
// LLT / SimplicialLLT solves (/root/reference/proj/src/schwarz.cpp:155-167).
//
// Each supernode is ONE dense mat-vec over its row-tiled panel (host/pack.cpp):
//   forward : [y_S ; u_S] = F (r_S - sum of incoming descendant updates u_D)
//   backward: x_S         = H [y_S ; -x_R]
// cut into work units of <= 44 KB of panel: runs of whole 32-row tiles, or
// balanced column chunks of one wide tile.
//
// Scheduling: resident CTAs take tickets; tickets follow a simulated
// critical-path list schedule (sim.cu), so forward and backward units
// interleave and a unit's dependencies always hold smaller tickets. A CTA
// holds up to two tickets (the unit it runs + one of lookahead whose
// descriptor and task record are fetched while it runs; deeper lookahead
// reserves critical units too early), and the lowest unfinished ticket is
// always running, so the sweep is deadlock-free without a grid barrier.
// A unit's panel is bulk-prefetched into L2 when the unit starts.
//
// Per unit the CTA splits by role: thread 0 polls the (at most two,
// precomputed) dependency counters, lane 1 of warp 0 fetches the lookahead
// unit, and warps 1-3 stage tile descriptors, gather maps and every input
// that does not depend on the awaited units. After the wait only one level of
// dependent loads (descendant update slices or ancestor x) and the mat-vec
// remain. Column chunks write 32 partial sums; the last chunk to arrive
// (atom.acq_rel) reduces them in chunk order, so results are deterministic.
// Results of other units are read with ld.cg; a unit publishes with barrier +
// one red.release.gpu. Counters are monotone across launches (sweep number
// `epoch`), so no memsets are needed between sweeps.
#include <cstdint>

#include "../host/problem.hpp"
#include "kernels.cuh"

#ifndef PDG_SPIN_NS
#define PDG_SPIN_NS 16  // back-off between dependency polls
#endif
#ifndef PDG_DOT_DEPTH
#define PDG_DOT_DEPTH 8
#endif
// PDG_SWEEP_MINB (build knob): minimum resident CTAs per SM the register
// allocation must allow. Unset = the compiler's own choice (58 registers,
// 8 CTAs/SM), which measured best; an explicit 1 lets it take 102.
#ifdef PDG_SWEEP_MINB
#define PDG_SWEEP_BOUNDS __launch_bounds__(NT, PDG_SWEEP_MINB)
#else
// 1024 resident threads per SM (8 CTAs of 128 or 16 of 64): at most 64 registers
#define PDG_SWEEP_BOUNDS __launch_bounds__(NT, 1024 / NT)
#endif
static_assert(PDG_DOT_DEPTH % 4 == 0, "tile_dot consumes loads four at a time");

namespace pdg {

namespace {

__device__ __forceinline__ int ld_acquire_s(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed_s(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_relaxed_add(int* p, int v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_acq_rel_add(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Spin with relaxed loads (each acquire load invalidates the SM's L1, which
// the other CTAs on the SM are using), then one acquire load for ordering.
// A count that never arrives is a schedule bug: fail the launch instead of
// hanging the device.
__device__ __forceinline__ void wait_count(const int* flag, int need) {
  // common case (the list schedule releases units after their dependencies):
  // one acquire load and done
  if (ld_acquire_s(flag) >= need) return;
  const long long t0 = clock64();
  do {
    __nanosleep(PDG_SPIN_NS);
    if (clock64() - t0 > (1LL << 33)) __trap();
  } while (ld_relaxed_s(flag) < need);
  (void)ld_acquire_s(flag);
}
// panel loads: read-only path; EF marks the lines evict-first in L2 once read,
// so consumed panel lines give way before prefetched, not-yet-read ones
template <bool EF>
__device__ __forceinline__ double2 ld_panel(const double2* p, unsigned long long pol) {
  if (!EF) return __ldg(p);
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(pol));
  return v;
}
// named barrier for the staging warps (1..kWarps-1) only
template <int NT>
__device__ __forceinline__ void staging_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(NT - 32) : "memory");
}

constexpr int kMaxSmemTiles = 32;
constexpr int kMetaCells = 160;  // staged in_ptr entries per unit
constexpr int kMetaIdx = 768;    // staged update offsets / row dof starts per unit
constexpr int kAhead = 2;  // ring: running unit + one lookahead unit

struct Ahead {
  DevUnit u;
  DevTask t;
  int tk;
};

struct UnitSmem {
  DevUnit u;  // running unit and its task
  DevTask t;
  int col_lo, col_hi, cell_lo, meta, last, ep, tk;
  union {
    struct {
      DevTile tiles[kMaxSmemTiles];
      int iptr[kMetaCells];
      long long idx[kMetaIdx];
    };
    alignas(16) int blob[kChunkMetaInts];  // a level chunk's record (host/problem.hpp LevelChunk)
  };
  Ahead q[kAhead];
  int qh;
  int seen_level;  // level chunks: the last level counter this CTA waited for (this sweep)
};

// takes the next ticket into lookahead slot `q`: descriptor, task record, and
// an L2 bulk prefetch of the unit's panel
__device__ __forceinline__ void fetch_ahead(const SweepArgs& a, Ahead& q) {
  const int tk = static_cast<int>(atomicAdd(a.ticket, 1u));
  q.tk = tk < a.n_units ? tk : a.n_units;
  if (tk < a.n_units) {
    q.u = a.units[tk];
    q.t = a.tasks[q.u.task];
    // a level chunk's record is the first thing its CTA needs: bring it to L2 now
    if (q.u.nchunk == 0)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.bmeta + q.u.in_e0), "r"(q.u.in_n * 4)
                   : "memory");
  }
}
// L2 bulk prefetch of the running unit's panel (issued when the unit starts:
// prefetching the lookahead units as well overcommits the L2)
__device__ __forceinline__ void prefetch_panel(const SweepArgs& a, const DevUnit& u) {
  const double* src = (u.dir == 0 ? a.fmat : a.hmat) + u.src_off;
  if (a.prefetch & 4) {  // prefetched lines evict-last until read (evict-first) by the unit
    unsigned long long pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(src), "r"(u.bytes), "l"(pol)
                 : "memory");
    return;
  }
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(u.bytes) : "memory");
}

// one warp: rows of tile `tl` restricted to input columns [j0, j1) of the
// panel `m` (tile base, global, L2-prefetched); (row 2*l2, row 2*l2+1) sums in half 0
template <bool EF>
__device__ __forceinline__ double2 tile_dot(const double* m, const DevTile& tl, const double* x, int j0, int j1) {
  unsigned long long pol = 0;
  if (EF) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const int lane = threadIdx.x & 31, half = lane >> 4, l2 = lane & 15;
  double2 acc0 = make_double2(0.0, 0.0), acc1 = acc0, acc2 = acc0, acc3 = acc0;
  if (2 * l2 < tl.rows) {
    const double2* mm = reinterpret_cast<const double2*>(m) + l2;
    const long long cs = tl.stride >> 1;
    int j = j0 + half;
    constexpr int D = PDG_DOT_DEPTH;  // double2 loads in flight per lane
    for (; j + 2 * D - 2 < j1; j += 2 * D) {
      double2 v[D];
#pragma unroll
      for (int u = 0; u < D; ++u) v[u] = ld_panel<EF>(mm + (j + 2 * u) * cs, pol);
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
      const double2 v0 = ld_panel<EF>(mm + j * cs, pol);
      acc0.x = fma(v0.x, x[j], acc0.x);
      acc0.y = fma(v0.y, x[j], acc0.y);
    }
  }
  double vx = (acc0.x + acc1.x) + (acc2.x + acc3.x), vy = (acc0.y + acc1.y) + (acc2.y + acc3.y);
  vx += __shfl_down_sync(0xffffffffu, vx, 16);
  vy += __shfl_down_sync(0xffffffffu, vy, 16);
  return make_double2(vx, vy);
}

// level chunks: one panel column entry per lane (row), read-only path with the
// same evict-first policy as the tiled panel loads
template <bool EF>
__device__ __forceinline__ double ld_col(const double* p, unsigned long long pol) {
  if (!EF) return __ldg(p);
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
// one warp, one tile of a level chunk (rows R <= 32, ncol a multiple of the
// block size BS), one row per lane. Tall tiles (R > 16): one column per load
// instruction, BS columns in flight, no predicates. Short tiles: the lanes form
// G = 32 / R column groups, G columns per load instruction, sixteen in flight;
// the group sums are added in group order. Row r's sum in lane r < R.
template <int BS, bool EF>
__device__ __forceinline__ double tile_rows(const double* m, int R, int stride, int ncol, const double* x,
                                            unsigned long long pol) {
  const int lane = threadIdx.x & 31;
  double acc0 = 0.0, acc1 = 0.0;
  if (R > 16) {
    if (lane < R) {
      const double* p = m + lane;
      for (int j = 0; j < ncol; j += BS) {
        double v[BS];
#pragma unroll
        for (int u = 0; u < BS; ++u) v[u] = ld_col<EF>(p + static_cast<long long>(j + u) * stride, pol);
#pragma unroll
        for (int u = 0; u < BS; ++u) {
          if (u & 1) acc1 = fma(v[u], x[j + u], acc1);
          else acc0 = fma(v[u], x[j + u], acc0);
        }
      }
    }
    return acc0 + acc1;
  }
  const int G = 32 / R, g = lane / R, r = lane - g * R;
  if (g < G) {
    const double* p = m + r;
    constexpr int D = 16;
    for (int j = g; j < ncol; j += D * G) {
      double v[D];
#pragma unroll
      for (int u = 0; u < D; ++u) {
        v[u] = 0.0;
        if (j + u * G < ncol) v[u] = ld_col<EF>(p + static_cast<long long>(j + u * G) * stride, pol);
      }
#pragma unroll
      for (int u = 0; u < D; ++u)
        if (j + u * G < ncol) {
          if (u & 1) acc1 = fma(v[u], x[j + u * G], acc1);
          else acc0 = fma(v[u], x[j + u * G], acc0);
        }
    }
  }
  const double acc = acc0 + acc1;
  double sum = acc;
  for (int k = 1; k < G; ++k) sum += __shfl_sync(0xffffffffu, acc, (lane + k * R) & 31);
  return sum;
}

// the tiles of a level chunk over the CTA's warps
template <int BS, bool FWD, bool EF, int NT>
__device__ __forceinline__ void chunk_tiles(const SweepArgs& a, const int* items, int nitem, const double* pan,
                                            const double* xin) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long pol = 0;
  if (EF) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  for (int it = warp; it < nitem; it += NT / 32) {
    const int4 e0 = *reinterpret_cast<const int4*>(items + 8 * it);
    const int4 e1 = *reinterpret_cast<const int4*>(items + 8 * it + 4);
    const int rows = e0.z & 63;
    const double val = tile_rows<BS, EF>(pan + e0.x, rows, e0.w, e0.y, xin + e1.x, pol);
    if (lane < rows && !(a.prefetch & 32)) {
      if (!FWD) a.z[e1.z + lane] = val;
      else if (lane < e1.y) ((e0.z >> 30) ? a.z : a.yf)[e1.z + lane] = val;
      else a.ubuf[e1.w + lane] = val;
    }
  }
}

template <bool FWD>
__device__ __forceinline__ void store_row(const SweepArgs& a, const DevTask& T, double* outv, int o, double v) {
  // forward y_S goes to its own buffer: a task's backward units read all of
  // y_S while their siblings already overwrite the output with x_S
  if (!FWD) outv[T.dof0 + o] = v;
  else if (T.pad) (T.coarse ? a.y0 : a.z)[T.dof0 + o] = v;  // dense root: x_S = inv(K_SS) t_S
  else if (o < T.w) (T.coarse ? a.yc : a.yf)[T.dof0 + o] = v;
  else a.ubuf[T.ubuf_off + (o - T.w)] = v;
}

// warps 1..3: everything that does not depend on the awaited units
template <bool FWD, int NT>
__device__ __forceinline__ void stage(const SweepArgs& a, UnitSmem& s, double* xin) {
  const int t = threadIdx.x - 32;  // 0 .. NT-33
  const int nst = NT - 32;
  const DevUnit& U = s.u;
  const DevTask& T = s.t;
  if (t == 0 && (a.prefetch & 1)) prefetch_panel(a, U);
  // every load below depends only on the (host-precomputed) descriptor, so
  // the whole staging is one round of independent loads
  const int tile0 = (FWD ? T.f_tile0 : T.h_tile0) + U.tile_begin;
  const int ntile = U.tile_end - U.tile_begin;
  const DevTile* tiles = FWD ? a.ftiles : a.htiles;
  for (int i = t; i < ntile && i < kMaxSmemTiles; i += nst) s.tiles[i] = tiles[tile0 + i];
  const int bs = T.bs, w = T.w;
  const int col_lo = U.col_lo, col_hi = U.col_hi;
  const int cell_lo = col_lo / bs, cell_hi = (col_hi + bs - 1) / bs;
  if (t == 0) {
    s.col_lo = col_lo;
    s.col_hi = col_hi;
    s.cell_lo = cell_lo;
  }
  int meta = 0;
  if (FWD) {
    // independent part of the inputs: r (or r0) itself
    if (T.coarse && a.r0part) {
      // r0 = sum of the restriction chunks of each coarse node, in chunk order
      // (the restrict_combine kernel folded into the coarse forward staging)
      for (int i = col_lo + t; i < col_hi; i += nst) {
        const int d = static_cast<int>(T.dof0) + i, node = d / bs, m = d - node * bs;
        double v = 0.0;
        for (int c = a.node_chunk_ptr[node]; c < a.node_chunk_ptr[node + 1]; ++c) v += a.r0part[c * bs + m];
        xin[i - col_lo] = v;
      }
    } else {
      const double* in = T.coarse ? a.r0 : a.r;
      for (int i = col_lo + t; i < col_hi; i += nst) xin[i - col_lo] = in[T.dof0 + i];
    }
    const int nc = cell_hi - cell_lo;
    if (nc + 1 <= kMetaCells && U.in_n <= kMetaIdx) {
      for (int c = t; c <= nc; c += nst) s.iptr[c] = a.in_ptr[T.in_off + cell_lo + c];
      for (int k = t; k < U.in_n; k += nst) s.idx[k] = a.in_idx[U.in_e0 + k];
      meta = 1;
    }
  } else {
    const int r_lo = max(col_lo, w);
    const int rc0 = (r_lo - w) / bs;
    const int nr_cells = col_hi > w ? (col_hi - w + bs - 1) / bs - rc0 : 0;
    if (nr_cells <= kMetaIdx) {
      for (int k = t; k < nr_cells; k += nst) s.idx[k] = a.row_dof[T.rows_off + rc0 + k];
      meta = 1;
    }
    // own y_S (this task's forward result) is independent of the awaited ancestors
    if (U.own_fwd >= 0 && col_lo < w) {
      if (t == 0) wait_count(a.flags + U.own_fwd, (s.ep + 1) * U.own_need);
      staging_sync<NT>();
      const double* ybuf = T.coarse ? a.yc : a.yf;
      for (int i = col_lo + t; i < min(col_hi, w); i += nst) xin[i - col_lo] = __ldcg(ybuf + T.dof0 + i);
    }
  }
  if (t == 0) {
    s.meta = meta;
    if (a.trace) a.trace[8LL * s.tk + 4] = gtimer();
  }
}

template <bool FWD, bool EF, int NT>
__device__ __forceinline__ void run_unit(const SweepArgs& a, UnitSmem& s, double* xin, double* part, int tk) {
  long long* tr = a.trace ? a.trace + 8LL * tk : nullptr;
  const int ep = s.ep;
  if (threadIdx.x == 0) {
    if (tr) tr[0] = gtimer();
    const DevUnit& U = s.u;
    if (U.n_dep <= 2) {
      for (int d = 0; d < U.n_dep; ++d) wait_count(a.flags + U.dep[d], (ep + 1) * U.need[d]);
    } else {  // many children: walk the task's child list
      const DevTask& T = s.t;
      for (int k = 0; k < T.n_child; ++k) {
        const int c = a.task_child[T.child_off + k];
        wait_count(a.flags + c, (ep + 1) * a.tasks[c].f_ntile);
      }
    }
    if (tr) tr[1] = gtimer();
  } else if (threadIdx.x == 1) {
    // lookahead: q[qh] is the next unit; the slot after it (freed when the
    // running unit was copied out) takes the next ticket
    const int target = (s.qh + kAhead - 2) % kAhead, latest = (target + kAhead - 1) % kAhead;
    Ahead& q = s.q[target];
    if (s.q[latest].tk < a.n_units) fetch_ahead(a, q);
    else q.tk = a.n_units;
  } else if (threadIdx.x >= 32) {
    stage<FWD, NT>(a, s, xin);
  }
  __syncthreads();
  const DevUnit& U = s.u;
  const DevTask& T = s.t;
  const int w = T.w, bs = T.bs;
  const int col_lo = s.col_lo, col_hi = s.col_hi, cell_lo = s.cell_lo;
  const bool meta = s.meta;
  double* outv = T.coarse ? a.y0 : a.z;
  // the one dependent gather level
  if (FWD && meta) {
    // two columns per pass, their update loads issued four at a time before
    // any is consumed; each column subtracts its updates in list order (same
    // sums as one load per step, fewer dependent round trips)
    const int e0 = s.iptr[0];
    for (int i0 = col_lo + threadIdx.x; i0 < col_hi; i0 += 2 * blockDim.x) {
      int kk[2], ke[2], rr[2];
      double v[2];
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const int i = i0 + g * blockDim.x;
        const bool on = i < col_hi;
        const int cell = on ? i / bs : cell_lo;
        rr[g] = on ? i - cell * bs : 0;
        kk[g] = on ? s.iptr[cell - cell_lo] : 0;
        ke[g] = on ? s.iptr[cell - cell_lo + 1] : 0;
        v[g] = on ? xin[i - col_lo] : 0.0;
      }
      while (kk[0] < ke[0] || kk[1] < ke[1]) {
        double t[2][4];
#pragma unroll
        for (int g = 0; g < 2; ++g)
#pragma unroll
          for (int u = 0; u < 4; ++u)
            t[g][u] = kk[g] + u < ke[g] ? __ldcg(a.ubuf + s.idx[kk[g] + u - e0] + rr[g]) : 0.0;
#pragma unroll
        for (int g = 0; g < 2; ++g) {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (kk[g] + u < ke[g]) v[g] -= t[g][u];
          kk[g] = min(kk[g] + 4, ke[g]);
        }
      }
#pragma unroll
      for (int g = 0; g < 2; ++g)
        if (i0 + g * static_cast<int>(blockDim.x) < col_hi) xin[i0 + g * blockDim.x - col_lo] = v[g];
    }
  } else if (FWD) {
    for (int i = col_lo + threadIdx.x; i < col_hi; i += blockDim.x) {
      const int cell = i / bs, rr = i - cell * bs;
      double v = xin[i - col_lo];
      {
        const int k0 = a.in_ptr[T.in_off + cell], k1 = a.in_ptr[T.in_off + cell + 1];
        for (int k = k0; k < k1; ++k) v -= __ldcg(a.ubuf + a.in_idx[k] + rr);
      }
      xin[i - col_lo] = v;
    }
  } else {
    const int rc0 = (max(col_lo, w) - w) / bs;
    const int i_start = (U.own_fwd >= 0) ? max(col_lo, w) : col_lo;  // own y already staged
    for (int i = i_start + threadIdx.x; i < col_hi; i += blockDim.x) {
      double v;
      if (i < w) {
        v = __ldcg((T.coarse ? a.yc : a.yf) + T.dof0 + i);
      } else {
        const int k = i - w, cell = k / bs, rr = k - cell * bs;
        const long long base = meta ? s.idx[cell - rc0] : a.row_dof[T.rows_off + cell];
        v = -__ldcg(outv + base + rr);
      }
      xin[i - col_lo] = v;
    }
  }
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[2] = gtimer();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, l2 = lane & 15;
  const int ntile = U.tile_end - U.tile_begin;
  if (U.nchunk > 1) {
    // one tile, columns [c0, c1): warps split the columns, partials to global
    const DevTile tl = s.tiles[0];
    const int nc = U.c1 - U.c0;
    const int per = (((nc + (NT / 32) - 1) / (NT / 32)) + 1) & ~1;
    const int j0 = warp * per, j1 = min(nc, j0 + per);
    const double2 v = tile_dot<EF>((FWD ? a.fmat : a.hmat) + U.src_off, tl, xin, j0, j1);
    if (lane < 16) {
      part[warp * 32 + 2 * l2] = v.x;
      part[warp * 32 + 2 * l2 + 1] = v.y;
    }
    if (tr && threadIdx.x == 0) tr[5] = gtimer();
    __syncthreads();
    double* gp = a.part + static_cast<long long>(U.part_base + U.chunk) * 32;
    if (threadIdx.x < 32) {
      double sum = 0.0;
      for (int q = 0; q < (NT / 32); ++q) sum += part[q * 32 + threadIdx.x];
      __stcg(gp + threadIdx.x, sum);
    }
    __syncthreads();
    if (threadIdx.x == 0) s.last = atom_acq_rel_add(a.tile_ctr + U.tile_ctr, 1) + 1 == (ep + 1) * U.nchunk;
    __syncthreads();
    if (!s.last) {
      if (tr && threadIdx.x == 0) tr[3] = gtimer();
      return;
    }
    if (threadIdx.x < tl.rows) {
      double sum = 0.0;
      const double* base = a.part + static_cast<long long>(U.part_base) * 32 + threadIdx.x;
      for (int c = 0; c < U.nchunk; ++c) sum += __ldcg(base + c * 32);
      store_row<FWD>(a, T, outv, U.tile_begin * 32 + threadIdx.x, sum);
    }
    __syncthreads();
    if (threadIdx.x == 0) red_release_add(a.flags + (FWD ? 0 : a.n_tasks) + U.task, 1);
    if (tr && threadIdx.x == 0) tr[3] = gtimer();
    return;
  }
  // whole tiles: items = (tile, column split) over the warps
  const int split = ntile >= (NT / 32) ? 1 : (NT / 32) / ntile;
  const int items = ntile * split;
  const DevTile* gtiles = (FWD ? a.ftiles : a.htiles) + (FWD ? T.f_tile0 : T.h_tile0) + U.tile_begin;
  for (int it = warp; it < items; it += (NT / 32)) {
    const int R = it / split, c = it - R * split;
    const DevTile tl = R < kMaxSmemTiles ? s.tiles[R] : gtiles[R];
    const double* m = (FWD ? a.fmat : a.hmat) + tl.off;
    const int chunk = (((tl.ncol + split - 1) / split) + 1) & ~1;
    const int j0 = c * chunk, j1 = min(tl.ncol, j0 + chunk);
    const double2 v = tile_dot<EF>(m, tl, xin + (tl.col0 - col_lo), j0, j1);
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
      if (l >= s.tiles[R].rows) continue;
      double v = 0.0;
      for (int c = 0; c < split; ++c) v += part[(R * split + c) * 32 + l];
      store_row<FWD>(a, T, outv, (U.tile_begin + R) * 32 + l, v);
    }
  }
  if (tr && threadIdx.x == 0) tr[5] = gtimer();
  __syncthreads();
  if (threadIdx.x == 0) red_release_add(a.flags + (FWD ? 0 : a.n_tasks) + U.task, ntile);
  if (tr && threadIdx.x == 0) tr[3] = gtimer();
}

// A level chunk (host/problem.hpp LevelChunk): some bottom-level supernodes of
// one tree height, all independent of each other. The CTA gathers the inputs
// of all of them into shared memory (forward: r_S minus the descendants'
// updates; backward: [y_S ; -x_R]), one barrier, then one warp per 32-row
// tile (tile_rows). A forward chunk waits for the previous level's counter,
// adds to its own level's, and publishes the task counters of its supernodes
// whose parent is scheduled individually; a backward chunk waits for the level
// above (the top level: for the last forward level) and for those parents.
template <bool FWD, bool EF, int NT>
__device__ __forceinline__ void run_chunk(const SweepArgs& a, UnitSmem& s, double* xin, int tk) {
  long long* tr = a.trace ? a.trace + 8LL * tk : nullptr;
  const int ep = s.ep;
  const DevUnit& U = s.u;
  if (threadIdx.x < 32) {
    if (tr && threadIdx.x == 0) tr[0] = gtimer();
    // the level counter this CTA already saw complete needs no second acquire
    if (threadIdx.x == 0 && U.n_dep && s.seen_level != U.dep[0]) {
      wait_count(a.flags + U.dep[0], (ep + 1) * U.need[0]);
      s.seen_level = U.dep[0];
    }
    if (!FWD)
      for (int d = threadIdx.x; d < U.c1; d += 32) {
        const int2 w = a.bdeps[U.c0 + d];
        wait_count(a.flags + w.x, (ep + 1) * w.y);
      }
    __syncwarp();
    if (tr && threadIdx.x == 0) tr[1] = gtimer();
  } else {
    const int t = threadIdx.x - 32;
    if (t == 0 && (a.prefetch & 1)) prefetch_panel(a, U);
    const int4* src = reinterpret_cast<const int4*>(a.bmeta + U.in_e0);
    int4* dst = reinterpret_cast<int4*>(s.blob);
    for (int i = t; i < (U.in_n >> 2); i += NT - 32) dst[i] = __ldg(src + i);
    if (tr && t == 0) tr[4] = gtimer();
  }
  __syncthreads();
  const int ncell = s.blob[0], nitem = s.blob[1], naux = s.blob[2];
  const int* cells = s.blob + 4;
  const int* aux = cells + (FWD ? 4 : 2) * ncell;
  // items start 16-byte aligned (the header, cells and aux are padded by the host)
  const int* items = aux + ((naux + 3) & ~3);
  const int bs = s.t.bs;
  const double* pan = (FWD ? a.fmat : a.hmat) + U.src_off;
  // warp 0 takes the lookahead ticket (three dependent round trips) while the
  // other warps gather
  if (threadIdx.x < 32) {
    if (threadIdx.x == 1) {
      const int target = (s.qh + kAhead - 2) % kAhead, latest = (target + kAhead - 1) % kAhead;
      Ahead& q = s.q[target];
      if (s.q[latest].tk < a.n_units) fetch_ahead(a, q);
      else q.tk = a.n_units;
    }
  } else if (FWD) {
    for (int q = threadIdx.x - 32; q < ncell * bs; q += NT - 32) {
      const int cc = q / bs, rr = q - cc * bs;
      const int* ce = cells + 4 * cc;
      double x = a.r[ce[0] + rr];
      const int ke = ce[3];
      for (int k = ce[2]; k < ke && !(a.prefetch & 16); k += 4) {
        double t[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) t[u] = k + u < ke ? __ldcg(a.ubuf + aux[k + u] + rr) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (k + u < ke) x -= t[u];
      }
      xin[ce[1] + rr] = x;
    }
  } else {
    // two independent loads per thread per pass
    const int n = ncell * bs;
    for (int q = threadIdx.x - 32; q < n; q += 2 * (NT - 32)) {
      const int q1 = q + NT - 32;
      const int c0 = q / bs, r0 = q - c0 * bs, s0 = cells[2 * c0];
      const bool two = q1 < n;
      const int c1 = two ? q1 / bs : c0, r1 = two ? q1 - c1 * bs : r0, s1 = cells[2 * c1];
      const bool dbg = (a.prefetch & 16) != 0;
      const double v0 = dbg ? 1.0 : s0 >= 0 ? __ldcg(a.yf + s0 + r0) : -__ldcg(a.z + (-1 - s0) + r0);
      const double v1 = dbg ? 1.0 : s1 >= 0 ? __ldcg(a.yf + s1 + r1) : -__ldcg(a.z + (-1 - s1) + r1);
      xin[cells[2 * c0 + 1] + r0] = v0;
      if (two) xin[cells[2 * c1 + 1] + r1] = v1;
    }
  }
  __syncthreads();
  if (tr && threadIdx.x == 0) tr[2] = gtimer();
  switch (bs) {
    case 3: chunk_tiles<3, FWD, EF, NT>(a, items, nitem, pan, xin); break;
    case 6: chunk_tiles<6, FWD, EF, NT>(a, items, nitem, pan, xin); break;
    case 10: chunk_tiles<10, FWD, EF, NT>(a, items, nitem, pan, xin); break;
    case 15: chunk_tiles<15, FWD, EF, NT>(a, items, nitem, pan, xin); break;
    default: chunk_tiles<1, FWD, EF, NT>(a, items, nitem, pan, xin); break;
  }
  __syncthreads();
  // publish: one release fence for warp 0 (the barrier ordered the CTA's
  // stores before it), then relaxed additions spread over its lanes
  if (threadIdx.x < 32) {
    if (tr && threadIdx.x == 0) {
      tr[5] = gtimer();
      tr[7] = nitem;
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    if (FWD)
      for (int k = threadIdx.x; k < U.tile_ctr; k += 32) {
        const int2 r = a.broots[U.part_base + k];
        red_relaxed_add(a.flags + r.x, r.y);
      }
    if (threadIdx.x == 0) {
      red_relaxed_add(a.flags + U.own_fwd, 1);
      if (U.chunk >= 0) red_relaxed_add(a.flags + U.chunk, 1);
    }
    if (tr && threadIdx.x == 0) tr[3] = gtimer();
  }
}

template <bool EF, int NT>
__global__ void PDG_SWEEP_BOUNDS sweep_kernel(SweepArgs a) {
  pdl_wait();
  if (a.S && a.S->stop) return;
  extern __shared__ __align__(128) double sm[];
  __shared__ UnitSmem s;
  double* part = sm;  // NT doubles
  double* xin = part + NT;
  if (threadIdx.x == 0) {
    // live duration of every launch (first CTA start -> last CTA end, read by
    // bench.py over its timed region)
    if (blockIdx.x == 0 && a.live) a.live[0] = static_cast<unsigned long long>(gtimer());
    s.ep = __ldcg(a.epoch);
    for (int i = 0; i + 1 < kAhead; ++i) {
      if (i == 0 || s.q[i - 1].tk < a.n_units) fetch_ahead(a, s.q[i]);
      else s.q[i].tk = a.n_units;
    }
    s.q[kAhead - 1].tk = a.n_units;
    s.qh = 0;
    s.seen_level = -1;
  }
  __syncthreads();
  // slot layout: q[qh] running, q[qh+1] next, q[qh+2] fetched during the run
  for (;;) {
    // warp 0 copies the descriptor and task record out of the ring and
    // advances the ring head; one barrier publishes both
    if (threadIdx.x < 32) {
      const Ahead& cur = s.q[s.qh];
      constexpr int nu = sizeof(DevUnit) / 4, nt = sizeof(DevTask) / 4;
      for (int i = threadIdx.x; i < nu + nt; i += 32) {
        if (i < nu) reinterpret_cast<int*>(&s.u)[i] = reinterpret_cast<const int*>(&cur.u)[i];
        else reinterpret_cast<int*>(&s.t)[i - nu] = reinterpret_cast<const int*>(&cur.t)[i - nu];
      }
      __syncwarp();
      if (threadIdx.x == 0) {
        s.tk = cur.tk;
        s.qh = s.qh == kAhead - 1 ? 0 : s.qh + 1;
      }
    }
    __syncthreads();
    const int tk = s.tk;
    if (tk >= a.n_units) break;
    if (s.u.nchunk == 0) {
      if (s.u.dir == 0) run_chunk<true, EF, NT>(a, s, xin, tk);
      else run_chunk<false, EF, NT>(a, s, xin, tk);
    } else if (s.u.dir == 0) {
      run_unit<true, EF, NT>(a, s, xin, part, tk);
    } else {
      run_unit<false, EF, NT>(a, s, xin, part, tk);
    }
    __syncthreads();
  }
  // the last CTA of this sweep resets the tickets and advances the epoch
  if (threadIdx.x == 0) {
    if (atomicAdd(a.epoch + 1, 1) == static_cast<int>(gridDim.x) - 1) {
      a.epoch[1] = 0;
      *a.ticket = 0u;
      a.epoch[0] = s.ep + 1;
      if (a.live) {
        a.live[1] += static_cast<unsigned long long>(gtimer()) - __ldcg(a.live);
        a.live[2] += 1;
      }
      __threadfence();
    }
  }
}


}  // namespace

int sweep_smem_bytes(int xcap, int threads) { return static_cast<int>(sizeof(double)) * (threads + xcap); }

template <int NT>
static int ctas_per_sm(int smem) {
  int per_sm = 0;
  PDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sweep_kernel<false, NT>, NT, smem));
  return per_sm > 0 ? per_sm : 1;
}

void launch_sweep(const SweepArgs& a, int smem, cudaStream_t st) {
  if (a.n_units == 0) return;
  static int cached_smem = -1, cached_threads = -1, resident = 0;
  if (cached_smem != smem || cached_threads != a.threads) {
    int sms = 0, dev = 0;
    PDG_CUDA(cudaGetDevice(&dev));
    PDG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    resident = (a.threads == 64 ? ctas_per_sm<64>(smem) : ctas_per_sm<128>(smem)) * sms;
    cached_smem = smem;
    cached_threads = a.threads;
  }
  const int grid = a.n_units < resident ? a.n_units : resident;
  const bool ef = (a.prefetch & 2) != 0;
  if (a.threads == 64) {
    if (ef) launch_pdl(sweep_kernel<true, 64>, grid, 64, smem, st, a);
    else launch_pdl(sweep_kernel<false, 64>, grid, 64, smem, st, a);
  } else {
    if (ef) launch_pdl(sweep_kernel<true, 128>, grid, 128, smem, st, a);
    else launch_pdl(sweep_kernel<false, 128>, grid, 128, smem, st, a);
  }
}

int sweep_ctas_per_sm(int smem, int threads) { return threads == 64 ? ctas_per_sm<64>(smem) : ctas_per_sm<128>(smem); }

void set_sweep_smem(int bytes) {
  PDG_CUDA(cudaFuncSetAttribute(sweep_kernel<false, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  PDG_CUDA(cudaFuncSetAttribute(sweep_kernel<true, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  PDG_CUDA(cudaFuncSetAttribute(sweep_kernel<false, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  PDG_CUDA(cudaFuncSetAttribute(sweep_kernel<true, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
}

}  // namespace pdg
