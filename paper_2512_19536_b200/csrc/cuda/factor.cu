// Numeric supernodal Cholesky of the Schwarz subdomain matrices on the device
// (replaces the host half of the reference's
// SimplicialLLT setup, schwarz.cpp:114-136, and host/factor.cpp's numeric
// loop). The host builds the symbolic plan (supernodes in nested-dissection
// order, below rows, left-looking updaters; Problem::FactorSn/FactorUpd);
// the GPU then, level by level of the elimination forest (all subdomains at
// once, one CTA per supernode):
//   1. assembles the panel P_S (H x w) from the device copy of K,
//   2. subtracts the left-looking updates L_D[rows >= S] L_D[rows in S]^T of
//      every descendant D (ascending, so the result is deterministic),
//   3. factors P_S with a blocked right-looking Cholesky (32-column panels,
//      smem-tiled FP64 trailing updates): L_SS and L_RS in place,
//   4. inverts L_SS by 32 x 32 blocks (X_ij = -X_ii sum_k L_ik X_kj),
//   5. writes inv(L_SS) (packed lower) and L_RS to the factor-value buffer
//      that panels.cu turns into the sweep panels.
// Everything is FP64; a non-positive pivot sets an error flag (the host
// raises SolverError like the reference, schwarz.cpp:130-134).
#include <cstdint>
#include <vector>

#include "common.cuh"
#include "sim.cuh"

namespace pdg {

namespace {

using FSn = Problem::FactorSn;
using FUpd = Problem::FactorUpd;

constexpr int kT = 256;  // threads per CTA

// P(i, j) of a column-major panel with leading dimension ld
__device__ __forceinline__ double& at(double* P, int ld, int i, int j) {
  return P[static_cast<long long>(j) * ld + i];
}

__global__ void __launch_bounds__(kT) assemble_kernel(const FSn* __restrict__ sn, const int* __restrict__ rows,
                                                      const int* __restrict__ kptr, const int* __restrict__ kcol,
                                                      const double* __restrict__ kval, int bs, double* P) {
  const FSn S = sn[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, b2 = bs * bs;
  const int nc = S.s1 - S.s0;
  double* Ps = P + S.p_off;
  const int* R = rows + S.rows_off;
  for (int jc = warp; jc < nc; jc += kT / 32) {
    const int row = S.cell0 + S.s0 + jc;
    for (int kk = kptr[row]; kk < kptr[row + 1]; ++kk) {
      const int ip = kcol[kk] - S.cell0;
      if (ip < S.s0 + jc || ip >= S.ucells) continue;  // lower part, inside the unit
      int rc;
      if (ip < S.s1) {
        rc = ip - S.s0;
      } else {
        int lo = 0, hi = S.nrows;  // rows are sorted
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (R[mid] < ip) lo = mid + 1;
          else hi = mid;
        }
        rc = nc + lo;
      }
      for (int q = lane; q < b2; q += 32) {
        const int rr = q / bs, c = q - rr * bs;
        at(Ps, S.H, rc * bs + rr, jc * bs + c) = kval[static_cast<long long>(kk) * b2 + q];
      }
    }
  }
}

// acc(lg + 8q, jj) += sum_t A(l, t) B(jj, t) over one 32-wide t chunk staged in As/Bs
__device__ __forceinline__ void tile_fma(const double (*As)[33], const double (*Bs)[33], int jj, int lg,
                                         double acc[4]) {
#pragma unroll 8
  for (int t = 0; t < 32; ++t) {
    const double bv = Bs[jj][t];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] = fma(As[lg + 8 * q][t], bv, acc[q]);
  }
}

__global__ void __launch_bounds__(kT) factor_level_kernel(const int* __restrict__ ids, const FSn* __restrict__ sn,
                                                          const int* __restrict__ rows, const FUpd* __restrict__ upd,
                                                          const int* __restrict__ map,
                                                          const long long* __restrict__ lv_off,  // (linv, b) per task
                                                          const long long* __restrict__ x_off, double* P,
                                                          double* lval, double* Xbuf, int bs, int* err) {
  __shared__ double As[32][33];
  __shared__ double Bs[32][33];
  __shared__ double s_inv;
  const int tid = threadIdx.x, jj = tid & 31, lg = tid >> 5, lane = tid & 31, warp = tid >> 5;
  const int task = ids[blockIdx.x];
  const FSn S = sn[task];
  const int w = S.w, H = S.H;
  double* Ps = P + S.p_off;

  // ---- 2. left-looking updates, descendants in ascending order ----
  for (int ui = 0; ui < S.nupd; ++ui) {
    const FUpd u = upd[S.upd_off + ui];
    const FSn D = sn[u.d];
    const int nrD = D.H - D.w, wD = D.w;
    const double* BD = lval + lv_off[2 * u.d + 1];  // L_RS of D, nrD x wD column-major
    const int* RD = rows + D.rows_off;
    const int ni = (u.nrd - u.a) * bs, nj = (u.ce - u.a) * bs, src0 = u.a * bs;
    for (int jt = 0; jt < nj; jt += 32) {
      for (int it = jt; it < ni; it += 32) {  // tile-level lower part (k >= l)
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int t0 = 0; t0 < wD; t0 += 32) {
          for (int e = tid; e < 32 * 32; e += kT) {
            const int l = e & 31, tt = e >> 5, t = t0 + tt;
            As[l][tt] = (it + l < ni && t < wD) ? BD[src0 + it + l + static_cast<long long>(t) * nrD] : 0.0;
            Bs[l][tt] = (jt + l < nj && t < wD) ? BD[src0 + jt + l + static_cast<long long>(t) * nrD] : 0.0;
          }
          __syncthreads();
          tile_fma(As, Bs, jj, lg, acc);
          __syncthreads();
        }
        const int jo = jt + jj;
        if (jo < nj) {
          const int lc = jo / bs, cc = jo - lc * bs;
          const int colP = (RD[u.a + lc] - S.s0) * bs + cc;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int io = it + lg + 8 * q;
            if (io >= ni) continue;
            const int kc = io / bs, rr = io - kc * bs;
            if (kc < lc) continue;  // strictly upper cell blocks are not part of the update
            at(Ps, H, map[u.map_off + kc] * bs + rr, colP) -= acc[q];
          }
        }
      }
    }
    __syncthreads();
  }

  // ---- 3. blocked right-looking Cholesky of P (w columns, H rows) ----
  for (int jb = 0; jb < w; jb += 32) {
    const int nb = min(32, w - jb);
    for (int j = jb; j < jb + nb; ++j) {
      if (tid == 0) {
        double d = at(Ps, H, j, j);
        if (!(d > 0.0) || !isfinite(d)) {
          atomicCAS(err, 0, task + 1);
          d = 1.0;
        }
        d = sqrt(d);
        at(Ps, H, j, j) = d;
        s_inv = 1.0 / d;
      }
      __syncthreads();
      const double inv = s_inv;
      for (int i = j + 1 + tid; i < H; i += kT) at(Ps, H, i, j) *= inv;
      __syncthreads();
      for (int k = j + 1 + warp; k < jb + nb; k += kT / 32) {
        const double lkj = at(Ps, H, k, j);
        for (int i = k + lane; i < H; i += 32) at(Ps, H, i, k) -= at(Ps, H, i, j) * lkj;
      }
      __syncthreads();
    }
    // trailing update: P(i, k) -= sum_{t in panel} P(i, t) P(k, t), k >= jb + nb, i >= k (tile level)
    for (int kt = jb + nb; kt < w; kt += 32) {
      for (int it = kt; it < H; it += 32) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int e = tid; e < 32 * 32; e += kT) {
          const int l = e & 31, tt = e >> 5;
          As[l][tt] = (it + l < H && tt < nb) ? at(Ps, H, it + l, jb + tt) : 0.0;
          Bs[l][tt] = (kt + l < w && tt < nb) ? at(Ps, H, kt + l, jb + tt) : 0.0;
        }
        __syncthreads();
        tile_fma(As, Bs, jj, lg, acc);
        __syncthreads();
        const int k = kt + jj;
        if (k < w) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int i = it + lg + 8 * q;
            if (i < H && i >= k) at(Ps, H, i, k) -= acc[q];
          }
        }
      }
    }
    __syncthreads();
  }

  // ---- 4. X = inv(L_SS), 32 x 32 blocks, column-major w x w scratch ----
  double* X = Xbuf + x_off[blockIdx.x];
  const int nbk = (w + 31) / 32;
  for (int ib = 0; ib < nbk; ++ib) {  // diagonal blocks by forward substitution, one column per thread
    const int r0 = ib * 32, nb = min(32, w - r0);
    for (int e = tid; e < 32 * 32; e += kT) {
      const int l = e & 31, c = e >> 5;
      As[l][c] = (l < nb && c < nb && l >= c) ? at(Ps, H, r0 + l, r0 + c) : 0.0;
    }
    __syncthreads();
    if (tid < nb) {
      const int c = tid;
      for (int r = 0; r < nb; ++r) {
        double v = r == c ? 1.0 : 0.0;
        if (r > c)
          for (int m = c; m < r; ++m) v -= As[r][m] * Bs[m][c];
        Bs[r][c] = r < c ? 0.0 : v / As[r][r];
      }
    }
    __syncthreads();
    for (int e = tid; e < 32 * 32; e += kT) {
      const int l = e & 31, c = e >> 5;
      if (l < nb && c < nb) X[static_cast<long long>(r0 + c) * w + r0 + l] = Bs[l][c];
    }
    __syncthreads();
  }
  for (int jbk = 0; jbk < nbk; ++jbk) {
    for (int ibk = jbk + 1; ibk < nbk; ++ibk) {
      // T = sum_{k = jbk}^{ibk - 1} L(ib, k) X(k, jb) ; then X(ib, jb) = -X(ib, ib) T
      const int i0 = ibk * 32, j0 = jbk * 32;
      double acc[4] = {0.0, 0.0, 0.0, 0.0};
      for (int kb = jbk; kb < ibk; ++kb) {
        const int k0 = kb * 32;
        for (int e = tid; e < 32 * 32; e += kT) {
          const int l = e & 31, tt = e >> 5;  // As[l][tt] = L(i0 + l, k0 + tt) ; Bs[l][tt] = X(k0 + tt, j0 + l)
          As[l][tt] = (i0 + l < w && k0 + tt < w) ? at(Ps, H, i0 + l, k0 + tt) : 0.0;
          Bs[l][tt] = (k0 + tt < w && j0 + l < w) ? X[static_cast<long long>(j0 + l) * w + k0 + tt] : 0.0;
        }
        __syncthreads();
        tile_fma(As, Bs, jj, lg, acc);
        __syncthreads();
      }
      // stage T (As) and X(ib, ib) (Bs, transposed for tile_fma), then X(ib, jb) = -X(ib, ib) T
#pragma unroll
      for (int q = 0; q < 4; ++q) As[lg + 8 * q][jj] = acc[q];  // As[i][j] = T(i, j)
      __syncthreads();
      double t2[4] = {0.0, 0.0, 0.0, 0.0};
      // X(ib, jb)(i, j) = -sum_m Xd(i, m) T(m, j): stage Xd rows in Bs as Bs[i][m]
      for (int e = tid; e < 32 * 32; e += kT) {
        const int l = e & 31, m = e >> 5;
        Bs[l][m] = (i0 + l < w && i0 + m < w) ? X[static_cast<long long>(i0 + m) * w + i0 + l] : 0.0;
      }
      __syncthreads();
#pragma unroll 8
      for (int m = 0; m < 32; ++m) {
        const double tv = As[m][jj];
#pragma unroll
        for (int q = 0; q < 4; ++q) t2[q] = fma(Bs[lg + 8 * q][m], tv, t2[q]);
      }
      __syncthreads();
      const int j = j0 + jj;
      if (j < w) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int i = i0 + lg + 8 * q;
          if (i < w) X[static_cast<long long>(j) * w + i] = -t2[q];
        }
      }
      __syncthreads();
    }
  }

  // ---- 5. write inv(L_SS) packed lower and L_RS ----
  double* Lo = lval + lv_off[2 * task];
  double* Bo = lval + lv_off[2 * task + 1];
  const int nr = H - w;
  for (int j = warp; j < w; j += kT / 32) {
    double* col = Lo + static_cast<long long>(j) * w - static_cast<long long>(j) * (j - 1) / 2 - j;
    for (int i = j + lane; i < w; i += 32) col[i] = X[static_cast<long long>(j) * w + i];
    for (int i = lane; i < nr; i += 32) Bo[static_cast<long long>(j) * nr + i] = at(Ps, H, w + i, j);
  }
}

}  // namespace

void DeviceSim::device_factor(double* d_lval) {
  const Problem& pr = *P;
  const int nf = static_cast<int>(pr.fsn.size());
  if (nf == 0) return;
  // tasks by height: a supernode's descendants all have smaller heights
  int hmax = 0;
  for (const auto& f : pr.fsn) hmax = std::max(hmax, f.height);
  std::vector<std::vector<int>> level(hmax + 1);
  for (int i = 0; i < nf; ++i) level[pr.fsn[i].height].push_back(i);
  std::vector<long long> lv(2 * static_cast<std::size_t>(nf));
  for (int i = 0; i < nf; ++i) {
    lv[2 * i] = pr.tasks[i].linv_off;
    lv[2 * i + 1] = pr.tasks[i].b_off;
  }
  // per-level scratch for inv(L_SS): offsets within the level, one buffer
  std::vector<long long> xoff(nf);
  long long xcap = 0;
  for (const auto& L : level) {
    long long o = 0;
    for (int i : L) {
      xoff[i] = o;
      o += static_cast<long long>(pr.fsn[i].w) * pr.fsn[i].w;
    }
    xcap = std::max(xcap, o);
  }
  std::vector<int> ids;
  std::vector<long long> xo;
  for (const auto& L : level)
    for (int i : L) {
      ids.push_back(i);
      xo.push_back(xoff[i]);
    }
  auto up = [&](const void* src, std::size_t bytes) {
    void* p = nullptr;
    PDG_CUDA(cudaMalloc(&p, bytes ? bytes : 1));
    if (bytes) PDG_CUDA(cudaMemcpyAsync(p, src, bytes, cudaMemcpyHostToDevice, st));
    return p;
  };
  auto* d_sn = static_cast<FSn*>(up(pr.fsn.data(), pr.fsn.size() * sizeof(FSn)));
  auto* d_rows = static_cast<int*>(up(pr.frows.data(), pr.frows.size() * sizeof(int)));
  auto* d_upd = static_cast<FUpd*>(up(pr.fupd.data(), pr.fupd.size() * sizeof(FUpd)));
  auto* d_map = static_cast<int*>(up(pr.fmap.data(), pr.fmap.size() * sizeof(int)));
  auto* d_lv = static_cast<long long*>(up(lv.data(), lv.size() * sizeof(long long)));
  auto* d_ids = static_cast<int*>(up(ids.data(), ids.size() * sizeof(int)));
  auto* d_xo = static_cast<long long*>(up(xo.data(), xo.size() * sizeof(long long)));
  double *d_P = nullptr, *d_X = nullptr;
  int* d_err = nullptr;
  PDG_CUDA(cudaMalloc(&d_P, std::max<long long>(pr.fp_len, 1) * sizeof(double)));
  PDG_CUDA(cudaMalloc(&d_X, std::max<long long>(xcap, 1) * sizeof(double)));
  PDG_CUDA(cudaMalloc(&d_err, sizeof(int)));
  PDG_CUDA(cudaMemsetAsync(d_P, 0, std::max<long long>(pr.fp_len, 1) * sizeof(double), st));
  PDG_CUDA(cudaMemsetAsync(d_err, 0, sizeof(int), st));
  assemble_kernel<<<nf, kT, 0, st>>>(d_sn, d_rows, d_ptr, d_col, d_kval, b, d_P);
  PDG_CUDA(cudaGetLastError());
  int first = 0;
  for (const auto& L : level) {
    const int cnt = static_cast<int>(L.size());
    if (cnt)
      factor_level_kernel<<<cnt, kT, 0, st>>>(d_ids + first, d_sn, d_rows, d_upd, d_map, d_lv, d_xo + first, d_P,
                                             d_lval, d_X, b, d_err);
    PDG_CUDA(cudaGetLastError());
    first += cnt;
  }
  int err = 0;
  PDG_CUDA(cudaMemcpyAsync(&err, d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
  PDG_CUDA(cudaStreamSynchronize(st));
  for (void* p : {static_cast<void*>(d_sn), static_cast<void*>(d_rows), static_cast<void*>(d_upd),
                  static_cast<void*>(d_map), static_cast<void*>(d_lv), static_cast<void*>(d_ids),
                  static_cast<void*>(d_xo), static_cast<void*>(d_P), static_cast<void*>(d_X),
                  static_cast<void*>(d_err)})
    cudaFree(p);
  if (err) throw SolverError("schwarz: subdomain factorization failed (not positive definite)");
}

}  // namespace pdg
