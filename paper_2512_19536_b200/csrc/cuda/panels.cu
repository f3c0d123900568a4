// Device-side formation of the Schwarz sweep panels (SURVEY.md §8(f) row 1,
// the packing half of the reference's factor setup, schwarz.cpp:99-146).
//
// The host computes the supernodal Cholesky factor (inv(L_SS) packed lower,
// L_RS column-major; host/factor.cpp) and lays the 32-row tiles out
// (host/pack.cpp). Here, per supernode S with w columns and nr below rows:
//   F = [ inv(L_SS) ; G ],  G = L_RS inv(L_SS)   (h x w, h = w + nr)
//   H = F^T
// G is an (nr x w) x (w x w, lower) product: smem-tiled FP64 (32 x 32 output
// blocks, 8 x 32 threads, 4 rows per thread), one CTA per forward tile.
// H is written by a tiled transpose of the finished forward tiles. All
// entries, including the zero upper triangle inside a tile and the padding
// row of odd tiles, are written explicitly.
#include <cstdint>

#include "common.cuh"
#include "sim.cuh"

namespace pdg {

namespace {

struct PanelTask {
  long long linv_off, b_off;
  int w, nr, f_tile0, dense;  // dense: root panel G = inv(L_SS)^T inv(L_SS) (full w x w)
};

__device__ __forceinline__ double linv_at(const double* L, int w, int m, int j) {
  // packed column-major lower: column j holds rows j..w-1
  return L[static_cast<long long>(j) * w - static_cast<long long>(j) * (j - 1) / 2 + (m - j)];
}

__global__ void __launch_bounds__(256) forward_panel_kernel(const PanelTask* __restrict__ tasks,
                                                            const int* __restrict__ tile_task,
                                                            const DevTile* __restrict__ tiles,
                                                            const double* __restrict__ lval,
                                                            double* __restrict__ fmat) {
  __shared__ double Bs[32][33];
  __shared__ double Ls[32][33];
  const int tid = threadIdx.x, jj = tid & 31, lg = tid >> 5;  // 8 row groups
  const int tix = blockIdx.x;
  const PanelTask T = tasks[tile_task[tix]];
  const DevTile tl = tiles[tix];
  const int r0 = (tix - T.f_tile0) * 32;
  const int w = T.w, nr = T.nr;
  const double* L = lval + T.linv_off;
  const double* B = lval + T.b_off;
  double* out = fmat + tl.off;
  for (int jb = 0; jb < tl.ncol; jb += 32) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    const bool any_g = T.dense || r0 + tl.rows > w;
    if (any_g) {
      // G rows of this tile: sum over m >= j of B(i - w, m) inv(L)(m, j);
      // dense root: sum over m >= max(i, j) of inv(L)(m, i) inv(L)(m, j)
      for (int mb = T.dense ? (min(r0, jb) & ~31) : jb; mb < w; mb += 32) {
        for (int e = tid; e < 32 * 32; e += 256) {
          const int l = e & 31, mm = e >> 5;  // Bs[l][mm] = B(r0 + l - w, mb + mm) or inv(L)(mb + mm, r0 + l)
          const int i = r0 + l, m = mb + mm;
          if (T.dense)
            Bs[l][mm] = (l < tl.rows && i < w && m < w && m >= i) ? linv_at(L, w, m, i) : 0.0;
          else
            Bs[l][mm] = (i >= w && l < tl.rows && m < w) ? B[static_cast<long long>(m) * nr + (i - w)] : 0.0;
          const int m2 = mb + l, j2 = jb + mm;  // Ls[l][mm] = inv(L)(mb + l, jb + mm)
          Ls[l][mm] = (m2 < w && j2 < w && m2 >= j2) ? linv_at(L, w, m2, j2) : 0.0;
        }
        __syncthreads();
#pragma unroll 8
        for (int mm = 0; mm < 32; ++mm) {
          const double lv = Ls[mm][jj];
#pragma unroll
          for (int q = 0; q < 4; ++q) acc[q] = fma(Bs[lg + 8 * q][mm], lv, acc[q]);
        }
        __syncthreads();
      }
    }
    const int j = jb + jj;
    if (j < tl.ncol) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int l = lg + 8 * q;
        if (l >= tl.stride) continue;
        const int i = r0 + l;
        double v = 0.0;
        if (l < tl.rows) v = T.dense ? acc[q] : i < w ? (i >= j ? linv_at(L, w, i, j) : 0.0) : acc[q];
        out[static_cast<long long>(j) * tl.stride + l] = v;
      }
    }
  }
}

// H tile (rows r0..r0+rows of H = columns of F, inputs i = r0 .. h-1):
// H(l, i - r0) = F(i, r0 + l), staged through shared memory one 32-row F tile
// at a time (reads along F's rows, writes along H's rows).
__global__ void __launch_bounds__(256) backward_panel_kernel(const PanelTask* __restrict__ tasks,
                                                             const int* __restrict__ tile_task,
                                                             const DevTile* __restrict__ htiles,
                                                             const DevTile* __restrict__ ftiles,
                                                             const double* __restrict__ fmat,
                                                             double* __restrict__ hmat) {
  __shared__ double S[32][33];
  const int tid = threadIdx.x;
  const int tix = blockIdx.x;
  const PanelTask T = tasks[tile_task[tix]];
  const DevTile ht = htiles[tix];
  const int r0 = ht.col0, h = T.w + T.nr;
  double* out = hmat + ht.off;
  for (int ib = r0; ib < h; ib += 32) {  // one forward tile: rows [ib, ib + 32)
    const DevTile ft = ftiles[T.f_tile0 + ib / 32];
    for (int e = tid; e < 32 * 32; e += 256) {
      const int ii = e & 31, l = e >> 5;  // S[l][ii] = F(ib + ii, r0 + l)
      const int j = r0 + l;
      S[l][ii] = (ii < ft.rows && l < ht.rows && j < ft.ncol) ? fmat[ft.off + static_cast<long long>(j) * ft.stride + ii]
                                                               : 0.0;
    }
    __syncthreads();
    for (int e = tid; e < 32 * 32; e += 256) {
      const int l = e & 31, ii = e >> 5;  // H(l, ib + ii - r0)
      if (l < ht.stride && ib + ii < h) out[static_cast<long long>(ib + ii - r0) * ht.stride + l] = S[l][ii];
    }
    __syncthreads();
  }
}

}  // namespace

// Builds d_fmat / d_hmat for every task from the factor values (Problem::lval).
void DeviceSim::build_panels() {
  const Problem& pr = *P;
  const int nt = static_cast<int>(pr.tasks.size());
  std::vector<PanelTask> pt(nt);
  std::vector<int> ft_task(pr.ftiles.size()), ht_task(pr.htiles.size());
  for (int i = 0; i < nt; ++i) {
    const TaskDesc& s = pr.tasks[i];
    pt[i] = PanelTask{s.linv_off, s.b_off, s.w, s.nr, s.f_tile0, s.root_dense};
    for (int k = 0; k < s.f_ntile; ++k) ft_task[s.f_tile0 + k] = i;
    for (int k = 0; k < s.h_ntile; ++k) ht_task[s.h_tile0 + k] = i;
  }
  auto up = [&](const void* src, std::size_t bytes) {
    void* p = nullptr;
    PDG_CUDA(cudaMalloc(&p, bytes ? bytes : 1));
    if (bytes) PDG_CUDA(cudaMemcpyAsync(p, src, bytes, cudaMemcpyHostToDevice, st));
    return p;
  };
  auto* d_pt = static_cast<PanelTask*>(up(pt.data(), pt.size() * sizeof(PanelTask)));
  auto* d_ftt = static_cast<int*>(up(ft_task.data(), ft_task.size() * sizeof(int)));
  auto* d_htt = static_cast<int*>(up(ht_task.data(), ht_task.size() * sizeof(int)));
  // factor values: host-computed ones (all tasks, or the coarse tail when the
  // device factors the subdomains) at lval_host0, then the device factor
  double* d_lval = nullptr;
  PDG_CUDA(cudaMalloc(&d_lval, std::max<std::int64_t>(pr.lval_len, 1) * sizeof(double)));
  if (!pr.lval.empty())
    PDG_CUDA(cudaMemcpyAsync(d_lval + pr.lval_host0, pr.lval.data(), pr.lval.size() * sizeof(double),
                             cudaMemcpyHostToDevice, st));
  if (pr.device_factor) device_factor(d_lval);
  PDG_CUDA(cudaMalloc(&d_fmat, std::max<std::int64_t>(pr.fmat_len, 1) * sizeof(double)));
  PDG_CUDA(cudaMalloc(&d_hmat, std::max<std::int64_t>(pr.hmat_len, 1) * sizeof(double)));
  // alignment gaps between tiles stay zero
  PDG_CUDA(cudaMemsetAsync(d_fmat, 0, std::max<std::int64_t>(pr.fmat_len, 1) * sizeof(double), st));
  PDG_CUDA(cudaMemsetAsync(d_hmat, 0, std::max<std::int64_t>(pr.hmat_len, 1) * sizeof(double), st));
  if (!pr.ftiles.empty())
    forward_panel_kernel<<<static_cast<unsigned>(pr.ftiles.size()), 256, 0, st>>>(d_pt, d_ftt, d_ftiles, d_lval, d_fmat);
  PDG_CUDA(cudaGetLastError());
  if (!pr.htiles.empty())
    backward_panel_kernel<<<static_cast<unsigned>(pr.htiles.size()), 256, 0, st>>>(d_pt, d_htt, d_htiles, d_ftiles,
                                                                                  d_fmat, d_hmat);
  PDG_CUDA(cudaGetLastError());
  PDG_CUDA(cudaStreamSynchronize(st));
  for (void* p : {static_cast<void*>(d_pt), static_cast<void*>(d_ftt), static_cast<void*>(d_htt),
                  static_cast<void*>(d_lval)})
    cudaFree(p);
}

}  // namespace pdg
