// Device assembly of the CN system: volume terms (mass
// and anisotropic stiffness, assembly.cpp:89-136), interior-face SIPG terms
// (assembly.cpp:138-181), K = C_m chi_m M + dt/2 A (assembly.cpp:197-202), the
// per-cell mass inverses, the L2 projections of the initial state
// (assembly.cpp:228-242, timestepper.cpp:108-123), the coarse embedding E
// (schwarz.cpp:49-75) and this rank's K0 = E^T K E (schwarz.cpp:141).
//
// Same values, bit for bit, as the host assembly (host/problem.cpp): this file
// is compiled with -fmad=false (the host is built with -ffp-contract=off), and
// every sum runs in the host's order — quadrature points in rule order, faces
// in face order, one warp per cell owning its entries. The host still lays
// out the geometry (fan triangles, face midpoints/directions, penalties).
#include "kernels.cuh"

namespace pdg {

namespace {

struct Basis {
  double v, gx, gy;
};

// mode m of the bbox-scaled tensor Legendre basis at (x, y) (dg_space.cpp:44-84,
// host/quadrature.cpp basis_at: same operation order)
__device__ Basis basis_mode(const double* box, int p, int m, double x, double y, bool grad) {
  const double wx = box[2] - box[0], wy = box[3] - box[1];
  const double xi = (2.0 * x - box[0] - box[2]) / wx;
  const double eta = (2.0 * y - box[1] - box[3]) / wy;
  int d = 0, mm = m;
  while (mm > d) {
    mm -= d + 1;
    ++d;
  }
  const int ax = d - mm, ay = d - ax;
  double px0 = 1.0, px1 = xi, dx0 = 0.0, dx1 = 1.0;
  double py0 = 1.0, py1 = eta, dy0 = 0.0, dy1 = 1.0;
  double pxa = ax == 0 ? 1.0 : xi, dxa = ax == 0 ? 0.0 : 1.0;
  for (int k = 1; k < ax; ++k) {
    const double v2 = ((2 * k + 1) * xi * px1 - k * px0) / (k + 1);
    const double d2 = dx0 + (2 * k + 1) * px1;
    px0 = px1;
    px1 = v2;
    dx0 = dx1;
    dx1 = d2;
  }
  if (ax >= 2) {
    pxa = px1;
    dxa = dx1;
  }
  double pya = ay == 0 ? 1.0 : eta, dya = ay == 0 ? 0.0 : 1.0;
  for (int k = 1; k < ay; ++k) {
    const double v2 = ((2 * k + 1) * eta * py1 - k * py0) / (k + 1);
    const double d2 = dy0 + (2 * k + 1) * py1;
    py0 = py1;
    py1 = v2;
    dy0 = dy1;
    dy1 = d2;
  }
  if (ay >= 2) {
    pya = py1;
    dya = dy1;
  }
  (void)p;
  const double inv = 1.0 / sqrt(wx * wy);
  const double sx = sqrt(2.0 * ax + 1.0), sy = sqrt(2.0 * ay + 1.0);
  const double fx = sx * pxa, fy = sy * pya;
  Basis out;
  out.v = inv * fx * fy;
  out.gx = grad ? inv * sx * dxa * (2.0 / wx) * fy : 0.0;
  out.gy = grad ? inv * fx * sy * dya * (2.0 / wy) : 0.0;
  return out;
}

__device__ double init_value_d(const AsmArgs& a, double x, double y) {
  switch (a.init_kind) {
    case PDG_INIT_DISC: {
      const double dx = x - a.omega0[0], dy = y - a.omega0[1];
      return dx * dx + dy * dy < a.omega0_r2 ? a.u_patch : a.u_rest;
    }
    case PDG_INIT_CONSTANT:
      return a.ip[0];
    case PDG_INIT_COSINE:
      return a.ip[0] * cos(M_PI * x) * cos(M_PI * y) + a.ip[1];
    case PDG_INIT_BILINEAR:
      return a.ip[0] + a.ip[1] * x + a.ip[2] * y + a.ip[3] * x * y;
  }
  return 0.0;
}

// upper-triangle entry e (column-major, ii <= jj) -> (ii, jj): e = jj (jj + 1) / 2 + ii
__device__ __forceinline__ void up_index(int e, int& ii, int& jj) {
  jj = static_cast<int>((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
  while ((jj + 1) * (jj + 2) / 2 <= e) ++jj;
  while (jj * (jj + 1) / 2 > e) --jj;
  ii = e - jj * (jj + 1) / 2;
}

// Cholesky of the full symmetric n x n block `a` (column-major, lower part
// read) into L, one warp: column j's diagonal by lane 0, then its entries
// below by one lane each (host/problem.cpp spd_inverse: same sums).
__device__ bool warp_cholesky(int n, const double* a, double* L) {
  const int lane = threadIdx.x & 31;
  for (int e = lane; e < n * n; e += 32) L[e] = 0.0;
  __syncwarp();
  bool ok = true;
  for (int j = 0; j < n; ++j) {
    if (lane == 0) {
      double d = a[j * n + j];
      for (int k = 0; k < j; ++k) d -= L[k * n + j] * L[k * n + j];
      L[j * n + j] = d > 0.0 ? sqrt(d) : -1.0;
    }
    __syncwarp();
    const double d = L[j * n + j];
    if (!(d > 0.0)) ok = false;
    for (int i = j + 1 + lane; i < n; i += 32) {
      double s = a[j * n + i];
      for (int k = 0; k < j; ++k) s -= L[k * n + i] * L[k * n + j];
      L[j * n + i] = s / d;
    }
    __syncwarp();
  }
  return ok;
}

// x <- L^-T L^-1 x for one column x (host spd_inverse / spd_solve substitutions)
__device__ void chol_solve_col(int n, const double* L, double* x) {
  for (int i = 0; i < n; ++i) {
    double s = x[i];
    for (int k = 0; k < i; ++k) s -= L[k * n + i] * x[k];
    x[i] = s / L[i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = x[i];
    for (int k = i + 1; k < n; ++k) s -= L[i * n + k] * x[k];
    x[i] = s / L[i * n + i];
  }
}

__device__ __forceinline__ long long find_block(const int* kptr, const int* kcol, int row, int col) {
  int lo = kptr[row], hi = kptr[row + 1];
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (kcol[mid] < col) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// ---- volume terms: one warp (CTA) per local cell ----
__global__ void __launch_bounds__(32) volume_kernel(AsmArgs a) {
  extern __shared__ double sh[];
  const int c = blockIdx.x, lane = threadIdx.x;
  const int b = a.b, bq = a.bq, nup = b * (b + 1) / 2;
  double* v = sh;                       // b
  double* X = v + 32;                   // b
  double* Y = X + 32;                   // b
  double* cv = Y + 32;                  // bq
  double* Mup = cv + 32;                // nup
  double* Aup = Mup + nup;              // nup
  double* ru = Aup + nup;               // b
  double* ry = ru + b;                  // n_comp * b
  double* em = ry + 4 * b;              // b * b (E mass)
  double* er = em + b * b;              // b * bq
  double* F = er + b * bq;              // b * b full block scratch
  double* L = F + b * b;                // b * b Cholesky factor
  const bool withE = a.two_level != 0;
  for (int e = lane; e < nup; e += 32) Mup[e] = Aup[e] = 0.0;
  for (int e = lane; e < 5 * b; e += 32) ru[e] = 0.0;
  if (withE)
    for (int e = lane; e < b * b + b * bq; e += 32) em[e] = 0.0;
  const double* box = a.bbox + 4LL * c;
  const double s00 = a.sigma[4LL * c], s01 = a.sigma[4LL * c + 1], s10 = a.sigma[4LL * c + 2],
               s11 = a.sigma[4LL * c + 3];
  const double* abox = withE ? a.abox + 4LL * a.cell_label[c] : nullptr;
  __syncwarp();
  for (int t = a.tri_ptr[c]; t < a.tri_ptr[c + 1]; ++t) {
    const double* tr = a.tri + 6LL * t;
    const double ax = tr[0], ay = tr[1], bx = tr[2], by = tr[3], cx = tr[4], cy = tr[5];
    const double area2 = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax);
    for (int i = 0; i < a.ngl; ++i) {
      const double s = 0.5 * (a.glx[i] + 1.0);
      for (int j = 0; j < a.ngl; ++j) {
        const double tt = 0.5 * (a.glx[j] + 1.0);
        const double eta = tt * (1.0 - s);
        const double px = ax + (bx - ax) * s + (cx - ax) * eta;
        const double py = ay + (by - ay) * s + (cy - ay) * eta;
        const double w = a.glw[i] * a.glw[j] * 0.25 * (1.0 - s) * area2;
        if (lane < b) {
          const Basis bs = basis_mode(box, a.p, lane, px, py, true);
          v[lane] = bs.v;
          X[lane] = bs.gx;
          Y[lane] = bs.gy;
        }
        if (withE && lane < bq) cv[lane] = basis_mode(abox, a.q, lane, px, py, false).v;
        __syncwarp();
        for (int e = lane; e < nup; e += 32) {
          int ii, jj;
          up_index(e, ii, jj);
          Mup[e] += w * v[ii] * v[jj];
          const double sx = s00 * X[jj] + s01 * Y[jj];
          const double sy = s10 * X[jj] + s11 * Y[jj];
          Aup[e] += w * (X[ii] * sx + Y[ii] * sy);
        }
        const double g = init_value_d(a, px, py);
        for (int ii = lane; ii < b; ii += 32) {
          ru[ii] += w * g * v[ii];
          for (int l = 0; l < a.n_comp; ++l)
            if (a.y_rest[l] != 0.0) ry[l * b + ii] += w * a.y_rest[l] * v[ii];
        }
        if (withE) {
          for (int e = lane; e < b * b; e += 32) {
            const int jj = e / b, ii = e - jj * b;
            em[e] += w * v[ii] * v[jj];
          }
          for (int e = lane; e < b * bq; e += 32) {
            const int m = e / b, ii = e - m * b;
            er[e] += w * v[ii] * cv[m];
          }
        }
        __syncwarp();
      }
    }
  }
  // M (full), the volume part of A's diagonal block (into K's diagonal slot;
  // face_kernel adds the faces and forms K), M^-1, U0 / Y0 projections
  const long long b2 = static_cast<long long>(b) * b;
  const long long kd = find_block(a.kptr, a.kcol, c, a.cell0 + c);
  double* Mg = a.M + b2 * c;
  double* Kd = a.kval + b2 * kd;
  for (int e = lane; e < nup; e += 32) {
    int ii, jj;
    up_index(e, ii, jj);
    F[jj * b + ii] = F[ii * b + jj] = Mup[e];
    Mg[jj * b + ii] = Mg[ii * b + jj] = Mup[e];
    Kd[jj * b + ii] = Kd[ii * b + jj] = Aup[e];
  }
  __syncwarp();
  if (!warp_cholesky(b, F, L)) {
    if (lane == 0) atomicOr(a.err, 1);
    return;
  }
  double* Mi = a.Minv + b2 * c;
  for (int col = lane; col < b; col += 32) {
    double x[32];
    for (int i = 0; i < b; ++i) x[i] = 0.0;
    x[col] = 1.0;
    chol_solve_col(b, L, x);
    for (int i = 0; i < b; ++i) Mi[col * b + i] = x[i];
  }
  __syncwarp();
  for (int ii = lane; ii < b; ii += 32) {
    double acc = 0.0;
    for (int jj = 0; jj < b; ++jj) acc += Mi[jj * b + ii] * ru[jj];
    a.U0[static_cast<long long>(c) * b + ii] = acc;
    for (int l = 0; l < a.n_comp; ++l) {
      double y = 0.0;
      if (a.y_rest[l] != 0.0)
        for (int jj = 0; jj < b; ++jj) y += Mi[jj * b + ii] * ry[l * b + jj];
      a.Y0[static_cast<long long>(l) * a.ncells * b + static_cast<long long>(c) * b + ii] = y;
    }
  }
  if (!withE) return;
  // E_K = M_K^-1 int phi psi^T (host spd_solve on the separately summed mass)
  __syncwarp();
  if (!warp_cholesky(b, em, L)) {
    if (lane == 0) atomicOr(a.err, 2);
    return;
  }
  for (int m = lane; m < bq; m += 32) {
    double x[32];
    for (int i = 0; i < b; ++i) x[i] = er[m * b + i];
    chol_solve_col(b, L, x);
    for (int i = 0; i < b; ++i) a.E[static_cast<long long>(c) * b * bq + m * b + i] = x[i];
  }
}

// ---- interior faces + K = a M + hb A: one warp (CTA) per local cell ----
__global__ void __launch_bounds__(32) face_kernel(AsmArgs a) {
  extern __shared__ double sh[];
  const int c = blockIdx.x, lane = threadIdx.x;
  const int b = a.b, nup = b * (b + 1) / 2;
  double* vk = sh;
  double* vl = vk + 32;
  double* ak = vl + 32;
  double* al = ak + 32;
  double* D = al + 32;        // b * b: A's diagonal block
  double* fd = D + b * b;     // nup: this face's diagonal term
  double* fo = fd + nup;      // b * b: this face's coupling block (kl)
  const long long b2 = static_cast<long long>(b) * b;
  const long long kd = find_block(a.kptr, a.kcol, c, a.cell0 + c);
  double* Kd = a.kval + b2 * kd;
  for (int e = lane; e < b * b; e += 32) D[e] = Kd[e];
  __syncwarp();
  for (int q = a.fptr[c]; q < a.fptr[c + 1]; ++q) {
    const int f = a.fent[q] >> 1, side = a.fent[q] & 1;
    const int K = a.fcell[2 * f], Lc = a.fcell[2 * f + 1];
    const double* g = a.fgeo + 8LL * f;
    const double midx = g[0], midy = g[1], dirx = g[2], diry = g[3], half = g[4], nx = g[5], ny = g[6], eta = g[7];
    const double* sk = a.sigma + 4LL * K;
    const double* sl = a.sigma + 4LL * Lc;
    for (int e = lane; e < nup; e += 32) fd[e] = 0.0;
    for (int e = lane; e < b * b; e += 32) fo[e] = 0.0;
    __syncwarp();
    for (int i = 0; i < a.ngs; ++i) {
      const double px = midx + dirx * a.gsx[i], py = midy + diry * a.gsx[i];
      const double w = a.gsw[i] * half;
      if (lane < b) {
        const Basis bk = basis_mode(a.bbox + 4LL * K, a.p, lane, px, py, true);
        const Basis bl = basis_mode(a.bbox + 4LL * Lc, a.p, lane, px, py, true);
        vk[lane] = bk.v;
        vl[lane] = bl.v;
        ak[lane] = (sk[0] * bk.gx + sk[1] * bk.gy) * nx + (sk[2] * bk.gx + sk[3] * bk.gy) * ny;
        al[lane] = (sl[0] * bl.gx + sl[1] * bl.gy) * nx + (sl[2] * bl.gx + sl[3] * bl.gy) * ny;
      }
      __syncwarp();
      for (int e = lane; e < nup; e += 32) {
        int ii, jj;
        up_index(e, ii, jj);
        if (side == 0) {
          const double vki = vk[ii];
          fd[e] += w * (-0.5 * (ak[jj] * vki + ak[ii] * vk[jj]) + eta * vk[jj] * vki);
        } else {
          const double vli = vl[ii];
          fd[e] += w * (0.5 * (al[jj] * vli + al[ii] * vl[jj]) + eta * vl[jj] * vli);
        }
      }
      for (int e = lane; e < b * b; e += 32) {
        const int jj = e / b, ii = e - jj * b;
        const double vki = vk[ii];
        fo[e] += w * (-0.5 * al[jj] * vki + 0.5 * ak[ii] * vl[jj] - eta * vl[jj] * vki);
      }
      __syncwarp();
    }
    // the face's diagonal term into D (symmetric), the coupling block into K
    for (int e = lane; e < nup; e += 32) {
      int ii, jj;
      up_index(e, ii, jj);
      D[jj * b + ii] += fd[e];
      if (ii != jj) D[ii * b + jj] += fd[e];
    }
    const int other = side == 0 ? Lc : K;
    double* Ko = a.kval + b2 * find_block(a.kptr, a.kcol, c, other);
    for (int e = lane; e < b * b; e += 32) {
      const int jj = e / b, ii = e - jj * b;
      const double o = side == 0 ? fo[e] : fo[ii * b + jj];
      Ko[e] = a.hb * (0.0 + o);
    }
    __syncwarp();
  }
  const double* Mg = a.M + b2 * c;
  for (int e = lane; e < b * b; e += 32) Kd[e] = a.am * Mg[e] + a.hb * D[e];
}

// ---- K0 partial = E^T K E over this rank's rows: one CTA per coarse row ----
__global__ void __launch_bounds__(128) k0_kernel(AsmArgs a) {
  extern __shared__ double sh[];
  const int ai = blockIdx.x;
  const int b = a.b, bq = a.bq;
  double* KE = sh;  // b * bq
  const long long bbq = static_cast<long long>(b) * bq;
  for (int ci = a.agg_ptr[ai]; ci < a.agg_ptr[ai + 1]; ++ci) {
    const int i = a.agg_cells[ci];
    const double* Ei = a.E + bbq * i;
    for (int k = a.kptr[i]; k < a.kptr[i + 1]; ++k) {
      const int j = a.kcol[k] - a.cell0;
      const int aj2 = a.cell_agg[j];
      const double* Ej = a.E + bbq * j;
      const double* Kb = a.kval + static_cast<long long>(k) * b * b;
      __syncthreads();
      for (int e = threadIdx.x; e < b * bq; e += blockDim.x) {
        const int m = e / b, r = e - m * b;
        double s = 0.0;
        for (int cc = 0; cc < b; ++cc) s += Kb[cc * b + r] * Ej[m * b + cc];
        KE[m * b + r] = s;
      }
      __syncthreads();
      const long long blk = find_block(a.k0ptr, a.k0col, ai, aj2);
      double* out = a.k0val + blk * bq * bq;
      for (int e = threadIdx.x; e < bq * bq; e += blockDim.x) {
        const int m2 = e / bq, m1 = e - m2 * bq;
        double s = 0.0;
        for (int r = 0; r < b; ++r) s += Ei[m1 * b + r] * KE[m2 * b + r];
        out[m2 * bq + m1] += s;
      }
    }
  }
}

}  // namespace

void launch_assembly(const AsmArgs& a, cudaStream_t st) {
  const int b = a.b, bq = a.bq > 0 ? a.bq : 1;
  const int nup = b * (b + 1) / 2;
  const int vol_smem = static_cast<int>(sizeof(double)) * (4 * 32 + 2 * nup + 5 * b + b * b + b * bq + 2 * b * b);
  const int face_smem = static_cast<int>(sizeof(double)) * (4 * 32 + b * b + nup + b * b);
  if (vol_smem > 48 * 1024) PDG_CUDA(cudaFuncSetAttribute(volume_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, vol_smem));
  if (face_smem > 48 * 1024) PDG_CUDA(cudaFuncSetAttribute(face_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, face_smem));
  if (a.ncells == 0) return;
  volume_kernel<<<a.ncells, 32, vol_smem, st>>>(a);
  PDG_CUDA(cudaGetLastError());
  face_kernel<<<a.ncells, 32, face_smem, st>>>(a);
  PDG_CUDA(cudaGetLastError());
}

void launch_k0(const AsmArgs& a, int n_agg, cudaStream_t st) {
  if (n_agg == 0) return;
  k0_kernel<<<n_agg, 128, static_cast<int>(sizeof(double)) * a.b * a.bq, st>>>(a);
  PDG_CUDA(cudaGetLastError());
}

}  // namespace pdg
