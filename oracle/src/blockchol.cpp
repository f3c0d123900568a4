// TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// Exact local and coarse solves of schwarz.cpp:99-146 / :165-168. The
// reference factors each K_i with Eigen's SimplicialLLT (AMD ordering); the
// oracle uses its own, deliberately different, exact factorisation so it stays
// independent of the product (nested dissection + supernodes on the device):
//   * ordering: minimum degree on the block (cell / agglomerate) graph,
//     eliminated on an explicit elimination graph, ties broken by index;
//   * symbolic: block elimination tree and column structures;
//   * numeric: left-looking block Cholesky (b x b dense blocks, row-major),
//     George-Liu linked lists of pending updates.
// Memory is nnz(L) blocks, so the BASELINE config-4/5 subdomains (up to 3,626
// cells x 10-15 dofs) fit where an envelope factor would not.
#include <algorithm>
#include <numeric>
#include <queue>

#include "oracle.hpp"

namespace orc {

namespace {

// minimum degree on an explicit elimination graph (adjacency without self)
std::vector<int> min_degree(std::vector<std::vector<int>> adj) {
  const int n = static_cast<int>(adj.size());
  using Key = std::pair<int, int>;  // (degree, node)
  std::priority_queue<Key, std::vector<Key>, std::greater<Key>> heap;
  for (int v = 0; v < n; ++v) heap.push({static_cast<int>(adj[v].size()), v});
  std::vector<char> done(n, 0);
  std::vector<int> order;
  order.reserve(n);
  std::vector<int> merged;
  while (!heap.empty()) {
    const auto [d, v] = heap.top();
    heap.pop();
    if (done[v] || d != static_cast<int>(adj[v].size())) continue;  // stale entry
    done[v] = 1;
    order.push_back(v);
    const std::vector<int> nb = std::move(adj[v]);
    adj[v].clear();
    for (int u : nb) {
      // adj[u] <- (adj[u] u nb) \ {u, v}
      merged.clear();
      std::set_union(adj[u].begin(), adj[u].end(), nb.begin(), nb.end(), std::back_inserter(merged));
      auto& a = adj[u];
      a.clear();
      for (int w : merged)
        if (w != u && w != v) a.push_back(w);
      heap.push({static_cast<int>(a.size()), u});
    }
  }
  return order;
}

// C -= X * Y^T for b x b row-major blocks
inline void sub_xyt(int b, const double* X, const double* Y, double* C) {
  for (int i = 0; i < b; ++i)
    for (int j = 0; j < b; ++j) {
      double s = 0.0;
      for (int k = 0; k < b; ++k) s += X[i * b + k] * Y[j * b + k];
      C[i * b + j] -= s;
    }
}

}  // namespace

void BlockChol::factor(const Csr& A, int block) {
  b = block;
  const int64_t n = A.rows;
  if (n % b != 0) throw SolverError("block factor: dimension is not a multiple of the block size");
  nb = static_cast<int>(n / b);
  // block graph of A
  std::vector<std::vector<int>> adj(nb);
  for (int64_t r = 0; r < n; ++r) {
    const int bi = static_cast<int>(r / b);
    for (int64_t k = A.ptr[r]; k < A.ptr[r + 1]; ++k) {
      const int bj = static_cast<int>(A.idx[k] / b);
      if (bj != bi) adj[bi].push_back(bj);
    }
  }
  for (auto& a : adj) {
    std::sort(a.begin(), a.end());
    a.erase(std::unique(a.begin(), a.end()), a.end());
  }
  perm = min_degree(adj);  // new -> old
  std::vector<int> inv(nb);
  for (int i = 0; i < nb; ++i) inv[perm[i]] = i;

  // symbolic: struct(j) = {j} u {i > j : A_ij != 0} u (struct(c) \ {c}) over children c
  std::vector<std::vector<int>> cols(nb), kids(nb);
  std::vector<int> parent(nb, -1), tmp;
  for (int j = 0; j < nb; ++j) {
    std::vector<int>& s = cols[j];
    for (int o : adj[perm[j]])
      if (inv[o] > j) s.push_back(inv[o]);
    std::sort(s.begin(), s.end());
    for (int c : kids[j]) {
      tmp.clear();
      std::set_union(s.begin(), s.end(), cols[c].begin() + 2, cols[c].end(), std::back_inserter(tmp));
      s.swap(tmp);
    }
    s.insert(s.begin(), j);
    if (s.size() > 1) {
      parent[j] = s[1];
      kids[s[1]].push_back(j);
    }
  }
  colptr.assign(nb + 1, 0);
  for (int j = 0; j < nb; ++j) colptr[j + 1] = colptr[j] + static_cast<int64_t>(cols[j].size());
  rowidx.resize(colptr[nb]);
  for (int j = 0; j < nb; ++j) std::copy(cols[j].begin(), cols[j].end(), rowidx.begin() + colptr[j]);
  cols.clear();
  cols.shrink_to_fit();
  const int bb = b * b;
  L.assign(colptr[nb] * bb, 0.0);

  // scatter the lower triangle of A, in its ORIGINAL numbering, mirrored
  // (what SimplicialLLT<.., Lower> factors for a not bit-symmetric K0 = E^T K E);
  // inside a diagonal block R >= C keeps to its lower triangle
  std::vector<int64_t> pos(nb, -1);
  for (int64_t R = 0; R < n; ++R) {
    const int nr = inv[static_cast<int>(R / b)];
    for (int64_t k = A.ptr[R]; k < A.ptr[R + 1]; ++k) {
      const int64_t Cc = A.idx[k];
      if (Cc > R) continue;
      const int nc = inv[static_cast<int>(Cc / b)];
      const int col = std::min(nr, nc), row = std::max(nr, nc);
      const int li = static_cast<int>(nr >= nc ? R % b : Cc % b);
      const int lc = static_cast<int>(nr >= nc ? Cc % b : R % b);
      const auto b0 = rowidx.begin() + colptr[col], e0 = rowidx.begin() + colptr[col + 1];
      const int64_t at = std::lower_bound(b0, e0, row) - rowidx.begin();
      L[at * bb + li * b + lc] = A.val[k];
    }
  }

  // numeric: left-looking block Cholesky
  std::vector<int64_t> next(nb, -1);   // next unprocessed entry of column k
  std::vector<int> head(nb, -1), link(nb, -1);
  for (int j = 0; j < nb; ++j) {
    for (int64_t k = colptr[j]; k < colptr[j + 1]; ++k) pos[rowidx[k]] = k;
    int k = head[j];
    while (k >= 0) {
      const int knext = link[k];
      const int64_t p = next[k];  // rowidx[p] == j
      const double* Ljk = &L[p * bb];
      for (int64_t q = p; q < colptr[k + 1]; ++q) sub_xyt(b, &L[q * bb], Ljk, &L[pos[rowidx[q]] * bb]);
      if (p + 1 < colptr[k + 1]) {
        next[k] = p + 1;
        const int i = rowidx[p + 1];
        link[k] = head[i];
        head[i] = k;
      }
      k = knext;
    }
    // dense Cholesky of the diagonal block (lower), then L_ij = C_ij L_jj^{-T}
    double* D = &L[colptr[j] * bb];
    for (int c = 0; c < b; ++c) {
      double d = D[c * b + c];
      for (int t = 0; t < c; ++t) d -= D[c * b + t] * D[c * b + t];
      if (!(d > 0.0) || !std::isfinite(d)) throw SolverError("factorization failed (not positive definite)");
      D[c * b + c] = std::sqrt(d);
      for (int r = c + 1; r < b; ++r) {
        double s = D[r * b + c];
        for (int t = 0; t < c; ++t) s -= D[r * b + t] * D[c * b + t];
        D[r * b + c] = s / D[c * b + c];
      }
      for (int r = 0; r < c; ++r) D[r * b + c] = 0.0;
    }
    for (int64_t q = colptr[j] + 1; q < colptr[j + 1]; ++q) {
      double* X = &L[q * bb];
      for (int r = 0; r < b; ++r)
        for (int c = 0; c < b; ++c) {
          double s = X[r * b + c];
          for (int t = 0; t < c; ++t) s -= X[r * b + t] * D[c * b + t];
          X[r * b + c] = s / D[c * b + c];
        }
    }
    if (colptr[j + 1] - colptr[j] > 1) {
      next[j] = colptr[j] + 1;
      const int i = rowidx[colptr[j] + 1];
      link[j] = head[i];
      head[i] = j;
    }
    for (int64_t q = colptr[j]; q < colptr[j + 1]; ++q) pos[rowidx[q]] = -1;
  }
}

void BlockChol::solve(Vec& x) const {
  const int bb = b * b;
  Vec y(static_cast<std::size_t>(nb) * b);
  for (int j = 0; j < nb; ++j)
    for (int c = 0; c < b; ++c) y[static_cast<int64_t>(j) * b + c] = x[static_cast<int64_t>(perm[j]) * b + c];
  // forward: L y = x
  for (int j = 0; j < nb; ++j) {
    double* yj = &y[static_cast<int64_t>(j) * b];
    const double* D = &L[colptr[j] * bb];
    for (int r = 0; r < b; ++r) {
      double s = yj[r];
      for (int t = 0; t < r; ++t) s -= D[r * b + t] * yj[t];
      yj[r] = s / D[r * b + r];
    }
    for (int64_t q = colptr[j] + 1; q < colptr[j + 1]; ++q) {
      const double* X = &L[q * bb];
      double* yi = &y[static_cast<int64_t>(rowidx[q]) * b];
      for (int r = 0; r < b; ++r) {
        double s = 0.0;
        for (int c = 0; c < b; ++c) s += X[r * b + c] * yj[c];
        yi[r] -= s;
      }
    }
  }
  // backward: L^T x = y
  for (int j = nb - 1; j >= 0; --j) {
    double* yj = &y[static_cast<int64_t>(j) * b];
    for (int64_t q = colptr[j] + 1; q < colptr[j + 1]; ++q) {
      const double* X = &L[q * bb];
      const double* yi = &y[static_cast<int64_t>(rowidx[q]) * b];
      for (int c = 0; c < b; ++c) {
        double s = 0.0;
        for (int r = 0; r < b; ++r) s += X[r * b + c] * yi[r];
        yj[c] -= s;
      }
    }
    const double* D = &L[colptr[j] * bb];
    for (int r = b - 1; r >= 0; --r) {
      double s = yj[r];
      for (int t = r + 1; t < b; ++t) s -= D[t * b + r] * yj[t];
      yj[r] = s / D[r * b + r];
    }
  }
  for (int j = 0; j < nb; ++j)
    for (int c = 0; c < b; ++c) x[static_cast<int64_t>(perm[j]) * b + c] = y[static_cast<int64_t>(j) * b + c];
}

}  // namespace orc
