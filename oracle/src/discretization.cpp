// TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// Restates quadrature.cpp:19-198, dg_space.cpp:17-84, mesh.cpp:17-106,
// assembly.cpp:13-242 and ionics.cpp:20-113 of /root/reference/proj/src.
#include <algorithm>
#include <cstdlib>
#include <map>
#include <numeric>
#include <random>
#include <thread>

#include "oracle.hpp"

namespace orc {

// parallel.cpp:13-41
int thread_count() {
  int n = static_cast<int>(std::thread::hardware_concurrency());
  if (n < 1) n = 1;
  if (const char* env = std::getenv("POLYDG_THREADS")) {
    const int cap = std::atoi(env);
    if (cap >= 1) n = std::min(n, cap);
  }
  return n;
}

void parallel_for(std::size_t n, const std::function<void(std::size_t)>& fn) {
  const int workers = thread_count();
  if (workers <= 1 || n < 2) {
    for (std::size_t i = 0; i < n; ++i) fn(i);
    return;
  }
  const std::size_t chunk = (n + workers - 1) / workers;
  std::vector<std::thread> pool;
  for (int w = 0; w < workers; ++w) {
    const std::size_t b = static_cast<std::size_t>(w) * chunk;
    if (b >= n) break;
    const std::size_t e = std::min(n, b + chunk);
    pool.emplace_back([&fn, b, e] {
      for (std::size_t i = b; i < e; ++i) fn(i);
    });
  }
  for (auto& t : pool) t.join();
}

// ---------------- CSR ----------------
// Row-parallel kernels give the same bits as the serial loops (every row is
// computed by one thread in the serial order). Csr::apply stays single-threaded
// like Eigen's SpMV unless parallel operators are switched on (large parity
// runs; the timed CPU baseline keeps the reference's threading).
namespace {
bool g_parallel_ops = false;
int g_lean = 0;  // 1: drop M and A after K / K_rhs; 2: also skip K_rhs (single solves)

void parallel_rows(int64_t n, const std::function<void(int64_t, int64_t)>& fn) {
  const int workers = thread_count();
  if (workers <= 1 || n < 64) {
    fn(0, n);
    return;
  }
  const int64_t parts = std::min<int64_t>(n, static_cast<int64_t>(workers) * 8);
  const int64_t chunk = (n + parts - 1) / parts;
  parallel_for(static_cast<std::size_t>(parts), [&](std::size_t w) {
    const int64_t b = static_cast<int64_t>(w) * chunk, e = std::min(n, b + chunk);
    if (b < e) fn(b, e);
  });
}

// builds ptr from per-row counts, then fills rows in parallel
template <class Count, class Fill>
Csr build_rows(int64_t rows, int64_t cols, Count count, Fill fill) {
  Csr C;
  C.rows = rows;
  C.cols = cols;
  C.ptr.assign(rows + 1, 0);
  parallel_rows(rows, [&](int64_t b, int64_t e) {
    for (int64_t r = b; r < e; ++r) C.ptr[r + 1] = count(r);
  });
  for (int64_t r = 0; r < rows; ++r) C.ptr[r + 1] += C.ptr[r];
  C.idx.resize(C.ptr[rows]);
  C.val.resize(C.ptr[rows]);
  parallel_rows(rows, [&](int64_t b, int64_t e) {
    for (int64_t r = b; r < e; ++r) fill(r, &C.idx[C.ptr[r]], &C.val[C.ptr[r]]);
  });
  return C;
}
}  // namespace

void set_parallel_ops(bool on) { g_parallel_ops = on; }
void set_lean(int level) { g_lean = level; }

void Csr::apply(const Vec& x, Vec& y) const {
  y.assign(rows, 0.0);
  auto body = [&](int64_t b, int64_t e) {
    for (int64_t r = b; r < e; ++r) {
      double s = 0.0;
      for (int64_t k = ptr[r]; k < ptr[r + 1]; ++k) s += val[k] * x[idx[k]];
      y[r] = s;
    }
  };
  if (g_parallel_ops) parallel_rows(rows, body);
  else body(0, rows);
}

double Csr::at(int64_t r, int64_t c) const {
  const auto b = idx.begin() + ptr[r], e = idx.begin() + ptr[r + 1];
  const auto it = std::lower_bound(b, e, c);
  return (it != e && *it == c) ? val[it - idx.begin()] : 0.0;
}

Csr from_triplets(int64_t rows, int64_t cols, std::vector<Triplet>& t) {
  // stable order by (row, col); duplicates summed in insertion order
  // (Eigen's setFromTriplets): bucket by row keeping insertion order, then a
  // stable sort by column inside each row
  std::vector<int64_t> start(rows + 1, 0);
  for (const Triplet& e : t) ++start[e.r + 1];
  for (int64_t r = 0; r < rows; ++r) start[r + 1] += start[r];
  std::vector<int64_t> order(t.size()), fillp(start.begin(), start.end() - 1);
  for (int64_t i = 0; i < static_cast<int64_t>(t.size()); ++i) order[fillp[t[i].r]++] = i;
  fillp.clear();
  fillp.shrink_to_fit();
  std::vector<int64_t> rowlen(rows, 0);
  parallel_rows(rows, [&](int64_t b, int64_t e) {
    for (int64_t r = b; r < e; ++r) {
      auto* o = &order[start[r]];
      const int64_t m = start[r + 1] - start[r];
      std::stable_sort(o, o + m, [&](int64_t a, int64_t c) { return t[a].c < t[c].c; });
      int64_t distinct = 0;
      for (int64_t i = 0; i < m; ++i)
        if (i == 0 || t[o[i]].c != t[o[i - 1]].c) ++distinct;
      rowlen[r] = distinct;
    }
  });
  return build_rows(rows, cols, [&](int64_t r) { return rowlen[r]; },
                    [&](int64_t r, int64_t* idx, double* val) {
                      int64_t w = -1;
                      for (int64_t i = start[r]; i < start[r + 1]; ++i) {
                        const Triplet& e = t[order[i]];
                        if (w >= 0 && idx[w] == e.c) {
                          val[w] += e.v;
                        } else {
                          ++w;
                          idx[w] = e.c;
                          val[w] = e.v;
                        }
                      }
                    });
}

Csr transpose(const Csr& A) {
  std::vector<Triplet> t;
  t.reserve(A.val.size());
  for (int64_t r = 0; r < A.rows; ++r)
    for (int64_t k = A.ptr[r]; k < A.ptr[r + 1]; ++k) t.push_back({A.idx[k], r, A.val[k]});
  return from_triplets(A.cols, A.rows, t);
}

Csr multiply(const Csr& A, const Csr& B) {
  // Gustavson row by row; each row accumulates in A's then B's entry order
  std::vector<std::vector<int64_t>> rows_cols(A.rows);
  std::vector<std::vector<double>> rows_vals(A.rows);
  parallel_rows(A.rows, [&](int64_t b, int64_t e) {
    std::vector<double> a(B.cols, 0.0);
    std::vector<int64_t> mk(B.cols, -1);
    std::vector<int64_t> used;
    for (int64_t r = b; r < e; ++r) {
      used.clear();
      for (int64_t k = A.ptr[r]; k < A.ptr[r + 1]; ++k) {
        const int64_t j = A.idx[k];
        for (int64_t l = B.ptr[j]; l < B.ptr[j + 1]; ++l) {
          const int64_t c = B.idx[l];
          if (mk[c] != r) {
            mk[c] = r;
            a[c] = 0.0;
            used.push_back(c);
          }
          a[c] += A.val[k] * B.val[l];
        }
      }
      std::sort(used.begin(), used.end());
      rows_cols[r] = used;
      auto& v = rows_vals[r];
      v.resize(used.size());
      for (std::size_t i = 0; i < used.size(); ++i) v[i] = a[used[i]];
    }
  });
  return build_rows(A.rows, B.cols, [&](int64_t r) { return static_cast<int64_t>(rows_cols[r].size()); },
                    [&](int64_t r, int64_t* idx, double* val) {
                      std::copy(rows_cols[r].begin(), rows_cols[r].end(), idx);
                      std::copy(rows_vals[r].begin(), rows_vals[r].end(), val);
                    });
}

Csr combine(const Csr& A, double a, const Csr& B, double b) {
  auto merge = [&](int64_t r, int64_t* idx, double* val) {
    int64_t i = A.ptr[r], j = B.ptr[r], w = 0;
    while (i < A.ptr[r + 1] || j < B.ptr[r + 1]) {
      const int64_t ca = i < A.ptr[r + 1] ? A.idx[i] : INT64_MAX;
      const int64_t cb = j < B.ptr[r + 1] ? B.idx[j] : INT64_MAX;
      const int64_t c = std::min(ca, cb);
      if (idx) {
        idx[w] = c;
        val[w] = ca == cb ? a * A.val[i] + b * B.val[j] : (ca < cb ? a * A.val[i] : b * B.val[j]);
      }
      if (ca == cb) ++i, ++j;
      else if (ca < cb) ++i;
      else ++j;
      ++w;
    }
    return w;
  };
  return build_rows(A.rows, A.cols, [&](int64_t r) { return merge(r, nullptr, nullptr); },
                    [&](int64_t r, int64_t* idx, double* val) { merge(r, idx, val); });
}

// ---------------- quadrature ----------------
void gauss_legendre(int n, Vec& x, Vec& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  auto leg = [n](double t, double& p0, double& p1) {
    p0 = 1.0;
    p1 = t;
    for (int k = 2; k <= n; ++k) {
      const double p2 = ((2 * k - 1) * t * p1 - (k - 1) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
  };
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double t = std::cos(M_PI * (i + 0.75) / (n + 0.5)), dp = 0.0, p0, p1;
    for (int it = 0; it < 100; ++it) {
      leg(t, p0, p1);
      dp = n * (t * p1 - p0) / (t * t - 1.0);
      const double dx = p1 / dp;
      t -= dx;
      if (std::abs(dx) < 1e-15) {
        leg(t, p0, p1);
        dp = n * (t * p1 - p0) / (t * t - 1.0);
        t -= p1 / dp;
        break;
      }
    }
    const double wt = 2.0 / ((1.0 - t * t) * dp * dp);
    x[i] = -std::abs(t);
    x[n - 1 - i] = std::abs(t);
    w[i] = w[n - 1 - i] = wt;
  }
  if (n % 2 == 1) x[n / 2] = 0.0;
}

static void tri_rule(P2 a, P2 b, P2 c, int order, Rule& r) {
  const int n = (order + 3) / 2;
  Vec gx, gw;
  gauss_legendre(n, gx, gw);
  const double area2 = cross(b - a, c - a);
  for (int i = 0; i < n; ++i) {
    const double s = 0.5 * (gx[i] + 1.0);
    for (int j = 0; j < n; ++j) {
      const double t = 0.5 * (gx[j] + 1.0);
      r.pts.push_back(a + (b - a) * s + (c - a) * (t * (1.0 - s)));
      r.w.push_back(gw[i] * gw[j] * 0.25 * (1.0 - s) * area2);
    }
  }
}

static double signed_area(const std::vector<P2>& p) {
  double s = 0.0;
  for (std::size_t i = 0; i < p.size(); ++i) s += cross(p[i], p[(i + 1) % p.size()]);
  return 0.5 * s;
}

static P2 centroid(const std::vector<P2>& p) {
  double tw = 0, cx = 0, cy = 0;
  for (std::size_t i = 0; i < p.size(); ++i) {
    const P2 a = p[i], b = p[(i + 1) % p.size()];
    const double w = cross(a, b);
    tw += w;
    cx += (a.x + b.x) * w;
    cy += (a.y + b.y) * w;
  }
  return {cx / (3.0 * tw), cy / (3.0 * tw)};
}

Rule polygon_rule(const std::vector<P2>& poly, int order) {
  order = std::max(order, 1);
  const std::size_t n = poly.size();
  const P2 c = centroid(poly);
  const double area = signed_area(poly);
  bool fan = true;
  for (std::size_t i = 0; i < n; ++i)
    if (cross(poly[i] - c, poly[(i + 1) % n] - c) <= 1e-14 * std::abs(area)) fan = false;
  Rule r;
  if (fan) {
    for (std::size_t i = 0; i < n; ++i) tri_rule(c, poly[i], poly[(i + 1) % n], order, r);
    return r;
  }
  // ear clipping (quadrature.cpp:91-142)
  std::vector<int> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  while (idx.size() > 3) {
    const int m = static_cast<int>(idx.size());
    bool clipped = false;
    for (int e = 0; e < m && !clipped; ++e) {
      const int i = idx[(e + m - 1) % m], j = idx[e], k = idx[(e + 1) % m];
      if (cross(poly[j] - poly[i], poly[k] - poly[i]) <= 0.0) continue;
      bool ear = true;
      for (int q : idx) {
        if (q == i || q == j || q == k) continue;
        const P2 p = poly[q];
        if (cross(poly[j] - poly[i], p - poly[i]) >= 0 && cross(poly[k] - poly[j], p - poly[j]) >= 0 &&
            cross(poly[i] - poly[k], p - poly[k]) >= 0) {
          ear = false;
          break;
        }
      }
      if (!ear) continue;
      tri_rule(poly[i], poly[j], poly[k], order, r);
      idx.erase(idx.begin() + e);
      clipped = true;
    }
    if (!clipped) throw std::runtime_error("ear_clip: no ear found");
  }
  tri_rule(poly[idx[0]], poly[idx[1]], poly[idx[2]], order, r);
  return r;
}

Rule segment_rule(P2 a, P2 b, int order) {
  const int n = (std::max(order, 1) + 2) / 2;
  Vec gx, gw;
  gauss_legendre(n, gx, gw);
  Rule r;
  const double half = 0.5 * std::hypot(a.x - b.x, a.y - b.y);
  const P2 mid = (a + b) * 0.5, dir = (b - a) * 0.5;
  for (int i = 0; i < n; ++i) {
    r.pts.push_back(mid + dir * gx[i]);
    r.w.push_back(gw[i] * half);
  }
  return r;
}

int n_modes(int p) { return (p + 1) * (p + 2) / 2; }

void eval_basis(const Box& box, int p, const std::vector<P2>& pts, Vec& val, Vec* gx, Vec* gy) {
  const int nl = n_modes(p);
  const std::size_t np = pts.size();
  val.assign(np * nl, 0.0);
  if (gx) gx->assign(np * nl, 0.0);
  if (gy) gy->assign(np * nl, 0.0);
  Vec px(p + 1), dpx(p + 1), py(p + 1), dpy(p + 1);
  auto leg = [p](double t, Vec& v, Vec& d) {
    v[0] = 1.0;
    d[0] = 0.0;
    if (p == 0) return;
    v[1] = t;
    d[1] = 1.0;
    for (int k = 1; k < p; ++k) {
      v[k + 1] = ((2 * k + 1) * t * v[k] - k * v[k - 1]) / (k + 1);
      d[k + 1] = d[k - 1] + (2 * k + 1) * v[k];
    }
  };
  const double wx = box.w(), wy = box.h();
  for (std::size_t q = 0; q < np; ++q) {
    leg((2.0 * pts[q].x - box.x0 - box.x1) / wx, px, dpx);
    leg((2.0 * pts[q].y - box.y0 - box.y1) / wy, py, dpy);
    const double inv = 1.0 / std::sqrt(wx * wy);
    int m = 0;
    for (int d = 0; d <= p; ++d)
      for (int ax = d; ax >= 0; --ax, ++m) {
        const int ay = d - ax;
        const double sx = std::sqrt(2.0 * ax + 1.0), sy = std::sqrt(2.0 * ay + 1.0);
        const double fx = sx * px[ax], fy = sy * py[ay];
        val[q * nl + m] = inv * fx * fy;
        if (gx) (*gx)[q * nl + m] = inv * sx * dpx[ax] * (2.0 / wx) * fy;
        if (gy) (*gy)[q * nl + m] = inv * fx * sy * dpy[ay] * (2.0 / wy);
      }
  }
}

// ---------------- mesh view ----------------
std::vector<P2> MeshView::cell(int c) const {
  std::vector<P2> p;
  for (int k = off[c]; k < off[c + 1]; ++k) p.push_back(verts[idx[k]]);
  return p;
}

void MeshView::build() {
  const int nc = n_cells();
  diam.resize(nc);
  bbox.resize(nc);
  for (int c = 0; c < nc; ++c) {
    const auto p = cell(c);
    double d2 = 0.0;
    Box b{1e300, 1e300, -1e300, -1e300};
    for (std::size_t i = 0; i < p.size(); ++i) {
      for (std::size_t j = i + 1; j < p.size(); ++j) {
        const P2 d = p[i] - p[j];
        d2 = std::max(d2, d.x * d.x + d.y * d.y);
      }
      b.x0 = std::min(b.x0, p[i].x);
      b.x1 = std::max(b.x1, p[i].x);
      b.y0 = std::min(b.y0, p[i].y);
      b.y1 = std::max(b.y1, p[i].y);
    }
    diam[c] = std::sqrt(d2);
    bbox[c] = b;
  }
  // faces in first-occurrence order of the (min,max) vertex key
  std::map<std::pair<int, int>, int> key;
  struct Use {
    int cell, va, vb, n = 0, other = -1;
  };
  std::vector<Use> uses;
  for (int c = 0; c < nc; ++c) {
    const int k = off[c + 1] - off[c];
    for (int e = 0; e < k; ++e) {
      const int va = idx[off[c] + e], vb = idx[off[c] + (e + 1) % k];
      auto [it, ins] = key.try_emplace({std::min(va, vb), std::max(va, vb)}, static_cast<int>(uses.size()));
      if (ins) uses.push_back({c, va, vb, 1, -1});
      else {
        uses[it->second].other = c;
        uses[it->second].n++;
      }
    }
  }
  faces.clear();
  for (const Use& u : uses) {
    if (u.n != 2) continue;
    Face f;
    f.a = verts[u.va];
    f.b = verts[u.vb];
    f.in = u.cell;
    f.out = u.other;
    f.len = std::hypot(f.a.x - f.b.x, f.a.y - f.b.y);
    f.n = {(f.b.y - f.a.y) / f.len, -(f.b.x - f.a.x) / f.len};
    faces.push_back(f);
  }
}

// ---------------- assembly ----------------
namespace {
struct Tensor {
  double a00, a01, a10, a11;
};
Tensor tensor(double sl, double sn, P2 f) {
  const double len = std::hypot(f.x, f.y);
  if (!(len > 0.0)) throw ConfigError("conductivity: zero fiber direction");
  const double nx = -f.y / len, ny = f.x / len;
  return {sl + (sn - sl) * nx * nx, (sn - sl) * nx * ny, (sn - sl) * ny * nx, sl + (sn - sl) * ny * ny};
}
void dense_llt(int n, const double* a, double* L) {  // row-major
  std::fill(L, L + n * n, 0.0);
  for (int j = 0; j < n; ++j) {
    double d = a[j * n + j];
    for (int k = 0; k < j; ++k) d -= L[j * n + k] * L[j * n + k];
    if (!(d > 0.0)) throw SolverError("dense block is not positive definite");
    L[j * n + j] = std::sqrt(d);
    for (int i = j + 1; i < n; ++i) {
      double s = a[i * n + j];
      for (int k = 0; k < j; ++k) s -= L[i * n + k] * L[j * n + k];
      L[i * n + j] = s / L[j * n + j];
    }
  }
}
void dense_llt_solve(int n, const double* L, double* x) {
  for (int i = 0; i < n; ++i) {
    double s = x[i];
    for (int k = 0; k < i; ++k) s -= L[i * n + k] * x[k];
    x[i] = s / L[i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = x[i];
    for (int k = i + 1; k < n; ++k) s -= L[k * n + i] * x[k];
    x[i] = s / L[i * n + i];
  }
}
}  // namespace

void Discretization::build(const MeshView& m, const Config& c) {
  mesh = &m;
  p = c.degree;
  nloc = n_modes(p);
  const int nc = m.n_cells(), order = 2 * p + 2;
  const int64_t n = static_cast<int64_t>(nc) * nloc;
  if (!(c.sgl > 0 && c.sgn > 0 && c.swl > 0 && c.swn > 0))
    throw ConfigError("conductivity: all sigma values must be positive");
  std::vector<Tensor> sig(nc);
  std::vector<double> snorm(nc);
  for (int e = 0; e < nc; ++e) {
    const bool grey = m.region[e] == 0;
    const double sl = grey ? c.sgl : c.swl, sn = grey ? c.sgn : c.swn;
    P2 fib = grey ? c.fiber_grey : c.fiber_white;
    sig[e] = tensor(sl, sn, fib);
    snorm[e] = std::max(sl, sn);
  }
  if (c.fiber_random) {
    // ext: theta_K = pi * (rng()>>11) * 2^-53 from mt19937_64(fiber_seed), cell order
    std::mt19937_64 rng(c.fiber_seed);
    for (int e = 0; e < nc; ++e) {
      const double th = M_PI * (static_cast<double>(rng() >> 11) * 0x1.0p-53);
      const bool grey = m.region[e] == 0;
      sig[e] = tensor(grey ? c.sgl : c.swl, grey ? c.sgn : c.swn, {std::cos(th), std::sin(th)});
    }
  }
  // Direct CSR assembly with the SAME per-entry summation order as
  // setFromTriplets over the reference's triplet stream (assembly.cpp:52-84):
  // all volume blocks first (cell order), then per interior face, in face
  // order, the K-K block, the L-L block and the K-L / L-K pair. Local blocks
  // are computed in parallel; accumulation into each entry follows the stream.
  const int nl = nloc, nl2 = nl * nl;
  std::vector<std::vector<int>> nbr(nc);
  for (int e = 0; e < nc; ++e) nbr[e].push_back(e);
  for (const Face& f : m.faces) {
    nbr[f.in].push_back(f.out);
    nbr[f.out].push_back(f.in);
  }
  for (auto& v : nbr) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
  auto block_pattern = [&](bool diag_only) {
    return build_rows(n, n, [&](int64_t r) { return static_cast<int64_t>(diag_only ? 1 : nbr[r / nl].size()) * nl; },
                      [&](int64_t r, int64_t* idx, double* val) {
                        const int e = static_cast<int>(r / nl);
                        int w = 0;
                        for (int cb : nbr[e]) {
                          if (diag_only && cb != e) continue;
                          for (int j = 0; j < nl; ++j, ++w) {
                            idx[w] = static_cast<int64_t>(cb) * nl + j;
                            val[w] = 0.0;
                          }
                        }
                      });
  };
  M = block_pattern(true);
  A = block_pattern(false);
  auto slot = [&](int e, int cb) {  // block position of column block cb in row block e
    return static_cast<int64_t>(std::lower_bound(nbr[e].begin(), nbr[e].end(), cb) - nbr[e].begin()) * nl;
  };
  auto add_diag = [&](Csr& X, int e, int64_t pos, const double* Lu) {  // upper triangle mirrored
    const int64_t r0 = static_cast<int64_t>(e) * nl;
    for (int i = 0; i < nl; ++i) {
      X.val[X.ptr[r0 + i] + pos + i] += Lu[i * nl + i];
      for (int j = i + 1; j < nl; ++j) {
        X.val[X.ptr[r0 + i] + pos + j] += Lu[i * nl + j];
        X.val[X.ptr[r0 + j] + pos + i] += Lu[i * nl + j];
      }
    }
  };
  Mchol.assign(nc, Vec());
  parallel_rows(nc, [&](int64_t e0, int64_t e1) {
    Vec val, gx, gy, lm(nl2), la(nl2), full(nl2);
    for (int64_t ee = e0; ee < e1; ++ee) {
      const int e = static_cast<int>(ee);
      const Rule r = polygon_rule(m.cell(e), order);
      eval_basis(m.bbox[e], p, r.pts, val, &gx, &gy);
      std::fill(lm.begin(), lm.end(), 0.0);
      std::fill(la.begin(), la.end(), 0.0);
      for (std::size_t q = 0; q < r.w.size(); ++q) {
        const double* v = &val[q * nloc];
        for (int i = 0; i < nloc; ++i)
          for (int j = i; j < nloc; ++j) lm[i * nloc + j] += r.w[q] * v[i] * v[j];
      }
      const Tensor& s = sig[e];
      for (std::size_t q = 0; q < r.w.size(); ++q) {
        const double* X = &gx[q * nloc];
        const double* Y = &gy[q * nloc];
        for (int j = 0; j < nloc; ++j) {
          const double sx = s.a00 * X[j] + s.a01 * Y[j], sy = s.a10 * X[j] + s.a11 * Y[j];
          for (int i = 0; i <= j; ++i) la[i * nloc + j] += r.w[q] * (X[i] * sx + Y[i] * sy);
        }
      }
      // volume blocks are the first contribution to their entries and touch
      // only this cell's rows: safe to add from any thread
      add_diag(M, e, 0, lm.data());
      add_diag(A, e, slot(e, e), la.data());
      for (int i = 0; i < nloc; ++i)
        for (int j = 0; j < nloc; ++j) full[i * nloc + j] = lm[std::min(i, j) * nloc + std::max(i, j)];
      Mchol[e].resize(nl2);
      dense_llt(nloc, full.data(), Mchol[e].data());
    }
  });
  const int64_t nf = static_cast<int64_t>(m.faces.size());
  const int64_t chunk = 1 << 17;
  Vec buf(static_cast<std::size_t>(std::min(nf, chunk)) * 3 * nl2);
  for (int64_t f0 = 0; f0 < nf; f0 += chunk) {
    const int64_t f1 = std::min(nf, f0 + chunk);
    parallel_rows(f1 - f0, [&](int64_t b0, int64_t b1) {
      Vec vk, vl, gxk, gyk, gxl, gyl, ak(nl), al(nl);
      for (int64_t fi = f0 + b0; fi < f0 + b1; ++fi) {
        const Face& f = m.faces[fi];
        const int K = f.in, L = f.out;
        const double hk = m.diam[K], hl = m.diam[L];
        const double eta = c.eta0 * (0.5 * (snorm[K] + snorm[L])) * p * p / (2.0 * hk * hl / (hk + hl));
        const Rule r = segment_rule(f.a, f.b, order);
        eval_basis(m.bbox[K], p, r.pts, vk, &gxk, &gyk);
        eval_basis(m.bbox[L], p, r.pts, vl, &gxl, &gyl);
        double* kk = &buf[static_cast<std::size_t>(fi - f0) * 3 * nl2];
        double* ll = kk + nl2;
        double* kl = ll + nl2;
        std::fill(kk, kk + 3 * nl2, 0.0);
        const Tensor &sk = sig[K], &sl = sig[L];
        for (std::size_t q = 0; q < r.w.size(); ++q) {
          const double w = r.w[q];
          const double *VK = &vk[q * nloc], *VL = &vl[q * nloc];
          for (int mm = 0; mm < nloc; ++mm) {
            const double xk = gxk[q * nloc + mm], yk = gyk[q * nloc + mm];
            const double xl = gxl[q * nloc + mm], yl = gyl[q * nloc + mm];
            ak[mm] = (sk.a00 * xk + sk.a01 * yk) * f.n.x + (sk.a10 * xk + sk.a11 * yk) * f.n.y;
            al[mm] = (sl.a00 * xl + sl.a01 * yl) * f.n.x + (sl.a10 * xl + sl.a11 * yl) * f.n.y;
          }
          for (int i = 0; i < nloc; ++i) {
            for (int j = i; j < nloc; ++j) {
              kk[i * nloc + j] += w * (-0.5 * (ak[j] * VK[i] + ak[i] * VK[j]) + eta * VK[j] * VK[i]);
              ll[i * nloc + j] += w * (0.5 * (al[j] * VL[i] + al[i] * VL[j]) + eta * VL[j] * VL[i]);
            }
            for (int j = 0; j < nloc; ++j)
              kl[i * nloc + j] += w * (-0.5 * al[j] * VK[i] + 0.5 * ak[i] * VL[j] - eta * VL[j] * VK[i]);
          }
        }
      }
    });
    // accumulate in stream order: every thread owns a range of row cells and
    // walks the faces one after the other, adding only into its own rows, so
    // each entry still receives its contributions in face order
    const int parts = std::max(1, thread_count());
    parallel_for(static_cast<std::size_t>(parts), [&](std::size_t w) {
      const int lo = static_cast<int>(static_cast<int64_t>(nc) * w / parts);
      const int hi = static_cast<int>(static_cast<int64_t>(nc) * (w + 1) / parts);
      auto mine = [&](int e) { return e >= lo && e < hi; };
      for (int64_t fi = f0; fi < f1; ++fi) {
        const Face& f = m.faces[fi];
        const int K = f.in, L = f.out;
        if (!mine(K) && !mine(L)) continue;
        const double* kk = &buf[static_cast<std::size_t>(fi - f0) * 3 * nl2];
        const double* kl = kk + 2 * nl2;
        if (mine(K)) {
          add_diag(A, K, slot(K, K), kk);
          const int64_t pKL = slot(K, L), rK = static_cast<int64_t>(K) * nl;
          for (int i = 0; i < nl; ++i)
            for (int j = 0; j < nl; ++j) A.val[A.ptr[rK + i] + pKL + j] += kl[i * nl + j];
        }
        if (mine(L)) {
          add_diag(A, L, slot(L, L), kk + nl2);
          const int64_t pLK = slot(L, K), rL = static_cast<int64_t>(L) * nl;
          for (int i = 0; i < nl; ++i)
            for (int j = 0; j < nl; ++j) A.val[A.ptr[rL + j] + pLK + i] += kl[i * nl + j];
        }
      }
    });
  }
  K = combine(M, c.C_m * c.chi_m, A, 0.5 * c.dt);
  if (g_lean < 2) Krhs = combine(M, c.chi_m * c.C_m, A, -0.5 * c.dt);
  if (g_lean >= 1) {  // large parity runs: only K (and K_rhs) are needed after setup
    A = Csr();
    M = Csr();
  }
}

Vec Discretization::mass_solve(const Vec& rhs) const {
  Vec x(rhs.size());
  for (int e = 0; e < mesh->n_cells(); ++e) {
    double* xe = &x[static_cast<int64_t>(e) * nloc];
    std::copy(rhs.begin() + static_cast<int64_t>(e) * nloc, rhs.begin() + static_cast<int64_t>(e + 1) * nloc, xe);
    dense_llt_solve(nloc, Mchol[e].data(), xe);
  }
  return x;
}

Vec Discretization::l2_project(const std::function<double(P2)>& g) const {
  Vec rhs(static_cast<int64_t>(mesh->n_cells()) * nloc, 0.0), val;
  for (int e = 0; e < mesh->n_cells(); ++e) {
    const Rule r = polygon_rule(mesh->cell(e), 2 * p + 2);
    eval_basis(mesh->bbox[e], p, r.pts, val, nullptr, nullptr);
    for (std::size_t q = 0; q < r.w.size(); ++q) {
      const double wg = r.w[q] * g(r.pts[q]);
      for (int i = 0; i < nloc; ++i) rhs[static_cast<int64_t>(e) * nloc + i] += wg * val[q * nloc + i];
    }
  }
  return mass_solve(rhs);
}

// cell_means (snapshot.cpp:13-28): (1/|K|) sum_q w_q (Phi U_K)_q at order 2p+2,
// |K| the shoelace area of the cell (mesh.cpp:36, geometry.cpp:11-20)
Vec cell_means(const Discretization& D, const Vec& U) {
  const int nl = D.nloc, nc = D.mesh->n_cells();
  Vec means(nc, 0.0), val;
  for (int e = 0; e < nc; ++e) {
    const std::vector<P2> poly = D.mesh->cell(e);
    const Rule r = polygon_rule(poly, 2 * D.p + 2);
    eval_basis(D.mesh->bbox[e], D.p, r.pts, val, nullptr, nullptr);
    double acc = 0.0;
    for (std::size_t q = 0; q < r.w.size(); ++q) {
      double u = 0.0;
      for (int i = 0; i < nl; ++i) u += val[q * nl + i] * U[static_cast<int64_t>(e) * nl + i];
      acc += r.w[q] * u;
    }
    means[e] = acc / signed_area(poly);
  }
  return means;
}

// l2_error (dg_space.cpp:94-115): sqrt(sum_K sum_q w_q (u_h - g)^2) at order 2p+2
double l2_error(const Discretization& D, const Vec& U, const std::function<double(P2)>& g) {
  const int nl = D.nloc, nc = D.mesh->n_cells();
  double acc = 0.0;
  Vec val;
  for (int e = 0; e < nc; ++e) {
    const Rule r = polygon_rule(D.mesh->cell(e), 2 * D.p + 2);
    eval_basis(D.mesh->bbox[e], D.p, r.pts, val, nullptr, nullptr);
    for (std::size_t q = 0; q < r.w.size(); ++q) {
      double u = 0.0;
      for (int i = 0; i < nl; ++i) u += val[q * nl + i] * U[static_cast<int64_t>(e) * nl + i];
      const double diff = u - g(r.pts[q]);
      acc += r.w[q] * diff * diff;
    }
  }
  return std::sqrt(acc);
}

double MeshView::mesh_size() const { return *std::max_element(diam.begin(), diam.end()); }

// ---------------- ionics ----------------
double fhn_current(const double* P, double u, double w) {
  if (!std::isfinite(u) || !std::isfinite(w)) throw SolverError("fhn: non-finite state in current evaluation");
  const double span = P[6] - P[5];
  const double v = (u - P[5]) / span;
  return P[7] * (P[2] * v * (v - P[0]) * (v - 1.0) + P[3] * v * w) * span;
}

double fhn_rate(const double* P, double u, double w) {
  if (!std::isfinite(u) || !std::isfinite(w)) throw SolverError("fhn: non-finite state in rate evaluation");
  const double v = (u - P[5]) / (P[6] - P[5]);
  return -P[1] * (v - P[4] * w);
}

// ---- Barreto-Cressman (Cressman et al. 2009, J Comput Neurosci 26:159-170) ----
namespace {
double x_over_1mexp(double x) { return x == 0.0 ? 1.0 : x / (1.0 - std::exp(-x)); }
struct BcParts {
  double i_na, i_k, i_cl;
};
BcParts bc_parts(const double* P, double u, const double* y) {
  const double n = y[0], h = y[1], ko = y[2], nai = y[3];
  if (!std::isfinite(u) || !std::isfinite(n) || !std::isfinite(h) || !std::isfinite(ko) || !std::isfinite(nai))
    throw SolverError("barreto-cressman: non-finite state in current evaluation");
  const double alpha_m = x_over_1mexp(0.1 * (u + 30.0)), beta_m = 4.0 * std::exp(-(u + 55.0) / 18.0);
  const double m_inf = alpha_m / (alpha_m + beta_m);
  const double k_in = P[17] + (P[16] - nai);            // [K]i
  const double na_out = P[18] - P[11] * (nai - P[16]);  // [Na]o
  const double e_na = P[13] * std::log(na_out / nai);
  const double e_k = P[13] * std::log(ko / k_in);
  const double e_cl = P[13] * std::log(P[14] / P[15]);
  BcParts r;
  r.i_na = P[0] * m_inf * m_inf * m_inf * h * (u - e_na) + P[2] * (u - e_na);
  r.i_k = P[1] * std::pow(n, 4) * (u - e_k) + P[3] * (u - e_k);
  r.i_cl = P[4] * (u - e_cl);
  return r;
}
}  // namespace

double bc_current(const double* P, double u, const double* y) {
  const BcParts c = bc_parts(P, u, y);
  const double f = P[19] * (c.i_na + c.i_k + c.i_cl);
  if (!std::isfinite(f)) throw SolverError("barreto-cressman: non-finite state in current evaluation");
  return f;
}

void bc_rates(const double* P, double u, const double* y, double* m) {
  const BcParts c = bc_parts(P, u, y);
  const double alpha_n = 0.1 * x_over_1mexp(0.1 * (u + 34.0)), beta_n = 0.125 * std::exp(-(u + 44.0) / 80.0);
  const double alpha_h = 0.07 * std::exp(-(u + 44.0) / 20.0), beta_h = 1.0 / (1.0 + std::exp(-0.1 * (u + 14.0)));
  const double pump = P[6] / ((1.0 + std::exp((25.0 - y[3]) / 3.0)) * (1.0 + std::exp(5.5 - y[2])));
  const double glia = P[7] / (1.0 + std::exp((18.0 - y[2]) / 2.5));
  const double diff = P[8] * (y[2] - P[9]);
  const double dn = P[5] * (alpha_n * (1.0 - y[0]) - beta_n * y[0]);
  const double dh = P[5] * (alpha_h * (1.0 - y[1]) - beta_h * y[1]);
  const double dko = (P[10] * P[11] * c.i_k - 2.0 * P[11] * pump - glia - diff) / P[12];
  const double dnai = (-P[10] * c.i_na - 3.0 * pump) / P[12];
  m[0] = -dn;
  m[1] = -dh;
  m[2] = -dko;
  m[3] = -dnai;
  for (int l = 0; l < 4; ++l)
    if (!std::isfinite(m[l])) throw SolverError("barreto-cressman: non-finite state in rate evaluation");
}

int model_rest(const Config& c, double* u, double* y) {
  if (c.ionic == 1) {
    *u = c.fhn[5];
    y[0] = 0.0;
    return 1;
  }
  if (c.ionic != 2) return 0;
  // Newton on F(u, Ko, Nai) = (I, dKo/dt, dNai/dt) with n, h at steady state;
  // central-difference Jacobian, partial-pivot elimination
  auto gates = [](double v, double* g) {
    const double an = 0.1 * x_over_1mexp(0.1 * (v + 34.0)), bn = 0.125 * std::exp(-(v + 44.0) / 80.0);
    const double ah = 0.07 * std::exp(-(v + 44.0) / 20.0), bh = 1.0 / (1.0 + std::exp(-0.1 * (v + 14.0)));
    g[0] = an / (an + bn);
    g[1] = ah / (ah + bh);
  };
  auto F = [&](const double* z, double* f) {
    double yy[4];
    gates(z[0], yy);
    yy[2] = z[1];
    yy[3] = z[2];
    double m[4];
    bc_rates(c.bc, z[0], yy, m);
    f[0] = bc_current(c.bc, z[0], yy);
    f[1] = m[2] * c.bc[12];
    f[2] = m[3] * c.bc[12];
  };
  double z[3] = {-68.0, c.bc[9], c.bc[16]};
  for (int it = 0; it < 100; ++it) {
    double f[3], J[3][4];
    F(z, f);
    for (int j = 0; j < 3; ++j) {
      double zp[3] = {z[0], z[1], z[2]}, zm[3] = {z[0], z[1], z[2]}, fp[3], fm[3];
      const double h = 1e-6 * std::max(1.0, std::fabs(z[j]));
      zp[j] += h;
      zm[j] -= h;
      F(zp, fp);
      F(zm, fm);
      for (int i = 0; i < 3; ++i) J[i][j] = (fp[i] - fm[i]) / (2.0 * h);
    }
    for (int i = 0; i < 3; ++i) J[i][3] = -f[i];
    for (int col = 0; col < 3; ++col) {
      int piv = col;
      for (int r = col + 1; r < 3; ++r)
        if (std::fabs(J[r][col]) > std::fabs(J[piv][col])) piv = r;
      for (int k = 0; k < 4; ++k) std::swap(J[col][k], J[piv][k]);
      for (int r = col + 1; r < 3; ++r) {
        const double l = J[r][col] / J[col][col];
        for (int k = col; k < 4; ++k) J[r][k] -= l * J[col][k];
      }
    }
    double dz[3];
    for (int i = 2; i >= 0; --i) {
      double s = J[i][3];
      for (int k = i + 1; k < 3; ++k) s -= J[i][k] * dz[k];
      dz[i] = s / J[i][i];
    }
    double step = 0.0;
    for (int j = 0; j < 3; ++j) {
      z[j] += dz[j];
      step = std::max(step, std::fabs(dz[j]) / std::max(1.0, std::fabs(z[j])));
    }
    if (!std::isfinite(step)) break;
    if (step < 1e-14) {
      *u = z[0];
      gates(z[0], y);
      y[2] = z[1];
      y[3] = z[2];
      return 4;
    }
  }
  throw ConfigError("barreto-cressman: no resting state found for these parameters");
}

IonicTerms ionic_terms(const Discretization& D, const Vec& U, const std::vector<Vec>& Y, const Config& cfg,
                       bool* out_of_box) {
  const int nl = D.nloc, nc = D.mesh->n_cells();
  const int ncomp = static_cast<int>(Y.size());
  const bool bc = cfg.ionic == 2;
  const double* P = cfg.fhn;
  IonicTerms out;
  out.I.assign(U.size(), 0.0);
  out.G.assign(Y.size(), Vec(U.size(), 0.0));
  const double umin = bc ? -100.0 : P[5], umax = bc ? 60.0 : P[6];
  const double slack = 10.0 * (umax - umin);
  std::vector<char> oob(nc, 0);
  std::vector<std::string> err(nc);
  parallel_for(nc, [&](std::size_t ci) {
    const int e = static_cast<int>(ci);
    try {
      const Rule r = polygon_rule(D.mesh->cell(e), 2 * D.p + 2);
      Vec val;
      eval_basis(D.mesh->bbox[e], D.p, r.pts, val, nullptr, nullptr);
      const int64_t b0 = static_cast<int64_t>(e) * nl;
      for (std::size_t q = 0; q < r.w.size(); ++q) {
        double u = 0.0, y[4] = {0.0, 0.0, 0.0, 0.0}, m[4] = {0.0, 0.0, 0.0, 0.0};
        for (int i = 0; i < nl; ++i) u += val[q * nl + i] * U[b0 + i];
        for (int l = 0; l < ncomp; ++l)
          for (int i = 0; i < nl; ++i) y[l] += val[q * nl + i] * Y[l][b0 + i];
        if (u < umin - slack || u > umax + slack) oob[e] = 1;
        double f;
        if (bc) {
          f = bc_current(cfg.bc, u, y);
          bc_rates(cfg.bc, u, y, m);
        } else {
          f = fhn_current(P, u, y[0]);
          m[0] = fhn_rate(P, u, y[0]);
        }
        const double wf = r.w[q] * f;
        for (int i = 0; i < nl; ++i) out.I[b0 + i] += wf * val[q * nl + i];
        for (int l = 0; l < ncomp; ++l) {
          const double wm = r.w[q] * m[l];
          for (int i = 0; i < nl; ++i) out.G[l][b0 + i] += wm * val[q * nl + i];
        }
      }
    } catch (const std::exception& ex) {
      err[e] = ex.what();
    }
  });
  for (const auto& s : err)
    if (!s.empty()) throw SolverError(s);
  if (out_of_box) *out_of_box = std::any_of(oob.begin(), oob.end(), [](char c) { return c != 0; });
  return out;
}

}  // namespace orc
