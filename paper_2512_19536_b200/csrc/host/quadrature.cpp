#include "quadrature.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>

namespace pdg {

namespace {
// P_0..P_n at xi and their derivatives, P'_{k+1} = P'_{k-1} + (2k+1) P_k
// (dg_space.cpp:17-27)
void legendre(int n, double xi, double* v, double* d) {
  v[0] = 1.0;
  d[0] = 0.0;
  if (n == 0) return;
  v[1] = xi;
  d[1] = 1.0;
  for (int k = 1; k < n; ++k) {
    v[k + 1] = ((2 * k + 1) * xi * v[k] - k * v[k - 1]) / (k + 1);
    d[k + 1] = d[k - 1] + (2 * k + 1) * v[k];
  }
}

void legendre_p(int n, double x, double& p0, double& p1) {
  p0 = 1.0;
  p1 = x;
  for (int k = 2; k <= n; ++k) {
    const double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
}
}  // namespace

void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  const int half = (n + 1) / 2;
  for (int i = 0; i < half; ++i) {
    double t = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0, p1;
      legendre_p(n, t, p0, p1);
      dp = n * (t * p1 - p0) / (t * t - 1.0);
      const double dx = p1 / dp;
      t -= dx;
      if (std::abs(dx) < 1e-15) {
        legendre_p(n, t, p0, p1);
        dp = n * (t * p1 - p0) / (t * t - 1.0);
        t -= p1 / dp;
        break;
      }
    }
    const double wt = 2.0 / ((1.0 - t * t) * dp * dp);
    x[i] = -std::abs(t);
    x[n - 1 - i] = std::abs(t);
    w[i] = wt;
    w[n - 1 - i] = wt;
  }
  if (n % 2 == 1) x[n / 2] = 0.0;
}

// The Newton-iterated nodes are the same for every cell and face of a given
// order: compute each n once (thread-safe static init), same bits as before.
const std::pair<std::vector<double>, std::vector<double>>& gauss_legendre_cached(int n) {
  static const auto table = [] {
    std::vector<std::pair<std::vector<double>, std::vector<double>>> t(33);
    for (int k = 1; k < 33; ++k) gauss_legendre(k, t[k].first, t[k].second);
    return t;
  }();
  static thread_local std::pair<std::vector<double>, std::vector<double>> big;
  if (n > 0 && n < 33) return table[n];
  gauss_legendre(n, big.first, big.second);
  return big;
}

void triangle_rule(Pt a, Pt b, Pt c, int order, Rule& out) {
  const int n = (order + 3) / 2;
  const auto& gl = gauss_legendre_cached(n);
  const std::vector<double>& gx = gl.first;
  const std::vector<double>& gw = gl.second;
  const double area2 = cross(b - a, c - a);
  for (int i = 0; i < n; ++i) {
    const double s = 0.5 * (gx[i] + 1.0);
    for (int j = 0; j < n; ++j) {
      const double t = 0.5 * (gx[j] + 1.0);
      const double eta = t * (1.0 - s);
      out.pts.push_back(a + (b - a) * s + (c - a) * eta);
      out.w.push_back(gw[i] * gw[j] * 0.25 * (1.0 - s) * area2);
    }
  }
}

std::vector<std::array<int, 3>> ear_clip(const std::vector<Pt>& poly) {
  const int n = static_cast<int>(poly.size());
  if (n < 3) throw MeshError("ear_clip: polygon has fewer than 3 vertices");
  std::vector<int> idx(n);
  std::iota(idx.begin(), idx.end(), 0);
  auto inside = [&](int i, int j, int k, int q) {
    const Pt p = poly[q], A = poly[i], B = poly[j], C = poly[k];
    return cross(B - A, p - A) >= 0.0 && cross(C - B, p - B) >= 0.0 && cross(A - C, p - C) >= 0.0;
  };
  std::vector<std::array<int, 3>> tris;
  int guard = 0;
  while (idx.size() > 3) {
    const int m = static_cast<int>(idx.size());
    bool clipped = false;
    for (int e = 0; e < m; ++e) {
      const int i = idx[(e + m - 1) % m], j = idx[e], k = idx[(e + 1) % m];
      if (cross(poly[j] - poly[i], poly[k] - poly[i]) <= 0.0) continue;
      bool ear = true;
      for (int q : idx) {
        if (q == i || q == j || q == k) continue;
        if (inside(i, j, k, q)) {
          ear = false;
          break;
        }
      }
      if (!ear) continue;
      tris.push_back({i, j, k});
      idx.erase(idx.begin() + e);
      clipped = true;
      break;
    }
    if (!clipped) throw MeshError("ear_clip: no ear found (polygon not simple?)");
    if (++guard > 4 * n) throw MeshError("ear_clip: failed to terminate");
  }
  tris.push_back({idx[0], idx[1], idx[2]});
  return tris;
}

bool cell_triangles(const std::vector<Pt>& poly, std::vector<std::array<Pt, 3>>& tris) {
  if (poly.size() < 3) throw MeshError("polygon_quadrature: fewer than 3 vertices");
  tris.clear();
  const int n = static_cast<int>(poly.size());
  const Pt c = poly_centroid(poly.data(), n);
  const double area = poly_area(poly.data(), n);
  bool fan = true;
  for (int i = 0; i < n; ++i)
    if (cross(poly[i] - c, poly[(i + 1) % n] - c) <= 1e-14 * std::abs(area)) {
      fan = false;
      break;
    }
  if (fan) {
    for (int i = 0; i < n; ++i) tris.push_back({c, poly[i], poly[(i + 1) % n]});
  } else {
    for (const auto& t : ear_clip(poly)) tris.push_back({poly[t[0]], poly[t[1]], poly[t[2]]});
  }
  return fan;
}

Rule polygon_rule(const std::vector<Pt>& poly, int order) {
  order = std::max(order, 1);
  std::vector<std::array<Pt, 3>> tris;
  cell_triangles(poly, tris);
  Rule r;
  for (const auto& t : tris) triangle_rule(t[0], t[1], t[2], order, r);
  return r;
}

Rule segment_rule(Pt p0, Pt p1, int order) {
  const int n = (std::max(order, 1) + 2) / 2;
  const auto& gl = gauss_legendre_cached(n);
  const std::vector<double>& gx = gl.first;
  const std::vector<double>& gw = gl.second;
  Rule r;
  const double half = 0.5 * dist(p0, p1);
  const Pt mid = (p0 + p1) * 0.5;
  const Pt dir = (p1 - p0) * 0.5;
  for (int i = 0; i < n; ++i) {
    r.pts.push_back(mid + dir * gx[i]);
    r.w.push_back(gw[i] * half);
  }
  return r;
}

void basis_at(const Box& box, int p, Pt x, double* val, double* gx, double* gy) {
  double px[16], dpx[16], py[16], dpy[16];
  const double wx = box.width(), wy = box.height();
  const double xi = (2.0 * x.x - box.xmin - box.xmax) / wx;
  const double eta = (2.0 * x.y - box.ymin - box.ymax) / wy;
  legendre(p, xi, px, dpx);
  legendre(p, eta, py, dpy);
  const double inv = 1.0 / std::sqrt(wx * wy);
  int m = 0;
  for (int d = 0; d <= p; ++d)
    for (int ax = d; ax >= 0; --ax, ++m) {
      const int ay = d - ax;
      const double sx = std::sqrt(2.0 * ax + 1.0), sy = std::sqrt(2.0 * ay + 1.0);
      const double fx = sx * px[ax], fy = sy * py[ay];
      val[m] = inv * fx * fy;
      if (gx) gx[m] = inv * sx * dpx[ax] * (2.0 / wx) * fy;
      if (gy) gy[m] = inv * fx * sy * dpy[ay] * (2.0 / wy);
    }
}

}  // namespace pdg
