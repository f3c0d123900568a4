// Quadrature rules and the bounding-box Legendre modal basis (host side).
//
// Rules follow /root/reference/proj/src/quadrature.cpp:19-198: Newton-iterated
// Gauss-Legendre, collapsed-Gauss triangles with n = (order+3)/2 points per
// direction (s outer, t inner), centroid fans with an ear-clip fallback. The
// SAME rule is regenerated on the device by the ionic kernel (non-exact
// integrands make the rule part of the parity contract): the
// device receives the 1-D Gauss nodes/weights computed here and the cell
// triangulation from `cell_triangles`.
// Basis: /root/reference/proj/src/dg_space.cpp:17-84 (P1 in SURVEY.md App. A).
#pragma once

#include <array>
#include <vector>

#include "core.hpp"

namespace pdg {

void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w);

struct Rule {
  std::vector<Pt> pts;
  std::vector<double> w;
  std::size_t size() const { return w.size(); }
};

void triangle_rule(Pt a, Pt b, Pt c, int order, Rule& out);  // appends
Rule polygon_rule(const std::vector<Pt>& poly, int order);
Rule segment_rule(Pt p0, Pt p1, int order);
std::vector<std::array<int, 3>> ear_clip(const std::vector<Pt>& poly);
// Triangles the polygon rule integrates over, as corner triples; the first
// corner of a fan triangle is the centroid. Returns true for a centroid fan.
bool cell_triangles(const std::vector<Pt>& poly, std::vector<std::array<Pt, 3>>& tris);

inline int n_modes(int p) { return (p + 1) * (p + 2) / 2; }

// Values (and optionally gradients) of the degree-p bbox-Legendre basis at one
// point; arrays of length n_modes(p).
void basis_at(const Box& box, int p, Pt x, double* val, double* gx = nullptr,
              double* gy = nullptr);

}  // namespace pdg
