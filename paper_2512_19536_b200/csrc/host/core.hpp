// polydg-b200 host core: points, boxes, polygon primitives, error types.
//
// Host-side setup code for the B200 solver. Everything here is one-time setup
// (mesh, agglomeration, assembly inputs), compiled with -ffp-contract=off so
// the floating-point sequence matches the reference's non-FMA build
// (SURVEY.md Appendix A, P15). Semantics follow
//   /root/reference/proj/include/polydg/geometry.hpp:12-55
//   /root/reference/proj/src/geometry.cpp:11-92
//   /root/reference/proj/include/polydg/errors.hpp:13-35
#pragma once

#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace pdg {

// Error taxonomy of the reference (errors.hpp:13-35). The C-ABI maps these to
// PDG_ERR_CONFIG / PDG_ERR_MESH / PDG_ERR_SOLVER / PDG_ERR_IO.
struct ConfigError : std::runtime_error {
  explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};
struct MeshError : std::runtime_error {
  explicit MeshError(const std::string& w) : std::runtime_error(w) {}
};
struct SolverError : std::runtime_error {
  explicit SolverError(const std::string& w) : std::runtime_error(w) {}
};
struct IoError : std::runtime_error {
  explicit IoError(const std::string& w) : std::runtime_error(w) {}
};

struct Pt {
  double x = 0.0, y = 0.0;
};
inline Pt operator+(Pt a, Pt b) { return {a.x + b.x, a.y + b.y}; }
inline Pt operator-(Pt a, Pt b) { return {a.x - b.x, a.y - b.y}; }
inline Pt operator*(Pt a, double s) { return {a.x * s, a.y * s}; }
inline double dot(Pt a, Pt b) { return a.x * b.x + a.y * b.y; }
inline double cross(Pt a, Pt b) { return a.x * b.y - a.y * b.x; }
inline double dist(Pt a, Pt b) {
  const Pt d = a - b;
  return std::hypot(d.x, d.y);
}

struct Box {
  double xmin = 0.0, ymin = 0.0, xmax = 1.0, ymax = 1.0;
  double width() const { return xmax - xmin; }
  double height() const { return ymax - ymin; }
  double area() const { return width() * height(); }
  bool contains(Pt p) const { return p.x >= xmin && p.x <= xmax && p.y >= ymin && p.y <= ymax; }
};

// 0 = Grey, 1 = White (mesh.hpp:15 order).
enum : std::uint8_t { kGrey = 0, kWhite = 1 };

// Polygon primitives over a contiguous point loop (geometry.cpp:11-60).
double poly_area(const Pt* p, int n);
Pt poly_centroid(const Pt* p, int n);
double poly_diameter(const Pt* p, int n);
Box bbox_of(const Pt* p, int n);
// Monotone-chain hull, CCW, collinear points dropped (geometry.cpp:62-87).
std::vector<Pt> hull_of(std::vector<Pt> pts);
// Diameter through the hull (geometry.cpp:89-92).
double point_set_diameter(const std::vector<Pt>& pts);

}  // namespace pdg
