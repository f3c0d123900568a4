// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-ABI shim over the reference's own Eigen-free mesh half, compiled straight
// from /root/reference/proj/src/{geometry,quadrature,mesh,voronoi,agglomerate,
// parallel}.cpp by oracle/Makefile into oracle/_ref/libpolydg_ref.so. It is
// the golden generator for the bit-exact mesh / face / region / partition
// index maps and for quadrature rules
// (quadrature.cpp:19-198). No reference source is copied into this repo.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include "polydg/mesh.hpp"
#include "polydg/quadrature.hpp"

using namespace polydg;

namespace {
thread_local std::string g_err;
}

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// Generates assign_regions(generate_polygonal_mesh(n, box, seed, lloyd), split)
// (split <= domain ymin skips region assignment). Returns an opaque handle.
void* ref_mesh_generate(int n, double x0, double y0, double x1, double y1, std::uint64_t seed,
                        int lloyd, double split_y) {
  try {
    PolygonalMesh m = generate_polygonal_mesh(n, Rect{x0, y0, x1, y1}, seed, lloyd);
    if (split_y > y0) m = assign_regions(m, split_y);
    return new PolygonalMesh(std::move(m));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_mesh_free(void* h) { delete static_cast<PolygonalMesh*>(h); }

// counts[0..4] = n_cells, n_vertices, n_corners, n_interior, n_boundary
void ref_mesh_counts(void* h, int* counts) {
  const auto& m = *static_cast<PolygonalMesh*>(h);
  int corners = 0;
  for (const auto& c : m.cells()) corners += static_cast<int>(c.size());
  counts[0] = m.n_cells();
  counts[1] = m.n_vertices();
  counts[2] = corners;
  counts[3] = static_cast<int>(m.interior_faces().size());
  counts[4] = static_cast<int>(m.boundary_faces().size());
}

// verts: 2*nv doubles; off: nc+1; idx: corners; regions: nc bytes
void ref_mesh_arrays(void* h, double* verts, int* off, int* idx, std::uint8_t* regions) {
  const auto& m = *static_cast<PolygonalMesh*>(h);
  for (int v = 0; v < m.n_vertices(); ++v) {
    verts[2 * v] = m.vertices()[v].x;
    verts[2 * v + 1] = m.vertices()[v].y;
  }
  int k = 0;
  off[0] = 0;
  for (int c = 0; c < m.n_cells(); ++c) {
    for (int v : m.cells()[c]) idx[k++] = v;
    off[c + 1] = k;
    regions[c] = static_cast<std::uint8_t>(m.region(c));
  }
}

// per interior face: cell_in, cell_out; geo: a.x a.y b.x b.y n.x n.y length
void ref_mesh_faces(void* h, int interior, int* cells, double* geo) {
  const auto& m = *static_cast<PolygonalMesh*>(h);
  const auto& fs = interior ? m.interior_faces() : m.boundary_faces();
  for (std::size_t i = 0; i < fs.size(); ++i) {
    const Face& f = fs[i];
    cells[2 * i] = f.cell_in;
    cells[2 * i + 1] = f.cell_out;
    const double g[7] = {f.a.x, f.a.y, f.b.x, f.b.y, f.normal.x, f.normal.y, f.length};
    std::memcpy(geo + 7 * i, g, sizeof g);
  }
}

// per cell: area, centroid x, centroid y, diameter
void ref_mesh_cell_geometry(void* h, double* out) {
  const auto& m = *static_cast<PolygonalMesh*>(h);
  for (int c = 0; c < m.n_cells(); ++c) {
    out[4 * c] = m.cell_area(c);
    out[4 * c + 1] = m.cell_centroid(c).x;
    out[4 * c + 2] = m.cell_centroid(c).y;
    out[4 * c + 3] = m.cell_diameter(c);
  }
}

// agglomerate(mesh, target) -> count (owner filled), or -1 on error
int ref_agglomerate(void* h, int target, int* owner, double* H) {
  try {
    const auto& m = *static_cast<PolygonalMesh*>(h);
    const AgglomeratedPartition p = agglomerate(m, target);
    for (int c = 0; c < m.n_cells(); ++c) owner[c] = p.owner[c];
    if (H)
      for (int a = 0; a < p.count; ++a) H[a] = p.H_K[a];
    return p.count;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// last level of agglomerate_hierarchy(mesh, levels)
int ref_agglomerate_hierarchy(void* h, int levels, int* owner) {
  try {
    const auto& m = *static_cast<PolygonalMesh*>(h);
    const auto hier = agglomerate_hierarchy(m, levels);
    for (int c = 0; c < m.n_cells(); ++c) owner[c] = hier.back().owner[c];
    return hier.back().count;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// polygon_quadrature(poly, order): returns #points, fills pts (2*cap), w (cap)
int ref_polygon_quadrature(const double* poly, int n, int order, double* pts, double* w,
                           int cap) {
  try {
    std::vector<Point2> p(n);
    for (int i = 0; i < n; ++i) p[i] = {poly[2 * i], poly[2 * i + 1]};
    const QuadratureRule r = polygon_quadrature(p, order);
    const int np = static_cast<int>(r.size());
    for (int i = 0; i < np && i < cap; ++i) {
      pts[2 * i] = r.points[i].x;
      pts[2 * i + 1] = r.points[i].y;
      w[i] = r.weights[i];
    }
    return np;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

int ref_gauss_legendre(int n, double* x, double* w) {
  std::vector<double> a, b;
  gauss_legendre(n, a, b);
  for (int i = 0; i < n; ++i) {
    x[i] = a[i];
    w[i] = b[i];
  }
  return n;
}

}  // extern "C"
