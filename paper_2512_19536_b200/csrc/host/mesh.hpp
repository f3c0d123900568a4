// Polygonal mesh, faces, region labels and agglomerated partitions.
//
// Host setup for the B200 path. Semantics (and, where the north star asks for
// bit-exact index maps, arithmetic) follow
//   /root/reference/proj/include/polydg/mesh.hpp:15-130
//   /root/reference/proj/src/mesh.cpp:17-185        (ctor, faces, regions)
//   /root/reference/proj/src/voronoi.cpp:15-289     (generator)
//   /root/reference/proj/src/agglomerate.cpp:19-186 (greedy agglomeration)
// Storage is CSR (corner offsets + vertex ids) instead of vector<vector<int>>.
#pragma once

#include <cstdint>
#include <vector>

#include "core.hpp"

namespace pdg {

struct Face {
  Pt a, b;
  int cell_in = -1;   // normal points out of this cell
  int cell_out = -1;  // -1 on the boundary
  Pt normal;
  double length = 0.0;
};

class Mesh {
 public:
  Mesh() = default;
  Mesh(std::vector<Pt> verts, std::vector<int> cell_off, std::vector<int> cell_vtx,
       std::vector<std::uint8_t> regions);

  int n_cells() const { return static_cast<int>(cell_off_.size()) - 1; }
  int n_vertices() const { return static_cast<int>(verts_.size()); }
  int cell_size(int c) const { return cell_off_[c + 1] - cell_off_[c]; }
  const int* cell_vertices(int c) const { return cell_vtx_.data() + cell_off_[c]; }
  void cell_points(int c, std::vector<Pt>& out) const;
  std::vector<Pt> cell_points(int c) const {
    std::vector<Pt> p;
    cell_points(c, p);
    return p;
  }

  const std::vector<Pt>& vertices() const { return verts_; }
  const std::vector<int>& cell_offsets() const { return cell_off_; }
  const std::vector<int>& cell_vertex_ids() const { return cell_vtx_; }
  const std::vector<std::uint8_t>& regions() const { return regions_; }
  std::uint8_t region(int c) const { return regions_[c]; }
  const std::vector<Face>& interior_faces() const { return interior_; }
  const std::vector<Face>& boundary_faces() const { return boundary_; }
  double diameter(int c) const { return h_[c]; }
  double area(int c) const { return area_[c]; }
  Pt centroid(int c) const { return centroid_[c]; }
  double mesh_size() const;
  double total_area() const;

 private:
  std::vector<Pt> verts_;
  std::vector<int> cell_off_{0};
  std::vector<int> cell_vtx_;
  std::vector<std::uint8_t> regions_;
  std::vector<Face> interior_, boundary_;
  std::vector<double> h_, area_;
  std::vector<Pt> centroid_;
  void build_faces();
};

struct Partition {
  std::vector<int> owner;  // cell -> agglomerate
  int count = 0;
  std::vector<double> H;   // agglomerate diameters
  bool target_achieved = true;
  std::vector<std::vector<int>> members() const;
};

Mesh generate_mesh(int n_cells, const Box& domain, std::uint64_t seed, int lloyd);
Mesh voronoi_mesh(const std::vector<Pt>& seeds, const Box& domain);
Mesh assign_regions(const Mesh& m, double split_y);
Partition identity_partition(const Mesh& m);
Partition agglomerate(const Mesh& m, int target);
Partition agglomerate(const Mesh& m, const Partition& p, int target);
std::vector<Partition> agglomerate_hierarchy(const Mesh& m, int levels);

}  // namespace pdg
