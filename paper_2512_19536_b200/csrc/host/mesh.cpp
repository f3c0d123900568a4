// Mesh construction, face extraction and region labels.
// Face order and orientation reproduce /root/reference/proj/src/mesh.cpp:65-106:
// faces appear in first-occurrence order of their (min, max) vertex key when
// cells are walked in index order; the first using cell is `cell_in`.
#include "mesh.hpp"

#include <algorithm>
#include <unordered_map>

namespace pdg {

Mesh::Mesh(std::vector<Pt> verts, std::vector<int> cell_off, std::vector<int> cell_vtx,
           std::vector<std::uint8_t> regions)
    : verts_(std::move(verts)),
      cell_off_(std::move(cell_off)),
      cell_vtx_(std::move(cell_vtx)),
      regions_(std::move(regions)) {
  const int nc = n_cells();
  if (static_cast<int>(regions_.size()) != nc)
    throw MeshError("mesh: region count does not match cell count");
  h_.resize(nc);
  area_.resize(nc);
  centroid_.resize(nc);
  std::vector<Pt> pts;
  for (int c = 0; c < nc; ++c) {
    if (cell_size(c) < 3)
      throw MeshError("mesh: cell " + std::to_string(c) + " has fewer than 3 vertices");
    for (int k = cell_off_[c]; k < cell_off_[c + 1]; ++k)
      if (cell_vtx_[k] < 0 || cell_vtx_[k] >= n_vertices())
        throw MeshError("mesh: cell " + std::to_string(c) + " references vertex " +
                        std::to_string(cell_vtx_[k]) + " out of range");
    cell_points(c, pts);
    const int n = static_cast<int>(pts.size());
    const double a = poly_area(pts.data(), n);
    if (!(a > 0.0))
      throw MeshError("mesh: cell " + std::to_string(c) +
                      " is not counter-clockwise with positive area");
    area_[c] = a;
    centroid_[c] = poly_centroid(pts.data(), n);
    h_[c] = poly_diameter(pts.data(), n);
  }
  build_faces();
}

void Mesh::cell_points(int c, std::vector<Pt>& out) const {
  out.clear();
  for (int k = cell_off_[c]; k < cell_off_[c + 1]; ++k) out.push_back(verts_[cell_vtx_[k]]);
}

double Mesh::mesh_size() const { return *std::max_element(h_.begin(), h_.end()); }

double Mesh::total_area() const {
  double s = 0.0;
  for (double a : area_) s += a;
  return s;
}

void Mesh::build_faces() {
  struct Use {
    int cell, va, vb;
  };
  struct Slot {
    Use u[2];
    int n = 0;
  };
  std::unordered_map<std::uint64_t, int> key_to_slot;
  key_to_slot.reserve(cell_vtx_.size());
  std::vector<Slot> slots;
  slots.reserve(cell_vtx_.size() / 2 + 8);
  for (int c = 0; c < n_cells(); ++c) {
    const int k = cell_size(c);
    const int* loop = cell_vertices(c);
    for (int e = 0; e < k; ++e) {
      const int va = loop[e], vb = loop[(e + 1) % k];
      const std::uint64_t key =
          (static_cast<std::uint64_t>(std::min(va, vb)) << 32) | static_cast<std::uint32_t>(std::max(va, vb));
      auto [it, inserted] = key_to_slot.try_emplace(key, static_cast<int>(slots.size()));
      if (inserted) slots.emplace_back();
      Slot& s = slots[it->second];
      if (s.n >= 2) throw MeshError("mesh: edge shared by more than two cells (non-manifold)");
      s.u[s.n++] = {c, va, vb};
    }
  }
  for (const Slot& s : slots) {
    const Use& first = s.u[0];
    Face f;
    f.a = verts_[first.va];
    f.b = verts_[first.vb];
    f.cell_in = first.cell;
    f.length = dist(f.a, f.b);
    if (!(f.length > 0.0)) throw MeshError("mesh: zero-length face");
    f.normal = Pt{(f.b.y - f.a.y) / f.length, -(f.b.x - f.a.x) / f.length};
    if (s.n == 2) {
      f.cell_out = s.u[1].cell;
      if (f.cell_out == f.cell_in) throw MeshError("mesh: interior face with identical incident cells");
      interior_.push_back(f);
    } else {
      boundary_.push_back(f);
    }
  }
}

Mesh assign_regions(const Mesh& m, double split_y) {
  const Box box = bbox_of(m.vertices().data(), m.n_vertices());
  if (!(split_y > box.ymin && split_y < box.ymax))
    throw ConfigError("assign_regions: split_y outside the domain height");
  std::vector<std::uint8_t> reg(m.n_cells());
  for (int c = 0; c < m.n_cells(); ++c) reg[c] = m.centroid(c).y >= split_y ? kGrey : kWhite;
  return Mesh(m.vertices(), m.cell_offsets(), m.cell_vertex_ids(), std::move(reg));
}

std::vector<std::vector<int>> Partition::members() const {
  std::vector<std::vector<int>> out(count);
  for (std::size_t c = 0; c < owner.size(); ++c) out[owner[c]].push_back(static_cast<int>(c));
  return out;
}

Partition identity_partition(const Mesh& m) {
  Partition p;
  p.count = m.n_cells();
  p.owner.resize(m.n_cells());
  p.H.resize(m.n_cells());
  for (int c = 0; c < m.n_cells(); ++c) {
    p.owner[c] = c;
    p.H[c] = m.diameter(c);
  }
  return p;
}

}  // namespace pdg
