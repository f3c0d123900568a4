// Snapshot writer (export_snapshot, /root/reference/proj/src/snapshot.cpp:30-75):
// the per-cell means come from the device (cell_means_kernel); this host half
// only formats them, with the reference's two formats and error behaviour.
#include "snapshot.hpp"

#include <cstdio>
#include <fstream>

namespace pdg {

void write_snapshot(const Mesh& mesh, const std::vector<double>& means, double t, const std::string& path,
                    const std::string& format) {
  if (format != "vtk-legacy" && format != "csv-cellmeans")
    throw ConfigError("unknown snapshot format '" + format + "'");
  std::ofstream out(path);
  if (!out) throw IoError("cannot open snapshot for writing: " + path);
  char buf[96];
  const int nc = mesh.n_cells();
  const auto& off = mesh.cell_offsets();
  const auto& idx = mesh.cell_vertex_ids();
  if (format == "vtk-legacy") {
    out << "# vtk DataFile Version 3.0\n";
    std::snprintf(buf, sizeof buf, "polydg transmembrane potential t=%.17g ms\n", t);
    out << buf << "ASCII\nDATASET POLYDATA\n";
    out << "POINTS " << mesh.n_vertices() << " double\n";
    for (const Pt& v : mesh.vertices()) {
      std::snprintf(buf, sizeof buf, "%.17g %.17g 0\n", v.x, v.y);
      out << buf;
    }
    out << "POLYGONS " << nc << ' ' << (idx.size() + static_cast<std::size_t>(nc)) << '\n';
    for (int c = 0; c < nc; ++c) {
      out << (off[c + 1] - off[c]);
      for (int k = off[c]; k < off[c + 1]; ++k) out << ' ' << idx[k];
      out << '\n';
    }
    out << "CELL_DATA " << nc << "\nSCALARS u_mean double 1\nLOOKUP_TABLE default\n";
    for (double m : means) {
      std::snprintf(buf, sizeof buf, "%.17g\n", m);
      out << buf;
    }
  } else {
    out << "cell_id,centroid_x,centroid_y,u_mean\n";
    for (int c = 0; c < nc; ++c) {
      const Pt ctr = mesh.centroid(c);
      std::snprintf(buf, sizeof buf, "%d,%.17g,%.17g,%.17g\n", c, ctr.x, ctr.y, means[c]);
      out << buf;
    }
  }
  if (!out) throw IoError("snapshot write failed: " + path);
}

}  // namespace pdg
