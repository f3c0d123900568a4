// Snapshot output (snapshot.hpp:13-22 of the reference): formats per-cell
// means computed on the device.
#pragma once

#include <string>
#include <vector>

#include "mesh.hpp"

namespace pdg {

// vtk-legacy (POLYDATA + CELL_DATA u_mean) or csv-cellmeans; means in
// reference cell order. Throws ConfigError (format) / IoError (file).
void write_snapshot(const Mesh& mesh, const std::vector<double>& means, double t, const std::string& path,
                    const std::string& format);

}  // namespace pdg
