// Device packing of the exact local factors (see problem.hpp pack_unit_tasks).
//
// For a supernode S with w columns and nr below rows (h = w + nr), the sweep
// reads ONE dense panel per direction:
//   forward   F = [ inv(L_SS) ; L_RS inv(L_SS) ]     (h x w):   [y_S ; u_S] = F t_S
//   backward  H = F^T                                 (w x h):   x_S = H [y_S ; -x_R]
// since x_S = inv(L_SS)^T (y_S - L_RS^T x_R) = inv(L_SS)^T y_S - (L_RS inv(L_SS))^T x_R.
// Each task is therefore a single independent mat-vec (no intra-task
// dependency chain). Panels are stored in 32-row tiles (column-major inside a
// tile, last tile not padded) so a warp reads one coalesced 8*rows-byte row
// segment per input column; the zero upper triangle of inv(L_SS) is skipped
// at tile granularity. This file only lays the tiles out; F and H are formed
// on the device from inv(L_SS) and L_RS (cuda/panels.cu).
#include <algorithm>
#include <cstdlib>

#include "problem.hpp"

namespace pdg {

void pack_unit_tasks(Problem& pr, const SupernodalFactor& F, int coarse, std::int64_t dof_base) {
  constexpr int kTile = 32;
  // Rows per column segment are padded to an even count (each lane streams
  // double2 row pairs); PDG_ROW_ALIGN=8 pads to whole 64-byte bursts, which
  // only added bytes once the L2 re-reads were fixed (config4 sweep 6.40 ms
  // at 2 vs 6.51 ms at 8, profiles/r02e).
  static const int kRowAlign = std::getenv("PDG_ROW_ALIGN") ? std::max(2, std::atoi(std::getenv("PDG_ROW_ALIGN"))) : 2;
  constexpr int kTileAlign = 16;    // 128 bytes
  const int bs = F.bs;
  const int base = static_cast<int>(pr.tasks.size());
  const int nsn = static_cast<int>(F.sn.size());
  std::vector<std::vector<int>> kids(nsn);
  for (int s = 0; s < nsn; ++s)
    if (F.sn[s].parent >= 0) kids[F.sn[s].parent].push_back(s);
  std::vector<int> height(nsn, 0), depth(nsn, 0);
  for (int s = 0; s < nsn; ++s)
    for (int c : kids[s]) height[s] = std::max(height[s], height[c] + 1);
  for (int s = nsn - 1; s >= 0; --s)
    if (F.sn[s].parent >= 0) depth[s] = depth[F.sn[s].parent] + 1;

  std::vector<int> slot(nsn);
  for (int s = 0; s < nsn; ++s) {
    const Supernode& S = F.sn[s];
    const int w = S.w(bs), nr = static_cast<int>(S.rows.size()) * bs, h = w + nr;
    TaskDesc t;
    t.coarse = coarse;
    t.bs = bs;
    t.w = w;
    t.nr = nr;
    t.dof0 = dof_base + static_cast<std::int64_t>(S.s0) * bs;
    // factor values for the device panel builder (cuda/panels.cu); a
    // symbolic-only factor (device factorisation, cuda/factor.cu) reserves
    // the space
    t.linv_off = pr.lval_len;
    pr.lval_len += static_cast<std::int64_t>(w) * (w + 1) / 2;
    t.b_off = pr.lval_len;
    pr.lval_len += static_cast<std::int64_t>(nr) * w;
    if (!S.Linv.empty()) {
      if (pr.lval.empty()) pr.lval_host0 = t.linv_off;
      if (pr.lval_host0 + static_cast<std::int64_t>(pr.lval.size()) != t.linv_off)
        throw SolverError("pack: host factor values must follow the device-factored tasks");
      pr.lval.insert(pr.lval.end(), S.Linv.begin(), S.Linv.end());
      pr.lval.insert(pr.lval.end(), S.B.begin(), S.B.end());
    }
    // a root with no below rows takes one dense symmetric panel
    t.root_dense = S.parent < 0 && nr == 0 ? 1 : 0;
    // forward tiles: output rows of F
    // Tiles start 128-byte aligned; each lane streams double2 pairs of rows.
    auto seg = [&](int rows) { return (rows + kRowAlign - 1) / kRowAlign * kRowAlign; };
    auto align = [](std::int64_t off) { return (off + kTileAlign - 1) / kTileAlign * kTileAlign; };
    t.f_tile0 = static_cast<int>(pr.ftiles.size());
    for (int r0 = 0; r0 < h; r0 += kTile) {
      const int rows = std::min(kTile, h - r0), rs = seg(rows);
      const int ncol = t.root_dense ? w : std::min(w, r0 + rows);
      pr.fmat_len = align(pr.fmat_len);
      pr.ftiles.push_back({pr.fmat_len, ncol, 0, rows, rs});
      pr.fmat_len += static_cast<std::int64_t>(ncol) * rs;
    }
    t.f_ntile = static_cast<int>(pr.ftiles.size()) - t.f_tile0;
    // backward tiles: output rows of H = F^T (columns of F), inputs i >= r0
    t.h_tile0 = static_cast<int>(pr.htiles.size());
    for (int r0 = 0; r0 < (t.root_dense ? 0 : w); r0 += kTile) {
      const int rows = std::min(kTile, w - r0), rs = seg(rows);
      const int ncol = h - r0;
      pr.hmat_len = align(pr.hmat_len);
      pr.htiles.push_back({pr.hmat_len, ncol, r0, rows, rs});
      pr.hmat_len += static_cast<std::int64_t>(ncol) * rs;
    }
    t.h_ntile = static_cast<int>(pr.htiles.size()) - t.h_tile0;
    t.rows_off = static_cast<int>(pr.row_dof.size());
    for (int qpos : S.rows) pr.row_dof.push_back(dof_base + static_cast<std::int64_t>(qpos) * bs);
    t.ubuf_off = pr.ubuf_size;
    pr.ubuf_size += nr;
    t.parent = S.parent >= 0 ? base + S.parent : -1;
    t.child_off = static_cast<int>(pr.task_child.size());
    for (int c : kids[s]) pr.task_child.push_back(base + c);
    t.n_child = static_cast<int>(kids[s].size());
    t.height = height[s];
    t.depth = depth[s];
    slot[s] = static_cast<int>(pr.in_ptr.size()) - 1;
    t.in_off = slot[s];
    for (int cc = S.s0; cc < S.s1; ++cc) pr.in_ptr.push_back(pr.in_ptr.back());  // filled below
    pr.tasks.push_back(t);
  }
  // incoming lists: (S, cell) <- ubuf slices of descendants D, in D order
  std::vector<std::vector<std::int64_t>> inc(F.m);
  for (int d = 0; d < nsn; ++d) {
    const Supernode& D = F.sn[d];
    for (std::size_t k = 0; k < D.rows.size(); ++k)
      inc[D.rows[k]].push_back(pr.tasks[base + d].ubuf_off + static_cast<std::int64_t>(k) * bs);
  }
  for (int s = 0; s < nsn; ++s) {
    const Supernode& S = F.sn[s];
    int at = slot[s];
    for (int cc = S.s0; cc < S.s1; ++cc) {
      pr.in_idx.insert(pr.in_idx.end(), inc[cc].begin(), inc[cc].end());
      pr.in_ptr[at + 1] = static_cast<int>(pr.in_idx.size());
      ++at;
    }
  }
  pr.factor_values = pr.fmat_len + pr.hmat_len;
}

}  // namespace pdg

namespace pdg {

void halo_plan(const Problem& pr, std::vector<std::vector<int>>& send, std::vector<std::vector<int>>& recv) {
  const int w = pr.cfg.world, r = pr.cfg.rank;
  auto owner_rank = [&](int g) {
    return static_cast<int>(std::upper_bound(pr.rank_cell_start.begin(), pr.rank_cell_start.end(), g) -
                            pr.rank_cell_start.begin()) - 1;
  };
  send.assign(w, {});
  recv.assign(w, {});
  for (const Face& f : pr.mesh.interior_faces()) {
    const int a = pr.iperm[f.cell_in], c = pr.iperm[f.cell_out];
    const int ra = owner_rank(a), rc = owner_rank(c);
    if (ra == rc) continue;
    if (ra == r) {
      send[rc].push_back(a - pr.cell_begin);
      recv[rc].push_back(c);
    }
    if (rc == r) {
      send[ra].push_back(c - pr.cell_begin);
      recv[ra].push_back(a);
    }
  }
  for (int p = 0; p < w; ++p) {
    for (auto* v : {&send[p], &recv[p]}) {
      std::sort(v->begin(), v->end());
      v->erase(std::unique(v->begin(), v->end()), v->end());
    }
  }
}

}  // namespace pdg
