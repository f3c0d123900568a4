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

namespace {

// Per-subtree totals used to decide what fits into one bundle.
struct BundleAcc {
  std::int64_t fb = 0, hb = 0;  // panel bytes (F, H)
  int mf = 4, mb = 4;           // bmeta ints (forward, backward), header included
  int nt = 0, hmax = 0;
  int x = 0;                    // shared-memory doubles: sum of 2 w + nr (backward inputs + results)
  void add(const BundleAcc& o) {
    fb += o.fb;
    hb += o.hb;
    mf += o.mf - 4;
    mb += o.mb - 4;
    nt += o.nt;
    x += o.x;
    hmax = std::max(hmax, o.hmax);
  }
};

struct BundleCaps {
  std::int64_t bytes;
  int meta, x, tasks;
  bool fits(const BundleAcc& a) const {
    if (a.fb > bytes || a.hb > bytes || a.nt > tasks || a.x > x) return false;
    return a.mf + 2 * (a.hmax + 1) + 8 <= meta && a.mb + 2 * (a.hmax + 1) + 8 <= meta;
  }
};

int env_int(const char* k, int d) {
  const char* e = std::getenv(k);
  return e ? std::atoi(e) : d;
}

}  // namespace

void pack_unit_tasks(Problem& pr, const SupernodalFactor& F, int coarse, std::int64_t dof_base) {
  constexpr int kTile = 32;
  // Rows per column segment are padded to an even count (each lane streams
  // double2 row pairs); PDG_ROW_ALIGN=8 pads to whole 64-byte bursts, which
  // only added bytes once the L2 re-reads were fixed (config4 sweep 6.40 ms
  // at 2 vs 6.51 ms at 8, profiles/r02e).
  static const int kRowAlign = std::getenv("PDG_ROW_ALIGN") ? std::max(2, std::atoi(std::getenv("PDG_ROW_ALIGN"))) : 2;
  constexpr int kTileAlign = 16;    // 128 bytes
  // Subtree bundles: bottom subtrees of the elimination tree whose panels
  // total <= PDG_BUNDLE_KB per direction go to one CTA as one unit (0: off).
  // Default: only where the sweep is bandwidth bound (>= 2M dofs); smaller
  // problems have idle CTAs and want every supernode on its own one.
  const BundleCaps caps{1024LL * env_int("PDG_BUNDLE_KB", 0), kBundleMetaInts,
                               std::max(64, env_int("PDG_BUNDLE_X", 1536)), std::max(2, env_int("PDG_BUNDLE_TASKS", 64))};
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

  auto seg = [&](int rows) { return (rows + kRowAlign - 1) / kRowAlign * kRowAlign; };
  auto align = [](std::int64_t off) { return (off + kTileAlign - 1) / kTileAlign * kTileAlign; };
  auto tile_len = [&](const Problem::Tile& t) { return align(static_cast<std::int64_t>(t.ncol) * t.stride); };

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
    // forward tiles: output rows of F. Each lane streams double2 pairs of
    // rows; the offsets (128-byte aligned) are assigned below, bundles first.
    t.f_tile0 = static_cast<int>(pr.ftiles.size());
    for (int r0 = 0; r0 < h; r0 += kTile) {
      const int rows = std::min(kTile, h - r0), rs = seg(rows);
      const int ncol = t.root_dense ? w : std::min(w, r0 + rows);
      pr.ftiles.push_back({-1, ncol, 0, rows, rs});
    }
    t.f_ntile = static_cast<int>(pr.ftiles.size()) - t.f_tile0;
    // backward tiles: output rows of H = F^T (columns of F), inputs i >= r0
    t.h_tile0 = static_cast<int>(pr.htiles.size());
    for (int r0 = 0; r0 < (t.root_dense ? 0 : w); r0 += kTile) {
      const int rows = std::min(kTile, w - r0), rs = seg(rows);
      const int ncol = h - r0;
      pr.htiles.push_back({-1, ncol, r0, rows, rs});
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
  std::vector<std::vector<int>> inc_d(F.m);  // the descendant behind each entry
  for (int d = 0; d < nsn; ++d) {
    const Supernode& D = F.sn[d];
    for (std::size_t k = 0; k < D.rows.size(); ++k) {
      inc[D.rows[k]].push_back(pr.tasks[base + d].ubuf_off + static_cast<std::int64_t>(k) * bs);
      inc_d[D.rows[k]].push_back(d);
    }
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

  // ---- subtree bundles ----
  // Bottom-up: a supernode "fits" when its whole subtree stays under the caps;
  // the maximal fitting subtrees, taken in postorder, are packed greedily into
  // bundles (neighbours in postorder are neighbours in the tree). Offsets into
  // dof / ubuf vectors are kept as ints in the bundle records.
  std::vector<std::vector<int>> groups;
  const bool int_ok = pr.ubuf_size < (1LL << 31) - (1 << 20) && dof_base + static_cast<std::int64_t>(F.m) * bs < (1LL << 31) - 1;
  if (!coarse && caps.bytes > 0 && nsn >= 2 && int_ok) {
    std::vector<BundleAcc> acc(nsn);
    std::vector<char> fit(nsn, 1);
    auto own = [&](int s) {
      const TaskDesc& t = pr.tasks[base + s];
      BundleAcc a;
      for (int k = 0; k < t.f_ntile; ++k) a.fb += 8 * tile_len(pr.ftiles[t.f_tile0 + k]);
      for (int k = 0; k < t.h_ntile; ++k) a.hb += 8 * tile_len(pr.htiles[t.h_tile0 + k]);
      const Supernode& S = F.sn[s];
      int nin = 0;
      for (int cc = S.s0; cc < S.s1; ++cc) nin += static_cast<int>(inc[cc].size());
      a.mf += 4 * (S.s1 - S.s0) + nin + 9 * t.f_ntile;
      a.mb += t.h_ntile ? 2 * ((t.w + t.nr) / bs) + 9 * t.h_ntile : 0;
      a.nt = 1;
      a.hmax = height[s];
      a.x = 2 * t.w + t.nr;
      return a;
    };
    for (int s = 0; s < nsn; ++s) {
      bool ok = true;
      for (int c : kids[s]) ok = ok && fit[c];
      if (ok) {
        BundleAcc a = own(s);
        for (int c : kids[s]) a.add(acc[c]);
        ok = caps.fits(a);
        if (ok) acc[s] = std::move(a);
      }
      fit[s] = ok;
      // children's records are only needed while their parent is undecided
      if (ok)
        for (int c : kids[s]) acc[c] = BundleAcc{};
    }
    BundleAcc cur;
    std::vector<int> cur_roots;
    auto flush = [&]() {
      if (cur.nt >= 2) groups.push_back(cur_roots);
      cur = BundleAcc{};
      cur_roots.clear();
    };
    for (int s = 0; s < nsn; ++s) {
      const int p = F.sn[s].parent;
      if (!fit[s] || (p >= 0 && fit[p])) continue;  // maximal fitting subtrees only
      BundleAcc tryacc = cur;
      tryacc.add(acc[s]);
      if (!cur_roots.empty() && !caps.fits(tryacc)) {
        flush();
        tryacc = acc[s];
      }
      cur = std::move(tryacc);
      cur_roots.push_back(s);
    }
    flush();
  }
  // members of each bundle (subtrees are contiguous in postorder), ordered
  // by level for the forward pass
  std::vector<std::vector<int>> members(groups.size());
  {
    std::vector<int> first_desc(nsn);
    for (int s = 0; s < nsn; ++s) {
      first_desc[s] = s;
      for (int c : kids[s]) first_desc[s] = std::min(first_desc[s], first_desc[c]);
    }
    for (std::size_t g = 0; g < groups.size(); ++g) {
      for (int r : groups[g])
        for (int s = first_desc[r]; s <= r; ++s) {
          members[g].push_back(s);
          pr.tasks[base + s].bundle = static_cast<int>(pr.bundles.size() + g);
        }
      std::stable_sort(members[g].begin(), members[g].end(), [&](int a, int c) { return height[a] < height[c]; });
    }
  }
  // ---- panel offsets: bundles first (each contiguous per direction), then
  // the remaining supernodes in order ----
  auto place_f = [&](int s) {
    const TaskDesc& t = pr.tasks[base + s];
    for (int k = 0; k < t.f_ntile; ++k) {
      Problem::Tile& tl = pr.ftiles[t.f_tile0 + k];
      pr.fmat_len = align(pr.fmat_len);
      tl.off = pr.fmat_len;
      pr.fmat_len += static_cast<std::int64_t>(tl.ncol) * tl.stride;
    }
  };
  auto place_h = [&](int s) {
    const TaskDesc& t = pr.tasks[base + s];
    for (int k = 0; k < t.h_ntile; ++k) {
      Problem::Tile& tl = pr.htiles[t.h_tile0 + k];
      pr.hmat_len = align(pr.hmat_len);
      tl.off = pr.hmat_len;
      pr.hmat_len += static_cast<std::int64_t>(tl.ncol) * tl.stride;
    }
  };
  for (std::size_t g = 0; g < groups.size(); ++g) {
    const std::vector<int>& mem = members[g];
    Bundle B;
    B.n_task = static_cast<int>(mem.size());
    pr.fmat_len = align(pr.fmat_len);
    pr.hmat_len = align(pr.hmat_len);
    B.src_off[0] = pr.fmat_len;
    B.src_off[1] = pr.hmat_len;
    for (int s : mem) place_f(s);
    for (auto it = mem.rbegin(); it != mem.rend(); ++it) place_h(*it);  // top level first
    B.bytes[0] = static_cast<int>(8 * (align(pr.fmat_len) - B.src_off[0]));
    B.bytes[1] = static_cast<int>(8 * (align(pr.hmat_len) - B.src_off[1]));
    B.root_off = static_cast<int>(pr.bundle_roots.size());
    B.par_off = static_cast<int>(pr.bundle_parents.size());
    for (int r : groups[g]) {
      pr.bundle_roots.push_back(base + r);
      const int p = F.sn[r].parent;
      if (p >= 0 && std::find(pr.bundle_parents.begin() + B.par_off, pr.bundle_parents.end(), base + p) ==
                        pr.bundle_parents.end())
        pr.bundle_parents.push_back(base + p);
    }
    B.n_root = static_cast<int>(groups[g].size());
    B.n_par = static_cast<int>(pr.bundle_parents.size()) - B.par_off;
    B.nlev = height[mem.back()] + 1;
    // shared-memory layout of the CTA's vector block (doubles). Forward:
    // [t_S of every member][u_S of every member]; backward: [[y_S ; -x_R] of
    // every member with backward tiles][x_S of every member].
    std::vector<int> vx(nsn, -1), ul(nsn, -1), bin(nsn, -1), xs(nsn, -1);
    int sw = 0, snr = 0, sh = 0;
    for (int s : mem) {
      const TaskDesc& t = pr.tasks[base + s];
      vx[s] = sw;
      xs[s] = sw;
      sw += t.w;
    }
    for (int s : mem) {
      const TaskDesc& t = pr.tasks[base + s];
      ul[s] = sw + snr;
      snr += t.nr;
      if (t.h_ntile) {
        bin[s] = sh;
        sh += t.w + t.nr;
      }
    }
    for (int s : mem) xs[s] += sh;
    B.xneed = std::max(sw + snr, sh + sw);
    for (int dir = 0; dir < 2; ++dir) {
      std::vector<int> lev, cells, aux, items;
      int ncell = 0, nitem = 0;
      for (int l = 0; l < B.nlev; ++l) {
        const int hgt = dir == 0 ? l : B.nlev - 1 - l;
        for (int s : mem) {
          if (height[s] != hgt) continue;
          const TaskDesc& t = pr.tasks[base + s];
          const Supernode& S = F.sn[s];
          if (dir == 0) {
            for (int cc = S.s0; cc < S.s1; ++cc) {
              cells.push_back(static_cast<int>(dof_base + static_cast<std::int64_t>(cc) * bs));
              cells.push_back(vx[s] + (cc - S.s0) * bs);
              cells.push_back(static_cast<int>(aux.size()));
              for (std::size_t e = 0; e < inc[cc].size(); ++e) {
                const int d = inc_d[cc][e];  // a descendant, hence a member
                aux.push_back(ul[d] + static_cast<int>(inc[cc][e] - pr.tasks[base + d].ubuf_off));
              }
              cells.push_back(static_cast<int>(aux.size()));
              ++ncell;
            }
            for (int k = 0; k < t.f_ntile; ++k) {
              const Problem::Tile& tl = pr.ftiles[t.f_tile0 + k];
              const int r0 = k * kTile;
              items.push_back(static_cast<int>(tl.off - B.src_off[0]));
              items.push_back(tl.ncol);
              items.push_back(tl.rows | (t.root_dense << 30));
              items.push_back(tl.stride);
              items.push_back(vx[s]);
              items.push_back(t.root_dense ? tl.rows : std::clamp(t.w - r0, 0, tl.rows));
              items.push_back(static_cast<int>(t.dof0) + r0);
              items.push_back(static_cast<int>(t.ubuf_off) + r0 - t.w);
              items.push_back(ul[s] + r0 - t.w);
              ++nitem;
            }
          } else if (t.h_ntile) {
            // own y_S and the rows owned by supernodes outside the bundle (or
            // by its dense root, whose x_S the forward pass left in z) are
            // known when the unit starts; rows of members are copied level by
            // level from the x_S block
            for (int cc = S.s0; cc < S.s1; ++cc) {
              aux.push_back(static_cast<int>(dof_base + static_cast<std::int64_t>(cc) * bs));
              aux.push_back(bin[s] + (cc - S.s0) * bs);
            }
            for (std::size_t k = 0; k < S.rows.size(); ++k) {
              const int q = S.rows[k], m = F.sn_of[q];
              const int xo = bin[s] + t.w + static_cast<int>(k) * bs;
              if (pr.tasks[base + m].bundle == pr.tasks[base + s].bundle && !pr.tasks[base + m].root_dense) {
                cells.push_back(xs[m] + (q - F.sn[m].s0) * bs);
                cells.push_back(xo);
                ++ncell;
              } else {
                aux.push_back(-1 - static_cast<int>(dof_base + static_cast<std::int64_t>(q) * bs));
                aux.push_back(xo);
              }
            }
            for (int k = 0; k < t.h_ntile; ++k) {
              const Problem::Tile& tl = pr.htiles[t.h_tile0 + k];
              items.push_back(static_cast<int>(tl.off - B.src_off[1]));
              items.push_back(tl.ncol);
              items.push_back(tl.rows);
              items.push_back(tl.stride);
              items.push_back(bin[s] + tl.col0);
              items.push_back(tl.rows);
              items.push_back(static_cast<int>(t.dof0) + tl.col0);
              items.push_back(0);
              items.push_back(xs[s] + tl.col0);
              ++nitem;
            }
          }
        }
        lev.push_back(ncell);
        lev.push_back(nitem);
      }
      while (pr.bmeta.size() % 4) pr.bmeta.push_back(0);  // 16-byte aligned records (L2 bulk prefetch)
      B.meta_off[dir] = static_cast<int>(pr.bmeta.size());
      pr.bmeta.push_back(B.nlev);
      pr.bmeta.push_back(ncell);
      pr.bmeta.push_back(nitem);
      pr.bmeta.push_back(static_cast<int>(dir == 0 ? aux.size() : aux.size() / 2));
      pr.bmeta.insert(pr.bmeta.end(), lev.begin(), lev.end());
      pr.bmeta.insert(pr.bmeta.end(), cells.begin(), cells.end());
      pr.bmeta.insert(pr.bmeta.end(), aux.begin(), aux.end());
      pr.bmeta.insert(pr.bmeta.end(), items.begin(), items.end());
      while (pr.bmeta.size() % 4) pr.bmeta.push_back(0);
      B.meta_n[dir] = static_cast<int>(pr.bmeta.size()) - B.meta_off[dir];
      if (B.meta_n[dir] > kBundleMetaInts) throw SolverError("pack: bundle record exceeds its shared-memory block");
    }
    pr.bundles.push_back(B);
  }
  for (int s = 0; s < nsn; ++s)
    if (pr.tasks[base + s].bundle < 0) {
      place_f(s);
      place_h(s);
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
