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

int env_int(const char* k, int d) {
  const char* e = std::getenv(k);
  return e ? std::atoi(e) : d;
}

// doubles of a level chunk's input vectors in the sweep CTA's shared block
int chunk_x_cap() { return std::max(64, env_int("PDG_CHUNK_X", 1536)); }

constexpr int kTileAlign = 16;  // panel tiles start 128-byte aligned
std::int64_t align_tile(std::int64_t off) { return (off + kTileAlign - 1) / kTileAlign * kTileAlign; }

}  // namespace

long long bottom_level_bytes(long long dofs_per_rank, int b) {
  return 1024LL * env_int("PDG_BOTTOM_KB", dofs_per_rank >= 2000000 && b >= 6 ? kBottomDefaultKB : 0);
}

void pack_unit_tasks(Problem& pr, const SupernodalFactor& F, int coarse, std::int64_t dof_base) {
  constexpr int kTile = 32;
  // Rows per column segment are padded to an even count (each lane streams
  // double2 row pairs); PDG_ROW_ALIGN=8 pads to whole 64-byte bursts, which
  // only added bytes once the L2 re-reads were fixed (config4 sweep 6.40 ms
  // at 2 vs 6.51 ms at 8, profiles/r02e).
  static const int kRowAlign = std::getenv("PDG_ROW_ALIGN") ? std::max(2, std::atoi(std::getenv("PDG_ROW_ALIGN"))) : 2;
  // Bottom levels: the supernodes of every subtree whose panels total <=
  // PDG_BOTTOM_KB per direction are not scheduled one by one; they are solved
  // level by level in chunks (finish_bottom_levels below). 0: off.
  const std::int64_t bottom_bytes = bottom_level_bytes(pr.n_global_dofs() / std::max(1, pr.cfg.world), pr.b);
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
  auto align = [](std::int64_t off) { return align_tile(off); };

  // ---- bottom levels: whole subtrees under the byte cap, at most
  // PDG_BOTTOM_LEVELS high, supernodes at most 32 columns wide ----
  std::vector<char> bottom(nsn, 0);
  if (!coarse && bottom_bytes > 0 && pr.n_global_dofs() < (1LL << 30)) {  // chunk records hold int offsets
    const int max_levels = std::max(1, env_int("PDG_BOTTOM_LEVELS", kBottomDefaultLevels));
    const int chunk_x = chunk_x_cap();
    // incoming updates per cell (one per descendant row block): part of a chunk record's size
    std::vector<int> incount(F.m, 0);
    for (const Supernode& D : F.sn)
      for (int q : D.rows) ++incount[q];
    std::vector<std::int64_t> fb(nsn, 0);
    for (int s = 0; s < nsn; ++s) {
      const Supernode& S = F.sn[s];
      const int w = S.w(bs), h = w + static_cast<int>(S.rows.size()) * bs;
      int ntile = 0, nin = 0;
      for (int r0 = 0; r0 < h; r0 += kTile, ++ntile)
        fb[s] += 8 * align(static_cast<std::int64_t>(w) * seg(std::min(kTile, h - r0)));
      for (int cc = S.s0; cc < S.s1; ++cc) nin += incount[cc];
      // a supernode must fit a level chunk on its own: its input vector in the
      // CTA's shared block and its share of the record in half the record block
      const int rec = 4 * (S.s1 - S.s0) + nin + 2 * (h / bs) + 8 * (ntile + 1);
      bool ok = w <= 32 && height[s] < max_levels && h <= chunk_x && rec <= kChunkMetaInts / 2;
      for (int c : kids[s]) {
        ok = ok && bottom[c];
        fb[s] += fb[c];
      }
      bottom[s] = ok && fb[s] <= bottom_bytes;
    }
  }

  std::vector<int> slot(nsn);
  for (int s = 0; s < nsn; ++s) {
    const Supernode& S = F.sn[s];
    const int w = S.w(bs), nr = static_cast<int>(S.rows.size()) * bs, h = w + nr;
    TaskDesc t;
    t.bottom = bottom[s] ? 0 : -1;
    t.unit = pr.n_packed_units;
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
    // rows; the offsets (128-byte aligned) are assigned below (the bottom levels in finish_bottom_levels).
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

  ++pr.n_packed_units;
  // ---- panel offsets of the individually scheduled supernodes (the bottom
  // levels are laid out level by level in finish_bottom_levels) ----
  for (int s = 0; s < nsn; ++s) {
    const TaskDesc& t = pr.tasks[base + s];
    if (t.bottom >= 0) continue;
    for (int k = 0; k < t.f_ntile; ++k) {
      Problem::Tile& tl = pr.ftiles[t.f_tile0 + k];
      pr.fmat_len = align(pr.fmat_len);
      tl.off = pr.fmat_len;
      pr.fmat_len += static_cast<std::int64_t>(tl.ncol) * tl.stride;
    }
    for (int k = 0; k < t.h_ntile; ++k) {
      Problem::Tile& tl = pr.htiles[t.h_tile0 + k];
      pr.hmat_len = align(pr.hmat_len);
      tl.off = pr.hmat_len;
      pr.hmat_len += static_cast<std::int64_t>(tl.ncol) * tl.stride;
    }
  }
  pr.factor_values = pr.fmat_len + pr.hmat_len;
}

// The bottom levels of all subdomains as level chunks (problem.hpp LevelChunk):
// per direction and per height, the bottom supernodes in task order are cut
// into chunks of <= PDG_CHUNK_KB of panel whose input vectors fit the sweep
// CTA's shared block; each chunk's panels are contiguous and its record lists
// where every input comes from and where every tile's rows go.
void finish_bottom_levels(Problem& pr) {
  constexpr int kTile = 32;
  const std::int64_t chunk_bytes = 1024LL * std::max(4, env_int("PDG_CHUNK_KB", 64));
  const int xcap = chunk_x_cap();
  const int nt = static_cast<int>(pr.tasks.size());
  int lmax = -1;
  for (const TaskDesc& t : pr.tasks)
    if (t.bottom >= 0) lmax = std::max(lmax, t.height);
  pr.n_bottom_levels = lmax + 1;
  pr.n_bottom_groups = 0;
  pr.level_chunks[0].clear();
  pr.level_chunks[1].clear();
  if (lmax < 0) return;
  if (pr.ubuf_size >= (1LL << 31)) throw SolverError("pack: update buffer too large for the level chunk records");
  const int nlev = lmax + 1;
  // groups of consecutive subdomains holding about group_bytes of bottom forward panel
  const std::int64_t group_bytes = (1LL << 20) * std::max(1, env_int("PDG_BOTTOM_GROUP_MB", 192));
  std::vector<int> group_of_unit(std::max(pr.n_packed_units, 1), 0);
  {
    std::vector<std::int64_t> ub(group_of_unit.size(), 0);
    for (const TaskDesc& t : pr.tasks)
      if (t.bottom >= 0) ub[t.unit] += 8LL * t.w * (t.w + t.nr);
    std::int64_t acc = 0;
    int g = 0;
    for (std::size_t u = 0; u < ub.size(); ++u) {
      if (acc > 0 && acc + ub[u] > group_bytes) {
        ++g;
        acc = 0;
      }
      group_of_unit[u] = g;
      acc += ub[u];
    }
    pr.n_bottom_groups = g + 1;
  }
  // Levels below PDG_BOTTOM_GROUP_LEVELS run group by group (group counters),
  // the few supernodes above them level by level over all groups (global
  // counters, slots ngroups * nlev + level): near the top a group has too few
  // chunks to keep a level's dependencies a safe distance behind it.
  // Default: every level grouped, in the skewed order below with groups of
  // ~192 MB (config 4 sweep 5.55 -> 5.45 ms, config 5 p=2 2.21 -> 2.10 ms,
  // profiles/r02af, r02ag). Smaller groups or the block-interleaved order
  // (PDG_BOTTOM_INTERLEAVE > 0) put a level's dependencies too close behind it
  // in the ticket order and the CTAs wait (>= 7 ms, profiles/r02y).
  const int glev = std::clamp(env_int("PDG_BOTTOM_GROUP_LEVELS", 99), 0, nlev);
  const int inter = std::max(0, env_int("PDG_BOTTOM_INTERLEAVE", 0));
  const int ngroups = pr.n_bottom_groups, nslots = ngroups * nlev + nlev;
  auto gslot = [&](int level) { return ngroups * nlev + level; };
  pr.level_chunks[0].assign(nslots, 0);
  pr.level_chunks[1].assign(nslots, 0);
  std::vector<std::vector<int>> by_slot(nslots);
  std::vector<int> gmax(ngroups, -1);  // highest bottom level of each group
  for (int i = 0; i < nt; ++i)
    if (pr.tasks[i].bottom >= 0) {
      const int g = group_of_unit[pr.tasks[i].unit], l = pr.tasks[i].height;
      by_slot[l < glev ? g * nlev + l : gslot(l)].push_back(i);
      gmax[g] = std::max(gmax[g], l);
    }
  auto is_regular = [&](int p) { return p >= 0 && pr.tasks[p].bottom < 0; };
  for (int dir = 0; dir < 2; ++dir) {
    auto& tiles = dir == 0 ? pr.ftiles : pr.htiles;
    std::int64_t& mat_len = dir == 0 ? pr.fmat_len : pr.hmat_len;
    // slots in ticket order. Forward: `inter` groups at a time, level by level,
    // then the global levels; backward the reverse (top level first).
    std::vector<int> slot_order;
    if (dir == 1)
      for (int l = nlev - 1; l >= glev; --l) slot_order.push_back(gslot(l));
    if (inter > 0) {  // `inter` groups at a time, level by level
      for (int g0 = 0; g0 < ngroups; g0 += inter)
        for (int li = 0; li < glev; ++li)
          for (int g = g0; g < std::min(ngroups, g0 + inter); ++g)
            slot_order.push_back(g * nlev + (dir == 0 ? li : glev - 1 - li));
    } else {
      // skewed: step t runs level li of group t - li for every li, so a
      // group's consecutive levels are always one whole step (about one
      // group's worth of chunks from glev different groups) apart
      for (int t = 0; t < ngroups + glev - 1; ++t)
        for (int li = 0; li < glev; ++li) {
          const int g = t - li;
          if (g >= 0 && g < ngroups) slot_order.push_back(g * nlev + (dir == 0 ? li : glev - 1 - li));
        }
    }
    if (dir == 0)
      for (int l = glev; l < nlev; ++l) slot_order.push_back(gslot(l));
    for (int slot : slot_order) {
      const bool global = slot >= ngroups * nlev;
      const int level = global ? slot - ngroups * nlev : slot % nlev, group = global ? -1 : slot / nlev;
      const std::vector<int>& lt = by_slot[slot];
      std::size_t at = 0;
      while (at < lt.size()) {
        // greedy: tasks [at, e) while the chunk stays under every cap
        std::int64_t bytes = 0;
        int x = 0, meta = 4;
        std::size_t e = at;
        while (e < lt.size()) {
          const TaskDesc& t = pr.tasks[lt[e]];
          const int t0 = dir == 0 ? t.f_tile0 : t.h_tile0, n = dir == 0 ? t.f_ntile : t.h_ntile;
          std::int64_t tb = 0;
          for (int k = 0; k < n; ++k) tb += 8 * align_tile(static_cast<std::int64_t>(tiles[t0 + k].ncol) * tiles[t0 + k].stride);
          int tm = 8 * n, tx = 0;
          if (dir == 0) {
            const int nc = t.w / t.bs;
            tm += 4 * nc + pr.in_ptr[t.in_off + nc] - pr.in_ptr[t.in_off];
            tx = t.w;
          } else if (n) {
            tm += 2 * ((t.w + t.nr) / t.bs);
            tx = t.w + t.nr;
          }
          if (e > at && (bytes + tb > chunk_bytes || x + tx > xcap || meta + tm + 12 > kChunkMetaInts)) break;
          if (tx > xcap || meta + tm + 12 > kChunkMetaInts)
            throw SolverError("pack: a bottom-level supernode does not fit a level chunk");
          bytes += tb;
          x += tx;
          meta += tm;
          ++e;
        }
        LevelChunk C;
        C.dir = dir;
        C.level = level;
        // counters: every chunk adds to its global level counter, a grouped
        // one also to its group's; it waits for the level before it (backward:
        // above it) in the same scope, the first backward level for the last
        // forward one
        C.slot = global ? -1 : slot;
        C.gslot = gslot(level);
        if (dir == 0 && level > 0) {
          C.dep_dir = 0;
          C.dep_slot = global ? gslot(level - 1) : slot - 1;
        } else if (dir == 1) {
          if (global) {
            C.dep_dir = level < lmax ? 1 : 0;
            C.dep_slot = level < lmax ? gslot(level + 1) : gslot(lmax);
          } else if (level + 1 < glev && level < gmax[group]) {
            C.dep_dir = 1;
            C.dep_slot = slot + 1;
          } else if (level + 1 == glev && glev <= lmax) {
            C.dep_dir = 1;
            C.dep_slot = gslot(glev);
          } else {  // the group's top level
            C.dep_dir = 0;
            C.dep_slot = group * nlev + gmax[group];
          }
        }
        C.first_task = lt[at];
        C.n_task = static_cast<int>(e - at);
        mat_len = align_tile(mat_len);
        C.src_off = mat_len;
        C.root_off = static_cast<int>(pr.chunk_roots.size());
        C.par_off = static_cast<int>(pr.chunk_parents.size());
        std::vector<int> cells, aux, items;
        int ncell = 0, nitem = 0, xo = 0;
        for (std::size_t q = at; q < e; ++q) {
          const int ti = lt[q];
          const TaskDesc& t = pr.tasks[ti];
          const int t0 = dir == 0 ? t.f_tile0 : t.h_tile0, n = dir == 0 ? t.f_ntile : t.h_ntile;
          for (int k = 0; k < n; ++k) {  // panels: contiguous in chunk order
            Problem::Tile& tl = tiles[t0 + k];
            mat_len = align_tile(mat_len);
            tl.off = mat_len;
            mat_len += static_cast<std::int64_t>(tl.ncol) * tl.stride;
            if (tl.ncol % t.bs) throw SolverError("pack: bottom-level tile width is not a whole number of blocks");
          }
          if (dir == 0) {
            if (is_regular(t.parent)) pr.chunk_roots.push_back(ti);
            const int nc = t.w / t.bs;
            for (int c = 0; c < nc; ++c) {
              cells.push_back(static_cast<int>(t.dof0) + c * t.bs);
              cells.push_back(xo + c * t.bs);
              cells.push_back(static_cast<int>(aux.size()));
              for (int k = pr.in_ptr[t.in_off + c]; k < pr.in_ptr[t.in_off + c + 1]; ++k)
                aux.push_back(static_cast<int>(pr.in_idx[k]));
              cells.push_back(static_cast<int>(aux.size()));
              ++ncell;
            }
            for (int k = 0; k < n; ++k) {
              const Problem::Tile& tl = tiles[t0 + k];
              const int r0 = k * kTile;
              items.push_back(static_cast<int>(tl.off - C.src_off));
              items.push_back(tl.ncol);
              items.push_back(tl.rows | (t.root_dense << 30));
              items.push_back(tl.stride);
              items.push_back(xo);
              items.push_back(t.root_dense ? tl.rows : std::clamp(t.w - r0, 0, tl.rows));
              items.push_back(static_cast<int>(t.dof0) + r0);
              items.push_back(static_cast<int>(t.ubuf_off) + r0 - t.w);
              ++nitem;
            }
            xo += t.w;
          } else if (n) {
            if (is_regular(t.parent) &&
                std::find(pr.chunk_parents.begin() + C.par_off, pr.chunk_parents.end(), t.parent) == pr.chunk_parents.end())
              pr.chunk_parents.push_back(t.parent);
            for (int c = 0; c < t.w / t.bs; ++c) {
              cells.push_back(static_cast<int>(t.dof0) + c * t.bs);
              cells.push_back(xo + c * t.bs);
              ++ncell;
            }
            for (int c = 0; c < t.nr / t.bs; ++c) {
              cells.push_back(-1 - static_cast<int>(pr.row_dof[t.rows_off + c]));
              cells.push_back(xo + t.w + c * t.bs);
              ++ncell;
            }
            for (int k = 0; k < n; ++k) {
              const Problem::Tile& tl = tiles[t0 + k];
              items.push_back(static_cast<int>(tl.off - C.src_off));
              items.push_back(tl.ncol);
              items.push_back(tl.rows);
              items.push_back(tl.stride);
              items.push_back(xo + tl.col0);
              items.push_back(tl.rows);
              items.push_back(static_cast<int>(t.dof0) + tl.col0);
              items.push_back(0);
              ++nitem;
            }
            xo += t.w + t.nr;
          }
        }
        C.bytes = static_cast<int>(8 * (align_tile(mat_len) - C.src_off));
        C.n_root = static_cast<int>(pr.chunk_roots.size()) - C.root_off;
        C.n_par = static_cast<int>(pr.chunk_parents.size()) - C.par_off;
        C.xneed = xo;
        while (pr.bmeta.size() % 4) pr.bmeta.push_back(0);  // 16-byte aligned records
        C.meta_off = static_cast<int>(pr.bmeta.size());
        // the items are read as int4 pairs: an even number of backward cells
        // (2 ints each) and the aux list padded to a multiple of 4 ints
        if (dir == 1 && (ncell & 1)) {
          cells.push_back(cells[cells.size() - 2]);  // repeat the last cell (same value, same slot)
          cells.push_back(cells[cells.size() - 2]);
          ++ncell;
        }
        pr.bmeta.push_back(ncell);
        pr.bmeta.push_back(nitem);
        pr.bmeta.push_back(static_cast<int>(aux.size()));
        pr.bmeta.push_back(0);
        while (aux.size() % 4) aux.push_back(0);
        pr.bmeta.insert(pr.bmeta.end(), cells.begin(), cells.end());
        pr.bmeta.insert(pr.bmeta.end(), aux.begin(), aux.end());
        pr.bmeta.insert(pr.bmeta.end(), items.begin(), items.end());
        while (pr.bmeta.size() % 4) pr.bmeta.push_back(0);
        C.meta_n = static_cast<int>(pr.bmeta.size()) - C.meta_off;
        if (C.meta_n > kChunkMetaInts) throw SolverError("pack: level chunk record exceeds its shared-memory block");
        // a chunk with no tiles (backward, dense roots only) still counts for its level
        pr.chunks.push_back(C);
        if (C.slot >= 0) ++pr.level_chunks[dir][C.slot];
        ++pr.level_chunks[dir][C.gslot];
        at = e;
      }
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
