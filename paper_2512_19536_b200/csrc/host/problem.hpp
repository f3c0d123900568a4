// Host-side problem setup: config -> mesh -> partitions -> internal ordering
// -> assembly (BSR) -> Schwarz factors -> coarse space, packed as flat
// arrays ("device image") that the CUDA side uploads once.
//
// Mirrors the setup half of Simulation::Simulation
// (/root/reference/proj/src/timestepper.cpp:67-126) with the BASELINE.json
// extensions (multi-cell subdomains, explicit coarse count, per-element
// fibres). K_h is time-independent (timestepper.hpp:113-115), so everything
// here runs once.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "../../../include/polydg_b200.h"
#include "factor.hpp"
#include "mesh.hpp"

namespace pdg {

// Block-sparse rows over internal cells. Block (row i, col j) at
// val[k*b*b + c*b + r] = entry (r, c) (column-major blocks).
struct Bsr {
  int rows = 0, b = 0;
  std::vector<int> ptr, col;
  std::vector<double> val;
};

// One supernode task of the device sweep (fine subdomain or coarse problem).
struct TaskDesc {
  int coarse = 0;      // 0 = fine vector set (r -> z), 1 = coarse (r0 -> y0)
  int bs = 0;          // block size of this unit
  int w = 0;           // supernode columns (cells * bs)
  int nr = 0;          // below rows (|R| * bs)
  std::int64_t dof0 = 0;    // first dof of the supernode in its vector
  int f_tile0 = 0, f_ntile = 0;  // forward tiles of F = [inv(L_SS); L_RS inv(L_SS)]
  int h_tile0 = 0, h_ntile = 0;  // backward tiles of H = F^T
  int rows_off = 0;    // R cell dof-starts in row_dof[rows_off .. + nr/bs)
  std::int64_t ubuf_off = 0;  // update buffer slot (nr doubles)
  int in_off = 0;      // incoming CSR: in_ptr[in_off .. in_off + w/bs]
  int parent = -1;     // task id (ND parent), -1 = root
  int child_off = 0, n_child = 0;  // children ids in task_child[]
  int height = 0, depth = 0;
  // root supernode applied as ONE dense symmetric mat-vec x_S = inv(K_SS) t_S
  // (G = inv(L_SS)^T inv(L_SS) in the forward tiles, no backward tiles): its
  // forward and backward solves collapse into one level of the sweep
  int root_dense = 0;
  std::int64_t linv_off = 0, b_off = 0;  // inv(L_SS) and L_RS of this supernode in Problem::lval
  int bottom = -1;     // >= 0: a bottom-level supernode, solved inside level chunks (LevelChunk)
  int unit = 0;        // which pack_unit_tasks call (subdomain) it came from
};

// Bottom levels of the sweep. The supernodes of every small bottom subtree
// (TaskDesc::bottom >= 0; host/pack.cpp) are not scheduled one by one: per
// direction and per tree height they are cut into LEVEL CHUNKS, each solved by
// one CTA as one unit (cuda/sweep.cu run_chunk): gather the inputs of all its
// supernodes into shared memory, one barrier, one warp per 32-row tile. All
// chunks of a level are independent; a level waits for the previous one
// through one counter per level, so no per-supernode dependency is tracked.
// The subdomains are taken in GROUPS of about PDG_BOTTOM_GROUP_MB of bottom
// panel, each with its own level counters, in a skewed ticket order (step t
// runs level l of group t - l): part of a level's updates is then read back
// from the L2 instead of DRAM, and a level's dependencies were issued one
// whole step (about a group's worth of chunks) earlier.
// A chunk's panels are contiguous and its record is one block of ints in
// bmeta (16-byte aligned):
//   [ncell, nitem, naux, 0] ,
//   cells, forward {dof, xoff, in0, in1}: t = r[dof..] minus ubuf[aux[in0..in1)] ,
//          backward {src, xoff}: y_S (src >= 0) or -x_R (z at -1-src) ,
//   aux (forward): ubuf offsets of the incoming updates ,
//   items (one 32-row tile each): {panel offset - src_off, ncol, rows | dense_root << 30, stride,
//                                  xoff, wsplit, dst_a, dst_b}: rows < wsplit go to y_S (dense
//                                  root: x_S) at dst_a, the rest to ubuf at dst_b; backward rows to z at dst_a.
constexpr int kChunkMetaInts = 2560;  // shared-memory block of the sweep CTA (cuda/sweep.cu)
constexpr int kBottomDefaultKB = 160;  // PDG_BOTTOM_KB
constexpr int kBottomDefaultLevels = 8;  // PDG_BOTTOM_LEVELS
// Bottom levels on? Default: where the sweep is bandwidth bound (>= 2M dofs
// per rank, the minimum-degree ordering) and b >= 6 (config 5 p=2, b = 6: 2.35 -> 2.22 ms
// with 128-thread CTAs and supernodes of <= 2 cells; profiles/r02aa).
// Smaller problems have idle CTAs and want every supernode on its own one.
// PDG_BOTTOM_KB overrides (0: off). Returns the subtree byte cap.
long long bottom_level_bytes(long long dofs_per_rank, int b);
struct LevelChunk {
  int dir = 0, level = 0, first_task = 0, n_task = 0;
  // counters (Problem::level_chunks[dir][slot], slot = group * levels + level): the one this
  // chunk adds to, and the one it waits for (dep_slot < 0: none)
  int slot = 0, gslot = 0, dep_dir = 0, dep_slot = -1;  // slot < 0: a global level (no group counter)
  std::int64_t src_off = 0;  // first panel double (F or H)
  int bytes = 0;
  int meta_off = 0, meta_n = 0, xneed = 0;
  int root_off = 0, n_root = 0;  // forward: chunk_roots, its supernodes with an individually scheduled parent
  int par_off = 0, n_par = 0;    // backward: chunk_parents, the distinct such parents
};

struct Problem {
  pdg_config cfg{};
  Mesh mesh;
  int p = 1, b = 3, q = 1, bq = 3;
  Partition sub, coarse;  // subdomain / coarse partitions (reference cell ids)
  bool two_level = false, has_precond = false;

  // internal order
  std::vector<int> perm, iperm;  // internal -> reference cell, inverse
  int cell_begin = 0, cell_end = 0;   // this rank's internal cell range
  std::vector<int> rank_cell_start;   // world+1

  // operators (local rows, global internal columns)
  Bsr K, A;                  // A kept only when keep_matrices
  std::vector<double> M;     // local diag mass blocks (b*b each, column-major)
  std::vector<double> Minv;  // inverses
  bool keep_matrices = true;

  // Schwarz local solves
  std::vector<TaskDesc> tasks;
  std::vector<int> task_child, fwd_order, bwd_order;
  std::vector<LevelChunk> chunks;  // forward chunks (levels bottom-up), then backward ones (top-down)
  std::vector<int> bmeta, chunk_roots, chunk_parents;
  int n_bottom_levels = 0, n_bottom_groups = 0, n_packed_units = 0;
  std::vector<int> level_chunks[2];  // chunks per (group, level) slot (forward, backward)
  // Row-tiled dense panels: tile t covers output rows [32k, 32k+rows) of its
  // task; element (row r0+l, input col0+j) at mat[off + j*stride + l]. The
  // panels themselves are formed on the device (cuda/panels.cu) from the
  // factor values in lval; the host only lays the tiles out.
  struct Tile {
    std::int64_t off;
    int ncol, col0, rows, stride;  // stride = rows rounded up to even
  };
  std::int64_t fmat_len = 0, hmat_len = 0;  // forward / backward panel doubles
  // Factor values, per task: inv(L_SS) packed lower, then L_RS (column-major),
  // at TaskDesc::linv_off / b_off of a device buffer of lval_len doubles.
  // Host-computed values cover [lval_host0, lval_len) (all tasks when the
  // host factors; only the coarse tasks when the device does, cuda/factor.cu).
  std::int64_t lval_len = 0, lval_host0 = 0;
  std::vector<double> lval;

  // Device factorisation plan of the fine supernodes (one per fine task, same
  // index): scratch panel P (H x w, column-major, ld H) at p_off, its unit's
  // first internal local cell and size, position range, below rows
  // (unit-relative positions) and the descendants that update it.
  struct FactorSn {
    std::int64_t p_off;
    int cell0, ucells, s0, s1, w, H, rows_off, nrows, upd_off, nupd, height, pad;
  };
  // One left-looking update of S by descendant d (a task id): D's below rows
  // [a, ce) are columns of S; rows [a, nrd) map to P_S row cells map[map_off + k - a].
  struct FactorUpd {
    int d, a, ce, nrd;
    std::int64_t map_off;
  };
  bool device_factor = false;
  std::vector<FactorSn> fsn;
  std::vector<int> frows, fmap;
  std::vector<FactorUpd> fupd;
  std::int64_t fp_len = 0;
  std::vector<Tile> ftiles, htiles;
  std::vector<std::int64_t> row_dof;  // below-row cell dof starts
  std::vector<int> in_ptr;       // incoming CSR (per supernode cell slot)
  std::vector<std::int64_t> in_idx;   // ubuf offsets
  std::int64_t ubuf_size = 0;
  int n_fine_tasks = 0;

  // coarse space: per local cell E block (b x bq, column-major) and coarse dof start
  std::vector<double> E;
  std::vector<int> cell_agg;            // local cell -> coarse internal node
  std::vector<int> agg_cell_ptr, agg_cells;  // coarse node -> local cells (for E^T r)
  int n_agg = 0;                        // coarse nodes
  std::vector<int> agg_order;           // coarse internal node -> coarse label
  NdTree coarse_nd;                     // coarse supernode tree (positions)
  Bsr K0;                               // coarse matrix in coarse internal order
  std::int64_t factor_values = 0;
  // structural nnz(L) (scalar, lower incl. diagonal) of this rank's local
  // factors and of the coarse factor, for the SURVEY §8(d) byte count
  std::int64_t l_struct = 0, l0_struct = 0;

  // ionic geometry per local cell: bbox (4) and fan triangles
  std::vector<double> bbox;
  std::vector<int> tri_ptr;
  std::vector<double> tri;   // 6 doubles per triangle
  std::vector<double> gl_x, gl_w;  // 1-D Gauss nodes for the volume rule

  // initial state (local, internal order)
  std::vector<double> U0;
  std::vector<double> Y0;    // n_comp fields
  int n_comp = 0;

  int n_cells_global = 0;
  bool from_operator = false;  // built from caller data (no mesh, no time stepper)

  // device assembly (cuda/assemble.cu): the host keeps the geometry only
  bool device_assembly = false;
  std::vector<double> sigma;             // 4 per internal cell: conductivity tensor
  std::vector<int> fptr, fent, fcell;    // per local cell its faces (2 f + side); per face (K, L)
  std::vector<double> fgeo;              // per face: mid, half direction, half length, normal, penalty
  std::vector<double> gs_x, gs_w;        // segment-rule Gauss nodes
  std::vector<double> abox;              // 4 per coarse label: agglomerate bounding box
  std::vector<int> cell_label;           // local cell -> coarse label
  double y_rest[4] = {0.0, 0.0, 0.0, 0.0};

  std::int64_t n_local_dofs() const { return static_cast<std::int64_t>(cell_end - cell_begin) * b; }
  std::int64_t n_global_dofs() const { return static_cast<std::int64_t>(n_cells_global) * b; }
};

// Appends the supernodes of one exact local factor (fine subdomain, coarse=0,
// or the coarse problem, coarse=1) as device tasks: panels, tiles, row maps,
// incoming update lists and the tree links (host/pack.cpp).
void pack_unit_tasks(Problem& pr, const SupernodalFactor& F, int coarse, std::int64_t dof_base);
// After the last fine pack_unit_tasks: level chunks of the bottom supernodes.
void finish_bottom_levels(Problem& pr);

// Multi-rank SpMV halo, identical on every rank:
// send[peer] = this rank's local cells adjacent to peer's cells (ascending),
// recv[peer] = peer's global internal cells this rank's rows touch (ascending).
void halo_plan(const Problem& pr, std::vector<std::vector<int>>& send, std::vector<std::vector<int>>& recv);

void validate_config(const pdg_config& cfg);
// IonicModel::state_dim / resting_potential / resting_state (ionics.hpp:25-31)
int ionic_rest(const pdg_config& cfg, double& u_rest, double* y_rest);
std::unique_ptr<Problem> build_problem(const pdg_config& cfg, bool device = false);
// Solver setup from a caller's K, subdomain partition and coarse embedding
// (pdg_sim_create_from_operator): one rank, graph-only orderings.
std::unique_ptr<Problem> build_problem_from_operator(const pdg_operator_desc& d);
// build_coarse_embedding (schwarz.cpp:13-77): per cell b x bq blocks of E for
// agglomerates `owner` (count) with degree-q bbox-Legendre coarse modes.
std::vector<double> coarse_embedding(const Mesh& mesh, int p, const std::vector<int>& owner, int count, int q);
// coarse factorisation + task packing; split out so a multi-rank run can sum
// K0 partials before factorising.
void finish_coarse(Problem& P);

}  // namespace pdg
