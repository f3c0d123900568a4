// Exact local solvers for the Schwarz preconditioner: geometric nested
// dissection + block supernodal Cholesky, packed for the device sweep.
//
// Replaces the reference's per-subdomain Eigen::LLT / SimplicialLLT factors
// (/root/reference/proj/src/schwarz.cpp:99-146) and the coarse SimplicialLLT
// (:138-146). Any exact factorisation satisfies the preconditioner contract
// z_i = K_i^{-1} r_i (P9); the ordering here is chosen for the GPU: every
// nested-dissection separator and leaf is a dense supernode, and the device
// stores inv(L_SS) so each supernode's triangular solve is one parallel
// triangular mat-vec instead of a w-step dependency chain.
#pragma once

#include <cstdint>
#include <vector>

#include "core.hpp"

namespace pdg {

// Symmetric block matrix over m nodes with bs x bs blocks (column-major
// blocks, both triangles stored, diagonal present).
struct BlockMatrix {
  int m = 0, bs = 0;
  std::vector<int> ptr, col;
  std::vector<double> val;
  const double* block(int k) const { return val.data() + static_cast<std::size_t>(k) * bs * bs; }
};

struct NdTree {
  std::vector<int> order;     // position -> node
  std::vector<int> sn_start;  // supernode s covers positions [sn_start[s], sn_start[s+1])
  std::vector<int> parent;    // supernode parent, -1 for roots (postorder: parent > child)
};

// Recursive coordinate bisection; separators are the smaller one-sided
// boundary of the cut. Deterministic (ties broken by node id). `merge`
// consecutive separator levels form one supernode.
// consecutive separator levels form one supernode; the root supernode takes
// the top `top` levels (0: same as merge).
NdTree nested_dissection(int m, const std::vector<int>& adj_ptr, const std::vector<int>& adj,
                         const std::vector<Pt>& pos, int leaf_nodes, int merge = 1, int top = 0);

struct Supernode {
  int s0 = 0, s1 = 0;         // positions
  int parent = -1;
  std::vector<int> rows;      // below-diagonal row nodes (positions, ascending)
  std::vector<double> Linv;   // inv(L_SS), packed column-major lower (w(w+1)/2)
  std::vector<double> B;      // L_{R,S}, column-major (rows.size()*bs x w)
  int w(int bs) const { return (s1 - s0) * bs; }
};

struct SupernodalFactor {
  int m = 0, bs = 0;
  std::vector<Supernode> sn;
  std::vector<int> sn_of;     // position -> supernode
  std::int64_t values() const;
};

// A must already be in position order (node i of A == position i).
// Throws SolverError("... not positive definite") on a non-positive pivot.
SupernodalFactor supernodal_cholesky(const BlockMatrix& A, const NdTree& nd);

// The symbolic half: supernode ranges, below rows and, per supernode, the
// descendants whose rows touch it (ascending; the left-looking update order).
// No values (A.val may be empty); Linv and B stay empty.
SupernodalFactor symbolic_factor(const BlockMatrix& A, const NdTree& nd, std::vector<std::vector<int>>& upd);

// Structural blocks of the Cholesky factor of a graph (adjacency without
// self loops) eliminated in `order` (position -> node): diagonal blocks plus
// the strictly lower nonzero blocks, by elimination tree + row subtrees
// (Liu). The SURVEY §8(d) byte count uses nnz(L) = offdiag*bs^2 + m*bs(bs+1)/2.
struct FillCount {
  std::int64_t diag = 0, offdiag = 0;
  std::int64_t scalar(int bs) const {
    return offdiag * bs * bs + diag * static_cast<std::int64_t>(bs) * (bs + 1) / 2;
  }
};
FillCount structural_fill(int m, const std::vector<int>& adj_ptr, const std::vector<int>& adj,
                          const std::vector<int>& order);

// Permutes a block matrix: out node i = in node order[i].
BlockMatrix permute(const BlockMatrix& A, const std::vector<int>& order);

}  // namespace pdg
