// Fill-reducing orderings and supernode partitions for the Schwarz local
// factors (the reference factors each subdomain with Eigen's SimplicialLLT
// under an AMD ordering, /root/reference/proj/src/schwarz.cpp:128-129).
//
// Any ordering gives the same exact local solve z_i = K_i^{-1} r_i (P9); the
// choice only moves bytes: the sweep streams every stored supernode panel
// twice per PCG iteration, so the bytes are 2 x 8 x (stored entries).
//   * min_degree_order: exact minimum degree on the explicit elimination graph
//     (ties by lowest node id; the subdomains hold <= ~4K cells);
//   * etree_supernodes: elimination tree of an ordering, postordered,
//     fundamental supernodes, then relaxed amalgamation (merge a child into
//     its parent while the merged dense panel adds few explicit zeros), so the
//     sweep gets supernodes of >= `relax` cells where it costs little.
#pragma once

#include <cstdint>
#include <vector>

#include "factor.hpp"

namespace pdg {

std::vector<int> min_degree_order(int m, const std::vector<int>& adj_ptr, const std::vector<int>& adj);

// Supernode partition (postordered, parent > child) of the elimination of the
// graph in `order` (position -> node). Relaxed amalgamation: a child merges
// into its parent when the merged supernode has <= relax cells, or when the
// explicit zeros it adds stay under a size-dependent fraction of its entries.
NdTree etree_supernodes(int m, const std::vector<int>& adj_ptr, const std::vector<int>& adj,
                        const std::vector<int>& order, int relax);

NdTree md_supernodes(int m, const std::vector<int>& adj_ptr, const std::vector<int>& adj, int relax);

// Nested-dissection separators on top, minimum degree inside every leaf of
// `nd`, then etree_supernodes on the combined order.
NdTree hybrid_md_supernodes(int m, const std::vector<int>& adj_ptr, const std::vector<int>& adj, const NdTree& nd,
                            int relax);

// Stored element blocks of a supernode partition: sum over supernodes of the
// dense lower triangle w(w+1)/2 plus w x |below rows| (cells).
struct SupernodeStorage {
  std::int64_t blocks = 0;
  int supernodes = 0;
};
SupernodeStorage supernode_storage(int m, const std::vector<int>& adj_ptr, const std::vector<int>& adj,
                                   const NdTree& t);

}  // namespace pdg
