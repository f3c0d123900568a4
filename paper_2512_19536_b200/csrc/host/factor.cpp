#include "factor.hpp"

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <functional>
#include <string>

namespace pdg {

std::int64_t SupernodalFactor::values() const {
  std::int64_t n = 0;
  for (const auto& s : sn) n += static_cast<std::int64_t>(s.Linv.size() + s.B.size());
  return n;
}

namespace {

// Minimum vertex cover of the bipartite graph of edges between side 0 and
// side 1 (nodes of `ord`, side[] in {0,1}): maximum matching by augmenting
// paths (Kuhn, sides scanned in `ord` order, so deterministic), then Koenig's
// construction: Z = nodes reachable from unmatched side-0 nodes by
// alternating paths; cover = (side0 \ Z) u (side1 n Z). Returned in `ord` order.
std::vector<int> min_cut_cover(const std::vector<int>& ord, const std::vector<int>& side,
                               const std::vector<int>& ap, const std::vector<int>& aj, std::vector<int>& mate,
                               std::vector<int>& seen, std::vector<int>& par) {
  std::vector<int> L;
  for (int v : ord) {
    if (side[v] != 0) continue;
    for (int k = ap[v]; k < ap[v + 1]; ++k)
      if (side[aj[k]] == 1) {
        L.push_back(v);
        break;
      }
  }
  int stamp = 0;
  // BFS for an augmenting path from the free side-0 node u; par[w] = side-0
  // node that reached side-1 node w
  std::vector<int> q;
  auto augment = [&](int u) -> bool {
    ++stamp;
    q.assign(1, u);
    for (std::size_t h = 0; h < q.size(); ++h) {
      const int x = q[h];
      for (int k = ap[x]; k < ap[x + 1]; ++k) {
        int w = aj[k];
        if (side[w] != 1 || seen[w] == stamp) continue;
        seen[w] = stamp;
        par[w] = x;
        if (mate[w] < 0) {
          while (w >= 0) {  // flip the alternating path back to u
            const int y = par[w], next = mate[y];
            mate[y] = w;
            mate[w] = y;
            w = next;
          }
          return true;
        }
        q.push_back(mate[w]);
      }
    }
    return false;
  };
  for (int u : L) augment(u);
  // Koenig: alternating BFS from unmatched left nodes
  ++stamp;
  q.clear();
  std::vector<char> inZ;
  for (int u : L)
    if (mate[u] < 0) {
      q.push_back(u);
      seen[u] = stamp;
    }
  for (std::size_t h = 0; h < q.size(); ++h) {
    const int u = q[h];
    if (side[u] == 0) {
      for (int k = ap[u]; k < ap[u + 1]; ++k) {
        const int w = aj[k];
        if (side[w] == 1 && seen[w] != stamp && mate[u] != w) {
          seen[w] = stamp;
          q.push_back(w);
        }
      }
    } else if (mate[u] >= 0 && seen[mate[u]] != stamp) {
      seen[mate[u]] = stamp;
      q.push_back(mate[u]);
    }
  }
  std::vector<int> cover;
  for (int v : ord) {
    if (side[v] == 0) {
      if (mate[v] >= 0 && seen[v] != stamp) cover.push_back(v);
    } else if (side[v] == 1 && mate[v] >= 0 && seen[v] == stamp) {
      cover.push_back(v);
    }
  }
  for (int v : ord) mate[v] = seen[v] = -1;
  return cover;
}

}  // namespace

NdTree nested_dissection(int m, const std::vector<int>& adj_ptr, const std::vector<int>& adj,
                         const std::vector<Pt>& pos, int leaf, int merge, int top) {
  NdTree t;
  merge = std::max(1, merge);
  top = top > 0 ? top : merge;
  t.order.reserve(m);
  t.sn_start.push_back(0);
  std::vector<int> side(m, -1), mate(m, -1), seen(m, -1), par(m, -1);
  constexpr int n_dirs = 4;
  auto emit = [&](const std::vector<int>& nodes) {
    for (int v : nodes) t.order.push_back(v);
    t.sn_start.push_back(static_cast<int>(t.order.size()));
    t.parent.push_back(-1);
    return static_cast<int>(t.parent.size()) - 1;
  };
  // Separators of `merge` consecutive levels form one supernode (a level
  // whose depth % merge != 0 hands its separator up as `pending`): the
  // elimination tree gets `merge` times shallower, which shortens the
  // dependency chain of the triangular sweeps, at the price of storing the
  // (zero) couplings between the merged separators.
  std::function<void(std::vector<int>&, std::vector<int>&, std::vector<int>&, int)> rec =
      [&](std::vector<int>& nodes, std::vector<int>& roots, std::vector<int>& pending, int depth) {
        roots.clear();
        pending.clear();
        if (nodes.empty()) return;
        if (static_cast<int>(nodes.size()) <= leaf) {
          roots.push_back(emit(nodes));
          return;
        }
        // median cuts along 4 directions; keep the smallest one-sided separator
        const std::size_t half = nodes.size() / 2;
        std::vector<int> best_order, sep;
        bool have = false;
        static const double kDir[4][2] = {{1, 0}, {0, 1}, {0.7071067811865476, 0.7071067811865476},
                                          {0.7071067811865476, -0.7071067811865476}};
        for (int d = 0; d < n_dirs; ++d) {
          std::vector<int> ord = nodes;
          const double dx = kDir[d][0], dy = kDir[d][1];
          std::sort(ord.begin(), ord.end(), [&](int a, int b) {
            const double ca = pos[a].x * dx + pos[a].y * dy, cb = pos[b].x * dx + pos[b].y * dy;
            return ca < cb || (ca == cb && a < b);
          });
          for (std::size_t i = 0; i < ord.size(); ++i) side[ord[i]] = i < half ? 0 : 1;
          std::vector<int> sep_l, sep_r;
          for (std::size_t i = 0; i < ord.size(); ++i) {
            const int v = ord[i];
            const int sv = side[v];
            for (int k = adj_ptr[v]; k < adj_ptr[v + 1]; ++k) {
              const int u = adj[k];
              if (side[u] >= 0 && side[u] != sv) {
                (sv == 0 ? sep_l : sep_r).push_back(v);
                break;
              }
            }
          }
          {
            // minimum vertex cover of the cut edges (Koenig): the smallest
            // separator whose removal disconnects the two halves
            std::vector<int> cover = min_cut_cover(ord, side, adj_ptr, adj, mate, seen, par);
            if (cover.size() < sep_l.size() && cover.size() < sep_r.size()) sep_l = std::move(cover);
          }
          for (int v : ord) side[v] = -1;
          std::vector<int>& s = sep_r.size() < sep_l.size() ? sep_r : sep_l;
          if (!have || s.size() < sep.size()) {
            have = true;
            sep = s;
            best_order = std::move(ord);
          }
        }
        nodes = std::move(best_order);
        if (2 * sep.size() > nodes.size()) {
          roots.push_back(emit(nodes));
          return;
        }
        for (int v : sep) side[v] = 2;
        std::vector<int> left, right;
        for (std::size_t i = 0; i < nodes.size(); ++i) {
          const int v = nodes[i];
          if (side[v] == 2) continue;
          (i < half ? left : right).push_back(v);
        }
        for (int v : sep) side[v] = -1;
        std::vector<int> rl, rr, pl, pr;
        rec(left, rl, pl, depth + 1);
        rec(right, rr, pr, depth + 1);
        std::vector<int> sep_nodes = pl;
        sep_nodes.insert(sep_nodes.end(), pr.begin(), pr.end());
        sep_nodes.insert(sep_nodes.end(), sep.begin(), sep.end());
        roots = rl;
        roots.insert(roots.end(), rr.begin(), rr.end());
        // defer: the ancestor level emits it (the top `top` levels form the
        // root supernode, below that every `merge` levels form one)
        if (depth < top ? depth != 0 : (depth - top) % merge != 0) {
          pending = sep_nodes;
          return;
        }
        if (sep_nodes.empty()) return;
        const int id = emit(sep_nodes);
        for (int c : roots) t.parent[c] = id;
        roots.assign(1, id);
      };
  std::vector<int> all(m);
  for (int i = 0; i < m; ++i) all[i] = i;
  std::vector<int> roots, pending;
  rec(all, roots, pending, 0);
  if (!pending.empty()) {
    const int id = emit(pending);
    for (int c : roots) t.parent[c] = id;
  }
  return t;
}

BlockMatrix permute(const BlockMatrix& A, const std::vector<int>& order) {
  const int m = A.m, bs2 = A.bs * A.bs;
  std::vector<int> inv(m);
  for (int i = 0; i < m; ++i) inv[order[i]] = i;
  BlockMatrix P;
  P.m = m;
  P.bs = A.bs;
  P.ptr.assign(m + 1, 0);
  for (int i = 0; i < m; ++i) P.ptr[i + 1] = P.ptr[i] + (A.ptr[order[i] + 1] - A.ptr[order[i]]);
  P.col.resize(A.col.size());
  P.val.resize(A.val.size());
  std::vector<std::pair<int, int>> row;
  for (int i = 0; i < m; ++i) {
    const int o = order[i];
    row.clear();
    for (int k = A.ptr[o]; k < A.ptr[o + 1]; ++k) row.emplace_back(inv[A.col[k]], k);
    std::sort(row.begin(), row.end());
    int dst = P.ptr[i];
    for (const auto& [c, k] : row) {
      P.col[dst] = c;
      std::copy(A.val.begin() + static_cast<std::size_t>(k) * bs2,
                A.val.begin() + static_cast<std::size_t>(k + 1) * bs2,
                P.val.begin() + static_cast<std::size_t>(dst) * bs2);
      ++dst;
    }
  }
  return P;
}

SupernodalFactor symbolic_factor(const BlockMatrix& A, const NdTree& nd, std::vector<std::vector<int>>& upd) {
  const int m = A.m, bs = A.bs;
  const int nsn = static_cast<int>(nd.sn_start.size()) - 1;
  SupernodalFactor F;
  F.m = m;
  F.bs = bs;
  F.sn.resize(nsn);
  F.sn_of.resize(m);
  std::vector<std::vector<int>> children(nsn);
  for (int s = 0; s < nsn; ++s) {
    F.sn[s].s0 = nd.sn_start[s];
    F.sn[s].s1 = nd.sn_start[s + 1];
    F.sn[s].parent = nd.parent[s];
    for (int p = F.sn[s].s0; p < F.sn[s].s1; ++p) F.sn_of[p] = s;
    if (nd.parent[s] >= 0) children[nd.parent[s]].push_back(s);
  }
  // symbolic: rows(S) = (adj(S) u rows(children)) restricted to positions >= s1
  std::vector<int> mark(m, -1);
  for (int s = 0; s < nsn; ++s) {
    Supernode& S = F.sn[s];
    auto add = [&](int q) {
      if (q >= S.s1 && mark[q] != s) {
        mark[q] = s;
        S.rows.push_back(q);
      }
    };
    for (int p = S.s0; p < S.s1; ++p)
      for (int k = A.ptr[p]; k < A.ptr[p + 1]; ++k) add(A.col[k]);
    for (int c : children[s])
      for (int q : F.sn[c].rows) add(q);
    std::sort(S.rows.begin(), S.rows.end());
  }
  // updaters of S: descendants D whose rows touch S (ascending D)
  upd.assign(nsn, {});
  std::vector<int> last(nsn, -1);
  for (int d = 0; d < nsn; ++d)
    for (int q : F.sn[d].rows) {
      const int s = F.sn_of[q];
      if (last[s] != d) {
        last[s] = d;
        upd[s].push_back(d);
      }
    }
  return F;
}

SupernodalFactor supernodal_cholesky(const BlockMatrix& A, const NdTree& nd) {
  const int m = A.m, bs = A.bs;
  const int nsn = static_cast<int>(nd.sn_start.size()) - 1;
  std::vector<std::vector<int>> upd;
  SupernodalFactor F = symbolic_factor(A, nd, upd);

  std::vector<int> rowcell(m, -1);
  std::vector<double> P, x;
  for (int s = 0; s < nsn; ++s) {
    Supernode& S = F.sn[s];
    const int nc = S.s1 - S.s0, w = nc * bs, r = static_cast<int>(S.rows.size());
    const int H = w + r * bs;
    P.assign(static_cast<std::size_t>(H) * w, 0.0);
    for (int p = S.s0; p < S.s1; ++p) rowcell[p] = p - S.s0;
    for (int k = 0; k < r; ++k) rowcell[S.rows[k]] = nc + k;
    auto at = [&](int row, int col) -> double& { return P[static_cast<std::size_t>(col) * H + row]; };
    // original entries (lower part): A_ij for i >= j, j in S
    for (int j = S.s0; j < S.s1; ++j) {
      const int jc = j - S.s0;
      for (int k = A.ptr[j]; k < A.ptr[j + 1]; ++k) {
        const int i = A.col[k];
        if (i < j) continue;
        const int rc = rowcell[i];
        const double* blk = A.block(k);  // A_{j,i}, column-major
        for (int c = 0; c < bs; ++c)
          for (int rr = 0; rr < bs; ++rr) at(rc * bs + rr, jc * bs + c) = blk[rr * bs + c];
      }
    }
    // left-looking updates from descendants
    for (int d : upd[s]) {
      const Supernode& D = F.sn[d];
      const int wD = D.w(bs), nrD = static_cast<int>(D.rows.size());
      const int ld = nrD * bs;
      const int a = static_cast<int>(std::lower_bound(D.rows.begin(), D.rows.end(), S.s0) - D.rows.begin());
      const int ce = static_cast<int>(std::lower_bound(D.rows.begin(), D.rows.end(), S.s1) - D.rows.begin());
      for (int l = a; l < ce; ++l) {
        const int colcell = rowcell[D.rows[l]];
        for (int cc = 0; cc < bs; ++cc) {
          const int colP = colcell * bs + cc;
          double* pcol = P.data() + static_cast<std::size_t>(colP) * H;
          for (int t = 0; t < wD; ++t) {
            const double* bcol = D.B.data() + static_cast<std::size_t>(t) * ld;
            const double coef = bcol[l * bs + cc];
            if (coef == 0.0) continue;
            for (int k = l; k < nrD; ++k) {
              const int rb = rowcell[D.rows[k]] * bs;
              const double* src = bcol + k * bs;
              for (int rr = 0; rr < bs; ++rr) pcol[rb + rr] -= src[rr] * coef;
            }
          }
        }
      }
    }
    // right-looking Cholesky of the diagonal block, with the below rows solved in the same sweep
    for (int j = 0; j < w; ++j) {
      double* cj = P.data() + static_cast<std::size_t>(j) * H;
      double d = cj[j];
      if (!(d > 0.0) || !std::isfinite(d))
        throw SolverError("factorization failed (not positive definite)");
      d = std::sqrt(d);
      cj[j] = d;
      const double inv = 1.0 / d;
      for (int i = j + 1; i < H; ++i) cj[i] *= inv;
      for (int k = j + 1; k < w; ++k) {
        const double lkj = cj[k];
        if (lkj == 0.0) continue;
        double* ck = P.data() + static_cast<std::size_t>(k) * H;
        for (int i = k; i < H; ++i) ck[i] -= cj[i] * lkj;
      }
    }
    // inv(L_SS), packed column-major lower
    S.Linv.assign(static_cast<std::size_t>(w) * (w + 1) / 2, 0.0);
    x.resize(w);
    std::size_t off = 0;
    for (int j = 0; j < w; ++j) {
      std::fill(x.begin(), x.end(), 0.0);
      x[j] = 1.0;
      for (int k = j; k < w; ++k) {
        const double* ck = P.data() + static_cast<std::size_t>(k) * H;
        x[k] /= ck[k];
        const double xk = x[k];
        if (xk == 0.0) continue;
        for (int i = k + 1; i < w; ++i) x[i] -= ck[i] * xk;
      }
      for (int i = j; i < w; ++i) S.Linv[off++] = x[i];
    }
    S.B.resize(static_cast<std::size_t>(r) * bs * w);
    for (int j = 0; j < w; ++j)
      std::copy(P.begin() + static_cast<std::size_t>(j) * H + w, P.begin() + static_cast<std::size_t>(j + 1) * H,
                S.B.begin() + static_cast<std::size_t>(j) * r * bs);
    for (int p = S.s0; p < S.s1; ++p) rowcell[p] = -1;
    for (int q : S.rows) rowcell[q] = -1;
  }
  return F;
}

FillCount structural_fill(int m, const std::vector<int>& adj_ptr, const std::vector<int>& adj,
                          const std::vector<int>& order) {
  std::vector<int> pos(m);
  for (int i = 0; i < m; ++i) pos[order[i]] = i;
  std::vector<int> parent(m, -1), anc(m, -1), mark(m, -1);
  // elimination tree with path-compressed ancestors
  for (int i = 0; i < m; ++i) {
    const int node = order[i];
    for (int k = adj_ptr[node]; k < adj_ptr[node + 1]; ++k) {
      int r = pos[adj[k]];
      if (r >= i) continue;
      while (anc[r] != -1 && anc[r] != i) {
        const int t = anc[r];
        anc[r] = i;
        r = t;
      }
      if (anc[r] == -1) {
        anc[r] = i;
        parent[r] = i;
      }
    }
  }
  FillCount f;
  f.diag = m;
  // row i of L: the union of the etree paths from its lower neighbours up to i
  for (int i = 0; i < m; ++i) {
    mark[i] = i;
    const int node = order[i];
    for (int k = adj_ptr[node]; k < adj_ptr[node + 1]; ++k) {
      for (int j = pos[adj[k]]; j < i && mark[j] != i; j = parent[j]) {
        mark[j] = i;
        ++f.offdiag;
      }
    }
  }
  return f;
}

}  // namespace pdg
