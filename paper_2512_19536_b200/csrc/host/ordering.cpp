#include "ordering.hpp"

#include <algorithm>
#include <cstdlib>
#include <set>

namespace pdg {

namespace {

std::vector<std::vector<int>> graph_of(int m, const std::vector<int>& ap, const std::vector<int>& aj) {
  std::vector<std::vector<int>> g(m);
  for (int v = 0; v < m; ++v) {
    for (int k = ap[v]; k < ap[v + 1]; ++k)
      if (aj[k] != v) g[v].push_back(aj[k]);
    std::sort(g[v].begin(), g[v].end());
    g[v].erase(std::unique(g[v].begin(), g[v].end()), g[v].end());
  }
  return g;
}

// elimination tree of the graph in positions (padj[i] = neighbour positions)
std::vector<int> etree(int m, const std::vector<std::vector<int>>& padj) {
  std::vector<int> parent(m, -1), anc(m, -1);
  for (int i = 0; i < m; ++i)
    for (int r : padj[i]) {
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
  return parent;
}

double relax_z() {
  static const double z = std::getenv("PDG_RELAX_Z") ? std::atof(std::getenv("PDG_RELAX_Z")) : 0.5;
  return z;
}

}  // namespace

std::vector<int> min_degree_order(int m, const std::vector<int>& adj_ptr, const std::vector<int>& adj) {
  auto g = graph_of(m, adj_ptr, adj);
  std::set<std::pair<int, int>> q;
  for (int v = 0; v < m; ++v) q.insert({static_cast<int>(g[v].size()), v});
  std::vector<int> order;
  order.reserve(m);
  std::vector<int> tmp;
  while (!q.empty()) {
    const int v = q.begin()->second;
    q.erase(q.begin());
    order.push_back(v);
    const std::vector<int> nb = std::move(g[v]);
    g[v].clear();
    // the neighbours of v become a clique
    for (int u : nb) {
      q.erase({static_cast<int>(g[u].size()), u});
      tmp.clear();
      std::set_union(g[u].begin(), g[u].end(), nb.begin(), nb.end(), std::back_inserter(tmp));
      tmp.erase(std::remove_if(tmp.begin(), tmp.end(), [&](int x) { return x == u || x == v; }), tmp.end());
      g[u].swap(tmp);
      q.insert({static_cast<int>(g[u].size()), u});
    }
  }
  return order;
}

NdTree etree_supernodes(int m, const std::vector<int>& adj_ptr, const std::vector<int>& adj,
                        const std::vector<int>& order_in, int relax) {
  NdTree out;
  if (m == 0) {
    out.sn_start.push_back(0);
    return out;
  }
  // ---- elimination tree of the given order, then a postorder of it ----
  std::vector<int> pos(m);
  for (int i = 0; i < m; ++i) pos[order_in[i]] = i;
  std::vector<std::vector<int>> padj(m);
  for (int i = 0; i < m; ++i) {
    const int v = order_in[i];
    for (int k = adj_ptr[v]; k < adj_ptr[v + 1]; ++k)
      if (adj[k] != v) padj[i].push_back(pos[adj[k]]);
  }
  std::vector<int> par0 = etree(m, padj);
  std::vector<std::vector<int>> kids(m);
  std::vector<int> roots;
  for (int i = 0; i < m; ++i) (par0[i] < 0 ? roots : kids[par0[i]]).push_back(i);
  std::vector<int> post;  // new position -> old position
  post.reserve(m);
  {
    std::vector<std::pair<int, int>> st;
    for (int r : roots) {
      st.push_back({r, 0});
      while (!st.empty()) {
        auto& [x, k] = st.back();
        if (k < static_cast<int>(kids[x].size())) {
          const int c = kids[x][k++];
          st.push_back({c, 0});
        } else {
          post.push_back(x);
          st.pop_back();
        }
      }
    }
  }
  std::vector<int> newpos(m), order(m);
  for (int k = 0; k < m; ++k) {
    newpos[post[k]] = k;
    order[k] = order_in[post[k]];
  }
  std::vector<int> parent(m, -1);
  for (int k = 0; k < m; ++k) parent[k] = par0[post[k]] < 0 ? -1 : newpos[par0[post[k]]];
  std::vector<std::vector<int>> nadj(m);
  for (int k = 0; k < m; ++k) {
    for (int j : padj[post[k]]) nadj[k].push_back(newpos[j]);
    std::sort(nadj[k].begin(), nadj[k].end());
  }
  // ---- column counts (row subtrees) ----
  std::vector<int> cc(m, 1), mark(m, -1), nchild(m, 0);
  for (int i = 0; i < m; ++i) {
    if (parent[i] >= 0) ++nchild[parent[i]];
    mark[i] = i;
    for (int j0 : nadj[i])
      for (int j = j0; j < i && mark[j] != i; j = parent[j]) {
        mark[j] = i;
        ++cc[j];
      }
  }
  // ---- fundamental supernodes ----
  std::vector<int> sn_of(m), s_start{0};
  for (int j = 0; j < m; ++j) {
    if (j > 0 && parent[j - 1] == j && cc[j - 1] == cc[j] + 1 && nchild[j] == 1) {
      sn_of[j] = static_cast<int>(s_start.size()) - 1;
      continue;
    }
    if (j > 0) s_start.push_back(j);
    sn_of[j] = static_cast<int>(s_start.size()) - 1;
  }
  const int ns = static_cast<int>(s_start.size());
  s_start.push_back(m);
  // ---- supernode rows, tree, structural entries ----
  struct Node {
    std::vector<int> cols;  // positions (topological inside)
    std::vector<int> rows;  // below rows (positions), sorted
    std::vector<int> kids;
    std::int64_t nz = 0;    // true structural entries (cells)
    int parent = -1;
    bool alive = true;
  };
  std::vector<Node> sn(ns);
  std::vector<int> smark(m, -1);
  for (int s = 0; s < ns; ++s) {
    Node& S = sn[s];
    const int a = s_start[s], e = s_start[s + 1];
    for (int p = a; p < e; ++p) S.cols.push_back(p);
    const int last = e - 1;
    S.parent = parent[last] < 0 ? -1 : sn_of[parent[last]];
    if (S.parent >= 0) sn[S.parent].kids.push_back(s);
    // rows = struct of the first column minus the supernode's own columns
    for (int p = a; p < e; ++p)
      for (int q : nadj[p])
        if (q >= e && smark[q] != s) {
          smark[q] = s;
          S.rows.push_back(q);
        }
  }
  for (int s = 0; s < ns; ++s) {
    Node& S = sn[s];
    const int e = s_start[s + 1];
    for (int c : S.kids)
      for (int q : sn[c].rows)
        if (q >= e && smark[q] != s) {
          smark[q] = s;
          S.rows.push_back(q);
        }
    std::sort(S.rows.begin(), S.rows.end());
    const std::int64_t w = static_cast<std::int64_t>(S.cols.size());
    S.nz = w * (w + 1) / 2 + w * static_cast<std::int64_t>(S.rows.size());
  }
  // ---- relaxed amalgamation (children merge into parents, bottom-up) ----
  auto stored = [](std::int64_t w, std::int64_t r) { return w * (w + 1) / 2 + w * r; };
  const double zr = relax_z();
  // PDG_RELAX_MIN_SUBTREE = T: a child is only merged when its subtree holds
  // at least T cells. The small bottom subtrees then keep their fundamental
  // supernodes (no explicit zeros; the sweep solves them in level chunks,
  // host/pack.cpp) while the supernodes above them are amalgamated as usual.
  static const int min_subtree = std::getenv("PDG_RELAX_MIN_SUBTREE") ? std::atoi(std::getenv("PDG_RELAX_MIN_SUBTREE")) : 0;
  std::vector<int> subtree_cells(ns, 0);
  for (int s = 0; s < ns; ++s) {
    subtree_cells[s] += static_cast<int>(sn[s].cols.size());
    if (sn[s].parent >= 0) subtree_cells[sn[s].parent] += subtree_cells[s];
  }
  for (int p = 0; p < ns; ++p) {
    Node& P = sn[p];
    if (P.kids.empty()) continue;
    std::vector<int> kids_sorted = P.kids;
    std::sort(kids_sorted.begin(), kids_sorted.end(), [&](int x, int y) {
      return sn[x].cols.size() < sn[y].cols.size() || (sn[x].cols.size() == sn[y].cols.size() && x < y);
    });
    std::vector<int> new_kids;
    for (int c : kids_sorted) {
      Node& Cn = sn[c];
      const std::int64_t w = static_cast<std::int64_t>(P.cols.size() + Cn.cols.size());
      const std::int64_t st = stored(w, static_cast<std::int64_t>(P.rows.size()));
      const double z = 1.0 - static_cast<double>(P.nz + Cn.nz) / static_cast<double>(st);
      const bool merge = ((w <= relax && z < zr) || z < 0.02) && subtree_cells[c] >= min_subtree;
      if (!merge) {
        new_kids.push_back(c);
        continue;
      }
      // child's columns go first (topological: they precede the parent's)
      std::vector<int> cols = Cn.cols;
      cols.insert(cols.end(), P.cols.begin(), P.cols.end());
      std::sort(cols.begin(), cols.end());
      P.cols.swap(cols);
      P.nz += Cn.nz;
      for (int g : Cn.kids) {
        sn[g].parent = p;
        new_kids.push_back(g);
      }
      Cn.alive = false;
    }
    P.kids.swap(new_kids);
  }
  // ---- emit in a postorder of the merged tree ----
  out.sn_start.push_back(0);
  std::vector<int> id(ns, -1);
  std::vector<int> sroots;
  for (int s = 0; s < ns; ++s)
    if (sn[s].alive && sn[s].parent < 0) sroots.push_back(s);
  for (auto& S : sn) std::sort(S.kids.begin(), S.kids.end());
  std::vector<std::pair<int, int>> st;
  for (int r : sroots) {
    st.push_back({r, 0});
    while (!st.empty()) {
      auto& [x, k] = st.back();
      if (k < static_cast<int>(sn[x].kids.size())) {
        const int c = sn[x].kids[k++];
        st.push_back({c, 0});
      } else {
        for (int p : sn[x].cols) out.order.push_back(order[p]);
        out.sn_start.push_back(static_cast<int>(out.order.size()));
        id[x] = static_cast<int>(out.parent.size());
        out.parent.push_back(-1);
        for (int c : sn[x].kids) out.parent[id[c]] = id[x];
        st.pop_back();
      }
    }
  }
  return out;
}

NdTree md_supernodes(int m, const std::vector<int>& adj_ptr, const std::vector<int>& adj, int relax) {
  return etree_supernodes(m, adj_ptr, adj, min_degree_order(m, adj_ptr, adj), relax);
}

NdTree hybrid_md_supernodes(int m, const std::vector<int>& adj_ptr, const std::vector<int>& adj, const NdTree& nd,
                            int relax) {
  const int ns = static_cast<int>(nd.parent.size());
  std::vector<char> has_child(ns, 0);
  for (int s = 0; s < ns; ++s)
    if (nd.parent[s] >= 0) has_child[nd.parent[s]] = 1;
  std::vector<int> order = nd.order;
  std::vector<int> loc(m, -1);
  for (int s = 0; s < ns; ++s) {
    if (has_child[s]) continue;
    const int a = nd.sn_start[s], e = nd.sn_start[s + 1], k = e - a;
    if (k <= 2) continue;
    for (int i = 0; i < k; ++i) loc[order[a + i]] = i;
    std::vector<int> ap{0}, aj;
    for (int i = 0; i < k; ++i) {
      const int v = order[a + i];
      for (int q = adj_ptr[v]; q < adj_ptr[v + 1]; ++q)
        if (loc[adj[q]] >= 0) aj.push_back(loc[adj[q]]);
      ap.push_back(static_cast<int>(aj.size()));
    }
    std::vector<int> o = min_degree_order(k, ap, aj);
    std::vector<int> nodes(order.begin() + a, order.begin() + e);
    for (int i = 0; i < k; ++i) order[a + i] = nodes[o[i]];
    for (int v : nodes) loc[v] = -1;
  }
  return etree_supernodes(m, adj_ptr, adj, order, relax);
}

SupernodeStorage supernode_storage(int m, const std::vector<int>& adj_ptr, const std::vector<int>& adj,
                                   const NdTree& t) {
  SupernodeStorage out;
  const int ns = static_cast<int>(t.parent.size());
  out.supernodes = ns;
  std::vector<int> pos(m);
  for (int i = 0; i < m; ++i) pos[t.order[i]] = i;
  std::vector<std::vector<int>> rows(ns), kids(ns);
  for (int s = 0; s < ns; ++s)
    if (t.parent[s] >= 0) kids[t.parent[s]].push_back(s);
  std::vector<int> mark(m, -1);
  for (int s = 0; s < ns; ++s) {
    const int a = t.sn_start[s], e = t.sn_start[s + 1];
    auto add = [&](int q) {
      if (q >= e && mark[q] != s) {
        mark[q] = s;
        rows[s].push_back(q);
      }
    };
    for (int p = a; p < e; ++p) {
      const int v = t.order[p];
      for (int k = adj_ptr[v]; k < adj_ptr[v + 1]; ++k) add(pos[adj[k]]);
    }
    for (int c : kids[s])
      for (int q : rows[c]) add(q);
    const std::int64_t w = e - a;
    out.blocks += w * (w + 1) / 2 + w * static_cast<std::int64_t>(rows[s].size());
  }
  return out;
}

}  // namespace pdg
