// Fill study for the Schwarz local factors (development tool, not product):
// structural nnz(L) and stored supernodal bytes of several orderings on a
// sample of the subdomains of a seeded mesh.
//   g++ -O2 -std=c++20 -I paper_2512_19536_b200/csrc/host scripts/fill_study.cpp build/csrc/host/*.o -lpthread
//   ./a.out N S sample_every
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <numeric>

#include "factor.hpp"
#include "mesh.hpp"
#include "ordering.hpp"

using namespace pdg;

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 1048576;
  const int S = argc > 2 ? atoi(argv[2]) : 512;
  const int every = argc > 3 ? atoi(argv[3]) : 16;
  const int bs = argc > 4 ? atoi(argv[4]) : 10;
  auto t0 = std::chrono::steady_clock::now();
  Mesh mesh = assign_regions(generate_mesh(N, Box{0, 0, 1, 1}, 42, 5), 0.5);
  Partition part = agglomerate(mesh, S);
  auto t1 = std::chrono::steady_clock::now();
  fprintf(stderr, "mesh+partition %.1f s\n", std::chrono::duration<double>(t1 - t0).count());
  std::vector<std::vector<int>> nbr(mesh.n_cells());
  for (const Face& f : mesh.interior_faces()) {
    nbr[f.cell_in].push_back(f.cell_out);
    nbr[f.cell_out].push_back(f.cell_in);
  }
  auto members = part.members();
  struct Acc {
    double cells = 0, structural = 0, stored = 0, nsn = 0, height = 0, n = 0;
    double panel[4] = {0, 0, 0, 0};  // panel doubles (fwd + bwd): align 8 / align 2 / tri16+align8 / tri16+align2
    double bundled_bytes = 0, bundled_tasks = 0, bundles = 0, free_tasks = 0, leaves = 0, leaf_bytes = 0, all_bytes = 0;
  };
  std::map<std::string, Acc> acc;
  for (int u = 0; u < part.count; u += every) {
    const auto& cells = members[u];
    const int m = static_cast<int>(cells.size());
    std::map<int, int> loc;
    for (int i = 0; i < m; ++i) loc[cells[i]] = i;
    std::vector<int> ap{0}, aj;
    std::vector<Pt> pos(m);
    for (int i = 0; i < m; ++i) {
      for (int nb : nbr[cells[i]]) {
        auto it = loc.find(nb);
        if (it != loc.end()) aj.push_back(it->second);
      }
      ap.push_back(static_cast<int>(aj.size()));
      pos[i] = mesh.centroid(cells[i]);
    }
    auto add = [&](const std::string& name, const NdTree& t) {
      FillCount f = structural_fill(m, ap, aj, t.order);
      auto st = supernode_storage(m, ap, aj, t);
      Acc& a = acc[name];
      a.cells += m;
      a.structural += f.offdiag + f.diag;
      a.stored += st.blocks;
      a.nsn += st.supernodes;
      // panel layout of host/pack.cpp: 32-row tiles, staircase triangle, rows padded
      {
        std::vector<int> pos(m);
        for (int i = 0; i < m; ++i) pos[t.order[i]] = i;
        const int ns = static_cast<int>(t.parent.size());
        std::vector<std::vector<int>> rows(ns), kids(ns);
        for (int q = 0; q < ns; ++q)
          if (t.parent[q] >= 0) kids[t.parent[q]].push_back(q);
        std::vector<int> mark(m, -1);
        std::vector<double> fbytes_of(ns, 0.0);
        for (int q = 0; q < ns; ++q) {
          const int a0 = t.sn_start[q], e = t.sn_start[q + 1];
          auto addr = [&](int r) { if (r >= e && mark[r] != q) { mark[r] = q; rows[q].push_back(r); } };
          for (int pp = a0; pp < e; ++pp) { const int v = t.order[pp]; for (int k = ap[v]; k < ap[v + 1]; ++k) addr(pos[aj[k]]); }
          for (int c : kids[q]) for (int r : rows[c]) addr(r);
          const long w = (long)(e - a0) * bs, h = w + (long)rows[q].size() * bs;
          for (int var = 0; var < 4; ++var) {
            const int al = (var & 1) ? 2 : 8, trit = (var & 2) ? 16 : 32;
            auto seg = [&](long r) { return (r + al - 1) / al * al; };
            double tot = 0;
            // forward: triangle rows [0, w) in trit-row tiles, below rows in 32-row tiles
            for (long r0 = 0; r0 < w; r0 += trit) { long rr = std::min<long>(trit, w - r0); tot += (double)std::min(w, r0 + rr) * seg(rr); }
            for (long r0 = w; r0 < h; r0 += 32) { long rr = std::min<long>(32, h - r0); tot += (double)w * seg(rr); }
            // backward: rows of H = columns of F, inputs i >= r0
            for (long r0 = 0; r0 < w; r0 += trit) { long rr = std::min<long>(trit, w - r0); tot += (double)(h - r0) * seg(rr); }
            a.panel[var] += tot;
            if (var == 1) fbytes_of[q] = tot * 8 / 2;  // ~forward half
          }
        }
        // bundles: maximal complete subtrees (non-root) with <= 64 KB of forward
        // panel, siblings grouped while the group stays <= 64 KB
        std::vector<double> sub(ns, 0.0);
        for (int q = 0; q < ns; ++q) {
          sub[q] += fbytes_of[q];
          if (t.parent[q] >= 0) sub[t.parent[q]] += sub[q];
        }
        const double Bmax = 65536;
        std::vector<char> in_bundle(ns, 0);
        for (int q = 0; q < ns; ++q) {
          // children of q that are small complete subtrees, grouped greedily
          double acc = 0; int cnt = 0;
          for (int c : kids[q]) {
            if (sub[c] > Bmax) continue;
            if (acc + sub[c] > Bmax && cnt > 0) { a.bundles += 1; acc = 0; cnt = 0; }
            acc += sub[c]; ++cnt;
          }
          if (cnt > 0) a.bundles += 1;
        }
        for (int q = 0; q < ns; ++q) {
          const int pp = t.parent[q];
          if (pp >= 0 && sub[q] <= Bmax) in_bundle[q] = 1;
        }
        // a task is bundled if it or an ancestor (below a big node) is a small subtree root
        for (int q = ns - 1; q >= 0; --q) {
          const int pp = t.parent[q];
          if (pp >= 0 && in_bundle[pp]) in_bundle[q] = 1;
        }
        for (int q = 0; q < ns; ++q) (in_bundle[q] ? a.bundled_tasks : a.free_tasks) += 1;
        for (int q = 0; q < ns; ++q) if (in_bundle[q]) a.bundled_bytes += fbytes_of[q];
        for (int q = 0; q < ns; ++q) {
          a.all_bytes += fbytes_of[q];
          if (kids[q].empty()) { a.leaves += 1; a.leaf_bytes += fbytes_of[q]; }
        }
      }
      std::vector<int> h(t.parent.size(), 1);
      int hmax = 0;
      for (size_t s = 0; s < t.parent.size(); ++s) {
        hmax = std::max(hmax, h[s]);
        if (t.parent[s] >= 0) h[t.parent[s]] = std::max(h[t.parent[s]], h[s] + 1);
      }
      a.height += hmax;
      a.n += 1;
    };
    add("nd_leaf6", nested_dissection(m, ap, aj, pos, 6, 1, 1));
    for (int relax : {1, 2, 4, 8}) add("md relax" + std::to_string(relax), md_supernodes(m, ap, aj, relax));
  }
  for (auto& [k, a] : acc)
    printf("%-28s tasks %.0f leaves %.0f (%.0f%% of fwd bytes) per subdomain\n", k.c_str(),
           (a.bundled_tasks + a.free_tasks) / a.n, a.leaves / a.n, 100.0 * a.leaf_bytes / a.all_bytes);
  for (auto& [k, a] : acc)
    printf("%-28s bundles %.0f holding %.0f tasks (%.0f%% of fwd bytes), free tasks %.0f per subdomain\n", k.c_str(),
           a.bundles / a.n, a.bundled_tasks / a.n, 100.0 * a.bundled_bytes / a.all_bytes, a.free_tasks / a.n);
  for (auto& [k, a] : acc)
    printf("%-28s panel/cell (fwd+bwd doubles): a8 %.0f a2 %.0f tri16a8 %.0f tri16a2 %.0f | 2x structural %.0f\n", k.c_str(),
           a.panel[0] / a.cells, a.panel[1] / a.cells, a.panel[2] / a.cells, a.panel[3] / a.cells,
           2 * (a.structural * bs * bs - a.cells * bs * (bs - 1) / 2.0) / a.cells);
  for (auto& [k, a] : acc)
    printf("%-28s structural %.2f blocks/cell  stored %.2f blocks/cell (x%.3f)  cells/supernode %.1f height %.0f\n", k.c_str(),
           a.structural / a.cells, a.stored / a.cells, a.stored / a.structural, a.cells / a.nsn, a.height / a.n);
}
