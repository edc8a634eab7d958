// Hierarchical cell reordering (host C++), the paper's locality optimisation
// (no reference implementation exists).
// Deterministic algorithm, bit-exact
// with the oracle restatement oracle/ref_reorder.py:
//   order(G): |G| <= 512 -> cuthill_mckee(G); else groups = bfs_groups(G),
//             C = coarsen(G, groups), concat(groups[c] for c in order(C)).
#include <algorithm>
#include <climits>
#include <cstdint>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/tetmf_b200.h"

namespace {

struct Graph {  // CSR, neighbours ascending, integer edge weights
  std::vector<int64_t> ptr;
  std::vector<int64_t> nbr;
  std::vector<int64_t> w;
  int64_t n() const { return (int64_t)ptr.size() - 1; }
};

Graph from_edges(int64_t n, std::vector<std::pair<int64_t, int64_t>>& e, const std::vector<int64_t>* ew) {
  // e: directed edges (both directions present); merge duplicates summing weights
  std::vector<int64_t> idx(e.size());
  std::iota(idx.begin(), idx.end(), 0);
  std::sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return e[a] < e[b]; });
  Graph g;
  g.ptr.assign(n + 1, 0);
  for (size_t k = 0; k < idx.size();) {
    size_t j = k;
    int64_t wsum = 0;
    while (j < idx.size() && e[idx[j]] == e[idx[k]]) {
      wsum += ew ? (*ew)[idx[j]] : 1;
      ++j;
    }
    g.nbr.push_back(e[idx[k]].second);
    g.w.push_back(wsum);
    g.ptr[e[idx[k]].first + 1]++;
    k = j;
  }
  for (int64_t i = 0; i < n; ++i) g.ptr[i + 1] += g.ptr[i];
  return g;
}

std::vector<int64_t> by_degree(const Graph& g) {
  std::vector<int64_t> s(g.n());
  std::iota(s.begin(), s.end(), 0);
  std::stable_sort(s.begin(), s.end(), [&](int64_t a, int64_t b) {
    return (g.ptr[a + 1] - g.ptr[a]) < (g.ptr[b + 1] - g.ptr[b]);
  });
  return s;
}

std::vector<std::vector<int64_t>> bfs_groups(const Graph& g, int gs) {
  const int64_t n = g.n();
  std::vector<char> vis(n, 0);
  std::vector<std::vector<int64_t>> groups;
  std::vector<int64_t> queue;
  const std::vector<int64_t> seeds = by_degree(g);
  size_t si = 0;
  const std::vector<int64_t>* last = nullptr;
  while (true) {
    int64_t seed = -1;
    if (last) {  // continue next to the previous group: fewest free neighbours, then lowest id
      int64_t best_free = INT64_MAX;
      for (int64_t v : *last)
        for (int64_t k = g.ptr[v]; k < g.ptr[v + 1]; ++k) {
          const int64_t u = g.nbr[k];
          if (vis[u]) continue;
          int64_t free = 0;
          for (int64_t m = g.ptr[u]; m < g.ptr[u + 1]; ++m) free += vis[g.nbr[m]] ? 0 : 1;
          if (free < best_free || (free == best_free && u < seed)) {
            best_free = free;
            seed = u;
          }
        }
    }
    if (seed < 0) {
      while (si < seeds.size() && vis[seeds[si]]) ++si;
      if (si == seeds.size()) break;
      seed = seeds[si];
    }
    vis[seed] = 1;
    std::vector<int64_t> grp{seed};
    queue.assign(1, seed);
    size_t head = 0;
    while (head < queue.size() && (int)grp.size() < gs) {
      const int64_t v = queue[head++];
      for (int64_t k = g.ptr[v]; k < g.ptr[v + 1] && (int)grp.size() < gs; ++k) {
        const int64_t u = g.nbr[k];
        if (!vis[u]) {
          vis[u] = 1;
          grp.push_back(u);
          queue.push_back(u);
        }
      }
    }
    groups.push_back(std::move(grp));
    last = &groups.back();
  }
  return groups;
}

Graph coarsen(const Graph& g, const std::vector<std::vector<int64_t>>& groups) {
  std::vector<int64_t> gid(g.n());
  for (size_t k = 0; k < groups.size(); ++k)
    for (int64_t v : groups[k]) gid[v] = (int64_t)k;
  std::vector<std::pair<int64_t, int64_t>> e;
  std::vector<int64_t> w;
  for (int64_t v = 0; v < g.n(); ++v)
    for (int64_t k = g.ptr[v]; k < g.ptr[v + 1]; ++k)
      if (gid[g.nbr[k]] != gid[v]) {
        e.emplace_back(gid[v], gid[g.nbr[k]]);
        w.push_back(g.w[k]);
      }
  return from_edges((int64_t)groups.size(), e, &w);
}

// Cuthill-McKee level structure (the top of the hierarchy): BFS from the lowest-degree
// node, neighbours appended by (degree, id); restart per component.
std::vector<int64_t> cuthill_mckee(const Graph& g) {
  const int64_t n = g.n();
  std::vector<char> seen(n, 0);
  const std::vector<int64_t> seeds = by_degree(g);
  std::vector<int64_t> out;
  out.reserve(n);
  size_t si = 0;
  std::vector<int64_t> nb;
  while ((int64_t)out.size() < n) {
    while (seen[seeds[si]]) ++si;
    const int64_t s = seeds[si];
    seen[s] = 1;
    size_t head = out.size();
    out.push_back(s);
    while (head < out.size()) {
      const int64_t v = out[head++];
      nb.assign(g.nbr.begin() + g.ptr[v], g.nbr.begin() + g.ptr[v + 1]);
      std::sort(nb.begin(), nb.end(), [&](int64_t a, int64_t b) {
        const int64_t da = g.ptr[a + 1] - g.ptr[a], db = g.ptr[b + 1] - g.ptr[b];
        return da != db ? da < db : a < b;
      });
      for (int64_t u : nb)
        if (!seen[u]) {
          seen[u] = 1;
          out.push_back(u);
        }
    }
  }
  return out;
}

std::vector<int64_t> order(const Graph& g, int gs, int64_t base) {
  if (g.n() <= base) return cuthill_mckee(g);
  auto groups = bfs_groups(g, gs);
  const Graph c = coarsen(g, groups);
  const std::vector<int64_t> co = order(c, gs, base);
  std::vector<int64_t> out;
  out.reserve(g.n());
  for (int64_t k : co) out.insert(out.end(), groups[k].begin(), groups[k].end());
  return out;
}

constexpr int64_t kBaseNodes = 512;  // coarsest level ordered as a Cuthill-McKee level structure

}  // namespace

extern "C" int tmf_hierarchical_reorder(int64_t n_cells, int64_t n_interior_faces,
                                        const int32_t* interior_faces, int32_t group_size,
                                        int64_t* new_of_old) {
  if (n_cells <= 0 || !new_of_old || group_size < 2 || (n_interior_faces > 0 && !interior_faces))
    return TMF_EINVAL;
  std::vector<std::pair<int64_t, int64_t>> e;
  e.reserve(2 * n_interior_faces);
  for (int64_t f = 0; f < n_interior_faces; ++f) {
    const int64_t a = interior_faces[5 * f], b = interior_faces[5 * f + 2];
    if (a < 0 || b < 0 || a >= n_cells || b >= n_cells) return TMF_EINVAL;
    e.emplace_back(a, b);
    e.emplace_back(b, a);
  }
  const Graph g = from_edges(n_cells, e, nullptr);
  const std::vector<int64_t> seq = order(g, group_size, kBaseNodes);
  for (int64_t i = 0; i < n_cells; ++i) new_of_old[seq[i]] = i;
  return TMF_OK;
}
