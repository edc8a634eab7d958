// Host-side mesh/DoF setup at scale (C++), bit-identical to the reference's
// Python setup (the reference needs minutes to tens of
// minutes for these at 12.6 M cells).
//
//   tmf_build_faces    <- mesh._build_faces   (mesh.py:84-120)
//   tmf_build_cg_dofs  <- dofmap.build_dof_map, CG branch (dofmap.py:67-123)
//                         + the documented P4 extension
//
// Both are O(n) bucket sorts keyed by the smallest vertex id instead of the
// reference's Python dicts; first-encounter numbering is reproduced exactly.
#include <algorithm>
#include <cstdint>
#include <numeric>
#include <vector>

#include "../../include/tetmf_b200.h"

namespace {

const int FV[4][3] = {{1, 2, 3}, {0, 2, 3}, {0, 1, 3}, {0, 1, 2}};
const int EV[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
const int PERMS[6][3] = {{0, 1, 2}, {1, 2, 0}, {2, 0, 1}, {0, 2, 1}, {2, 1, 0}, {1, 0, 2}};

struct Key3 {
  int32_t a, b, c;  // sorted a < b < c (or a < b, c = -1 for edges)
};

// Group items (pos = 0..n-1) by key; returns items sorted by (key, pos) and the
// bucket layout (counting sort on key.a, then sort by (b, c, pos) inside buckets).
std::vector<int64_t> sort_keys(const std::vector<Key3>& k, int64_t n_vertices) {
  const int64_t n = (int64_t)k.size();
  std::vector<int64_t> cnt(n_vertices + 1, 0);
  for (int64_t i = 0; i < n; ++i) cnt[k[i].a + 1]++;
  for (int64_t v = 0; v < n_vertices; ++v) cnt[v + 1] += cnt[v];
  std::vector<int64_t> out(n);
  {
    std::vector<int64_t> fill(cnt.begin(), cnt.end() - 1);
    for (int64_t i = 0; i < n; ++i) out[fill[k[i].a]++] = i;  // pos ascending inside a bucket
  }
  for (int64_t v = 0; v < n_vertices; ++v) {
    auto b = out.begin() + cnt[v], e = out.begin() + cnt[v + 1];
    if (e - b > 1)
      std::sort(b, e, [&](int64_t x, int64_t y) {
        if (k[x].b != k[y].b) return k[x].b < k[y].b;
        if (k[x].c != k[y].c) return k[x].c < k[y].c;
        return x < y;
      });
  }
  return out;
}

bool same(const Key3& x, const Key3& y) { return x.a == y.a && x.b == y.b && x.c == y.c; }

// First-encounter ids: id[pos] = rank of pos's key by its earliest position.
int64_t first_encounter(const std::vector<Key3>& k, int64_t n_vertices, std::vector<int64_t>& id) {
  const int64_t n = (int64_t)k.size();
  const std::vector<int64_t> s = sort_keys(k, n_vertices);
  std::vector<int64_t> first_of(n);        // pos -> first pos of its key
  std::vector<char> is_first(n, 0);
  for (int64_t i = 0; i < n;) {
    int64_t j = i;
    while (j < n && same(k[s[j]], k[s[i]])) ++j;
    const int64_t f = s[i];                 // smallest pos (sorted by pos inside equal keys)
    is_first[f] = 1;
    for (int64_t t = i; t < j; ++t) first_of[s[t]] = f;
    i = j;
  }
  std::vector<int64_t> rank(n, -1);
  int64_t next = 0;
  for (int64_t p = 0; p < n; ++p)
    if (is_first[p]) rank[p] = next++;
  id.resize(n);
  for (int64_t p = 0; p < n; ++p) id[p] = rank[first_of[p]];
  return next;
}

Key3 sorted3(int32_t x, int32_t y, int32_t z) {
  if (x > y) std::swap(x, y);
  if (y > z) std::swap(y, z);
  if (x > y) std::swap(x, y);
  return Key3{x, y, z};
}

}  // namespace

extern "C" int tmf_build_faces(int64_t n_cells, const int32_t* cells, int64_t n_vertices,
                               int32_t* interior_out, int64_t* n_interior, int32_t* boundary_out,
                               int64_t* n_boundary) {
  if (n_cells <= 0 || !cells || !interior_out || !boundary_out || !n_interior || !n_boundary)
    return TMF_EINVAL;
  for (int64_t i = 0; i < 4 * n_cells; ++i)
    if (cells[i] < 0 || cells[i] >= n_vertices) return TMF_EINVAL;
  const int64_t n = 4 * n_cells;
  std::vector<Key3> k(n);
  for (int64_t e = 0; e < n_cells; ++e)
    for (int lf = 0; lf < 4; ++lf) {
      const int32_t* c = cells + 4 * e;
      k[4 * e + lf] = sorted3(c[FV[lf][0]], c[FV[lf][1]], c[FV[lf][2]]);
    }
  const std::vector<int64_t> s = sort_keys(k, n_vertices);
  std::vector<int64_t> partner(n, -1);
  for (int64_t i = 0; i < n;) {
    int64_t j = i;
    while (j < n && same(k[s[j]], k[s[i]])) ++j;
    if (j - i > 2) return TMF_EINVAL;  // face referenced by more than two cells
    if (j - i == 2) {
      partner[s[i]] = s[i + 1];
      partner[s[i + 1]] = s[i];
    }
    i = j;
  }
  // interior faces sorted by (c-, lf-) == ascending flat position of the minus side;
  // boundary faces by (cell, lf) (mesh.py:117-119)
  int64_t ni = 0, nb = 0;
  for (int64_t p = 0; p < n; ++p) {
    const int64_t q = partner[p];
    if (q < 0) {
      boundary_out[3 * nb] = (int32_t)(p / 4);
      boundary_out[3 * nb + 1] = (int32_t)(p % 4);
      boundary_out[3 * nb + 2] = 0;
      ++nb;
    } else if (p < q) {
      const int64_t c0 = p / 4, f0 = p % 4, c1 = q / 4, f1 = q % 4;
      const int32_t* a = cells + 4 * c0;
      const int32_t* b = cells + 4 * c1;
      const int32_t tm[3] = {a[FV[f0][0]], a[FV[f0][1]], a[FV[f0][2]]};
      const int32_t tp[3] = {b[FV[f1][0]], b[FV[f1][1]], b[FV[f1][2]]};
      int code = -1;
      for (int o = 0; o < 6 && code < 0; ++o)
        if (tp[PERMS[o][0]] == tm[0] && tp[PERMS[o][1]] == tm[1] && tp[PERMS[o][2]] == tm[2]) code = o;
      if (code < 0) return TMF_EINVAL;
      int32_t* r = interior_out + 5 * ni;
      r[0] = (int32_t)c0;
      r[1] = (int32_t)f0;
      r[2] = (int32_t)c1;
      r[3] = (int32_t)f1;
      r[4] = code;
      ++ni;
    }
  }
  *n_interior = ni;
  *n_boundary = nb;
  return TMF_OK;
}

extern "C" int tmf_build_cg_dofs(int64_t n_cells, const int32_t* cells, int64_t n_vertices,
                                 int32_t degree, int32_t* cell_dofs, int64_t* n_scalar_dofs) {
  const int p = degree;
  if (n_cells <= 0 || !cells || !cell_dofs || !n_scalar_dofs || p < 1 || p > 4) return TMF_EINVAL;
  for (int64_t i = 0; i < 4 * n_cells; ++i)
    if (cells[i] < 0 || cells[i] >= n_vertices) return TMF_EINVAL;
  const int nd = (p + 1) * (p + 2) * (p + 3) / 6;
  const int per_edge = p - 1;
  std::vector<int64_t> eid, fid;
  int64_t n_edges = 0, n_faces = 0;
  if (p >= 2) {  // first-encounter pass over (cell, local edge), dofmap.py:93-97
    std::vector<Key3> k(6 * n_cells);
    for (int64_t e = 0; e < n_cells; ++e)
      for (int le = 0; le < 6; ++le) {
        int32_t x = cells[4 * e + EV[le][0]], y = cells[4 * e + EV[le][1]];
        k[6 * e + le] = Key3{std::min(x, y), std::max(x, y), -1};
      }
    n_edges = first_encounter(k, n_vertices, eid);
  }
  if (p >= 3) {  // separate, later pass over (cell, local face), dofmap.py:98-102
    std::vector<Key3> k(4 * n_cells);
    for (int64_t e = 0; e < n_cells; ++e)
      for (int lf = 0; lf < 4; ++lf) {
        const int32_t* c = cells + 4 * e;
        k[4 * e + lf] = sorted3(c[FV[lf][0]], c[FV[lf][1]], c[FV[lf][2]]);
      }
    n_faces = first_encounter(k, n_vertices, fid);
  }
  const int64_t edge_base = n_vertices;
  const int64_t face_base = edge_base + per_edge * n_edges;
  const int64_t per_face = p == 3 ? 1 : (p == 4 ? 3 : 0);
  const int64_t interior_base = face_base + per_face * n_faces;
  const int64_t n_scalar = interior_base + (p == 4 ? n_cells : 0);
  if (n_scalar >= ((int64_t)1 << 31)) return TMF_EINVAL;
  for (int64_t e = 0; e < n_cells; ++e) {
    const int32_t* c = cells + 4 * e;
    int32_t* out = cell_dofs + (int64_t)nd * e;
    int j = 0;
    for (int v = 0; v < 4; ++v) out[j++] = c[v];
    for (int le = 0; le < 6; ++le) {
      const bool asc = c[EV[le][0]] < c[EV[le][1]];
      for (int slot = 0; slot < per_edge; ++slot)
        out[j++] = (int32_t)(edge_base + per_edge * eid[6 * e + le] + (asc ? slot : per_edge - 1 - slot));
    }
    if (p == 3)
      for (int lf = 0; lf < 4; ++lf) out[j++] = (int32_t)(face_base + fid[4 * e + lf]);
    if (p == 4) {
      for (int lf = 0; lf < 4; ++lf) {
        const int32_t g[3] = {c[FV[lf][0]], c[FV[lf][1]], c[FV[lf][2]]};
        for (int slot = 0; slot < 3; ++slot) {
          const int rank = (g[0] < g[slot]) + (g[1] < g[slot]) + (g[2] < g[slot]);
          out[j++] = (int32_t)(face_base + 3 * fid[4 * e + lf] + rank);
        }
      }
      out[j++] = (int32_t)(interior_base + e);
    }
  }
  *n_scalar_dofs = n_scalar;
  return TMF_OK;
}

// Greedy distance-1 colouring of the face-adjacency graph of the cells (cells in order, each
// gets the smallest colour not used by an already coloured face neighbour) -- the cell-level
// analogue of the reference's batch colouring (dofmap.py:269-292).  Used to probe the exact
// diagonal of DG operators: cells of one colour share no face, so one apply per
// (colour, local DoF) reads their diagonal entries (multigrid.py: dg_diagonal).
extern "C" int tmf_color_cells(int64_t n_cells, int64_t n_interior_faces, const int32_t* interior_faces,
                               int32_t* colors, int32_t* n_colors) {
  if (n_cells < 0 || n_interior_faces < 0 || !colors || !n_colors || (n_interior_faces && !interior_faces))
    return TMF_EINVAL;
  std::vector<int64_t> start(n_cells + 1, 0);
  for (int64_t f = 0; f < n_interior_faces; ++f) {
    const int32_t a = interior_faces[5 * f], b = interior_faces[5 * f + 2];
    if (a < 0 || a >= n_cells || b < 0 || b >= n_cells) return TMF_EINVAL;
    start[a + 1]++;
    start[b + 1]++;
  }
  for (int64_t e = 0; e < n_cells; ++e) start[e + 1] += start[e];
  std::vector<int32_t> adj(start[n_cells]);
  {
    std::vector<int64_t> fill(start.begin(), start.end() - 1);
    for (int64_t f = 0; f < n_interior_faces; ++f) {
      const int32_t a = interior_faces[5 * f], b = interior_faces[5 * f + 2];
      adj[fill[a]++] = b;
      adj[fill[b]++] = a;
    }
  }
  int32_t nc = 0;
  for (int64_t e = 0; e < n_cells; ++e) colors[e] = -1;
  for (int64_t e = 0; e < n_cells; ++e) {
    uint64_t used = 0;
    for (int64_t k = start[e]; k < start[e + 1]; ++k) {
      const int32_t c = colors[adj[k]];
      if (c >= 0 && c < 64) used |= 1ull << c;
    }
    int32_t c = 0;
    while (c < 64 && (used >> c & 1)) ++c;
    colors[e] = c;   // a cell has <= 4 face neighbours, so c <= 4
    if (c + 1 > nc) nc = c + 1;
  }
  *n_colors = nc;
  return TMF_OK;
}
