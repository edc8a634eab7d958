"""Pure-Python restatement of hierarchical cell reordering (oracle only).

The reference package has no implementation (SURVEY finding 3); this restates
the SPEC with the deterministic choices
recorded in SURVEY Appendix B12 and DESIGN.md.  Parity of the product's C++
implementation (csrc/reorder.cpp) against this file is bit-exact on the
permutation; parity against the reference itself is unpinned.

    order(G):  if |G| <= base: cuthill_mckee(G)
               groups = bfs_groups(G)            # members in BFS growth order
               C = coarsen(G, groups)           # weight = number of shared faces
               return concat(groups[c] for c in order(C))
    cuthill_mckee: BFS from the lowest-degree node (ties: lowest id), each
               node's unvisited neighbours appended by (degree, id); restart at
               the lowest-degree unvisited node for another component.  Ordering
               the top of the hierarchy (<= base = 512 groups) as a level
               structure bounds the bandwidth, the groups below keep locality.
    bfs_groups: seed = the unvisited neighbour of the previous group with the
               fewest unvisited neighbours (ties: lowest id); if there is none,
               the lowest-degree unvisited node (ties: lowest id).  Grow by BFS
               over unvisited neighbours in ascending id until g nodes (a group
               closes early if its frontier empties).
"""

from __future__ import annotations

import numpy as np


def cell_graph(n_cells, interior_faces):
    adj = [dict() for _ in range(n_cells)]
    for r in interior_faces:
        a, b = int(r[0]), int(r[2])
        adj[a][b] = adj[a].get(b, 0) + 1
        adj[b][a] = adj[b].get(a, 0) + 1
    return adj


def _by_degree(adj):
    return sorted(range(len(adj)), key=lambda v: (len(adj[v]), v))


def bfs_groups(adj, g):
    n = len(adj)
    visited = [False] * n
    groups = []
    seeds = _by_degree(adj)
    si = 0
    last = None
    while True:
        seed = None
        if last is not None:           # continue next to the previous group
            best = None
            for v in last:
                for nb in adj[v]:
                    if not visited[nb]:
                        free = sum(1 for x in adj[nb] if not visited[x])
                        if best is None or (free, nb) < best:
                            best = (free, nb)
            if best is not None:
                seed = best[1]
        if seed is None:
            while si < n and visited[seeds[si]]:
                si += 1
            if si == n:
                break
            seed = seeds[si]
        visited[seed] = True
        grp, queue, head = [seed], [seed], 0
        while head < len(queue) and len(grp) < g:
            v = queue[head]
            head += 1
            for nb in sorted(adj[v]):
                if len(grp) >= g:
                    break
                if not visited[nb]:
                    visited[nb] = True
                    grp.append(nb)
                    queue.append(nb)
        groups.append(grp)
        last = grp
    return groups


def coarsen(adj, groups):
    gid = [0] * len(adj)
    for k, grp in enumerate(groups):
        for v in grp:
            gid[v] = k
    cadj = [dict() for _ in groups]
    for v, nbrs in enumerate(adj):
        for u, w in nbrs.items():
            if gid[u] != gid[v]:
                cadj[gid[v]][gid[u]] = cadj[gid[v]].get(gid[u], 0) + w
    return cadj


def cuthill_mckee(adj):
    n = len(adj)
    seen = [False] * n
    seeds = _by_degree(adj)
    out, si = [], 0
    while len(out) < n:
        while seen[seeds[si]]:
            si += 1
        s = seeds[si]
        seen[s] = True
        queue, head = [s], 0
        while head < len(queue):
            v = queue[head]
            head += 1
            out.append(v)
            for u in sorted(adj[v], key=lambda x: (len(adj[x]), x)):
                if not seen[u]:
                    seen[u] = True
                    queue.append(u)
    return out


def order(adj, g, base=512):
    if len(adj) <= base:
        return cuthill_mckee(adj)
    groups = bfs_groups(adj, g)
    corder = order(coarsen(adj, groups), g, base)
    return [v for c in corder for v in groups[c]]


def hierarchical_reorder(n_cells, interior_faces, group_size=8, base=512):
    """new_of_old permutation (cell e moves to position new_of_old[e])."""
    if group_size < 2:
        raise ValueError("group_size must be >= 2")
    seq = order(cell_graph(n_cells, interior_faces), group_size, base)
    new_of_old = np.empty(n_cells, dtype=np.int64)
    new_of_old[np.asarray(seq, dtype=np.int64)] = np.arange(n_cells)
    return new_of_old


def locality_metrics(n_cells, interior_faces):
    """(mean |i-j|, max |i-j|) over face-adjacent cell pairs."""
    d = np.abs(interior_faces[:, 0].astype(np.int64) - interior_faces[:, 2])
    return (float(d.mean()) if len(d) else 0.0, int(d.max()) if len(d) else 0)
