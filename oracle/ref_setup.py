"""Pure-Python restatements of the reference's integer setup (oracle only).

Deliberately loop/dict based, following the reference line by line in
behaviour, so that the vectorised product versions can be checked against an
independent statement of the algorithm on small meshes.
"""

from __future__ import annotations

import numpy as np

FACE_VERTICES = ((1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2))
EDGE_VERTICES = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))
PERMS = ((0, 1, 2), (1, 2, 0), (2, 0, 1), (0, 2, 1), (2, 1, 0), (1, 0, 2))


def orientation_code(tm, tp) -> int:
    """reference.py:43-48."""
    for o, p in enumerate(PERMS):
        if (tp[p[0]], tp[p[1]], tp[p[2]]) == tuple(tm):
            return o
    raise ValueError("face corner sets differ")


def build_faces(cells, boundary_id_fn=None, vertices=None):
    """mesh.py:84-120: dict pairing keyed by sorted vertex triples."""
    fmap = {}
    for e in range(len(cells)):
        for lf in range(4):
            key = tuple(sorted(int(cells[e][c]) for c in FACE_VERTICES[lf]))
            fmap.setdefault(key, []).append((e, lf))
    interior, boundary = [], []
    for key, refs in fmap.items():
        if len(refs) == 2:
            (c0, f0), (c1, f1) = refs
            if c0 > c1:
                c0, f0, c1, f1 = c1, f1, c0, f0
            tm = tuple(int(cells[c0][c]) for c in FACE_VERTICES[f0])
            tp = tuple(int(cells[c1][c]) for c in FACE_VERTICES[f1])
            interior.append((c0, f0, c1, f1, orientation_code(tm, tp)))
        elif len(refs) == 1:
            e, lf = refs[0]
            bid = 0
            if boundary_id_fn is not None:
                bid = int(boundary_id_fn(vertices[[cells[e][c] for c in FACE_VERTICES[lf]]]))
            boundary.append((e, lf, bid))
        else:
            raise ValueError("face shared by more than two cells")
    return (np.array(sorted(interior), dtype=np.int32).reshape(-1, 5),
            np.array(sorted(boundary), dtype=np.int32).reshape(-1, 3))


def node_tags(p: int):
    """basis.py:48-69 tags (+ the documented P4 extension)."""
    tags = [("v", i, 0) for i in range(4)]
    tags += [("e", e, k) for e in range(6) for k in range(p - 1)]
    if p == 3:
        tags += [("f", f, 0) for f in range(4)]
    if p == 4:
        tags += [("f", f, j) for f in range(4) for j in range(3)]
        tags += [("c", 0, 0)]
    return tags


def build_cg_dofs(cells, n_vertices: int, p: int, boundary_faces=(), dirichlet_ids=()):
    """dofmap.py:67-144 (CG branch), first-encounter numbering with dicts."""
    edge_ids, face_ids = {}, {}
    if p >= 2:
        for e in range(len(cells)):
            for a, b in EDGE_VERTICES:
                key = tuple(sorted((int(cells[e][a]), int(cells[e][b]))))
                edge_ids.setdefault(key, len(edge_ids))
    if p >= 3:
        for e in range(len(cells)):
            for fv in FACE_VERTICES:
                key = tuple(sorted(int(cells[e][c]) for c in fv))
                face_ids.setdefault(key, len(face_ids))
    per_edge = p - 1
    edge_base = n_vertices
    face_base = edge_base + per_edge * len(edge_ids)
    per_face = 3 if p == 4 else 1
    interior_base = face_base + per_face * len(face_ids)
    n_scalar = interior_base + (len(cells) if p == 4 else 0)
    tags = node_tags(p)
    cd = np.empty((len(cells), len(tags)), dtype=np.int64)
    for e in range(len(cells)):
        cell = [int(v) for v in cells[e]]
        for j, (kind, ent, slot) in enumerate(tags):
            if kind == "v":
                cd[e, j] = cell[ent]
            elif kind == "e":
                a, b = EDGE_VERTICES[ent]
                ga, gb = cell[a], cell[b]
                k = slot if ga < gb else per_edge - 1 - slot
                cd[e, j] = edge_base + per_edge * edge_ids[(min(ga, gb), max(ga, gb))] + k
            elif kind == "f":
                corners = [cell[c] for c in FACE_VERTICES[ent]]
                fid = face_ids[tuple(sorted(corners))]
                if p == 3:
                    cd[e, j] = face_base + fid
                else:
                    cd[e, j] = face_base + 3 * fid + sorted(corners).index(corners[slot])
            else:
                cd[e, j] = interior_base + e
    mask = np.zeros(n_scalar, dtype=bool)
    dset = set(int(b) for b in dirichlet_ids)
    for c, lf, bid in (boundary_faces if len(boundary_faces) else []):
        if int(bid) not in dset:
            continue
        for j, (kind, ent, _) in enumerate(tags):
            on = ((kind == "v" and ent in FACE_VERTICES[lf])
                  or (kind == "e" and set(EDGE_VERTICES[ent]) <= set(FACE_VERTICES[lf]))
                  or (kind == "f" and ent == lf))
            if on:
                mask[cd[c, j]] = True
    return cd.astype(np.int32), mask, n_scalar


def color_batches(cell_dofs, cell_ids, active, space="cg"):
    """dofmap.py:269-292: greedy, smallest colour unused by adjacent earlier batches."""
    nb = len(cell_ids)
    colors = np.zeros(nb, dtype=np.int32)
    if space == "dg":
        return colors
    owner = {}
    for b in range(nb):
        for d in np.unique(cell_dofs[np.asarray(cell_ids[b])[np.asarray(active[b])]]).tolist():
            owner.setdefault(d, []).append(b)
    adj = [set() for _ in range(nb)]
    for bs in owner.values():
        for i in bs:
            for j in bs:
                if i != j:
                    adj[i].add(j)
    for b in range(nb):
        used = {colors[j] for j in adj[b] if j < b}
        c = 0
        while c in used:
            c += 1
        colors[b] = c
    return colors
