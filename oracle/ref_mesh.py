"""Vectorised NumPy restatement of the reference's integer setup (oracle only).

Test / measurement infrastructure: the bench's reference arm (``bench.py --impl
reference``) builds its whole workload with this module, ``ref_reorder`` and
``ref_apply`` -- nothing from the product package or its shared library -- and
``tests/test_oracle_setup.py`` pins every function here bit-for-bit against the
dict/loop restatements in ``ref_setup`` (which follow the reference line by line)
and against the reference fixtures.

    kuhn_mesh            the BASELINE mesh generator (mesh.py:123-130 orientation)
    build_faces          mesh.py:84-120   (_build_faces: sorted-triple pairing, codes, order)
    orientation_codes    reference.py:43-48
    cg_dofs              dofmap.py:67-144 (first-encounter edge / face numbering, p <= 3;
                                           P4 per SURVEY Appendix B6)
    dirichlet_mask       dofmap.py:125-142
    permute_cells        mesh.py:291-293  (apply_cell_permutation; faces rebuilt)
    first_touch_vertices renumber vertices by first touch in cell order
"""

from __future__ import annotations

import itertools

import numpy as np

FACE_VERTICES = np.array(((1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2)))
EDGE_VERTICES = np.array(((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3)))
PERMS = ((0, 1, 2), (1, 2, 0), (2, 0, 1), (0, 2, 1), (2, 1, 0), (1, 0, 2))


def orientation_codes(tm: np.ndarray, tp: np.ndarray) -> np.ndarray:
    """reference.py:43-48 row-wise: o with tp[PERMS[o]] == tm."""
    code = np.full(len(tm), -1, dtype=np.int64)
    for o, p in enumerate(PERMS):
        hit = np.all(tp[:, list(p)] == tm, axis=1) & (code < 0)
        code[hit] = o
    if np.any(code < 0):
        raise ValueError("face corner sets differ")
    return code


def _cube_ids(coords: np.ndarray) -> np.ndarray:
    """Boundary ids 0..5 = -x, +x, -y, +y, -z, +z of faces on the unit cube's sides."""
    out = np.zeros(len(coords), dtype=np.int64)
    done = np.zeros(len(coords), dtype=bool)
    for axis in range(3):
        for side, val in ((0, 0.0), (1, 1.0)):
            hit = np.all(np.abs(coords[:, :, axis] - val) < 1e-9, axis=1) & ~done
            out[hit] = 2 * axis + side
            done |= hit
    return out


def build_faces(cells: np.ndarray, vertices: np.ndarray | None = None):
    """mesh.py:84-120: faces keyed by the sorted global vertex triple; a key seen twice is
    an interior face (c-, lf-, c+, lf+, code) with c- < c+ (first reference), a key seen once
    a boundary face (c, lf, id); both lists sorted lexicographically."""
    cells = np.asarray(cells, dtype=np.int64)
    n = len(cells)
    tri = cells[:, FACE_VERTICES].reshape(-1, 3)                 # row 4 e + lf
    key = np.sort(tri, axis=1)
    order = np.lexsort((np.arange(4 * n), key[:, 2], key[:, 1], key[:, 0]))
    ks = key[order]
    same = np.all(ks[1:] == ks[:-1], axis=1)
    if len(same) > 1 and np.any(same[1:] & same[:-1]):
        raise ValueError("face shared by more than two cells")
    first = np.flatnonzero(same)
    a, b = order[first], order[first + 1]                         # a < b: minus = lower cell
    interior = np.stack([a // 4, a % 4, b // 4, b % 4, orientation_codes(tri[a], tri[b])], axis=1)
    interior = interior[np.lexsort((interior[:, 1], interior[:, 0]))]
    paired = np.zeros(4 * n, dtype=bool)
    paired[first] = paired[first + 1] = True
    single = np.sort(order[~paired])
    bid = _cube_ids(vertices[tri[single]]) if vertices is not None else np.zeros(len(single), np.int64)
    boundary = np.stack([single // 4, single % 4, bid], axis=1)
    return interior.astype(np.int32).reshape(-1, 5), boundary.astype(np.int32).reshape(-1, 3)


def kuhn_mesh(n: int, seed: int = 0, jitter: float = 0.2, permute: bool = True):
    """BASELINE mesh: unit cube, n^3 subcubes x 6 Kuhn tets (v0, v0+e_a,
    v0+e_a+e_b, v0+e_a+e_b+e_c) over the 6 axis permutations, interior vertices jittered
    U[-jitter h, jitter h] per coordinate, negative cells fixed by swapping local vertices
    2 <-> 3 (mesh.py:123-130), cells randomly permuted; default_rng(seed): jitter first,
    then the permutation.  Returns (vertices, cells, interior_faces, boundary_faces)."""
    h, m = 1.0 / n, n + 1
    g = np.arange(m, dtype=np.float64) * h
    vertices = np.stack(np.meshgrid(g, g, g, indexing="ij"), axis=-1).reshape(-1, 3)
    ijk = np.stack(np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij"), -1).reshape(-1, 3)
    inner = np.all((ijk > 0) & (ijk < n), axis=1)
    rng = np.random.default_rng(seed)
    if jitter:
        vertices[inner] += rng.uniform(-jitter * h, jitter * h, size=(int(inner.sum()), 3))
    base = np.stack(np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij"), -1).reshape(-1, 3)
    tets = []
    for perm in itertools.permutations(range(3)):
        c = [np.zeros(3, np.int64)]
        for ax in perm:
            c.append(c[-1] + np.eye(3, dtype=np.int64)[ax])
        tets.append(c)
    pts = base[:, None, None, :] + np.array(tets)[None]
    cells = ((pts[..., 0] * m + pts[..., 1]) * m + pts[..., 2]).reshape(-1, 4)
    v = vertices[cells]
    det = np.linalg.det(np.stack([v[:, 1] - v[:, 0], v[:, 2] - v[:, 0], v[:, 3] - v[:, 0]], axis=2))
    neg = det < 0
    cells[neg] = cells[neg][:, [0, 1, 3, 2]]
    if permute:
        cells = cells[rng.permutation(len(cells))]
    cells = cells.astype(np.int32)
    inter, bnd = build_faces(cells, vertices)
    return vertices, cells, inter, bnd


def _carry_ids(old_cells, old_bnd, new_cells, new_bnd):
    """Boundary ids follow the face's vertex triple (mesh.py:268-282)."""
    if not len(new_bnd):
        return new_bnd
    okey = np.sort(old_cells[old_bnd[:, 0, None], FACE_VERTICES[old_bnd[:, 1]]], axis=1).astype(np.int64)
    nkey = np.sort(new_cells[new_bnd[:, 0, None], FACE_VERTICES[new_bnd[:, 1]]], axis=1).astype(np.int64)
    big = int(max(okey.max(), nkey.max())) + 1
    oc = (okey[:, 0] * big + okey[:, 1]) * big + okey[:, 2]
    nc = (nkey[:, 0] * big + nkey[:, 1]) * big + nkey[:, 2]
    srt = np.argsort(oc)
    pos = np.searchsorted(oc[srt], nc)
    out = new_bnd.copy()
    out[:, 2] = old_bnd[srt[pos], 2]
    return out


def permute_cells(cells, boundary_faces, new_of_old):
    """mesh.py:291-293: cell e moves to position new_of_old[e]; faces rebuilt."""
    order = np.argsort(np.asarray(new_of_old))
    nc = np.asarray(cells)[order]
    inter, bnd = build_faces(nc)
    return nc, inter, _carry_ids(np.asarray(cells), np.asarray(boundary_faces), nc, bnd)


def first_touch_vertices(vertices, cells, boundary_faces):
    """Vertices renumbered by first appearance in the cell list (unused vertices last);
    faces rebuilt (orientation codes follow global ids).  Returns (vertices, cells, if, bf)."""
    flat = np.asarray(cells).ravel()
    uniq, first = np.unique(flat, return_index=True)
    order = uniq[np.argsort(first, kind="stable")]
    nv = len(vertices)
    order = np.concatenate([order, np.setdiff1d(np.arange(nv), order, assume_unique=True)])
    new_of_old = np.empty(nv, dtype=np.int64)
    new_of_old[order] = np.arange(nv)
    verts = np.empty_like(vertices)
    verts[new_of_old] = vertices
    nc = new_of_old[np.asarray(cells)].astype(np.int32)
    inter, bnd = build_faces(nc)
    old = new_of_old[np.asarray(cells)]
    return verts, nc, inter, _carry_ids(old, np.asarray(boundary_faces), nc, bnd)


def _first_encounter(keys: np.ndarray):
    """Ids of the rows of keys numbered by first appearance (dict.setdefault order)."""
    keys = np.asarray(keys, dtype=np.int64)
    big = int(keys.max()) + 1 if len(keys) else 1
    if big ** keys.shape[1] < 2 ** 62:       # rows packed into one int64 (same order)
        packed = np.zeros(len(keys), dtype=np.int64)
        for c in range(keys.shape[1]):
            packed = packed * big + keys[:, c]
        keys = packed
        _, first, inv = np.unique(keys, return_index=True, return_inverse=True)
    else:
        _, first, inv = np.unique(keys, axis=0, return_index=True, return_inverse=True)
    rank = np.empty(len(first), dtype=np.int64)
    rank[np.argsort(first, kind="stable")] = np.arange(len(first))
    return rank[inv.ravel()], len(first)


def node_tags(p: int):
    """basis.py:48-69 node order (+ SURVEY B6 at P4)."""
    tags = [("v", i, 0) for i in range(4)]
    tags += [("e", e, k) for e in range(6) for k in range(p - 1)]
    if p == 3:
        tags += [("f", f, 0) for f in range(4)]
    if p == 4:
        tags += [("f", f, j) for f in range(4) for j in range(3)] + [("c", 0, 0)]
    return tags


def cg_dofs(cells: np.ndarray, n_vertices: int, p: int):
    """dofmap.py:67-144 (CG): vertex DoF = vertex id; edge ids by first encounter over
    (cell, local edge), p-1 DoFs per edge oriented by global vertex id; face ids by a later
    first-encounter pass; P4: 3 DoFs per face ranked by global corner id, 1 per cell.
    Returns (cell_dofs (n, n_dpc) int32, n_scalar_dofs)."""
    cells = np.asarray(cells, dtype=np.int64)
    n = len(cells)
    per_edge = p - 1
    n_edges = n_faces = 0
    if p >= 2:
        ev = cells[:, EDGE_VERTICES]
        eid, n_edges = _first_encounter(np.sort(ev, axis=2).reshape(-1, 2))
        eid = eid.reshape(n, 6)
        asc = ev[:, :, 0] < ev[:, :, 1]
    face_base = n_vertices + per_edge * n_edges
    if p >= 3:
        fv = cells[:, FACE_VERTICES]
        fid, n_faces = _first_encounter(np.sort(fv, axis=2).reshape(-1, 3))
        fid = fid.reshape(n, 4)
    interior_base = face_base + {3: 1, 4: 3}.get(p, 0) * n_faces
    n_scalar = interior_base + (n if p == 4 else 0)
    tags = node_tags(p)
    cd = np.empty((n, len(tags)), dtype=np.int64)
    for j, (kind, ent, slot) in enumerate(tags):
        if kind == "v":
            cd[:, j] = cells[:, ent]
        elif kind == "e":
            cd[:, j] = n_vertices + per_edge * eid[:, ent] + np.where(asc[:, ent], slot, per_edge - 1 - slot)
        elif kind == "f":
            if p == 3:
                cd[:, j] = face_base + fid[:, ent]
            else:
                corners = fv[:, ent]
                cd[:, j] = face_base + 3 * fid[:, ent] + (corners < corners[:, slot, None]).sum(axis=1)
        else:
            cd[:, j] = interior_base + np.arange(n)
    return cd.astype(np.int32), int(n_scalar)


def dirichlet_mask(cell_dofs, n_scalar, p, boundary_faces, dirichlet_ids):
    """dofmap.py:125-142: closure of the selected boundary faces."""
    mask = np.zeros(n_scalar, dtype=bool)
    bf = np.asarray(boundary_faces)
    if not len(bf) or not len(dirichlet_ids):
        return mask
    tags = node_tags(p)
    sel = np.isin(bf[:, 2], np.array(sorted(int(b) for b in dirichlet_ids)))
    for lf in range(4):
        fvs = set(FACE_VERTICES[lf].tolist())
        on = [j for j, (k, e, _) in enumerate(tags)
              if (k == "v" and e in fvs) or (k == "e" and set(EDGE_VERTICES[e].tolist()) <= fvs)
              or (k == "f" and e == lf)]
        rows = bf[sel & (bf[:, 1] == lf), 0]
        mask[np.asarray(cell_dofs)[rows[:, None], np.array(on)[None, :]].ravel()] = True
    return mask
