"""Tetrahedral meshes: the reference ``TetMesh`` container, face pairing, and
the BASELINE.json Kuhn-cube generator.

``TetMesh`` mirrors mesh.py:33-81.  :func:`build_faces` is a vectorised,
bit-identical restatement of ``_build_faces`` (mesh.py:84-120):

* every (cell e, local face lf) is keyed by the sorted global vertex triple of
  ``cells[e, FACE_VERTICES[lf]]``;
* a key seen twice is an interior face ``(c0, f0, c1, f1, code)`` with
  ``c0 < c1`` and ``code = orientation_code(cells[c0, FV[f0]], cells[c1, FV[f1]])``;
* a key seen once is a boundary face ``(e, lf, bid)``;
* both lists are sorted lexicographically (mesh.py:117-119).

The generator follows SURVEY §8(d): unit cube, n^3 subcubes of 6 Kuhn tets
``(v0, v0+e_a, v0+e_a+e_b, v0+e_a+e_b+e_c)`` for the 6 axis permutations,
interior vertices jittered by U[-0.2h, 0.2h] per coordinate, negative cells
repaired by swapping local vertices 2<->3 (mesh.py:123-130), then cells
randomly permuted.  RNG: ``numpy.random.default_rng(seed)``, jitter drawn
first, then the permutation.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

from .reference import FACE_VERTICES_ARR, orientation_codes

__all__ = ["TetMesh", "build_faces", "orient_positive", "kuhn_cube_mesh",
           "apply_cell_permutation", "cube_boundary_ids"]


@dataclass
class TetMesh:
    vertices: np.ndarray            # (n_v, 3) float64
    cells: np.ndarray               # (n_cells, 4) int32
    interior_faces: np.ndarray      # (n_if, 5) int32: c-, lf-, c+, lf+, code
    boundary_faces: np.ndarray      # (n_bf, 3) int32: cell, lf, boundary id
    geometry_nodes: np.ndarray | None = None
    parent_cells: np.ndarray | None = None

    @property
    def n_vertices(self) -> int:
        return len(self.vertices)

    @property
    def n_cells(self) -> int:
        return len(self.cells)

    @property
    def is_curved(self) -> bool:
        return self.geometry_nodes is not None

    def cell_jacobians(self) -> np.ndarray:
        v = self.vertices[self.cells]
        return np.stack([v[:, 1] - v[:, 0], v[:, 2] - v[:, 0], v[:, 3] - v[:, 0]], axis=2)

    def cell_volumes(self) -> np.ndarray:
        return np.linalg.det(self.cell_jacobians()) / 6.0

    def validate(self) -> None:
        assert self.cells.min() >= 0 and self.cells.max() < self.n_vertices
        assert np.all(self.cell_volumes() > 0)
        assert 4 * self.n_cells == 2 * len(self.interior_faces) + len(self.boundary_faces)
        f = self.interior_faces
        if len(f):
            tm = self.cells[f[:, 0, None], FACE_VERTICES_ARR[f[:, 1]]]
            tp = self.cells[f[:, 2, None], FACE_VERTICES_ARR[f[:, 3]]]
            assert np.array_equal(orientation_codes(tm, tp), f[:, 4])


def _face_keys(cells: np.ndarray):
    tri = cells[:, FACE_VERTICES_ARR].reshape(-1, 3).astype(np.int64)   # (4N, 3), row = 4e+lf
    return tri, np.sort(tri, axis=1)


def build_faces(cells: np.ndarray, vertices: np.ndarray | None = None, boundary_id_fn=None,
                method: str = "native"):
    """``_build_faces`` restated; ``boundary_id_fn(coords (F,3,3)) -> (F,)``.

    method "native": O(n) bucket sort in C++ (csrc/setup.cpp, tmf_build_faces);
    "numpy": vectorised lexsort.  Both are bit-identical to the reference."""
    cells = np.asarray(cells)
    if method == "native":
        interior, boundary = _build_faces_native(cells)
        if boundary_id_fn is not None and len(boundary):
            tri = cells[boundary[:, 0, None], FACE_VERTICES_ARR[boundary[:, 1]]]
            boundary[:, 2] = np.asarray(boundary_id_fn(vertices[tri]), dtype=np.int64)
        return interior, boundary
    if method != "numpy":
        raise ValueError(f"unknown method {method!r}")
    n = len(cells)
    tri, key = _face_keys(cells)
    order = np.lexsort((np.arange(4 * n), key[:, 2], key[:, 1], key[:, 0]))
    ks = key[order]
    same_next = np.all(ks[1:] == ks[:-1], axis=1)
    if len(same_next) > 1 and np.any(same_next[1:] & same_next[:-1]):
        raise ValueError("face referenced by more than 2 cells")
    first = np.flatnonzero(same_next)                  # start of each interior pair
    paired = np.zeros(len(ks), dtype=bool)
    paired[first] = True
    paired[first + 1] = True
    a, b = order[first], order[first + 1]              # a < b as flat (4e+lf) ids
    c0, f0, c1, f1 = a // 4, a % 4, b // 4, b % 4
    codes = orientation_codes(tri[a], tri[b])
    interior = np.stack([c0, f0, c1, f1, codes], axis=1)
    interior = interior[np.lexsort((interior[:, 1], interior[:, 0]))].astype(np.int32)

    single = np.sort(order[~paired])
    be, bl = single // 4, single % 4
    if boundary_id_fn is not None and len(single):
        bid = np.asarray(boundary_id_fn(vertices[tri[single]]), dtype=np.int64)
    else:
        bid = np.zeros(len(single), dtype=np.int64)
    boundary = np.stack([be, bl, bid], axis=1).astype(np.int32).reshape(-1, 3)
    return interior.reshape(-1, 5), boundary


def _build_faces_native(cells: np.ndarray):
    import ctypes as C

    from . import _lib

    c = np.ascontiguousarray(cells, dtype=np.int32)
    n = len(c)
    nv = int(c.max()) + 1 if n else 0
    inter = np.empty((2 * n, 5), dtype=np.int32)
    bnd = np.empty((4 * n, 3), dtype=np.int32)
    ni, nb = C.c_int64(), C.c_int64()
    rc = _lib.lib().tmf_build_faces(n, _lib.ptr(c, C.c_int32), nv, _lib.ptr(inter, C.c_int32), C.byref(ni),
                                    _lib.ptr(bnd, C.c_int32), C.byref(nb))
    if rc:
        raise ValueError("face pairing failed: a face is referenced by more than two cells "
                         "or the cell array is invalid")
    return inter[:ni.value].copy(), bnd[:nb.value].copy()


def orient_positive(vertices: np.ndarray, cells: np.ndarray) -> np.ndarray:
    cells = cells.copy()
    v = vertices[cells]
    jac = np.stack([v[:, 1] - v[:, 0], v[:, 2] - v[:, 0], v[:, 3] - v[:, 0]], axis=2)
    neg = np.linalg.det(jac) < 0
    cells[neg] = cells[neg][:, [0, 1, 3, 2]]
    return cells


def cube_boundary_ids(coords: np.ndarray, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    """Ids 0..5 = -x,+x,-y,+y,-z,+z for faces lying on the box sides (else 0)."""
    out = np.zeros(len(coords), dtype=np.int64)
    done = np.zeros(len(coords), dtype=bool)
    for axis in range(3):
        for side, val in ((0, lo), (1, hi)):
            hit = np.all(np.abs(coords[:, :, axis] - val) < 1e-9, axis=1) & ~done
            out[hit] = 2 * axis + side
            done |= hit
    return out


def kuhn_cube_mesh(n: int, seed: int = 0, jitter: float = 0.2, permute: bool = True) -> TetMesh:
    """Jittered, randomly permuted 6-tet Kuhn split of [0,1]^3 with n^3 subcubes."""
    n = int(n)
    if n < 1:
        raise ValueError("n must be >= 1")
    h = 1.0 / n
    m = n + 1
    ax = np.arange(m, dtype=np.float64) * h
    ii, jj, kk = np.meshgrid(ax, ax, ax, indexing="ij")
    vertices = np.stack([ii.ravel(), jj.ravel(), kk.ravel()], axis=1)
    rng = np.random.default_rng(seed)
    ijk = np.stack(np.meshgrid(np.arange(m), np.arange(m), np.arange(m), indexing="ij"), -1).reshape(-1, 3)
    interior = np.all((ijk > 0) & (ijk < n), axis=1)
    if jitter:
        vertices[interior] += rng.uniform(-jitter * h, jitter * h, size=(int(interior.sum()), 3))

    I, J, K = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    base = np.stack([I.ravel(), J.ravel(), K.ravel()], axis=1)          # cube origins, lexicographic
    unit = np.eye(3, dtype=np.int64)
    tets = []
    for perm in itertools.permutations(range(3)):
        corners = [np.zeros(3, np.int64)]
        for a in perm:
            corners.append(corners[-1] + unit[a])
        tets.append(corners)
    tets = np.array(tets)                                                 # (6, 4, 3)
    pts = base[:, None, None, :] + tets[None]                             # (n^3, 6, 4, 3)
    gid = (pts[..., 0] * m + pts[..., 1]) * m + pts[..., 2]
    cells = gid.reshape(-1, 4).astype(np.int32)
    cells = orient_positive(vertices, cells)
    if permute:
        cells = cells[rng.permutation(len(cells))]
    interior_f, boundary_f = build_faces(cells, vertices, cube_boundary_ids)
    return TetMesh(vertices, cells, interior_f, boundary_f)


def apply_cell_permutation(mesh: TetMesh, new_of_old: np.ndarray) -> TetMesh:
    """Cell e moves to position new_of_old[e] (mesh.py:291-293); faces rebuilt,
    boundary ids carried over by vertex triple (mesh.py:268-282)."""
    order = np.argsort(new_of_old)
    cells = mesh.cells[order]
    interior, bnd = build_faces(cells)
    if len(bnd):
        old_tri = np.sort(mesh.cells[mesh.boundary_faces[:, 0, None],
                                     FACE_VERTICES_ARR[mesh.boundary_faces[:, 1]]], axis=1)
        new_tri = np.sort(cells[bnd[:, 0, None], FACE_VERTICES_ARR[bnd[:, 1]]], axis=1)
        lookup = {tuple(t): int(b) for t, b in zip(old_tri.tolist(), mesh.boundary_faces[:, 2].tolist())}
        bnd = bnd.copy()
        bnd[:, 2] = [lookup.get(tuple(t), 0) for t in new_tri.tolist()]
    geom = mesh.geometry_nodes[order] if mesh.geometry_nodes is not None else None
    par = mesh.parent_cells[order] if mesh.parent_cells is not None else None
    return TetMesh(mesh.vertices.copy(), cells, interior, bnd, geom, par)


def apply_vertex_permutation(mesh: TetMesh, new_of_old: np.ndarray) -> TetMesh:
    """Vertex v is renumbered new_of_old[v] (cells keep their order and local vertex
    order, so orientation is unchanged); faces are rebuilt because their orientation
    codes follow global vertex ids (reference.py orientation_code), boundary ids are
    carried over by vertex triple.  The reference has no vertex renumbering; the CG DoF
    map of the result (vertex DoF = vertex id, dofmap.py:113-114) follows the new ids."""
    new_of_old = np.asarray(new_of_old, dtype=np.int64)
    nv = len(mesh.vertices)
    if new_of_old.shape != (nv,) or not np.array_equal(np.sort(new_of_old), np.arange(nv)):
        raise ValueError("new_of_old must be a permutation of the vertex ids")
    verts = np.empty_like(mesh.vertices)
    verts[new_of_old] = mesh.vertices
    cells = new_of_old[mesh.cells].astype(mesh.cells.dtype)
    interior, bnd = build_faces(cells)
    if len(bnd):
        old_tri = np.sort(new_of_old[mesh.cells[mesh.boundary_faces[:, 0, None],
                                                FACE_VERTICES_ARR[mesh.boundary_faces[:, 1]]]], axis=1)
        new_tri = np.sort(cells[bnd[:, 0, None], FACE_VERTICES_ARR[bnd[:, 1]]], axis=1)
        lookup = {tuple(t): int(b) for t, b in zip(old_tri.tolist(), mesh.boundary_faces[:, 2].tolist())}
        bnd = bnd.copy()
        bnd[:, 2] = [lookup.get(tuple(t), 0) for t in new_tri.tolist()]
    # curved geometry nodes are per-cell coordinates: unaffected by vertex ids
    return TetMesh(verts, cells, interior, bnd, mesh.geometry_nodes, mesh.parent_cells)


def first_touch_vertex_order(mesh: TetMesh) -> np.ndarray:
    """new_of_old for apply_vertex_permutation: vertices numbered in order of first
    appearance in the cell list (cell order, then local vertex order), so the vertices
    of consecutive cells get nearby ids.  Vertices no cell touches go last."""
    flat = mesh.cells.ravel()
    uniq, first = np.unique(flat, return_index=True)
    order = uniq[np.argsort(first, kind="stable")]
    nv = len(mesh.vertices)
    rest = np.setdiff1d(np.arange(nv), order, assume_unique=True)
    order = np.concatenate([order, rest])
    new_of_old = np.empty(nv, dtype=np.int64)
    new_of_old[order] = np.arange(nv)
    return new_of_old
