"""Global DoF enumeration and Dirichlet masks (CG and DG).

``DoFMap`` mirrors dofmap.py:41-64.  :func:`build_dof_map` is a vectorised,
bit-identical restatement of dofmap.py:67-144 for p <= 3:

* vertex DoF = global vertex id (dofmap.py:113-114);
* edge ids by first encounter over (cell, local edge in EDGE_VERTICES order),
  keyed by the sorted global pair; edge DoF = ``n_v + (p-1)*eid + k`` with
  ``k = slot`` if the local endpoints are in ascending global order else
  ``p-2-slot`` (dofmap.py:93-97, 115-120);
* face ids by a separate, later first-encounter pass (dofmap.py:98-102);
  face DoF = ``face_base + fid`` (dofmap.py:121-123);
* Dirichlet mask = closure of the selected boundary faces (dofmap.py:125-142);
* DG: ``cell_dofs[e] = e*n_dpc + [0..n_dpc)`` with no mask (dofmap.py:84-88).

P4 (no reference): 3 face DoFs per face at
``face_base + 3*fid + rank(global id of local corner j)`` and one interior DoF
``interior_base + e`` with ``interior_base = face_base + 3*n_faces``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .basis import n_dofs_per_cell, reference_nodes
from .mesh import TetMesh
from .reference import EDGE_VERTICES_ARR, FACE_VERTICES_ARR

__all__ = ["DoFMap", "build_dof_map", "face_local_dofs", "first_encounter_ids", "dof_coordinates"]

CG = "cg"
DG = "dg"


@dataclass
class DoFMap:
    space: str
    degree: int
    n_components: int
    n_scalar_dofs: int
    cell_dofs: np.ndarray           # (n_cells, n_dpc) int32
    dirichlet_mask: np.ndarray      # (n_scalar_dofs,) bool

    @property
    def n_global_dofs(self) -> int:
        return self.n_scalar_dofs * self.n_components

    @property
    def n_dofs_per_cell(self) -> int:
        return self.cell_dofs.shape[1]

    @property
    def n_cells(self) -> int:
        return self.cell_dofs.shape[0]

    def vector_mask(self) -> np.ndarray:
        return np.repeat(self.dirichlet_mask, self.n_components)


def first_encounter_ids(keys: np.ndarray):
    """Number unique rows of ``keys`` (K, m) in order of first appearance.

    Returns (ids (K,), n_unique)."""
    keys = np.ascontiguousarray(keys)
    if keys.ndim == 1:
        keys = keys[:, None]
    order = np.lexsort(tuple(keys[:, c] for c in range(keys.shape[1] - 1, -1, -1)))
    ks = keys[order]
    new = np.ones(len(ks), dtype=bool)
    new[1:] = np.any(ks[1:] != ks[:-1], axis=1)
    group = np.cumsum(new) - 1                      # sorted-unique index per sorted row
    first_pos = np.empty(int(new.sum()), dtype=np.int64)
    # lexsort is stable, so the first row of each group is the earliest occurrence
    first_pos[:] = order[new]
    rank = np.empty_like(first_pos)
    rank[np.argsort(first_pos, kind="stable")] = np.arange(len(first_pos))
    ids = np.empty(len(keys), dtype=np.int64)
    ids[order] = rank[group]
    return ids, len(first_pos)


def face_local_dofs(p: int) -> list[np.ndarray]:
    """Local DoF indices lying on the closure of each local face."""
    _, tags = reference_nodes(p)
    from .reference import FACE_EDGES, FACE_VERTICES
    out = []
    for f in range(4):
        sel = [j for j, (kind, ent, _) in enumerate(tags)
               if (kind == "v" and ent in FACE_VERTICES[f])
               or (kind == "e" and ent in FACE_EDGES[f])
               or (kind == "f" and ent == f)]
        out.append(np.array(sel, dtype=np.int64))
    return out


def _cg_dofs_native(cells: np.ndarray, n_vertices: int, p: int):
    import ctypes as C

    from . import _lib

    c = np.ascontiguousarray(cells, dtype=np.int32)
    out = np.empty((len(c), n_dofs_per_cell(p)), dtype=np.int32)
    ns = C.c_int64()
    _lib.check(_lib.lib().tmf_build_cg_dofs(len(c), _lib.ptr(c, C.c_int32), int(n_vertices), int(p),
                                            _lib.ptr(out, C.c_int32), C.byref(ns)))
    return out, int(ns.value)


def build_dof_map(mesh: TetMesh, p: int, space: str, n_components: int = 1,
                  dirichlet_boundary_ids=(), method: str = "native") -> DoFMap:
    """``method``: "native" (C++ bucket sort, csrc/setup.cpp) or "numpy" (vectorised);
    both bit-identical to the reference numbering."""
    if space not in (CG, DG):
        raise ValueError(f"unknown space {space!r}")
    if n_components not in (1, 3):
        raise ValueError("n_components must be 1 or 3")
    known = set(int(b) for b in mesh.boundary_faces[:, 2]) if len(mesh.boundary_faces) else set()
    for bid in dirichlet_boundary_ids:
        if bid not in known:
            raise ValueError(f"unknown boundary id {bid} (mesh has {sorted(known)})")
    nd = n_dofs_per_cell(p)
    n = mesh.n_cells
    if space == DG:
        cell_dofs = np.arange(n * nd, dtype=np.int32).reshape(n, nd)
        return DoFMap(DG, p, n_components, n * nd, cell_dofs, np.zeros(n * nd, dtype=bool))

    if method == "native":
        cell_dofs, n_scalar = _cg_dofs_native(mesh.cells, mesh.n_vertices, p)
        return DoFMap(CG, p, n_components, n_scalar, cell_dofs,
                      _dirichlet_mask(mesh, p, cell_dofs, n_scalar, dirichlet_boundary_ids))
    if method != "numpy":
        raise ValueError(f"unknown method {method!r}")
    cells = mesh.cells.astype(np.int64)
    _, tags = reference_nodes(p)
    per_edge = p - 1
    edge_base = mesh.n_vertices
    n_edges = 0
    if p >= 2:
        ev = cells[:, EDGE_VERTICES_ARR]                    # (n, 6, 2) in (cell, local edge) order
        lo, hi = ev.min(axis=2).reshape(-1), ev.max(axis=2).reshape(-1)
        edge_id, n_edges = first_encounter_ids(np.stack([lo, hi], axis=1))
        edge_id = edge_id.reshape(n, 6)
        ascending = ev[:, :, 0] < ev[:, :, 1]
    face_base = edge_base + per_edge * n_edges
    n_faces = 0
    if p >= 3:
        fv = cells[:, FACE_VERTICES_ARR]                    # (n, 4, 3)
        face_id, n_faces = first_encounter_ids(np.sort(fv, axis=2).reshape(-1, 3))
        face_id = face_id.reshape(n, 4)
    per_face = {3: 1, 4: 3}.get(p, 0)
    interior_base = face_base + per_face * n_faces
    n_scalar = interior_base + (n if p >= 4 else 0)

    cell_dofs = np.empty((n, nd), dtype=np.int64)
    for j, (kind, ent, slot) in enumerate(tags):
        if kind == "v":
            cell_dofs[:, j] = cells[:, ent]
        elif kind == "e":
            k = np.where(ascending[:, ent], slot, per_edge - 1 - slot)
            cell_dofs[:, j] = edge_base + per_edge * edge_id[:, ent] + k
        elif kind == "f":
            if p == 3:
                cell_dofs[:, j] = face_base + face_id[:, ent]
            else:
                corners = fv[:, ent]                          # (n, 3) global ids, local order
                rank = (corners < corners[:, slot, None]).sum(axis=1)
                cell_dofs[:, j] = face_base + 3 * face_id[:, ent] + rank
        else:
            cell_dofs[:, j] = interior_base + np.arange(n)
    if n_scalar >= 2 ** 31:
        raise ValueError("DoF count exceeds int32 indexing")

    cell_dofs = cell_dofs.astype(np.int32)
    return DoFMap(CG, p, n_components, int(n_scalar), cell_dofs,
                  _dirichlet_mask(mesh, p, cell_dofs, n_scalar, dirichlet_boundary_ids))


def _dirichlet_mask(mesh, p, cell_dofs, n_scalar, dirichlet_boundary_ids):
    """Closure of the selected boundary faces (dofmap.py:125-142)."""
    mask = np.zeros(n_scalar, dtype=bool)
    if len(dirichlet_boundary_ids) and len(mesh.boundary_faces):
        bf = mesh.boundary_faces
        sel = np.isin(bf[:, 2], np.array(list(dirichlet_boundary_ids), dtype=np.int64))
        fl = face_local_dofs(p)
        for lf in range(4):
            rows = bf[sel & (bf[:, 1] == lf), 0]
            mask[cell_dofs[rows[:, None], fl[lf][None, :]].reshape(-1)] = True
    return mask


def dof_coordinates(mesh: TetMesh, dofmap: DoFMap, ref_nodes: np.ndarray) -> np.ndarray:
    """Physical coordinates of the scalar DoFs (dofmap.py:295-303, vectorised)."""
    v = mesh.vertices[mesh.cells]
    jac = np.stack([v[:, 1] - v[:, 0], v[:, 2] - v[:, 0], v[:, 3] - v[:, 0]], axis=2)
    phys = v[:, 0][:, None, :] + np.einsum("eij,aj->eai", jac, ref_nodes)
    coords = np.empty((dofmap.n_scalar_dofs, 3))
    coords[dofmap.cell_dofs.reshape(-1)] = phys.reshape(-1, 3)
    return coords
