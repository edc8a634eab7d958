"""Nodal Lagrange bases on the reference tetrahedron and their tabulation.

Mirrors the reference's ``BasisTable``/``tabulate_basis`` (basis.py:92-174):
value table (n_q, n_dofs), gradient table (3 n_q, n_dofs) with row ``3*i + k``
(basis.py:155), face tables per (local face, orientation code) of shape
(4, 6, n_qf, n_dofs) and (4, 6, 3 n_qf, n_dofs) (basis.py:159-166).

Node order follows basis.py:48-69 -- vertices, then p-1 equispaced nodes per
edge in EDGE_VERTICES order counted from the lower local endpoint, then (p=3)
face centroids.  The reference stops at p=3 (basis.py:146); P4 is this
package's documented extension: 3 nodes per face at
barycentrics (1/2,1/4,1/4) and permutations (slot j = node nearest local face
corner j), then one interior node at the centroid.  Shape functions are the
monomial basis times the inverse nodal Vandermonde matrix.

These tables are host-side setup; the GPU consumes them through the C-ABI.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .quadrature import QuadratureRule
from .reference import EDGE_VERTICES, FACE_VERTICES, N_ORIENTATIONS, REF_VERTICES, face_quad_points

__all__ = ["BasisTable", "tabulate_basis", "n_dofs_per_cell", "reference_nodes",
           "lagrange_values", "lagrange_grads"]

MAX_DEGREE = 4


def n_dofs_per_cell(p: int) -> int:
    return (p + 1) * (p + 2) * (p + 3) // 6


def _exponents(p: int):
    out = []
    for d in range(p + 1):
        for a in range(d, -1, -1):
            for b in range(d - a, -1, -1):
                out.append((a, b, d - a - b))
    return out


def reference_nodes(p: int):
    """(nodes (n_dofs, 3), tags).  Tags: ("v", vertex, 0), ("e", edge, slot),
    ("f", face, slot), ("c", 0, 0)."""
    if p < 1 or p > MAX_DEGREE:
        raise ValueError(f"unsupported polynomial degree {p}")
    nodes = [REF_VERTICES[i].copy() for i in range(4)]
    tags = [("v", i, 0) for i in range(4)]
    for e, (a, b) in enumerate(EDGE_VERTICES):
        for k in range(p - 1):
            t = (k + 1) / p
            nodes.append((1.0 - t) * REF_VERTICES[a] + t * REF_VERTICES[b])
            tags.append(("e", e, k))
    if p == 3:
        for f, corners in enumerate(FACE_VERTICES):
            nodes.append(REF_VERTICES[list(corners)].mean(axis=0))
            tags.append(("f", f, 0))
    elif p == 4:
        for f, corners in enumerate(FACE_VERTICES):
            cv = REF_VERTICES[list(corners)]
            for j in range(3):
                bary = np.full(3, 0.25)
                bary[j] = 0.5
                nodes.append(bary @ cv)
                tags.append(("f", f, j))
        nodes.append(REF_VERTICES.mean(axis=0))
        tags.append(("c", 0, 0))
    return np.array(nodes), tags


def _mono(points: np.ndarray, exps) -> np.ndarray:
    x, y, z = points[:, 0], points[:, 1], points[:, 2]
    return np.stack([x ** a * y ** b * z ** c for a, b, c in exps], axis=1)


def _mono_grad(points: np.ndarray, exps) -> np.ndarray:
    """(n_pts, 3, n_mono)."""
    x, y, z = points[:, 0], points[:, 1], points[:, 2]
    out = np.zeros((len(points), 3, len(exps)))
    for j, (a, b, c) in enumerate(exps):
        if a:
            out[:, 0, j] = a * x ** (a - 1) * y ** b * z ** c
        if b:
            out[:, 1, j] = b * x ** a * y ** (b - 1) * z ** c
        if c:
            out[:, 2, j] = c * x ** a * y ** b * z ** (c - 1)
    return out


def _coeffs(p: int) -> np.ndarray:
    nodes, _ = reference_nodes(p)
    return np.linalg.inv(_mono(nodes, _exponents(p)))


def lagrange_values(p: int, points: np.ndarray) -> np.ndarray:
    return _mono(points, _exponents(p)) @ _coeffs(p)


def lagrange_grads(p: int, points: np.ndarray) -> np.ndarray:
    """(n_pts, 3, n_dofs)."""
    return _mono_grad(points, _exponents(p)) @ _coeffs(p)


@dataclass
class BasisTable:
    degree: int
    nodes: np.ndarray
    node_tags: list
    cell_rule: QuadratureRule
    face_rule: QuadratureRule
    value_matrix: np.ndarray      # (n_q, n_dofs)
    grad_matrix: np.ndarray       # (3 n_q, n_dofs), row 3*i + k
    face_values: np.ndarray       # (4, 6, n_qf, n_dofs)
    face_grads: np.ndarray        # (4, 6, 3 n_qf, n_dofs)

    @property
    def n_dofs(self) -> int:
        return self.nodes.shape[0]

    @property
    def n_q(self) -> int:
        return self.value_matrix.shape[0]

    @property
    def n_qf(self) -> int:
        return self.face_values.shape[2]


def tabulate_basis(p: int, cell_rule: QuadratureRule, face_rule: QuadratureRule) -> BasisTable:
    nodes, tags = reference_nodes(p)
    exps = _exponents(p)
    coeffs = np.linalg.inv(_mono(nodes, exps))
    nd = len(nodes)
    values = _mono(cell_rule.points, exps) @ coeffs
    grads = (_mono_grad(cell_rule.points, exps) @ coeffs).reshape(3 * cell_rule.n_points, nd)
    nqf = face_rule.n_points
    fv = np.empty((4, N_ORIENTATIONS, nqf, nd))
    fg = np.empty((4, N_ORIENTATIONS, 3 * nqf, nd))
    for f in range(4):
        for o in range(N_ORIENTATIONS):
            pts = face_quad_points(f, o, face_rule.points)
            fv[f, o] = _mono(pts, exps) @ coeffs
            fg[f, o] = (_mono_grad(pts, exps) @ coeffs).reshape(3 * nqf, nd)
    return BasisTable(p, nodes, tags, cell_rule, face_rule, values, grads, fv, fg)
