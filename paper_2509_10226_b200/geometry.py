"""Geometry container mirroring the reference ``GeometryData`` (geometry.py:31-74).

The plan computes every geometric factor itself from the vertex coordinates, once, at plan
creation (``cell_geometry_kernel`` / ``face_geometry_kernel``: 64-byte cell records G = det J
J^-1 J^-T and the mass factor, and the face records; the P1 block kernel recomputes G from
staged vertices instead), so the only fields the operators read from this container are
``mode`` (must be "affine") and the quadrature rules.  :func:`build_geometry`
still fills the affine arrays (vectorised restatement of geometry.py:145-151,
202-240, with the reference's compact per-face storage) so that code written
against the reference (e.g. ``compute_sipg_tau``) keeps working.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .mesh import TetMesh
from .quadrature import QuadratureRule
from .reference import FACE_VERTICES_ARR, REF_VERTICES

__all__ = ["GeometryData", "build_geometry", "AFFINE", "PER_POINT"]

AFFINE = "affine"
PER_POINT = "per_point"


@dataclass
class GeometryData:
    mode: str
    cell_rule: QuadratureRule
    face_rule: QuadratureRule | None
    jac_inv_t: np.ndarray
    jxw: np.ndarray
    det: np.ndarray | None
    cell_volumes: np.ndarray
    face_normals: np.ndarray | None = None
    face_jxw: np.ndarray | None = None
    face_m_minus: np.ndarray | None = None
    face_m_plus: np.ndarray | None = None
    face_areas: np.ndarray | None = None
    bnd_normals: np.ndarray | None = None
    bnd_jxw: np.ndarray | None = None
    bnd_m: np.ndarray | None = None
    bnd_areas: np.ndarray | None = None

    @property
    def n_cells(self) -> int:
        return len(self.jxw)

    @property
    def is_affine(self) -> bool:
        return self.mode == AFFINE


def _face_block(mesh: TetMesh, jac, c_minus, lf_minus, w, c_plus=None):
    jm = jac[c_minus]
    corners = REF_VERTICES[FACE_VERTICES_ARR[lf_minus]]
    t_s = np.einsum("fij,fj->fi", jm, corners[:, 1] - corners[:, 0])
    t_t = np.einsum("fij,fj->fi", jm, corners[:, 2] - corners[:, 0])
    cr = np.cross(t_s, t_t)
    norm = np.linalg.norm(cr, axis=1)
    n = cr / norm[:, None]
    opp = mesh.vertices[mesh.cells[c_minus, lf_minus]]
    fv0 = mesh.vertices[mesh.cells[c_minus, FACE_VERTICES_ARR[lf_minus, 0]]]
    n *= np.where(np.einsum("fi,fi->f", n, fv0 - opp) < 0, -1.0, 1.0)[:, None]
    sjxw = norm[:, None] * w[None, :]
    m_minus = np.linalg.solve(jm, n[..., None])[..., 0]
    m_plus = None if c_plus is None else np.linalg.solve(jac[c_plus], n[..., None])[..., 0]
    return n, sjxw, m_minus, m_plus, sjxw.sum(axis=1)


def build_geometry(mesh: TetMesh, cell_rule: QuadratureRule, mode: str = AFFINE,
                   face_rule: QuadratureRule | None = None) -> GeometryData:
    if mode not in (AFFINE, PER_POINT):
        raise ValueError(f"unknown geometry mode {mode!r}")
    if mode != AFFINE or getattr(mesh, "is_curved", False):
        raise ValueError("the B200 operators support straight-sided (affine) cells only")
    jac = mesh.cell_jacobians()
    det = np.linalg.det(jac)
    bad = np.flatnonzero(det <= 0)
    if len(bad):
        raise ValueError(f"non-positive Jacobian determinant in cell geometry for cells {bad[:20].tolist()}")
    geo = GeometryData(mode, cell_rule, face_rule, np.transpose(np.linalg.inv(jac), (0, 2, 1)),
                       det[:, None] * cell_rule.weights[None, :], det, det / 6.0)
    if face_rule is not None:
        w = face_rule.weights
        f = mesh.interior_faces.astype(np.int64)
        n, s, mm, mp, a = _face_block(mesh, jac, f[:, 0], f[:, 1], w, f[:, 2])
        geo.face_normals, geo.face_jxw, geo.face_m_minus, geo.face_m_plus, geo.face_areas = n, s, mm, mp, a
        b = mesh.boundary_faces.astype(np.int64)
        n, s, m, _, a = _face_block(mesh, jac, b[:, 0], b[:, 1], w)
        geo.bnd_normals, geo.bnd_jxw, geo.bnd_m, geo.bnd_areas = n, s, m, a
    return geo
