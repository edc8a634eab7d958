"""Reference-tetrahedron conventions (local numbering, face orientation codes).

Mirrors the conventions of the reference package so that integer data (DoF maps,
face lists, orientation codes) is bit-identical:

* vertices (0,0,0), (1,0,0), (0,1,0), (0,0,1)          -- reference.py:19-23
* local face f is opposite local vertex f, corners ascending -- reference.py:25-26
* local edge order                                        -- reference.py:28-29
* the six triangle symmetries; code o means
  ``minus[k] == plus[PERMS[o][k]]`` in global vertex ids  -- reference.py:31-48
* triangle point (s,t) -> barycentrics (1-s-t, s, t) in minus-side corner
  order, permuted onto the plus side by the code          -- reference.py:66-81
"""

from __future__ import annotations

import numpy as np

REF_VERTICES = np.array([[0.0, 0.0, 0.0],
                         [1.0, 0.0, 0.0],
                         [0.0, 1.0, 0.0],
                         [0.0, 0.0, 1.0]])
REF_VOLUME = 1.0 / 6.0

FACE_VERTICES = ((1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2))
EDGE_VERTICES = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))
PERMS = ((0, 1, 2), (1, 2, 0), (2, 0, 1), (0, 2, 1), (2, 1, 0), (1, 0, 2))
N_ORIENTATIONS = 6

FACE_VERTICES_ARR = np.array(FACE_VERTICES, dtype=np.int64)
EDGE_VERTICES_ARR = np.array(EDGE_VERTICES, dtype=np.int64)
PERMS_ARR = np.array(PERMS, dtype=np.int64)

# local edges lying inside each local face (used by Dirichlet masking)
FACE_EDGES = tuple(
    tuple(e for e, (a, b) in enumerate(EDGE_VERTICES) if a in fv and b in fv)
    for fv in FACE_VERTICES)


def orientation_code(minus_triple, plus_triple) -> int:
    """Code ``o`` with ``minus_triple[k] == plus_triple[PERMS[o][k]]``."""
    m = tuple(int(v) for v in minus_triple)
    for o, p in enumerate(PERMS):
        if tuple(int(plus_triple[p[k]]) for k in range(3)) == m:
            return o
    raise ValueError(f"face corner sets differ: {minus_triple} vs {plus_triple}")


def orientation_codes(minus: np.ndarray, plus: np.ndarray) -> np.ndarray:
    """Vectorised :func:`orientation_code` over (F, 3) corner arrays."""
    codes = np.full(len(minus), -1, dtype=np.int64)
    for o, p in enumerate(PERMS):
        hit = np.all(plus[:, list(p)] == minus, axis=1) & (codes < 0)
        codes[hit] = o
    if len(codes) and codes.min() < 0:
        bad = int(np.flatnonzero(codes < 0)[0])
        raise ValueError(f"face corner sets differ: {minus[bad]} vs {plus[bad]}")
    return codes


def face_quad_points(local_face: int, code: int, pts2d: np.ndarray) -> np.ndarray:
    """Reference-tet coordinates of triangle points on ``local_face`` seen with
    orientation ``code`` (minus side uses code 0)."""
    s, t = pts2d[:, 0], pts2d[:, 1]
    bary = np.stack([1.0 - s - t, s, t], axis=1)
    side = np.empty_like(bary)
    side[:, list(PERMS[code])] = bary
    return side @ REF_VERTICES[list(FACE_VERTICES[local_face])]
