"""Simplex quadrature rules.

``QuadratureRule`` mirrors the reference dataclass (quadrature.py:30-46).  The
reference ships Witherden-Vincent-type orbit tables for p <= 3 only
(quadrature.py:72-101); BASELINE.json asks for Grundmann-Moller rules exact to
degree 2p for P1..P4, so this module generates those:

    Grundmann & Moeller (1978), n-simplex, degree d = 2s+1, i = 0..s:
      points  lambda_j = (2 beta_j + 1) / (d + n - 2i),  beta in N^{n+1}, |beta| = s - i
      weight  (-1)^i 2^{-2s} (d + n - 2i)^d / (i! (d + n - i)!)

The weights sum to 1/n! (the reference-simplex volume); coordinates drop
lambda_0 exactly as the reference does (quadrature.py:134).  s = p gives
n_q = 5/15/35/70 (tet) and n_qf = 4/10/20/35 (triangle) for p = 1..4.

Both rule families are fully symmetric under permutations of the barycentric
coordinates, which the DG face kernel relies on (plus-side tables are row
permutations of the code-0 tables, see :func:`symmetric_point_permutation`).
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass, field

import numpy as np

__all__ = ["QuadratureRule", "grundmann_moller", "make_cell_quadrature",
           "make_face_quadrature", "symmetric_point_permutation"]


@dataclass(frozen=True)
class QuadratureRule:
    points: np.ndarray          # (n_q, dim)
    weights: np.ndarray         # (n_q,)
    exactness_degree: int
    dim: int = field(default=3)

    @property
    def n_points(self) -> int:
        return len(self.weights)


def _compositions(total: int, parts: int):
    """All beta in N^parts with sum == total, in lexicographic order."""
    if parts == 1:
        yield (total,)
        return
    for first in range(total, -1, -1):
        for rest in _compositions(total - first, parts - 1):
            yield (first,) + rest


def grundmann_moller(s: int, dim: int) -> QuadratureRule:
    """Grundmann-Moller rule of degree 2s+1 on the unit ``dim``-simplex."""
    if s < 0:
        raise ValueError("s must be >= 0")
    d = 2 * s + 1
    n = dim
    pts, wts = [], []
    for i in range(s + 1):
        denom = d + n - 2 * i
        w = (-1.0) ** i * 2.0 ** (-2 * s) * float(denom) ** d / (
            math.factorial(i) * math.factorial(d + n - i))
        for beta in _compositions(s - i, n + 1):
            lam = [(2 * b + 1) / denom for b in beta]
            pts.append(lam[1:])
            wts.append(w)
    return QuadratureRule(np.asarray(pts, dtype=np.float64),
                          np.asarray(wts, dtype=np.float64), d, dim)


def make_cell_quadrature(p: int, variant: str = "standard") -> QuadratureRule:
    """Tet rule exact to 2p ("standard") or 2p-2 ("modified"; degree >= 1)."""
    if p not in (1, 2, 3, 4):
        raise ValueError(f"unsupported polynomial degree {p}")
    if variant == "standard":
        need = 2 * p
    elif variant == "modified":
        need = max(2 * p - 2, 1)
    else:
        raise ValueError(f"unknown quadrature variant {variant!r}")
    return grundmann_moller(need // 2, 3)   # degree 2s+1 >= need


def make_face_quadrature(p: int) -> QuadratureRule:
    """Triangle rule exact to 2p for the face terms."""
    if p not in (1, 2, 3, 4):
        raise ValueError(f"unsupported polynomial degree {p}")
    return grundmann_moller(p, 2)


def symmetric_point_permutation(points2d: np.ndarray, perm) -> np.ndarray | None:
    """Index map ``pi`` with bary(points[q]) permuted by ``perm`` == bary(points[pi[q]]).

    Returns None when the rule is not invariant under ``perm``.
    """
    s, t = points2d[:, 0], points2d[:, 1]
    bary = np.stack([1.0 - s - t, s, t], axis=1)
    moved = np.empty_like(bary)
    moved[:, list(perm)] = bary
    out = np.empty(len(bary), dtype=np.int64)
    for q in range(len(bary)):
        dist = np.abs(bary - moved[q]).max(axis=1)
        k = int(np.argmin(dist))
        if dist[k] > 1e-12:
            return None
        out[q] = k
    return out


def monomial_exactness(rule: QuadratureRule) -> int:
    """Largest total degree integrated exactly (rel. 1e-12); for tests."""
    deg = 0
    while deg < 20:
        ok = True
        for exps in itertools.product(range(deg + 2), repeat=rule.dim):
            if sum(exps) != deg + 1:
                continue
            num = np.sum(rule.weights * np.prod(rule.points ** np.array(exps), axis=1))
            exact = math.prod(math.factorial(e) for e in exps) / math.factorial(sum(exps) + rule.dim)
            if abs(num - exact) > 1e-12 * max(1.0, abs(exact)):
                ok = False
                break
        if not ok:
            return deg
        deg += 1
    return deg
