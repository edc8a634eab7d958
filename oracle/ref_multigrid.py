"""CPU restatement of the p-multigrid solver layer (TEST INFRASTRUCTURE ONLY: imported by
tests/, never by the product path).

The reference specifies the solver layer (Chebyshev
smoothing, p-transfers, CG with a multigrid preconditioner) but ships no code, so this is
the builder's restatement of the textbook algorithms, used as the checker for
paper_2509_10226_b200/multigrid.py ("parity unpinned" against the reference itself):

* global prolongation matrix: row f (fine DoF) = P_loc[i, :] scattered to the coarse
  DoFs of the FIRST cell containing f (any containing cell gives the same row up to
  rounding: the coarse function is continuous); Dirichlet rows / columns are zero;
* Chebyshev-Jacobi smoothing (Saad, Iterative Methods for Sparse Linear Systems,
  Alg. 12.1) on [lmax/range, lmax];
* V-cycle: pre-smooth from 0, residual, restrict (P^T), recurse, prolongate-add,
  post-smooth; coarsest level: fixed-count Jacobi-PCG (ref_apply.jacobi_pcg);
* flexible (Polak-Ribiere) PCG outer loop.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from .ref_apply import jacobi_pcg


def prolongation_matrix(fine_cell_dofs, coarse_cell_dofs, P_loc, n_fine, n_coarse,
                        fine_dirichlet=None, coarse_dirichlet=None):
    rows, cols, vals = [], [], []
    seen = np.zeros(n_fine, dtype=bool)
    fd = np.asarray(fine_cell_dofs)
    cd = np.asarray(coarse_cell_dofs)
    for e in range(fd.shape[0]):
        for i, f in enumerate(fd[e]):
            if seen[f]:
                continue
            seen[f] = True
            if fine_dirichlet is not None and fine_dirichlet[f]:
                continue
            for j, c in enumerate(cd[e]):
                if coarse_dirichlet is not None and coarse_dirichlet[c]:
                    continue
                if P_loc[i, j] != 0.0:
                    rows.append(f)
                    cols.append(c)
                    vals.append(P_loc[i, j])
    return sp.csr_matrix((vals, (rows, cols)), shape=(n_fine, n_coarse))


def lanczos_lmax(apply, diag, r0, iters):
    """Largest Ritz value of D^-1 A after ``iters`` Jacobi-PCG steps from r0 (the
    tridiagonal Lanczos matrix from the CG coefficients)."""
    r = r0.copy()
    z = r / diag
    p = z.copy()
    rz = float(r @ z)
    al, be = [], []
    for _ in range(iters):
        q = apply(p)
        pq = float(p @ q)
        if pq <= 0.0 or rz <= 0.0:
            break
        a = rz / pq
        r = r - a * q
        z = r / diag
        rz_new = float(r @ z)
        al.append(a)
        be.append(rz_new / rz)
        p = z + be[-1] * p
        rz = rz_new
    k = len(al)
    T = np.zeros((k, k))
    for j in range(k):
        T[j, j] = 1.0 / al[j] + (be[j - 1] / al[j - 1] if j else 0.0)
        if j + 1 < k:
            T[j, j + 1] = T[j + 1, j] = np.sqrt(be[j]) / al[j]
    return float(np.linalg.eigvalsh(T)[-1])


def chebyshev_coefficients(lmax, smoothing_range, degree):
    a, b = lmax / smoothing_range, lmax
    theta, delta = 0.5 * (b + a), 0.5 * (b - a)
    sigma = theta / delta
    rho = 1.0 / sigma
    out = [(0.0, 1.0 / theta)]
    for _ in range(1, degree):
        rho_new = 1.0 / (2.0 * sigma - rho)
        out.append((rho_new * rho, 2.0 * rho_new / delta))
        rho = rho_new
    return out


def chebyshev(apply, dinv, b, x, coeffs):
    """x = None: start from 0.  Returns the smoothed x."""
    d = None
    for k, (c1, c2) in enumerate(coeffs):
        if k == 0 and x is None:
            d = c2 * dinv * b
            x = d.copy()
            continue
        r = b - apply(x)
        d = c2 * dinv * r if d is None else c1 * d + c2 * dinv * r
        x = x + d
    return x


def vcycle(levels, transfers, b, coarse_iterations, i=0):
    """levels[i] = dict(apply, diag, coeffs); transfers[i] = CSR prolongation i+1 -> i."""
    lv = levels[i]
    if i == len(levels) - 1:
        x, _ = jacobi_pcg(lv["apply"], lv["diag"], b, coarse_iterations)
        return x
    dinv = 1.0 / lv["diag"]
    x = chebyshev(lv["apply"], dinv, b, None, lv["coeffs"])
    r = b - lv["apply"](x)
    xc = vcycle(levels, transfers, transfers[i].T @ r, coarse_iterations, i + 1)
    x = x + transfers[i] @ xc
    return chebyshev(lv["apply"], dinv, b, x, lv["coeffs"])


def flexible_pcg(apply, precond, b, tol, maxiter):
    x = np.zeros_like(b)
    r = b.copy()
    z = precond(r)
    p = z.copy()
    rz = float(r @ z)
    hist = [float(np.linalg.norm(r))]
    for _ in range(maxiter):
        if hist[-1] <= tol * hist[0]:
            break
        q = apply(p)
        alpha = rz / float(p @ q)
        x += alpha * p
        r -= alpha * q
        hist.append(float(np.linalg.norm(r)))
        z_new = precond(r)
        beta = float(r @ (z_new - z)) / rz
        rz = float(r @ z_new)
        z = z_new
        p = z + beta * p
    return x, np.array(hist)
