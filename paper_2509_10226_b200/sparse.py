"""Matrix-based baseline on the GPU: CSR assembly + cuSPARSE SpMV.

Mirrors the reference's ``sparse.assemble`` / ``CsrMatrix.matvec``
(sparse.py:173-230, :225-228), which the reference uses as the oracle and as
the throughput baseline of the paper's matrix-free vs sparse-matrix comparison
(PAPER.md:300-309).  SURVEY §8f row 3: this is the "next" row, a baseline, not
the product path -- the SpMV is a plain library call (torch -> cuSPARSE).

CG Laplace: element matrices K_e = sum_kl G_kl(e) S_kl with the reference
stiffness tensors S_kl[a, b] = sum_q w_q dphi_a/dxi_k dphi_b/dxi_l (exactly the
quadrature sum of sparse._cell_matrices, reorganised) and
G = det J J^-1 J^-T; Dirichlet rows/columns are replaced by identity
(sparse.py:210-217).
"""

from __future__ import annotations

import numpy as np

__all__ = ["CsrOperator", "assemble_cg_csr"]


def _metric(vertices, cells):
    v = vertices[cells]
    J = np.stack([v[:, 1] - v[:, 0], v[:, 2] - v[:, 0], v[:, 3] - v[:, 0]], axis=2)
    det = np.linalg.det(J)
    inv = np.linalg.inv(J)
    G = det[:, None, None] * inv @ np.transpose(inv, (0, 2, 1))
    return G


def assemble_cg_csr(mesh, dofmap, geometry, basis, device="cuda", kappa=None):
    """torch sparse CSR matrix (fp64, on ``device``) of the CG Laplace operator
    (``kappa``: per-cell coefficient, -div(kappa grad u))."""
    import torch

    nq = len(geometry.cell_rule.weights)
    nd = dofmap.cell_dofs.shape[1]
    w = np.asarray(geometry.cell_rule.weights)
    Eg = np.asarray(basis.grad_matrix).reshape(nq, 3, nd)
    S = np.einsum("q,qka,qlb->klab", w, Eg, Eg).reshape(9, nd * nd)            # (9, nd^2)
    Gn = _metric(mesh.vertices, mesh.cells).reshape(-1, 9)
    if kappa is not None:
        Gn = Gn * np.asarray(kappa, dtype=np.float64)[:, None]
    G = torch.from_numpy(Gn).to(device)
    Ke = G @ torch.from_numpy(S).to(device)                                      # (n_cells, nd^2)
    cd = torch.from_numpy(dofmap.cell_dofs.astype(np.int64)).to(device)
    rows = cd[:, :, None].expand(-1, nd, nd).reshape(-1)
    cols = cd[:, None, :].expand(-1, nd, nd).reshape(-1)
    vals = Ke.reshape(-1)
    n = dofmap.n_scalar_dofs
    mask = np.asarray(dofmap.dirichlet_mask, dtype=bool)
    if mask.any():
        m = torch.from_numpy(mask).to(device)
        keep = ~(m[rows] | m[cols])
        rows, cols, vals = rows[keep], cols[keep], vals[keep]
        c = torch.from_numpy(np.flatnonzero(mask)).to(device)
        rows = torch.cat([rows, c])
        cols = torch.cat([cols, c])
        vals = torch.cat([vals, torch.ones(len(c), dtype=vals.dtype, device=device)])
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        A = torch.sparse_coo_tensor(torch.stack([rows, cols]), vals, (n, n), check_invariants=False).coalesce()
        return A.to_sparse_csr()


class CsrOperator:
    """y = A u with an assembled CSR matrix (cuSPARSE through torch)."""

    def __init__(self, mesh, dofmap, geometry, basis, device="cuda"):
        if dofmap.space != "cg" or dofmap.n_components != 1:
            raise ValueError("the CSR baseline covers the scalar CG operator")
        self.A = assemble_cg_csr(mesh, dofmap, geometry, basis, device)
        self.nnz = int(self.A.values().numel())
        self.n = dofmap.n_scalar_dofs

    @property
    def nbytes(self) -> int:
        """reference CsrMatrix.nbytes accounting (sparse.py:52-53) with int32 columns."""
        return 12 * self.nnz + 8 * (self.n + 1)

    def apply(self, u):
        import torch

        if isinstance(u, np.ndarray):
            return (self.A @ torch.from_numpy(u).to(self.A.device).unsqueeze(1)).squeeze(1).cpu().numpy()
        return (self.A @ u.unsqueeze(1)).squeeze(1)
