"""p-multigrid preconditioned CG on the matrix-free operators.

The paper's solver layer is the main consumer of
the apply; the reference package specifies it but ships no implementation.  This is
the fp64 p-multigrid part of it, built on the B200 operator apply:

* levels: CG spaces of decreasing degree on the same mesh (default p, p-1, ..., 1),
  each a :class:`CgPoissonOperator` with its matrix-free diagonal;
* transfers: ``tmf_prolongate`` / ``tmf_restrict`` (interpolation of the coarse
  function at the fine nodes and its exact transpose, csrc/multigrid.cu);
* smoother: Chebyshev-accelerated point Jacobi of degree ``smoothing_degree`` (default 2:
  fastest to 1e-8 on the C5 problem among 2 / 3 / 4, tools/mg_sweep.py) on
  [lambda_max / smoothing_range, lambda_max] (Saad, Iterative Methods, Alg. 12.1;
  fused update ``tmf_chebyshev_step``); lambda_max of D^-1 A from a short Lanczos
  (Jacobi-PCG coefficients) times 1.1;
* optional DG finest level (``fine_operator``) over the CG levels via a c-transfer (DG p ->
  CG p, "transferred to an auxiliary continuous space"), smoothed with the
  exact DG diagonal probed by colouring (:func:`dg_diagonal`);
* coarse level (P1): ``coarse_iterations`` native Jacobi-PCG iterations (``tmf_pcg``);
* outer loop: flexible (Polak-Ribiere) PCG, since a fixed-count inner CG makes the
  V-cycle slightly nonlinear.

``precision="mixed"``: the whole V-cycle in fp32 (``tmf_apply_f32``: the modal cell form on
FFMA, fp32 transfers / Chebyshev steps / coarse Jacobi-PCG) inside the fp64 flexible PCG,
as the paper does ("the multigrid V-cycle runs in single precision").

``h_coarse=(n1, n2, ...)``: h-levels below the fine-mesh P1 level on unjittered Kuhn meshes of
the unit cube with n1 > n2 > ... cubes per side (non-nested: the BASELINE meshes are jittered, not
refinements), linked by point transfers (``tmf_transfer_create_points``: each fine vertex takes
the coarse P1 function at its position).

Not built (out of scope this round): Chebyshev on the coarse level, refinement genealogies.  No CPU fallback: every vector operation
is a native kernel or a device tensor op; the CPU restatement is
``oracle/ref_multigrid.py`` (tests only).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import basis as B
from . import dofmap as D
from . import quadrature as Q
from .geometry import GeometryData

__all__ = ["interpolation_matrix", "Transfer", "PointTransfer", "kuhn_point_weights", "PMultigrid",
           "chebyshev_coefficients", "color_cells",
           "dg_diagonal", "n10"]


def interpolation_matrix(p_fine: int, p_coarse: int) -> np.ndarray:
    """(n_fine_dpc, n_coarse_dpc): coarse Lagrange basis at the fine reference nodes;
    entries below 1e-13 (where a coarse function vanishes at a fine node) are exact 0."""
    if not 1 <= p_coarse < p_fine <= B.MAX_DEGREE:
        raise ValueError(f"need 1 <= p_coarse < p_fine <= {B.MAX_DEGREE}")
    nodes, _ = B.reference_nodes(p_fine)
    P = B.lagrange_values(p_coarse, nodes)
    P[np.abs(P) < 1e-13] = 0.0
    return np.ascontiguousarray(P)


def color_cells(mesh):
    """Greedy face-adjacency colouring of the cells (``tmf_color_cells``): (colors, n_colors)."""
    f = np.ascontiguousarray(mesh.interior_faces, dtype=np.int32)
    col = np.empty(mesh.n_cells, dtype=np.int32)
    nc = C.c_int32()
    rc = _lib.lib().tmf_color_cells(mesh.n_cells, len(f), _lib.ptr(f, C.c_int32), _lib.ptr(col, C.c_int32),
                                    C.byref(nc))
    if rc != _lib.TMF_OK:
        raise ValueError("bad interior-face table")
    return col, int(nc.value)


def dg_diagonal(A, mesh, stream: int = 0):
    """Exact diagonal of a DG operator (a device tensor): cells of one colour share no face,
    so applying A to the indicator of local DoF j on all cells of a colour returns their
    diagonal entries at those positions (n_colours x n_dofs_per_cell applies)."""
    import torch

    N = A.dofmap.n_dofs_per_cell
    nc_ = int(A.dofmap.n_components)
    col, ncol = color_cells(mesh)
    dev = torch.device(f"cuda:{A.config.device}")
    n = A.n_global_dofs
    diag = torch.empty(n, dtype=torch.float64, device=dev)
    u = torch.zeros(n, dtype=torch.float64, device=dev)
    y = torch.empty_like(u)
    # every probe (torch writes of u, the apply, torch reads of y) runs on ONE stream: the
    # caller's ``stream`` if given (made torch's current stream for the loop), else torch's own
    ext = torch.cuda.ExternalStream(stream, device=dev) if stream else torch.cuda.current_stream(dev)
    with torch.cuda.stream(ext):
        for c in range(ncol):
            cells = torch.from_numpy(np.nonzero(col == c)[0].astype(np.int64)).to(dev)
            for j in range(N):
                for k in range(nc_):
                    idx = (cells * N + j) * nc_ + k
                    u.zero_()
                    u[idx] = 1.0
                    A.apply_into(u.data_ptr(), y.data_ptr(), ext.cuda_stream)
                    diag[idx] = y[idx]
    return diag


def chebyshev_coefficients(lmax: float, smoothing_range: float, degree: int):
    """[(c1, c2)] per step of the Chebyshev-Jacobi iteration on [lmax/range, lmax]:
    step k: d = c1 d + c2 D^-1 (b - A x), x += d (step 0: c1 = 0)."""
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


def _vp(t):
    return C.c_void_p(t.data_ptr())


class Transfer:
    """Degree transfer between two CG dof maps on the same mesh (device resident)."""

    def __init__(self, fine_dm, coarse_dm, device: int = 0):
        if fine_dm.n_cells != coarse_dm.n_cells:
            raise ValueError("fine and coarse dof maps must live on the same mesh")
        if fine_dm.space == "dg" and coarse_dm.space == "cg" and fine_dm.degree == coarse_dm.degree:
            self.P = np.eye(fine_dm.n_dofs_per_cell)          # c-transfer: DG p -> CG p
        elif fine_dm.space == "cg" and coarse_dm.space == "cg":
            self.P = interpolation_matrix(fine_dm.degree, coarse_dm.degree)
        else:
            raise ValueError("transfers are CG p -> CG q < p, or DG p -> CG p")
        fd = np.ascontiguousarray(fine_dm.cell_dofs, dtype=np.int32)
        cd = np.ascontiguousarray(coarse_dm.cell_dofs, dtype=np.int32)
        fm = np.ascontiguousarray(fine_dm.dirichlet_mask, dtype=np.uint8)
        cm = np.ascontiguousarray(coarse_dm.dirichlet_mask, dtype=np.uint8)
        d = _lib.TransferDesc()
        d.n_cells = fine_dm.n_cells
        d.n_fine_dpc, d.n_coarse_dpc = fd.shape[1], cd.shape[1]
        d.n_fine_dofs, d.n_coarse_dofs = fine_dm.n_scalar_dofs, coarse_dm.n_scalar_dofs
        d.fine_cell_dofs = _lib.ptr(fd, C.c_int32)
        d.coarse_cell_dofs = _lib.ptr(cd, C.c_int32)
        d.fine_dirichlet = _lib.ptr(fm, C.c_uint8) if fm.any() else _lib.ptr(None, C.c_uint8)
        d.coarse_dirichlet = _lib.ptr(cm, C.c_uint8) if cm.any() else _lib.ptr(None, C.c_uint8)
        d.interp = _lib.ptr(self.P, C.c_double)
        d.device = int(device)
        self._t = C.c_void_p()
        _lib.check(_lib.lib().tmf_transfer_create(C.byref(d), C.byref(self._t)))
        self.n_fine, self.n_coarse = fine_dm.n_scalar_dofs, coarse_dm.n_scalar_dofs

    def prolongate(self, xc, xf, add: bool = False, stream: int = 0):
        """xf = P xc (add: xf += P xc), device tensors (both float64 or both float32)."""
        import torch

        f = _lib.lib().tmf_prolongate_f32 if xc.dtype == torch.float32 else _lib.lib().tmf_prolongate
        if xf.dtype != xc.dtype:
            raise ValueError("prolongate: mixed dtypes")
        _lib.check(f(self._t, _vp(xc), _vp(xf), int(bool(add)), C.c_void_p(stream)))

    def restrict(self, rf, rc, stream: int = 0):
        """rc = P^T rf, device tensors (both float64 or both float32)."""
        import torch

        f = _lib.lib().tmf_restrict_f32 if rf.dtype == torch.float32 else _lib.lib().tmf_restrict
        if rc.dtype != rf.dtype:
            raise ValueError("restrict: mixed dtypes")
        _lib.check(f(self._t, _vp(rf), _vp(rc), C.c_void_p(stream)))

    def close(self):
        if self._t:
            _lib.lib().tmf_transfer_destroy(self._t)
            self._t = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def kuhn_point_weights(points: np.ndarray, n_coarse: int):
    """(idx (n, 4) int32, w (n, 4)): for each point of [0,1]^3, the 4 vertices of the cell of
    the unjittered, unpermuted Kuhn mesh ``mesh.kuhn_cube_mesh(n_coarse, jitter=0,
    permute=False)`` containing it and its barycentric coordinates there.  In the cube with
    origin c and local coordinates t, sorted t_a >= t_b >= t_c, the Kuhn cell is
    (c, c + e_a, c + e_a + e_b, c + 1) with weights (1 - t_a, t_a - t_b, t_b - t_c, t_c)."""
    x = np.clip(np.asarray(points, dtype=np.float64), 0.0, 1.0) * n_coarse
    c = np.minimum(np.floor(x), n_coarse - 1).astype(np.int64)
    t = x - c
    order = np.argsort(-t, axis=1, kind="stable")
    ts = np.take_along_axis(t, order, axis=1)
    w = np.stack([1.0 - ts[:, 0], ts[:, 0] - ts[:, 1], ts[:, 1] - ts[:, 2], ts[:, 2]], axis=1)
    corners = np.zeros((len(x), 4, 3), dtype=np.int64)
    corners[:, 0] = c
    for k in range(3):
        corners[:, k + 1] = corners[:, k]
        np.add.at(corners[:, k + 1], (np.arange(len(x)), order[:, k]), 1)
    m = n_coarse + 1
    idx = (corners[..., 0] * m + corners[..., 1]) * m + corners[..., 2]
    return idx.astype(np.int32), w


class PointTransfer(Transfer):
    """P1 -> P1 transfer onto a non-nested, coarser Kuhn mesh of the unit cube (h-coarsening):
    each fine DoF (= fine vertex) takes the coarse P1 function at its position."""

    def __init__(self, fine_mesh, fine_dm, coarse_n: int, coarse_dm, device: int = 0):
        if fine_dm.degree != 1 or coarse_dm.degree != 1 or fine_dm.space != "cg":
            raise ValueError("h-transfers link P1 CG spaces")
        idx, w = kuhn_point_weights(fine_mesh.vertices, coarse_n)
        self.P = None
        self.index, self.weights = idx, np.ascontiguousarray(w)
        fm = np.ascontiguousarray(fine_dm.dirichlet_mask, dtype=np.uint8)
        cm = np.ascontiguousarray(coarse_dm.dirichlet_mask, dtype=np.uint8)
        d = _lib.PointTransferDesc()
        d.n_fine_dofs, d.n_coarse_dofs, d.entries_per_row = fine_dm.n_scalar_dofs, coarse_dm.n_scalar_dofs, 4
        d.coarse_index = _lib.ptr(self.index, C.c_int32)
        d.weights = _lib.ptr(self.weights, C.c_double)
        d.fine_dirichlet = _lib.ptr(fm, C.c_uint8) if fm.any() else _lib.ptr(None, C.c_uint8)
        d.coarse_dirichlet = _lib.ptr(cm, C.c_uint8) if cm.any() else _lib.ptr(None, C.c_uint8)
        d.device = int(device)
        self._t = C.c_void_p()
        _lib.check(_lib.lib().tmf_transfer_create_points(C.byref(d), C.byref(self._t)))
        self.n_fine, self.n_coarse = fine_dm.n_scalar_dofs, coarse_dm.n_scalar_dofs


@dataclass
class _Level:
    p: int
    dm: object
    A: object
    dinv: object
    lmax: float
    coeffs: list
    x: object = None
    b: object = None
    r: object = None
    d: object = None
    ax: object = None
    csr: object = None      # assembled operator (cuSPARSE) used instead of the matrix-free apply
    mesh: object = None


class PMultigrid:
    """p-multigrid V-cycle on CG Laplace (homogeneous Dirichlet on ``dirichlet_ids``).

    ``kappa``: per-cell coefficient of the CG levels' Laplacians (with a KappaHelmholtzOperator
    on top: the C4 operator's auxiliary CG space).
    ``fine_operator``: a DG operator (DgSipgOperator / HelmholtzOperator / KappaHelmholtzOperator
    of degree ``degrees[0]``, weak Dirichlet on ``dirichlet_ids``) to put on top of the CG levels
    through a c-transfer (the paper's cp-MG); its smoother uses the exact
    diagonal probed by :func:`dg_diagonal`."""

    def __init__(self, mesh, degrees=(3, 2, 1), dirichlet_ids=tuple(range(6)), smoothing_degree: int = 2,
                 smoothing_range: float = 15.0, coarse_iterations: int = 30, eig_iterations: int = 15,
                 lmax=None, config=None, seed: int = 0, fine_operator=None, precision: str = "f64",
                 coarse_matrix: bool = False, h_coarse=(), fine_smoothing_degree: int | None = None,
                 graph: bool = True, kappa=None):
        import torch

        from . import operator as op

        if precision not in ("f64", "mixed"):
            raise ValueError("precision must be 'f64' or 'mixed' (fp32 V-cycle, fp64 outer CG)")
        if precision == "mixed" and fine_operator is not None:
            raise ValueError("the mixed-precision V-cycle has fp32 operators for the CG levels only")
        self.mixed = precision == "mixed"
        # CUDA-graph replay of the V-cycle: needs device-side scalars everywhere (the mixed
        # cycle's coarse PCG); the fp64 cycle's native coarse PCG syncs with the host
        self.use_graph = bool(graph) and self.mixed
        self._graph, self._graph_failed = None, False
        degrees = tuple(int(p) for p in degrees)
        if len(degrees) < 2 or any(a <= b for a, b in zip(degrees, degrees[1:])):
            raise ValueError("degrees must be strictly decreasing, at least two levels")
        self.config = config or op.OperatorConfig()
        if self.mixed:
            import dataclasses

            self.config = dataclasses.replace(self.config, f32_mirror=True)
        dev = int(self.config.device)
        self.device = torch.device(f"cuda:{dev}")
        self.smoothing_degree, self.smoothing_range = int(smoothing_degree), float(smoothing_range)
        self.coarse_iterations = int(coarse_iterations)
        self.levels: list[_Level] = []
        from . import mesh as M

        h_coarse = tuple(int(n) for n in h_coarse)
        if kappa is not None and h_coarse:
            raise ValueError("a per-cell kappa lives on the fine mesh: no h-levels with kappa")
        if h_coarse and degrees[-1] != 1:
            raise ValueError("h-coarsening continues from a P1 level: degrees must end with 1")
        specs = [("cg", p, mesh) for p in degrees]
        specs += [("cg", 1, M.kuhn_cube_mesh(n, jitter=0.0, permute=False)) for n in h_coarse]
        self.p1_fine_level = len(degrees) - 1
        if fine_operator is not None:
            if fine_operator.dofmap.space != "dg" or fine_operator.dofmap.degree != degrees[0]:
                raise ValueError("fine_operator must be a DG operator of degree degrees[0]")
            if int(fine_operator.dofmap.n_components) != 1:
                raise ValueError("fine_operator must be scalar")
            specs.insert(0, ("dg", degrees[0], mesh))
            self.p1_fine_level += 1
        for i, (space, p, lmesh) in enumerate(specs):
            if space == "dg":
                A, dm = fine_operator, fine_operator.dofmap
                dinv = 1.0 / dg_diagonal(A, mesh)
            else:
                cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
                bas = B.tabulate_basis(p, cr, fr)
                geo = GeometryData("affine", cr, fr, None, None, None, None)
                dm = D.build_dof_map(lmesh, p, "cg", 1, tuple(dirichlet_ids))
                A = op.CgPoissonOperator(lmesh, dm, geo, bas, self.config, kappa=kappa)
                dinv = 1.0 / A.diagonal()
            lv = _Level(p, dm, A, dinv, 0.0, [])
            lv.mesh = lmesh
            n = dm.n_global_dofs
            vt = torch.float32 if self.mixed else torch.float64
            lv.x, lv.b, lv.r, lv.d, lv.ax = (torch.zeros(n, dtype=vt, device=self.device) for _ in range(5))
            if i < len(specs) - 1:
                given = None if lmax is None else float(lmax[i])
                lv.lmax = given if given is not None else 1.1 * self.estimate_lmax(lv, eig_iterations, seed)
                deg = self.smoothing_degree
                if space == "dg":   # the DG level sets the cp-MG rate: degree 4 by default
                    # (DG P3 32^3 to 1e-8: degree 2 / 4 / 6 -> 15 / 9 / 8 iterations, 53 / 41 / 45 ms)
                    deg = 4 if fine_smoothing_degree is None else int(fine_smoothing_degree)
                lv.coeffs = chebyshev_coefficients(lv.lmax, self.smoothing_range, deg)
            self.levels.append(lv)
        if self.mixed:   # the fp64 diagonals served the eigenvalue estimates; the cycle runs in fp32
            for lv in self.levels:
                lv.dinv = lv.dinv.to(torch.float32)
        # matrix-based P1 level on the fine mesh (the paper switches to the assembled operator
        # where it is faster): P1 there has 6 cells per DoF, so its CSR SpMV
        # (cuSPARSE) moves far fewer bytes than the matrix-free cell loop
        self.coarse_csr = None
        if coarse_matrix:
            from .sparse import assemble_cg_csr

            lv = self.levels[self.p1_fine_level]
            cr, fr = Q.make_cell_quadrature(lv.p), Q.make_face_quadrature(lv.p)
            A = assemble_cg_csr(lv.mesh, lv.dm, GeometryData("affine", cr, fr, None, None, None, None),
                                B.tabulate_basis(lv.p, cr, fr), device=self.device, kappa=kappa)
            lv.csr = A.to(torch.float32) if self.mixed else A
            self.coarse_csr = lv.csr
        self.transfers = []
        for i in range(len(self.levels) - 1):
            f, c = self.levels[i], self.levels[i + 1]
            if f.mesh is c.mesh:
                self.transfers.append(Transfer(f.dm, c.dm, dev))
            else:
                self.transfers.append(PointTransfer(f.mesh, f.dm, h_coarse[i - self.p1_fine_level], c.dm, dev))
        self.n_global_dofs = self.levels[0].dm.n_global_dofs

    # ------------------------------------------------------------------ setup
    def estimate_lmax(self, lv, iters: int, seed: int) -> float:
        """Largest eigenvalue of D^-1 A from ``iters`` Jacobi-PCG (Lanczos) steps."""
        import torch

        n = lv.dm.n_global_dofs
        g = np.random.default_rng(seed).uniform(-1, 1, n)
        g[np.asarray(lv.dm.dirichlet_mask, dtype=bool)] = 0.0
        r = torch.from_numpy(g).to(self.device)
        z = r * lv.dinv
        p = z.clone()
        q = torch.empty_like(p)
        rz = float(r @ z)
        alphas, betas = [], []
        for _ in range(iters):
            lv.A.apply_into(p.data_ptr(), q.data_ptr(), self._st())
            pq = float(p @ q)
            if pq <= 0.0:
                # SPEC.md:514 "indefiniteness detected (p^T A p <= 0)"
                raise ValueError(f"level P{lv.p} ({lv.dm.space}) is not positive definite: p.Ap = {pq:.3e} "
                                 f"after {len(alphas)} Lanczos steps (DG: penalty too small for the mesh?)")
            if rz <= 0.0:
                break
            a = rz / pq
            r -= a * q
            z = r * lv.dinv
            rz_new = float(r @ z)
            alphas.append(a)
            betas.append(rz_new / rz)
            p = z + betas[-1] * p
            rz = rz_new
        k = len(alphas)
        T = np.zeros((k, k))
        for j in range(k):
            T[j, j] = 1.0 / alphas[j] + (betas[j - 1] / alphas[j - 1] if j else 0.0)
            if j + 1 < k:
                T[j, j + 1] = T[j + 1, j] = np.sqrt(betas[j]) / alphas[j]
        return float(np.linalg.eigvalsh(T)[-1])

    @staticmethod
    def _st():
        import torch

        return torch.cuda.current_stream().cuda_stream

    # ------------------------------------------------------------------ cycle
    def _apply(self, lv, x, y, st):
        if lv.csr is not None:
            y.copy_((lv.csr @ x.unsqueeze(1)).squeeze(1))
        elif self.mixed:
            lv.A.apply_f32(x, out=y, stream=st)
        else:
            lv.A.apply_into(x.data_ptr(), y.data_ptr(), st)

    def _smooth(self, lv, first: bool):
        """Chebyshev-Jacobi on A x = b (lv.x, lv.b); first: x = 0 on entry."""
        L = _lib.lib()
        stp = self._st()
        st = C.c_void_p(stp)
        n = lv.dm.n_global_dofs
        step = L.tmf_chebyshev_step_f32 if self.mixed else L.tmf_chebyshev_step
        for k, (c1, c2) in enumerate(lv.coeffs):
            if k == 0 and first:
                _lib.check(step(n, None, _vp(lv.b), _vp(lv.dinv), _vp(lv.x), _vp(lv.d), c1, c2, st))
                continue
            self._apply(lv, lv.x, lv.ax, stp)
            _lib.check(step(n, _vp(lv.ax), _vp(lv.b), _vp(lv.dinv), _vp(lv.x), _vp(lv.d), c1, c2, st))

    def _coarse_pcg(self, lv):
        """Jacobi-PCG in the cycle's precision (x0 = 0, fixed iteration count) with the scalars
        on the device; the operator is the matrix-free apply or the assembled coarse matrix."""
        import torch

        st = self._st()
        x, b, dinv, q = lv.x, lv.b, lv.dinv, lv.ax
        x.zero_()
        r = b.clone()
        z = r * dinv
        p = z.clone()
        rz = torch.dot(r, z)
        zero = torch.zeros((), dtype=x.dtype, device=self.device)
        for _ in range(self.coarse_iterations):
            self._apply(lv, p, q, st)
            pq = torch.dot(p, q)
            alpha = torch.where(pq != 0, rz / pq, zero)
            x.add_(alpha * p)
            r.sub_(alpha * q)
            torch.mul(r, dinv, out=z)
            rz_new = torch.dot(r, z)
            beta = torch.where(rz != 0, rz_new / rz, zero)
            p = z + beta * p
            rz = rz_new

    def _cycle(self, i: int):
        from .solvers import jacobi_pcg

        lv = self.levels[i]
        if i == len(self.levels) - 1:
            if self.mixed or lv.csr is not None:
                self._coarse_pcg(lv)
            else:
                x, _ = jacobi_pcg(lv.A, lv.b, self.coarse_iterations)
                lv.x.copy_(x)
            return
        st = self._st()
        L = _lib.lib()
        self._smooth(lv, first=True)
        self._apply(lv, lv.x, lv.ax, st)
        axpby = L.tmf_vec_axpby_f32 if self.mixed else L.tmf_vec_axpby
        _lib.check(axpby(lv.dm.n_global_dofs, 1.0, _vp(lv.b), -1.0, _vp(lv.ax), _vp(lv.r), C.c_void_p(st)))
        nxt = self.levels[i + 1]
        self.transfers[i].restrict(lv.r, nxt.b, st)
        self._cycle(i + 1)
        self.transfers[i].prolongate(nxt.x, lv.x, add=True, stream=st)
        self._smooth(lv, first=False)

    def _capture(self):
        """Capture the whole V-cycle (every level's kernels, the coarse PCG with device scalars)
        into one CUDA graph: its hundreds of small launches on the coarse levels would
        otherwise be host-bound.  Returns None where capture is not possible."""
        import torch

        lv = self.levels[0]
        try:
            s = torch.cuda.Stream(device=self.device)
            s.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(s):
                for _ in range(2):   # warm-up (allocator, cuSPARSE workspaces) off the capture
                    self._cycle(0)
            torch.cuda.current_stream(self.device).wait_stream(s)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._cycle(0)
            return g
        except Exception:   # noqa: BLE001 -- eager cycles instead
            torch.cuda.synchronize(self.device)
            return None

    def vcycle(self, r, out=None):
        """z = V r (one V-cycle from a zero initial guess); device tensors.  Mixed precision:
        r is rounded to fp32, the cycle runs in fp32 and z is returned in r's dtype.  With
        ``graph=True`` (mixed precision) the cycle is replayed from a captured CUDA graph."""
        lv = self.levels[0]
        lv.b.copy_(r)
        if self.use_graph and self._graph is None and not self._graph_failed:
            self._graph = self._capture()
            self._graph_failed = self._graph is None
        if self._graph is not None:
            self._graph.replay()
        else:
            self._cycle(0)
        if out is None:
            return lv.x.to(r.dtype, copy=True)
        out.copy_(lv.x)
        return out

    # ------------------------------------------------------------------ solve
    def solve(self, b, tol: float = 1e-8, maxiter: int = 200):
        """Flexible PCG with one V-cycle per iteration; stops when ||r|| <= tol ||b||.
        Returns (x, residual norms)."""
        import torch

        A = self.levels[0].A
        st = self._st()
        x = torch.zeros_like(b)
        r = b.clone()
        z = self.vcycle(r)
        p = z.clone()
        q = torch.empty_like(b)
        rz = float(r @ z)
        hist = [float(torch.linalg.vector_norm(r))]
        stop = tol * hist[0]
        for _ in range(maxiter):
            if hist[-1] <= stop:
                break
            A.apply_into(p.data_ptr(), q.data_ptr(), st)
            pq = float(p @ q)
            if pq <= 0.0:
                raise ValueError(f"indefinite operator or preconditioner: p.Ap = {pq:.3e}")
            alpha = rz / pq
            x.add_(p, alpha=alpha)
            r.add_(q, alpha=-alpha)
            hist.append(float(torch.linalg.vector_norm(r)))
            z_new = self.vcycle(r)
            beta = float(r @ (z_new - z)) / rz
            rz = float(r @ z_new)
            z = z_new
            p = z + beta * p
        return x, np.array(hist)

    def close(self):
        for t in self.transfers:
            t.close()
        for lv in self.levels:
            if lv.dm.space == "cg":   # a caller's fine operator stays open
                lv.A.close()


def n10(hist) -> float:
    """Fractional iteration count to reduce the residual by 1e10 ([Fehn2019]):
    linear interpolation of log10 ||r|| between the bracketing iterations."""
    h = np.log10(np.asarray(hist, dtype=float) / float(hist[0]))
    hit = np.nonzero(h <= -10.0)[0]
    if not len(hit):
        raise ValueError("the residual was not reduced by ten orders of magnitude")
    k = int(hit[0])
    if k == 0:
        return 0.0
    return float(k - 1 + (h[k - 1] + 10.0) / (h[k - 1] - h[k]))
