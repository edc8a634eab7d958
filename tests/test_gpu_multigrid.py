"""GPU tests of the p-multigrid layer (paper_2509_10226_b200/multigrid.py, csrc/multigrid.cu)
against the CPU restatement oracle/ref_multigrid.py."""

import numpy as np
import pytest

from conftest import rel_l2
from oracle import ref_apply, ref_multigrid as RM

pytestmark = pytest.mark.gpu


def _dm(m, p, dids):
    from paper_2509_10226_b200 import dofmap as D

    return D.build_dof_map(m, p, "cg", 1, dids)


@pytest.mark.parametrize("pf,pc", [(2, 1), (3, 1), (3, 2), (4, 1), (4, 2), (4, 3)])
@pytest.mark.parametrize("dirichlet", [False, True])
def test_transfers_match_oracle(pf, pc, dirichlet):
    import torch

    from paper_2509_10226_b200 import mesh as M
    from paper_2509_10226_b200.multigrid import Transfer, interpolation_matrix

    m = M.kuhn_cube_mesh(4, seed=0)
    dids = tuple(range(6)) if dirichlet else ()
    dmf, dmc = _dm(m, pf, dids), _dm(m, pc, dids)
    T = Transfer(dmf, dmc)
    Pg = RM.prolongation_matrix(dmf.cell_dofs, dmc.cell_dofs, interpolation_matrix(pf, pc), dmf.n_scalar_dofs,
                                dmc.n_scalar_dofs, dmf.dirichlet_mask if dirichlet else None,
                                dmc.dirichlet_mask if dirichlet else None)
    rng = np.random.default_rng(3)
    xc = rng.uniform(-1, 1, dmc.n_scalar_dofs)
    rf = rng.uniform(-1, 1, dmf.n_scalar_dofs)
    xf0 = rng.uniform(-1, 1, dmf.n_scalar_dofs)
    xc_t, rf_t = torch.from_numpy(xc).cuda(), torch.from_numpy(rf).cuda()
    xf_t = torch.from_numpy(xf0).cuda()
    T.prolongate(xc_t, xf_t)                      # overwrite
    assert rel_l2(xf_t.cpu().numpy(), Pg @ xc) <= 1e-14
    xf_t = torch.from_numpy(xf0).cuda()
    T.prolongate(xc_t, xf_t, add=True)            # accumulate
    assert rel_l2(xf_t.cpu().numpy(), xf0 + Pg @ xc) <= 1e-14
    rc_t = torch.full((dmc.n_scalar_dofs,), 7.0, dtype=torch.float64, device="cuda")
    T.restrict(rf_t, rc_t)
    torch.cuda.synchronize()
    assert rel_l2(rc_t.cpu().numpy(), Pg.T @ rf) <= 1e-14
    if dirichlet:
        assert np.all(rc_t.cpu().numpy()[dmc.dirichlet_mask] == 0.0)


def test_transfer_rejects_bad_input():
    from paper_2509_10226_b200 import mesh as M
    from paper_2509_10226_b200.multigrid import Transfer

    m = M.kuhn_cube_mesh(2, seed=0)
    with pytest.raises(ValueError):
        Transfer(_dm(m, 1, ()), _dm(m, 2, ()))        # coarse has more DoFs per cell
    m2 = M.kuhn_cube_mesh(3, seed=0)
    with pytest.raises(ValueError):
        Transfer(_dm(m2, 2, ()), _dm(m, 1, ()))       # different meshes


def _oracle_levels(m, mg):
    from paper_2509_10226_b200 import basis as B, quadrature as Q

    levels, transfers = [], []
    for i, lv in enumerate(mg.levels):
        p = lv.p
        cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
        bas = B.tabulate_basis(p, cr, fr)
        dm = lv.dm
        A = (lambda dm, bas, w: lambda v: ref_apply.cg_apply(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask,
                                                             bas.grad_matrix, w, v))(dm, bas, cr.weights)
        diag = ref_apply.cg_diagonal(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask, bas.grad_matrix,
                                     cr.weights, dm.n_global_dofs)
        levels.append(dict(apply=A, diag=diag, coeffs=lv.coeffs))
        if i + 1 < len(mg.levels):
            nx = mg.levels[i + 1].dm
            transfers.append(RM.prolongation_matrix(dm.cell_dofs, nx.cell_dofs, mg.transfers[i].P, dm.n_scalar_dofs,
                                                    nx.n_scalar_dofs, dm.dirichlet_mask, nx.dirichlet_mask))
    return levels, transfers


@pytest.mark.parametrize("degrees", [(2, 1), (3, 2, 1), (4, 2, 1)])
def test_vcycle_matches_oracle(degrees):
    import torch

    from paper_2509_10226_b200 import mesh as M
    from paper_2509_10226_b200.multigrid import PMultigrid

    m = M.kuhn_cube_mesh(4, seed=0)
    mg = PMultigrid(m, degrees, coarse_iterations=12)
    levels, transfers = _oracle_levels(m, mg)
    # the Lanczos estimate agrees with the oracle's (same start vector, same iteration)
    lv = mg.levels[0]
    r0 = np.where(lv.dm.dirichlet_mask, 0.0, np.random.default_rng(0).uniform(-1, 1, lv.dm.n_global_dofs))
    assert abs(lv.lmax - 1.1 * RM.lanczos_lmax(levels[0]["apply"], levels[0]["diag"], r0, 15)) <= 1e-10 * lv.lmax
    b = np.where(lv.dm.dirichlet_mask, 0.0, np.random.default_rng(1).uniform(-1, 1, lv.dm.n_global_dofs))
    z = mg.vcycle(torch.from_numpy(b).cuda()).cpu().numpy()
    zr = RM.vcycle(levels, transfers, b, 12)
    assert rel_l2(z, zr) <= 1e-11
    assert np.all(z[lv.dm.dirichlet_mask] == 0.0)


def test_multigrid_pcg_converges_and_matches_oracle():
    import torch

    from paper_2509_10226_b200 import mesh as M
    from paper_2509_10226_b200.multigrid import PMultigrid
    from paper_2509_10226_b200.solvers import jacobi_pcg

    m = M.kuhn_cube_mesh(6, seed=0)
    mg = PMultigrid(m, (3, 2, 1), coarse_iterations=30)
    dm = mg.levels[0].dm
    b = np.where(dm.dirichlet_mask, 0.0, np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs))
    bt = torch.from_numpy(b).cuda()
    x, hist = mg.solve(bt, tol=1e-10, maxiter=50)
    assert hist[-1] <= 1e-10 * hist[0]
    assert len(hist) - 1 <= 20
    levels, transfers = _oracle_levels(m, mg)
    xr, hr = RM.flexible_pcg(levels[0]["apply"], lambda r: RM.vcycle(levels, transfers, r, 30), b, 1e-10, 50)
    assert len(hr) == len(hist)
    assert rel_l2(x.cpu().numpy(), xr) <= 1e-9
    # the true residual, and Jacobi-PCG with the same iteration count is far behind
    Ax = mg.levels[0].A.apply(x)
    assert rel_l2(Ax.cpu().numpy(), b) <= 1e-9
    _, hj = jacobi_pcg(mg.levels[0].A, bt, len(hist) - 1)
    assert hj[-1] > 1e3 * hist[-1]
    mg.close()


def _dg_problem(n, p):
    from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, operator as op, quadrature as Q
    from paper_2509_10226_b200.geometry import GeometryData

    m = M.kuhn_cube_mesh(n, seed=0)
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    dm = D.build_dof_map(m, p, "dg")
    sipg = op.baseline_sipg_tau(m, p, 1.0 / n)
    A = op.DgSipgOperator(m, dm, geo, bas, sipg, dirichlet_ids=range(6))
    Aref = lambda v: ref_apply.dg_apply(m.vertices, m.cells, dm.n_dofs_per_cell, m.interior_faces,  # noqa: E731
                                        m.boundary_faces, set(range(6)), bas.value_matrix, bas.grad_matrix,
                                        cr.weights, bas.face_values, bas.face_grads, fr.weights,
                                        sipg.tau_interior, sipg.tau_boundary, v)
    return m, dm, A, Aref


@pytest.mark.parametrize("p", [1, 2])
def test_dg_diagonal_by_colouring(p):
    import torch

    from paper_2509_10226_b200.multigrid import dg_diagonal

    m, dm, A, Aref = _dg_problem(2, p)
    d = dg_diagonal(A, m).cpu().numpy()
    n = dm.n_global_dofs
    ref = np.array([Aref(np.eye(1, n, i).ravel())[i] for i in range(n)])
    assert rel_l2(d, ref) <= 1e-13
    assert np.all(d > 0)


def test_c_transfer_matches_oracle():
    import torch

    from paper_2509_10226_b200.multigrid import Transfer

    m, dm, A, _ = _dg_problem(3, 2)
    dmc = _dm(m, 2, tuple(range(6)))
    T = Transfer(dm, dmc)
    assert np.array_equal(T.P, np.eye(10))
    Pg = RM.prolongation_matrix(dm.cell_dofs, dmc.cell_dofs, T.P, dm.n_scalar_dofs, dmc.n_scalar_dofs,
                                None, dmc.dirichlet_mask)
    rng = np.random.default_rng(5)
    xc, rf = rng.uniform(-1, 1, dmc.n_scalar_dofs), rng.uniform(-1, 1, dm.n_scalar_dofs)
    xf = torch.empty(dm.n_scalar_dofs, dtype=torch.float64, device="cuda")
    T.prolongate(torch.from_numpy(xc).cuda(), xf)
    assert rel_l2(xf.cpu().numpy(), Pg @ xc) <= 1e-15
    rc = torch.empty(dmc.n_scalar_dofs, dtype=torch.float64, device="cuda")
    T.restrict(torch.from_numpy(rf).cuda(), rc)
    assert rel_l2(rc.cpu().numpy(), Pg.T @ rf) <= 1e-14
    with pytest.raises(ValueError):
        Transfer(dm, _dm(m, 1, ()))                  # DG -> CG of another degree


def test_dg_cp_multigrid_matches_oracle_and_converges():
    import torch

    from paper_2509_10226_b200.multigrid import PMultigrid, n10
    from paper_2509_10226_b200.solvers import pcg_loop

    m, dm, A, Aref = _dg_problem(4, 2)
    mg = PMultigrid(m, (2, 1), fine_operator=A, coarse_iterations=20)
    assert [lv.dm.space for lv in mg.levels] == ["dg", "cg", "cg"]
    b = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    bt = torch.from_numpy(b).cuda()
    x, hist = mg.solve(bt, tol=1e-10, maxiter=60)
    assert hist[-1] <= 1e-10 * hist[0]
    # oracle: the same hierarchy on the CPU restatement
    levels, transfers = [], []
    diag0 = 1.0 / mg.levels[0].dinv.cpu().numpy()
    levels.append(dict(apply=Aref, diag=diag0, coeffs=mg.levels[0].coeffs))
    sub, subt = _oracle_levels(m, type("H", (), {"levels": mg.levels[1:], "transfers": mg.transfers[1:]})())
    levels += sub
    transfers.append(RM.prolongation_matrix(dm.cell_dofs, mg.levels[1].dm.cell_dofs, mg.transfers[0].P,
                                            dm.n_scalar_dofs, mg.levels[1].dm.n_scalar_dofs, None,
                                            mg.levels[1].dm.dirichlet_mask))
    transfers += subt
    xr, hr = RM.flexible_pcg(Aref, lambda r: RM.vcycle(levels, transfers, r, 20), b, 1e-10, 60)
    assert len(hr) == len(hist)
    assert rel_l2(x.cpu().numpy(), xr) <= 1e-8
    assert rel_l2(A.apply(x).cpu().numpy(), b) <= 1e-9
    # Jacobi-PCG (same diagonal) needs far more iterations for ten orders of magnitude
    _, hj = pcg_loop(lambda v, out: out.copy_(A.apply(v)), 1.0 / mg.levels[0].dinv, bt, 3 * len(hist))
    assert hj[-1] > 1e2 * hist[-1]
    assert n10(hist) < len(hist)


def test_indefinite_operator_is_reported():
    """cg_solve reports indefiniteness (p.Ap <= 0); a DG-SIPG penalty far below the
    coercivity threshold makes the operator indefinite and the hierarchy set-up raises."""
    from paper_2509_10226_b200 import operator as op
    from paper_2509_10226_b200.multigrid import PMultigrid

    m, dm, A, _ = _dg_problem(3, 2)
    sipg = op.baseline_sipg_tau(m, 2, 1.0 / 3)
    sipg.tau_interior *= 1e-3
    sipg.tau_boundary *= 1e-3
    B = op.DgSipgOperator(m, dm, A.geo, A.basis, sipg, dirichlet_ids=range(6))
    with pytest.raises(ValueError, match="positive definite"):
        PMultigrid(m, (2, 1), fine_operator=B, eig_iterations=60)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("dirichlet", [False, True])
def test_apply_f32_matches_fp64(p, dirichlet):
    """fp32 mirror of the CG Laplace apply (modal form on FFMA) vs the fp64 apply and the oracle."""
    import torch

    from paper_2509_10226_b200 import basis as B, mesh as M, operator as op, quadrature as Q
    from paper_2509_10226_b200.geometry import GeometryData

    m = M.kuhn_cube_mesh(4, seed=0)
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    dm = _dm(m, p, tuple(range(6)) if dirichlet else ())
    A = op.CgPoissonOperator(m, dm, geo, bas, op.OperatorConfig(f32_mirror=True))
    u = np.random.default_rng(2).uniform(-1, 1, dm.n_global_dofs)
    y64 = A.apply(u)
    y32 = A.apply_f32(torch.from_numpy(u).float().cuda()).double().cpu().numpy()
    assert rel_l2(y32, y64) <= 2e-6
    yr = ref_apply.cg_apply(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask, bas.grad_matrix, cr.weights, u)
    assert rel_l2(y64, yr) <= 1e-12
    if dirichlet:
        assert np.array_equal(y32[dm.dirichlet_mask], u.astype(np.float32).astype(np.float64)[dm.dirichlet_mask])


def test_apply_f32_needs_the_mirror():
    import torch

    from paper_2509_10226_b200 import mesh as M
    from paper_2509_10226_b200 import basis as B, operator as op, quadrature as Q
    from paper_2509_10226_b200.geometry import GeometryData

    m = M.kuhn_cube_mesh(2, seed=0)
    cr, fr = Q.make_cell_quadrature(2), Q.make_face_quadrature(2)
    bas = B.tabulate_basis(2, cr, fr)
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    dm = _dm(m, 2, ())
    A = op.CgPoissonOperator(m, dm, geo, bas)
    with pytest.raises(ValueError, match="fp32 mirror"):
        A.apply_f32(torch.zeros(dm.n_global_dofs, dtype=torch.float32, device="cuda"))
    with pytest.raises(ValueError):
        A.apply_f32(torch.zeros(dm.n_global_dofs, dtype=torch.float64, device="cuda"))
    from paper_2509_10226_b200 import dofmap as D

    ddm = D.build_dof_map(m, 2, "dg")
    with pytest.raises(ValueError, match="fp32 mirror"):
        op.DgSipgOperator(m, ddm, geo, bas, op.baseline_sipg_tau(m, 2, 0.5), op.OperatorConfig(f32_mirror=True))


def test_transfers_f32_match_fp64():
    import torch

    from paper_2509_10226_b200 import mesh as M
    from paper_2509_10226_b200.multigrid import Transfer

    m = M.kuhn_cube_mesh(4, seed=0)
    dmf, dmc = _dm(m, 3, tuple(range(6))), _dm(m, 1, tuple(range(6)))
    T = Transfer(dmf, dmc)
    rng = np.random.default_rng(4)
    xc = torch.from_numpy(rng.uniform(-1, 1, dmc.n_scalar_dofs)).cuda()
    rf = torch.from_numpy(rng.uniform(-1, 1, dmf.n_scalar_dofs)).cuda()
    xf64, xf32 = torch.empty(dmf.n_scalar_dofs, dtype=torch.float64, device="cuda"), \
        torch.empty(dmf.n_scalar_dofs, dtype=torch.float32, device="cuda")
    T.prolongate(xc, xf64)
    T.prolongate(xc.float(), xf32)
    assert rel_l2(xf32.double().cpu().numpy(), xf64.cpu().numpy()) <= 1e-6
    rc64, rc32 = torch.empty(dmc.n_scalar_dofs, dtype=torch.float64, device="cuda"), \
        torch.empty(dmc.n_scalar_dofs, dtype=torch.float32, device="cuda")
    T.restrict(rf, rc64)
    T.restrict(rf.float(), rc32)
    assert rel_l2(rc32.double().cpu().numpy(), rc64.cpu().numpy()) <= 1e-6
    with pytest.raises(ValueError):
        T.restrict(rf, rc32)


def test_mixed_precision_multigrid_converges_like_fp64():
    """fp32 V-cycle inside the fp64 flexible PCG reaches 1e-10 (far below fp32 round-off) in
    about the fp64 iteration count."""
    import torch

    from paper_2509_10226_b200 import mesh as M
    from paper_2509_10226_b200.multigrid import PMultigrid

    m = M.kuhn_cube_mesh(6, seed=0)
    mg64 = PMultigrid(m, (3, 2, 1), coarse_iterations=30)
    mg32 = PMultigrid(m, (3, 2, 1), coarse_iterations=30, precision="mixed")
    assert mg32.levels[0].x.dtype == torch.float32
    dm = mg64.levels[0].dm
    b = np.where(dm.dirichlet_mask, 0.0, np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs))
    bt = torch.from_numpy(b).cuda()
    x64, h64 = mg64.solve(bt, tol=1e-10, maxiter=60)
    x32, h32 = mg32.solve(bt, tol=1e-10, maxiter=60)
    assert h32[-1] <= 1e-10 * h32[0]
    assert len(h32) <= len(h64) + 3
    assert rel_l2(x32.cpu().numpy(), x64.cpu().numpy()) <= 1e-8
    z = mg32.vcycle(bt)
    assert z.dtype == torch.float64
    with pytest.raises(ValueError):
        PMultigrid(m, (2, 1), precision="half")


@pytest.mark.parametrize("precision", ["f64", "mixed"])
def test_matrix_based_coarse_level(precision):
    """Assembled (cuSPARSE) P1 coarse level: same V-cycle as the matrix-free one up to the
    coarse solver's round-off, same convergence."""
    import torch

    from paper_2509_10226_b200 import mesh as M
    from paper_2509_10226_b200.multigrid import PMultigrid

    m = M.kuhn_cube_mesh(5, seed=0)
    a = PMultigrid(m, (3, 1), coarse_iterations=20, precision=precision)
    b_ = PMultigrid(m, (3, 1), coarse_iterations=20, precision=precision, coarse_matrix=True)
    dm = a.levels[0].dm
    r = torch.from_numpy(np.where(dm.dirichlet_mask, 0.0,
                                  np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs))).cuda()
    za, zb = a.vcycle(r), b_.vcycle(r)
    tol = 1e-10 if precision == "f64" else 1e-4
    assert rel_l2(zb.cpu().numpy(), za.cpu().numpy()) <= tol
    _, ha = a.solve(r, tol=1e-10, maxiter=60)
    _, hb = b_.solve(r, tol=1e-10, maxiter=60)
    assert hb[-1] <= 1e-10 * hb[0] and abs(len(ha) - len(hb)) <= 2


@pytest.mark.parametrize("dirichlet", [False, True])
def test_point_transfer_matches_oracle(dirichlet):
    import scipy.sparse as sp
    import torch

    from paper_2509_10226_b200 import mesh as M
    from paper_2509_10226_b200.multigrid import PointTransfer

    mf = M.kuhn_cube_mesh(6, seed=0)
    mc = M.kuhn_cube_mesh(3, jitter=0.0, permute=False)
    dids = tuple(range(6)) if dirichlet else ()
    dmf, dmc = _dm(mf, 1, dids), _dm(mc, 1, dids)
    T = PointTransfer(mf, dmf, 3, dmc)
    nf_, nc_ = dmf.n_scalar_dofs, dmc.n_scalar_dofs
    rows = np.repeat(np.arange(nf_), 4)
    w = T.weights.ravel().copy()
    keep = np.ones_like(w, dtype=bool)
    if dirichlet:
        keep &= ~dmf.dirichlet_mask[rows] & ~dmc.dirichlet_mask[T.index.ravel()]
    Pg = sp.csr_matrix((w[keep], (rows[keep], T.index.ravel()[keep])), shape=(nf_, nc_))
    rng = np.random.default_rng(6)
    xc, rf = rng.uniform(-1, 1, nc_), rng.uniform(-1, 1, nf_)
    for dt, tol in ((torch.float64, 1e-14), (torch.float32, 1e-6)):
        xf = torch.empty(nf_, dtype=dt, device="cuda")
        T.prolongate(torch.from_numpy(xc).to("cuda", dt), xf)
        assert rel_l2(xf.double().cpu().numpy(), Pg @ xc) <= tol
        rc = torch.empty(nc_, dtype=dt, device="cuda")
        T.restrict(torch.from_numpy(rf).to("cuda", dt), rc)
        assert rel_l2(rc.double().cpu().numpy(), Pg.T @ rf) <= tol


@pytest.mark.parametrize("precision", ["f64", "mixed"])
def test_hp_multigrid_mesh_independent_iterations(precision):
    """SPEC.md:549 (mesh-independent iterations): p-levels then h-levels down to a 2^3 Kuhn
    mesh; the iteration count to 1e-10 stays within 3 across three refinements."""
    import torch

    from paper_2509_10226_b200 import mesh as M
    from paper_2509_10226_b200.multigrid import PMultigrid, n10

    its = []
    for n, hc in ((8, (4, 2)), (16, (8, 4, 2)), (24, (12, 6, 3))):
        m = M.kuhn_cube_mesh(n, seed=0)
        mg = PMultigrid(m, (2, 1), h_coarse=hc, coarse_iterations=40, precision=precision)
        assert [lv.dm.n_scalar_dofs for lv in mg.levels][-1] == (hc[-1] + 1) ** 3
        dm = mg.levels[0].dm
        b = torch.from_numpy(np.where(dm.dirichlet_mask, 0.0,
                                      np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs))).cuda()
        x, hist = mg.solve(b, tol=1e-10, maxiter=80)
        assert hist[-1] <= 1e-10 * hist[0]
        assert rel_l2(mg.levels[0].A.apply(x).cpu().numpy(), b.cpu().numpy()) <= 1e-9
        its.append(n10(hist))
        mg.close()
    assert max(its) - min(its) <= 3.0, its


def test_graph_replayed_vcycle_matches_eager():
    """The mixed-precision V-cycle captured in a CUDA graph gives the eager cycle's result."""
    import torch

    from paper_2509_10226_b200 import mesh as M
    from paper_2509_10226_b200.multigrid import PMultigrid

    m = M.kuhn_cube_mesh(8, seed=0)
    kw = dict(precision="mixed", h_coarse=(4, 2), coarse_iterations=20, coarse_matrix=True)
    eager = PMultigrid(m, (2, 1), graph=False, **kw)
    graph = PMultigrid(m, (2, 1), graph=True, **kw)
    dm = eager.levels[0].dm
    r = torch.from_numpy(np.where(dm.dirichlet_mask, 0.0,
                                  np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs))).cuda()
    z0 = eager.vcycle(r)
    z1 = graph.vcycle(r)
    z2 = graph.vcycle(2.0 * r)          # replayed with new input
    assert graph._graph is not None
    assert rel_l2(z1.cpu().numpy(), z0.cpu().numpy()) <= 1e-5
    assert rel_l2(z2.cpu().numpy(), 2.0 * z0.cpu().numpy()) <= 1e-4
    _, h = graph.solve(r, tol=1e-10, maxiter=60)
    assert h[-1] <= 1e-10 * h[0]


def test_transfer_c_abi_rejects_bad_input():
    """C-ABI argument checks of the transfer entry points (TMF_EINVAL -> ValueError)."""
    import ctypes as C

    from paper_2509_10226_b200 import _lib

    L = _lib.lib()
    fd = np.zeros((1, 10), np.int32)
    cd = np.zeros((1, 4), np.int32)
    P = np.zeros((10, 4))
    d = _lib.TransferDesc()
    d.n_cells, d.n_fine_dpc, d.n_coarse_dpc, d.n_fine_dofs, d.n_coarse_dofs = 1, 10, 4, 1, 1
    d.fine_cell_dofs, d.coarse_cell_dofs = _lib.ptr(fd, C.c_int32), _lib.ptr(cd, C.c_int32)
    d.interp = _lib.ptr(P, C.c_double)
    t = C.c_void_p()
    fd[0, 3] = 7                                     # fine DoF out of range
    with pytest.raises(ValueError, match="out of range"):
        _lib.check(L.tmf_transfer_create(C.byref(d), C.byref(t)))
    d.n_coarse_dpc = 5                               # unsupported coarse space
    with pytest.raises(ValueError):
        _lib.check(L.tmf_transfer_create(C.byref(d), C.byref(t)))
    pd = _lib.PointTransferDesc()
    pd.n_fine_dofs, pd.n_coarse_dofs, pd.entries_per_row = 1, 1, 3
    with pytest.raises(ValueError):
        _lib.check(L.tmf_transfer_create_points(C.byref(pd), C.byref(t)))
    with pytest.raises(ValueError):
        _lib.check(L.tmf_prolongate(None, None, None, 0, None))


@pytest.mark.parametrize("p", [1, 2, 3])
def test_cg_kappa_operator_and_diagonal(p):
    """CG -div(kappa grad u) with a per-cell coefficient (apply, diagonal, fp32 mirror, CSR) vs
    the oracle with the stiffness JxW scaled by kappa_e."""
    import torch

    from paper_2509_10226_b200 import basis as B, mesh as M, operator as op, quadrature as Q
    from paper_2509_10226_b200.geometry import GeometryData
    from paper_2509_10226_b200.sparse import assemble_cg_csr

    m = M.kuhn_cube_mesh(4, seed=0)
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    dm = _dm(m, p, tuple(range(6)))
    kap = 10.0 ** np.random.default_rng(2).uniform(-1, 1, m.n_cells)
    A = op.CgPoissonOperator(m, dm, geo, bas, op.OperatorConfig(f32_mirror=True), kappa=kap)
    u = np.random.default_rng(3).uniform(-1, 1, dm.n_global_dofs)
    yr = ref_apply.cg_apply(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask, bas.grad_matrix, cr.weights, u,
                            kappa=kap)
    assert rel_l2(A.apply(u), yr) <= 1e-12
    dr = ref_apply.cg_diagonal(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask, bas.grad_matrix, cr.weights,
                               dm.n_global_dofs, kappa=kap)
    assert rel_l2(A.diagonal().cpu().numpy(), dr) <= 1e-13
    y32 = A.apply_f32(torch.from_numpy(u).float().cuda()).double().cpu().numpy()
    assert rel_l2(y32, yr) <= 2e-6
    C = assemble_cg_csr(m, dm, geo, bas, kappa=kap)
    yc = (C @ torch.from_numpy(u).cuda().unsqueeze(1)).squeeze(1).cpu().numpy()
    assert rel_l2(yc, yr) <= 1e-12


def test_cp_multigrid_for_kappa_helmholtz():
    """C4-type operator (DG mass + kappa-Laplace, kappa log-uniform in [0.1, 10]) under the
    cp-multigrid with kappa-weighted CG levels: converges far faster than Jacobi-PCG."""
    import torch

    from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, operator as op, quadrature as Q
    from paper_2509_10226_b200.geometry import GeometryData
    from paper_2509_10226_b200.multigrid import PMultigrid
    from paper_2509_10226_b200.solvers import pcg_loop

    n, p = 8, 2
    m = M.kuhn_cube_mesh(n, seed=0)
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    dm = D.build_dof_map(m, p, "dg")
    kap = 10.0 ** np.random.default_rng(2).uniform(-1, 1, m.n_cells)
    sipg = op.baseline_sipg_tau(m, p, 1.0 / n)
    H = op.KappaHelmholtzOperator(m, dm, geo, bas, sipg, kap, 1.0, dirichlet_ids=range(6))
    mg = PMultigrid(m, (2, 1), fine_operator=H, kappa=kap, coarse_iterations=40)
    b = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)).cuda()
    x, hist = mg.solve(b, tol=1e-10, maxiter=80)
    assert hist[-1] <= 1e-10 * hist[0]
    assert rel_l2(H.apply(x).cpu().numpy(), b.cpu().numpy()) <= 1e-9
    _, hj = pcg_loop(lambda v, out: out.copy_(H.apply(v)), 1.0 / mg.levels[0].dinv, b, len(hist) - 1)
    assert hj[-1] > 1e3 * hist[-1]
    with pytest.raises(ValueError):
        PMultigrid(m, (2, 1), kappa=kap, h_coarse=(4,))
