"""GPU tests: matrix-free diagonal, Jacobi-PCG (native loop and the Python-driven
loop used by the multi-GPU solver), properties of the operators, and the
partitioned operator classes on one rank."""

import numpy as np
import pytest

from conftest import rel_l2
from oracle import ref_apply

pytestmark = pytest.mark.gpu


def _cg(n, p, dids=(), seed=0):
    from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, operator as op, quadrature as Q
    from paper_2509_10226_b200.geometry import GeometryData

    m = M.kuhn_cube_mesh(n, seed=seed)
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    dm = D.build_dof_map(m, p, "cg", 1, dids)
    return m, dm, geo, bas, op.CgPoissonOperator(m, dm, geo, bas)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_diagonal_matches_oracle(p):
    import torch

    m, dm, geo, bas, A = _cg(4, p, (0, 1, 2, 3, 4, 5))
    d = A.diagonal()
    torch.cuda.synchronize()
    ref = ref_apply.cg_diagonal(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask, bas.grad_matrix,
                                geo.cell_rule.weights, dm.n_global_dofs)
    assert rel_l2(d.cpu().numpy(), ref) <= 1e-13


@pytest.mark.parametrize("p", [1, 3])
def test_native_pcg_matches_oracle(p):
    import torch

    from paper_2509_10226_b200.solvers import jacobi_pcg, pcg_loop

    m, dm, geo, bas, A = _cg(5, p, tuple(range(6)))
    rng = np.random.default_rng(1)
    b = np.where(dm.dirichlet_mask, 0.0, rng.uniform(-1, 1, dm.n_global_dofs))
    bt = torch.from_numpy(b).cuda()
    x, hist = jacobi_pcg(A, bt, 25)
    diag = ref_apply.cg_diagonal(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask, bas.grad_matrix,
                                 geo.cell_rule.weights, dm.n_global_dofs)
    Aref = lambda v: ref_apply.cg_apply(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask,  # noqa: E731
                                        bas.grad_matrix, geo.cell_rule.weights, v)
    xr, hr = ref_apply.jacobi_pcg(Aref, diag, b, 25)
    assert rel_l2(x.cpu().numpy(), xr) <= 1e-10
    assert np.allclose(hist, hr, rtol=1e-8)
    assert hist[-1] < 0.05 * hist[0]
    # the Python-driven loop (multi-GPU code path, single process) agrees
    x2, h2 = pcg_loop(lambda v, out: A.apply(v) if out is None else out.copy_(A.apply(v)), A.diagonal(), bt, 25)
    assert rel_l2(x2.cpu().numpy(), xr) <= 1e-10
    assert np.allclose(h2, hr, rtol=1e-8)


def test_cg_properties_nullspace_symmetry():
    m, dm, geo, bas, A = _cg(6, 3)
    one = np.ones(dm.n_global_dofs)
    assert np.linalg.norm(A.apply(one)) <= 1e-11 * np.sqrt(dm.n_global_dofs)
    rng = np.random.default_rng(3)
    u, v = rng.standard_normal((2, dm.n_global_dofs))
    a, b = u @ A.apply(v), v @ A.apply(u)
    assert abs(a - b) <= 1e-12 * max(abs(a), 1.0)
    assert u @ A.apply(u) > 0


def test_dg_symmetry_and_coercivity():
    from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, operator as op, quadrature as Q
    from paper_2509_10226_b200.geometry import GeometryData

    p, n = 2, 4
    m = M.kuhn_cube_mesh(n, seed=4)
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    dm = D.build_dof_map(m, p, "dg")
    A = op.DgSipgOperator(m, dm, geo, bas, op.baseline_sipg_tau(m, p, 1.0 / n), dirichlet_ids=range(6))
    rng = np.random.default_rng(5)
    u, v = rng.standard_normal((2, dm.n_global_dofs))
    a, b = u @ A.apply(v), v @ A.apply(u)
    assert abs(a - b) <= 1e-11 * max(abs(a), 1.0)
    assert u @ A.apply(u) > 0


def test_distributed_operator_single_rank_on_gpu():
    """The partitioned operator classes with the B200 local plan, world size 1 (NCCL)."""
    import os

    import torch
    import torch.distributed as dist

    from paper_2509_10226_b200 import distributed as DD

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    created = False
    if not dist.is_initialized():
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
        dist.barrier()
        created = True
    try:
        m, dm, geo, bas, A = _cg(4, 2, (1, 2))
        D = DD.DistributedCgOperator(m, dm, geo, bas, 0, 1)
        u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
        ids = D.owned_global_ids
        y = D.apply(torch.from_numpy(u[ids]).cuda()).cpu().numpy()
        ref = A.apply(u)
        assert rel_l2(y, ref[ids]) <= 1e-14
        # DG-SIPG through the partitioned class (owned cells' volume terms, then faces)
        from paper_2509_10226_b200 import basis as B, dofmap as Dm, operator as op, quadrature as Q
        from paper_2509_10226_b200.geometry import GeometryData

        p = 2
        cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
        bas2 = B.tabulate_basis(p, cr, fr)
        geo2 = GeometryData("affine", cr, fr, None, None, None, None)
        dm2 = Dm.build_dof_map(m, p, "dg")
        sipg = op.baseline_sipg_tau(m, p, 0.25)
        Dg = DD.DistributedDgOperator(m, dm2, geo2, bas2, sipg, 0, 1, dirichlet_ids=range(6))
        Ag = op.DgSipgOperator(m, dm2, geo2, bas2, sipg, dirichlet_ids=range(6))
        ug = np.random.default_rng(2).uniform(-1, 1, dm2.n_global_dofs)
        gids = Dg.owned_global_ids()
        yg = torch.empty(Dg.n_local, dtype=torch.float64, device="cuda")
        Dg.apply(torch.from_numpy(ug[gids]).cuda(), out=yg)
        assert rel_l2(yg.cpu().numpy()[: Dg.n_owned], Ag.apply(ug)[gids]) <= 1e-14
    finally:
        if created:
            dist.destroy_process_group()


@pytest.mark.parametrize("engine", ["modal", "tensor"])
@pytest.mark.parametrize("p", [2, 3])
def test_fused_pcg_matches_unfused(p, engine):
    """tmf_pcg's fused iteration (tensor / modal cell engines: p.Ap from the element energies plus
    the identity rows, x update and zeroing of A p folded into the direction update) against
    the unfused loop (quadrature-point engine: memset / dot / update / direction), with b
    nonzero on the constrained rows too so the identity-row energy term matters."""
    import torch

    from paper_2509_10226_b200 import operator as op
    from paper_2509_10226_b200.solvers import jacobi_pcg

    m, dm, geo, bas, _ = _cg(5, p, (0, 3))
    A = op.CgPoissonOperator(m, dm, geo, bas, op.OperatorConfig(cell_engine=engine))
    assert A.info["cell_engine"] == {"modal": 4, "tensor": 3}[engine]
    B = op.CgPoissonOperator(m, dm, geo, bas, op.OperatorConfig(cell_engine="dmma"))
    b = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, dm.n_global_dofs)).cuda()
    x1, h1 = jacobi_pcg(A, b, 30)
    x2, h2 = jacobi_pcg(B, b, 30)
    assert rel_l2(x1.cpu().numpy(), x2.cpu().numpy()) <= 1e-10
    assert np.allclose(h1, h2, rtol=1e-8)
    assert h1[-1] < 0.1 * h1[0]
