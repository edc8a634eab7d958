"""GPU parity at BASELINE sizes through size-independent properties, and against
the CPU oracle at the largest sizes the oracle finishes in seconds.

C2 (48^3 x 6, P1-P4): constant nullspace (no Dirichlet), symmetry, linearity,
reordering invariance of the energy; C3 (64^3 x 6 DG-SIPG P3): symmetry and
coercivity; C4-type kappa-Helmholtz P2 (48^3): symmetry and positivity; GPU vs
oracle on 16^3 (CG P3, DG P2) meshes.
"""

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu


def _setup(n, p, space, reorder=False, dids=()):
    from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, quadrature as Q
    from paper_2509_10226_b200.geometry import GeometryData

    m = M.kuhn_cube_mesh(n, seed=0)
    if reorder:
        from paper_2509_10226_b200.reorder import hierarchical_reorder

        m = M.apply_cell_permutation(m, hierarchical_reorder(m))
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    return m, D.build_dof_map(m, p, space, 1, dids), geo, bas


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_c2_full_size_properties(p):
    import torch

    from paper_2509_10226_b200 import operator as op

    m, dm, geo, bas = _setup(48, p, "cg")
    A = op.CgPoissonOperator(m, dm, geo, bas)
    n = dm.n_global_dofs
    g = torch.Generator(device="cuda").manual_seed(p)
    u = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    v = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    one = torch.ones(n, dtype=torch.float64, device="cuda")
    Au, Av, A1 = A.apply(u), A.apply(v), A.apply(one)
    scale = torch.linalg.vector_norm(Au)
    # constant nullspace of the pure-Neumann Laplacian
    assert torch.linalg.vector_norm(A1) <= 1e-12 * scale
    # symmetry
    a, b = float(u @ Av), float(v @ Au)
    assert abs(a - b) <= 1e-12 * float(torch.linalg.vector_norm(u) * torch.linalg.vector_norm(Av))
    # linearity
    w = A.apply(2.5 * u - v)
    assert float(torch.linalg.vector_norm(w - (2.5 * Au - Av))) <= 1e-13 * float(scale)
    # positive semi-definite
    assert float(u @ Au) > 0


@pytest.mark.parametrize("p", [2, 3])
def test_c2_reordering_preserves_energy(p):
    """x^T A x for the interpolant of a smooth function does not depend on the cell order."""
    from paper_2509_10226_b200 import operator as op
    from paper_2509_10226_b200.dofmap import dof_coordinates

    vals = []
    for reorder in (False, True):
        m, dm, geo, bas = _setup(24, p, "cg", reorder)
        x = dof_coordinates(m, dm, bas.nodes)
        u = np.sin(np.pi * x[:, 0]) * np.cos(2 * x[:, 1]) + x[:, 2] ** 2
        vals.append(float(u @ op.CgPoissonOperator(m, dm, geo, bas).apply(u)))
    assert abs(vals[0] - vals[1]) <= 1e-12 * abs(vals[0])


def test_c3_full_size_symmetry_coercivity():
    import torch

    from paper_2509_10226_b200 import operator as op

    n, p = 64, 3
    m, dm, geo, bas = _setup(n, p, "dg", True)
    A = op.DgSipgOperator(m, dm, geo, bas, op.baseline_sipg_tau(m, p, 1.0 / n), dirichlet_ids=range(6))
    g = torch.Generator(device="cuda").manual_seed(7)
    u = torch.rand(dm.n_global_dofs, dtype=torch.float64, device="cuda", generator=g) - 0.5
    v = torch.rand(dm.n_global_dofs, dtype=torch.float64, device="cuda", generator=g) - 0.5
    Au, Av = A.apply(u), A.apply(v)
    a, b = float(u @ Av), float(v @ Au)
    assert abs(a - b) <= 1e-12 * float(torch.linalg.vector_norm(u) * torch.linalg.vector_norm(Av))
    assert float(u @ Au) > 0


def test_c4_kappa_helmholtz_symmetry_positivity():
    import torch

    from paper_2509_10226_b200 import operator as op

    n, p = 48, 2
    m, dm, geo, bas = _setup(n, p, "dg", True)
    kap = 10.0 ** np.random.default_rng(2).uniform(-1, 1, m.n_cells)
    A = op.KappaHelmholtzOperator(m, dm, geo, bas, op.baseline_sipg_tau(m, p, 1.0 / n), kap, 1.0,
                                  dirichlet_ids=range(6))
    g = torch.Generator(device="cuda").manual_seed(3)
    u = torch.rand(dm.n_global_dofs, dtype=torch.float64, device="cuda", generator=g) - 0.5
    v = torch.rand(dm.n_global_dofs, dtype=torch.float64, device="cuda", generator=g) - 0.5
    Au, Av = A.apply(u), A.apply(v)
    a, b = float(u @ Av), float(v @ Au)
    assert abs(a - b) <= 1e-12 * float(torch.linalg.vector_norm(u) * torch.linalg.vector_norm(Av))
    assert float(u @ Au) > 0


def test_oracle_parity_16cubed_cg_p3_dirichlet():
    from oracle import ref_apply
    from paper_2509_10226_b200 import operator as op

    m, dm, geo, bas = _setup(16, 3, "cg", False, tuple(range(6)))
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    y = op.CgPoissonOperator(m, dm, geo, bas).apply(u)
    ref = ref_apply.cg_apply(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask, bas.grad_matrix,
                             geo.cell_rule.weights, u)
    assert rel_l2(y, ref) <= 1e-12


def test_oracle_parity_16cubed_dg_p2():
    from oracle import ref_apply
    from paper_2509_10226_b200 import operator as op

    n, p = 16, 2
    m, dm, geo, bas = _setup(n, p, "dg", True)
    sipg = op.baseline_sipg_tau(m, p, 1.0 / n)
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    y = op.DgSipgOperator(m, dm, geo, bas, sipg, dirichlet_ids=(0, 2, 4)).apply(u)
    ref = ref_apply.dg_apply(m.vertices, m.cells, dm.n_dofs_per_cell, m.interior_faces, m.boundary_faces,
                             {0, 2, 4}, bas.value_matrix, bas.grad_matrix, geo.cell_rule.weights,
                             bas.face_values, bas.face_grads, geo.face_rule.weights, sipg.tau_interior,
                             sipg.tau_boundary, u)
    assert rel_l2(y, ref) <= 1e-12
