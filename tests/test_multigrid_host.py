"""CPU tests of the p-multigrid layer: interpolation tables, Chebyshev coefficients, and the
oracle's transfer / V-cycle restatement (oracle/ref_multigrid.py) on small meshes."""

import numpy as np
import pytest

from conftest import rel_l2
from oracle import ref_apply, ref_multigrid as RM
from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, quadrature as Q
from paper_2509_10226_b200.multigrid import chebyshev_coefficients, interpolation_matrix

PAIRS = [(2, 1), (3, 1), (3, 2), (4, 1), (4, 2), (4, 3)]


@pytest.mark.parametrize("pf,pc", PAIRS)
def test_interpolation_matrix_reproduces_coarse_polynomials(pf, pc):
    P = interpolation_matrix(pf, pc)
    nf, nc = B.n_dofs_per_cell(pf), B.n_dofs_per_cell(pc)
    assert P.shape == (nf, nc)
    assert np.allclose(P.sum(axis=1), 1.0, atol=1e-13)          # partition of unity
    fine, _ = B.reference_nodes(pf)
    coarse, _ = B.reference_nodes(pc)
    rng = np.random.default_rng(0)
    for _ in range(3):   # a random polynomial of degree pc, sampled at both node sets
        c = rng.standard_normal(B.n_dofs_per_cell(pc))
        f = lambda x: B._mono(x, B._exponents(pc)) @ c  # noqa: E731
        assert np.allclose(P @ f(coarse), f(fine), atol=1e-12)
    # vertex DoFs of the fine space are the coarse vertex DoFs
    assert np.array_equal(P[:4, :4], np.eye(4))


def test_interpolation_matrix_rejects_bad_degrees():
    with pytest.raises(ValueError):
        interpolation_matrix(2, 2)
    with pytest.raises(ValueError):
        interpolation_matrix(5, 1)


def test_chebyshev_coefficients_match_oracle():
    for deg in (1, 2, 3, 5):
        a = chebyshev_coefficients(1.7, 15.0, deg)
        b = RM.chebyshev_coefficients(1.7, 15.0, deg)
        assert np.allclose(a, b, rtol=0, atol=0)


def _space(m, p, dids=()):
    dm = D.build_dof_map(m, p, "cg", 1, dids)
    return dm


@pytest.mark.parametrize("pf,pc", [(2, 1), (3, 2), (4, 2)])
def test_oracle_prolongation_interpolates(pf, pc):
    """The oracle's global prolongation maps the interpolant of a degree-pc polynomial on
    the coarse space to its interpolant on the fine space (continuity across cells)."""
    m = M.kuhn_cube_mesh(3, seed=0)
    dmf, dmc = _space(m, pf), _space(m, pc)
    Pg = RM.prolongation_matrix(dmf.cell_dofs, dmc.cell_dofs, interpolation_matrix(pf, pc),
                                dmf.n_scalar_dofs, dmc.n_scalar_dofs)
    xf = D.dof_coordinates(m, dmf, B.reference_nodes(pf)[0])
    xc = D.dof_coordinates(m, dmc, B.reference_nodes(pc)[0])
    f = lambda x: 1.0 + x[:, 0] - 2.0 * x[:, 1] * (pc >= 2) * x[:, 2] + 0.5 * x[:, 2] ** pc  # noqa: E731
    assert rel_l2(Pg @ f(xc), f(xf)) <= 1e-13
    # each fine row is a partition of unity
    assert np.allclose(np.asarray(Pg.sum(axis=1)).ravel(), 1.0, atol=1e-13)


def test_oracle_multigrid_pcg_converges_fast():
    """p-MG (3 -> 2 -> 1) flexible PCG reaches 1e-8 in far fewer iterations than Jacobi-PCG."""
    m = M.kuhn_cube_mesh(3, seed=0)
    dids = tuple(range(6))
    levels, dms = [], []
    for p in (3, 2, 1):
        cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
        bas = B.tabulate_basis(p, cr, fr)
        dm = _space(m, p, dids)
        A = (lambda dm, bas, w: lambda v: ref_apply.cg_apply(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask,
                                                             bas.grad_matrix, w, v))(dm, bas, cr.weights)
        diag = ref_apply.cg_diagonal(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask, bas.grad_matrix,
                                     cr.weights, dm.n_global_dofs)
        r0 = np.where(dm.dirichlet_mask, 0.0, np.random.default_rng(0).uniform(-1, 1, dm.n_global_dofs))
        lmax = 1.1 * RM.lanczos_lmax(A, diag, r0, 15)
        assert 1.0 < lmax < 5.0
        levels.append(dict(apply=A, diag=diag, coeffs=RM.chebyshev_coefficients(lmax, 15.0, 3)))
        dms.append(dm)
    transfers = [RM.prolongation_matrix(dms[i].cell_dofs, dms[i + 1].cell_dofs,
                                        interpolation_matrix(dms[i].degree, dms[i + 1].degree),
                                        dms[i].n_scalar_dofs, dms[i + 1].n_scalar_dofs,
                                        dms[i].dirichlet_mask, dms[i + 1].dirichlet_mask) for i in range(2)]
    b = np.where(dms[0].dirichlet_mask, 0.0, np.random.default_rng(1).uniform(-1, 1, dms[0].n_global_dofs))
    x, hist = RM.flexible_pcg(levels[0]["apply"], lambda r: RM.vcycle(levels, transfers, r, 40), b, 1e-8, 60)
    assert hist[-1] <= 1e-8 * hist[0]
    assert len(hist) - 1 <= 10
    assert rel_l2(levels[0]["apply"](x), b) <= 1e-7
    _, hj = ref_apply.jacobi_pcg(levels[0]["apply"], levels[0]["diag"], b, len(hist) - 1)
    assert hj[-1] > 100 * hist[-1]


def test_color_cells_is_a_proper_colouring():
    from paper_2509_10226_b200.multigrid import color_cells

    m = M.kuhn_cube_mesh(5, seed=0)
    col, nc = color_cells(m)
    f = m.interior_faces
    assert np.all(col[f[:, 0]] != col[f[:, 2]])
    assert 2 <= nc <= 5 and col.min() == 0 and col.max() == nc - 1
    # greedy in cell order: every cell's colour is the smallest not used by an earlier neighbour
    nbr = [[] for _ in range(m.n_cells)]
    for a, b in zip(f[:, 0], f[:, 2]):
        nbr[a].append(b)
        nbr[b].append(a)
    for e in range(m.n_cells):
        used = {col[x] for x in nbr[e] if x < e}
        assert col[e] == min(set(range(6)) - used)


def test_n10_metric():
    from paper_2509_10226_b200.multigrid import n10

    assert n10(10.0 ** -np.arange(12)) == pytest.approx(10.0)        # 10x per iteration
    h = [1.0, 1e-4, 1e-8, 1e-12]                                        # 1e-10 reached mid-way
    assert n10(h) == pytest.approx(2.5)
    with pytest.raises(ValueError):
        n10([1.0, 1e-3])


@pytest.mark.parametrize("nf,nc", [(7, 4), (8, 4), (16, 8), (5, 2)])
def test_kuhn_point_weights_locate_and_interpolate(nf, nc):
    """h-transfer weights: each fine vertex lies in a real cell of the coarse Kuhn mesh, with
    nonnegative barycentric weights summing to 1 that reproduce linear functions exactly."""
    from paper_2509_10226_b200.multigrid import kuhn_point_weights

    mc = M.kuhn_cube_mesh(nc, jitter=0.0, permute=False)
    mf = M.kuhn_cube_mesh(nf, seed=3)
    idx, w = kuhn_point_weights(mf.vertices, nc)
    assert w.min() >= -1e-15 and np.allclose(w.sum(axis=1), 1.0, atol=1e-15)
    f = lambda x: 1.0 + 2.0 * x[:, 0] - 3.0 * x[:, 1] + 0.5 * x[:, 2]  # noqa: E731
    assert np.abs((w * f(mc.vertices)[idx]).sum(axis=1) - f(mf.vertices)).max() <= 1e-14
    cells = {tuple(sorted(c)) for c in mc.cells.tolist()}
    assert all(tuple(sorted(r)) in cells for r in idx.tolist())
    # a fine vertex that coincides with a coarse vertex maps onto it alone
    idx2, w2 = kuhn_point_weights(mc.vertices, nc)
    assert np.allclose(np.take_along_axis(w2, np.argmax(w2, axis=1)[:, None], 1), 1.0)


def test_color_cells_rejects_bad_faces():
    from paper_2509_10226_b200.multigrid import color_cells

    m = M.kuhn_cube_mesh(2, seed=0)
    bad = type("Mesh", (), {"n_cells": m.n_cells, "interior_faces": m.interior_faces.copy()})()
    bad.interior_faces[0, 2] = m.n_cells + 5
    with pytest.raises(ValueError):
        color_cells(bad)
    empty = type("Mesh", (), {"n_cells": 1, "interior_faces": np.zeros((0, 5), np.int32)})()
    col, nc = color_cells(empty)
    assert nc == 1 and col.tolist() == [0]
