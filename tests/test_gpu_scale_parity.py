"""Value-level GPU parity at the BASELINE sizes the bench runs.

Every test compares the B200 apply with the CPU oracle (oracle/ref_apply.py, the
NumPy restatement of the reference loop, one vectorised pass over all cells) on
the SAME seeded arrays, at relative L2 <= 1e-12 (north_star):

* C2: CG Laplace P1-P4 on the 48^3 x 6 jittered permuted Kuhn mesh, unordered and
  reordered exactly as ``bench.py`` builds it (``reorder_mesh``: hierarchical cell
  order + first-touch vertex renumbering), no Dirichlet (the bench's case), plus an
  all-Dirichlet P3 variant;
* C3: DG-SIPG P3 on the full 64^3 x 6 mesh (1,572,864 cells: 48 face windows of
  32,768 cells), reordered, weak Dirichlet on all 6 sides, BASELINE tau;
  plus DG-SIPG P3 on the unordered 48^3 mesh (faces in random cell order);
* C4-type: kappa-Helmholtz P2 (log-uniform per-cell kappa, mass 1) on 64^3, reordered;
* C5-type: 100 Jacobi-PCG iterations of CG P3 with homogeneous Dirichlet on 24^3,
  residual history and solution against the oracle PCG.

The oracle sizes were timed in the build container: CG P4 48^3 12 s, DG P3 48^3
13 s, kappa-Helmholtz P2 48^3 7 s (single thread).
"""

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu

_MESHES = {}


def _mesh(n, reorder):
    from paper_2509_10226_b200 import mesh as M
    from paper_2509_10226_b200.reorder import reorder_mesh

    key = (n, reorder)
    if key not in _MESHES:
        m = M.kuhn_cube_mesh(n, seed=0)
        _MESHES[key] = reorder_mesh(m) if reorder else m
    return _MESHES[key]


def _tables(p):
    from paper_2509_10226_b200 import basis as B, quadrature as Q
    from paper_2509_10226_b200.geometry import GeometryData

    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    return GeometryData("affine", cr, fr, None, None, None, None), B.tabulate_basis(p, cr, fr)


def _cg_oracle(m, dm, geo, bas, u, kappa=None):
    from oracle import ref_apply

    return ref_apply.cg_apply(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask, bas.grad_matrix,
                              geo.cell_rule.weights, u, kappa=kappa, chunk=65536)


def _dg_oracle(m, dm, geo, bas, sipg, dids, u, kappa=None, mass_scale=0.0):
    from oracle import ref_apply

    return ref_apply.dg_apply(m.vertices, m.cells, dm.n_dofs_per_cell, m.interior_faces, m.boundary_faces,
                              set(dids), bas.value_matrix, bas.grad_matrix, geo.cell_rule.weights,
                              bas.face_values, bas.face_grads, geo.face_rule.weights, sipg.tau_interior,
                              sipg.tau_boundary, u, kappa=kappa, mass_scale=mass_scale, chunk=65536)


@pytest.mark.parametrize("reorder", [False, True], ids=["unordered", "reordered"])
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_c2_48cubed_value_parity(p, reorder):
    from paper_2509_10226_b200 import dofmap as D, operator as op

    m = _mesh(48, reorder)
    geo, bas = _tables(p)
    dm = D.build_dof_map(m, p, "cg")
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    A = op.CgPoissonOperator(m, dm, geo, bas)
    y = A.apply(u)
    ref = _cg_oracle(m, dm, geo, bas, u)
    assert rel_l2(y, ref) <= 1e-12
    # the device-resident path the bench times (torch tensors in HBM) gives the same vector
    import torch

    yd = A.apply(torch.from_numpy(u).cuda())
    assert rel_l2(yd.cpu().numpy(), ref) <= 1e-12


def test_c2_48cubed_p3_all_dirichlet_value_parity():
    from paper_2509_10226_b200 import dofmap as D, operator as op

    m = _mesh(48, True)
    geo, bas = _tables(3)
    dm = D.build_dof_map(m, 3, "cg", 1, tuple(range(6)))
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    y = op.CgPoissonOperator(m, dm, geo, bas).apply(u)
    assert rel_l2(y, _cg_oracle(m, dm, geo, bas, u)) <= 1e-12
    assert np.array_equal(y[dm.dirichlet_mask], u[dm.dirichlet_mask])


def test_c3_64cubed_dg_sipg_p3_value_parity():
    """The full C3 mesh: 1,572,864 cells, 48 face windows."""
    from paper_2509_10226_b200 import dofmap as D, operator as op

    n, p = 64, 3
    m = _mesh(n, True)
    geo, bas = _tables(p)
    dm = D.build_dof_map(m, p, "dg")
    sipg = op.baseline_sipg_tau(m, p, 1.0 / n)
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    A = op.DgSipgOperator(m, dm, geo, bas, sipg, dirichlet_ids=range(6))
    assert m.n_cells > 32 * 32768
    y = A.apply(u)
    ref = _dg_oracle(m, dm, geo, bas, sipg, range(6), u)
    assert rel_l2(y, ref) <= 1e-12


def test_dg_sipg_p3_48cubed_unordered_value_parity():
    """Faces of the randomly permuted mesh: signatures and windows interleave at random."""
    from paper_2509_10226_b200 import dofmap as D, operator as op

    n, p = 48, 3
    m = _mesh(n, False)
    geo, bas = _tables(p)
    dm = D.build_dof_map(m, p, "dg")
    sipg = op.baseline_sipg_tau(m, p, 1.0 / n)
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    y = op.DgSipgOperator(m, dm, geo, bas, sipg, dirichlet_ids=(0, 3, 4)).apply(u)
    assert rel_l2(y, _dg_oracle(m, dm, geo, bas, sipg, (0, 3, 4), u)) <= 1e-12


def test_c4_kappa_helmholtz_p2_64cubed_value_parity():
    from paper_2509_10226_b200 import dofmap as D, operator as op

    n, p = 64, 2
    m = _mesh(n, True)
    geo, bas = _tables(p)
    dm = D.build_dof_map(m, p, "dg")
    sipg = op.baseline_sipg_tau(m, p, 1.0 / n)
    kap = 10.0 ** np.random.default_rng(2).uniform(-1, 1, m.n_cells)
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    y = op.KappaHelmholtzOperator(m, dm, geo, bas, sipg, kap, 1.0, dirichlet_ids=range(6)).apply(u)
    ref = _dg_oracle(m, dm, geo, bas, sipg, range(6), u, kappa=kap, mass_scale=1.0)
    assert rel_l2(y, ref) <= 1e-12


@pytest.mark.parametrize("engine", ["modal", "tensor"])
@pytest.mark.parametrize("p,n", [(2, 12), (3, 8), (4, 6)])
def test_kappa_helmholtz_cell_engines_vs_oracle(p, n, engine):
    """kappa-Helmholtz at P2-P4 (no reference golden above P2): the modal cell engine with the
    mass term as its own GEMM, and the reference tensor, against the oracle."""
    from paper_2509_10226_b200 import dofmap as D, operator as op

    m = _mesh(n, True)
    geo, bas = _tables(p)
    dm = D.build_dof_map(m, p, "dg")
    sipg = op.baseline_sipg_tau(m, p, 1.0 / n)
    kap = 10.0 ** np.random.default_rng(2).uniform(-1, 1, m.n_cells)
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    A = op.KappaHelmholtzOperator(m, dm, geo, bas, sipg, kap, 0.7, op.OperatorConfig(cell_engine=engine),
                                  dirichlet_ids=(0, 2, 5))
    assert A.info["cell_engine"] == {"modal": 4, "tensor": 3}[engine]
    ref = _dg_oracle(m, dm, geo, bas, sipg, (0, 2, 5), u, kappa=kap, mass_scale=0.7)
    assert rel_l2(A.apply(u), ref) <= 1e-12


def test_c5_jacobi_pcg_p3_24cubed_history():
    """C5's solver (CG P3, homogeneous Dirichlet, RHS U[-1,1] zero on constrained rows,
    100 Jacobi-PCG iterations) against the oracle PCG on the oracle apply."""
    import torch

    from oracle import ref_apply
    from paper_2509_10226_b200 import dofmap as D, operator as op
    from paper_2509_10226_b200.solvers import jacobi_pcg

    n, p, iters = 24, 3, 100
    m = _mesh(n, True)
    geo, bas = _tables(p)
    dm = D.build_dof_map(m, p, "cg", 1, tuple(range(6)))
    A = op.CgPoissonOperator(m, dm, geo, bas)
    b = np.where(dm.dirichlet_mask, 0.0, np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs))
    x, hist = jacobi_pcg(A, torch.from_numpy(b).cuda(), iters)
    diag = ref_apply.cg_diagonal(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask, bas.grad_matrix,
                                 geo.cell_rule.weights, dm.n_global_dofs)
    xr, hr = ref_apply.jacobi_pcg(lambda v: _cg_oracle(m, dm, geo, bas, v), diag, b, iters)
    assert len(hist) == len(hr) == iters + 1
    # each apply agrees to ~1e-15 (fp64 RED summation order differs from np.add.at); CG
    # amplifies that over the iterations: measured on B200 the histories agree to 1e-13 for
    # the first iterations and to 5e-8 after 100 (0.86105737 vs 0.86105733)
    assert np.allclose(hist[:21], hr[:21], rtol=1e-10, atol=0)
    assert np.allclose(hist, hr, rtol=1e-6, atol=0)
    assert rel_l2(x.cpu().numpy(), xr) <= 1e-6
    assert hist[-1] < 1e-2 * hist[0]


@pytest.mark.parametrize("kind", ["dg", "helmk"])
@pytest.mark.parametrize("p", [2, 3, 4])
def test_dg_cell_kernels_are_bitwise_repeatable(p, kind):
    """Race smoke test (no racecheck on this pool, DESIGN 3.3): the DG cell kernels store their
    rows (no REDs), so repeated launches must agree BIT FOR BIT; a race in the per-warp cp.async
    gather rings (DG P2 / P4, Helmholtz P2) or the staged tables would show up as run-to-run
    differences.  24^3 x 6 cells: several tiles per warp, the rings wrap."""
    import torch

    from paper_2509_10226_b200 import _lib, dofmap as D, operator as op

    n = 24
    m = _mesh(n, True)
    geo, bas = _tables(p)
    dm = D.build_dof_map(m, p, "dg")
    sipg = op.baseline_sipg_tau(m, p, 1.0 / n)
    if kind == "dg":
        A = op.DgSipgOperator(m, dm, geo, bas, sipg, dirichlet_ids=range(6))
    else:
        kap = 10.0 ** np.random.default_rng(2).uniform(-1, 1, m.n_cells)
        A = op.KappaHelmholtzOperator(m, dm, geo, bas, sipg, kap, 1.0, dirichlet_ids=range(6))
    u = torch.from_numpy(np.random.default_rng(p).uniform(-1, 1, dm.n_global_dofs)).cuda()
    st = torch.cuda.current_stream().cuda_stream
    ys = []
    for _ in range(6):
        y = torch.full_like(u, float("nan"))
        A.apply_stages(u.data_ptr(), y.data_ptr(), _lib.STAGE_CELLS, stream=st)
        torch.cuda.synchronize()
        ys.append(y)
    assert bool(torch.isfinite(ys[0]).all())
    for y in ys[1:]:
        assert torch.equal(y, ys[0])


@pytest.mark.parametrize("p,n,nu", [(1, 20, 0.3), (2, 20, 0.3), (3, 20, 0.3), (4, 10, 0.3), (2, 20, 0.0)])
def test_three_component_helmholtz_value_parity(p, n, nu):
    """HelmholtzOperator (operator.py:469-493: mass_scale M + nu A_sipg on 3 interleaved components)
    beyond the 48-cell goldens: 48,000 cells at n = 20 (more than one 32,768-cell face window,
    ragged last tile), against the oracle's 3-component loop; nu = 0 is the mass-only operator
    (no face kernels)."""
    from oracle import ref_apply
    from paper_2509_10226_b200 import dofmap as D, operator as op

    m = _mesh(n, True)
    geo, bas = _tables(p)
    dm = D.build_dof_map(m, p, "dg", 3)
    sipg = op.baseline_sipg_tau(m, p, 1.0 / n)
    co = op.HelmholtzCoefficients(0.8, nu)
    u = np.random.default_rng(7).uniform(-1, 1, dm.n_global_dofs)
    y = op.HelmholtzOperator(m, dm, geo, bas, sipg, co, dirichlet_ids=(0, 3)).apply(u)
    ref = ref_apply.dg_apply(m.vertices, m.cells, dm.n_dofs_per_cell, m.interior_faces, m.boundary_faces,
                             {0, 3}, bas.value_matrix, bas.grad_matrix, geo.cell_rule.weights,
                             bas.face_values, bas.face_grads, geo.face_rule.weights, sipg.tau_interior,
                             sipg.tau_boundary, u, mass_scale=0.8, stiff_scale=nu, n_components=3, chunk=65536)
    assert rel_l2(y, ref) <= 1e-12


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_three_component_cg_value_parity(p):
    """CG Laplace on 3 interleaved components (the reference's vector CG space; golden only at
    162 cells) at 24,576 cells with Dirichlet rows, component by component against the oracle."""
    from paper_2509_10226_b200 import dofmap as D, operator as op

    m = _mesh(16, True)
    geo, bas = _tables(p)
    dm = D.build_dof_map(m, p, "cg", 3, dirichlet_boundary_ids=(0, 5))
    u = np.random.default_rng(11).uniform(-1, 1, dm.n_global_dofs)
    y = op.CgPoissonOperator(m, dm, geo, bas).apply(u).reshape(-1, 3)
    uc = u.reshape(-1, 3)
    for c in range(3):
        ref = _cg_oracle(m, dm, geo, bas, uc[:, c])
        assert rel_l2(y[:, c], ref) <= 1e-12


@pytest.mark.parametrize("p,n", [(1, 24), (2, 24), (3, 24), (4, 24), (1, 48), (4, 48)])
def test_dependent_launch_clear_is_ordered_before_the_scatter(p, n):
    """Stress test of the y clear + programmatic dependent cell kernel (DESIGN 4.8): 40 applies
    back to back into a y refilled with garbage each time.  A RED that landed before the clear
    would be lost (or a stale value survive): every result must match the oracle-checked first
    one to RED-order round-off.  24^3: the P1 block kernel's CTAs are all resident while the
    clear runs (largest overlap); 48^3 P4: the longest clear."""
    import torch

    from paper_2509_10226_b200 import dofmap as D, operator as op

    m = _mesh(n, True)
    geo, bas = _tables(p)
    dm = D.build_dof_map(m, p, "cg")
    A = op.CgPoissonOperator(m, dm, geo, bas)
    u = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, dm.n_global_dofs)).cuda()
    st = torch.cuda.current_stream().cuda_stream
    y0 = torch.empty_like(u)
    A.apply_into(u.data_ptr(), y0.data_ptr(), st)
    if n <= 24:
        ref = _cg_oracle(m, dm, geo, bas, u.cpu().numpy())
        assert rel_l2(y0.cpu().numpy(), ref) <= 1e-12
    ys = [torch.empty_like(u) for _ in range(4)]
    worst = 0.0
    for r in range(10):
        for y in ys:
            y.fill_(1e300 if r % 2 else -7.0)
        for y in ys:                       # four applies queued back to back
            A.apply_into(u.data_ptr(), y.data_ptr(), st)
        torch.cuda.synchronize()
        for y in ys:
            worst = max(worst, float(torch.linalg.vector_norm(y - y0) / torch.linalg.vector_norm(y0)))
    assert worst <= 1e-13


@pytest.mark.parametrize("kind,p,n", [("dg", 3, 16), ("helmk", 2, 24), ("dg", 1, 24)])
def test_dg_dependent_launch_chain_is_ordered(kind, p, n):
    """The DG face kernels are programmatic dependents of the kernel before them (cell -> interior
    faces -> boundary faces): queued applies into garbage-filled y must all match the
    oracle-checked first result to RED-order round-off (a face RED overtaken by the cell kernel's
    row store would be lost)."""
    import torch

    from paper_2509_10226_b200 import dofmap as D, operator as op

    m = _mesh(n, True)
    geo, bas = _tables(p)
    dm = D.build_dof_map(m, p, "dg")
    sipg = op.baseline_sipg_tau(m, p, 1.0 / n)
    kap = 10.0 ** np.random.default_rng(2).uniform(-1, 1, m.n_cells) if kind == "helmk" else None
    if kind == "dg":
        A = op.DgSipgOperator(m, dm, geo, bas, sipg, dirichlet_ids=range(6))
    else:
        A = op.KappaHelmholtzOperator(m, dm, geo, bas, sipg, kap, 1.0, dirichlet_ids=range(6))
    un = np.random.default_rng(3).uniform(-1, 1, dm.n_global_dofs)
    u = torch.from_numpy(un).cuda()
    st = torch.cuda.current_stream().cuda_stream
    y0 = torch.empty_like(u)
    A.apply_into(u.data_ptr(), y0.data_ptr(), st)
    ref = _dg_oracle(m, dm, geo, bas, sipg, range(6), un, kappa=kap, mass_scale=1.0 if kind == "helmk" else 0.0)
    assert rel_l2(y0.cpu().numpy(), ref) <= 1e-12
    ys = [torch.empty_like(u) for _ in range(4)]
    worst = 0.0
    for r in range(8):
        for y in ys:
            y.fill_(1e300 if r % 2 else -7.0)
        for y in ys:
            A.apply_into(u.data_ptr(), y.data_ptr(), st)
        torch.cuda.synchronize()
        for y in ys:
            worst = max(worst, float(torch.linalg.vector_norm(y - y0) / torch.linalg.vector_norm(y0)))
    assert worst <= 1e-13
