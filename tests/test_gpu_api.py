"""GPU tests of the operator API surface (reference-compatible behaviour)."""

import numpy as np
import pytest

from conftest import load_golden, rel_l2
from helpers import fixture_objects, operator_from_fixture

pytestmark = pytest.mark.gpu


def test_length_mismatch_raises_value_error():
    A = operator_from_fixture(load_golden("cg_p1_n4_ref"))
    with pytest.raises(ValueError, match="does not match"):
        A.apply(np.zeros(A.n_global_dofs + 1))


def test_torch_cuda_tensor_roundtrip_and_counters():
    import torch

    g = load_golden("dg_p2_n3_gm_dir")
    A = operator_from_fixture(g)
    u = torch.from_numpy(g["u"]).cuda()
    y = A.apply(u)
    assert y.is_cuda and y.dtype == torch.float64
    assert rel_l2(y.cpu().numpy(), g["y"]) <= 1e-12
    y2 = A.apply(g["u"])
    assert A.n_applies == 2
    assert A.counters.total_flops == 2 * A._apply_counts["cell_interp_flops"] + 2 * (
        A._apply_counts["cell_qpoint_flops"] + A._apply_counts["cell_sum_flops"]
        + A._apply_counts["face_interp_flops"] + A._apply_counts["face_qpoint_flops"])
    assert A.counters["vector_bytes"] == 2 * 24 * A.n_global_dofs
    assert rel_l2(y2, g["y"]) <= 1e-12


def test_out_buffer_and_async_host_path():
    import torch

    g = load_golden("cg_p2_n8_gm_dir")
    A = operator_from_fixture(g)
    out = np.empty_like(g["u"])
    A.apply(g["u"], out=out)
    assert rel_l2(out, g["y"]) <= 1e-12
    u_pin = torch.from_numpy(g["u"]).pin_memory()
    y_pin = torch.empty_like(u_pin).pin_memory()
    s = torch.cuda.Stream()
    A.apply_host_async(u_pin, y_pin, s.cuda_stream)
    s.synchronize()
    assert rel_l2(y_pin.numpy(), g["y"]) <= 1e-12


def test_host_multi_pipeline_matches_goldens():
    """tmf_apply_host_multi: CG and DG plans (mixed sizes, one plan twice) in one pipelined
    call give the golden results; a length mismatch or an empty list is handled."""
    import torch

    from paper_2509_10226_b200 import operator as op

    names = ["cg_p2_n8_gm_dir", "dg_p3_n3_gm_dir", "cg_p4_n3_gm", "helmk_p2_n3_gm_dir"]
    gs = [load_golden(n) for n in names]
    ops = [operator_from_fixture(g) for g in gs]
    ops.append(ops[0])
    gs.append(gs[0])
    us = [torch.from_numpy(np.ascontiguousarray(g["u"])).pin_memory() for g in gs]
    ys = [torch.full_like(u, np.nan).pin_memory() for u in us]
    s = torch.cuda.Stream()
    op.apply_host_multi(ops, us, ys, s.cuda_stream)
    s.synchronize()
    for g, y in zip(gs, ys):
        assert rel_l2(y.numpy(), g["y"]) <= 1e-12
    assert ops[0].n_applies == 2
    op.apply_host_multi([], [], [], s.cuda_stream)
    with pytest.raises(ValueError, match="operator size"):
        op.apply_host_multi(ops[:1], us[1:2], ys[1:2])
    # host buffers must be float64, contiguous, on the host
    with pytest.raises(ValueError, match="host buffers"):
        op.apply_host_multi(ops[:1], [us[0].float()], ys[:1])
    with pytest.raises(ValueError, match="host buffers"):
        op.apply_host_multi(ops[:1], [us[0].cuda()], ys[:1])
    with pytest.raises(ValueError, match="host buffers"):
        ops[0].apply_host_async(us[0], ys[0][::1].cuda(), s.cuda_stream)
    with pytest.raises(ValueError, match="differ in length"):
        op.apply_host_multi(ops[:2], us[:1], ys[:2])


def test_wrong_space_and_missing_faces():
    from paper_2509_10226_b200 import operator as op

    g = load_golden("dg_p1_n3_ref_dir")
    mesh, dofmap, geo, basis = fixture_objects(g)
    with pytest.raises(ValueError, match="CG operator needs a CG dof map"):
        op.CgPoissonOperator(mesh, dofmap, geo, basis)
    geo.face_rule = None
    with pytest.raises(ValueError, match="face data"):
        op.DgSipgOperator(mesh, dofmap, geo, basis, op.SipgConfig(1.0, g["tau_i"], g["tau_b"]))


def test_nonpositive_penalty_rejected():
    from paper_2509_10226_b200 import operator as op

    g = load_golden("dg_p1_n3_ref_dir")
    mesh, dofmap, geo, basis = fixture_objects(g)
    tau = g["tau_i"].copy()
    tau[3] = 0.0
    with pytest.raises(ValueError, match="penalty"):
        op.DgSipgOperator(mesh, dofmap, geo, basis, op.SipgConfig(1.0, tau, g["tau_b"]))


def test_reference_objects_are_accepted_duck_typed():
    """The shim reads only array fields, so objects shaped like the reference's work."""
    g = load_golden("helm3_p1_n2_ref_dir")
    A = operator_from_fixture(g)
    assert A.n_global_dofs == len(g["u"])
    assert rel_l2(A.apply(g["u"]), g["y"]) <= 1e-12


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_reordered_mesh_gives_same_operator(p):
    """Hierarchical reordering permutes cells (and so the CG numbering); the operator
    applied to the correspondingly permuted vector is the permuted result."""
    from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, operator as op, quadrature as Q
    from paper_2509_10226_b200.geometry import GeometryData
    from paper_2509_10226_b200.reorder import hierarchical_reorder

    m = M.kuhn_cube_mesh(4, seed=1)
    m2 = M.apply_cell_permutation(m, hierarchical_reorder(m))
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    d1, d2 = D.build_dof_map(m, p, "cg"), D.build_dof_map(m2, p, "cg")
    # DoF correspondence through the (identical) physical node positions of each cell
    order = np.argsort(hierarchical_reorder(m))
    perm = np.empty(d1.n_global_dofs, dtype=np.int64)
    perm[d2.cell_dofs.ravel()] = d1.cell_dofs[order].ravel()      # new dof -> old dof
    u1 = np.random.default_rng(0).uniform(-1, 1, d1.n_global_dofs)
    y1 = op.CgPoissonOperator(m, d1, geo, bas).apply(u1)
    y2 = op.CgPoissonOperator(m2, d2, geo, bas).apply(u1[perm])
    assert rel_l2(y2, y1[perm]) <= 1e-13


@pytest.mark.parametrize("name", ["cg_p2_n8_gm", "cg_p3_n4_ref_dir", "cg_p4_n3_gm_dir"])
def test_gpu_csr_baseline_matches_reference_csr(name):
    from paper_2509_10226_b200.sparse import CsrOperator

    g = load_golden(name)
    mesh, dofmap, geo, basis = fixture_objects(g)
    A = CsrOperator(mesh, dofmap, geo, basis)
    assert rel_l2(A.apply(g["u"]), g["y_csr"]) <= 1e-12


def _single_tet_problem(p, space):
    from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, quadrature as Q
    from paper_2509_10226_b200.geometry import GeometryData

    v = np.array([[0.1, 0.0, 0.0], [1.0, 0.2, 0.0], [0.0, 1.1, 0.1], [0.2, 0.1, 0.9]])
    cells = np.array([[0, 1, 2, 3]], dtype=np.int32)
    ifc, bfc = M.build_faces(cells, v, lambda c: np.arange(len(c)) % 6)
    m = M.TetMesh(v, cells, ifc, bfc)
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    return m, D.build_dof_map(m, p, space), geo, bas


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_single_cell_edge_case(p):
    """One cell: 1 tile with 7 padded slots, no interior faces, 4 boundary faces."""
    from oracle import ref_apply
    from paper_2509_10226_b200 import operator as op

    m, dm, geo, bas = _single_tet_problem(p, "cg")
    u = np.random.default_rng(p).uniform(-1, 1, dm.n_global_dofs)
    y = op.CgPoissonOperator(m, dm, geo, bas).apply(u)
    ref = ref_apply.cg_apply(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask, bas.grad_matrix,
                             geo.cell_rule.weights, u)
    assert rel_l2(y, ref) <= 1e-12
    m, dm, geo, bas = _single_tet_problem(p, "dg")
    sipg = op.SipgConfig(1.0, np.zeros(0), np.full(4, 10.0))
    y = op.DgSipgOperator(m, dm, geo, bas, sipg, dirichlet_ids=(1, 3)).apply(u)
    ref = ref_apply.dg_apply(m.vertices, m.cells, dm.n_dofs_per_cell, m.interior_faces, m.boundary_faces, {1, 3},
                             bas.value_matrix, bas.grad_matrix, geo.cell_rule.weights, bas.face_values,
                             bas.face_grads, geo.face_rule.weights, np.zeros(0), np.full(4, 10.0), u)
    assert rel_l2(y, ref) <= 1e-12


def test_all_dofs_constrained_is_identity():
    from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, operator as op, quadrature as Q
    from paper_2509_10226_b200.geometry import GeometryData

    m = M.kuhn_cube_mesh(1, seed=0)   # every vertex is on the boundary
    cr, fr = Q.make_cell_quadrature(1), Q.make_face_quadrature(1)
    dm = D.build_dof_map(m, 1, "cg", 1, tuple(range(6)))
    assert dm.dirichlet_mask.all()
    A = op.CgPoissonOperator(m, dm, GeometryData("affine", cr, fr, None, None, None, None),
                             B.tabulate_basis(1, cr, fr))
    u = np.arange(dm.n_global_dofs, dtype=np.float64)
    assert np.array_equal(A.apply(u), u)


@pytest.mark.parametrize("n", [1, 2, 5])
def test_ragged_tile_counts(n):
    """Cell counts that are not multiples of the 8-cell tile / 2-tile super-tile."""
    from oracle import ref_apply
    from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, operator as op, quadrature as Q
    from paper_2509_10226_b200.geometry import GeometryData

    m = M.kuhn_cube_mesh(n, seed=9)
    m = M.TetMesh(m.vertices, m.cells[:-3], *M.build_faces(m.cells[:-3], m.vertices, M.cube_boundary_ids))
    for p in (1, 2, 3):
        cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
        bas = B.tabulate_basis(p, cr, fr)
        geo = GeometryData("affine", cr, fr, None, None, None, None)
        dm = D.build_dof_map(m, p, "cg")
        used = np.zeros(dm.n_scalar_dofs, bool)
        used[dm.cell_dofs.ravel()] = True
        u = np.random.default_rng(p).uniform(-1, 1, dm.n_global_dofs) * used
        y = op.CgPoissonOperator(m, dm, geo, bas).apply(u)
        ref = ref_apply.cg_apply(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask, bas.grad_matrix,
                                 geo.cell_rule.weights, u)
        assert rel_l2(y, ref) <= 1e-12


def test_c_abi_demo_runs():
    """The plain-C demo (examples/c_abi_demo.c) passes on the GPU."""
    import os
    import shutil
    import subprocess

    from conftest import ROOT
    from paper_2509_10226_b200 import _lib

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    out = os.path.join(ROOT, "examples", "c_abi_demo")
    subprocess.run(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "examples", "c_abi_demo.c"),
                    "-L", os.path.dirname(_lib.LIB_PATH), "-ltetmf_b200",
                    f"-Wl,-rpath,{os.path.dirname(_lib.LIB_PATH)}", "-lm", "-o", out], check=True)
    r = subprocess.run([out], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout


def test_host_multi_same_plan_adjacent_different_inputs():
    """one plan twice in a row with DIFFERENT inputs, and the plan's
    async host apply on another stream right after: the staging buffers are ordered by the
    plan's stage event, so every output is its own input's apply."""
    import torch

    from paper_2509_10226_b200 import operator as op

    g = load_golden("cg_p2_n8_gm_dir")
    A = operator_from_fixture(g)
    rng = np.random.default_rng(9)
    us = [torch.from_numpy(rng.uniform(-1, 1, A.n_global_dofs)).pin_memory() for _ in range(3)]
    ys = [torch.full_like(u, np.nan).pin_memory() for u in us]
    refs = [A.apply(u.numpy()) for u in us]
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        for y in ys:
            y.fill_(np.nan)
        op.apply_host_multi([A, A], us[:2], ys[:2], s1.cuda_stream)
        A.apply_host_async(us[2], ys[2], s2.cuda_stream)
        torch.cuda.synchronize()
        for y, r in zip(ys, refs):
            assert rel_l2(y.numpy(), r) <= 1e-14


def test_counters_follow_reference_batching():
    """Row a23: the reference counter categories, per apply, from the reference's batching
    (the values themselves are pinned against the real reference in tests/test_counters.py)."""
    from paper_2509_10226_b200 import operator as op
    from paper_2509_10226_b200.counters import reference_apply_counts

    g = load_golden("dg_p3_n3_gm_dir")
    mesh, dofmap, geo, basis = fixture_objects(g)
    sipg = op.SipgConfig(1.0, g["tau_i"], g["tau_b"])
    cfg = op.OperatorConfig(kernel_stage="ref", lane_width=8)
    A = op.DgSipgOperator(mesh, dofmap, geo, basis, sipg, cfg, dirichlet_ids=range(6))
    A.apply(g["u"])
    inc = reference_apply_counts(cfg, dofmap, len(geo.cell_rule.weights), len(geo.face_rule.weights),
                                 interior_faces=mesh.interior_faces, boundary_faces=mesh.boundary_faces,
                                 dirichlet_ids=range(6), faces=True)
    d = A.counters.as_dict()
    assert all(d[k] == v for k, v in inc.items())
    assert d["face_interp_flops"] > 0 and d["index_bytes"] > 0 and d["geometry_bytes"] > 0


def test_geometry_mode_and_precision_boundary():
    """geometry.py:139-142 (unknown mode, affine on curved), per-point geometry of straight
    cells (= the affine map), precision="f32" (CG: float32 result; DG: rejected)."""
    from types import SimpleNamespace as NS

    import torch

    from paper_2509_10226_b200 import operator as op

    g = load_golden("cg_p2_n8_gm_dir")
    mesh, dofmap, geo, basis = fixture_objects(g)
    geo.mode = "bogus"
    with pytest.raises(ValueError, match="unknown geometry mode"):
        op.CgPoissonOperator(mesh, dofmap, geo, basis)
    geo.mode = "affine"
    curved = NS(**vars(mesh), geometry_nodes=np.zeros((len(g["cells"]), 10, 3)), is_curved=True)
    with pytest.raises(ValueError, match="curved"):
        op.CgPoissonOperator(curved, dofmap, geo, basis)
    geo.mode = "per_point"
    with pytest.raises(ValueError, match="curved"):
        op.CgPoissonOperator(curved, dofmap, geo, basis)
    A = op.CgPoissonOperator(mesh, dofmap, geo, basis)          # straight cells: same operator
    assert rel_l2(A.apply(g["u"]), g["y"]) <= 1e-12
    assert A.counters["geometry_bytes"] > 0
    geo.mode = "affine"
    A32 = op.CgPoissonOperator(mesh, dofmap, geo, basis, op.OperatorConfig(precision="f32"))
    y32 = A32.apply(g["u"])
    assert y32.dtype == np.float32
    assert rel_l2(y32.astype(np.float64), g["y"]) <= 1e-5
    yt = A32.apply(torch.from_numpy(g["u"]).cuda())
    assert yt.dtype == torch.float32 and rel_l2(yt.cpu().double().numpy(), g["y"]) <= 1e-5
    gd = load_golden("dg_p2_n3_gm_dir")
    mesh, dofmap, geo, basis = fixture_objects(gd)
    with pytest.raises(ValueError, match="f32"):
        op.DgSipgOperator(mesh, dofmap, geo, basis, op.SipgConfig(1.0, gd["tau_i"], gd["tau_b"]),
                          op.OperatorConfig(precision="f32"))


@pytest.mark.parametrize("name", ["cg_p1_n4_ref", "cg_p2_n8_gm_dir", "cg_p3_n4_ref_dir", "cg_p4_n3_gm_dir"])
def test_y_clear_kernel_unaligned_and_stale_output(name):
    """The CG apply clears y with its own kernel (16-byte stores behind an 8-byte head / tail) and
    launches the cell kernel as its programmatic dependent: a y that starts 8 bytes off a 16-byte
    boundary and holds stale values must come out the same, with the neighbouring entries untouched."""
    import torch

    g = load_golden(name)
    A = operator_from_fixture(g)
    n = A.n_global_dofs
    u = torch.from_numpy(g["u"]).cuda()
    st = torch.cuda.current_stream().cuda_stream
    for off in (0, 1):
        buf = torch.full((n + 4,), 7.5, dtype=torch.float64, device="cuda")
        y = buf[off + 1: off + 1 + n]
        for _ in range(3):   # repeated applies: the clear must not race the previous apply's REDs
            A.apply_into(u.data_ptr(), y.data_ptr(), st)
        torch.cuda.synchronize()
        assert rel_l2(y.cpu().numpy(), g["y"]) <= 1e-12
        assert float(buf[off]) == 7.5 and float(buf[off + 1 + n]) == 7.5


def test_plain_launch_path_matches(tmp_path):
    """TMF_PDL=0 (cudaMemsetAsync + plain launch) gives the same y as the default dependent launch."""
    import os
    import subprocess
    import sys

    g = load_golden("cg_p2_n8_gm_dir")
    y_pdl = operator_from_fixture(g).apply(g["u"])
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r);"
            "from conftest import load_golden; from helpers import operator_from_fixture;"
            "g = load_golden('cg_p2_n8_gm_dir'); np.save(%r, operator_from_fixture(g).apply(g['u']))"
            % (root, os.path.join(root, "tests"), str(tmp_path / "y.npy")))
    subprocess.run([sys.executable, "-c", code], check=True, env=dict(os.environ, TMF_PDL="0"), timeout=300)
    y_plain = np.load(tmp_path / "y.npy")
    assert rel_l2(y_plain, g["y"]) <= 1e-12
    assert rel_l2(y_plain, y_pdl) <= 1e-14
