"""CPU tests: host setup vs the oracle restatements, the C-ABI library surface,
quadrature/basis properties.  No GPU needed."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden_names, load_golden
from oracle import ref_reorder, ref_setup
from paper_2509_10226_b200 import _lib, basis as B, dofmap as D, mesh as M, quadrature as Q, reorder as R
from paper_2509_10226_b200.reference import PERMS


# ------------------------------------------------------------------ C-ABI surface
def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "tetmf_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char\*)\s+(tmf_\w+)\s*\(", hdr, re.M))
    assert declared == set(_lib.EXPORTED)
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(L, name), name
    assert b"sm_100a" in _lib.lib().tmf_version()


def test_plan_create_rejects_bad_descriptors():
    d = _lib.PlanDesc()
    d.operator_kind = 7
    plan = ctypes.c_void_p()
    with pytest.raises(ValueError, match="unknown operator kind"):
        _lib.check(_lib.lib().tmf_plan_create(ctypes.byref(d), ctypes.byref(plan)))
    d.operator_kind = _lib.TMF_CG_LAPLACE
    d.degree = 5
    with pytest.raises(ValueError, match="unsupported polynomial degree"):
        _lib.check(_lib.lib().tmf_plan_create(ctypes.byref(d), ctypes.byref(plan)))


@pytest.mark.parametrize("blocked,run", [(0, 0), (1, 0), (1, 1), (1, 2), (1, 8)])
@pytest.mark.parametrize("n_work,grid", [(0, 4), (1, 296), (295, 296), (296, 296), (1000, 296), (12345, 148), (37, 5)])
def test_face_chunk_walk_visits_every_chunk_once(n_work, grid, blocked, run):
    """The CTA walks of the face kernels (face_kernel.cuh ChunkWalk, through the host test
    hook): over all CTAs every chunk exactly once; blocked runs are consecutive chunks."""
    L = _lib.lib()
    seen = []
    for b in range(grid):
        out = (ctypes.c_int64 * (n_work + 1))()
        n = ctypes.c_int64()
        _lib.check(L.tmf_debug_chunk_walk(n_work, grid, b, blocked, run, out, n_work + 1, ctypes.byref(n)))
        w = list(out[: n.value])
        if blocked and run == 0:
            assert w == list(range(w[0], w[0] + len(w))) if w else True
        if blocked and run > 0:
            for k in range(0, len(w), run):   # each run: consecutive chunks starting at a multiple of run
                r = w[k:k + run]
                assert r[0] % run == 0 and r == list(range(r[0], r[0] + len(r)))
        seen += w
    assert sorted(seen) == list(range(n_work))


# ------------------------------------------------------------------ mesh / faces
@pytest.mark.parametrize("n,seed", [(1, 0), (2, 5), (3, 1)])
def test_build_faces_matches_oracle(n, seed):
    m = M.kuhn_cube_mesh(n, seed=seed)
    ifc, bfc = ref_setup.build_faces(m.cells, lambda c: int(M.cube_boundary_ids(c[None])[0]), m.vertices)
    assert np.array_equal(ifc, m.interior_faces)
    assert np.array_equal(bfc, m.boundary_faces)
    m.validate()
    assert len(m.interior_faces) == 12 * n ** 3 - 6 * n ** 2
    assert len(m.boundary_faces) == 12 * n ** 2


def test_mesh_generator_deterministic_and_positive():
    a, b = M.kuhn_cube_mesh(4, seed=7), M.kuhn_cube_mesh(4, seed=7)
    assert np.array_equal(a.cells, b.cells) and np.array_equal(a.vertices, b.vertices)
    assert np.all(a.cell_volumes() > 0)
    assert abs(a.cell_volumes().sum() - 1.0) < 1e-12
    assert sorted(set(a.boundary_faces[:, 2].tolist())) == [0, 1, 2, 3, 4, 5]


def test_golden_meshes_rebuild_identically():
    for name in golden_names("cg_p2_n8"):
        g = load_golden(name)
        ifc, bfc = M.build_faces(g["cells"], g["vertices"], M.cube_boundary_ids)
        assert np.array_equal(ifc, g["interior_faces"])
        assert np.array_equal(bfc, g["boundary_faces"])


# ------------------------------------------------------------------ DoF maps
@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("dids", [(), (0, 1, 2, 3, 4, 5), (2, 5)])
def test_cg_dofmap_matches_oracle(p, dids):
    m = M.kuhn_cube_mesh(3, seed=2)
    dm = D.build_dof_map(m, p, "cg", 1, dids)
    cd, mask, n = ref_setup.build_cg_dofs(m.cells, m.n_vertices, p, m.boundary_faces, dids)
    assert dm.n_scalar_dofs == n == (3 * p + 1) ** 3
    assert np.array_equal(dm.cell_dofs, cd)
    assert np.array_equal(dm.dirichlet_mask, mask)


def test_dofmap_errors():
    m = M.kuhn_cube_mesh(2)
    with pytest.raises(ValueError):
        D.build_dof_map(m, 2, "xx")
    with pytest.raises(ValueError):
        D.build_dof_map(m, 2, "cg", dirichlet_boundary_ids=(9,))
    with pytest.raises(ValueError):
        D.build_dof_map(m, 2, "cg", n_components=2)


def test_golden_dofmaps_rebuild_identically():
    for name in golden_names("cg_"):
        g = load_golden(name)
        m = M.TetMesh(g["vertices"], g["cells"], g["interior_faces"], g["boundary_faces"])
        dm = D.build_dof_map(m, int(g["p"]), "cg", 1, tuple(g["dirichlet_ids"].tolist()))
        assert np.array_equal(dm.cell_dofs, g["cell_dofs"]), name
        assert np.array_equal(dm.dirichlet_mask, g["dirichlet_mask"]), name


def test_colouring_oracle_smoke():
    m = M.kuhn_cube_mesh(2, seed=0)
    dm = D.build_dof_map(m, 1, "cg")
    ids = np.arange(m.n_cells).reshape(-1, 16)
    col = ref_setup.color_batches(dm.cell_dofs, ids, np.ones_like(ids, bool))
    for b in range(len(ids)):
        for c in range(b):
            if col[b] == col[c]:
                assert not set(dm.cell_dofs[ids[b]].ravel()) & set(dm.cell_dofs[ids[c]].ravel())


# ------------------------------------------------------------------ quadrature / basis
@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_gm_rules(p):
    c, f = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    assert (c.n_points, f.n_points) == ({1: 5, 2: 15, 3: 35, 4: 70}[p], {1: 4, 2: 10, 3: 20, 4: 35}[p])
    assert Q.monomial_exactness(c) >= 2 * p and Q.monomial_exactness(f) >= 2 * p
    for perm in PERMS:
        assert Q.symmetric_point_permutation(f.points, perm) is not None


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_basis_nodal_and_partition_of_unity(p):
    nodes, tags = B.reference_nodes(p)
    assert len(nodes) == B.n_dofs_per_cell(p) == len(tags)
    assert np.allclose(B.lagrange_values(p, nodes), np.eye(len(nodes)), atol=1e-10)
    b = B.tabulate_basis(p, Q.make_cell_quadrature(p), Q.make_face_quadrature(p))
    assert np.allclose(b.value_matrix.sum(axis=1), 1.0)
    assert np.allclose(b.grad_matrix.sum(axis=1), 0.0, atol=1e-10)
    assert b.face_values.shape == (4, 6, b.n_qf, len(nodes))


def test_basis_tables_match_reference_fixtures():
    for name in golden_names("cg_p"):
        g = load_golden(name)
        p = int(g["p"])
        cr = Q.QuadratureRule(g["cell_points"], g["cell_weights"], 2 * p, 3)
        fr = Q.QuadratureRule(g["face_points"], g["face_weights"], 2 * p, 2)
        b = B.tabulate_basis(p, cr, fr)
        assert np.allclose(b.grad_matrix, g["grad_matrix"], atol=1e-11), name
        assert np.allclose(b.face_grads, g["face_grads"], atol=1e-11), name


# ------------------------------------------------------------------ reordering
@pytest.mark.parametrize("n,seed", [(2, 0), (3, 4), (5, 1)])
def test_reorder_bit_exact_vs_oracle(n, seed):
    m = M.kuhn_cube_mesh(n, seed=seed)
    a = R.hierarchical_reorder(m)
    b = ref_reorder.hierarchical_reorder(m.n_cells, m.interior_faces)
    assert np.array_equal(a, b)
    assert np.array_equal(np.sort(a), np.arange(m.n_cells))


def test_reorder_spec_acceptance_on_reference_fixture():
    """on the reference's seed-42 shuffled 5*8^3 mesh the reordering cuts the
    mean neighbour index distance >= 2x and the max bandwidth >= 4x."""
    g = load_golden("mesh_5tet_n8_shuffled42")
    m = M.TetMesh(g["vertices"], g["cells"], g["interior_faces"], g["boundary_faces"])
    nb = R.hierarchical_reorder(m)
    assert np.array_equal(nb, ref_reorder.hierarchical_reorder(m.n_cells, m.interior_faces))
    m2 = M.apply_cell_permutation(m, nb)
    before, after = R.locality_metrics(m), R.locality_metrics(m2)
    assert after["mean_neighbor_index_distance"] * 2 <= before["mean_neighbor_index_distance"]
    assert after["max_bandwidth"] * 4 <= before["max_bandwidth"]
    m2.validate()


def test_reorder_improves_locality_spec_acceptance():
    m = M.kuhn_cube_mesh(8, seed=0)
    m2 = M.apply_cell_permutation(m, R.hierarchical_reorder(m))
    before, after = R.locality_metrics(m), R.locality_metrics(m2)
    assert after["mean_neighbor_index_distance"] * 2 <= before["mean_neighbor_index_distance"]
    m2.validate()


def test_reorder_chain_and_determinism():
    # shuffled chain of 256 cells as a face graph: bandwidth must collapse
    rng = np.random.default_rng(0)
    perm = rng.permutation(256)
    faces = np.array([[perm[i], 0, perm[i + 1], 0, 0] for i in range(255)], dtype=np.int32)
    faces[:, [0, 2]] = np.sort(faces[:, [0, 2]], axis=1)
    nb = ref_reorder.hierarchical_reorder(256, faces)
    nb2 = ref_reorder.hierarchical_reorder(256, faces)
    assert np.array_equal(nb, nb2)
    d = np.abs(nb[faces[:, 0]] - nb[faces[:, 2]])
    assert d.max() <= 16


# ------------------------------------------------------------------ native (C++) vs numpy setup
@pytest.mark.parametrize("n,seed", [(2, 0), (4, 3)])
def test_native_setup_matches_numpy_path(n, seed):
    m = M.kuhn_cube_mesh(n, seed=seed)
    a = M.build_faces(m.cells, m.vertices, M.cube_boundary_ids, method="native")
    b = M.build_faces(m.cells, m.vertices, M.cube_boundary_ids, method="numpy")
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    for p in (1, 2, 3, 4):
        x = D.build_dof_map(m, p, "cg", 1, (0, 3), method="native")
        y = D.build_dof_map(m, p, "cg", 1, (0, 3), method="numpy")
        assert x.n_scalar_dofs == y.n_scalar_dofs
        assert np.array_equal(x.cell_dofs, y.cell_dofs)
        assert np.array_equal(x.dirichlet_mask, y.dirichlet_mask)


def test_native_faces_reject_nonmanifold():
    cells = np.array([[0, 1, 2, 3], [0, 1, 2, 4], [0, 1, 2, 5]], dtype=np.int32)
    with pytest.raises(ValueError):
        M.build_faces(cells)


def test_c_abi_demo_compiles_against_header_and_library():
    """A plain-C caller of include/tetmf_b200.h links against libtetmf_b200.so (gcc)."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    out = os.path.join(ROOT, "examples", "c_abi_demo")
    r = subprocess.run(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "examples", "c_abi_demo.c"), "-L", os.path.dirname(_lib.LIB_PATH),
                        "-ltetmf_b200", f"-Wl,-rpath,{os.path.dirname(_lib.LIB_PATH)}", "-lm", "-o", out],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


@pytest.mark.parametrize("p", [1, 2])
def test_vertex_renumbering_is_a_permutation_of_the_operator(p):
    """reorder_mesh's first-touch vertex numbering relabels vertices only: the mesh stays
    valid and positive, boundary ids survive, and the CG operator (oracle) on the new mesh
    equals the old one up to the DoF relabelling (P1: DoF = vertex id)."""
    from oracle import ref_apply

    m = M.apply_cell_permutation(M.kuhn_cube_mesh(4, seed=3), R.hierarchical_reorder(M.kuhn_cube_mesh(4, seed=3)))
    nov = M.first_touch_vertex_order(m)
    m2 = M.apply_vertex_permutation(m, nov)
    m2.validate()
    assert np.all(np.linalg.det(m2.cell_jacobians()) > 0)
    assert np.array_equal(np.sort(nov), np.arange(m.n_vertices))
    assert np.array_equal(np.bincount(m2.boundary_faces[:, 2]), np.bincount(m.boundary_faces[:, 2]))
    # first touch: the vertices of the first cell are 0..3
    assert sorted(m2.cells[0].tolist()) == [0, 1, 2, 3]
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    d1, d2 = D.build_dof_map(m, p, "cg"), D.build_dof_map(m2, p, "cg")
    u1 = np.random.default_rng(1).uniform(-1, 1, d1.n_global_dofs)
    y1 = ref_apply.cg_apply(m.vertices, m.cells, d1.cell_dofs, d1.dirichlet_mask, bas.grad_matrix, cr.weights, u1)
    # DoF relabelling old -> new through the cell-local DoF lists (same cells, same local order)
    new_of_old = np.empty(d1.n_global_dofs, dtype=np.int64)
    new_of_old[d1.cell_dofs.ravel()] = d2.cell_dofs.ravel()
    u2 = np.empty_like(u1)
    u2[new_of_old] = u1
    y2 = ref_apply.cg_apply(m2.vertices, m2.cells, d2.cell_dofs, d2.dirichlet_mask, bas.grad_matrix, cr.weights, u2)
    assert np.linalg.norm(y2[new_of_old] - y1) <= 1e-13 * np.linalg.norm(y1)
    with pytest.raises(ValueError):
        M.apply_vertex_permutation(m, np.zeros(m.n_vertices, dtype=np.int64))
