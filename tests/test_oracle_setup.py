"""The vectorised oracle setup (oracle/ref_mesh.py) -- what the bench's reference arm
builds its workload with -- against the loop restatements (oracle/ref_setup.py), the
reference fixtures, and the product's native setup (bit-exact integer data)."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import ref_mesh, ref_reorder, ref_setup


def test_faces_match_loop_oracle_and_product():
    from paper_2509_10226_b200 import mesh as M

    v, c, fi, fb = ref_mesh.kuhn_mesh(5, seed=3)
    li, lb = ref_setup.build_faces(c, lambda x: int(ref_mesh._cube_ids(x[None])[0]), v)
    assert np.array_equal(fi, li) and np.array_equal(fb, lb)
    m = M.kuhn_cube_mesh(5, seed=3)
    assert np.array_equal(m.vertices, v) and np.array_equal(m.cells, c)
    assert np.array_equal(m.interior_faces, fi) and np.array_equal(m.boundary_faces, fb)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_cg_dofs_match_loop_oracle(p):
    v, c, fi, fb = ref_mesh.kuhn_mesh(4, seed=1)
    cd, ns = ref_mesh.cg_dofs(c, len(v), p)
    lcd, lmask, lns = ref_setup.build_cg_dofs(c, len(v), p, fb, (0, 3, 5))
    assert ns == lns and np.array_equal(cd, lcd)
    assert np.array_equal(ref_mesh.dirichlet_mask(cd, ns, p, fb, (0, 3, 5)), lmask)


@pytest.mark.parametrize("name", ["cg_p1_n4_ref_dir", "cg_p2_n8_gm_dir", "cg_p3_n4_ref_dir", "cg_p4_n3_gm_dir"])
def test_cg_dofs_match_reference_fixtures(name):
    g = load_golden(name)
    cd, ns = ref_mesh.cg_dofs(g["cells"], len(g["vertices"]), int(g["p"]))
    assert np.array_equal(cd, g["cell_dofs"]) and ns == len(g["dirichlet_mask"])
    mask = ref_mesh.dirichlet_mask(cd, ns, int(g["p"]), g["boundary_faces"], [int(x) for x in g["dirichlet_ids"]])
    assert np.array_equal(mask, g["dirichlet_mask"])
    fi, fb = ref_mesh.build_faces(g["cells"], g["vertices"])
    assert np.array_equal(fi, g["interior_faces"]) and np.array_equal(fb, g["boundary_faces"])


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_bench_workload_matches_product_setup(p):
    """The reordered C2 workload as the reference arm builds it (oracle only) equals the
    one the B200 arm builds (native C++ setup + reorder_mesh) on a 10^3 mesh."""
    from paper_2509_10226_b200 import dofmap as D, mesh as M
    from paper_2509_10226_b200.reorder import reorder_mesh

    v, c, fi, fb = ref_mesh.kuhn_mesh(10, seed=0)
    c2, fi2, fb2 = ref_mesh.permute_cells(c, fb, ref_reorder.hierarchical_reorder(len(c), fi))
    v3, c3, fi3, fb3 = ref_mesh.first_touch_vertices(v, c2, fb2)
    m = reorder_mesh(M.kuhn_cube_mesh(10, seed=0))
    assert np.array_equal(m.vertices, v3) and np.array_equal(m.cells, c3)
    assert np.array_equal(m.interior_faces, fi3) and np.array_equal(m.boundary_faces, fb3)
    cd, ns = ref_mesh.cg_dofs(c3, len(v3), p)
    dm = D.build_dof_map(m, p, "cg")
    assert ns == dm.n_scalar_dofs and np.array_equal(cd, dm.cell_dofs)


def test_reorder_bit_exact_at_bench_size():
    """The product's C++ hierarchical reordering equals the oracle's restatement on the 48^3
    C2 mesh the bench reorders (663,552 cells)."""
    from paper_2509_10226_b200 import mesh as M
    from paper_2509_10226_b200.reorder import hierarchical_reorder

    m = M.kuhn_cube_mesh(48, seed=0)
    assert np.array_equal(hierarchical_reorder(m), ref_reorder.hierarchical_reorder(m.n_cells, m.interior_faces))
