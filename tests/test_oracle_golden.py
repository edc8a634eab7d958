"""Pin the CPU oracle against the real reference's outputs (tests/golden)."""

import numpy as np
import pytest

from conftest import golden_names, load_golden, rel_l2
from oracle import ref_apply, ref_setup

TOL = 1e-12   # north_star: relative L2 <= 1e-12 in fp64


def _oracle_y(g):
    kind = str(g["kind"])
    if kind == "cg":
        nc = int(g["n_components"]) if "n_components" in g else 1
        if nc == 1:
            return ref_apply.cg_apply(g["vertices"], g["cells"], g["cell_dofs"], g["dirichlet_mask"],
                                      g["grad_matrix"], g["cell_weights"], g["u"])
        u = g["u"].reshape(-1, nc)
        return np.stack([ref_apply.cg_apply(g["vertices"], g["cells"], g["cell_dofs"], g["dirichlet_mask"],
                                            g["grad_matrix"], g["cell_weights"], u[:, c])
                         for c in range(nc)], axis=1).ravel()
    nd = g["cell_dofs"].shape[1]
    common = (g["vertices"], g["cells"], nd, g["interior_faces"], g["boundary_faces"],
              set(g["dirichlet_ids"].tolist()), g["value_matrix"], g["grad_matrix"], g["cell_weights"],
              g["face_values"], g["face_grads"], g["face_weights"], g["tau_i"], g["tau_b"], g["u"])
    if kind == "dg":
        return ref_apply.dg_apply(*common)
    if kind == "helm_kappa":
        return ref_apply.dg_apply(*common, kappa=g["kappa"], mass_scale=1.0, stiff_scale=1.0)
    if kind == "helm3":
        return ref_apply.dg_apply(*common, mass_scale=float(g["mass_scale"]),
                                  stiff_scale=float(g["nu"]), n_components=3)
    raise AssertionError(kind)


@pytest.mark.parametrize("name", golden_names())
def test_oracle_matches_reference(name):
    g = load_golden(name)
    y = _oracle_y(g)
    assert rel_l2(y, g["y"]) <= TOL


@pytest.mark.parametrize("name", golden_names("cg_p"))
def test_oracle_integer_setup_matches_reference(name):
    g = load_golden(name)
    p = int(g["p"])
    ifc, bfc = ref_setup.build_faces(g["cells"])
    assert np.array_equal(ifc, g["interior_faces"])
    assert np.array_equal(bfc[:, :2], g["boundary_faces"][:, :2])
    cd, mask, n = ref_setup.build_cg_dofs(g["cells"], len(g["vertices"]), p, g["boundary_faces"],
                                          g["dirichlet_ids"].tolist())
    assert n == len(g["u"])
    assert np.array_equal(cd, g["cell_dofs"])
    assert np.array_equal(mask, g["dirichlet_mask"])
