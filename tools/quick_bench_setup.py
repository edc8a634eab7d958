"""Operator construction from a spec kind:p:n[:variant[:engine[:patches]]] (developer tools)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2509_10226_b200 import basis as B, dofmap as D, geometry as G, mesh as M, operator as op  # noqa: E402
from paper_2509_10226_b200 import quadrature as Q  # noqa: E402


def build(spec):
    parts = spec.split(":")
    kind, p, n = parts[0], int(parts[1]), int(parts[2])
    variant = int(parts[3]) if len(parts) > 3 else 0
    engine = parts[4] if len(parts) > 4 else "auto"
    patches = parts[5] if len(parts) > 5 else "auto"
    m = M.kuhn_cube_mesh(n, seed=0)
    if kind.endswith("r"):
        from paper_2509_10226_b200.reorder import hierarchical_reorder
        m = M.apply_cell_permutation(m, hierarchical_reorder(m))
    base = kind.rstrip("r")
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = G.GeometryData("affine", cr, fr, None, None, None, None)
    cfg = op.OperatorConfig(kernel_variant=variant & 0xF, face_variant=(variant >> 4) & 0xF,
                            face_chunk=((variant >> 8) & 0xF) * 8, concurrent_dg=bool(variant >> 12),
                            cell_engine=engine, cell_patches=patches)
    if base == "cg":
        dm = D.build_dof_map(m, p, "cg")
        A = op.CgPoissonOperator(m, dm, geo, bas, cfg)
    elif base == "dg":
        dm = D.build_dof_map(m, p, "dg")
        A = op.DgSipgOperator(m, dm, geo, bas, op.baseline_sipg_tau(m, p, 1.0 / n), cfg, dirichlet_ids=range(6))
    else:
        dm = D.build_dof_map(m, p, "dg")
        kap = 10.0 ** np.random.default_rng(2).uniform(-1, 1, m.n_cells)
        A = op.KappaHelmholtzOperator(m, dm, geo, bas, op.baseline_sipg_tau(m, p, 1.0 / n), kap, 1.0, cfg,
                                      dirichlet_ids=range(6))
    meta = dict(spec=spec, patch_cells=A.info["patch_cells"], patch_ratio=round(A.info["patch_ratio"], 3))
    return A, A.n_global_dofs, meta
