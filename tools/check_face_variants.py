"""GPU check: face-kernel variants give the default variant's apply (developer tool)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, operator as op, quadrature as Q
from paper_2509_10226_b200.geometry import GeometryData

for kind, p, n in (("dg", 2, 12), ("dg", 3, 10), ("hh", 2, 12), ("dg", 4, 6), ("dg", 1, 12)):
    m = M.kuhn_cube_mesh(n, seed=0)
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    dm = D.build_dof_map(m, p, "dg")
    u = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)).cuda()
    ys = {}
    for v in (0, 11, 12):
        cfg = op.OperatorConfig(face_variant=v)
        if kind == "dg":
            A = op.DgSipgOperator(m, dm, geo, bas, op.baseline_sipg_tau(m, p, 1.0 / n), cfg, dirichlet_ids=range(6))
        else:
            kap = 10.0 ** np.random.default_rng(2).uniform(-1, 1, m.n_cells)
            A = op.KappaHelmholtzOperator(m, dm, geo, bas, op.baseline_sipg_tau(m, p, 1.0 / n), kap, 1.0, cfg,
                                          dirichlet_ids=range(6))
        ys[v] = A.apply(u)
    rel = {v: float(torch.linalg.vector_norm(ys[v] - ys[0]) / torch.linalg.vector_norm(ys[0])) for v in (11, 12)}
    print(json.dumps({"kind": kind, "p": p, "n": n, "rel_vs_default": rel}), flush=True)
