"""Timing experiment: CG cell kernels on the reordered 48^3 mesh with the reference DoF
numbering (vertices | edges | faces | interiors) vs the same operator with ALL DoFs
renumbered by first touch in cell order (P A P^T; parity checked through the permutation)."""
import dataclasses, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_10226_b200 import basis as B, dofmap as D, geometry as G, mesh as M, operator as op, quadrature as Q
from paper_2509_10226_b200.reorder import reorder_mesh

n = int(sys.argv[1]) if len(sys.argv) > 1 else 48
m = reorder_mesh(M.kuhn_cube_mesh(n, seed=0))
st = torch.cuda.current_stream().cuda_stream
for p in (1, 2, 3, 4):
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = G.GeometryData("affine", cr, fr, None, None, None, None)
    dm = D.build_dof_map(m, p, "cg")
    flat = dm.cell_dofs.reshape(-1)
    _, first = np.unique(flat, return_index=True)
    order = np.argsort(first, kind="stable")          # old ids in first-touch order
    new_of_old = np.empty_like(order)
    new_of_old[order] = np.arange(len(order))
    dm2 = dataclasses.replace(dm, cell_dofs=new_of_old[dm.cell_dofs].astype(np.int32),
                              dirichlet_mask=dm.dirichlet_mask[order])
    row = {"p": p, "n": n, "ndof": dm.n_global_dofs}
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    ys = []
    for name, d in (("reference_numbering", dm), ("first_touch", dm2)):
        A = op.CgPoissonOperator(m, d, geo, bas, op.OperatorConfig())
        uu = u if d is dm else u[order]
        ut = torch.from_numpy(uu).cuda()
        yt = torch.empty_like(ut)
        A.timed(ut.data_ptr(), yt.data_ptr(), st, 3)
        row[name + "_ms"] = round(float(A.timed(ut.data_ptr(), yt.data_ptr(), st, 20)[0]), 4)
        y = yt.cpu().numpy()
        ys.append(y if d is dm else y[new_of_old])
    row["rel_l2"] = float(np.linalg.norm(ys[0] - ys[1]) / np.linalg.norm(ys[0]))
    print(json.dumps(row), flush=True)
