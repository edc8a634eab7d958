"""A/B timing of the C2 cell kernels of two checkouts on the same box (developer tool):
    python tools/ab_time.py <repo root> p:reorder ...   (e.g. 4:1 3:0)"""
import json
import os
import sys

root = os.path.abspath(sys.argv[1])
sys.path.insert(0, root)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, operator as op, quadrature as Q  # noqa: E402
from paper_2509_10226_b200.geometry import GeometryData  # noqa: E402
from paper_2509_10226_b200.reorder import reorder_mesh  # noqa: E402

meshes = {}
for spec in sys.argv[2:]:
    p, r = (int(x) for x in spec.split(":"))
    if r not in meshes:
        m = M.kuhn_cube_mesh(48, seed=0)
        meshes[r] = reorder_mesh(m) if r else m
    m = meshes[r]
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    A = op.CgPoissonOperator(m, D.build_dof_map(m, p, "cg"), GeometryData("affine", cr, fr, None, None, None, None),
                             B.tabulate_basis(p, cr, fr))
    u = torch.rand(A.n_global_dofs, dtype=torch.float64, device="cuda")
    y = torch.empty_like(u)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for _ in range(5):
        A.apply_into(u.data_ptr(), y.data_ptr(), st)
    ts = []
    for _ in range(30):
        flush.fill_(1.0)
        ts.append(A.timed(u.data_ptr(), y.data_ptr(), st, 1)[1])
    print(json.dumps({"root": os.path.basename(root), "spec": spec, "cell_ms": round(float(np.median(ts)), 4),
                      "engine": A.info["cell_engine"]}), flush=True)
