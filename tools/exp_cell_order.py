"""Experiment: the unordered C2 mesh's cell traversal re-sorted in Morton order of the
centroids, DoF numbering unchanged (cells and cell_dofs rows permuted together) -- what a
plan-internal traversal order would give the tile kernels.  Developer tool."""
import json
import os
import sys
from types import SimpleNamespace as NS

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, operator as op, quadrature as Q  # noqa: E402
from paper_2509_10226_b200.geometry import GeometryData  # noqa: E402


def morton(vertices, cells):
    c = vertices[cells].mean(axis=1)
    lo, hi = c.min(0), c.max(0)
    q = np.minimum(((c - lo) / (hi - lo) * 2097152).astype(np.uint64), 2097151)

    def spread(x):
        x = x & np.uint64(0x1fffff)
        for s, m in ((32, 0x1f00000000ffff), (16, 0x1f0000ff0000ff), (8, 0x100f00f00f00f00f),
                     (4, 0x10c30c30c30c30c3), (2, 0x1249249249249249)):
            x = (x | (x << np.uint64(s))) & np.uint64(m)
        return x
    code = spread(q[:, 0]) | (spread(q[:, 1]) << np.uint64(1)) | (spread(q[:, 2]) << np.uint64(2))
    return np.argsort(code, kind="stable")


m = M.kuhn_cube_mesh(48, seed=0)
if len(sys.argv) > 1 and sys.argv[1] == "reordered":
    from paper_2509_10226_b200.reorder import reorder_mesh
    m = reorder_mesh(m)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for p in (2, 3, 4):
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    dm = D.build_dof_map(m, p, "cg")
    perm = morton(m.vertices, m.cells)
    for name, order in (("input", None), ("morton", perm)):
        cells = m.cells if order is None else m.cells[order]
        cd = dm.cell_dofs if order is None else dm.cell_dofs[order]
        mesh = NS(vertices=m.vertices, cells=np.ascontiguousarray(cells), interior_faces=None, boundary_faces=None)
        dmap = NS(space="cg", degree=p, n_components=1, n_scalar_dofs=dm.n_scalar_dofs,
                  cell_dofs=np.ascontiguousarray(cd), dirichlet_mask=dm.dirichlet_mask)
        A = op.CgPoissonOperator(mesh, dmap, geo, bas)
        u = torch.rand(A.n_global_dofs, dtype=torch.float64, device="cuda")
        y = torch.empty_like(u)
        for _ in range(5):
            A.apply_into(u.data_ptr(), y.data_ptr(), st)
        ts = []
        for _ in range(30):
            flush.fill_(1.0)
            ts.append(A.timed(u.data_ptr(), y.data_ptr(), st, 1)[1])
        print(json.dumps({"p": p, "order": name, "cell_ms": round(float(np.median(ts)), 4)}), flush=True)
