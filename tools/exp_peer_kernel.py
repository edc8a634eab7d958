"""Time the fused peer-memory CG cell kernels with WORLD ranks emulated on one GPU (developer
experiment; every rank's p2p_compute in turn, CUDA events):
    python tools/exp_peer_kernel.py <degree> <n> <world>"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2509_10226_b200 import basis as B, distributed as DD, dofmap as D, mesh as M, quadrature as Q  # noqa: E402
from paper_2509_10226_b200.geometry import GeometryData  # noqa: E402
from paper_2509_10226_b200.reorder import reorder_mesh  # noqa: E402

p, n, world = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
m = reorder_mesh(M.kuhn_cube_mesh(n, seed=0))
cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
bas = B.tabulate_basis(p, cr, fr)
geo = GeometryData("affine", cr, fr, None, None, None, None)
dm = D.build_dof_map(m, p, "cg")
part = DD.partition_cells(m, world)
ops = [DD.DistributedCgOperator(m, dm, geo, bas, r, world, part=part, transport="p2p") for r in range(world)]
DD.DistributedCgOperator.connect_local(ops)
u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
for o in ops:
    ids = o.owned_global_ids
    o.p2p_stage_in(torch.from_numpy(u[ids() if callable(ids) else ids]).cuda())
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
ts = []
for rep in range(8):
    tot = 0.0
    for o in ops:
        flush.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        o.p2p_compute()
        e1.record()
        e1.synchronize()
        tot += e0.elapsed_time(e1)
    ts.append(tot)
print(json.dumps({"lib": os.environ.get("TMF_LIB", "head"), "p": p, "n": n, "world": world,
                  "sum_of_rank_compute_ms": round(float(np.median(ts[2:])), 4)}), flush=True)
