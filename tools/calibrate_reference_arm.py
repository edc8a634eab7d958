"""Calibration of the bench reference arm (build container only: imports the REAL reference
from /root/reference): one core, same mesh and tables, the reference CgPoissonOperator.apply
(kernel_stage "mm") vs the port bench._ref_batches uses.  Output: profiles/r02/reference_arm_calibration.jsonl"""

import sys, time, os
os.environ["OPENBLAS_NUM_THREADS"] = "1"
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests/golden")
import numpy as np
import make_golden as G
from tetmf import geometry as rgeo, operator as rop
import bench
for p, n in ((1, 24), (2, 24), (3, 16)):
    tm = G.ref_mesh(n, 0)
    cr, fr = G.rules(p, "gm")
    basis = G.ref_basis(p, cr, fr)
    dm = G.ref_dofmap(tm, p, "cg")
    geo = rgeo.build_geometry(tm, cr, "affine")
    A = rop.CgPoissonOperator(tm, dm, geo, basis, rop.OperatorConfig(kernel_stage="mm"))
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    A.apply(u)
    t = time.perf_counter(); y = A.apply(u); t_ref = time.perf_counter() - t
    from oracle import ref_apply
    jit, jxw, _ = ref_apply.affine_cell_geometry(tm.vertices, tm.cells, cr.weights)
    ids, act = ref_apply._cell_batches(tm.n_cells, 4, 4)
    pr = dict(cd=dm.cell_dofs.astype(np.int64), u=u, Eg=basis.grad_matrix, jit=jit, jxw=jxw, ids=ids, act=act,
              y=np.zeros(len(u)))
    bench._ref_batches(pr, 0, 10)
    pr["y"][:] = 0
    t = time.perf_counter(); bench._ref_batches(pr, 0, len(ids)); t_port = time.perf_counter() - t
    err = np.linalg.norm(pr["y"] - y) / np.linalg.norm(y)
    print({"p": p, "n": n, "ndof": len(u), "reference_apply_s": round(t_ref, 3), "port_s": round(t_port, 3),
           "reference_over_port": round(t_ref / t_port, 2), "port_vs_reference_rel_l2": float(err)}, flush=True)
