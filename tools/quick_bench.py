"""Developer timing of single applies (not the official bench.py)."""
import sys, time, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_10226_b200 import mesh as M, dofmap as D, basis as B, quadrature as Q, geometry as G, operator as op

def run(kind, p, n, reps=20, variant=0, engine="auto", patches="auto", face="auto", runs="plain"):
    reordered = kind[-1] in "rv"
    suffix = kind[-1] if reordered else ""
    t0 = time.time()
    m = M.kuhn_cube_mesh(n, seed=0)
    if reordered:   # r: cells only, v: cells + first-touch vertex renumbering
        from paper_2509_10226_b200.reorder import reorder_mesh
        m = reorder_mesh(m, renumber_vertices=suffix == "v")
        kind = kind[:-1]
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = G.GeometryData("affine", cr, fr, None, None, None, None)
    if kind == "cg":
        dm = D.build_dof_map(m, p, "cg")
        A = op.CgPoissonOperator(m, dm, geo, bas, op.OperatorConfig(kernel_variant=variant, cell_engine=engine, cell_patches=patches))
    elif kind == "dg":
        dm = D.build_dof_map(m, p, "dg")
        A = op.DgSipgOperator(m, dm, geo, bas, op.baseline_sipg_tau(m, p, 1.0 / n),
                              op.OperatorConfig(kernel_variant=variant & 0xF, face_variant=(variant >> 4) & 0xF, face_chunk=((variant >> 8) & 0xF) * 8, concurrent_dg=bool(variant >> 12), cell_engine=engine, face_engine=face, face_runs=runs),
                              dirichlet_ids=range(6))
    else:
        dm = D.build_dof_map(m, p, "dg")
        kap = 10.0 ** np.random.default_rng(2).uniform(-1, 1, m.n_cells)
        A = op.KappaHelmholtzOperator(m, dm, geo, bas, op.baseline_sipg_tau(m, p, 1.0 / n), kap, 1.0,
                                      op.OperatorConfig(kernel_variant=variant & 0xF, face_variant=(variant >> 4) & 0xF, face_chunk=((variant >> 8) & 0xF) * 8, concurrent_dg=bool(variant >> 12), cell_engine=engine, face_engine=face, face_runs=runs),
                                      dirichlet_ids=range(6))
    setup = time.time() - t0
    nd = A.n_global_dofs
    u = torch.rand(nd, dtype=torch.float64, device="cuda") * 2 - 1
    y = torch.empty_like(u)
    st = torch.cuda.current_stream().cuda_stream
    A.timed(u.data_ptr(), y.data_ptr(), st, 3)
    ms = A.timed(u.data_ptr(), y.data_ptr(), st, reps)
    info = A.info
    gdofs = nd / (ms[0] * 1e-3) / 1e9
    tf_alg = info["flops_alg"] / (ms[0] * 1e-3) / 1e12
    tf_iss = info["flops_issued"] / (ms[0] * 1e-3) / 1e12
    print(json.dumps(dict(kind=kind + suffix, p=p, n=n, variant=variant, engine=engine, face=face, runs=runs, patch_cells=A.info['patch_cells'], patch_ratio=round(A.info['patch_ratio'], 3), ndof=nd, setup_s=round(setup, 1), ms=[round(x, 4) for x in ms],
                          gdofs=round(gdofs, 3), tflops_alg=round(tf_alg, 2), tflops_issued=round(tf_iss, 2),
                          frac_fp64=round(tf_alg / 37.1, 3))), flush=True)

if __name__ == "__main__":
    for spec in sys.argv[1:]:
        parts = spec.split(":")
        run(parts[0], int(parts[1]), int(parts[2]), variant=int(parts[3]) if len(parts) > 3 else 0,
            engine=parts[4] if len(parts) > 4 else "auto", patches=parts[5] if len(parts) > 5 else "auto",
            face=parts[6] if len(parts) > 6 else "auto", runs=parts[7] if len(parts) > 7 else "plain")
