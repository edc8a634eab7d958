"""Developer timing of one operator apply (not the driver bench).

    python tools/loop_bench.py cg:2:48:r:auto:auto [dg:3:64:r:auto:auto ...]

spec = kind (cg | dg | helmk) : degree : n (n^3 x 6 Kuhn mesh) : u (unordered) | r
(reorder_mesh) : cell engine : cell blocks [: face engine].  Prints one JSON line per spec: the apply
time per tmf_apply_timed with a 256 MiB L2 flush before every apply (the bench's
protocol, CUDA events on the launch stream), its cell / face split, and back-to-back
"hot" applies.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

_MESH = {}


def build(spec):
    from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, operator as op, quadrature as Q
    from paper_2509_10226_b200.geometry import GeometryData
    from paper_2509_10226_b200.reorder import reorder_mesh

    parts = spec.split(":")
    kind, p, n, order, eng, blocks = parts[:6]
    face = parts[6] if len(parts) > 6 else "auto"
    p, n = int(p), int(n)
    if (n, order) not in _MESH:
        m = M.kuhn_cube_mesh(n, seed=0)
        _MESH[(n, order)] = reorder_mesh(m) if order == "r" else m
    m = _MESH[(n, order)]
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    cfg = op.OperatorConfig(cell_engine=eng, cell_blocks=blocks, face_engine=face)
    if kind == "cg":
        dm = D.build_dof_map(m, p, "cg")
        A = op.CgPoissonOperator(m, dm, geo, bas, cfg)
    else:
        dm = D.build_dof_map(m, p, "dg")
        sipg = op.baseline_sipg_tau(m, p, 1.0 / n)
        if kind == "dg":
            A = op.DgSipgOperator(m, dm, geo, bas, sipg, cfg, dirichlet_ids=range(6))
        else:
            kap = 10.0 ** np.random.default_rng(2).uniform(-1, 1, m.n_cells)
            A = op.KappaHelmholtzOperator(m, dm, geo, bas, sipg, kap, 1.0, cfg, dirichlet_ids=range(6))
    return A, dm.n_global_dofs


def main():
    for spec in sys.argv[1:]:
        A, nd = build(spec)
        u = torch.rand(nd, dtype=torch.float64, device="cuda") * 2 - 1
        y = torch.empty_like(u)
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
        st = torch.cuda.current_stream().cuda_stream
        for _ in range(5):
            A.apply_into(u.data_ptr(), y.data_ptr(), st)
        torch.cuda.synchronize()
        rows = []
        for _ in range(20):
            flush.fill_(1.0)
            rows.append(A.timed(u.data_ptr(), y.data_ptr(), st, 1))
        r = np.array(rows).mean(axis=0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            A.apply_into(u.data_ptr(), y.data_ptr(), st)
        e1.record()
        e1.synchronize()
        hot = e0.elapsed_time(e1) / 50
        info = A.info
        print(json.dumps({"spec": spec, "ndof": nd, "ms": round(float(r[0]), 4), "cell_ms": round(float(r[1]), 4),
                          "face_ms": round(float(r[2]), 4), "hot_ms": round(hot, 4),
                          "gdofs": round(nd / r[0] / 1e6, 3), "cell_engine": info["cell_engine"],
                          "face_engine": info["face_engine"], "block_cells": info["block_cells"],
                          "block_ratio": round(info["block_ratio"], 3),
                          "tflops_engine_cell": round(info["flops_engine"] / (r[1] * 1e-3) / 1e12, 2)}),
              flush=True)
        del A


if __name__ == "__main__":
    main()
