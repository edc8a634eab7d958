"""Diagnostics for the cp-multigrid on DG-SIPG P3 (developer tool)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from tools.bench_configs import setup
from paper_2509_10226_b200 import operator as op
from paper_2509_10226_b200.multigrid import PMultigrid, dg_diagonal

for n in [int(a) for a in sys.argv[1:]]:
    p = 3
    m, dm, geo, bas, ts = setup(n, p, "dg", True)
    A = op.DgSipgOperator(m, dm, geo, bas, op.baseline_sipg_tau(m, p, 1.0 / n), dirichlet_ids=range(6))
    nd = dm.n_global_dofs
    g = torch.Generator(device="cuda").manual_seed(7)
    u = torch.rand(nd, dtype=torch.float64, device="cuda", generator=g) - 0.5
    v = torch.rand(nd, dtype=torch.float64, device="cuda", generator=g) - 0.5
    Au, Av = A.apply(u), A.apply(v)
    sym = abs(float(u @ Av) - float(v @ Au)) / float(torch.linalg.vector_norm(u) * torch.linalg.vector_norm(Av))
    det = float(torch.linalg.vector_norm(A.apply(u) - Au) / torch.linalg.vector_norm(Au))
    d = dg_diagonal(A, m)
    rng = np.random.default_rng(0)
    errs = []
    for i in rng.integers(0, nd, 10):
        e = torch.zeros(nd, dtype=torch.float64, device="cuda"); e[int(i)] = 1.0
        errs.append(abs(float(A.apply(e)[int(i)]) - float(d[int(i)])) / abs(float(d[int(i)])))
    row = {"n": n, "ndof": nd, "sym": sym, "repeat_rel": det, "diag_probe_err": max(errs),
           "diag_min": float(d.min()), "diag_max": float(d.max())}
    for ci in (30,):
        mg = PMultigrid(m, (3, 2, 1), fine_operator=A, coarse_iterations=ci)
        bt = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, nd)).cuda()
        x, hist = mg.solve(bt, tol=1e-8, maxiter=40)
        row["mg_hist"] = [float(h / hist[0]) for h in hist[::4]]
        # V-cycle as a preconditioner: r.V(r) > 0 and linearity-ish
        r1 = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, nd)).cuda()
        z1 = mg.vcycle(r1)
        row["rVr"] = float(r1 @ z1)
        # CG-only MG on the same mesh for comparison
        mg.close()
    print(json.dumps(row), flush=True)
