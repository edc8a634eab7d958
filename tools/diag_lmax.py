"""Lanczos lambda_max(D^-1 A) convergence for the DG-SIPG P3 level (developer tool)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from tools.bench_configs import setup
from paper_2509_10226_b200 import operator as op
from paper_2509_10226_b200.multigrid import PMultigrid, dg_diagonal, _Level

n = int(sys.argv[1])
p = 3
m, dm, geo, bas, ts = setup(n, p, "dg", True)
A = op.DgSipgOperator(m, dm, geo, bas, op.baseline_sipg_tau(m, p, 1.0 / n), dirichlet_ids=range(6))
mg = PMultigrid(m, (3, 2, 1), fine_operator=A, coarse_iterations=30)
lv = mg.levels[0]
est = {}
for it in (15, 30, 60, 120):
    for seed in (0, 1):
        est[f"{it}_{seed}"] = mg.estimate_lmax(lv, it, seed)
row = {"n": n, "lmax_estimates": est}
nd = dm.n_global_dofs
bt = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, nd)).cuda()
from paper_2509_10226_b200.multigrid import chebyshev_coefficients
for fac in (1.1, 1.3):
    top = max(est.values()) * fac
    for lv_ in mg.levels[:1]:
        lv_.lmax = top
        lv_.coeffs = chebyshev_coefficients(top, mg.smoothing_range, mg.smoothing_degree)
    x, hist = mg.solve(bt, tol=1e-8, maxiter=60)
    row[f"fac{fac}"] = {"iterations": len(hist) - 1, "final": float(hist[-1] / hist[0])}
print(json.dumps(row), flush=True)
