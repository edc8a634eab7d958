"""p-multigrid parameter sweep on the C5 problem (developer tool): time to 1e-8."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2509_10226_b200 import mesh as M
from paper_2509_10226_b200.multigrid import PMultigrid
from paper_2509_10226_b200.reorder import reorder_mesh

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
m = reorder_mesh(M.kuhn_cube_mesh(n, seed=0))
for spec in sys.argv[2:]:
    parts = spec.split(":")
    lev, sdeg, ci = parts[:3]
    prec = parts[3] if len(parts) > 3 else "f64"
    cm = len(parts) > 4 and parts[4] == "csr"
    hc = tuple(int(v) for v in parts[5].split("-")) if len(parts) > 5 and parts[5] else ()
    degs = tuple(int(c) for c in lev)
    t0 = time.time()
    mg = PMultigrid(m, degs, smoothing_degree=int(sdeg), coarse_iterations=int(ci), precision=prec, coarse_matrix=cm,
                    h_coarse=hc)
    setup = time.time() - t0
    dm = mg.levels[0].dm
    b = np.where(dm.dirichlet_mask, 0.0, np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs))
    bt = torch.from_numpy(b).cuda()
    mg.solve(bt, tol=1e-2, maxiter=2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, hist = mg.solve(bt, tol=1e-8, maxiter=200)
    e1.record()
    e1.synchronize()
    print(json.dumps({"n": n, "levels": degs, "precision": prec, "coarse_matrix": cm, "h_levels": hc, "smoothing_degree": int(sdeg), "coarse_iterations": int(ci),
                      "iterations": len(hist) - 1, "solve_ms": round(e0.elapsed_time(e1), 2),
                      "final_rel": float(hist[-1] / hist[0]), "setup_s": round(setup, 1)}), flush=True)
    mg.close()
    del mg
    torch.cuda.empty_cache()
