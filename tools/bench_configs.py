"""Measure every BASELINE.json config on one GPU (developer tool; bench.py is the contract).

    python tools/bench_configs.py [c1 c2 c3 c4 c5] [--n4 128] [--n5 128]

Prints one JSON line per config: GDoF/s (fp64), per-kernel CUDA-event times, the
roofline fraction against the measured FP64 DMMA peak, and for C1 the parity vs
the CPU oracle.  Reordering (hierarchical) is applied as setup for C3-C5.
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

PEAK = 37.1


def setup(n, p, space, reorder, dids=()):
    from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, quadrature as Q
    from paper_2509_10226_b200.geometry import GeometryData

    t = time.time()
    m = M.kuhn_cube_mesh(n, seed=0)
    if reorder:
        from paper_2509_10226_b200.reorder import reorder_mesh

        m = reorder_mesh(m)
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    dm = D.build_dof_map(m, p, space, 1, dids)
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    return m, dm, geo, bas, time.time() - t


def timed(A, nd, reps=10):
    import torch

    u = torch.rand(nd, dtype=torch.float64, device="cuda") * 2 - 1
    y = torch.empty_like(u)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    A.timed(u.data_ptr(), y.data_ptr(), st, 3)
    acc = np.zeros(4)
    for _ in range(reps):
        flush.fill_(1.0)
        acc += A.timed(u.data_ptr(), y.data_ptr(), st, 1)
    return acc / reps


def line(name, A, nd, ms, extra=None):
    info = A.info
    d = {"config": name, "ndof": nd, "ms": round(float(ms[0]), 4), "cell_ms": round(float(ms[1]), 4),
         "face_ms": round(float(ms[2]), 4), "gdofs": round(nd / ms[0] / 1e6, 3),
         "tflops_engine": round(info["flops_engine"] / ms[0] / 1e9, 2),
         "frac_fp64_roofline": round(info["flops_engine"] / ms[0] / 1e9 / PEAK, 3),
         "tflops_ref_formula": round(info["flops_alg"] / ms[0] / 1e9, 2), "cell_engine": int(info["cell_engine"]),
         "flops_alg_per_dof": round(info["flops_alg"] / nd, 1), "bytes_alg_per_dof": round(info["bytes_alg"] / nd, 1),
         "issued_over_engine": round(info["flops_issued"] / info["flops_engine"], 3)}
    if extra:
        d.update(extra)
    print(json.dumps(d), flush=True)


def c1():
    from oracle import ref_apply
    from paper_2509_10226_b200 import operator as op

    m, dm, geo, bas, ts = setup(8, 2, "cg", False)
    A = op.CgPoissonOperator(m, dm, geo, bas)
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    y = A.apply(u)
    yr = ref_apply.cg_apply(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask, bas.grad_matrix,
                            geo.cell_rule.weights, u)
    ms = timed(A, dm.n_global_dofs, 50)
    line("C1 CG P2 8^3x6", A, dm.n_global_dofs, ms,
         {"rel_l2_vs_oracle": float(np.linalg.norm(y - yr) / np.linalg.norm(yr)), "setup_s": round(ts, 1)})


def c2():
    from paper_2509_10226_b200 import operator as op

    for reorder in (False, True):
        for p in (1, 2, 3, 4):
            m, dm, geo, bas, ts = setup(48, p, "cg", reorder)
            A = op.CgPoissonOperator(m, dm, geo, bas)
            ms = timed(A, dm.n_global_dofs)
            line(f"C2 CG P{p} 48^3x6{' reordered' if reorder else ''}", A, dm.n_global_dofs, ms,
                 {"setup_s": round(ts, 1)})


def c3(n=64):
    from paper_2509_10226_b200 import operator as op

    for reorder in (False, True):
        m, dm, geo, bas, ts = setup(n, 3, "dg", reorder)
        A = op.DgSipgOperator(m, dm, geo, bas, op.baseline_sipg_tau(m, 3, 1.0 / n), dirichlet_ids=range(6))
        ms = timed(A, dm.n_global_dofs)
        line(f"C3 DG-SIPG P3 {n}^3x6{' reordered' if reorder else ''}", A, dm.n_global_dofs, ms,
             {"setup_s": round(ts, 1)})


def c4(n=128):
    from paper_2509_10226_b200 import operator as op

    m, dm, geo, bas, ts = setup(n, 2, "dg", True)
    kap = 10.0 ** np.random.default_rng(2).uniform(-1, 1, m.n_cells)
    A = op.KappaHelmholtzOperator(m, dm, geo, bas, op.baseline_sipg_tau(m, 2, 1.0 / n), kap, 1.0,
                                  dirichlet_ids=range(6))
    ms = timed(A, dm.n_global_dofs, 5)
    line(f"C4 DG Helmholtz (mass + kappa-Laplace) P2 {n}^3x6 reordered, 1 GPU", A, dm.n_global_dofs, ms,
         {"setup_s": round(ts, 1)})


def c5(n=128, iters=100):
    import torch

    from paper_2509_10226_b200 import operator as op
    from paper_2509_10226_b200.solvers import jacobi_pcg

    m, dm, geo, bas, ts = setup(n, 3, "cg", True, tuple(range(6)))
    A = op.CgPoissonOperator(m, dm, geo, bas)
    b = np.where(dm.dirichlet_mask, 0.0, np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs))
    bt = torch.from_numpy(b).cuda()
    jacobi_pcg(A, bt, 3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, hist = jacobi_pcg(A, bt, iters)
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1)
    ms = timed(A, dm.n_global_dofs, 5)
    nd = dm.n_global_dofs
    print(json.dumps({"config": f"C5 Jacobi-PCG CG P3 {n}^3x6 reordered, {iters} iterations, 1 GPU", "ndof": nd,
                      "solve_ms": round(t, 2), "ms_per_iteration": round(t / iters, 4),
                      "apply_ms": round(float(ms[0]), 4),
                      "apply_gdofs": round(nd / ms[0] / 1e6, 3),
                      "solver_gdofs_per_iteration": round(nd * iters / t / 1e6, 3),
                      "apply_frac_fp64_roofline": round(A.info["flops_engine"] / ms[0] / 1e9 / PEAK, 3),
                      "residual_first_last": [float(hist[0]), float(hist[-1])], "setup_s": round(ts, 1)}),
          flush=True)


def csr(n=48):
    """Matrix-free vs assembled CSR (cuSPARSE) on the C2 meshes: the paper's comparison on B200."""
    import torch

    from paper_2509_10226_b200 import operator as op
    from paper_2509_10226_b200.sparse import CsrOperator

    for p in (1, 2, 3, 4):
        m, dm, geo, bas, ts = setup(n, p, "cg", True)
        A = op.CgPoissonOperator(m, dm, geo, bas)
        ms_mf = timed(A, dm.n_global_dofs)
        t0 = time.time()
        S = CsrOperator(m, dm, geo, bas)
        torch.cuda.synchronize()
        t_asm = time.time() - t0
        u = torch.rand(dm.n_global_dofs, dtype=torch.float64, device="cuda")
        flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
        for _ in range(3):
            S.apply(u)
        tt = []
        for _ in range(10):
            flush.fill_(1.0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            S.apply(u)
            e1.record()
            e1.synchronize()
            tt.append(e0.elapsed_time(e1))
        ms = float(np.mean(tt))
        print(json.dumps({"config": f"C2 P{p} {n}^3x6 reordered: matrix-free vs CSR SpMV (cuSPARSE)",
                          "ndof": dm.n_global_dofs, "nnz": S.nnz, "csr_bytes": S.nbytes,
                          "mf_ms": round(float(ms_mf[0]), 4), "csr_spmv_ms": round(ms, 4),
                          "csr_assembly_s": round(t_asm, 2),
                          "csr_spmv_gbps": round(S.nbytes / ms / 1e6, 1),
                          "mf_speedup_over_csr": round(ms / float(ms_mf[0]), 3)}), flush=True)
        del S
        torch.cuda.empty_cache()


def mg(n=128, degrees=(3, 2, 1), tol=1e-8, precision="f64", coarse_matrix=False, h_coarse=(), coarse_iterations=30,
       smoothing_degree=2):
    """p-multigrid flexible PCG vs Jacobi-PCG on the C5 problem (CG P3, homogeneous
    Dirichlet, RHS uniform[-1,1]): iterations and device time to ||r|| <= tol ||b||."""
    import torch

    from paper_2509_10226_b200.multigrid import PMultigrid
    from paper_2509_10226_b200.solvers import jacobi_pcg

    from paper_2509_10226_b200 import mesh as M
    from paper_2509_10226_b200.reorder import reorder_mesh

    t0 = time.time()
    m = reorder_mesh(M.kuhn_cube_mesh(n, seed=0))
    mg_ = PMultigrid(m, degrees, coarse_iterations=coarse_iterations, precision=precision,
                     coarse_matrix=coarse_matrix, h_coarse=h_coarse, smoothing_degree=smoothing_degree)
    setup = time.time() - t0
    dm = mg_.levels[0].dm
    nd = dm.n_global_dofs
    b = np.where(dm.dirichlet_mask, 0.0, np.random.default_rng(1).uniform(-1, 1, nd))
    bt = torch.from_numpy(b).cuda()
    mg_.solve(bt, tol=1e-2, maxiter=3)   # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, hist = mg_.solve(bt, tol=tol, maxiter=200)
    e1.record()
    e1.synchronize()
    t_mg = e0.elapsed_time(e1)
    # one V-cycle alone
    r = bt.clone()
    e0.record()
    for _ in range(5):
        mg_.vcycle(r)
    e1.record()
    e1.synchronize()
    t_v = e0.elapsed_time(e1) / 5
    true_res = float(torch.linalg.vector_norm(mg_.levels[0].A.apply(x) - bt) / torch.linalg.vector_norm(bt))
    # Jacobi-PCG: iterations to the same tolerance (fixed-count native loop, residual history)
    jit = 4000
    e0.record()
    _, hj = jacobi_pcg(mg_.levels[0].A, bt, jit)
    e1.record()
    e1.synchronize()
    t_j = e0.elapsed_time(e1)
    hit = np.nonzero(hj <= tol * hj[0])[0]
    kj = int(hit[0]) if len(hit) else None
    print(json.dumps({"config": f"p-multigrid PCG vs Jacobi-PCG, CG P3 {n}^3x6 reordered, Dirichlet, tol {tol}",
                      "precision": "fp32 V-cycle, fp64 outer CG" if precision == "mixed" else "fp64",
                      "ndof": nd, "levels": list(degrees), "lmax": [round(lv.lmax, 4) for lv in mg_.levels[:-1]],
                      "smoother": f"Chebyshev-Jacobi degree {mg_.smoothing_degree}, range {mg_.smoothing_range}",
                      "p1_fine_level": "assembled CSR (cuSPARSE)" if coarse_matrix else "matrix-free",
                      "h_levels": list(h_coarse),
                      "coarse": f"Jacobi-PCG {mg_.coarse_iterations} iterations on {mg_.levels[-1].dm.n_scalar_dofs} DoFs",
                      "mg_iterations": len(hist) - 1, "mg_solve_ms": round(t_mg, 2), "vcycle_ms": round(t_v, 3),
                      "mg_true_rel_residual": true_res,
                      "jacobi_iterations_to_tol": kj, "jacobi_ms_per_iteration": round(t_j / jit, 4),
                      "jacobi_ms_to_tol": round(t_j / jit * kj, 2) if kj else None,
                      "speedup_time_to_tol": round(t_j / jit * kj / t_mg, 2) if kj else None,
                      "setup_s": round(setup, 1)}), flush=True)
    mg_.close()


def mgdg(n=64, p=3, tol=1e-8, tau_scale=1.0, h_coarse=(), precision="f64", fine_smoothing_degree=None,
         helmholtz=False):
    """cp-multigrid (DG p -> CG p -> ... -> CG 1) flexible PCG vs Jacobi-PCG on the C3 problem
    (DG-SIPG P3, weak Dirichlet on all sides, RHS uniform[-1,1]): iterations / time to tol."""
    import torch

    from paper_2509_10226_b200 import operator as op
    from paper_2509_10226_b200.multigrid import PMultigrid, n10
    from paper_2509_10226_b200.solvers import pcg_loop

    m, dm, geo, bas, ts = setup(n, p, "dg", True)
    t0 = time.time()
    sipg = op.baseline_sipg_tau(m, p, 1.0 / n)
    sipg.tau_interior *= tau_scale
    sipg.tau_boundary *= tau_scale
    kap = None
    if helmholtz:   # C4: mass + kappa-Laplace, kappa log-uniform in [0.1, 10] (seed 2)
        kap = 10.0 ** np.random.default_rng(2).uniform(-1, 1, m.n_cells)
        A = op.KappaHelmholtzOperator(m, dm, geo, bas, sipg, kap, 1.0, dirichlet_ids=range(6))
    else:
        A = op.DgSipgOperator(m, dm, geo, bas, sipg, dirichlet_ids=range(6))
    mg_ = PMultigrid(m, tuple(range(p, 0, -1)), fine_operator=A, coarse_iterations=50 if h_coarse else 30,
                     h_coarse=h_coarse, fine_smoothing_degree=fine_smoothing_degree, kappa=kap)
    setup_mg = time.time() - t0
    nd = dm.n_global_dofs
    bt = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, nd)).cuda()
    mg_.solve(bt, tol=1e-2, maxiter=2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, hist = mg_.solve(bt, tol=tol, maxiter=300)
    e1.record()
    e1.synchronize()
    t_mg = e0.elapsed_time(e1)
    true_res = float(torch.linalg.vector_norm(A.apply(x) - bt) / torch.linalg.vector_norm(bt))
    diag = 1.0 / mg_.levels[0].dinv
    jit = 3000
    e0.record()
    _, hj = pcg_loop(lambda v, out: A.apply_into(v.data_ptr(), out.data_ptr(),
                                                 torch.cuda.current_stream().cuda_stream), diag, bt, jit)
    e1.record()
    e1.synchronize()
    t_j = e0.elapsed_time(e1)
    hit = np.nonzero(hj <= tol * hj[0])[0]
    kj = int(hit[0]) if len(hit) else None
    what = "DG kappa-Helmholtz (C4 operator)" if helmholtz else "DG-SIPG"
    print(json.dumps({"config": f"cp-multigrid PCG vs Jacobi-PCG, {what} P{p} {n}^3x6 reordered, weak Dirichlet, "
                      f"tol {tol}", "tau": f"{tau_scale} x 2.5 (p+1)^2 / h", "h_levels": list(h_coarse),
                      "dg_smoothing_degree": len(mg_.levels[0].coeffs), "ndof": nd, "levels": ["dg%d" % p] + ["cg%d" % lv.p for lv in mg_.levels[1:]],
                      "lmax": [round(lv.lmax, 4) for lv in mg_.levels[:-1]],
                      "mg_iterations": len(hist) - 1, "mg_solve_ms": round(t_mg, 2),
                      "mg_true_rel_residual": true_res,
                      "jacobi_iterations_to_tol": kj, "jacobi_ms_per_iteration": round(t_j / jit, 4),
                      "jacobi_rel_residual_after_%d" % jit: float(hj[-1] / hj[0]),
                      "jacobi_ms_to_tol": round(t_j / jit * kj, 2) if kj else None,
                      "speedup_time_to_tol": round(t_j / jit * kj / t_mg, 2) if kj else None,
                      "setup_s": round(ts, 1), "mg_setup_s": round(setup_mg, 1)}), flush=True)
    mg_.close()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--n3", type=int, default=64)
    ap.add_argument("--n4", type=int, default=128)
    ap.add_argument("--n5", type=int, default=128)
    ap.add_argument("--tau-scale", type=float, default=1.0)
    ap.add_argument("--precision", default="f64", choices=["f64", "mixed"])
    ap.add_argument("--coarse-matrix", action="store_true")
    ap.add_argument("--h-coarse", default="", help="comma-separated coarse Kuhn sizes, e.g. 64,32,16,8")
    ap.add_argument("--coarse-iterations", type=int, default=30)
    ap.add_argument("--dg-smoothing-degree", type=int, default=None)
    ap.add_argument("--smoothing-degree", type=int, default=2)
    ap.add_argument("--best", action="store_true",
                    help="mg: the fastest measured hierarchy (fp32 V-cycle in a CUDA graph, CSR P1 level, "
                         "h-levels n/2..n/16, Chebyshev degree 3, 10 coarse iterations)")
    a = ap.parse_args()
    for c in a.configs:
        {"c1": c1, "c2": c2, "c3": lambda: c3(a.n3), "c4": lambda: c4(a.n4), "c5": lambda: c5(a.n5),
         "csr": csr, "mg": (lambda: mg(a.n5, precision="mixed", coarse_matrix=True,
                          h_coarse=tuple(a.n5 // 2 ** k for k in range(1, 5) if a.n5 // 2 ** k >= 2),
                          coarse_iterations=10, smoothing_degree=3)) if a.best else
              (lambda: mg(a.n5, precision=a.precision, coarse_matrix=a.coarse_matrix,
                          h_coarse=tuple(int(v) for v in a.h_coarse.split(",") if v),
                          coarse_iterations=a.coarse_iterations, smoothing_degree=a.smoothing_degree)), "mgc4": lambda: mgdg(a.n4, p=2, tau_scale=a.tau_scale, helmholtz=True),
         "mgdg": lambda: mgdg(a.n3, tau_scale=a.tau_scale,
                             h_coarse=tuple(int(v) for v in a.h_coarse.split(",") if v),
                             fine_smoothing_degree=a.dg_smoothing_degree)}[c]()
