"""Strong-scaling runs of BASELINE configs 4 and 5 on 1/2/4/8 GPUs (one process per GPU).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/bench_scaling.py c4 [--n 128]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/bench_scaling.py c5 [--n 128] [--iters 100]
    python tools/bench_scaling.py c4 --n 64          # world size 1 (same partitioned code path)

C4: DG Helmholtz (mass + per-cell kappa Laplace) P2 on the jittered, reordered
n^3 x 6 mesh split by recursive coordinate bisection; every apply = forward NCCL
halo of ghost cells overlapped with the owned cells' volume kernel, then the
face kernel.  C5: Jacobi-PCG (CG P3, homogeneous Dirichlet) with the
partitioned apply (forward + reverse halo) and two NCCL all_reduce per
iteration.  Times: CUDA events on the compute stream, max over ranks; L2 is
flushed between timed applies.  Rank 0 prints one JSON line.
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

PEAK = 37.1


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=["c4", "c5"])
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--iters", type=int, default=100)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"])
    a = ap.parse_args()

    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29571")
    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    # eager communicator init + a collective first (halo P2P involves only neighbouring ranks)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
    dist.barrier()

    from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, operator as op, quadrature as Q
    from paper_2509_10226_b200 import distributed as DD
    from paper_2509_10226_b200.geometry import GeometryData
    from paper_2509_10226_b200.reorder import hierarchical_reorder
    from paper_2509_10226_b200.solvers import pcg_loop

    t0 = time.time()
    n = a.n
    p = 2 if a.config == "c4" else 3
    m = M.kuhn_cube_mesh(n, seed=0)
    m = M.apply_cell_permutation(m, hierarchical_reorder(m))
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    part = DD.partition_cells(m, world)
    if a.config == "c4":
        dm = D.build_dof_map(m, p, "dg")
        kap = 10.0 ** np.random.default_rng(2).uniform(-1, 1, m.n_cells)
        A = DD.DistributedDgOperator(m, dm, geo, bas, op.baseline_sipg_tau(m, p, 1.0 / n), rank, world,
                                     kind="helmholtz", dirichlet_ids=range(6), kappa=kap, part=part,
                                     transport=a.transport)
        ids = A.owned_global_ids()
    else:
        dm = D.build_dof_map(m, p, "cg", 1, tuple(range(6)))
        A = DD.DistributedCgOperator(m, dm, geo, bas, rank, world, part=part, transport=a.transport)
        ids = A.owned_global_ids
    if a.transport == "p2p":
        A.connect_ipc()
    setup_s = time.time() - t0
    ng = dm.n_global_dofs
    rng = np.random.default_rng(1).uniform(-1, 1, ng)
    u = torch.from_numpy(np.ascontiguousarray(rng[ids])).cuda()
    y = torch.empty_like(u)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")

    def maxr(x):
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t[0])

    for _ in range(3):
        A.apply(u, out=y)
    torch.cuda.synchronize()
    dist.barrier()
    ts = []
    for _ in range(a.reps):
        flush.fill_(1.0)
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        A.apply(u, out=y)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    apply_ms = maxr(float(np.mean(ts)))
    out = {"config": a.config, "n_gpus": world, "transport": a.transport, "mesh": f"{n}^3 x 6", "ndof": ng,
           "apply_ms_max_over_ranks": round(apply_ms, 4), "apply_gdofs": round(ng / apply_ms / 1e6, 3),
           "setup_s_rank0": round(setup_s, 1), "scaling": "strong"}
    if a.config == "c5":
        b = torch.from_numpy(np.ascontiguousarray(np.where(dm.dirichlet_mask, 0.0, rng)[ids])).cuda()
        diag = A.diagonal()
        pcg_loop(A.apply, diag, b, 2, allreduce=lambda t: dist.all_reduce(t), n_local=A.n_local)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x, hist = pcg_loop(A.apply, diag, b, a.iters, allreduce=lambda t: dist.all_reduce(t), n_local=A.n_local)
        e1.record()
        e1.synchronize()
        solve = maxr(e0.elapsed_time(e1))
        out.update(solve_ms=round(solve, 2), iters=a.iters, ms_per_iteration=round(solve / a.iters, 4),
                   solver_gdofs_per_iteration=round(ng * a.iters / solve / 1e6, 3),
                   residual_first_last=[float(hist[0]), float(hist[-1])])
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
