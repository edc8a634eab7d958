"""Peer-memory multi-GPU transport (transport="p2p"): the cell / face kernels read
ghost u (and RED ghost y) directly in the owner rank's registered buffers.

Only one GPU is available to this build, so the ranks are emulated the way the
B200 profiling guide prescribes: (1) all rank operators in ONE process on one
device, linked with plain device pointers and run phase by phase on one stream
(no kernel waits on another); (2) two processes on the same device linked with
CUDA IPC handles and separated by host barriers (gloo).  Both check the gathered
result against the unpartitioned B200 apply.
"""

import os
import socket
import sys

import numpy as np
import pytest

from conftest import rel_l2

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _setup(kind, n, p, dids):
    from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, quadrature as Q
    from paper_2509_10226_b200.geometry import GeometryData
    from paper_2509_10226_b200.reorder import hierarchical_reorder

    m = M.kuhn_cube_mesh(n, seed=0)
    m = M.apply_cell_permutation(m, hierarchical_reorder(m))
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    dm = D.build_dof_map(m, p, "cg" if kind == "cg" else "dg", 1, dids if kind == "cg" else ())
    return m, dm, geo, bas


def _ops(kind, n, m, dm, geo, bas, world, dids, rank=None):
    from paper_2509_10226_b200 import distributed as DD
    from paper_2509_10226_b200 import operator as op

    part = DD.partition_cells(m, world)
    ranks = range(world) if rank is None else [rank]
    if kind == "cg":
        return [DD.DistributedCgOperator(m, dm, geo, bas, r, world, part=part, transport="p2p") for r in ranks]
    sipg = op.baseline_sipg_tau(m, dm.degree, 1.0 / n)
    kap = 10.0 ** np.random.default_rng(2).uniform(-1, 1, m.n_cells) if kind == "helm" else None
    return [DD.DistributedDgOperator(m, dm, geo, bas, sipg, r, world, part=part, transport="p2p",
                                     kind="helmholtz" if kind == "helm" else "sipg", dirichlet_ids=dids,
                                     kappa=kap) for r in ranks], sipg, kap


def _global(kind, m, dm, geo, bas, dids, sipg=None, kap=None):
    from paper_2509_10226_b200 import operator as op

    if kind == "cg":
        return op.CgPoissonOperator(m, dm, geo, bas)
    if kind == "helm":
        return op.KappaHelmholtzOperator(m, dm, geo, bas, sipg, kap, 1.0, dirichlet_ids=dids)
    return op.DgSipgOperator(m, dm, geo, bas, sipg, dirichlet_ids=dids)


def _owned_ids(o):
    ids = o.owned_global_ids
    return ids() if callable(ids) else ids


@pytest.mark.parametrize("kind,world,n,p,dids", [("cg", 2, 6, 2, (0, 3)), ("cg", 4, 6, 3, ()), ("cg", 8, 8, 1, (1,)),
                                                 ("dg", 2, 5, 2, tuple(range(6))), ("helm", 4, 5, 3, (0, 5)),
                                                 ("dg", 8, 6, 1, ())])
def test_p2p_emulated_ranks_match_global_apply(kind, world, n, p, dids):
    import torch

    from paper_2509_10226_b200.distributed import DistributedCgOperator

    m, dm, geo, bas = _setup(kind, n, p, dids)
    built = _ops(kind, n, m, dm, geo, bas, world, dids)
    ops, sipg, kap = (built, None, None) if kind == "cg" else built
    DistributedCgOperator.connect_local(ops)
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    for o in ops:
        o.p2p_stage_in(torch.from_numpy(u[_owned_ids(o)]).cuda())
    for o in ops:   # every rank's kernel: peer loads (and CG peer REDs) into the other ranks' buffers
        o.p2p_compute()
    y = np.full(dm.n_global_dofs, np.nan)
    for o in ops:
        y[_owned_ids(o)] = o.p2p_result(None).cpu().numpy()
    assert not np.isnan(y).any()
    ref = _global(kind, m, dm, geo, bas, dids, sipg, kap).apply(u)
    assert rel_l2(y, ref) <= 1e-13
    # the SASS of the product path has the peer accesses inside the compute kernel:
    # the cell / face kernels were the only launches of p2p_compute
    for o in ops:
        assert o.connected


def _ipc_worker(rank, world, port, kind, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dids = (0, 3) if kind == "cg" else tuple(range(6))
        m, dm, geo, bas = _setup(kind, 5, 2, dids)
        built = _ops(kind, 5, m, dm, geo, bas, world, dids, rank=rank)
        o = built[0] if kind == "cg" else built[0][0]
        o.connect_ipc()
        u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
        ids = _owned_ids(o)
        y = o.apply(torch.from_numpy(u[ids]).cuda()).cpu().numpy()
        y2 = o.apply(torch.from_numpy(u[ids]).cuda()).cpu().numpy()   # buffers reused
        parts = [None] * world
        dist.all_gather_object(parts, (ids, y, y2))
        if rank == 0:
            full = np.full(dm.n_global_dofs, np.nan)
            full2 = full.copy()
            for i, a, b in parts:
                full[i] = a
                full2[i] = b
            sipg = kap = None
            if kind != "cg":
                sipg = built[1]
            ref = _global(kind, m, dm, geo, bas, dids, sipg, kap).apply(u)
            q.put((float(rel_l2(full, ref)), float(rel_l2(full2, ref))))
        dist.barrier()
        o.bufs.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["cg", "dg"])
def test_p2p_ipc_two_processes_one_device(kind):
    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, kind, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    e1, e2 = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    assert e1 <= 1e-13 and e2 <= 1e-13, (e1, e2)
