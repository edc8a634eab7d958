"""Multi-process (gloo, CPU) tests of the domain-decomposed apply and PCG.

The partition, ownership and halo logic of paper_2509_10226_b200.distributed
run exactly as on the GPUs; the per-rank local apply is the CPU oracle (the
GPU path plugs the B200 plan into the same slot), and the result gathered from
all ranks must equal the unpartitioned oracle apply.
"""

import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(kind, n, p):
    from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, quadrature as Q
    from paper_2509_10226_b200 import operator as op
    from paper_2509_10226_b200.geometry import GeometryData

    m = M.kuhn_cube_mesh(n, seed=0)
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    if kind.startswith("cg"):
        dids = (0, 3, 5) if kind == "cg_dir" else ()
        dm = D.build_dof_map(m, p, "cg", 1, dids)
        return m, dm, geo, bas, None, dids
    dm = D.build_dof_map(m, p, "dg")
    return m, dm, geo, bas, op.baseline_sipg_tau(m, p, 1.0 / n), tuple(range(6))


def _cg_local_factory(mesh, dofmap, geometry, basis):
    from oracle import ref_apply

    def f(u):
        y = ref_apply.cg_apply(mesh.vertices, mesh.cells, dofmap.cell_dofs, dofmap.dirichlet_mask,
                               basis.grad_matrix, geometry.cell_rule.weights, u.numpy())
        return torch.from_numpy(y)
    return f


def _dg_local_factory(kappa_on):
    def factory(mesh, dofmap, geometry, basis, sipg, kappa, dirichlet_ids):
        from oracle import ref_apply

        def f(u):
            y = ref_apply.dg_apply(mesh.vertices, mesh.cells, dofmap.n_dofs_per_cell, mesh.interior_faces,
                                   mesh.boundary_faces, set(dirichlet_ids), basis.value_matrix,
                                   basis.grad_matrix, geometry.cell_rule.weights, basis.face_values,
                                   basis.face_grads, geometry.face_rule.weights, sipg.tau_interior,
                                   sipg.tau_boundary, u.numpy(), kappa=kappa if kappa_on else None,
                                   mass_scale=1.0 if kappa_on else 0.0)
            return torch.from_numpy(y)
        return f
    return factory


class CpuVecOps:
    """Torch-CPU stand-in for the native fused PCG kernels (test scaffolding)."""

    def dot(self, a, b, out):
        out += torch.dot(a, b)

    def init(self, b, d, x, r, z, p, rz, rr):
        x.zero_(); r.copy_(b); z.copy_(r / d); p.copy_(z)
        rz += torch.dot(r, z); rr += torch.dot(r, r)

    def update(self, p, q, d, x, r, z, rz_k, pq_k, rz_next, rr_next):
        alpha = rz_k / pq_k
        x.add_(alpha * p); r.sub_(alpha * q); z.copy_(r / d)
        rz_next += torch.dot(r, z); rr_next += torch.dot(r, r)

    def direction(self, z, p, rz_k, rz_next):
        p.mul_(rz_next / rz_k).add_(z)


def _worker(rank, world, port, kind, n, p, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2509_10226_b200 import distributed as DD
        from paper_2509_10226_b200.solvers import pcg_loop

        shared = kind.endswith("_shared")
        kind = kind.replace("_shared", "")
        if shared:
            # global setup built by rank 0 only and mapped read-only by the others (NodeShared)
            from paper_2509_10226_b200.dofmap import DoFMap
            from paper_2509_10226_b200.mesh import TetMesh

            ns = DD.NodeShared(rank, DD.NodeShared.job_token())

            def build():
                assert rank == 0, "only the node's first rank builds"
                m0, dm0 = _problem(kind, n, p)[:2]
                return {"vertices": m0.vertices, "cells": m0.cells, "interior_faces": m0.interior_faces,
                        "boundary_faces": m0.boundary_faces, "cell_dofs": dm0.cell_dofs,
                        "dirichlet_mask": dm0.dirichlet_mask, "part": DD.partition_cells(m0, world)}

            a = ns.get("problem", build)
            if rank != 0:
                assert not a["cells"].flags.writeable   # mapped, not copied
            _, _, geo, bas, sipg, dids = _problem(kind, 2, p)   # tables only (tiny mesh)
            m = TetMesh(a["vertices"], a["cells"], a["interior_faces"], a["boundary_faces"])
            dm = DoFMap("cg", p, 1, len(a["dirichlet_mask"]), a["cell_dofs"], a["dirichlet_mask"])
            part = a["part"]
        else:
            m, dm, geo, bas, sipg, dids = _problem(kind, n, p)
            part = None
        u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
        out = {}
        if kind.startswith("cg"):
            A = DD.DistributedCgOperator(m, dm, geo, bas, rank, world, part=part, device="cpu",
                                         local_factory=_cg_local_factory)
            ids = A.owned_global_ids
            y = A.apply(torch.from_numpy(u[ids])).numpy()
            out["apply"] = (ids, y)
            # local layout (owned + ghost slots), used in place
            ul = torch.zeros(A.n_local, dtype=torch.float64)
            ul[: A.n_owned] = torch.from_numpy(u[ids])
            yl = torch.empty_like(ul)
            assert A.apply(ul, out=yl) is yl
            assert np.array_equal(yl[: A.n_owned].numpy(), y)
            if kind == "cg_dir":
                from oracle import ref_apply

                diag_g = ref_apply.cg_diagonal(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask,
                                               bas.grad_matrix, geo.cell_rule.weights, dm.n_global_dofs)
                b = torch.from_numpy(np.where(dm.dirichlet_mask, 0.0, u)[ids])
                x, hist = pcg_loop(A.apply, torch.from_numpy(diag_g[ids]), b, 12,
                                   allreduce=lambda t: dist.all_reduce(t), ops=CpuVecOps())
                out["pcg"] = (ids, x.numpy(), hist)
                # the same solve with the direction / A p in rank-local buffers (in place)
                x2, hist2 = pcg_loop(A.apply, torch.from_numpy(diag_g[ids]), b, 12,
                                     allreduce=lambda t: dist.all_reduce(t), ops=CpuVecOps(), n_local=A.n_local)
                assert np.array_equal(x2.numpy(), x.numpy()) and np.array_equal(hist2, hist)
        else:
            kap = 10.0 ** np.random.default_rng(2).uniform(-1, 1, m.n_cells) if kind == "helm" else None
            A = DD.DistributedDgOperator(m, dm, geo, bas, sipg, rank, world,
                                         kind="helmholtz" if kind == "helm" else "sipg", dirichlet_ids=dids,
                                         kappa=kap, device="cpu", local_factory=_dg_local_factory(kind == "helm"))
            ids = A.owned_global_ids()
            y = A.apply(torch.from_numpy(u[ids])).numpy()
            out["apply"] = (ids, y)
            ul = torch.zeros(A.n_local, dtype=torch.float64)
            ul[: A.n_owned] = torch.from_numpy(u[ids])
            yl = torch.empty_like(ul)
            assert A.apply(ul, out=yl) is yl
            assert np.array_equal(yl[: A.n_owned].numpy(), y)
        gathered = [None] * world
        dist.all_gather_object(gathered, out)
        if shared:
            dist.barrier()
            ns.close()
        if rank == 0:
            q.put(gathered)
    finally:
        dist.destroy_process_group()


def _run(kind, world, n, p):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, n, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    return res


def _assemble(parts, key, n):
    y = np.full(n, np.nan)
    for part in parts:
        ids, v = part[key][0], part[key][1]
        assert np.all(np.isnan(y[ids])), "a DoF is owned by two ranks"
        y[ids] = v
    assert not np.any(np.isnan(y)), "a DoF is owned by no rank"
    return y


@pytest.mark.parametrize("kind,world,n,p", [("cg", 2, 4, 2), ("cg_dir", 2, 4, 3), ("cg_dir", 4, 4, 1),
                                            ("dg", 2, 3, 2), ("helm", 4, 3, 1), ("cg_shared", 2, 4, 2)])
def test_partitioned_apply_matches_global(kind, world, n, p):
    from oracle import ref_apply

    parts = _run(kind, world, n, p)
    kind = kind.replace("_shared", "")   # same problem, global setup published by rank 0 (NodeShared)
    m, dm, geo, bas, sipg, dids = _problem(kind, n, p)
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    y = _assemble(parts, "apply", dm.n_global_dofs)
    if kind.startswith("cg"):
        ref = ref_apply.cg_apply(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask, bas.grad_matrix,
                                 geo.cell_rule.weights, u)
    else:
        kap = 10.0 ** np.random.default_rng(2).uniform(-1, 1, m.n_cells) if kind == "helm" else None
        ref = ref_apply.dg_apply(m.vertices, m.cells, dm.n_dofs_per_cell, m.interior_faces, m.boundary_faces,
                                 set(dids), bas.value_matrix, bas.grad_matrix, geo.cell_rule.weights,
                                 bas.face_values, bas.face_grads, geo.face_rule.weights, sipg.tau_interior,
                                 sipg.tau_boundary, u, kappa=kap, mass_scale=1.0 if kind == "helm" else 0.0)
    err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
    assert err <= 1e-12, err
    if kind == "cg_dir":
        x = _assemble(parts, "pcg", dm.n_global_dofs)
        diag = ref_apply.cg_diagonal(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask, bas.grad_matrix,
                                     geo.cell_rule.weights, dm.n_global_dofs)
        A = lambda v: ref_apply.cg_apply(m.vertices, m.cells, dm.cell_dofs, dm.dirichlet_mask,  # noqa: E731
                                         bas.grad_matrix, geo.cell_rule.weights, v)
        b = np.where(dm.dirichlet_mask, 0.0, u)
        xr, hist = ref_apply.jacobi_pcg(A, diag, b, 12)
        assert np.linalg.norm(x - xr) / np.linalg.norm(xr) <= 1e-10
        assert np.allclose(parts[0]["pcg"][2], hist, rtol=1e-9)


def test_partition_is_balanced_and_deterministic():
    from paper_2509_10226_b200 import distributed as DD, mesh as M

    m = M.kuhn_cube_mesh(6, seed=0)
    for k in (1, 2, 4, 8):
        a, b = DD.partition_cells(m, k), DD.partition_cells(m, k)
        assert np.array_equal(a, b)
        counts = np.bincount(a, minlength=k)
        assert counts.max() - counts.min() <= 1
    with pytest.raises(ValueError):
        DD.partition_cells(m, 3)


def test_cg_subdomain_interior_cells_touch_no_ghosts():
    """Cells [0, n_interior) are applied while the forward halo is in flight, so they
    must not read any ghost DoF; together the subdomains cover every cell once."""
    from paper_2509_10226_b200 import distributed as DD, dofmap as D, mesh as M

    m = M.kuhn_cube_mesh(5, seed=2)
    dm = D.build_dof_map(m, 2, "cg", 1, (0, 1))
    part = DD.partition_cells(m, 4)
    seen = []
    for r in range(4):
        sub = DD.build_cg_subdomain(m, dm.cell_dofs, dm.dirichlet_mask, part, r, 4)
        ni = sub.n_interior_cells
        assert 0 < ni <= len(sub.cell_dofs)
        if r > 0:        # rank 0 owns every DoF it touches (owner = lowest touching rank)
            assert ni < len(sub.cell_dofs)
        assert np.all(sub.cell_dofs[:ni] < sub.n_owned)
        assert np.any(sub.cell_dofs[ni:] >= sub.n_owned, axis=1).all()
        assert np.array_equal(dm.cell_dofs[sub.cells_global], sub.l2g[sub.cell_dofs])
        seen.append(sub.cells_global)
    assert np.array_equal(np.sort(np.concatenate(seen)), np.arange(m.n_cells))


def test_ghost_owner_maps_point_at_the_owners_entries():
    """Peer-memory transport tables: ghost e of rank r is entry ghost_index[e] of rank
    ghost_owner[e]'s local layout, which holds the same global DoF / cell, owned there."""
    from paper_2509_10226_b200 import distributed as DD, dofmap as D, mesh as M

    m = M.kuhn_cube_mesh(5, seed=1)
    dm = D.build_dof_map(m, 2, "cg", 1, (0, 4))
    for k in (2, 4, 8):
        part = DD.partition_cells(m, k)
        subs = [DD.build_cg_subdomain(m, dm.cell_dofs, dm.dirichlet_mask, part, r, k) for r in range(k)]
        for r, s in enumerate(subs):
            gh = s.l2g[s.n_owned:]
            assert len(gh) == len(s.ghost_owner) == len(s.ghost_index)
            assert np.all(s.ghost_owner != r)
            for o in np.unique(s.ghost_owner):
                sel = s.ghost_owner == o
                assert np.all(s.ghost_index[sel] < subs[o].n_owned)
                assert np.array_equal(subs[o].l2g[s.ghost_index[sel]], gh[sel])
        dsubs = [DD.build_dg_subdomain(m, part, r, k) for r in range(k)]
        for r, s in enumerate(dsubs):
            gh = s.cell_l2g[s.n_owned_cells:]
            assert np.all(s.ghost_owner != r)
            for o in np.unique(s.ghost_owner):
                sel = s.ghost_owner == o
                assert np.all(s.ghost_index[sel] < dsubs[o].n_owned_cells)
                assert np.array_equal(dsubs[o].cell_l2g[s.ghost_index[sel]], gh[sel])


def _bench_shared_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), LOCAL_RANK=str(rank))
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench

        ns = bench.node_shared(world)
        assert ns is not None and ns.publisher == (rank == 0)
        ok = True
        for reorder in (False, True):
            for p in (1, 3):
                m, dm, _, _ = bench.build_problem(5, p, reorder, cache={}, ns=ns)
                m0, dm0, _, _ = bench.build_problem(5, p, reorder, cache={})
                ok &= all(np.array_equal(getattr(m, k), getattr(m0, k)) for k in bench._MESH_FIELDS)
                ok &= np.array_equal(dm.cell_dofs, dm0.cell_dofs) and np.array_equal(dm.dirichlet_mask, dm0.dirichlet_mask)
                ok &= dm.n_global_dofs == dm0.n_global_dofs
                if rank != 0:
                    ok &= not m.cells.flags.writeable and not dm.cell_dofs.flags.writeable
        shared_dir = ns.dir
        dist.barrier()
        ns.close()
        dist.barrier()
        res = [None] * world
        dist.all_gather_object(res, (bool(ok), os.path.isdir(shared_dir)))
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


def test_bench_builds_the_global_problem_once_per_node():
    """bench.py at N > 1: the global mesh / DoF maps come from the node's first rank through
    distributed.NodeShared, bit-identical to a rank's own build, and are removed afterwards."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_shared_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res == [(True, False), (True, False)]
