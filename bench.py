"""Benchmark of the B200 matrix-free operator apply (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config c2]

Workload (BASELINE.json configs[1], "C2"): CG Laplace operator apply, degree
sweep P1..P4, fp64, on the 48^3 x 6 = 663,552-cell jittered, randomly permuted
Kuhn mesh (seed 0), Grundmann-Moller quadrature exact to 2p, u ~ U[-1,1]
(seed 1).  One *step* = one apply at each degree, on the unordered mesh and on
the hierarchically reordered mesh (8 applies); ``value`` = DoFs processed /
device time (GDoF/s).  Inputs and plans are resident in HBM before timing;
L2 is flushed (256 MiB write) before every apply, outside the timed events.

``e2e`` times the same step through the public API with host buffers
(``Operator.apply(numpy)`` -> ``tmf_apply_host``: pinned H2D of u, apply, D2H
of y), wall clock.  ``--impl reference`` times the CPU oracle port of the
reference's batched NumPy loop (oracle/ref_apply.py; the reference package
itself cannot travel to the GPU box) with one worker process per host core
on a bounded sample of batches of the same workload, extrapolated per DoF.

Multi-GPU (torchrun, N>1): ``scaling: "weak"``.  The global mesh grows to
round(48 N^(1/3))^3 x 6 cells, is split by recursive coordinate bisection into
N subdomains (paper_2509_10226_b200.distributed), and every apply runs the
forward NCCL halo, the local B200 kernel and the reverse (additive) halo;
``value`` = global DoFs per step / max-over-ranks step time.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")   # CPU arm: one BLAS thread per worker

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.1   # measured: DMMA m8n8k4 on this pool's B200 (profiles/r01_fp64_peak.json)
FP64_PEAK_SOURCE = "profiles/r01_fp64_peak.json (mma.sync m8n8k4 f64 microbench on B200, 1965 MHz)"
DEGREES = (1, 2, 3, 4)
ENGINE_NAMES = {1: "dmma-quadrature", 3: "dmma-reference-tensor",
                4: "dmma-modal (point kernel on M = dim P_(p-1) exact modes)"}
KERNEL_NAMES = {1: "cell_apply_kernel (n_q points)", 3: "cell_tensor_kernel",
                4: "cell_apply_kernel (modal tables)"}
N_MESH = 48


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=["c2"])
    ap.add_argument("--n", type=int, default=N_MESH)
    ap.add_argument("--no-reorder", action="store_true")
    ap.add_argument("--cpu-sample-s", type=float, default=2.5)
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline (e.g. under ncu)")
    ap.add_argument("--dist", action="store_true", help="use the partitioned (NCCL) path even at world size 1")
    ap.add_argument("--no-quadrature", action="store_true", help="skip the quadrature-point engine comparison")
    return ap.parse_args()


# ----------------------------------------------------------------- workload
_MESHES = {}


def build_problem(n, p, reorder):
    """Mesh (cached per (n, reorder): the reordering and the partition are shared by
    all degrees), DoF map, tables."""
    from paper_2509_10226_b200 import basis as B, dofmap as D, mesh as M, quadrature as Q
    from paper_2509_10226_b200.geometry import GeometryData

    key = (n, reorder)
    if key not in _MESHES:
        m = M.kuhn_cube_mesh(n, seed=0)
        if reorder:
            from paper_2509_10226_b200.reorder import reorder_mesh

            m = reorder_mesh(m)   # hierarchical cell order + first-touch vertex numbering
        _MESHES[key] = m
    m = _MESHES[key]
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    dm = D.build_dof_map(m, p, "cg")
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    return m, dm, geo, bas


_PARTS = {}


def partition_of(m, world):
    from paper_2509_10226_b200.distributed import partition_cells

    key = (id(m), world)
    if key not in _PARTS:
        _PARTS[key] = partition_cells(m, world)
    return _PARTS[key]


def variants(args):
    vs = [False]
    if not args.no_reorder:
        try:
            import paper_2509_10226_b200.reorder  # noqa: F401
            vs.append(True)
        except ImportError:
            pass
    return vs


# ----------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    NAMES = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
             0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, dev=0, period=0.005):
        self.samples, self.reasons, self.ok = [], 0, False
        self.period, self._stop = period, threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": ["unavailable"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max,
                "reasons": [v for k, v in self.NAMES.items() if self.reasons & k], "samples": len(self.samples)}


# ----------------------------------------------------------------- reference arm / cpu baseline
def _cpu_worker(args):
    p, n, b0, b1, reorder = args
    from oracle import ref_apply

    m, dm, geo, bas, jit, jxw = _CPU_CACHE[(p, reorder)]
    gidx = dm.cell_dofs.astype(np.int64)
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    y = np.zeros_like(u)
    ids, act = ref_apply._cell_batches(m.n_cells, 4, 4)
    t0 = time.perf_counter()
    for b in range(b0, b1):
        sub = ids[b]
        idx = gidx[sub].T.copy()
        idx[:, ~act[b]] = -1
        U = ref_apply.gather(u, idx)
        G = (bas.grad_matrix @ U).reshape(-1, 3, U.shape[1])
        Dd = ref_apply.d_action_affine(G, jit[sub], jxw[sub])
        R = bas.grad_matrix.T @ Dd.reshape(-1, U.shape[1])
        ref_apply.scatter_add(y, idx, R)
    return time.perf_counter() - t0, b1 - b0


_CPU_CACHE = {}


def cpu_reference(args, sample_s, workers=None):
    """Time the oracle port of the reference's batched NumPy loop (kernel_stage "mm":
    W=4 lanes x 4 cells per batch, operator.py:77-87) on all host cores; returns the
    aggregate GDoF/s over the P1..P4 sweep, extrapolated from a bounded sample."""
    import multiprocessing as mp

    workers = workers or os.cpu_count() or 1
    tot_dofs, tot_time, detail = 0.0, 0.0, {}
    for reorder in variants(args):
        for p in DEGREES:
            from oracle import ref_apply

            m, dm, geo, bas = build_problem(args.n, p, reorder)
            jit, jxw, _ = ref_apply.affine_cell_geometry(m.vertices, m.cells, geo.cell_rule.weights)
            _CPU_CACHE[(p, reorder)] = (m, dm, geo, bas, jit, jxw)
            n_batches = (m.n_cells + 15) // 16
            # calibrate batches/second on one worker, then give each worker ~sample_s
            dt, nb = _cpu_worker((p, args.n, 0, 20, reorder))
            per = max(1, int(sample_s * nb / dt))
            chunks = [(p, args.n, (w * per) % n_batches, min(n_batches, (w * per) % n_batches + per), reorder)
                      for w in range(workers)]
            ctx = mp.get_context("fork")
            with ctx.Pool(workers) as pool:
                res = pool.map(_cpu_worker, chunks)
            wall = max(r[0] for r in res)                # concurrent loops: slowest worker
            done = sum(r[1] for r in res)
            t_full = wall * n_batches / done            # extrapolated apply time, all cores
            tot_dofs += dm.n_global_dofs
            tot_time += t_full
            detail[f"p{p}{'_reordered' if reorder else ''}"] = {
                "gdofs": dm.n_global_dofs / t_full / 1e9, "batches_sampled": done, "n_batches": n_batches}
    return tot_dofs / tot_time / 1e9, workers, detail


# ----------------------------------------------------------------- GPU arm
def measure_link(problems, reps):
    """Pinned host <-> device copy rates of this box, measured live on the largest plan's
    vectors (H2D alone, D2H alone, both at once on two streams), and the lower bound they put
    on one e2e step: every plan's u goes up and its y comes down, a plan's D2H cannot start
    before its own H2D has finished, so a step takes at least max((H + D) / duplex,
    (H + s_max) / min(h2d, d2h)) whatever the order (two-stage flow shop, equal job sizes)."""
    import torch

    big = max(problems, key=lambda pr: pr["ndof"])
    nbytes = 8 * big["ndof"]
    dev_u = torch.empty(big["ndof"], dtype=torch.float64, device="cuda")
    dev_y = big["y"][: big["ndof"]]
    s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()
    reps = max(3, reps)

    def rate(up, dn):
        dev_u.copy_(big["u_pin"], non_blocking=True)   # warm
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            if up:
                with torch.cuda.stream(s_up):
                    dev_u.copy_(big["u_pin"], non_blocking=True)
            if dn:
                with torch.cuda.stream(s_dn):
                    big["y_pin"].copy_(dev_y, non_blocking=True)
        torch.cuda.synchronize()
        return (up + dn) * nbytes * reps / (time.perf_counter() - t0) / 1e9

    h2d, d2h, duplex = rate(True, False), rate(False, True), rate(True, True)
    tot = sum(8 * pr["ndof"] for pr in problems)
    bound_s = max(2 * tot / (duplex * 1e9), (tot + nbytes) / (min(h2d, d2h) * 1e9))
    del dev_u
    return {"h2d_GBs": round(h2d, 1), "d2h_GBs": round(d2h, 1), "duplex_GBs": round(duplex, 1),
            "step_bound_ms": round(bound_s * 1e3, 3)}


def gpu_bench(args, rank, world):
    import torch

    from paper_2509_10226_b200 import operator as op

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    cfg = op.OperatorConfig(device=dev)
    st = torch.cuda.current_stream().cuda_stream
    # weak scaling: each rank keeps ~n^3 x 6 cells (global mesh grows with the world size)
    n_glob = args.n if world == 1 else int(round(args.n * world ** (1.0 / 3.0)))
    # multi-GPU transport: "p2p" = ghost DoFs read / RED-scattered by the cell kernel in
    # the owner's buffers over NVLink (CUDA IPC), "nccl" = NCCL halo exchange
    transport = os.environ.get("TMF_TRANSPORT", "p2p")
    problems = []
    for reorder in variants(args):
        for p in DEGREES:
            m, dm, geo, bas = build_problem(n_glob, p, reorder)
            u_glob = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
            if world == 1 and not args.dist:
                A = op.CgPoissonOperator(m, dm, geo, bas, cfg)
                ids = None
                local = A
            else:
                from paper_2509_10226_b200.distributed import DistributedCgOperator

                A = DistributedCgOperator(m, dm, geo, bas, rank, world, part=partition_of(m, world),
                                          transport=transport)
                if transport == "p2p":
                    # CUDA-IPC mapping of the peers' buffers; if any rank cannot map them,
                    # every rank falls back to the NCCL halo transport
                    ok = 1.0
                    try:
                        A.connect_ipc()
                    except Exception as e:  # noqa: BLE001
                        print(f"rank {rank}: peer mapping failed ({e}); NCCL halo instead", file=sys.stderr)
                        ok = 0.0
                    flag = torch.tensor([ok], dtype=torch.float64, device="cuda")
                    if world > 1:
                        torch.distributed.all_reduce(flag, op=torch.distributed.ReduceOp.MIN)
                    if float(flag[0]) < 1.0:
                        transport = "nccl"
                        for q in problems:
                            if q["ids"] is not None:
                                q["A"].set_transport("nccl")
                        A.set_transport("nccl")
                ids = A.owned_global_ids
                local = A.local_op
            u_host = u_glob if ids is None else u_glob[ids]
            u = torch.from_numpy(np.ascontiguousarray(u_host)).cuda()
            if ids is not None and transport == "p2p" and A.transport == "p2p":
                # the registered (peer-visible) local buffers, used in place
                A.bufs.u[: len(u_host)].copy_(u)
                u, y = A.bufs.u, A.bufs.y
            elif ids is not None:
                # rank-local layout (owned DoFs, then ghost slots): the partitioned apply
                # works on these vectors in place (no owned <-> local copies)
                ul = torch.zeros(A.n_local, dtype=torch.float64, device="cuda")
                ul[: len(u_host)] = u
                u = ul
                y = torch.empty_like(u)
            else:
                y = torch.empty_like(u)
            u_pin = torch.from_numpy(np.ascontiguousarray(u_host)).pin_memory()
            y_pin = torch.empty_like(u_pin).pin_memory()
            problems.append(dict(p=p, reorder=reorder, A=A, local=local, u=u, y=y, u_pin=u_pin, y_pin=y_pin,
                                 ndof=len(u_host), ndof_global=dm.n_global_dofs, ids=ids))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    # self-check of the peer-memory transport against the NCCL halo path (same plans)
    p2p_check = None
    if (world > 1 or args.dist) and transport == "p2p":
        err = 0.0
        for pr in problems:
            A, n = pr["A"], pr["ndof"]
            y1 = A.apply(pr["u"])
            A.set_transport("nccl")
            y2 = A.apply(pr["u"])
            A.set_transport("p2p")
            err = max(err, float(torch.linalg.vector_norm(y1[:n] - y2[:n]) / torch.linalg.vector_norm(y2[:n])))
        t = torch.tensor([err], dtype=torch.float64, device="cuda")
        if world > 1:
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        p2p_check = float(t[0])
        if not p2p_check <= 1e-12:
            for pr in problems:
                pr["A"].set_transport("nccl")
            transport = "nccl"

    def timed_apply(pr):
        """(total, cell-kernel) ms of one apply, CUDA events on the launch stream."""
        if world == 1 and not args.dist:
            ms = pr["A"].timed(pr["u"].data_ptr(), pr["y"].data_ptr(), st, 1)
            return float(ms[0]), float(ms[1])
        A = pr["A"]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        A.kernel_events = []
        e0.record()
        A.apply(pr["u"], out=pr["y"])
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1), sum(k0.elapsed_time(k1) for k0, k1 in A.kernel_events)

    def step(record):
        for pr in problems:
            flush.fill_(1.0)
            ms = timed_apply(pr)
            if record is not None:
                record.append((pr, ms))

    for _ in range(args.warmup):
        step(None)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    rec = []
    with ClockSampler(dev) as clk:
        for _ in range(args.steps):
            step(rec)
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    total_ms = sum(ms[0] for _, ms in rec)
    dofs = sum(pr["ndof"] for pr, _ in rec)   # owned DoFs of this rank

    # e2e through the public API with host (pinned) buffers
    n_streams = int(os.environ.get("TMF_E2E_STREAMS", "8"))
    # largest plans first: the D2H of the big vectors starts as early as possible
    e2e_order = sorted(problems, key=lambda pr: -pr["ndof"]) if os.environ.get("TMF_E2E_ORDER", "desc") == "desc" \
        else list(problems)
    streams = [torch.cuda.Stream() for _ in range(n_streams)]
    e2e_path = os.environ.get("TMF_E2E_PATH", "streams")
    e2e_multi = e2e_path in ("multi", "blocks")
    e2e_sched = None
    if e2e_path == "blocks":
        # reordered plans streamed in cell blocks (their cells touch narrow DoF windows), each
        # ahead of its unordered twin; schedules built here, outside the timed region
        nblk = int(os.environ.get("TMF_E2E_BLOCKS", "16"))
        e2e_order = sorted(problems, key=lambda pr: (-pr["ndof"], not pr["reorder"]))
        e2e_sched = [pr["A"].host_schedule(nblk) if pr["reorder"] else None for pr in e2e_order]

    def e2e_step():
        if world == 1 and not args.dist:
            # public C-ABI with host buffers; the plans' H2D / kernels / D2H are
            # pipelined on one stream per plan, so the H2D and D2H copy engines and the
            # SMs work on different plans at the same time
            if e2e_multi:
                op.apply_host_multi([pr["A"] for pr in e2e_order], [pr["u_pin"] for pr in e2e_order],
                                    [pr["y_pin"] for pr in e2e_order], streams[0].cuda_stream,
                                    schedules=e2e_sched)
            else:
                for i, pr in enumerate(e2e_order):
                    pr["A"].apply_host_async(pr["u_pin"], pr["y_pin"], streams[i % len(streams)].cuda_stream)
            torch.cuda.synchronize()
            return
        for pr in problems:   # host -> device, partitioned apply (NCCL halo), device -> host
            u = pr["u_pin"].cuda(non_blocking=True)
            pr["y_pin"].copy_(pr["A"].apply(u), non_blocking=True)
        torch.cuda.synchronize()
    e2e_step()
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_s = time.perf_counter() - t0

    # parity spot check of the timed path against the e2e path (P2, unordered)
    pr0 = problems[1]
    y0 = pr0["y"][: pr0["ndof"]].cpu()
    err = float(torch.linalg.vector_norm(y0 - pr0["y_pin"]) / torch.linalg.vector_norm(pr0["y_pin"]))

    link = measure_link(problems, args.steps) if (world == 1 and not args.dist) else None

    per = {}
    for pr in problems:
        key = f"p{pr['p']}{'_reordered' if pr['reorder'] else ''}"
        ms = np.array([m for q, m in rec if q is pr])
        t = ms[:, 0].mean()
        tc = ms[:, 1].mean()
        info = pr["local"].info
        per[key] = {"ndof": pr["ndof"], "ms": round(float(t), 4), "gdofs": round(pr["ndof"] / t / 1e6, 3),
                    "cell_kernel_ms": round(float(tc), 4), "cell_engine": ENGINE_NAMES.get(info["cell_engine"]),
                    # useful flops of the algorithm the kernel runs (reference tensor: 12 N^2 + 12 N + N per cell)
                    "tflops_engine": round(info["flops_engine"] / tc / 1e9, 2),
                    "frac_fp64": round(info["flops_engine"] / tc / 1e9 / FP64_PEAK_TFLOPS, 3),
                    # the reference counter formula (quadrature-point loop, operator.py:227-242) / the same time:
                    # the rate the reference's own algorithm would need to match this time (> peak possible)
                    "tflops_ref_formula": round(info["flops_alg"] / tc / 1e9, 2)}
    # dominant kernel = the cell kernel of the slowest apply
    dom = max(problems, key=lambda q: per[f"p{q['p']}{'_reordered' if q['reorder'] else ''}"]["cell_kernel_ms"])
    dk = f"p{dom['p']}{'_reordered' if dom['reorder'] else ''}"
    tc = per[dk]["cell_kernel_ms"]
    achieved = dom["local"].info["flops_engine"] / tc / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("cell_kernel_p4", {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    n_kern = sum(pr["local"].info["kernels_per_apply"] for pr in problems) * args.steps

    # the paper's own algorithm (quadrature-point DMMA engine) on the reordered meshes, timed the
    # same way after the main timed region (reported beside it, not part of ``value``)
    quad = None
    if world == 1 and not args.dist and not args.no_quadrature:
        quad = {}
        for pr in problems:
            if not pr["reorder"] and len(variants(args)) > 1:
                continue
            m, dm, geo, bas = build_problem(n_glob, pr["p"], pr["reorder"])
            Aq = op.CgPoissonOperator(m, dm, geo, bas, op.OperatorConfig(device=dev, cell_engine="dmma"))
            Aq.timed(pr["u"].data_ptr(), pr["y"].data_ptr(), st, 2)
            tq = []
            for _ in range(args.steps):
                flush.fill_(1.0)
                tq.append(Aq.timed(pr["u"].data_ptr(), pr["y"].data_ptr(), st, 1))
            tq = np.array(tq)
            t, tc = float(tq[:, 0].mean()), float(tq[:, 1].mean())
            quad[f"p{pr['p']}"] = {"ms": round(t, 4), "gdofs": round(pr["ndof"] / t / 1e6, 3),
                                   "cell_kernel_ms": round(tc, 4),
                                   "frac_fp64": round(Aq.info["flops_alg"] / tc / 1e9 / FP64_PEAK_TFLOPS, 3)}
            del Aq
    dofs_global = sum(pr["ndof_global"] for pr, _ in rec)
    return dict(total_ms=total_ms, dofs=dofs, dofs_global=dofs_global, n_glob=n_glob, e2e_s=e2e_s, per=per, clocks=clk.summary(),
                transport=transport, p2p_check=p2p_check, quadrature_engine=quad,
                roofline={"bound": "tensor", "kernel": f"{KERNEL_NAMES.get(dom['local'].info['cell_engine'])} ({dk})",
                          "achieved": round(achieved, 3),
                          "peak": FP64_PEAK_TFLOPS, "peak_source": FP64_PEAK_SOURCE, "unit": "TFLOP/s",
                          "frac": round(achieved / FP64_PEAK_TFLOPS, 4), "traffic": traffic,
                          "algorithmic": "useful flops of the algorithm the cell engine runs, per launch "
                                         "(tmf_plan_info.flops_engine: modal 12 M N + 18 M + N per cell, M = dim "
                                         "P_(p-1), N = DoFs per cell; reference tensor 12 N^2 + 13 N) / CUDA-event "
                                         "kernel time"},
                gpu_launches=n_kern, parity_rel_l2=err, link=link,
                e2e_desc={"streams": "Operator.apply_host_async(pinned host u, y) -> tmf_apply_host_async, one stream "
                                     "per plan, largest first",
                          "multi": "operator.apply_host_multi -> tmf_apply_host_multi (upload / compute / download "
                                   "pipeline), largest first",
                          "blocks": "operator.apply_host_multi(schedules) -> tmf_apply_host_multi_blocks: reordered "
                                    "plans streamed in cell blocks, each ahead of its unordered twin, largest first"
                          }.get(e2e_path, e2e_path) if (world == 1 and not args.dist) else
                "host -> device, partitioned apply, device -> host",
                h2d=sum(8 * pr["ndof"] for pr in problems), d2h=sum(8 * pr["ndof"] for pr in problems))


_STDOUT_FD = None


def emit(line):
    """The one JSON line, on the real stdout (everything else -- e.g. the NCCL version
    banner that libnccl prints on fd 1 -- was redirected to stderr)."""
    os.write(_STDOUT_FD if _STDOUT_FD is not None else 1, (json.dumps(line) + "\n").encode())


def main():
    global _STDOUT_FD
    sys.stdout.flush()
    _STDOUT_FD = os.dup(1)
    os.dup2(2, 1)
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    workload = (f"CG Laplace apply, P1-P4 sweep, {args.n}^3x6 jittered permuted Kuhn tets, GM quadrature 2p, "
                f"fp64, unordered{'' if args.no_reorder else ' + hierarchically reordered'}")
    metric, unit = "operator-apply GDoF/s (fp64), CG Laplace P1-P4 sweep", "GDoF/s"
    if args.impl == "reference":
        if rank != 0:
            return
        val, cores, detail = cpu_reference(args, args.cpu_sample_s)
        line = {"impl": "reference", "metric": metric, "value": val, "unit": unit, "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "dtype": "f64",
                "data": "synthetic",
                # same workload as the b200 arm at this world size; the bounded CPU sample is drawn
                # from the 48^3 mesh (the per-DoF rate of the batched loop does not depend on size)
                "config": {"workload": workload,
                           "global_mesh": f"{args.n if world == 1 else int(round(args.n * world ** (1.0 / 3.0)))}^3 x 6",
                           "sample_mesh": f"{args.n}^3 x 6"},
                "cpu_baseline": {"value": val, "unit": unit, "cores": cores, "kind": "port",
                                 "sample": f"oracle port of the reference batched NumPy loop (16-cell batches), "
                                           f"~{args.cpu_sample_s}s per worker per degree, extrapolated per DoF",
                                 "detail": detail},
                "e2e": {"value": val, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        emit(line)
        return

    if world > 1 or args.dist:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29561")
        dev = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(dev)
        # eager communicator init + a collective first: batch_isend_irecv requires that all
        # ranks take part in the first NCCL call, and halo peers are a subset of the ranks
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", dev))
        dist.barrier()
    r = gpu_bench(args, rank, world)
    total_ms = r["total_ms"]
    if world > 1:
        import torch
        import torch.distributed as dist

        t = torch.tensor([total_ms, r["e2e_s"]], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, e2e_s = float(t[0]), float(t[1])
    else:
        e2e_s = r["e2e_s"]
    value = r["dofs_global"] / (total_ms * 1e-3) / 1e9
    e2e_val = r["dofs_global"] / e2e_s / 1e9
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            v, cores, detail = cpu_reference(args, min(args.cpu_sample_s, 1.5))
            cpu = {"value": v, "unit": unit, "cores": cores, "kind": "port",
                   "sample": "oracle port of the reference batched NumPy loop, ~1.5 s per worker per degree, "
                             "extrapolated per DoF", "detail": detail}
        except Exception as e:  # the CPU baseline is reported, not required for the GPU number
            cpu = {"value": None, "error": str(e)[:200]}
    if rank == 0:
        line = {"metric": metric, "value": round(value, 4), "unit": unit, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload, "l2": "flushed (256 MiB write) before every apply",
                           "global_mesh": f"{r['n_glob']}^3 x 6",
                           "parallelism": (f"{world}-way RCB domain decomposition, "
                                           + ("ghost DoFs gathered / RED-scattered by the cell kernel in peer "
                                              "memory (NVLink, CUDA IPC)" if r["transport"] == "p2p" else "NCCL halo")
                                           + f" (weak scaling: ~{args.n}^3 x 6 cells per GPU)")
                           if (world > 1 or args.dist) else "single GPU",
                           "transport": r["transport"] if (world > 1 or args.dist) else None,
                           "p2p_vs_nccl_rel_l2": r["p2p_check"]},
                "per_degree": r["per"], "roofline": r["roofline"], "cpu_baseline": cpu,
                "quadrature_engine": r["quadrature_engine"],
                "e2e": {"value": round(e2e_val, 4), "unit": unit, "h2d_bytes_per_step": r["h2d"],
                        "d2h_bytes_per_step": r["d2h"], "path": r["e2e_desc"],
                        "ms_per_step": round(e2e_s / args.steps * 1e3, 3),
                        # the box's PCIe link measured live; frac = link lower bound / measured step
                        "link": None if r["link"] is None else dict(
                            r["link"], frac=round(r["link"]["step_bound_ms"] / (e2e_s / args.steps * 1e3), 3))},
                "gpu_launches": r["gpu_launches"], "clocks": r["clocks"], "parity_e2e_vs_timed_rel_l2": r["parity_rel_l2"]}
        emit(line)
    if world > 1 or args.dist:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
