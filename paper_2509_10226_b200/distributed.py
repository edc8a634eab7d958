"""Domain decomposition for multi-GPU applies (the reference is
single-process, SPEC.md:17 -- the paper scales with MPI + METIS).

One process per GPU.  The mesh is split into k subdomains by recursive
coordinate bisection of cell centroids (deterministic; k = 2^L gives the
2x2x2 blocks at k = 8).  Each rank runs the B200 plan of its local problem
and exchanges ghost data over NCCL (``torch.distributed`` P2P, grouped):

CG (identity Dirichlet rows kept):
    owner(d) = lowest rank whose cells touch DoF d; local vector = owned DoFs
    (ascending global id) then ghosts (by owner, then global id).
    apply: forward halo (owners -> ghost copies of u), local cell kernel,
    reverse halo (ghost partial y -> owner, added; constrained DoFs excluded,
    their rows are fixed by the owner), result = owned slice.
DG (SIPG / Helmholtz):
    local cells = owned cells (global order) + face-neighbour ghost cells;
    forward halo of the ghosts' u blocks only; partition faces are evaluated
    on both sides and each rank keeps its own cells' rows.  Artificial
    boundary faces of the ghost layer are never Dirichlet.
Krylov dot products: local partial sums over owned DoFs + all_reduce (sum).

The exchange lists are pure host data built identically on every rank.
``HaloExchange`` works with any torch.distributed backend: NCCL for GPU
tensors, gloo for the CPU tests (tests/test_distributed.py), where the local
apply is the CPU oracle; the GPU path plugs in the B200 plan.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .mesh import TetMesh, build_faces
from .reference import FACE_VERTICES_ARR

__all__ = ["partition_cells", "CgSubdomain", "DgSubdomain", "build_cg_subdomain",
           "build_dg_subdomain", "HaloExchange", "NodeShared"]


class NodeShared:
    """Global setup arrays built ONCE per node and mapped read-only by the other ranks.

    The subdomain builders need the global mesh, DoF map and partition (the reference's
    first-encounter DoF numbering is a global construction).  With one process per GPU,
    every rank building them itself costs world x the host time and memory (a 128^3 mesh
    and its DoF maps are several GB).  ``get(tag, build)``: the node's first rank calls
    ``build() -> {name: ndarray}`` and publishes the arrays as ``.npy`` files under
    ``/dev/shm`` (atomic rename); the other ranks wait for the directory and
    ``np.load(..., mmap_mode="r")`` them, so the pages are shared.  ``token`` must be the
    same on all ranks of one job and unique to it (``NodeShared.job_token()`` broadcasts
    one); ``close()`` on the publishing rank removes the files (mapped pages stay valid).
    """

    def __init__(self, local_rank: int, token: str, root: str = "/dev/shm", timeout_s: float = 7200.0):
        import os

        self.publisher = int(local_rank) == 0
        self.dir = os.path.join(root, f"tmf_b200_{token}")
        self.timeout_s = timeout_s
        self._cache = {}
        if self.publisher:
            os.makedirs(self.dir, exist_ok=True)

    @staticmethod
    def job_token(group=None) -> str:
        """A token unique to this job, agreed by all ranks (torch.distributed must be up;
        without it: a token private to this process)."""
        import os
        import time

        tok = [f"{os.getpid()}_{time.time_ns()}"]
        try:
            import torch.distributed as dist

            if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
                dist.broadcast_object_list(tok, src=0, group=group)
        except ImportError:
            pass
        return tok[0]

    def get(self, tag: str, build):
        import os
        import time

        if tag in self._cache:
            return self._cache[tag]
        d = os.path.join(self.dir, tag)
        if self.publisher:
            arrays = {k: np.ascontiguousarray(v) for k, v in build().items()}
            tmp = d + ".tmp"
            os.makedirs(tmp, exist_ok=True)
            for k, a in arrays.items():
                np.save(os.path.join(tmp, k + ".npy"), a)
            os.rename(tmp, d)
            self._cache[tag] = arrays
            return arrays
        t0 = time.time()
        while not os.path.isdir(d):
            if time.time() - t0 > self.timeout_s:
                raise TimeoutError(f"NodeShared: {d} was not published within {self.timeout_s} s")
            time.sleep(0.05)
        self._cache[tag] = {f[:-4]: np.load(os.path.join(d, f), mmap_mode="r") for f in sorted(os.listdir(d))
                            if f.endswith(".npy")}
        return self._cache[tag]

    def close(self):
        import shutil

        self._cache = {}
        if self.publisher:
            shutil.rmtree(self.dir, ignore_errors=True)


def partition_cells(mesh: TetMesh, k: int) -> np.ndarray:
    """Recursive coordinate bisection of cell centroids into k parts (k a power of 2).

    Each split sorts by (coordinate along the widest axis, cell id) and cuts at
    the middle, so the partition is deterministic."""
    if k < 1 or (k & (k - 1)):
        raise ValueError("k must be a power of two")
    cen = mesh.vertices[mesh.cells].mean(axis=1)
    part = np.zeros(mesh.n_cells, dtype=np.int64)

    def split(ids, lo, nparts):
        if nparts == 1:
            part[ids] = lo
            return
        c = cen[ids]
        axis = int(np.argmax(c.max(axis=0) - c.min(axis=0)))
        order = np.lexsort((ids, c[:, axis]))
        half = len(ids) // 2
        split(ids[order[:half]], lo, nparts // 2)
        split(ids[order[half:]], lo + nparts // 2, nparts // 2)

    split(np.arange(mesh.n_cells), 0, k)
    return part


@dataclass
class Exchange:
    """Per-rank halo plan: for each peer, local indices to pack and to unpack."""

    peers: list = field(default_factory=list)
    send: dict = field(default_factory=dict)    # peer -> local indices (pack)
    recv: dict = field(default_factory=dict)    # peer -> local indices (unpack)


@dataclass
class CgSubdomain:
    rank: int
    mesh: TetMesh                 # local cells, local vertex numbering
    cell_dofs: np.ndarray         # (n_local_cells, n_dpc) local DoF ids
    dirichlet_mask: np.ndarray    # (n_local,) bool
    l2g: np.ndarray               # local -> global DoF
    n_owned: int
    forward: Exchange             # u: owners -> ghosts
    reverse: Exchange             # y: ghosts -> owners (added)
    n_interior_cells: int = 0     # local cells [0, n) touch no ghost DoF (overlap the forward halo)
    cells_global: np.ndarray = None   # local cell -> global cell
    ghost_owner: np.ndarray = None    # (n_local - n_owned,) owner rank of each ghost DoF
    ghost_index: np.ndarray = None    # its index in the owner's local layout


@dataclass
class DgSubdomain:
    rank: int
    mesh: TetMesh                 # owned + ghost cells, local numbering
    cell_l2g: np.ndarray          # local -> global cell
    n_owned_cells: int
    dirichlet_faces: np.ndarray   # (n_bf_local,) bool
    interior_face_g: np.ndarray   # local interior face -> global interior face
    boundary_face_g: np.ndarray   # local boundary face -> global boundary face (-1 = artificial)
    forward: Exchange             # cell blocks of u: owners -> ghosts (cell indices)
    ghost_owner: np.ndarray = None    # (n_ghost_cells,) owner rank of each ghost cell
    ghost_index: np.ndarray = None    # its cell index in the owner's local layout


def _index_in_owner(owner: np.ndarray, k: int) -> np.ndarray:
    """Position of every entry among the entries of the same owner, ascending ids:
    the owner's local index of an owned DoF / cell (owned entries come first, in
    ascending global order, in every subdomain layout)."""
    order = np.argsort(owner, kind="stable")
    starts = np.concatenate([[0], np.cumsum(np.bincount(owner, minlength=k))[:-1]])
    idx = np.empty(len(owner), dtype=np.int64)
    idx[order] = np.arange(len(owner)) - starts[owner[order]]
    return idx


def _local_mesh(mesh: TetMesh, cells_g: np.ndarray) -> tuple[TetMesh, np.ndarray]:
    verts_g, cells_l = np.unique(mesh.cells[cells_g], return_inverse=True)
    cells_l = cells_l.reshape(-1, 4).astype(np.int32)
    ifc, bfc = build_faces(cells_l)
    return TetMesh(mesh.vertices[verts_g], cells_l, ifc, bfc), verts_g


def _touch_masks(cell_dofs: np.ndarray, part: np.ndarray, n_dofs: int, k: int) -> np.ndarray:
    """Bit r of mask[d] is set iff a cell of rank r touches DoF d (k <= 64)."""
    dt = np.uint8 if k <= 8 else (np.uint16 if k <= 16 else np.uint64)
    mask = np.zeros(n_dofs, dtype=dt)
    for r in range(k):
        mask[cell_dofs[part == r].ravel()] |= dt(1 << r)
    return mask


def _lowest_bit(mask: np.ndarray, k: int) -> np.ndarray:
    owner = np.full(len(mask), k, dtype=np.int64)
    for r in range(k - 1, -1, -1):
        owner[(mask >> r) & 1 == 1] = r
    return owner


def build_cg_subdomain(mesh: TetMesh, cell_dofs: np.ndarray, dirichlet_mask: np.ndarray,
                       part: np.ndarray, rank: int, k: int) -> CgSubdomain:
    """O(n) vectorised: touch bitmasks per DoF give owners (lowest touching rank),
    the rank's local numbering and every peer list."""
    nd = cell_dofs.shape[1]
    n_dofs = len(dirichlet_mask)
    mask = _touch_masks(cell_dofs, part, n_dofs, k)
    owner = _lowest_bit(mask, k)
    mine = ((mask >> rank) & 1).astype(bool)
    own = np.flatnonzero(mine & (owner == rank))
    gh = np.flatnonzero(mine & (owner != rank))
    gh = gh[np.argsort(owner[gh], kind="stable")]          # by (owner, global id)
    l2g = np.concatenate([own, gh])
    g2l = np.full(n_dofs, -1, dtype=np.int64)
    g2l[l2g] = np.arange(len(l2g))
    fwd, rev = Exchange(), Exchange()
    for s in range(k):
        if s == rank:
            continue
        on_s = ((mask >> s) & 1).astype(bool)
        gh_s = np.flatnonzero(on_s & (owner == rank))      # s's ghosts that I own (ascending)
        gh_r = np.flatnonzero(mine & (owner == s))         # my ghosts owned by s (ascending)
        if len(gh_s) == 0 and len(gh_r) == 0:
            continue
        fwd.peers.append(s)
        rev.peers.append(s)
        fwd.send[s] = g2l[gh_s]
        fwd.recv[s] = g2l[gh_r]
        # reverse: constrained DoFs are never scattered -> excluded
        rev.send[s] = g2l[gh_r[~dirichlet_mask[gh_r]]]
        rev.recv[s] = g2l[gh_s[~dirichlet_mask[gh_s]]]
    cells_g = np.flatnonzero(part == rank)
    touches_ghost = np.any(g2l[cell_dofs[cells_g].astype(np.int64)] >= len(own), axis=1)
    cells_g = np.concatenate([cells_g[~touches_ghost], cells_g[touches_ghost]])  # interior first
    lmesh, _ = _local_mesh(mesh, cells_g)
    lcd = g2l[cell_dofs[cells_g].astype(np.int64)].astype(np.int32).reshape(-1, nd)
    in_owner = _index_in_owner(owner, k)
    return CgSubdomain(rank, lmesh, lcd, dirichlet_mask[l2g], l2g, len(own), fwd, rev,
                       int(np.count_nonzero(~touches_ghost)), cells_g,
                       owner[gh].astype(np.int32), in_owner[gh].astype(np.int32))


def _face_index_tables(mesh: TetMesh):
    """(4*cell + lf) -> interior face index / boundary face index (or -1)."""
    n4 = 4 * mesh.n_cells
    fi = np.full(n4, -1, dtype=np.int64)
    ifc = mesh.interior_faces.astype(np.int64)
    idx = np.arange(len(ifc))
    fi[4 * ifc[:, 0] + ifc[:, 1]] = idx
    fi[4 * ifc[:, 2] + ifc[:, 3]] = idx
    bi = np.full(n4, -1, dtype=np.int64)
    bfc = mesh.boundary_faces.astype(np.int64)
    bi[4 * bfc[:, 0] + bfc[:, 1]] = np.arange(len(bfc))
    return fi, bi


def build_dg_subdomain(mesh: TetMesh, part: np.ndarray, rank: int, k: int,
                       dirichlet_ids=()) -> DgSubdomain:
    ifc = mesh.interior_faces.astype(np.int64)
    cm, cp = ifc[:, 0], ifc[:, 2]
    cross = part[cm] != part[cp]

    def ghosts_of(r):
        a = cross & (part[cm] == r)
        b = cross & (part[cp] == r)
        g = np.unique(np.concatenate([cp[a], cm[b]]))
        return g[np.argsort(part[g], kind="stable")]       # by (owner, global id)

    owned = np.flatnonzero(part == rank)
    ghosts = ghosts_of(rank)
    cells_g = np.concatenate([owned, ghosts])
    lmesh, _ = _local_mesh(mesh, cells_g)
    # local faces -> global faces through (global cell, local face) (same local face numbering)
    fi, bi = _face_index_tables(mesh)
    li, lb = lmesh.interior_faces.astype(np.int64), lmesh.boundary_faces.astype(np.int64)
    if_g = fi[4 * cells_g[li[:, 0]] + li[:, 1]]
    bf_g = bi[4 * cells_g[lb[:, 0]] + lb[:, 1]]            # -1: artificial (ghost-layer) face
    bfc = mesh.boundary_faces.astype(np.int64)
    bids = np.where(bf_g >= 0, bfc[np.maximum(bf_g, 0), 2], -1)
    lb_out = lb.copy()
    lb_out[:, 2] = bids
    lmesh.boundary_faces = lb_out.astype(np.int32)
    dset = np.array(sorted(dirichlet_ids), dtype=np.int64)
    dfaces = np.isin(bids, dset) & (bids >= 0)

    fwd = Exchange()
    n_own = len(owned)
    for s in range(k):
        if s == rank:
            continue
        gh_r = ghosts[part[ghosts] == s]                       # my ghosts owned by s
        gh_s = ghosts_of(s)
        gh_s = gh_s[part[gh_s] == rank]                         # s's ghosts owned by me
        if len(gh_r) == 0 and len(gh_s) == 0:
            continue
        fwd.peers.append(s)
        fwd.send[s] = np.searchsorted(owned, gh_s)             # local owned cell index
        fwd.recv[s] = n_own + np.flatnonzero(part[ghosts] == s)
    in_owner = _index_in_owner(part.astype(np.int64), k)
    return DgSubdomain(rank, lmesh, cells_g, n_own, dfaces, if_g, bf_g, fwd,
                       part[ghosts].astype(np.int32), in_owner[ghosts].astype(np.int32))


class HaloExchange:
    """Grouped P2P exchange over torch.distributed (NCCL on GPUs, gloo on CPU).

    ``block`` = entries per index (1 for CG DoFs, n_dpc*n_comp for DG cells).
    Pack/unpack are device gathers/scatters on the vector's own device."""

    def __init__(self, ex: Exchange, block: int, device):
        import torch

        self.peers = list(ex.peers)
        self.block = block
        self.send = {p: torch.as_tensor(self._expand(ex.send[p], block), device=device) for p in self.peers}
        self.recv = {p: torch.as_tensor(self._expand(ex.recv[p], block), device=device) for p in self.peers}
        self.sbuf = {p: None for p in self.peers}
        self.rbuf = {p: None for p in self.peers}

    @staticmethod
    def _expand(idx, block):
        idx = np.asarray(idx, dtype=np.int64)
        if block == 1:
            return idx
        return (idx[:, None] * block + np.arange(block)[None, :]).ravel()

    def start(self, vec):
        """Pack the send buffers and post the grouped P2P operations (non-blocking)."""
        import torch
        import torch.distributed as dist

        ops = []
        for p in self.peers:
            self.sbuf[p] = vec.index_select(0, self.send[p])
            self.rbuf[p] = torch.empty(len(self.recv[p]), dtype=vec.dtype, device=vec.device)
            if len(self.sbuf[p]):
                ops.append(dist.P2POp(dist.isend, self.sbuf[p], p))
            if len(self.rbuf[p]):
                ops.append(dist.P2POp(dist.irecv, self.rbuf[p], p))
        return dist.batch_isend_irecv(ops) if ops else []

    def finish(self, reqs, vec, add: bool):
        """Wait for the posted operations and unpack into ``vec`` (overwrite or accumulate)."""
        for req in reqs:
            req.wait()
        for p in self.peers:
            if len(self.rbuf[p]):
                if add:
                    vec.index_add_(0, self.recv[p], self.rbuf[p])
                else:
                    vec.index_copy_(0, self.recv[p], self.rbuf[p])

    def forward(self, vec):
        """Owners -> ghost copies (overwrite)."""
        self.finish(self.start(vec), vec, add=False)

    def reverse_add(self, vec):
        """Ghost partials -> owners (accumulate)."""
        self.finish(self.start(vec), vec, add=True)


# --------------------------------------------------------------------------- operators
def _stream_of(t):
    import torch

    return torch.cuda.current_stream(t.device).cuda_stream if t.is_cuda else 0


# --------------------------------------------------------------------------- peer memory
class _CudaArray:
    """__cuda_array_interface__ view of a raw device allocation (zero-copy tensor)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}


class PeerBuffers:
    """This rank's registered local u / y vectors for the peer-memory transport:
    dedicated device allocations (CUDA-IPC exportable at offset 0) wrapped as
    tensors.  Peers read ghost u from them and RED ghost y into them."""

    def __init__(self, n_local: int, device):
        import ctypes as C

        import torch

        from . import _lib

        self.n, self.device = int(n_local), device
        self.ptrs = []
        for _ in range(2):
            p = C.c_void_p()
            _lib.check(_lib.lib().tmf_alloc(C.c_int64(8 * max(self.n, 1)), int(device.index or 0), C.byref(p)))
            self.ptrs.append(p.value)
        self.u = torch.as_tensor(_CudaArray(self.ptrs[0], self.n), device=device)
        self.y = torch.as_tensor(_CudaArray(self.ptrs[1], self.n), device=device)
        self.u.zero_()
        self.y.zero_()
        self.opened = []

    def handles(self):
        import ctypes as C

        from . import _lib

        out = []
        for p in self.ptrs:
            h = (C.c_uint8 * 64)()
            _lib.check(_lib.lib().tmf_ipc_get_handle(C.c_void_p(p), h))
            out.append(bytes(h))
        return out

    def open(self, handle: bytes) -> int:
        import ctypes as C

        from . import _lib

        h = (C.c_uint8 * 64).from_buffer_copy(handle)
        p = C.c_void_p()
        _lib.check(_lib.lib().tmf_ipc_open_handle(h, int(self.device.index or 0), C.byref(p)))
        self.opened.append(p.value)
        return p.value

    def close(self):
        import ctypes as C

        from . import _lib

        if _lib is None or not hasattr(self, "ptrs"):
            return
        for p in self.opened:
            _lib.lib().tmf_ipc_close_handle(C.c_void_p(p))
        self.opened = []
        for p in self.ptrs:
            _lib.lib().tmf_free(C.c_void_p(p))
        self.ptrs = []

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass


class _PeerTransport:
    """Multi-GPU apply without a halo exchange (transport="p2p"): ghost entries are
    read (and, for CG, RED-scattered) by the cell / face kernels directly in the
    owner's registered buffers over NVLink peer memory (tmf_plan_set_peers), with
    two cross-rank barriers per apply.  ``connect_ipc`` maps the peers' buffers of
    other processes (CUDA IPC); ``connect_local`` links operators that share one
    process (ranks emulated on one device: same kernels, same peer tables)."""

    def _peer_init(self, n_local, ghost_owner, ghost_index, n_own):
        self.bufs = PeerBuffers(n_local, self.device)
        self._ghost_owner = np.ascontiguousarray(ghost_owner, dtype=np.int32)
        self._ghost_index = np.ascontiguousarray(ghost_index, dtype=np.int32)
        self._peer_n_own = int(n_own)
        self._bar = None
        self.connected = False

    def connect_peers(self, ptrs_u, ptrs_y):
        import ctypes as C

        from . import _lib

        assert len(ptrs_u) == self.world
        u64 = (C.c_uint64 * self.world)(*[int(p) for p in ptrs_u])
        y64 = (C.c_uint64 * self.world)(*[int(p) for p in ptrs_y]) if ptrs_y is not None else None
        gr, gi = self._ghost_owner, self._ghost_index
        _lib.check(_lib.lib().tmf_plan_set_peers(
            self.local_op._plan, self.world, u64, y64, self.rank, self._peer_n_own, len(gr),
            _lib.ptr(gr, C.c_int32), _lib.ptr(gi, C.c_int32), int(getattr(self, "_peer_free_cells", 0))))
        self._peer_ptrs = (list(ptrs_u), None if ptrs_y is None else list(ptrs_y))
        self.connected = True

    def set_transport(self, transport: str):
        """Switch a connected operator between the peer-memory path and the NCCL halo
        path (e.g. to cross-check them); the plan's peer tables follow."""
        import ctypes as C

        from . import _lib

        if transport == "nccl":
            if getattr(self, "connected", False):
                _lib.check(_lib.lib().tmf_plan_set_peers(self.local_op._plan, 0, None, None, 0, 0, 0, None, None, 0))
        elif transport == "p2p":
            if not getattr(self, "_peer_ptrs", None):
                raise RuntimeError("peer transport: connect first")
            self.connect_peers(*self._peer_ptrs)
        else:
            raise ValueError(f"unknown transport {transport!r}")
        self.transport = transport
        del C

    def connect_ipc(self, group=None):
        """Exchange CUDA-IPC handles of every rank's registered buffers (collective)."""
        import torch.distributed as dist

        mine = self.bufs.handles()
        allh = [None] * self.world
        dist.all_gather_object(allh, mine, group=group)
        pu, py = [], []
        for r in range(self.world):
            if r == self.rank:
                pu.append(self.bufs.ptrs[0])
                py.append(self.bufs.ptrs[1])
            else:
                pu.append(self.bufs.open(allh[r][0]))
                py.append(self.bufs.open(allh[r][1]))
        self._group = group
        self.connect_peers(pu, py if self._peer_writes_y else None)

    @staticmethod
    def connect_local(ops):
        """Link the rank operators of one process (emulated ranks on one device)."""
        pu = [op.bufs.ptrs[0] for op in ops]
        py = [op.bufs.ptrs[1] for op in ops]
        for op in ops:
            op.connect_peers(pu, py if op._peer_writes_y else None)

    def barrier(self):
        """Cross-rank barrier ordered on the current stream (NCCL: a 1-element
        all_reduce; other backends: device sync + host barrier)."""
        import torch
        import torch.distributed as dist

        if not dist.is_initialized() or self.world == 1:
            return
        group = getattr(self, "_group", None)
        if dist.get_backend(group) == "nccl":
            if self._bar is None:
                self._bar = torch.zeros(1, dtype=torch.float64, device=self.device)
            dist.all_reduce(self._bar, group=group)
        else:
            torch.cuda.synchronize(self.device)
            dist.barrier(group=group)

    # phases (apply = stage_in | barrier | compute | barrier | result)
    def p2p_stage_in(self, u):
        from . import _lib

        n = self.n_owned
        if u.data_ptr() != self.bufs.u.data_ptr():
            self.bufs.u[:n].copy_(u[:n])
        if self._peer_writes_y:   # CG: zero y before any peer can RED into it
            self.local_op.apply_stages(self.bufs.u.data_ptr(), self.bufs.y.data_ptr(), _lib.STAGE_ZERO, 0, 0,
                                       _stream_of(self.bufs.u))

    def p2p_result(self, out):
        return _local_result(self.bufs.y, out, self.n_owned)

    def _apply_p2p(self, u, out):
        if not self.connected:
            raise RuntimeError("peer transport: call connect_ipc() (or connect_local) first")
        self.p2p_stage_in(u)
        self.barrier()
        ev = self._event_pair() if hasattr(self, "_event_pair") else None
        self.p2p_compute()
        if ev is not None:
            self._close_events(ev)
        self.barrier()
        return self.p2p_result(out)


def _local_buffers(op, u, out, n):
    """(u_loc, y_loc) for one apply: caller tensors of the local length are used in
    place; owned-length input is copied into the operator's local buffer."""
    nl = op.u_loc.numel()
    if u.numel() == nl:      # local layout (or a rank without ghosts): in place
        u_loc = u
    elif u.numel() == n:
        op.u_loc[:n].copy_(u)
        u_loc = op.u_loc
    else:
        raise ValueError(f"vector length {u.numel()} is neither the owned ({n}) nor the local ({nl}) size")
    y_loc = out if (out is not None and out.numel() == nl) else op.y_loc
    return u_loc, y_loc


def _local_result(y_loc, out, n):
    if out is None:
        return y_loc[:n].clone()
    if out.data_ptr() != y_loc.data_ptr():
        out.copy_(y_loc[:n])
    return out


class DistributedCgOperator(_PeerTransport):
    """CG Laplace apply on a k-way partition: y_owned = A u_owned.

    ``local_factory(mesh, dofmap, geometry, basis)`` may supply the local apply
    (a callable on local vectors); by default it is the rank's B200 plan, whose
    kernels run on the rank's current CUDA device."""

    def __init__(self, mesh, dofmap, geometry, basis, rank: int, world: int, part=None,
                 device=None, local_factory=None, transport: str = "nccl"):
        import torch

        from .dofmap import DoFMap
        from .operator import CgPoissonOperator, OperatorConfig

        if transport not in ("nccl", "p2p"):
            raise ValueError(f"unknown transport {transport!r}")
        self.transport = transport
        self.rank, self.world = rank, world
        self.part = partition_cells(mesh, world) if part is None else part
        self.sub = build_cg_subdomain(mesh, dofmap.cell_dofs, dofmap.dirichlet_mask, self.part, rank, world)
        n_local = len(self.sub.l2g)
        ldm = DoFMap("cg", dofmap.degree, 1, n_local, self.sub.cell_dofs, self.sub.dirichlet_mask)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if local_factory is None:
            # the halo overlap runs cell RANGES (interior cells first): the caller's order
            op = CgPoissonOperator(self.sub.mesh, ldm, geometry, basis,
                                   OperatorConfig(device=self.device.index or 0, cell_order="input"))
            self.local_op = op

            def local(u, y):
                op.apply_into(u.data_ptr(), y.data_ptr(), _stream_of(u))
        else:
            self.local_op = None
            fn = local_factory(self.sub.mesh, ldm, geometry, basis)

            def local(u, y):
                y.copy_(fn(u))
        self._local = local
        self.fwd = HaloExchange(self.sub.forward, 1, self.device)
        self.rev = HaloExchange(self.sub.reverse, 1, self.device)
        self.u_loc = torch.zeros(n_local, dtype=torch.float64, device=self.device)
        self.y_loc = torch.zeros(n_local, dtype=torch.float64, device=self.device)
        self._peer_writes_y = True
        if transport == "p2p":
            if self.local_op is None:
                raise ValueError("the p2p transport needs the B200 local plan")
            self._peer_init(n_local, self.sub.ghost_owner, self.sub.ghost_index, self.sub.n_owned)
            self._peer_free_cells = self.sub.n_interior_cells

    @property
    def n_owned(self) -> int:
        return self.sub.n_owned

    @property
    def owned_global_ids(self) -> np.ndarray:
        return self.sub.l2g[: self.sub.n_owned]

    kernel_events = None   # set to a list to record (start, end) CUDA events of the local apply

    def _event_pair(self):
        if self.kernel_events is None:
            return None
        import torch

        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        return (e0, e1)

    def _close_events(self, ev):
        if ev is not None:
            ev[1].record()
            self.kernel_events.append(ev)

    def _timed_local_on(self, u_loc, y_loc):
        import torch

        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        self._local(u_loc, y_loc)
        e1.record()
        self.kernel_events.append((e0, e1))

    @property
    def n_local(self) -> int:
        """Length of the rank-local layout (owned DoFs first, then ghost slots)."""
        return len(self.sub.l2g)

    def apply(self, u_owned, out=None):
        """Forward halo overlapped with the interior cells (no ghost DoF), then the
        boundary cells, the identity rows and the additive reverse halo.

        ``u_owned`` / ``out`` have the owned length (copied through internal local
        buffers) or the local length ``n_local`` (used in place, no copies: the ghost
        slots of ``u`` are overwritten by the halo, ``out[:n_owned]`` is the result)."""
        from . import _lib

        if self.transport == "p2p":
            return self._apply_p2p(u_owned, out)
        n = self.sub.n_owned
        u_loc, y_loc = _local_buffers(self, u_owned, out, n)
        reqs = self.fwd.start(u_loc)
        if self.local_op is None:           # external local apply (tests): no stages
            self.fwd.finish(reqs, u_loc, add=False)
            if self.kernel_events is None:
                self._local(u_loc, y_loc)
            else:
                self._timed_local_on(u_loc, y_loc)
        else:
            op, st = self.local_op, _stream_of(u_loc)
            up, yp = u_loc.data_ptr(), y_loc.data_ptr()
            ev = self._event_pair()
            op.apply_stages(up, yp, _lib.STAGE_ZERO | _lib.STAGE_CELLS, 0, self.sub.n_interior_cells, st)
            self._close_events(ev)
            self.fwd.finish(reqs, u_loc, add=False)
            ev = self._event_pair()
            op.apply_stages(up, yp, _lib.STAGE_CELLS | _lib.STAGE_FIXUP, self.sub.n_interior_cells, None, st)
            self._close_events(ev)
        self.rev.reverse_add(y_loc)
        return _local_result(y_loc, out, n)

    def p2p_compute(self):
        """All local cells in one kernel: ghost u by peer loads, ghost y by peer REDs."""
        from . import _lib

        b = self.bufs
        self.local_op.apply_stages(b.u.data_ptr(), b.y.data_ptr(), _lib.STAGE_CELLS | _lib.STAGE_FIXUP, 0, None,
                                   _stream_of(b.u))

    def diagonal(self):
        """Owned slice of diag(A): local matrix-free diagonal + reverse halo."""
        import torch

        from . import _lib
        import ctypes as C

        d = torch.zeros(len(self.sub.l2g), dtype=torch.float64, device=self.device)
        _lib.check(_lib.lib().tmf_diagonal(self.local_op._plan, C.c_void_p(d.data_ptr()),
                                            C.c_void_p(_stream_of(d))))
        self.rev.reverse_add(d)
        return d[: self.sub.n_owned].clone()


class DistributedDgOperator(_PeerTransport):
    """DG-SIPG / Helmholtz apply on a k-way partition (forward halo of ghost cells only).

    ``kind`` = "sipg" or "helmholtz" (scalar mass + per-cell kappa, KappaHelmholtzOperator)."""

    def __init__(self, mesh, dofmap, geometry, basis, sipg, rank: int, world: int, kind="sipg",
                 dirichlet_ids=(), kappa=None, mass_scale=1.0, part=None, device=None, local_factory=None,
                 transport: str = "nccl"):
        import torch

        if transport not in ("nccl", "p2p"):
            raise ValueError(f"unknown transport {transport!r}")
        self.transport = transport

        from .dofmap import DoFMap
        from .operator import DgSipgOperator, KappaHelmholtzOperator, OperatorConfig, SipgConfig

        self.rank, self.world = rank, world
        self.part = partition_cells(mesh, world) if part is None else part
        sub = self.sub = build_dg_subdomain(mesh, self.part, rank, world, dirichlet_ids)
        nd = dofmap.cell_dofs.shape[1]
        nc = dofmap.n_components
        self.block = nd * nc
        n_loc_cells = len(sub.cell_l2g)
        ldm = DoFMap("dg", dofmap.degree, nc, n_loc_cells * nd,
                     np.arange(n_loc_cells * nd, dtype=np.int32).reshape(n_loc_cells, nd),
                     np.zeros(n_loc_cells * nd, dtype=bool))
        tau_i = np.asarray(sipg.tau_interior)[sub.interior_face_g]
        tau_b = np.where(sub.boundary_face_g >= 0,
                         np.asarray(sipg.tau_boundary)[np.maximum(sub.boundary_face_g, 0)], 0.0)
        lsipg = SipgConfig(sipg.penalty_constant, tau_i, tau_b)
        lkappa = None if kappa is None else np.asarray(kappa)[sub.cell_l2g]
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        cfg = OperatorConfig(device=self.device.index or 0) if self.device.type == "cuda" else None
        if local_factory is None:
            if kind == "sipg":
                op = DgSipgOperator(sub.mesh, ldm, geometry, basis, lsipg, cfg, dirichlet_ids)
            else:
                op = KappaHelmholtzOperator(sub.mesh, ldm, geometry, basis, lsipg, lkappa, mass_scale, cfg,
                                            dirichlet_ids)
            self.local_op = op

            def local(u, y):
                op.apply_into(u.data_ptr(), y.data_ptr(), _stream_of(u))
        else:
            self.local_op = None
            fn = local_factory(sub.mesh, ldm, geometry, basis, lsipg, lkappa, dirichlet_ids)

            def local(u, y):
                y.copy_(fn(u))
        self._local = local
        self.fwd = HaloExchange(sub.forward, self.block, self.device)
        n_local = n_loc_cells * self.block
        self.u_loc = torch.zeros(n_local, dtype=torch.float64, device=self.device)
        self.y_loc = torch.zeros(n_local, dtype=torch.float64, device=self.device)
        self._peer_writes_y = False   # DG: ghost cells' u is read from the owner, nothing is written back
        if transport == "p2p":
            if self.local_op is None:
                raise ValueError("the p2p transport needs the B200 local plan")
            if nc != 1:
                raise ValueError("the p2p transport supports scalar DG (n_components = 1)")
            self._peer_init(n_local, sub.ghost_owner, sub.ghost_index, sub.n_owned_cells)

    @property
    def n_owned(self) -> int:
        return self.sub.n_owned_cells * self.block

    @property
    def n_local(self) -> int:
        """Length of the rank-local layout (owned cells' DoFs first, then ghost cells')."""
        return self.u_loc.numel()

    def owned_global_ids(self) -> np.ndarray:
        c = self.sub.cell_l2g[: self.sub.n_owned_cells]
        return (c[:, None] * self.block + np.arange(self.block)[None, :]).ravel()

    def apply(self, u_owned, out=None):
        """Forward halo overlapped with the owned cells' volume terms (ghost cells'
        volume terms are never needed), then all face terms."""
        from . import _lib

        if self.transport == "p2p":
            return self._apply_p2p(u_owned, out)
        n = self.n_owned
        u_loc, y_loc = _local_buffers(self, u_owned, out, n)
        reqs = self.fwd.start(u_loc)
        if self.local_op is None:
            self.fwd.finish(reqs, u_loc, add=False)
            self._local(u_loc, y_loc)
        else:
            op, st = self.local_op, _stream_of(u_loc)
            up, yp = u_loc.data_ptr(), y_loc.data_ptr()
            op.apply_stages(up, yp, _lib.STAGE_CELLS, 0, self.sub.n_owned_cells, st)
            self.fwd.finish(reqs, u_loc, add=False)
            op.apply_stages(up, yp, _lib.STAGE_FACES, 0, 0, st)
        return _local_result(y_loc, out, n)

    def p2p_compute(self):
        """Owned cells' volume terms, then every face (plus-side ghost cells' u by peer loads)."""
        from . import _lib

        b = self.bufs
        st = _stream_of(b.u)
        self.local_op.apply_stages(b.u.data_ptr(), b.y.data_ptr(), _lib.STAGE_CELLS, 0, self.sub.n_owned_cells, st)
        self.local_op.apply_stages(b.u.data_ptr(), b.y.data_ptr(), _lib.STAGE_FACES, 0, 0, st)
