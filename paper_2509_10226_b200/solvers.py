"""Point-Jacobi preconditioned conjugate gradients (BASELINE config 5).

The reference specifies ``cg_solve`` but ships no solver;
the builder's decisions: x0 = 0, z = D^-1 r with the matrix-free
diagonal, exactly ``iters`` iterations (no early exit), ||r_k||_2 recorded.

* :func:`jacobi_pcg` -- single GPU, the whole loop in native code
  (``tmf_pcg``: apply + fused vector kernels, scalars on the device).
* :func:`pcg_loop` -- the same iteration driven from Python for the
  partitioned operator: every dot product is a local partial sum (fused
  kernel) followed by ``allreduce`` (NCCL all_reduce in the multi-GPU run),
  and all scalars stay on the device (one host sync at the end).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

__all__ = ["jacobi_pcg", "pcg_loop", "DeviceVecOps"]


def jacobi_pcg(op, b, iters: int = 100, stream: int | None = None):
    """Solve op x = b (b: CUDA tensor) with ``iters`` Jacobi-PCG iterations on one GPU.

    Returns (x tensor, residual norms ndarray of length iters+1)."""
    import torch

    x = torch.empty_like(b)
    hist = np.zeros(iters + 1)
    st = torch.cuda.current_stream(b.device).cuda_stream if stream is None else stream
    _lib.check(_lib.lib().tmf_pcg(op._plan, C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()), int(iters),
                                  _lib.ptr(hist, C.c_double), C.c_void_p(st)))
    return x, hist


class DeviceVecOps:
    """Native fused PCG vector kernels (tmf_vec_dot / tmf_pcg_*), device scalars."""

    def __init__(self):
        self.L = _lib.lib()

    @staticmethod
    def _p(t):
        return C.c_void_p(t.data_ptr())

    @staticmethod
    def _st(t):
        import torch

        return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)

    def dot(self, a, b, out):
        _lib.check(self.L.tmf_vec_dot(self._p(a), self._p(b), a.numel(), self._p(out), self._st(a)))

    def init(self, b, d, x, r, z, p, rz, rr):
        _lib.check(self.L.tmf_pcg_init(self._p(b), self._p(d), self._p(x), self._p(r), self._p(z), self._p(p),
                                       b.numel(), self._p(rz), self._p(rr), self._st(b)))

    def update(self, p, q, d, x, r, z, rz_k, pq_k, rz_next, rr_next):
        _lib.check(self.L.tmf_pcg_update(self._p(p), self._p(q), self._p(d), self._p(x), self._p(r), self._p(z),
                                         p.numel(), self._p(rz_k), self._p(pq_k), self._p(rz_next),
                                         self._p(rr_next), self._st(p)))

    def direction(self, z, p, rz_k, rz_next):
        _lib.check(self.L.tmf_pcg_direction(self._p(z), self._p(p), p.numel(), self._p(rz_k), self._p(rz_next),
                                            self._st(p)))


def pcg_loop(apply, diag, b, iters: int, allreduce=None, ops=None, n_local=None):
    """Jacobi-PCG on (possibly partitioned) vectors.

    ``apply(p, out=q)`` computes the owned slice of A p; ``allreduce(t)`` sums a
    small contiguous tensor across ranks in place (None: single process).  With
    ``n_local`` (a partitioned operator's local length) the search direction and
    A p live in rank-local buffers that the operator uses in place; the vector
    updates and dot products run on their owned prefix."""
    import torch

    ops = ops or DeviceVecOps()
    red = allreduce or (lambda t: None)
    n = b.numel()
    x, r, z = (torch.empty_like(b) for _ in range(3))
    if n_local is not None and n_local > n:
        p_buf = torch.zeros(n_local, dtype=b.dtype, device=b.device)
        q_buf = torch.empty(n_local, dtype=b.dtype, device=b.device)
        p, q = p_buf[:n], q_buf[:n]
        apply_pq = lambda: apply(p_buf, out=q_buf)  # noqa: E731
    else:
        p, q = torch.empty_like(b), torch.empty_like(b)
        apply_pq = lambda: apply(p, out=q)  # noqa: E731
    sc = torch.zeros(iters + 1, 3, dtype=torch.float64, device=b.device)   # [rz, rr, pq] per iteration
    ops.init(b, diag, x, r, z, p, sc[0, 0], sc[0, 1])
    red(sc[0, 0:2])
    for k in range(iters):
        apply_pq()
        ops.dot(p, q, sc[k, 2])
        red(sc[k, 2:3])
        ops.update(p, q, diag, x, r, z, sc[k, 0], sc[k, 2], sc[k + 1, 0], sc[k + 1, 1])
        red(sc[k + 1, 0:2])
        ops.direction(z, p, sc[k, 0], sc[k + 1, 0])
    del n
    return x, np.sqrt(sc[:, 1].cpu().numpy())
