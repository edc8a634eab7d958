"""B200 matrix-free operators behind the reference's operator interface.

Drop-in mirrors of the reference classes (operator.py:57-134, 311-493):

* ``OperatorConfig``, ``SipgConfig``, ``HelmholtzCoefficients`` -- same fields
  and validation (operator.py:57-114);
* ``CgPoissonOperator(mesh, dofmap, geometry, basis, config=None)``;
* ``DgSipgOperator(mesh, dofmap, geometry, basis, sipg, config=None, dirichlet_ids=())``;
* ``HelmholtzOperator(mesh, dofmap, geometry, basis, sipg, coeffs, config=None, dirichlet_ids=())``
  -- the reference's 3-component constant-coefficient operator;
* ``KappaHelmholtzOperator`` -- BASELINE config 4's scalar mass + per-cell
  kappa Laplace (SURVEY §8c-3 convention);
* ``compute_sipg_tau``, ``baseline_sipg_tau`` and the ``apply_*`` wrappers.

``apply(u)`` accepts a NumPy vector (copied to and from the device, a fresh
``y`` is returned as in operator.py:324) or a CUDA ``torch.Tensor`` (zero
copy, ordered on torch's current stream).  Every apply runs the sm_100a
kernels of libtetmf_b200.so; there is no CPU path.  The constructor accepts
either this package's objects or the reference's own (duck-typed: only array
fields are read).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .counters import FlopCounters, reference_apply_counts

__all__ = ["OperatorConfig", "SipgConfig", "HelmholtzCoefficients", "CgPoissonOperator",
           "DgSipgOperator", "HelmholtzOperator", "KappaHelmholtzOperator", "compute_sipg_tau",
           "baseline_sipg_tau", "apply_cg_poisson", "apply_dg_sipg", "apply_helmholtz"]

_STAGES = ("ref", "data", "mm", "sched")
_ENGINES = {"auto": 0, "dmma": 1, "tensor": 3, "modal": 4}
_BLOCKS = {"auto": 0, "off": 1, "on": 2}
_ORDERS = {"auto": 0, "input": 1, "morton": 2}
_FACE_ENGINES = {"auto": 0, "quadrature": 1, "modal_flat": 2, "modal": 3}


@dataclass(frozen=True)
class OperatorConfig:
    """operator.py:57-91.  Stage/batching/lane-width select CPU SIMD layouts in the
    reference; on the B200 they are validated and recorded but the kernel layout
    (8-cell DMMA tiles) is fixed.  ``device`` selects the CUDA ordinal."""

    kernel_stage: str = "mm"
    batching: str = "cells"
    lane_width: int | None = None
    quadrature_variant: str = "standard"
    precision: str = "f64"
    threads: int = 1
    backend: str = "auto"
    device: int = 0
    face_chunk: int = 0          # 8-face batches per CTA chunk, multiple of 8 up to 120 (0 = default 32)
    cell_engine: str = "auto"    # B200 cell kernel: auto | dmma (quadrature points) | tensor (affine
    #                              reference tensor) | modal (points loop on the M = dim P_{p-1} exact modes)
    cell_blocks: str = "auto"    # B200 CG block assembly (low degrees on locality-ordered meshes): auto | off | on
    face_engine: str = "auto"    # B200 faces: auto (modal at P2-P4) | quadrature (points) | modal | modal_flat
    f32_mirror: bool = False     # B200 CG Laplace: also build the fp32 apply (apply_f32; mixed-precision multigrid)
    cell_order: str = "auto"     # B200 CG traversal: auto (Morton when the mesh order has no locality) | input | morton

    def __post_init__(self):
        if self.kernel_stage not in _STAGES:
            raise ValueError(f"unknown kernel stage {self.kernel_stage!r}")
        if self.batching not in ("cells", "components"):
            raise ValueError(f"unknown batching {self.batching!r}")
        if self.precision not in ("f32", "f64"):
            raise ValueError(f"unknown precision {self.precision!r}")
        if self.cell_engine not in _ENGINES:
            raise ValueError(f"unknown cell engine {self.cell_engine!r}")
        if self.cell_blocks not in _BLOCKS:
            raise ValueError(f"unknown cell block mode {self.cell_blocks!r}")
        if self.cell_order not in _ORDERS:
            raise ValueError(f"unknown cell order {self.cell_order!r}")
        if self.face_engine not in _FACE_ENGINES:
            raise ValueError(f"unknown face engine {self.face_engine!r}")
        if self.backend not in ("auto", "compiled", "python", "b200"):
            raise ValueError(f"unknown backend {self.backend!r}")

    @property
    def dtype(self):
        return np.float64


@dataclass
class HelmholtzCoefficients:
    mass_scale: float
    diffusivity: float

    def __post_init__(self):
        if self.mass_scale < 0 or self.diffusivity < 0:
            raise ValueError("coefficients must be non-negative")
        if self.mass_scale == 0 and self.diffusivity == 0:
            raise ValueError("mass_scale and diffusivity cannot both vanish")


@dataclass
class SipgConfig:
    penalty_constant: float = 1.0
    tau_interior: np.ndarray = field(default=None)
    tau_boundary: np.ndarray = field(default=None)


def compute_sipg_tau(mesh, geo, p: int, penalty_constant: float = 1.0) -> SipgConfig:
    """operator.py:117-134: tau = C (p+1)(p+3)/3 max(area/vol); boundary x2."""
    base = penalty_constant * (p + 1) * (p + 3) / 3.0
    vols = geo.cell_volumes
    ifc, bfc = mesh.interior_faces, mesh.boundary_faces
    tau_i = base * np.maximum(geo.face_areas / vols[ifc[:, 0]], geo.face_areas / vols[ifc[:, 2]]) \
        if len(ifc) else np.empty(0)
    tau_b = base * 2.0 * geo.bnd_areas / vols[bfc[:, 0]] if len(bfc) else np.empty(0)
    if len(tau_i) and not np.all(tau_i > 0):
        raise ValueError("non-positive interior penalty")
    return SipgConfig(penalty_constant, tau_i, tau_b)


def baseline_sipg_tau(mesh, p: int, h: float) -> SipgConfig:
    """BASELINE.json penalty tau = 2.5 (p+1)^2 / h on every interior and boundary face."""
    t = 2.5 * (p + 1) ** 2 / h
    return SipgConfig(1.0, np.full(len(mesh.interior_faces), t), np.full(len(mesh.boundary_faces), t))


def _c(a, dtype):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype)


class _B200Operator:
    _kind = None
    n_components = 1

    def __init__(self, mesh, dofmap, geometry, basis, config=None, *, sipg=None,
                 dirichlet_ids=(), mass_scale=0.0, diffusivity=1.0, kappa=None):
        if mesh is None:
            raise ValueError("the B200 operators need the mesh: geometry is recomputed from vertices")
        self.mesh, self.dofmap, self.geo, self.basis = mesh, dofmap, geometry, basis
        self.config = config or OperatorConfig()
        # geometry.py:139-142: unknown modes and affine-on-curved are errors in the reference.  The
        # kernels recompute the AFFINE map of every cell from its 4 vertices, which is the
        # reference's per-point geometry too whenever the cells are straight (its quadratic
        # geometry nodes are then the affine midpoints, geometry.py:77-83); curved cells have no
        # B200 path and are rejected instead of silently linearised.
        mode = getattr(geometry, "mode", "affine")
        if mode not in ("affine", "per_point"):
            raise ValueError(f"unknown geometry mode {mode!r}")
        if getattr(mesh, "is_curved", False) or getattr(mesh, "geometry_nodes", None) is not None:
            if mode == "affine":
                raise ValueError("affine geometry requested for a curved mesh; use per-point mode")
            raise ValueError("curved (per-point) geometry is not supported by the B200 operators: "
                             "the kernels use the affine map of each cell's vertices")
        if self.config.batching == "components" and int(dofmap.n_components) != 3:
            raise ValueError("components batching requires a 3-component space")   # operator.py:197-198
        self.precision = self.config.precision
        if self.precision == "f32" and (self._kind != _lib.TMF_CG_LAPLACE or int(dofmap.n_components) != 1
                                        or kappa is not None):
            raise ValueError("precision='f32' is implemented for the scalar CG Laplace operator only on "
                             "the B200 path (DG / Helmholtz run in f64)")
        self.counters = FlopCounters()
        self.n_applies = 0
        self.dirichlet_ids = frozenset(int(b) for b in dirichlet_ids)
        self._plan = C.c_void_p()
        p = int(dofmap.degree)
        nd = int(dofmap.cell_dofs.shape[1])
        keep = {}
        k = keep.setdefault
        d = _lib.PlanDesc()
        d.operator_kind = self._kind
        d.degree = p
        d.n_dofs_per_cell = nd
        d.n_components = int(dofmap.n_components)
        d.n_vertices = len(mesh.vertices)
        d.n_cells = len(mesh.cells)
        d.n_scalar_dofs = int(dofmap.n_scalar_dofs)
        d.vertices = _lib.ptr(k("v", _c(mesh.vertices, np.float64)), C.c_double)
        d.cells = _lib.ptr(k("c", _c(mesh.cells, np.int32)), C.c_int32)
        cell_rule = geometry.cell_rule
        d.n_q = int(len(cell_rule.weights))
        d.cell_weights = _lib.ptr(k("w", _c(cell_rule.weights, np.float64)), C.c_double)
        d.value_matrix = _lib.ptr(k("E", _c(basis.value_matrix, np.float64)), C.c_double)
        d.grad_matrix = _lib.ptr(k("G", _c(basis.grad_matrix, np.float64)), C.c_double)
        if dofmap.space == "cg":
            d.cell_dofs = _lib.ptr(k("cd", _c(dofmap.cell_dofs, np.int32)), C.c_int32)
            mask = np.asarray(dofmap.dirichlet_mask, dtype=bool)
            if mask.any():
                d.dirichlet_mask = _lib.ptr(k("m", mask.astype(np.uint8)), C.c_uint8)
        if sipg is not None:
            face_rule = geometry.face_rule
            if face_rule is None:
                raise ValueError("geometry was built without face data")
            d.n_qf = int(len(face_rule.weights))
            d.face_weights = _lib.ptr(k("fw", _c(face_rule.weights, np.float64)), C.c_double)
            d.face_values = _lib.ptr(k("fv", _c(basis.face_values, np.float64)), C.c_double)
            d.face_grads = _lib.ptr(k("fg", _c(basis.face_grads, np.float64)), C.c_double)
            ifc = _c(mesh.interior_faces, np.int32)
            bfc = _c(mesh.boundary_faces, np.int32)
            d.n_interior_faces = len(ifc)
            d.interior_faces = _lib.ptr(k("if", ifc), C.c_int32)
            d.tau_interior = _lib.ptr(k("ti", _c(sipg.tau_interior, np.float64)), C.c_double)
            d.n_boundary_faces = len(bfc)
            d.boundary_faces = _lib.ptr(k("bf", bfc), C.c_int32)
            if sipg.tau_boundary is not None and len(bfc):
                d.tau_boundary = _lib.ptr(k("tb", _c(sipg.tau_boundary, np.float64)), C.c_double)
            bd = np.isin(bfc[:, 2], np.array(sorted(self.dirichlet_ids), dtype=np.int64)).astype(np.uint8) \
                if len(bfc) else np.zeros(0, np.uint8)
            d.boundary_dirichlet = _lib.ptr(k("bd", bd), C.c_uint8)
        if kappa is not None:
            kap = k("kap", _c(kappa, np.float64))
            if kap.shape != (len(mesh.cells),):
                raise ValueError("kappa must hold one coefficient per cell")
            d.kappa = _lib.ptr(kap, C.c_double)
        d.mass_scale = float(mass_scale)
        d.diffusivity = float(diffusivity)
        d.device = int(self.config.device)
        eng = _ENGINES[getattr(self.config, "cell_engine", "auto")]
        d.flags = ((int(getattr(self.config, "face_chunk", 0)) // 8 & 0xF) << 8) | \
            ((eng & 3) << 13) | ((eng >> 2) << 19) | \
            (_BLOCKS[getattr(self.config, "cell_blocks", "auto")] << 15) | \
            (_FACE_ENGINES[getattr(self.config, "face_engine", "auto")] << 17) | \
            ((1 if (getattr(self.config, "f32_mirror", False) or self.precision == "f32") else 0) << 20) | \
            (_ORDERS[getattr(self.config, "cell_order", "auto")] << 22)
        _lib.check(_lib.lib().tmf_plan_create(C.byref(d), C.byref(self._plan)))
        info = _lib.PlanInfo()
        _lib.check(_lib.lib().tmf_plan_get_info(self._plan, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in info._fields_}
        # the reference's per-apply counter increments (operator.py:227-248, 416-437)
        self._apply_counts = reference_apply_counts(
            self.config, dofmap, d.n_q, int(d.n_qf), interior_faces=getattr(mesh, "interior_faces", None),
            boundary_faces=getattr(mesh, "boundary_faces", None), dirichlet_ids=self.dirichlet_ids,
            mass_scale=mass_scale, diffusivity=diffusivity, affine=mode == "affine", faces=sipg is not None)

    # -- lifecycle
    def close(self):
        if self._plan:
            _lib.lib().tmf_plan_destroy(self._plan)
            self._plan = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def n_global_dofs(self) -> int:
        return int(self.info["n_global_dofs"])

    def _check_length(self, u):
        if len(u) != self.n_global_dofs:
            raise ValueError(f"vector length {len(u)} does not match {self.n_global_dofs} DoFs")

    def _count(self):
        self.counters.add_all(self._apply_counts)
        self.n_applies += 1

    # -- apply
    def apply(self, u, out=None):
        """y = A u.  NumPy in -> fresh NumPy out (or ``out``, e.g. a pinned buffer);
        CUDA tensor in -> CUDA tensor out.  ``precision="f32"`` (CG Laplace) computes in
        single precision and returns float32, as the reference does (operator.py:323-324)."""
        self._check_length(u)
        if self.precision == "f32":
            return self._apply_single(u, out)
        if type(u).__module__.startswith("torch"):
            import torch

            if not u.is_cuda:
                u = u.detach().cpu().numpy()
            else:
                u = u.to(torch.float64).contiguous()
                y = torch.empty_like(u)
                self.apply_into(u.data_ptr(), y.data_ptr(), torch.cuda.current_stream(u.device).cuda_stream)
                return y
        u = np.ascontiguousarray(u, dtype=np.float64)
        y = np.empty_like(u) if out is None else out
        if y.dtype != np.float64 or not y.flags.c_contiguous or y.shape != u.shape:
            raise ValueError("out must be a contiguous float64 vector of the operator size")
        _lib.check(_lib.lib().tmf_apply_host(self._plan, _lib.ptr(u, C.c_double), _lib.ptr(y, C.c_double)))
        self._count()
        return y

    def _apply_single(self, u, out=None):
        import torch

        if type(u).__module__.startswith("torch") and u.is_cuda:
            ut = u.to(torch.float32).contiguous()
            y = torch.empty_like(ut)
            self.apply_f32(ut, out=y)
            self._count()
            return y
        un = np.ascontiguousarray(u.detach().cpu().numpy() if hasattr(u, "detach") else u, dtype=np.float32)
        ut = torch.from_numpy(un).to(torch.device("cuda", int(self.config.device)))
        yt = self.apply_f32(ut)
        y = yt.cpu().numpy()
        self._count()
        if out is not None:
            out[...] = y
            return out
        return y

    def apply_host_async(self, u_host, y_host, stream: int = 0):
        """Enqueue H2D(u), apply, D2H(y) on ``stream`` and return (pinned host arrays
        or tensors; they must outlive the stream work)."""
        up = _host_buffer(u_host, self.n_global_dofs)
        yp = _host_buffer(y_host, self.n_global_dofs)
        _lib.check(_lib.lib().tmf_apply_host_async(self._plan, C.c_void_p(up), C.c_void_p(yp), C.c_void_p(stream)))
        self._count()

    def apply_stages(self, u_ptr: int, y_ptr: int, stages: int, cell_begin: int = 0, cell_end: int | None = None,
                     stream: int = 0):
        """Part of the apply (``_lib.STAGE_*`` bits) on cells [cell_begin, cell_end)."""
        end = len(self.mesh.cells) if cell_end is None else cell_end
        _lib.check(_lib.lib().tmf_apply_stages(self._plan, C.c_void_p(u_ptr), C.c_void_p(y_ptr), int(stages),
                                                int(cell_begin), int(end), C.c_void_p(stream)))

    def apply_into(self, u_ptr: int, y_ptr: int, stream: int = 0):
        """Raw device-pointer apply (y overwritten), ordered on ``stream``."""
        _lib.check(_lib.lib().tmf_apply(self._plan, C.c_void_p(u_ptr), C.c_void_p(y_ptr), C.c_void_p(stream)))
        self._count()

    def apply_f32(self, u, out=None, stream: int | None = None):
        """y = A u in single precision (CUDA float32 tensors; plans built with
        ``OperatorConfig(f32_mirror=True)``): the mixed-precision V-cycle's operator."""
        import torch

        self._check_length(u)
        if u.dtype != torch.float32 or not u.is_cuda:
            raise ValueError("apply_f32 needs a CUDA float32 tensor")
        y = torch.empty_like(u) if out is None else out
        st = torch.cuda.current_stream(u.device).cuda_stream if stream is None else stream
        _lib.check(_lib.lib().tmf_apply_f32(self._plan, C.c_void_p(u.data_ptr()), C.c_void_p(y.data_ptr()),
                                            C.c_void_p(st)))
        return y

    def timed(self, u_ptr: int, y_ptr: int, stream: int = 0, reps: int = 1):
        """(total, cell, face, fixup) ms per apply from CUDA events on ``stream``."""
        out = np.zeros(4)
        _lib.check(_lib.lib().tmf_apply_timed(self._plan, C.c_void_p(u_ptr), C.c_void_p(y_ptr),
                                               C.c_void_p(stream), int(reps), _lib.ptr(out, C.c_double), 4))
        return out


class CgPoissonOperator(_B200Operator):
    """operator.py:311-331 (identity rows on Dirichlet DoFs)."""

    _kind = _lib.TMF_CG_LAPLACE

    def __init__(self, mesh, dofmap, geometry, basis, config=None, kappa=None):
        """``kappa`` (B200 extension, keyword only in practice): per-cell coefficient of the
        Laplacian, -div(kappa grad u); None = the reference operator."""
        if dofmap.space != "cg":
            raise ValueError("CG operator needs a CG dof map")
        super().__init__(mesh, dofmap, geometry, basis, config, kappa=kappa)

    def diagonal(self, stream: int = 0):
        """Matrix-free diag(A) as a CUDA tensor (identity on Dirichlet rows)."""
        import torch

        d = torch.empty(self.n_global_dofs, dtype=torch.float64, device=f"cuda:{self.config.device}")
        _lib.check(_lib.lib().tmf_diagonal(self._plan, C.c_void_p(d.data_ptr()),
                                            C.c_void_p(stream or torch.cuda.current_stream().cuda_stream)))
        return d


class DgSipgOperator(_B200Operator):
    """operator.py:446-466 (weak Dirichlet on ``dirichlet_ids``)."""

    _kind = _lib.TMF_DG_SIPG

    def __init__(self, mesh, dofmap, geometry, basis, sipg, config=None, dirichlet_ids=()):
        if dofmap.space != "dg":
            raise ValueError("DG operator needs a DG dof map")
        super().__init__(mesh, dofmap, geometry, basis, config, sipg=sipg,
                         dirichlet_ids=dirichlet_ids, diffusivity=1.0)


class HelmholtzOperator(_B200Operator):
    """operator.py:469-493: mass_scale*M + diffusivity*A_sipg on 3 interleaved components."""

    _kind = _lib.TMF_DG_HELMHOLTZ

    def __init__(self, mesh, dofmap, geometry, basis, sipg, coeffs, config=None, dirichlet_ids=()):
        if dofmap.space != "dg" or dofmap.n_components != 3:
            raise ValueError("Helmholtz operator needs a 3-component DG space")
        self.coeffs = coeffs
        super().__init__(mesh, dofmap, geometry, basis, config, sipg=sipg, dirichlet_ids=dirichlet_ids,
                         mass_scale=coeffs.mass_scale, diffusivity=coeffs.diffusivity)


class KappaHelmholtzOperator(_B200Operator):
    """BASELINE config 4: mass_scale*M + A_sipg(kappa) with a per-cell coefficient.

    Face convention: m± <- kappa± m±, tau_F <- tau max(kappa-, kappa+);
    boundary m <- kappa m, tau <- tau kappa."""

    _kind = _lib.TMF_DG_HELMHOLTZ

    def __init__(self, mesh, dofmap, geometry, basis, sipg, kappa, mass_scale=1.0, config=None,
                 dirichlet_ids=()):
        if dofmap.space != "dg":
            raise ValueError("Helmholtz operator needs a DG dof map")
        super().__init__(mesh, dofmap, geometry, basis, config, sipg=sipg, dirichlet_ids=dirichlet_ids,
                         mass_scale=mass_scale, diffusivity=1.0, kappa=kappa)


def apply_cg_poisson(config, dofmap, geometry, basis, u, mesh=None):
    return CgPoissonOperator(mesh, dofmap, geometry, basis, config).apply(u)


def apply_dg_sipg(config, mesh, dofmap, geometry, basis, sipg, u, dirichlet_ids=()):
    return DgSipgOperator(mesh, dofmap, geometry, basis, sipg, config, dirichlet_ids).apply(u)


def apply_helmholtz(config, mesh, dofmap, geometry, basis, sipg, coeffs, u, dirichlet_ids=()):
    return HelmholtzOperator(mesh, dofmap, geometry, basis, sipg, coeffs, config, dirichlet_ids).apply(u)


def _host_buffer(t, n: int) -> int:
    """Address of a host (CPU) float64 C-contiguous buffer of n entries (ideally pinned)."""
    if hasattr(t, "data_ptr"):
        import torch

        if t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous() or t.numel() != n:
            raise ValueError("host buffers must be contiguous float64 CPU tensors of the operator size")
        return t.data_ptr()
    a = np.asarray(t)
    if a.dtype != np.float64 or not a.flags.c_contiguous or a.size != n or a is not t:
        raise ValueError("host buffers must be contiguous float64 arrays of the operator size")
    return a.ctypes.data


def apply_host_multi(operators, u_hosts, y_hosts, stream: int = 0):
    """y_hosts[i] = operators[i] u_hosts[i] for several operators as one pipelined call
    (``tmf_apply_host_multi``): uploads back to back in the given order, each plan's
    kernels as soon as its own upload has landed, downloads overlapping the next plans'
    uploads.  Enqueued on ``stream`` and returns; the host buffers (pinned tensors or
    arrays) must outlive the stream work.  Replaces a caller's loop of
    ``operator.apply(u)`` calls (reference operator.py:320-331)."""
    ops, us, ys = list(operators), list(u_hosts), list(y_hosts)
    if not (len(ops) == len(us) == len(ys)):
        raise ValueError("operators, u_hosts and y_hosts differ in length")
    n = len(ops)
    arr = C.c_void_p * max(n, 1)
    plans = arr(*[A._plan.value for A in ops])
    up = arr(*[_host_buffer(u, A.n_global_dofs) for A, u in zip(ops, us)])
    yp = arr(*[_host_buffer(y, A.n_global_dofs) for A, y in zip(ops, ys)])
    _lib.check(_lib.lib().tmf_apply_host_multi(plans, up, yp, n, C.c_void_p(stream)))
    for A in ops:
        A._count()
