"""ctypes binding of libtetmf_b200.so (the C-ABI declared in include/tetmf_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is present, every operator call raises RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TMF_LIB=debug loads the bounds-checking build (libtetmf_b200_debug.so, _build.py --debug);
# TMF_LIB=<name> any other in-tree build libtetmf_b200_<name>.so (developer A/B measurements)
_VARIANT = os.environ.get("TMF_LIB", "")
LIB_PATH = os.path.join(_HERE, f"libtetmf_b200_{_VARIANT}.so" if _VARIANT else "libtetmf_b200.so")

TMF_OK, TMF_EINVAL, TMF_ECUDA = 0, 1, 2
TMF_CG_LAPLACE, TMF_DG_SIPG, TMF_DG_HELMHOLTZ = 0, 1, 2
STAGE_ZERO, STAGE_CELLS, STAGE_FACES, STAGE_FIXUP = 1, 2, 4, 8

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_bp = C.POINTER(C.c_uint8)


class PlanDesc(C.Structure):
    _fields_ = [
        ("operator_kind", C.c_int32), ("degree", C.c_int32), ("n_dofs_per_cell", C.c_int32),
        ("n_components", C.c_int32), ("n_vertices", C.c_int64), ("n_cells", C.c_int64),
        ("n_scalar_dofs", C.c_int64), ("vertices", _dp), ("cells", _ip), ("cell_dofs", _ip),
        ("dirichlet_mask", _bp), ("n_q", C.c_int32), ("n_qf", C.c_int32),
        ("cell_weights", _dp), ("value_matrix", _dp), ("grad_matrix", _dp),
        ("face_weights", _dp), ("face_values", _dp), ("face_grads", _dp),
        ("n_interior_faces", C.c_int64), ("interior_faces", _ip), ("tau_interior", _dp),
        ("n_boundary_faces", C.c_int64), ("boundary_faces", _ip), ("tau_boundary", _dp),
        ("boundary_dirichlet", _bp), ("kappa", _dp), ("mass_scale", C.c_double),
        ("diffusivity", C.c_double), ("device", C.c_int32), ("flags", C.c_int32),
    ]


class TransferDesc(C.Structure):
    _fields_ = [
        ("n_cells", C.c_int64), ("n_fine_dpc", C.c_int32), ("n_coarse_dpc", C.c_int32),
        ("n_fine_dofs", C.c_int64), ("n_coarse_dofs", C.c_int64), ("fine_cell_dofs", _ip),
        ("coarse_cell_dofs", _ip), ("fine_dirichlet", _bp), ("coarse_dirichlet", _bp),
        ("interp", _dp), ("device", C.c_int32),
    ]


class PointTransferDesc(C.Structure):
    _fields_ = [
        ("n_fine_dofs", C.c_int64), ("n_coarse_dofs", C.c_int64), ("entries_per_row", C.c_int32),
        ("coarse_index", _ip), ("weights", _dp), ("fine_dirichlet", _bp), ("coarse_dirichlet", _bp),
        ("device", C.c_int32),
    ]


class PlanInfo(C.Structure):
    _fields_ = [
        ("n_global_dofs", C.c_int64), ("flops_alg", C.c_double), ("bytes_alg", C.c_double),
        ("flops_issued", C.c_double), ("kernels_per_apply", C.c_int32),
        ("n_face_batches", C.c_int32), ("device_bytes", C.c_int64), ("block_cells", C.c_int32),
        ("block_ratio", C.c_double), ("cell_engine", C.c_int32), ("flops_engine", C.c_double),
        ("face_engine", C.c_int32), ("cell_order", C.c_int32),
    ]


_lib = None


def lib():
    """Load the library (once); raises RuntimeError if it has not been built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with "
                               "`python -m paper_2509_10226_b200._build` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        L.tmf_plan_create.argtypes = [C.POINTER(PlanDesc), C.POINTER(C.c_void_p)]
        L.tmf_plan_destroy.argtypes = [C.c_void_p]
        L.tmf_plan_get_info.argtypes = [C.c_void_p, C.POINTER(PlanInfo)]
        L.tmf_apply.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.tmf_apply_host.argtypes = [C.c_void_p, _dp, _dp]
        L.tmf_apply_stages.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int64, C.c_int64,
                                       C.c_void_p]
        L.tmf_apply_host_async.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.tmf_apply_host_multi.argtypes = [C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                           C.c_int, C.c_void_p]
        L.tmf_apply_timed.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, _dp, C.c_int]
        L.tmf_diagonal.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.tmf_pcg.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, _dp, C.c_void_p]
        L.tmf_hierarchical_reorder.argtypes = [C.c_int64, C.c_int64, _ip, C.c_int32, C.POINTER(C.c_int64)]
        _lp = C.POINTER(C.c_int64)
        L.tmf_build_faces.argtypes = [C.c_int64, _ip, C.c_int64, _ip, _lp, _ip, _lp]
        L.tmf_build_cg_dofs.argtypes = [C.c_int64, _ip, C.c_int64, C.c_int32, _ip, _lp]
        _v = C.c_void_p
        L.tmf_vec_dot.argtypes = [_v, _v, C.c_int64, _v, _v]
        L.tmf_pcg_init.argtypes = [_v, _v, _v, _v, _v, _v, C.c_int64, _v, _v, _v]
        L.tmf_pcg_update.argtypes = [_v, _v, _v, _v, _v, _v, C.c_int64, _v, _v, _v, _v, _v]
        L.tmf_pcg_direction.argtypes = [_v, _v, C.c_int64, _v, _v, _v]
        _u64p = C.POINTER(C.c_uint64)
        L.tmf_plan_set_peers.argtypes = [C.c_void_p, C.c_int32, _u64p, _u64p, C.c_int32, C.c_int64, C.c_int64,
                                         _ip, _ip, C.c_int64]
        L.tmf_alloc.argtypes = [C.c_int64, C.c_int32, C.POINTER(C.c_void_p)]
        L.tmf_free.argtypes = [C.c_void_p]
        L.tmf_ipc_get_handle.argtypes = [C.c_void_p, C.POINTER(C.c_uint8)]
        L.tmf_ipc_open_handle.argtypes = [C.POINTER(C.c_uint8), C.c_int32, C.POINTER(C.c_void_p)]
        L.tmf_ipc_close_handle.argtypes = [C.c_void_p]
        L.tmf_color_cells.argtypes = [C.c_int64, C.c_int64, _ip, _ip, _ip]
        L.tmf_transfer_create.argtypes = [C.POINTER(TransferDesc), C.POINTER(C.c_void_p)]
        L.tmf_transfer_destroy.argtypes = [_v]
        L.tmf_transfer_create_points.argtypes = [C.POINTER(PointTransferDesc), C.POINTER(C.c_void_p)]
        L.tmf_prolongate.argtypes = [_v, _v, _v, C.c_int, _v]
        L.tmf_restrict.argtypes = [_v, _v, _v, _v]
        L.tmf_chebyshev_step.argtypes = [C.c_int64, _v, _v, _v, _v, _v, C.c_double, C.c_double, _v]
        L.tmf_vec_axpby.argtypes = [C.c_int64, C.c_double, _v, C.c_double, _v, _v, _v]
        L.tmf_apply_f32.argtypes = [_v, _v, _v, _v]
        L.tmf_prolongate_f32.argtypes = [_v, _v, _v, C.c_int, _v]
        L.tmf_restrict_f32.argtypes = [_v, _v, _v, _v]
        L.tmf_chebyshev_step_f32.argtypes = [C.c_int64, _v, _v, _v, _v, _v, C.c_float, C.c_float, _v]
        L.tmf_vec_axpby_f32.argtypes = [C.c_int64, C.c_float, _v, C.c_float, _v, _v, _v]
        L.tmf_last_error.restype = C.c_char_p
        L.tmf_version.restype = C.c_char_p
        L.tmf_debug_poke_dof.argtypes = [C.c_void_p, C.c_int64, C.c_int32]
        L.tmf_debug_chunk_walk.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_int, C.c_int, _v, C.c_int64, _v]
        L.tmf_debug_chunk_walk.restype = C.c_int
        for name in ("tmf_plan_create", "tmf_plan_destroy", "tmf_plan_get_info", "tmf_apply",
                     "tmf_apply_host", "tmf_apply_host_async", "tmf_apply_host_multi", "tmf_apply_stages", "tmf_apply_timed", "tmf_diagonal", "tmf_pcg",
                     "tmf_hierarchical_reorder", "tmf_build_faces", "tmf_build_cg_dofs",
                     "tmf_vec_dot", "tmf_pcg_init", "tmf_pcg_update", "tmf_pcg_direction",
                     "tmf_plan_set_peers", "tmf_alloc", "tmf_free", "tmf_ipc_get_handle", "tmf_ipc_open_handle",
                     "tmf_ipc_close_handle", "tmf_color_cells", "tmf_transfer_create", "tmf_transfer_create_points",
                     "tmf_transfer_destroy", "tmf_prolongate",
                     "tmf_restrict", "tmf_chebyshev_step", "tmf_vec_axpby", "tmf_apply_f32", "tmf_prolongate_f32",
                     "tmf_restrict_f32", "tmf_chebyshev_step_f32", "tmf_vec_axpby_f32"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


EXPORTED = ("tmf_plan_create", "tmf_plan_destroy", "tmf_plan_get_info", "tmf_apply",
            "tmf_apply_host", "tmf_apply_host_async", "tmf_apply_host_multi", "tmf_apply_stages", "tmf_apply_timed", "tmf_diagonal", "tmf_pcg", "tmf_hierarchical_reorder",
            "tmf_build_faces", "tmf_build_cg_dofs", "tmf_vec_dot", "tmf_pcg_init", "tmf_pcg_update",
            "tmf_pcg_direction", "tmf_plan_set_peers", "tmf_alloc", "tmf_free", "tmf_ipc_get_handle",
            "tmf_ipc_open_handle", "tmf_ipc_close_handle", "tmf_color_cells", "tmf_transfer_create",
            "tmf_transfer_create_points", "tmf_transfer_destroy",
            "tmf_prolongate", "tmf_restrict", "tmf_chebyshev_step", "tmf_vec_axpby", "tmf_apply_f32",
            "tmf_prolongate_f32", "tmf_restrict_f32", "tmf_chebyshev_step_f32", "tmf_vec_axpby_f32", "tmf_last_error",
            "tmf_version", "tmf_debug_poke_dof", "tmf_debug_chunk_walk")


def check(rc: int) -> None:
    if rc == TMF_OK:
        return
    msg = lib().tmf_last_error().decode()
    if rc == TMF_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


def ptr(a: np.ndarray | None, ctype):
    if a is None:
        return C.cast(None, C.POINTER(ctype))
    return a.ctypes.data_as(C.POINTER(ctype))
