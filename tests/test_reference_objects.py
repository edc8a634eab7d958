"""The operator shim takes the REAL reference objects (tetmf.mesh.TetMesh, dofmap.DoFMap,
geometry.GeometryData, basis.BasisTable), not only look-alikes: built here by importing the
reference (this container only; skipped where /root/reference is absent, e.g. the GPU box).

Without a GPU the constructor must get as far as the C-ABI and fail LOUDLY there ("no CUDA
device ... no CPU path"): every attribute the shim reads from the reference objects exists and
converts, and nothing falls back to a CPU computation."""

import os
import sys

import numpy as np
import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not present")


def _ref_objects(p, space, nc=1, dids=(), mode="affine"):
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
    import make_golden as MG

    tm = MG.ref_mesh(3, 0)
    cr, fr = MG.rules(p, "ref")
    basis = MG.ref_basis(p, cr, fr)
    dm = MG.ref_dofmap(tm, p, space, nc, dids)
    geo = MG.rgeo.build_geometry(tm, cr, mode, face_rule=fr) if space == "dg" else MG.rgeo.build_geometry(tm, cr, mode)
    return MG, tm, dm, geo, basis


def _has_gpu():
    import torch

    return torch.cuda.is_available()


@pytest.mark.parametrize("mode", ["affine", "per_point"])
def test_real_reference_objects_reach_the_c_abi(mode):
    from paper_2509_10226_b200 import operator as op

    MG, tm, dm, geo, basis = _ref_objects(2, "cg", dids=(0,), mode=mode)
    assert type(tm).__module__ == "tetmf.mesh" and type(geo).__module__ == "tetmf.geometry"
    if _has_gpu():
        u = np.random.default_rng(0).uniform(-1, 1, dm.n_global_dofs)
        ref = MG.rop.CgPoissonOperator(tm, dm, geo, basis).apply(u)
        y = op.CgPoissonOperator(tm, dm, geo, basis).apply(u)
        assert np.linalg.norm(y - ref) <= 1e-12 * np.linalg.norm(ref)
    else:
        with pytest.raises(RuntimeError, match="no CUDA device"):
            op.CgPoissonOperator(tm, dm, geo, basis)


def test_real_reference_dg_objects_reach_the_c_abi():
    from paper_2509_10226_b200 import operator as op

    MG, tm, dm, geo, basis = _ref_objects(2, "dg")
    sipg = MG.rop.compute_sipg_tau(tm, geo, 2)    # the reference's own SipgConfig (operator.py:117)
    assert type(sipg).__module__ == "tetmf.operator"
    if _has_gpu():
        op.DgSipgOperator(tm, dm, geo, basis, sipg, dirichlet_ids=(0,))
    else:
        with pytest.raises(RuntimeError, match="no CUDA device"):
            op.DgSipgOperator(tm, dm, geo, basis, sipg, dirichlet_ids=(0,))


def test_real_reference_config_object_is_accepted():
    """A reference OperatorConfig (its own dataclass) passes the shim's checks: f64 + reference batching."""
    from paper_2509_10226_b200 import operator as op

    MG, tm, dm, geo, basis = _ref_objects(1, "cg")
    rcfg = MG.rop.OperatorConfig()
    cfg = op.OperatorConfig(**{k: getattr(rcfg, k) for k in ("lane_width", "cells_per_lane", "batching", "precision",
                                                             "kernel_stage") if hasattr(rcfg, k) and
                               k in op.OperatorConfig.__dataclass_fields__})
    if not _has_gpu():
        with pytest.raises(RuntimeError, match="no CUDA device"):
            op.CgPoissonOperator(tm, dm, geo, basis, cfg)


def test_real_curved_reference_mesh_is_rejected():
    """geometry.py:141-142 and the shim: a curved reference mesh (geometry_nodes set) has no B200
    path and must raise ValueError before any plan is built -- never be linearised silently."""
    from paper_2509_10226_b200 import operator as op

    MG, tm, dm, geo, basis = _ref_objects(2, "cg")
    curved = MG.rmesh.generate_cube_mesh(2, deformation="smooth")   # mesh.py:155
    assert curved.is_curved
    cr, fr = MG.rules(2, "ref")
    cgeo = MG.rgeo.build_geometry(curved, cr, "per_point")
    cdm = MG.rdof.build_dof_map(curved, 2, "cg", 1, ())
    with pytest.raises(ValueError, match="curved"):
        op.CgPoissonOperator(curved, cdm, cgeo, basis)
    with pytest.raises(ValueError, match="curved"):
        op.CgPoissonOperator(curved, cdm, geo, basis)   # affine container on a curved mesh
