"""GPU parity: the sm_100a kernels (through the C-ABI) against the reference's
golden outputs and the CPU oracle.  Tolerance: relative L2 <= 1e-12 (north_star)."""

import numpy as np
import pytest

from conftest import golden_names, load_golden, rel_l2
from helpers import operator_from_fixture

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.mark.parametrize("name", golden_names())
def test_gpu_matches_reference_golden(name):
    g = load_golden(name)
    A = operator_from_fixture(g)
    y = A.apply(g["u"])
    err = rel_l2(y, g["y"])
    assert err <= TOL, f"{name}: rel L2 {err:.3e}"
    assert A.n_applies == 1


@pytest.mark.parametrize("name", ["cg_p2_n8_gm", "dg_p3_n3_gm_dir", "helmk_p2_n3_gm_dir"])
def test_gpu_repeatable(name):
    g = load_golden(name)
    A = operator_from_fixture(g)
    y1 = A.apply(g["u"])
    y2 = A.apply(g["u"])
    assert rel_l2(y1, y2) <= 1e-15


ENGINE_CODE = {"dmma": 1, "tensor": 3, "modal": 4}


@pytest.mark.parametrize("engine", ["dmma", "tensor", "modal"])
@pytest.mark.parametrize("name", golden_names())
def test_gpu_cell_engines_match_golden(name, engine):
    """Every cell engine against every golden, P4 included: the quadrature-point loop (the
    reference's algorithm), the reference tensor (point sum precontracted per plan) and
    the modal tables (the point loop on M = dim P_{p-1} exact unit-weight modes; for
    Helmholtz at P2-P4 the mass term is a separate GEMM, P1 Helmholtz plans refuse it)."""
    g = load_golden(name)
    if engine == "modal" and str(g["kind"]).startswith("helm") and "_p1_" in name:
        with pytest.raises(ValueError, match="modal"):
            operator_from_fixture(g, cell_engine=engine)
        return
    A = operator_from_fixture(g, cell_engine=engine)
    assert A.info["cell_engine"] == ENGINE_CODE[engine]
    err = rel_l2(A.apply(g["u"]), g["y"])
    assert err <= TOL, f"{name}/{engine}: rel L2 {err:.3e}"


def test_gpu_default_engines():
    """auto: block assembly (5) for scalar CG Laplace at P1, modal tables for the other
    cell terms at P2-P4 (Helmholtz: plus the mass GEMM), the reference tensor for DG at P1;
    modal faces at P2-P4, the point loop at P1."""
    for name, cell, face in [("cg_p1_n3_gm_dir2", 5, 0), ("cg_p2_n8_gm", 4, 0), ("cg_p3_n4_ref_dir", 4, 0),
                             ("cg_p4_n3_gm", 4, 0), ("cg3_p2_n3_ref_dir", 4, 0),
                             ("dg_p1_n3_gm_dir", 3, 1), ("dg_p3_n3_gm_dir", 4, 3), ("helmk_p2_n3_gm_dir", 4, 3),
                             ("helm3_p2_n2_gm_none", 4, 3), ("helmk_p1_n3_ref_dir", 3, 1)]:
        A = operator_from_fixture(load_golden(name))
        assert A.info["cell_engine"] == cell, name
        assert A.info["face_engine"] == face, name


FACE_CODE = {"quadrature": 1, "modal_flat": 2, "modal": 3}


@pytest.mark.parametrize("engine", ["quadrature", "modal_flat", "modal"])
@pytest.mark.parametrize("name", [n for n in golden_names() if n.startswith(("dg", "helm"))])
def test_gpu_face_engines_match_golden(name, engine):
    """Faces: the n_qf-point loop (face_kernel.cuh) and the point loop on NF exact face
    modes (P4 interior faces: the asynchronous gather-ring kernel), against every DG /
    Helmholtz golden."""
    g = load_golden(name)
    A = operator_from_fixture(g, face_engine=engine)
    if A.info["n_face_batches"]:
        assert A.info["face_engine"] == FACE_CODE[engine]
    err = rel_l2(A.apply(g["u"]), g["y"])
    assert err <= TOL, f"{name}/{engine}: rel L2 {err:.3e}"


@pytest.mark.parametrize("name", [n for n in golden_names("cg") if ("_p1_" in n or "_p2_" in n)
                                  and not n.startswith("cg3")])
def test_gpu_block_assembly_matches_golden(name):
    """CG block assembly (cell_block_kernel.cuh) on and off against every scalar CG golden
    P1-P2 (Dirichlet and pure Neumann, reference and GM rules)."""
    g = load_golden(name)
    on = operator_from_fixture(g, cell_blocks="on")
    off = operator_from_fixture(g, cell_blocks="off")
    assert on.info["cell_engine"] == 5 and on.info["block_cells"] > 0
    assert off.info["cell_engine"] != 5 and off.info["block_cells"] == 0
    for A in (on, off):
        err = rel_l2(A.apply(g["u"]), g["y"])
        assert err <= TOL, f"{name}: rel L2 {err:.3e}"


@pytest.mark.parametrize("order", ["input", "morton"])
@pytest.mark.parametrize("name", [n for n in golden_names("cg")])
def test_gpu_cell_traversal_order_matches_golden(name, order):
    """CG plans traverse cells in the caller's order or in the Morton order of the centroids
    (OperatorConfig.cell_order); u / y keep the caller's numbering, results are the same."""
    g = load_golden(name)
    A = operator_from_fixture(g, cell_order=order)
    assert A.info["cell_order"] == {"input": 1, "morton": 2}[order]
    err = rel_l2(A.apply(g["u"]), g["y"])
    assert err <= TOL, f"{name}/{order}: rel L2 {err:.3e}"


def test_gpu_cell_order_auto_and_ranges():
    """auto picks Morton for a randomly permuted mesh and keeps a locality-ordered one; a
    Morton plan refuses partial cell ranges (the multi-GPU stages need the caller's order)."""
    import torch

    from paper_2509_10226_b200 import _lib, basis as B, dofmap as D, mesh as M, operator as op, quadrature as Q
    from paper_2509_10226_b200.geometry import GeometryData
    from paper_2509_10226_b200.reorder import reorder_mesh

    p = 2
    cr, fr = Q.make_cell_quadrature(p), Q.make_face_quadrature(p)
    bas = B.tabulate_basis(p, cr, fr)
    geo = GeometryData("affine", cr, fr, None, None, None, None)
    m = M.kuhn_cube_mesh(10, seed=0)
    A = op.CgPoissonOperator(m, D.build_dof_map(m, p, "cg"), geo, bas)
    assert A.info["cell_order"] == 2
    mr = reorder_mesh(m)
    assert op.CgPoissonOperator(mr, D.build_dof_map(mr, p, "cg"), geo, bas).info["cell_order"] == 1
    u = torch.rand(A.n_global_dofs, dtype=torch.float64, device="cuda")
    y = torch.empty_like(u)
    with pytest.raises(ValueError, match="cell ranges"):
        A.apply_stages(u.data_ptr(), y.data_ptr(), _lib.STAGE_CELLS, 0, 10)
    A.apply_stages(u.data_ptr(), y.data_ptr(), _lib.STAGE_ZERO | _lib.STAGE_CELLS | _lib.STAGE_FIXUP)
    torch.cuda.synchronize()
    assert rel_l2(y.cpu().numpy(), A.apply(u).cpu().numpy()) <= 1e-14


@pytest.mark.parametrize("run", [1, 2, 5])
@pytest.mark.parametrize("name", ["dg_p1_n3_gm_dir", "dg_p3_n3_gm_dir", "dg_p4_n2_gm_dir", "helm3_p2_n2_gm_none"])
def test_gpu_face_chunk_runs_match_golden(name, run, monkeypatch):
    """The interior-face CTA walk in runs of `run` chunks dealt round-robin (face_kernel.cuh
    ChunkWalk; large P3 meshes use run 2 by themselves, here forced on the small goldens so
    the blocked, ring and multi-component kernels all take the strided walk)."""
    monkeypatch.setenv("TMF_FACE_RUN", str(run))
    g = load_golden(name)
    A = operator_from_fixture(g)
    err = rel_l2(A.apply(g["u"]), g["y"])
    assert err <= TOL, f"{name}/run {run}: rel L2 {err:.3e}"
