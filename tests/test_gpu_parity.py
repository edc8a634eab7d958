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


@pytest.mark.parametrize("engine", ["dmma", "dfma"])
@pytest.mark.parametrize("name", [n for n in golden_names() if "_p4_" not in n])
def test_gpu_both_cell_engines_match_golden(name, engine):
    """The tensor-core (DMMA) and vector-pipe (DFMA) cell kernels are both exact
    restatements; the default picks one per degree (cell_dfma_kernel.cuh)."""
    g = load_golden(name)
    A = operator_from_fixture(g, cell_engine=engine)
    err = rel_l2(A.apply(g["u"]), g["y"])
    assert err <= TOL, f"{name}/{engine}: rel L2 {err:.3e}"


ENGINE_CODE = {"dmma": 1, "tensor": 3, "modal": 4}


@pytest.mark.parametrize("engine", ["dmma", "tensor", "modal"])
@pytest.mark.parametrize("name", golden_names())
def test_gpu_cell_engines_match_golden(name, engine):
    """Every cell engine against every golden, P4 included: the quadrature-point loop (the
    reference's algorithm), the reference tensor (point sum precontracted per plan) and
    the modal tables (the point loop on M = dim P_{p-1} exact unit-weight modes; Laplace
    cell terms only -- Helmholtz plans refuse it)."""
    g = load_golden(name)
    if engine == "modal" and str(g["kind"]).startswith("helm"):
        with pytest.raises(ValueError, match="modal"):
            operator_from_fixture(g, cell_engine=engine)
        return
    A = operator_from_fixture(g, cell_engine=engine)
    assert A.info["cell_engine"] == ENGINE_CODE[engine]
    err = rel_l2(A.apply(g["u"]), g["y"])
    assert err <= TOL, f"{name}/{engine}: rel L2 {err:.3e}"


def test_gpu_default_engines():
    """auto: modal tables for Laplace cell terms at P2-P4, the reference tensor at P1 and
    for Helmholtz; modal faces at P2-P4, the point loop at P1."""
    for name, cell, face in [("cg_p1_n3_gm_dir2", 3, 0), ("cg_p2_n8_gm", 4, 0), ("cg_p4_n3_gm", 4, 0),
                             ("dg_p1_n3_gm_dir", 3, 1), ("dg_p3_n3_gm_dir", 4, 3), ("helmk_p2_n3_gm_dir", 3, 3)]:
        A = operator_from_fixture(load_golden(name))
        assert A.info["cell_engine"] == cell, name
        assert A.info["face_engine"] == face, name


FACE_CODE = {"quadrature": 1, "tensor": 2, "modal": 3}


@pytest.mark.parametrize("engine", ["quadrature", "tensor", "modal"])
@pytest.mark.parametrize("name", [n for n in golden_names() if n.startswith(("dg", "helm"))])
def test_gpu_face_engines_match_golden(name, engine):
    """Faces: the n_qf-point loop (face_kernel.cuh), the reference-tensor form for interior
    faces (face_tensor_kernel.cuh, per-signature precontracted tables) and the point loop on
    NF exact face modes, against every DG / Helmholtz golden."""
    g = load_golden(name)
    A = operator_from_fixture(g, face_engine=engine)
    if A.info["n_face_batches"]:
        assert A.info["face_engine"] == FACE_CODE[engine]
    err = rel_l2(A.apply(g["u"]), g["y"])
    assert err <= TOL, f"{name}/{engine}: rel L2 {err:.3e}"


@pytest.mark.parametrize("variant", [1, 2, 4, 5, 9, 10, 13, 14, 15])
@pytest.mark.parametrize("name", ["dg_p2_n3_gm_dir", "dg_p3_n3_gm_dir", "dg_p4_n2_gm_dir", "helmk_p2_n3_gm_dir",
                                  "helm3_p2_n2_gm_none"])
def test_gpu_face_modal_variants_match_golden(name, variant):
    """Modal face tables under the face-kernel variants, including the asynchronous
    gather ring (13-15, face_async_kernel)."""
    g = load_golden(name)
    A = operator_from_fixture(g, face_engine="modal", face_variant=variant)
    err = rel_l2(A.apply(g["u"]), g["y"])
    assert err <= TOL, f"{name}/v{variant}: rel L2 {err:.3e}"


@pytest.mark.parametrize("variant", [0, 13, 14, 15])
@pytest.mark.parametrize("name", ["dg_p1_n3_gm_dir", "dg_p3_n3_gm_dir", "dg_p4_n2_gm_dir", "helm3_p1_n2_ref_dir"])
def test_gpu_face_quadrature_async_match_golden(name, variant):
    """The asynchronous gather ring on the n_qf-point face tables."""
    g = load_golden(name)
    A = operator_from_fixture(g, face_engine="quadrature", face_variant=variant)
    err = rel_l2(A.apply(g["u"]), g["y"])
    assert err <= TOL, f"{name}/v{variant}: rel L2 {err:.3e}"


@pytest.mark.parametrize("variant", range(1, 7))
@pytest.mark.parametrize("name", ["dg_p2_n3_gm_dir", "dg_p3_n3_gm_dir", "helmk_p2_n3_gm_dir", "helm3_p2_n2_gm_none"])
def test_gpu_face_tensor_variants_match_golden(name, variant):
    g = load_golden(name)
    A = operator_from_fixture(g, face_engine="tensor", face_variant=variant)
    err = rel_l2(A.apply(g["u"]), g["y"])
    assert err <= TOL, f"{name}/v{variant}: rel L2 {err:.3e}"


@pytest.mark.parametrize("variant", [2, 5, 6, 7, 8, 10, 11, 14, 15])
@pytest.mark.parametrize("name", ["cg_p2_n8_gm", "cg3_p2_n3_ref_dir", "cg_p3_n3_gm_dir2", "cg_p4_n3_gm_dir", "dg_p3_n3_gm_dir"])
def test_gpu_modal_variants_match_golden(name, variant):
    g = load_golden(name)
    A = operator_from_fixture(g, cell_engine="modal", kernel_variant=variant)
    err = rel_l2(A.apply(g["u"]), g["y"])
    assert err <= TOL, f"{name}/v{variant}: rel L2 {err:.3e}"


@pytest.mark.parametrize("variant", range(1, 8))
@pytest.mark.parametrize("name", ["cg_p1_n3_gm_dir2", "cg_p2_n8_gm", "cg3_p2_n3_ref_dir", "cg_p4_n3_gm_dir",
                                  "helmk_p2_n3_gm_dir", "dg_p3_n3_gm_dir"])
def test_gpu_tensor_variants_match_golden(name, variant):
    g = load_golden(name)
    A = operator_from_fixture(g, cell_engine="tensor", kernel_variant=variant)
    err = rel_l2(A.apply(g["u"]), g["y"])
    assert err <= TOL, f"{name}/v{variant}: rel L2 {err:.3e}"


@pytest.mark.parametrize("variant", range(1, 9))
@pytest.mark.parametrize("name", ["cg_p1_n3_gm_dir2", "cg_p2_n8_gm", "cg3_p2_n3_ref_dir", "helmk_p2_n3_gm_dir", "dg_p3_n3_gm_dir"])
def test_gpu_dfma_variants_match_golden(name, variant):
    g = load_golden(name)
    A = operator_from_fixture(g, cell_engine="dfma", kernel_variant=variant)
    err = rel_l2(A.apply(g["u"]), g["y"])
    assert err <= TOL, f"{name}/v{variant}: rel L2 {err:.3e}"


@pytest.mark.parametrize("variant", [0, 2, 3])
@pytest.mark.parametrize("name", [n for n in golden_names() if n.startswith("cg") and "_p4_" not in n])
def test_gpu_patch_local_assembly_matches_golden(name, variant):
    """CG patch-local assembly (shared-memory gather/scatter per cell patch) forced on."""
    g = load_golden(name)
    A = operator_from_fixture(g, cell_engine="dfma", cell_patches="on", kernel_variant=variant)
    assert A.info["patch_cells"] > 0
    err = rel_l2(A.apply(g["u"]), g["y"])
    assert err <= TOL, f"{name}: rel L2 {err:.3e}"


@pytest.mark.parametrize("face_variant", [11, 12, 13, 14])
@pytest.mark.parametrize("name", ["dg_p1_n3_gm_dir", "dg_p2_n3_gm_dir", "dg_p3_n3_gm_dir", "helmk_p2_n3_gm_dir",
                                  "helm3_p2_n2_gm_none", "dg_p4_n2_gm_dir"])
def test_gpu_face_variants_match_golden(name, face_variant):
    """Face-kernel scheduling variants (round-robin chunks + table prefetch)."""
    g = load_golden(name)
    A = operator_from_fixture(g, face_variant=face_variant, face_chunk=8)
    err = rel_l2(A.apply(g["u"]), g["y"])
    assert err <= TOL, f"{name}/f{face_variant}: rel L2 {err:.3e}"
