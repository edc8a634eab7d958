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


@pytest.mark.parametrize("engine", ["dmma", "tensor"])
@pytest.mark.parametrize("name", golden_names())
def test_gpu_quadrature_and_tensor_engines_match_golden(name, engine):
    """The quadrature-point DMMA engine (the reference's point loop) and the reference-
    tensor engine (the point sum precontracted per plan) against every golden, P4 included."""
    g = load_golden(name)
    A = operator_from_fixture(g, cell_engine=engine)
    assert A.info["cell_engine"] == (3 if engine == "tensor" else 1)
    err = rel_l2(A.apply(g["u"]), g["y"])
    assert err <= TOL, f"{name}/{engine}: rel L2 {err:.3e}"


@pytest.mark.parametrize("engine", ["quadrature", "tensor"])
@pytest.mark.parametrize("name", [n for n in golden_names() if n.startswith(("dg", "helm"))])
def test_gpu_face_engines_match_golden(name, engine):
    """Interior faces: the point loop (face_kernel.cuh) and the reference-tensor form
    (face_tensor_kernel.cuh, per-signature precontracted tables) against every DG golden."""
    g = load_golden(name)
    A = operator_from_fixture(g, face_engine=engine)
    if A.info["n_face_batches"]:
        assert A.info["face_engine"] == (2 if engine == "tensor" else 1)
    err = rel_l2(A.apply(g["u"]), g["y"])
    assert err <= TOL, f"{name}/{engine}: rel L2 {err:.3e}"


@pytest.mark.parametrize("variant", range(1, 7))
@pytest.mark.parametrize("name", ["dg_p2_n3_gm_dir", "dg_p3_n3_gm_dir", "helmk_p2_n3_gm_dir", "helm3_p2_n2_gm_none"])
def test_gpu_face_tensor_variants_match_golden(name, variant):
    g = load_golden(name)
    A = operator_from_fixture(g, face_engine="tensor", face_variant=variant)
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
