"""The bounds-checking build (libtetmf_b200_debug.so, common.cuh TMF_DEBUG_CHECKS) -- the
memcheck substitute on this GPU pool -- loads, passes a golden, and reports a corrupted
cell-DoF index instead of silently reading / writing out of range.  Run in a subprocess so
the release library of this process is untouched."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, {root!r}); sys.path.insert(0, {root!r} + "/tests")
from conftest import load_golden, rel_l2
from helpers import operator_from_fixture
from paper_2509_10226_b200 import _lib
assert b"DEBUG-CHECKS" in _lib.lib().tmf_version()
g = load_golden("cg_p2_n8_gm_dir")
for blocks in ("off", "on"):
    A = operator_from_fixture(g, cell_blocks=blocks)
    assert rel_l2(A.apply(g["u"]), g["y"]) <= 1e-12
# one DoF index pushed one past the vector: gathered / scattered inside the (padded)
# allocation, but outside the plan -- the apply must fail with the check's message
A = operator_from_fixture(g, cell_blocks="off")
n = A.n_global_dofs
u = torch.zeros(n + 4096, dtype=torch.float64, device="cuda")
y = torch.zeros_like(u)
_lib.check(_lib.lib().tmf_debug_poke_dof(A._plan, 7, n))
try:
    A.apply_into(u.data_ptr(), y.data_ptr(), torch.cuda.current_stream().cuda_stream)
except Exception as e:
    assert "debug bounds check failed" in str(e), e
    print("CAUGHT", e)
else:
    raise AssertionError("corrupted index not reported")
"""


def test_debug_build_checks_fire():
    lib = os.path.join(ROOT, "paper_2509_10226_b200", "libtetmf_b200_debug.so")
    if not os.path.exists(lib):
        pytest.skip("debug library not built")
    env = dict(os.environ, TMF_LIB="debug")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT)], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "CAUGHT" in r.stdout


def test_release_build_refuses_debug_hook():
    from helpers import operator_from_fixture

    from conftest import load_golden
    from paper_2509_10226_b200 import _lib

    if os.environ.get("TMF_LIB"):
        pytest.skip("not the release library (TMF_LIB is set)")
    A = operator_from_fixture(load_golden("cg_p2_n8_gm_dir"))
    with pytest.raises(Exception, match="TMF_DEBUG_CHECKS"):
        _lib.check(_lib.lib().tmf_debug_poke_dof(A._plan, 0, 0))
