"""The logical counters (row a23) against the reference's own counters.

tests/golden/counters_ref.json holds ``counters.as_dict()`` of REAL reference
operators after one apply (tests/golden/make_counters.py), for CG / DG / the
3-component Helmholtz under several OperatorConfigs (stages, lane widths, f32,
components batching).  ``reference_apply_counts`` must reproduce every key.
When /root/reference is present (the build container) the reference is also run
live on one case.
"""

import json
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN

from paper_2509_10226_b200 import dofmap as D, mesh as M
from paper_2509_10226_b200.counters import FlopCounters, reference_apply_counts
from paper_2509_10226_b200.operator import OperatorConfig

# reference tables (quadrature.py:30-46): n_q, n_qf for p = 1..3; GM rules s = p
_NQ = {"ref": {1: (4, 3), 2: (14, 6), 3: (35, 12)}, "gm": {1: (5, 4), 2: (15, 10), 3: (35, 20), 4: (70, 35)}}

with open(os.path.join(GOLDEN, "counters_ref.json")) as f:
    _CASES = json.load(f)


def _counts(case, cfg):
    m = M.kuhn_cube_mesh(case["n"], seed=0)
    p = case["p"]
    nq, nqf = _NQ[case["rule"]][p]
    kind = case["kind"]
    if kind == "cg":
        dm = D.build_dof_map(m, p, "cg", case.get("nc", 1), tuple(case["dids"]), method="numpy")
        return reference_apply_counts(cfg, dm, nq)
    dm = D.build_dof_map(m, p, "dg", 3 if kind == "helm3" else 1)
    ms, nu = (case["ms"], case["nu"]) if kind == "helm3" else (0.0, 1.0)
    return reference_apply_counts(cfg, dm, nq, nqf, interior_faces=m.interior_faces,
                                  boundary_faces=m.boundary_faces, dirichlet_ids=case["dids"],
                                  mass_scale=ms, diffusivity=nu, faces=True)


@pytest.mark.parametrize("i", range(len(_CASES)), ids=[f"{c['case']['kind']}-p{c['case']['p']}-{c['config']}"
                                                        for c in _CASES])
def test_counters_match_reference(i):
    rec = _CASES[i]
    cfg = OperatorConfig(**rec["config"])
    c = FlopCounters()
    c.add_all(_counts(rec["case"], cfg))
    assert c.as_dict() == rec["counters"]


def test_counters_accumulate_per_apply():
    rec = _CASES[0]
    cfg = OperatorConfig(**rec["config"])
    inc = _counts(rec["case"], cfg)
    c = FlopCounters()
    for _ in range(3):
        c.add_all(inc)
    assert c.as_dict() == {k: 3 * v for k, v in rec["counters"].items()}
    c.reset()
    assert c.total_flops == 0


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not present")
def test_counters_live_reference():
    sys.path.insert(0, os.path.join(GOLDEN))
    import make_counters as MC

    case, cfg = MC.CASES[6]
    live, _ = MC.run(case, cfg)
    c = FlopCounters()
    c.add_all(_counts({k: (list(v) if isinstance(v, tuple) else v) for k, v in case.items()},
                      OperatorConfig(**cfg)))
    assert c.as_dict() == live
    assert np.all(c.values >= 0)
