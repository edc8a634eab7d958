"""Record the REAL reference's logical counters (counters.py) after one apply.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_counters.py

Each case builds a reference operator on one of the golden fixtures' inputs (the
seeded Kuhn mesh and tables of tests/golden/<fixture>.npz, rebuilt here exactly as
make_golden.py builds them) with a given OperatorConfig, runs ``apply`` once and
stores ``counters.as_dict()``.  Output: tests/golden/counters_ref.json, which
tests/test_counters.py compares against paper_2509_10226_b200.counters (no
reference needed there).
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as G  # noqa: E402  (imports the reference from /root/reference/pkg/src)

from tetmf import geometry as rgeo  # noqa: E402
from tetmf import operator as rop  # noqa: E402

# (fixture-like case, config kwargs); kind/n/p/rule/dids/nc as in make_golden.cases()
CASES = [
    (dict(kind="cg", n=3, p=2, rule="gm", dids=G.ALL), {}),
    (dict(kind="cg", n=3, p=3, rule="ref", dids=(0, 3)), dict(kernel_stage="ref")),
    (dict(kind="cg", n=3, p=1, rule="gm", dids=(1, 4)), dict(precision="f32")),
    (dict(kind="cg", n=3, p=2, rule="ref", dids=(0, 2, 5), nc=3), dict(lane_width=8)),
    (dict(kind="cg", n=3, p=2, rule="ref", dids=(0, 2, 5), nc=3), dict(batching="components")),
    (dict(kind="cg", n=4, p=4, rule="gm", dids=()), dict(kernel_stage="sched")),
    (dict(kind="dg", n=3, p=2, rule="gm", dids=G.ALL), {}),
    (dict(kind="dg", n=3, p=3, rule="ref", dids=(1,)), dict(kernel_stage="data", lane_width=8)),
    (dict(kind="dg", n=2, p=1, rule="gm", dids=()), dict(kernel_stage="mm", lane_width=2)),
    (dict(kind="helm3", n=2, p=2, rule="gm", dids=G.ALL, ms=3.0, nu=1.0), dict(batching="components")),
    (dict(kind="helm3", n=2, p=1, rule="ref", dids=(), ms=2.0, nu=0.5), {}),
    (dict(kind="helm3", n=2, p=1, rule="ref", dids=G.ALL, ms=2.0, nu=0.0), dict(kernel_stage="ref")),
]


def run(case, cfg):
    tm = G.ref_mesh(case["n"], 0)
    p = case["p"]
    cr, fr = G.rules(p, case["rule"])
    basis = G.ref_basis(p, cr, fr)
    config = rop.OperatorConfig(**cfg)
    if case["kind"] == "cg":
        dm = G.ref_dofmap(tm, p, "cg", case.get("nc", 1), case["dids"])
        geo = rgeo.build_geometry(tm, cr, "affine")
        op = rop.CgPoissonOperator(tm, dm, geo, basis, config)
    else:
        nc = 3 if case["kind"] == "helm3" else 1
        dm = G.ref_dofmap(tm, p, "dg", nc)
        geo = rgeo.build_geometry(tm, cr, "affine", fr)
        G.broadcast_face_m(geo, fr.n_points)
        ti, tb = G.sipg_tau(tm, p, case["n"])
        sipg = rop.SipgConfig(1.0, ti, tb)
        if case["kind"] == "dg":
            op = rop.DgSipgOperator(tm, dm, geo, basis, sipg, config, case["dids"])
        else:
            co = rop.HelmholtzCoefficients(case["ms"], case["nu"])
            op = rop.HelmholtzOperator(tm, dm, geo, basis, sipg, co, config, case["dids"])
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    op.apply(u)
    return op.counters.as_dict(), op.n_applies


def main():
    out = []
    for case, cfg in CASES:
        counters, n_applies = run(case, cfg)
        out.append({"case": {k: (list(v) if isinstance(v, tuple) else v) for k, v in case.items()},
                    "config": cfg, "n_applies": n_applies, "counters": counters})
        print(case, cfg, counters["total_flops"])
    with open(os.path.join(HERE, "counters_ref.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
