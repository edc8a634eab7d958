"""Shared test helpers: build B200 operators from golden fixtures / generated meshes."""

from types import SimpleNamespace as NS

import numpy as np

from paper_2509_10226_b200 import operator as op


def fixture_objects(g):
    nd = g["cell_dofs"].shape[1]
    kind = str(g["kind"])
    nc = 3 if kind == "helm3" else int(g["n_components"]) if "n_components" in g else 1
    space = "cg" if kind == "cg" else "dg"
    n_scalar = len(g["u"]) // nc
    mesh = NS(vertices=g["vertices"], cells=g["cells"], interior_faces=g["interior_faces"],
              boundary_faces=g["boundary_faces"])
    dofmap = NS(space=space, degree=int(g["p"]), n_components=nc, n_scalar_dofs=n_scalar,
                cell_dofs=g["cell_dofs"], dirichlet_mask=g["dirichlet_mask"])
    geo = NS(cell_rule=NS(weights=g["cell_weights"], points=g["cell_points"]),
             face_rule=NS(weights=g["face_weights"], points=g["face_points"]))
    basis = NS(value_matrix=g["value_matrix"], grad_matrix=g["grad_matrix"],
               face_values=g["face_values"], face_grads=g["face_grads"])
    return mesh, dofmap, geo, basis


def operator_from_fixture(g, device=0, **config):
    mesh, dofmap, geo, basis = fixture_objects(g)
    kind = str(g["kind"])
    cfg = op.OperatorConfig(device=device, **config)
    dids = tuple(int(x) for x in g["dirichlet_ids"])
    if kind == "cg":
        return op.CgPoissonOperator(mesh, dofmap, geo, basis, cfg)
    sipg = op.SipgConfig(1.0, g["tau_i"], g["tau_b"])
    if kind == "dg":
        return op.DgSipgOperator(mesh, dofmap, geo, basis, sipg, cfg, dids)
    if kind == "helm_kappa":
        return op.KappaHelmholtzOperator(mesh, dofmap, geo, basis, sipg, g["kappa"], 1.0, cfg, dids)
    if kind == "helm3":
        co = op.HelmholtzCoefficients(float(g["mass_scale"]), float(g["nu"]))
        return op.HelmholtzOperator(mesh, dofmap, geo, basis, sipg, co, cfg, dids)
    raise AssertionError(kind)
