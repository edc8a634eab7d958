"""Generate golden fixtures by running the REAL reference package.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Every fixture is the reference's own output on a seeded Kuhn mesh built by
this package's generator and paired by the reference's ``_build_faces``
(mesh.py:84-120).  Workarounds documented in SURVEY §0-4 / §8c are applied
exactly as stated there and nowhere else:

* DG in affine mode: face m-vectors broadcast to (F, n_qf, 3) after
  ``build_geometry`` (the shipped backend crashes on the compact arrays);
* BASELINE penalty tau = 2.5 (p+1)^2 / h injected through ``SipgConfig``;
* scalar per-cell-kappa Helmholtz composed from the reference DG operator
  (jxw*kappa, m*kappa per side, tau*max(kappa)) plus the reference CSR mass
  (``sparse.assemble`` with ``HelmholtzCoefficients(1, 0)``);
* Grundmann-Moller rules injected as reference ``QuadratureRule`` objects
  ("gm" fixtures); "ref" fixtures use the reference's own tables;
* P4: the reference operator and CSR assembly run unchanged on this
  package's P4 tables and DoF map (the reference stops at p=3).

Outputs: tests/golden/<name>.npz (inputs, tables and outputs).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from tetmf import basis as rbasis  # noqa: E402
from tetmf import dofmap as rdof  # noqa: E402
from tetmf import geometry as rgeo  # noqa: E402
from tetmf import mesh as rmesh  # noqa: E402
from tetmf import operator as rop  # noqa: E402
from tetmf import quadrature as rquad  # noqa: E402
from tetmf import sparse as rsparse  # noqa: E402

from paper_2509_10226_b200 import basis as mybasis  # noqa: E402
from paper_2509_10226_b200 import dofmap as mydof  # noqa: E402
from paper_2509_10226_b200 import mesh as mymesh  # noqa: E402
from paper_2509_10226_b200 import quadrature as myquad  # noqa: E402


def ref_mesh(n, seed):
    m = mymesh.kuhn_cube_mesh(n, seed=seed)
    bid = lambda c: int(mymesh.cube_boundary_ids(c[None])[0])  # noqa: E731
    ri, rb = rmesh._build_faces(m.cells, bid, m.vertices)
    tm = rmesh.TetMesh(m.vertices, m.cells, ri, rb)
    tm.validate()
    return tm


def rules(p, kind):
    if kind == "ref":
        return rquad.make_cell_quadrature(p), rquad.make_face_quadrature(p)
    c, f = myquad.make_cell_quadrature(p), myquad.make_face_quadrature(p)
    return (rquad.QuadratureRule(c.points, c.weights, c.exactness_degree, 3),
            rquad.QuadratureRule(f.points, f.weights, f.exactness_degree, 2))


def ref_basis(p, cr, fr):
    if p <= 3:
        return rbasis.tabulate_basis(p, cr, fr)
    b = mybasis.tabulate_basis(p, cr, fr)
    return rbasis.BasisTable(p, b.nodes, b.node_tags, cr, fr, b.value_matrix, b.grad_matrix,
                             b.face_values, b.face_grads, np.eye(b.n_dofs))


def ref_dofmap(tm, p, space, nc=1, dids=()):
    if p <= 3 or space == "dg":
        return rdof.build_dof_map(tm, p, space, nc, dids)
    mm = mymesh.TetMesh(tm.vertices, tm.cells, tm.interior_faces, tm.boundary_faces)
    d = mydof.build_dof_map(mm, p, space, nc, dids)
    return rdof.DoFMap(d.space, d.degree, d.n_components, d.n_scalar_dofs, d.cell_dofs,
                       d.dirichlet_mask)


def broadcast_face_m(geo, nqf):
    for name in ("face_m_minus", "face_m_plus", "bnd_m", "face_normals", "bnd_normals"):
        a = getattr(geo, name)
        setattr(geo, name, np.ascontiguousarray(np.broadcast_to(a[:, None, :], (len(a), nqf, 3))))


def base_record(tm, p, rule_kind, cr, fr, basis, dm):
    return dict(
        p=p, rule=rule_kind, vertices=tm.vertices, cells=tm.cells,
        interior_faces=tm.interior_faces, boundary_faces=tm.boundary_faces,
        cell_dofs=dm.cell_dofs, dirichlet_mask=dm.dirichlet_mask,
        cell_points=cr.points, cell_weights=cr.weights,
        face_points=fr.points, face_weights=fr.weights,
        value_matrix=basis.value_matrix, grad_matrix=basis.grad_matrix,
        face_values=basis.face_values, face_grads=basis.face_grads)


def cg_case(n, p, rule_kind, dids, seed=0, nc=1):
    tm = ref_mesh(n, seed)
    cr, fr = rules(p, rule_kind)
    basis = ref_basis(p, cr, fr)
    dm = ref_dofmap(tm, p, "cg", nc, dids)
    geo = rgeo.build_geometry(tm, cr, "affine")
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    y = rop.CgPoissonOperator(tm, dm, geo, basis).apply(u)
    A = rsparse.assemble(dm, tm, geo, basis)
    rec = base_record(tm, p, rule_kind, cr, fr, basis, dm)
    rec.update(kind="cg", n=n, n_components=nc, dirichlet_ids=np.array(dids, dtype=np.int64), u=u, y=y,
               y_csr=A.matvec(u), diag=A.to_scipy().diagonal())
    return rec


def sipg_tau(tm, p, n):
    t = 2.5 * (p + 1) ** 2 * n
    return np.full(len(tm.interior_faces), t), np.full(len(tm.boundary_faces), t)


def dg_case(n, p, rule_kind, dids, seed=0):
    tm = ref_mesh(n, seed)
    cr, fr = rules(p, rule_kind)
    basis = ref_basis(p, cr, fr)
    dm = ref_dofmap(tm, p, "dg")
    geo = rgeo.build_geometry(tm, cr, "affine", fr)
    broadcast_face_m(geo, fr.n_points)
    ti, tb = sipg_tau(tm, p, n)
    sipg = rop.SipgConfig(1.0, ti, tb)
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    y = rop.DgSipgOperator(tm, dm, geo, basis, sipg, dirichlet_ids=dids).apply(u)
    A = rsparse.assemble(dm, tm, geo, basis, sipg, None, dids)
    rec = base_record(tm, p, rule_kind, cr, fr, basis, dm)
    rec.update(kind="dg", n=n, dirichlet_ids=np.array(dids, dtype=np.int64), tau_i=ti, tau_b=tb,
               u=u, y=y, y_csr=A.matvec(u))
    return rec


def helm_kappa_case(n, p, rule_kind, dids, seed=0):
    """Scalar mass + kappa-Laplace DG (BASELINE config 4), composed per SURVEY §8c-3."""
    tm = ref_mesh(n, seed)
    cr, fr = rules(p, rule_kind)
    basis = ref_basis(p, cr, fr)
    dm = ref_dofmap(tm, p, "dg")
    geo = rgeo.build_geometry(tm, cr, "affine", fr)
    broadcast_face_m(geo, fr.n_points)
    kappa = 10.0 ** np.random.default_rng(2).uniform(-1, 1, tm.n_cells)
    ti, tb = sipg_tau(tm, p, n)
    ifc, bfc = tm.interior_faces, tm.boundary_faces
    gk = rgeo.GeometryData(**{k: getattr(geo, k) for k in geo.__dataclass_fields__})
    gk.jxw = geo.jxw * kappa[:, None]
    gk.face_m_minus = geo.face_m_minus * kappa[ifc[:, 0], None, None]
    gk.face_m_plus = geo.face_m_plus * kappa[ifc[:, 2], None, None]
    gk.bnd_m = geo.bnd_m * kappa[bfc[:, 0], None, None]
    sipg = rop.SipgConfig(1.0, ti * np.maximum(kappa[ifc[:, 0]], kappa[ifc[:, 2]]),
                          tb * kappa[bfc[:, 0]])
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    y_lap = rop.DgSipgOperator(tm, dm, gk, basis, sipg, dirichlet_ids=dids).apply(u)
    M = rsparse.assemble(dm, tm, geo, basis, rop.SipgConfig(1.0, ti, tb),
                         rop.HelmholtzCoefficients(1.0, 0.0), ())
    rec = base_record(tm, p, rule_kind, cr, fr, basis, dm)
    rec.update(kind="helm_kappa", n=n, dirichlet_ids=np.array(dids, dtype=np.int64), tau_i=ti,
               tau_b=tb, kappa=kappa, u=u, y=y_lap + M.matvec(u))
    return rec


def helm3_case(n, p, rule_kind, dids, mass_scale, nu, seed=0):
    """The reference's own 3-component constant-coefficient Helmholtz (operator.py:469-493)."""
    tm = ref_mesh(n, seed)
    cr, fr = rules(p, rule_kind)
    basis = ref_basis(p, cr, fr)
    dm = ref_dofmap(tm, p, "dg", 3)
    geo = rgeo.build_geometry(tm, cr, "affine", fr)
    broadcast_face_m(geo, fr.n_points)
    ti, tb = sipg_tau(tm, p, n)
    sipg = rop.SipgConfig(1.0, ti, tb)
    co = rop.HelmholtzCoefficients(mass_scale, nu)
    u = np.random.default_rng(1).uniform(-1, 1, dm.n_global_dofs)
    y = rop.HelmholtzOperator(tm, dm, geo, basis, sipg, co, dirichlet_ids=dids).apply(u)
    A = rsparse.assemble(dm, tm, geo, basis, sipg, co, dids)
    rec = base_record(tm, p, rule_kind, cr, fr, basis, dm)
    rec.update(kind="helm3", n=n, dirichlet_ids=np.array(dids, dtype=np.int64), tau_i=ti, tau_b=tb,
               mass_scale=mass_scale, nu=nu, u=u, y=y, y_csr=A.matvec(u))
    return rec


def reorder_mesh_case():
    """SPEC.md:638 acceptance fixture: the reference's seed-42 shuffled 5-tet 8^3 cube mesh."""
    m = rmesh.shuffle_cells(rmesh.generate_cube_mesh(8), 42)
    return dict(kind="mesh", vertices=m.vertices, cells=m.cells, interior_faces=m.interior_faces,
                boundary_faces=m.boundary_faces)


ALL = tuple(range(6))


def cases():
    yield "mesh_5tet_n8_shuffled42", reorder_mesh_case
    yield "cg_p2_n8_gm", lambda: cg_case(8, 2, "gm", ())            # BASELINE config 1
    yield "cg_p2_n8_gm_dir", lambda: cg_case(8, 2, "gm", ALL)
    for p in (1, 2, 3):
        yield f"cg_p{p}_n4_ref", lambda p=p: cg_case(4, p, "ref", ())
        yield f"cg_p{p}_n4_ref_dir", lambda p=p: cg_case(4, p, "ref", ALL)
        yield f"cg_p{p}_n3_gm_dir2", lambda p=p: cg_case(3, p, "gm", (1, 4))
    yield "cg3_p2_n3_ref_dir", lambda: cg_case(3, 2, "ref", (0, 2, 5), nc=3)
    yield "cg_p4_n3_gm", lambda: cg_case(3, 4, "gm", ())
    yield "cg_p4_n3_gm_dir", lambda: cg_case(3, 4, "gm", ALL)
    for p in (1, 2, 3):
        yield f"dg_p{p}_n3_ref_dir", lambda p=p: dg_case(3, p, "ref", ALL)
        yield f"dg_p{p}_n3_gm_dir", lambda p=p: dg_case(3, p, "gm", ALL)
    yield "dg_p3_n2_gm_dir2", lambda: dg_case(2, 3, "gm", (0, 3))
    yield "dg_p4_n2_gm_dir", lambda: dg_case(2, 4, "gm", ALL)
    yield "helmk_p2_n3_gm_dir", lambda: helm_kappa_case(3, 2, "gm", ALL)
    yield "helmk_p1_n3_ref_dir", lambda: helm_kappa_case(3, 1, "ref", ALL)
    yield "helm3_p1_n2_ref_dir", lambda: helm3_case(2, 1, "ref", ALL, 10.0, 0.5)
    yield "helm3_p2_n2_gm_none", lambda: helm3_case(2, 2, "gm", (), 3.0, 1.0)


def main():
    only = set(sys.argv[1:])
    for name, fn in cases():
        if only and name not in only:
            continue
        rec = fn()
        path = os.path.join(HERE, name + ".npz")
        np.savez_compressed(path, **{k: np.asarray(v) for k, v in rec.items()})
        ref = rec.get("y_csr")
        extra = "" if ref is None else f" mf-vs-csr {np.linalg.norm(rec['y'] - ref) / np.linalg.norm(ref):.2e}"
        ndof = len(rec["u"]) if "u" in rec else 0
        print(f"{name}: {os.path.getsize(path) / 1024:.0f} KiB, n_dof {ndof}{extra}")


if __name__ == "__main__":
    main()
