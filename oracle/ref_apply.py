"""NumPy restatement of the reference matrix-free apply (oracle only).

Each function cites the reference code it restates.  Arrays are plain NumPy;
nothing here touches the GPU package.

Kernel functions (kernels/numpy_backend.py):
    gather                numpy_backend.py:23-27
    interp / interp_t     numpy_backend.py:48-65   (E @ U, E.T @ V)
    d_action_affine       numpy_backend.py:68-76   (J^-1 (jxw (J^-T g)))
    mass_action           numpy_backend.py:86-88
    face_qpoint           numpy_backend.py:91-109
    boundary_qpoint       numpy_backend.py:112-119
    scatter_add           numpy_backend.py:38-40   (np.add.at, masked skip)
Operator loops (operator.py):
    cell loop             operator.py:255-278
    CG apply + Dirichlet  operator.py:320-331
    face loop             operator.py:387-437
    DG / Helmholtz apply  operator.py:456-493
Geometry (geometry.py, affine mode):
    cells                 geometry.py:145-151
    faces                 geometry.py:202-236  (normals, surface JxW, m = J^-1 n)
"""

from __future__ import annotations

import numpy as np

REF_VERTICES = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]])
FACE_VERTICES = np.array(((1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2)))


# --------------------------------------------------------------------- kernels
def gather(u, idx):
    out = u[np.clip(idx, 0, None)]
    out[idx < 0] = 0.0
    return out


def scatter_add(y, idx, block):
    sel = idx >= 0
    np.add.at(y, idx[sel], block[sel])


def d_action_affine(G, jit, jxw):
    g1 = np.einsum("sij,qjs->qis", jit, G, optimize=True)
    g1 *= jxw.T[:, None, :]
    return np.einsum("sji,qjs->qis", jit, g1, optimize=True)


def face_qpoint(Vm, Vp, Gm, Gp, m_minus, m_plus, sjxw, tau, scale):
    dn_m = np.einsum("sqk,qks->qs", m_minus, Gm, optimize=True)
    dn_p = np.einsum("sqk,qks->qs", m_plus, Gp, optimize=True)
    jump = Vm - Vp
    avg = 0.5 * (dn_m + dn_p)
    w = sjxw.T * scale
    qv = w * (tau[None, :] * jump - avg)
    half_wj = -0.5 * (w * jump)
    qg_m = half_wj[:, None, :] * np.transpose(m_minus, (1, 2, 0))
    qg_p = half_wj[:, None, :] * np.transpose(m_plus, (1, 2, 0))
    return qv, qg_m, qg_p


def boundary_qpoint(Vm, Gm, m, sjxw, tau, scale):
    dn = np.einsum("sqk,qks->qs", m, Gm, optimize=True)
    w = sjxw.T * scale
    qv = w * (tau[None, :] * Vm - dn)
    qg = -(w * Vm)[:, None, :] * np.transpose(m, (1, 2, 0))
    return qv, qg


# -------------------------------------------------------------------- geometry
def cell_jacobians(vertices, cells):
    v = vertices[cells]
    return np.stack([v[:, 1] - v[:, 0], v[:, 2] - v[:, 0], v[:, 3] - v[:, 0]], axis=2)


def affine_cell_geometry(vertices, cells, weights):
    """geometry.py:145-151: J^-T (N,3,3), jxw = det * w (N, n_q)."""
    jac = cell_jacobians(vertices, cells)
    det = np.linalg.det(jac)
    if np.any(det <= 0):
        raise ValueError("non-positive Jacobian determinant")
    jit = np.transpose(np.linalg.inv(jac), (0, 2, 1))
    return jit, det[:, None] * weights[None, :], det


def affine_face_geometry(vertices, cells, c_minus, lf_minus, face_weights, c_plus=None):
    """geometry.py:202-236 for straight cells: per-face (constant) unit normal
    outward from the minus cell, surface JxW per point, m = J^-1 n per side."""
    jac = cell_jacobians(vertices, cells)
    jm = jac[c_minus]
    corners = REF_VERTICES[FACE_VERTICES[lf_minus]]                 # (F, 3, 3)
    t_s = np.einsum("fij,fj->fi", jm, corners[:, 1] - corners[:, 0])
    t_t = np.einsum("fij,fj->fi", jm, corners[:, 2] - corners[:, 0])
    cr = np.cross(t_s, t_t)
    norm = np.linalg.norm(cr, axis=1)
    nrm = cr / norm[:, None]
    cen = vertices[cells[c_minus]].mean(axis=1)
    fc = vertices[cells[c_minus[:, None], FACE_VERTICES[lf_minus]]].mean(axis=1)
    nrm *= np.sign(np.einsum("fi,fi->f", nrm, fc - cen))[:, None]
    sjxw = norm[:, None] * face_weights[None, :]
    m_minus = np.linalg.solve(jm, nrm[..., None])[..., 0]
    m_plus = None if c_plus is None else np.linalg.solve(jac[c_plus], nrm[..., None])[..., 0]
    return nrm, sjxw, m_minus, m_plus


# ------------------------------------------------------------------ cell loop
def _cell_batches(n_cells, lane_width, cells_per_lane):
    """dofmap.py:178-194 lane-major batches (slot c*W + l holds cell base + l*cpl + c)."""
    per = lane_width * cells_per_lane
    nb = (n_cells + per - 1) // per
    ids = np.empty((nb, per), dtype=np.int64)
    act = np.zeros((nb, per), dtype=bool)
    for l in range(lane_width):
        for c in range(cells_per_lane):
            cell = np.arange(nb) * per + l * cells_per_lane + c
            ids[:, c * lane_width + l] = np.minimum(cell, n_cells - 1)
            act[:, c * lane_width + l] = cell < n_cells
    return ids, act


def cell_loop(u, y, gidx, Eg, jit, jxw, Ev=None, mass_jxw=None, mass_scale=0.0,
              stiff_scale=1.0, batch_cells=None, max_batches=None, chunk=None):
    """operator.py:255-278 over batches of cells.

    gidx: (N, n_dpc) gather indices (-1 = masked).  jxw: stiffness JxW (N, n_q)
    (already scaled by any per-cell coefficient); mass_jxw: unscaled JxW for
    the mass term.  ``batch_cells`` = columns per batch (None: one batch of all
    cells).  ``chunk``: process contiguous ranges of this many cells instead (bounded
    memory at full BASELINE sizes; the sum is the same up to rounding order).  Returns
    the number of batches run.
    """
    n = len(gidx)
    nq = Eg.shape[0] // 3
    if chunk is not None:
        batches = ((np.arange(c0, min(n, c0 + chunk)), np.ones(min(n, c0 + chunk) - c0, bool))
                   for c0 in range(0, n, chunk))
    elif batch_cells is None:
        batches = [(np.arange(n), np.ones(n, bool))]
    else:
        W = 4
        ids, act = _cell_batches(n, W, batch_cells // W)
        batches = zip(ids, act)
    done = 0
    for cells, active in batches:
        if max_batches is not None and done >= max_batches:
            break
        idx = gidx[cells].T.copy()                         # (n_dpc, S)
        idx[:, ~active] = -1
        U = gather(u, idx)
        S = U.shape[1]
        G = (Eg @ U).reshape(nq, 3, S)
        D = d_action_affine(G, jit[cells], jxw[cells])
        if stiff_scale != 1.0:
            D *= stiff_scale
        R = Eg.T @ D.reshape(3 * nq, S)
        if mass_scale != 0.0:
            M = (Ev @ U) * (mass_scale * mass_jxw[cells].T)
            R += Ev.T @ M
        scatter_add(y, idx, R)
        done += 1
    return done


# ------------------------------------------------------------------ operators
def cg_apply(vertices, cells, cell_dofs, dirichlet_mask, grad_matrix, weights, u,
             batch_cells=None, kappa=None, chunk=None):
    """CgPoissonOperator.apply (operator.py:320-331); ``kappa``: per-cell coefficient of the
    stiffness term ("multiply the stiffness part by kappa_e")."""
    u = np.asarray(u, dtype=np.float64)
    jit, jxw, _ = affine_cell_geometry(vertices, cells, weights)
    if kappa is not None:
        jxw = jxw * np.asarray(kappa, dtype=np.float64)[:, None]
    gidx = cell_dofs.astype(np.int64).copy()
    if dirichlet_mask is not None and dirichlet_mask.any():
        gidx[dirichlet_mask[gidx]] = -1
    y = np.zeros(len(u))
    cell_loop(u, y, gidx, grad_matrix, jit, jxw, batch_cells=batch_cells, chunk=chunk)
    if dirichlet_mask is not None and dirichlet_mask.any():
        y[dirichlet_mask] = u[dirichlet_mask]
    return y


def _face_loop(u, y, vertices, cells, n_dpc, interior_faces, boundary_faces, dirichlet_ids,
               face_values, face_grads, face_weights, tau_i, tau_b, scale, kappa, comp, nc):
    """operator.py:387-437 with all faces of one signature processed together
    (the per-face tables make the grouping irrelevant numerically)."""
    nqf = len(face_weights)
    loc = np.arange(n_dpc)
    ifc = interior_faces.astype(np.int64)
    if len(ifc):
        cm, lfm, cp, lfp, code = ifc.T
        _, sjxw, mm, mp = affine_face_geometry(vertices, cells, cm, lfm, face_weights, cp)
        tau = np.asarray(tau_i, dtype=np.float64).copy()
        if kappa is not None:
            mm = mm * kappa[cm, None]
            mp = mp * kappa[cp, None]
            tau = tau * np.maximum(kappa[cm], kappa[cp])
        for sig in sorted(set(zip(lfm.tolist(), lfp.tolist(), code.tolist()))):
            sel = np.flatnonzero((lfm == sig[0]) & (lfp == sig[1]) & (code == sig[2]))
            F = len(sel)
            im = ((cm[sel, None] * n_dpc + loc[None, :]) * nc + comp).T
            ip = ((cp[sel, None] * n_dpc + loc[None, :]) * nc + comp).T
            Um, Up = gather(u, im), gather(u, ip)
            Fv_m, Fg_m = face_values[sig[0], 0], face_grads[sig[0], 0]
            Fv_p, Fg_p = face_values[sig[1], sig[2]], face_grads[sig[1], sig[2]]
            Vm, Gm = Fv_m @ Um, (Fg_m @ Um).reshape(nqf, 3, F)
            Vp, Gp = Fv_p @ Up, (Fg_p @ Up).reshape(nqf, 3, F)
            mmf = np.broadcast_to(mm[sel, None, :], (F, nqf, 3))
            mpf = np.broadcast_to(mp[sel, None, :], (F, nqf, 3))
            qv, qg_m, qg_p = face_qpoint(Vm, Vp, Gm, Gp, mmf, mpf, sjxw[sel], tau[sel], scale)
            Rm = Fv_m.T @ qv + Fg_m.T @ qg_m.reshape(3 * nqf, F)
            Rp = Fv_p.T @ (-qv) + Fg_p.T @ qg_p.reshape(3 * nqf, F)
            scatter_add(y, im, Rm)
            scatter_add(y, ip, Rp)
    bfc = boundary_faces.astype(np.int64)
    dsel = np.flatnonzero(np.isin(bfc[:, 2], np.array(sorted(dirichlet_ids), dtype=np.int64))) \
        if len(bfc) and len(dirichlet_ids) else np.zeros(0, np.int64)
    if len(dsel):
        c, lf = bfc[dsel, 0], bfc[dsel, 1]
        _, sjxw, m, _ = affine_face_geometry(vertices, cells, c, lf, face_weights)
        tau = np.asarray(tau_b, dtype=np.float64)[dsel].copy()
        if kappa is not None:
            m = m * kappa[c, None]
            tau = tau * kappa[c]
        for f in range(4):
            s = np.flatnonzero(lf == f)
            if not len(s):
                continue
            F = len(s)
            idx = ((c[s, None] * n_dpc + loc[None, :]) * nc + comp).T
            U = gather(u, idx)
            Fv, Fg = face_values[f, 0], face_grads[f, 0]
            V, G = Fv @ U, (Fg @ U).reshape(nqf, 3, F)
            mf = np.broadcast_to(m[s, None, :], (F, nqf, 3))
            qv, qg = boundary_qpoint(V, G, mf, sjxw[s], tau[s], scale)
            scatter_add(y, idx, Fv.T @ qv + Fg.T @ qg.reshape(3 * nqf, F))


def dg_apply(vertices, cells, n_dpc, interior_faces, boundary_faces, dirichlet_ids,
             value_matrix, grad_matrix, weights, face_values, face_grads, face_weights,
             tau_i, tau_b, u, kappa=None, mass_scale=0.0, stiff_scale=1.0, n_components=1, chunk=None):
    """DgSipgOperator.apply (operator.py:456-466), HelmholtzOperator.apply
    (operator.py:481-493; 3 interleaved components, constant coefficients) and
    the scalar per-cell-kappa Helmholtz of BASELINE config 4 (SURVEY §8c-3:
    jxw*kappa_e, m*kappa per side, tau*max(kappa), plus an unscaled mass)."""
    u = np.asarray(u, dtype=np.float64)
    n = len(cells)
    nc = n_components
    jit, jxw, _ = affine_cell_geometry(vertices, cells, weights)
    sjxw_cells = jxw if kappa is None else jxw * kappa[:, None]
    y = np.zeros(len(u))
    for comp in range(nc):
        gidx = (np.arange(n)[:, None] * n_dpc + np.arange(n_dpc)[None, :]) * nc + comp
        cell_loop(u, y, gidx, grad_matrix, jit, sjxw_cells, value_matrix, jxw,
                  mass_scale, stiff_scale, chunk=chunk)
        if stiff_scale != 0.0:
            _face_loop(u, y, vertices, cells, n_dpc, interior_faces, boundary_faces,
                       dirichlet_ids, face_values, face_grads, face_weights, tau_i, tau_b,
                       stiff_scale, kappa, comp, nc)
    return y


def cg_diagonal(vertices, cells, cell_dofs, dirichlet_mask, grad_matrix, weights, n_dofs, kappa=None):
    """Diagonal of the CG operator (identity on Dirichlet rows): the matrix-free
    equivalent of sparse.assemble(...).diagonal() (sparse.py:237-243)."""
    jit, jxw, _ = affine_cell_geometry(vertices, cells, weights)
    if kappa is not None:
        jxw = jxw * np.asarray(kappa, dtype=np.float64)[:, None]
    nq = grad_matrix.shape[0] // 3
    g3 = grad_matrix.reshape(nq, 3, -1)
    B = np.einsum("eij,qja->eqia", jit, g3)
    dloc = np.einsum("eqia,eqia,eq->ea", B, B, jxw)
    d = np.zeros(n_dofs)
    np.add.at(d, cell_dofs.astype(np.int64).ravel(), dloc.ravel())
    if dirichlet_mask is not None:
        d[dirichlet_mask] = 1.0
    return d


def jacobi_pcg(apply, diag, b, iters):
    """Point-Jacobi preconditioned CG, x0 = 0, fixed iteration count (SPEC.md:509-517
    restated; builder decision: no early exit).  Returns (x, residual norms)."""
    x = np.zeros_like(b)
    r = b.copy()
    z = r / diag
    p = z.copy()
    rz = float(r @ z)
    hist = [float(np.sqrt(r @ r))]
    for _ in range(iters):
        q = apply(p)
        pq = float(p @ q)
        alpha = rz / pq if pq != 0.0 else 0.0   # exact breakdown (converged): stay put
        x += alpha * p
        r -= alpha * q
        z = r / diag
        rz_new = float(r @ z)
        hist.append(float(np.sqrt(r @ r)))
        p = z + (rz_new / rz if rz != 0.0 else 0.0) * p
        rz = rz_new
    return x, np.array(hist)
