"""Logical flop/byte counters (mirrors counters.py:15-58 of the reference).

The reference adds, per 16-column batch it runs, the arithmetic volume of each
kernel call (operator.py:227-245 cells, :416-419 interior faces, :434-437
boundary faces) and the vector traffic once per apply (:247-248).  Every one of
those increments is fixed by the batch layout (lane width W, cells per lane,
components, face signature runs), not by the data, so the B200 operator computes
the whole per-apply increment once, at construction, with
:func:`reference_apply_counts` and adds it per apply: ``counters.as_dict()``
returns the same keys and the same values as the reference operator after the
same number of applies.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["FlopCounters", "reference_apply_counts", "COUNTER_NAMES"]

COUNTER_NAMES = (
    "cell_interp_flops",   # cell E / E^T products
    "cell_qpoint_flops",   # Jacobian transforms and JxW scaling
    "cell_sum_flops",      # accumulation into the result vector
    "face_interp_flops",   # face E_f / E_f^T products, both sides
    "face_qpoint_flops",   # jump/average/penalty arithmetic
    "index_bytes",         # gather/scatter index traffic (4 B each)
    "vector_bytes",        # unique DoF read/write traffic (24 B per DoF)
    "geometry_bytes",      # per-cell geometry pointer traffic
    "spmv_flops",
)

# operator.py:49-54
_D_FLOPS_PER_POINT = 33
_FACE_Q_FLOPS = 26
_BND_Q_FLOPS = 13


@dataclass
class FlopCounters:
    """counters.py:28-58: same names, same derived totals."""

    values: np.ndarray = field(default_factory=lambda: np.zeros(len(COUNTER_NAMES), dtype=np.int64))

    def reset(self) -> None:
        self.values[:] = 0

    def add(self, name: str, amount: int) -> None:
        self.values[COUNTER_NAMES.index(name)] += int(amount)

    def add_all(self, amounts: dict) -> None:
        for k, v in amounts.items():
            self.add(k, v)

    def __getitem__(self, name: str) -> int:
        return int(self.values[COUNTER_NAMES.index(name)])

    @property
    def cell_flops(self) -> int:
        return self["cell_interp_flops"] + self["cell_qpoint_flops"] + self["cell_sum_flops"]

    @property
    def face_flops(self) -> int:
        return self["face_interp_flops"] + self["face_qpoint_flops"]

    @property
    def total_flops(self) -> int:
        return self.cell_flops + self.face_flops + self["spmv_flops"]

    def as_dict(self) -> dict:
        out = {n: int(v) for n, v in zip(COUNTER_NAMES, self.values)}
        out["cell_flops"] = self.cell_flops
        out["face_flops"] = self.face_flops
        out["total_flops"] = self.total_flops
        return out


def _group_sizes(keys: np.ndarray, capacity: int) -> np.ndarray:
    """Sizes of operator._group_faces's groups (operator.py:151-170): maximal runs of
    equal key rows in list order, each cut into pieces of at most ``capacity``."""
    n = len(keys)
    if n == 0:
        return np.zeros(0, dtype=np.int64)
    change = np.ones(n, dtype=bool)
    change[1:] = np.any(keys[1:] != keys[:-1], axis=1)
    starts = np.flatnonzero(change)
    runs = np.diff(np.append(starts, n))
    full = runs // capacity
    rem = runs % capacity
    return np.concatenate([np.repeat(np.full(len(runs), capacity), full), rem[rem > 0]]).astype(np.int64)


def reference_apply_counts(config, dofmap, n_q: int, n_qf: int = 0, *, interior_faces=None,
                           boundary_faces=None, dirichlet_ids=(), mass_scale: float = 0.0,
                           diffusivity: float = 1.0, affine: bool = True, faces: bool = False) -> dict:
    """Per-apply increments of every reference counter for one operator.

    ``config``: the reference's OperatorConfig fields (kernel_stage, batching,
    lane_width, precision); ``dofmap``: space, n_components, cell_dofs,
    dirichlet_mask.  Follows build_batch_plan (dofmap.py:196-266: W lanes x
    cells_per_lane cells per batch, or one cell x 3 components per lane), the cell
    loop's per-batch increments (operator.py:227-245), the face loop's per-group
    increments (operator.py:416-419, 434-437) and _count_apply_vectors (:247-248)."""
    W = config.lane_width if config.lane_width is not None else (8 if config.precision == "f32" else 4)
    stage_mm = config.kernel_stage in ("mm", "sched")
    components = config.batching == "components"
    cpl = 4 if (stage_mm and not components) else 1
    nc = int(dofmap.n_components)
    cd = np.asarray(dofmap.cell_dofs)
    n_cells, nd = cd.shape
    dg = dofmap.space == "dg"
    # plans: one (components batching: 3 columns per lane), one per component (cells batching)
    n_plans = 1 if (components or nc == 1) else nc
    n_cols = 3 if components else cpl
    per_batch = W * (1 if components else cpl)
    n_batches = -(-n_cells // per_batch)
    S = n_cols * W
    slots_per_cell = 3 if components else 1
    n_active = n_cells * slots_per_cell
    mask = np.asarray(dofmap.dirichlet_mask, dtype=bool)
    masked = int(mask[cd].sum()) if (not dg and mask.any()) else 0
    n_unmasked = (n_cells * nd - masked) * slots_per_cell
    with_mass = mass_scale != 0.0

    c = dict.fromkeys(COUNTER_NAMES, 0)
    per_plan = {
        "cell_interp_flops": 2 * (3 * n_q * nd * 2) * S * n_batches,
        "cell_qpoint_flops": _D_FLOPS_PER_POINT * n_q * S * n_batches,
        "cell_sum_flops": n_unmasked,
        "index_bytes": 4 * (1 if dg else nd) * n_active,
        "geometry_bytes": ((14 if not dg else 18) * S // W) * n_batches,
    }
    if with_mass:
        per_plan["cell_interp_flops"] += 2 * (n_q * nd * 2) * S * n_batches
        per_plan["cell_qpoint_flops"] += (2 * n_q + 3 * n_q) * S * n_batches
        per_plan["cell_sum_flops"] += nd * S * n_batches
    if not affine:
        per_plan["geometry_bytes"] += 72 * n_q * n_active

    if faces and diffusivity != 0.0:
        cap = 4 * W if stage_mm else W
        cols = 3 if components else 1
        ifc = np.zeros((0, 5), np.int64) if interior_faces is None else np.asarray(interior_faces)
        gi = _group_sizes(ifc[:, [1, 3, 4]], cap) if len(ifc) else np.zeros(0, np.int64)
        Si = cols * gi
        per_plan["face_interp_flops"] = int((2 * 2 * 4 * n_qf * nd * 2 * Si).sum())
        per_plan["face_qpoint_flops"] = int((_FACE_Q_FLOPS * n_qf * Si).sum())
        per_plan["index_bytes"] += int(4 * 2 * gi.sum())
        per_plan["geometry_bytes"] += int((18 * Si // W).sum())
        bfc = np.zeros((0, 3), np.int64) if boundary_faces is None else np.asarray(boundary_faces)
        dsel = np.isin(bfc[:, 2], np.array(sorted(int(b) for b in dirichlet_ids), dtype=np.int64)) \
            if len(bfc) else np.zeros(0, bool)
        gb = _group_sizes(bfc[dsel][:, [1]], cap) if dsel.any() else np.zeros(0, np.int64)
        Sb = cols * gb
        per_plan["face_interp_flops"] += int((2 * 4 * n_qf * nd * 2 * Sb).sum())
        per_plan["face_qpoint_flops"] += int((_BND_Q_FLOPS * n_qf * Sb).sum())
        per_plan["index_bytes"] += int(4 * gb.sum())
        per_plan["geometry_bytes"] += int((18 * Sb // W).sum())

    for k, v in per_plan.items():
        c[k] += int(v) * n_plans
    c["vector_bytes"] = 24 * int(dofmap.n_scalar_dofs) * nc
    return c
