"""Normal-equation block assembly for one area, on the device.

API mirror of the reference's ``gridse.assembly`` fused path (reference
``pkg/src/gridse/assembly.py:32-53,116-163,172-326,486-524``):
``build_patterns(vmap, ms)`` runs the one-time symbolic analysis (here: a
single-area device plan) and ``fused_accumulate(vmap, ms, x_i, x_b, pattern)``
returns the area's ``AreaNormalBlocks`` in the reference's layout -- CSR
``g_ii`` / ``g_ib`` with the same sorted patterns, dense full ``g_bb``, ``b_i``,
``b_b`` -- computed by the template + accumulation kernels without
materialising the Jacobian.  ``explicit_assemble`` (the reference's test oracle, reference
``assembly.py:531-572``) is offered in the same spirit: the template layer comes from the device
(``gse_area_templates``: the partials exactly as the template kernel wrote them), the Jacobian is
materialised and the blocks are formed by sparse triple products on the host -- so a disagreement with
``fused_accumulate`` isolates the device accumulation program.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np
import scipy.sparse as sp

from . import _native
from .measurement import MeasurementSet
from .partition import AreaVariableMap, BoundaryOrdering, Partition


@dataclass
class AreaNormalBlocks:
    g_ii: sp.csr_matrix
    g_ib: sp.csr_matrix
    g_bb: np.ndarray
    b_i: np.ndarray
    b_b: np.ndarray

    @property
    def n_interior(self):
        return self.g_ii.shape[0]

    @property
    def n_boundary(self):
        return self.g_bb.shape[0]


@dataclass
class JacobianTriplets:
    """Materialized area Jacobian (oracle path only; reference assembly.py:57-72)."""

    rows: np.ndarray
    cols: np.ndarray
    vals: np.ndarray
    weights: np.ndarray
    residuals: np.ndarray
    n_rows: int
    n_cols: int

    def to_csr(self):
        return sp.csr_matrix((self.vals, (self.rows, self.cols)), shape=(self.n_rows, self.n_cols))


def area_row_ids(vmap: AreaVariableMap, ms: MeasurementSet) -> np.ndarray:
    """Rows owned by the area (bus owner for bus rows, from-bus for flows)."""
    owned = np.zeros(ms.net.n_bus, dtype=bool)
    owned[list(vmap.owned_buses)] = True
    return np.flatnonzero(owned[ms.owner_bus])


class AssemblyPattern:
    """One-time analysis of an area's measurement templates (a single-area plan)."""

    def __init__(self, vmap: AreaVariableMap, ms: MeasurementSet, device=0):
        import torch
        self.vmap = vmap
        self.row_ids = area_row_ids(vmap, ms)
        self.n_interior, self.n_boundary = vmap.n_interior, vmap.n_boundary
        net = ms.net
        # the area's rows as their own measurement set, one area, identity boundary layout
        keep = self.row_ids
        self._ms = replace(ms, mtype=ms.mtype[keep], target=ms.target[keep], z=ms.z[keep],
                           sigma=ms.sigma[keep], weight=ms.weight[keep], active=ms.active[keep],
                           owner_bus=ms.owner_bus[keep])
        lb_ang = [int(b) for b in vmap.local_boundary_angle_buses()]
        lb_mag = [int(b) for b in vmap.local_boundary_buses]
        entries = tuple([(b, "va") for b in lb_ang] + [(b, "vm") for b in lb_mag])
        bord = BoundaryOrdering(entries=entries,
                                angle_slot={b: i for i, b in enumerate(lb_ang)},
                                mag_slot={b: len(lb_ang) + i for i, b in enumerate(lb_mag)})
        local = replace(vmap, area=0, boundary_selector=np.arange(vmap.n_boundary, dtype=int))
        part = Partition(k=1, area_of_bus=np.zeros(net.n_bus, dtype=int),
                         cut_branches=np.zeros(0, dtype=int), boundary_buses=np.zeros(0, dtype=int),
                         area_pairs={})
        self.plan = _native.Plan(net, self._ms, part, bord, [local], device=device)
        ii_ptr, ii_idx, ib_ptr, ib_idx = self.plan.area_pattern(0)
        self.gii_indptr, self.gii_indices = ii_ptr.astype(int), ii_idx.astype(int)
        self.gib_indptr, self.gib_indices = ib_ptr.astype(int), ib_idx.astype(int)
        self._torch = torch
        self._dev = torch.device("cuda", device)
        self._state = torch.empty((2, net.n_bus), dtype=torch.float64, device=self._dev)
        self._weights = ms.weight[keep].copy()
        self._z = ms.z[keep].copy()

    def gii_pattern(self):
        n = self.n_interior
        return sp.csr_matrix((np.ones(len(self.gii_indices)), self.gii_indices, self.gii_indptr),
                             shape=(n, n))

    def refresh(self, ms: MeasurementSet):
        """Masking / new values on the same rows: weight and value refresh only."""
        w, z = ms.weight[self.row_ids], ms.z[self.row_ids]
        if not np.array_equal(w, self._weights):
            self.plan.set_weights(w)
            self._weights = w.copy()
        if not np.array_equal(z, self._z):
            self.plan.set_measurements(z)
            self._z = z.copy()

    def scatter_state(self, net, x_i, x_b):
        """(x_i, x_b) -> full (va, vm); unreferenced buses NaN, slack angle pinned
        (the reference's closure poisoning, assembly.py:407-420)."""
        vmap = self.vmap
        va = np.full(net.n_bus, np.nan)
        vm = np.full(net.n_bus, np.nan)
        na = len(vmap.interior_angle_buses)
        va[vmap.interior_angle_buses] = x_i[:na]
        vm[vmap.interior_mag_buses] = x_i[na:]
        lb_ang = vmap.local_boundary_angle_buses()
        va[lb_ang] = x_b[: len(lb_ang)]
        vm[vmap.local_boundary_buses] = x_b[len(lb_ang):]
        va[vmap.slack] = net.buses[vmap.slack].va_true
        return va, vm


def build_patterns(vmap: AreaVariableMap, ms: MeasurementSet) -> AssemblyPattern:
    return AssemblyPattern(vmap, ms)


def fused_accumulate(vmap: AreaVariableMap, ms: MeasurementSet, x_i, x_b,
                     pattern: AssemblyPattern = None) -> AreaNormalBlocks:
    """Assemble the area blocks on the device without materialising the Jacobian."""
    pat = pattern if pattern is not None else build_patterns(vmap, ms)
    pat.refresh(ms)
    net = ms.net
    va, vm = pat.scatter_state(net, np.asarray(x_i, float), np.asarray(x_b, float))
    torch = pat._torch
    pat._state.copy_(torch.from_numpy(np.stack([va, vm])))
    torch.cuda.current_stream(pat._dev).synchronize()
    pat.plan.phase_assemble(pat._state[0].data_ptr(), pat._state[1].data_ptr())
    data_ii, data_ib, g_bb, b_i, b_b = pat.plan.area_blocks(0)
    n_i, n_b = pat.n_interior, pat.n_boundary
    g_ii = sp.csr_matrix((data_ii, pat.gii_indices, pat.gii_indptr), shape=(n_i, n_i))
    g_ib = sp.csr_matrix((data_ib, pat.gib_indices, pat.gib_indptr), shape=(n_i, n_b))
    return AreaNormalBlocks(g_ii=g_ii, g_ib=g_ib, g_bb=g_bb, b_i=b_i, b_b=b_b)


def explicit_assemble(vmap: AreaVariableMap, ms: MeasurementSet, x_i, x_b, pattern: AssemblyPattern = None):
    """Materialize H and form the blocks by sparse triple products (reference assembly.py:531-572).

    The template values are the device's (one ``gse_phase_assemble``, read back with ``gse_area_templates``);
    the residuals are ``z - h`` from the host formulas; ``H^T W H`` and ``H^T W r`` are scipy products.  Returns
    ``(JacobianTriplets, AreaNormalBlocks)`` like the reference.
    """
    from .measurement import StateVector, eval_h_all
    pat = pattern if pattern is not None else build_patterns(vmap, ms)
    pat.refresh(ms)
    net = ms.net
    va, vm = pat.scatter_state(net, np.asarray(x_i, float), np.asarray(x_b, float))
    torch = pat._torch
    pat._state.copy_(torch.from_numpy(np.stack([va, vm])))
    torch.cuda.current_stream(pat._dev).synchronize()
    pat.plan.phase_assemble(pat._state[0].data_ptr(), pat._state[1].data_ptr())
    rows, slot_ptr, slot_var, g_flat, _ = pat.plan.area_templates(0)
    row_ids = pat.row_ids
    assert np.array_equal(rows, np.arange(len(row_ids)))         # the pattern's plan holds exactly the area's rows
    n_i, n_b = vmap.n_interior, vmap.n_boundary
    weights = ms.weight[row_ids]
    resid = ms.z[row_ids] - eval_h_all(pat._ms, StateVector(va=va, vm=vm))
    triplets = JacobianTriplets(rows=np.repeat(np.arange(len(row_ids)), np.diff(slot_ptr)), cols=slot_var.astype(int),
                                vals=g_flat, weights=weights, residuals=resid, n_rows=len(row_ids), n_cols=n_i + n_b)
    h_mat = triplets.to_csr()
    hw = h_mat.multiply(weights[:, None]).tocsr()
    g_full = (h_mat.T @ hw).tocsr()
    g_full.sort_indices()
    b_full = h_mat.T @ (weights * resid)
    blocks = AreaNormalBlocks(g_ii=g_full[:n_i, :n_i].tocsr(), g_ib=g_full[:n_i, n_i:].tocsr(),
                              g_bb=g_full[n_i:, n_i:].toarray(), b_i=b_full[:n_i], b_b=b_full[n_i:])
    return triplets, blocks
