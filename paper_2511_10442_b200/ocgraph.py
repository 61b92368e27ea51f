"""Association matrices for object-condensation training, on the GPU.

Mirrors the reference's ``gridknn.ocgraph`` front end (G/ocgraph.py:1-202):
``Associations``, ``UniqueObjects``, ``AssociationMatrices``, ``find_unique``,
``max_same_count`` and ``oc_helper`` with the same arguments, defaults,
result layout and errors.  The work runs in the sm_100a kernels of
``csrc/fg_oc.cu`` (``fg_oc_find_unique`` / ``fg_oc_matrices``); like the
reference, results are returned as read-only host numpy arrays, and the
device tensors stay available (``.device``) for callers that keep going on the
GPU.
"""

from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import ops
from .core import RowSplits, default_device
from .errors import BadCapacityError, BadShapeError, OutOfRangeError, ShapeMismatchError

__all__ = ["Associations", "UniqueObjects", "AssociationMatrices", "find_unique",
           "max_same_count", "oc_helper"]


def _frozen(t: Optional[torch.Tensor]):
    if t is None:
        return None
    a = t.detach().cpu().numpy()
    a.flags.writeable = False
    return a


class Associations:
    """Per-vertex association ids (negative = background) over a ragged batch
    (G/ocgraph.py:27-60).  Membership is always evaluated within a row split."""

    __slots__ = ("asso_idx", "row_splits", "_dev")

    def __init__(self, asso_idx, row_splits):
        if isinstance(asso_idx, torch.Tensor):
            asso_idx = asso_idx.detach().cpu().numpy()
        arr = np.ascontiguousarray(asso_idx, dtype=np.int64)
        if arr.ndim != 1:
            raise BadShapeError("association ids must be 1-d")
        if not isinstance(row_splits, RowSplits):
            row_splits = RowSplits(row_splits)
        if arr.size != row_splits.n_vertices:
            raise ShapeMismatchError(f"{arr.size} association ids for "
                                     f"{row_splits.n_vertices} vertices")
        arr.flags.writeable = False
        self.asso_idx = arr
        self.row_splits = row_splits
        self._dev = {}

    @property
    def n_vertices(self) -> int:
        return self.asso_idx.size

    def device_tensors(self, device=None):
        """(asso i64[N], row_splits i64[S+1]) on ``device`` (cached)."""
        device = torch.device(device) if device is not None else default_device()
        key = str(device)
        if key not in self._dev:
            self._dev[key] = torch.from_numpy(self.asso_idx.copy()).to(device)
        return self._dev[key], self.row_splits.device_tensor(device)

    def __repr__(self) -> str:
        return (f"Associations(n_vertices={self.n_vertices}, "
                f"n_splits={self.row_splits.n_splits})")


class UniqueObjects:
    """Objects in scan order: distinct ids per split, first occurrence first
    (G/ocgraph.py:63-84).  ``counts`` / ``max_count`` come from the same pass."""

    __slots__ = ("unique_idx", "unique_rs_asso", "counts", "max_count", "device")

    def __init__(self, unique_idx, unique_rs_asso, counts=None, max_count=None, device=None):
        ids = np.ascontiguousarray(unique_idx, dtype=np.int64)
        rs = np.ascontiguousarray(unique_rs_asso, dtype=np.int64)
        if ids.ndim != 1 or rs.shape != ids.shape:
            raise BadShapeError("unique ids and splits must be 1-d and equally long")
        ids.flags.writeable = False
        rs.flags.writeable = False
        self.unique_idx = ids
        self.unique_rs_asso = rs
        self.counts = counts
        self.max_count = max_count
        self.device = device  # (unique_idx, unique_rs) device tensors, when built here

    @property
    def n_unique(self) -> int:
        return self.unique_idx.size

    def device_tensors(self, device):
        if self.device is not None and self.device[0].device == torch.device(device):
            return self.device
        return (torch.from_numpy(self.unique_idx.copy()).to(device),
                torch.from_numpy(self.unique_rs_asso.copy()).to(device))

    def __repr__(self) -> str:
        return f"UniqueObjects(n_unique={self.n_unique})"


class AssociationMatrices:
    """M / M-not rows per object plus the visit counter (G/ocgraph.py:87-111):
    one visit per vertex of each object's window, M-not requested or not."""

    __slots__ = ("unique", "m", "m_not", "visit_count", "device")

    def __init__(self, unique, m, m_not, visit_count, device=None):
        self.unique = unique
        self.m = m
        self.m_not = m_not
        self.visit_count = int(visit_count)
        self.device = device  # (m, m_not) device tensors

    def __repr__(self) -> str:
        shape_not = None if self.m_not is None else self.m_not.shape
        return (f"AssociationMatrices(m={self.m.shape}, m_not={shape_not}, "
                f"visits={self.visit_count})")


def _unique_device(assoc: Associations, device=None) -> UniqueObjects:
    a, rs = assoc.device_tensors(device)
    uidx, urs, cnt, top = ops.oc_find_unique(a, rs)
    return UniqueObjects(uidx.cpu().numpy(), urs.cpu().numpy(), cnt.cpu().numpy(), top,
                         device=(uidx, urs))


def find_unique(assoc: Associations, *, device=None) -> UniqueObjects:
    """Distinct non-negative ids per split in first-occurrence order; the same
    id in two splits is two objects (G/ocgraph.py:114-134)."""
    return _unique_device(assoc, device)


def _check_objects(assoc: Associations, unique: UniqueObjects) -> None:
    """A caller-supplied object list must address existing splits before it
    reaches the device (the reference raises through RowSplits.bounds,
    G/core.py:80-84)."""
    ids, rs = np.asarray(unique.unique_idx), np.asarray(unique.unique_rs_asso)
    if ids.shape != rs.shape:
        raise ShapeMismatchError(f"unique_idx has {ids.size} entries, unique_rs_asso {rs.size}")
    n_splits = assoc.row_splits.n_splits
    bad = (rs < 0) | (rs >= n_splits)
    if bad.any():
        raise OutOfRangeError(f"split {int(rs[bad][0])} out of range [0, {n_splits})")


def max_same_count(assoc: Associations, unique: Optional[UniqueObjects] = None, *, device=None):
    """(largest member count, per-object counts in unique order)
    (G/ocgraph.py:137-149)."""
    if unique is not None:
        _check_objects(assoc, unique)
    if unique is None or unique.counts is None:
        fresh = _unique_device(assoc, device)
        if unique is None:
            unique = fresh
        else:  # counts for a caller-supplied object list: same keys, reorder
            pos = {(int(i), int(s)): j for j, (i, s) in
                   enumerate(zip(fresh.unique_idx, fresh.unique_rs_asso))}

            def count(i, s):
                if (i, s) in pos:
                    return int(fresh.counts[pos[(i, s)]])
                # ids the fresh table does not hold (negative / absent): count
                # them in the split the way the reference does
                lo, hi = assoc.row_splits.bounds(s)
                return int(np.count_nonzero(assoc.asso_idx[lo:hi] == i))

            counts = np.array([count(int(i), int(s)) for i, s in
                               zip(unique.unique_idx, unique.unique_rs_asso)], dtype=np.int64)
            return (int(counts.max()) if counts.size else 0), counts
    counts = np.asarray(unique.counts, dtype=np.int64)
    return (int(counts.max()) if counts.size else 0), counts


def oc_helper(assoc: Associations, unique: Optional[UniqueObjects] = None, *,
              n_maxuq: Optional[int] = None, n_maxrs: Optional[int] = None,
              calc_m_not: bool = True, device=None) -> AssociationMatrices:
    """M (members per object) and optionally M-not (non-members) rows
    (G/ocgraph.py:152-202).  Each object scans the first ``n_maxrs`` vertices of
    its split; rows are ascending vertex ids with a contiguous -1 suffix.
    Defaults: n_maxuq = largest member count, n_maxrs = largest split (>= 1)."""
    if unique is not None:
        _check_objects(assoc, unique)
    uniq = unique if unique is not None else _unique_device(assoc, device)
    if n_maxuq is None:
        top, _ = max_same_count(assoc, uniq, device=device)
        n_maxuq = max(1, top)
    sizes = assoc.row_splits.sizes()
    largest = int(sizes.max()) if sizes.size else 0
    if n_maxrs is None:
        n_maxrs = max(1, largest)
    n_maxuq, n_maxrs = int(n_maxuq), int(n_maxrs)
    if n_maxuq < 1 or n_maxrs < 1:
        raise BadCapacityError(f"capacities must be >= 1, got n_maxuq={n_maxuq}, "
                               f"n_maxrs={n_maxrs}")
    a, rs = assoc.device_tensors(device)
    ui, ur = uniq.device_tensors(a.device)
    m, m_not, visits = ops.oc_matrices(a, rs, ui, ur, n_maxuq, n_maxrs, largest, calc_m_not)
    return AssociationMatrices(uniq, _frozen(m), _frozen(m_not), int(visits.item()),
                               device=(m, m_not))
