"""GravNet distance-weighted aggregation on the device (mirror of G/gravnet.py)
and the GravNetOp layer built on the binned kNN.

``gravnet_aggregate`` / ``gravnet_aggregate_backward`` keep the reference's
semantics: w = exp(-scale * d2) over valid slots (idx >= 0; slot 0 only with
include_self), reducers in order, one F-wide block each, mean = sum / count,
max over valid slots, zeros for a row with no valid slot; the max block's
gradient goes to the lowest arg-max slot.  Arithmetic is float64 inside the
kernels, results are float32.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
from torch import nn

from . import ops
from .binning import BinningConfig, build_bin_index
from .core import NeighborMatrix, PointCloud
from .errors import BadShapeError, ShapeMismatchError

_REDUCERS = ("mean", "max")
_CODES = {"mean": 0, "max": 1}


@dataclass(frozen=True)
class AggregationSpec:
    """G/gravnet.py:29-49."""

    weight_scale: float = 10.0
    reducers: tuple[str, ...] = ("mean", "max")
    include_self: bool = True

    def __post_init__(self):
        if not self.reducers:
            raise BadShapeError("at least one reducer is required")
        if len(self.reducers) > 4:
            raise BadShapeError("at most 4 reducer blocks")
        for r in self.reducers:
            if r not in _REDUCERS:
                raise BadShapeError(f"unknown reducer {r!r}; expected {_REDUCERS}")
        if not (self.weight_scale > 0.0):
            raise BadShapeError(f"weight_scale must be > 0, got {self.weight_scale!r}")

    @property
    def codes(self) -> list[int]:
        return [_CODES[r] for r in self.reducers]


def _check_features(features: torch.Tensor, neighbors: NeighborMatrix) -> torch.Tensor:
    if features.dim() != 2:
        raise BadShapeError("features must be 2-d (n_vertices, n_features)")
    if features.shape[0] != neighbors.n_vertices:
        raise ShapeMismatchError(f"features cover {features.shape[0]} vertices, "
                                 f"neighbours have {neighbors.n_vertices}")
    return features


def neighbor_weights(neighbors: NeighborMatrix, spec: AggregationSpec):
    """G/gravnet.py:64-72 (elementwise helper; the kernels compute the same
    weights internally in float64)."""
    valid = neighbors.indices >= 0
    if not spec.include_self:
        valid = valid.clone()
        valid[:, 0] = False
    w = torch.exp(-spec.weight_scale * neighbors.dist2.to(torch.float64))
    return torch.where(valid, w, torch.zeros_like(w)), valid


def gravnet_aggregate(features, neighbors: NeighborMatrix,
                      spec: AggregationSpec = AggregationSpec(), order=None) -> torch.Tensor:
    """(n_vertices, n_features * n_reducers); differentiable w.r.t. features
    and neighbors.dist2.  ``order`` (optional, e.g. the bin index's
    sort_order) only changes the order rows are visited in, not the result."""
    f = _check_features(features, neighbors)
    return ops.gravnet_aggregate(f, neighbors.indices, neighbors.dist2, float(spec.weight_scale),
                                 spec.codes, bool(spec.include_self), order)


def gravnet_aggregate_backward(features, neighbors: NeighborMatrix, spec: AggregationSpec,
                               upstream, order=None) -> tuple[torch.Tensor, torch.Tensor]:
    """G/gravnet.py:100-150 -> (grad_features, grad_dist2)."""
    f = _check_features(features, neighbors)
    want = (f.shape[0], f.shape[1] * len(spec.reducers))
    if tuple(upstream.shape) != want:
        raise ShapeMismatchError(f"upstream shape {tuple(upstream.shape)} != {want}")
    return ops.gravnet_aggregate_grad(upstream, f, neighbors.indices, neighbors.dist2,
                                      float(spec.weight_scale), spec.codes,
                                      bool(spec.include_self), order)


class GravNetOp(nn.Module):
    """GravNet message passing on the binned kNN.

    x -> space = S(x) [d_space], props = P(x) [n_prop];
    neighbours = exact kNN in the learned space per row split (k incl. self);
    agg = [mean | max] of exp(-scale*d2) * props over the neighbours;
    out = O([x, agg]).  Gradients flow through the aggregation into props and
    d2, and through d2 into the learned coordinates (binned_select_knn_grad).
    ``space`` / ``prop`` / ``out`` may be disabled (pass ``linear=False``) to use
    the raw op: forward(coords, feats, row_splits) -> agg.
    """

    def __init__(self, in_features: int = 64, d_space: int = 4, n_prop: int = 64, k: int = 40,
                 out_features: int | None = None, weight_scale: float = 10.0,
                 reducers: tuple[str, ...] = ("mean", "max"), linear: bool = True):
        super().__init__()
        self.k = int(k)
        self.spec = AggregationSpec(weight_scale=weight_scale, reducers=reducers)
        self.linear = linear
        if linear:
            self.space = nn.Linear(in_features, d_space)
            self.prop = nn.Linear(in_features, n_prop)
            out_features = out_features or in_features
            self.out = nn.Linear(in_features + n_prop * len(reducers), out_features)

    def aggregate(self, coords: torch.Tensor, feats: torch.Tensor, row_splits):
        """Bin the learned coordinates, then ONE call of the fused op
        ``fastgraph::knn_gravnet`` (search + aggregation of its rows in sorted
        order; autograd into coords through d2 and into feats)."""
        cloud = PointCloud(coords, row_splits, check_finite=False)
        index = build_bin_index(cloud, BinningConfig(k_target=self.k))
        if feats.shape[0] != cloud.n_vertices:
            raise ShapeMismatchError(f"features cover {feats.shape[0]} vertices, "
                                     f"coords have {cloud.n_vertices}")
        rs = cloud.row_splits.device_tensor(cloud.coords.device)
        idx, d2, agg = ops.knn_gravnet(cloud.coords, rs, index.bin_idx, index.sort_order,
                                       index.bin_bounds, index.dim_mins, index.widths,
                                       index.sorted_coords, self.k, index.d_bin, index.n_bins,
                                       feats, float(self.spec.weight_scale), self.spec.codes,
                                       bool(self.spec.include_self))
        return agg, idx, d2

    def forward(self, x: torch.Tensor, row_splits, feats: torch.Tensor | None = None):
        if not self.linear:
            agg, _, _ = self.aggregate(x, feats, row_splits)
            return agg
        coords = self.space(x).float()
        props = self.prop(x).float()
        agg, _, _ = self.aggregate(coords, props, row_splits)
        return self.out(torch.cat([x, agg.to(x.dtype)], dim=1))
