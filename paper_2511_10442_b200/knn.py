"""Exact kNN front-end on the device (mirror of G/knn.py:1-180).

``binned_select_knn`` / ``brute_force_knn`` / ``knn_backward`` /
``knn_with_grad`` keep the reference's names, options and errors; the work is
done by the fastgraph:: ops (CUDA only).  Output rows are sorted by
(float64 d2, original index): slot 0 = self, ties -> lower index, padding
(-1, 0) -- the canonical instance of the reference's unordered contract.

``binned_select_knn`` is differentiable w.r.t. ``cloud.coords`` (autograd
runs fastgraph::binned_select_knn_grad).
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import ops
from .binning import BinIndex, BinningConfig, build_bin_index
from .core import DirectionMask, NeighborMatrix, PointCloud
from .errors import BadKError, IndexMismatchError, ShapeMismatchError

MAX_K = 960


@dataclass(frozen=True)
class KnnOptions:
    """G/knn.py:34-45: k counts the vertex itself; max_radius2 drops
    candidates with d2 strictly greater than the cutoff."""

    k: int
    mask: DirectionMask | None = None
    max_radius2: float | None = None


def _check_options(cloud: PointCloud, opts: KnnOptions):
    """G/knn.py:48-58."""
    if not isinstance(opts.k, int) or isinstance(opts.k, bool) or opts.k < 1:
        try:
            import numpy as np
            ok = isinstance(opts.k, np.integer) and opts.k >= 1
        except Exception:  # pragma: no cover
            ok = False
        if not ok:
            raise BadKError(f"k must be a positive integer, got {opts.k!r}")
    if int(opts.k) > MAX_K:
        raise BadKError(f"k must be <= {MAX_K}, got {opts.k}")
    if cloud.n_vertices >= 2 ** 31:
        raise ShapeMismatchError("vertex count exceeds int32 neighbour indices")
    if opts.mask is not None and opts.mask.dir.numel() != cloud.n_vertices:
        raise ShapeMismatchError(
            f"mask covers {opts.mask.dir.numel()} vertices, cloud has {cloud.n_vertices}")
    if opts.max_radius2 is not None and not (opts.max_radius2 >= 0.0):
        raise BadKError(f"max_radius2 must be >= 0, got {opts.max_radius2!r}")


def _direction(cloud: PointCloud, opts: KnnOptions):
    if opts.mask is not None and opts.mask.enabled:
        return opts.mask.dir.to(cloud.coords.device)
    return None


def _search(cloud: PointCloud, index: BinIndex, opts: KnnOptions, exhaustive: bool,
            d2_f64: bool) -> NeighborMatrix:
    rs = cloud.row_splits.device_tensor(cloud.coords.device)
    idx, d2 = ops.binned_select_knn(
        cloud.coords, rs, index.bin_idx, index.sort_order, index.bin_bounds, index.dim_mins,
        index.widths, index.sorted_coords, int(opts.k), index.d_bin, index.n_bins,
        _direction(cloud, opts), None if opts.max_radius2 is None else float(opts.max_radius2),
        bool(exhaustive), bool(d2_f64))
    return NeighborMatrix(idx, d2)


def binned_select_knn(cloud: PointCloud, index: BinIndex, opts: KnnOptions, *,
                      exhaustive_rings: bool = False, d2_f64: bool = False) -> NeighborMatrix:
    """Exact kNN over the bin index (G/knn.py:82-115).  ``d2_f64`` returns the
    bit-exact float64 distances of the reference instead of float32."""
    _check_options(cloud, opts)
    if index.n_vertices != cloud.n_vertices:
        raise IndexMismatchError(
            f"index built for {index.n_vertices} vertices, cloud has {cloud.n_vertices}")
    if index.row_splits != cloud.row_splits:
        raise IndexMismatchError("index row splits differ from the cloud's")
    if index.d_bin > cloud.n_coords:
        raise IndexMismatchError(f"index bins {index.d_bin} dims, cloud has {cloud.n_coords}")
    return _search(cloud, index, opts, exhaustive_rings, d2_f64)


def brute_force_knn(cloud: PointCloud, opts: KnnOptions, *, d2_f64: bool = False) -> NeighborMatrix:
    """Every vertex of the split is a candidate (G/knn.py:118-132): the
    brute-force kernel (csrc/fg_verify.cu), independent of the binned search;
    canonical (d2, index) rows, float64 distances (rounded to float32 unless
    ``d2_f64``)."""
    _check_options(cloud, opts)
    rs = cloud.row_splits.device_tensor(cloud.coords.device)
    idx, d2 = ops.brute_knn(cloud.coords.detach(), rs, int(opts.k), None, _direction(cloud, opts),
                            None if opts.max_radius2 is None else float(opts.max_radius2))
    return NeighborMatrix(idx, d2 if d2_f64 else d2.to(torch.float32))


def knn_backward(cloud: PointCloud, neighbors: NeighborMatrix, upstream) -> torch.Tensor:
    """G/knn.py:135-168: d(sum g*d2)/d coords.  Terms exact in float64, the
    upstream rounded to float32; bitwise repeatable like the reference's
    fixed-order accumulation (the deterministic transposed kernel) up to 2^23
    vertices, the atomic kernel above that."""
    up = upstream if isinstance(upstream, torch.Tensor) else torch.as_tensor(upstream)
    up = up.to(cloud.coords.device)
    if tuple(up.shape) != tuple(neighbors.dist2.shape):
        raise ShapeMismatchError(f"upstream shape {tuple(up.shape)} != neighbour shape "
                                 f"{tuple(neighbors.dist2.shape)}")
    if neighbors.n_vertices != cloud.n_vertices:
        raise ShapeMismatchError(f"neighbours cover {neighbors.n_vertices} vertices, "
                                 f"cloud has {cloud.n_vertices}")
    n, k = neighbors.indices.shape
    det = (n <= (1 << 23) and n * k < (1 << 32) and cloud.coords.dtype == torch.float32
           and up.dtype != torch.float64)
    return ops.binned_select_knn_grad(up, neighbors.indices, cloud.coords.detach(), None, det)


def knn_with_grad(cloud: PointCloud, index: BinIndex, opts: KnnOptions):
    """G/knn.py:171-180."""
    neighbors = binned_select_knn(cloud, index, opts)

    def grad_fn(upstream):
        return knn_backward(cloud, neighbors, upstream)

    return neighbors, grad_fn


def select_knn(coords: torch.Tensor, row_splits, K: int, *, direction=None,
               max_radius2: float | None = None, n_bins: int | None = None,
               d_bin: int | None = None, return_order: bool = False):
    """One-call FastGraph-style API: bin + search, differentiable w.r.t.
    ``coords``.  Returns (idx int32 [N, K], d2 float32 [N, K]), plus the bin
    index's sort_order (a spatially coherent row order for follow-up kernels)
    when ``return_order``."""
    cloud = PointCloud(coords, row_splits, check_finite=False)
    cfg = BinningConfig(k_target=int(K), d_bin=d_bin, n_bins=n_bins)
    index = build_bin_index(cloud, cfg)
    mask = None if direction is None else DirectionMask(direction)
    nm = binned_select_knn(cloud, index, KnnOptions(k=int(K), mask=mask, max_radius2=max_radius2))
    if return_order:
        return nm.indices, nm.dist2, index.sort_order
    return nm.indices, nm.dist2
