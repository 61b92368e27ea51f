"""The reference's kernel-backend protocol on the B200 path.

gridknn selects its kernels through ``gridknn._kernels.get_backend(name)``
(G/_kernels/__init__.py:23-38); a backend module exposes ``NAME``,
``build_index``, ``ring_cells``, ``binned_knn`` and ``brute_knn`` with the
signatures of _binned_cy.pyx (66-67, 145, 303-308, 394-397): host numpy
arrays in, host numpy arrays out, caller-allocated outputs filled in place.
This module is that backend, executed by the CUDA library.  ``install()``
makes an unmodified gridknn front-end route ``backend="cuda"`` here:

    import gridknn
    from paper_2511_10442_b200 import backend
    backend.install(gridknn)
    idx = gridknn.build_bin_index(cloud, cfg, backend="cuda")
    nm = gridknn.binned_select_knn(cloud, idx, opts, backend="cuda")

Coordinates stay float64 on the device: the bin index is built from the
float64 values (bit-identical arrays) and the search ranks exact float64 keys
computed from them in the reference's operation order (fg_knn_fwd_f64_ws), so
indices and float64 distances equal the reference's for any finite input.
Differences a caller can observe (all within the reference's contract): rows
come back sorted by (d2, index) with ties to the lower index (the reference
leaves slot order unspecified, G/core.py:163-166); ``binned_knn`` on float64
coordinates takes k <= 120 and n_bins <= 32 (the tile kernel's buffers;
BackendUnavailableError beyond).  The host copies make this a parity tool;
timing goes through the torch ops.
"""

from __future__ import annotations

import numpy as np
import torch

from . import ops

NAME = "cuda"


def _dev():
    return torch.device("cuda", torch.cuda.current_device())


def _upload_coords(coords) -> torch.Tensor:
    c = np.ascontiguousarray(coords, dtype=np.float64)
    return torch.from_numpy(c.copy()).to(_dev())


def build_index(coords, offsets, d_bin, n_bins):
    """pyx:66-139 -> (bin_idx i64, sort_order i64, bin_bounds i64,
    dim_mins f64, widths f64), bit-identical to the reference's."""
    c = _upload_coords(coords)
    rs = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.int64)).to(c.device)
    bi, so, bb, mins, widths, _ = ops.bin_by_coordinates(c, rs, int(d_bin), int(n_bins))
    return (bi.cpu().numpy(), so.to(torch.int64).cpu().numpy(), bb.to(torch.int64).cpu().numpy(),
            mins.cpu().numpy(), widths.cpu().numpy())


def ring_cells(bin_counts, center, radius):
    """pyx:145-182: in-bounds surface cells at one Chebyshev radius, ascending.
    A host enumeration utility (the device search walks row spans instead)."""
    bc = np.asarray(bin_counts, dtype=np.int64)
    ce = np.asarray(center, dtype=np.int64)
    r = int(radius)
    axes = [np.arange(c - r, c + r + 1) for c in ce]
    grid = np.stack(np.meshgrid(*axes, indexing="ij"), axis=-1).reshape(-1, bc.size)
    surface = np.any(np.abs(grid - ce) == r, axis=1) if r > 0 else np.ones(len(grid), bool)
    inside = np.all((grid >= 0) & (grid < bc), axis=1)
    keep = grid[surface & inside]
    flat = np.zeros(len(keep), dtype=np.int64)
    for i in range(bc.size):
        flat = flat * bc[i] + keep[:, i]
    return flat


def _offsets_from_bin_idx(bin_idx, total, n):
    """The protocol hands binned_knn no row splits; recover them from the
    split-major global cell ids (split = bin_idx // total)."""
    split = np.asarray(bin_idx, dtype=np.int64) // int(total)
    n_splits = int(split.max()) + 1 if n else 1
    counts = np.bincount(split, minlength=n_splits)
    off = np.zeros(n_splits + 1, dtype=np.int64)
    np.cumsum(counts, out=off[1:])
    return off


def _run_search(c, offsets, d_bin, n_bins, dir_mask, use_dir, max_r2, use_max_r2, exhaustive,
                k, out_idx, out_d2):
    rs = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.int64)).to(c.device)
    bi, so, bb, mins, widths, sc = ops.bin_by_coordinates(c, rs, int(d_bin), int(n_bins))
    direction = None
    if use_dir:
        direction = torch.from_numpy(np.ascontiguousarray(dir_mask, dtype=np.int8)).to(c.device)
    idx, d2 = ops.binned_select_knn(c, rs, bi, so, bb, mins, widths, sc, int(k), int(d_bin),
                                    int(n_bins), direction,
                                    float(max_r2) if use_max_r2 else None, bool(exhaustive), True)
    out_idx[...] = idx.cpu().numpy()
    out_d2[...] = d2.cpu().numpy()


def binned_knn(coords, bin_idx, sort_order, bin_bounds, bin_counts, min_widths, dir_mask,
               use_dir, max_r2, use_max_r2, exhaustive, k, out_idx, out_d2, threads):
    """pyx:303-329.  The device re-derives its grid from the same coordinates
    (build_index is deterministic and bit-identical), so only the grid shape
    is taken from the arguments."""
    del sort_order, bin_bounds, min_widths, threads
    bc = np.asarray(bin_counts, dtype=np.int64)
    if bc.size == 0 or np.any(bc != bc[0]):
        raise ValueError("the cuda backend supports uniform bin counts (as build_bin_index makes)")
    n = coords.shape[0]
    offsets = _offsets_from_bin_idx(bin_idx, int(np.prod(bc)), n)
    _run_search(_upload_coords(coords), offsets, bc.size, int(bc[0]), dir_mask, use_dir, max_r2,
                use_max_r2, exhaustive, k, out_idx, out_d2)


def brute_knn(coords, offsets, dir_mask, use_dir, max_r2, use_max_r2, k, out_idx, out_d2,
              threads):
    """pyx:394-409 on the brute-force kernel (csrc/fg_verify.cu)."""
    del threads
    c = _upload_coords(coords)
    rs = torch.from_numpy(np.ascontiguousarray(offsets, dtype=np.int64)).to(c.device)
    direction = None
    if use_dir:
        direction = torch.from_numpy(np.ascontiguousarray(dir_mask, dtype=np.int8)).to(c.device)
    if int(k) > 128:  # beyond the verifier kernel's list: the binned search on one cell per split
        _run_search(c, offsets, 1, 1, dir_mask, use_dir, max_r2, use_max_r2, False, k, out_idx,
                    out_d2)
        return
    idx, d2 = ops.brute_knn(c, rs, int(k), None, direction, float(max_r2) if use_max_r2 else None)
    out_idx[...] = idx.cpu().numpy()
    out_d2[...] = d2.cpu().numpy()


def install(gridknn_module) -> None:
    """Route ``backend="cuda"`` of an imported gridknn to this module."""
    kern = gridknn_module._kernels
    orig = kern.get_backend
    if getattr(orig, "_fastgraph_b200", False):
        return
    import sys
    me = sys.modules[__name__]

    def get_backend(name=None):
        if name == NAME:
            return me
        return orig(name)

    get_backend._fastgraph_b200 = True
    kern.get_backend = get_backend
