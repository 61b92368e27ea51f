"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of the library on inputs small enough for the
tools' 10-100x slowdown.  Run through tools/sanitize.sh; no oracle involved
(correctness is the parity tests' job, this only exercises the code paths).

Paths covered: binning (K1-K4), tile search (scan + finish + redo), the
warp-per-query kernel (float64 output, direction mask, max_radius2,
exhaustive, d = 10 with d_bin = 5), the clustered-data decline path, both
backward modes (atomic, deterministic), GravNet forward/backward, the brute
verifier, index_replacer, association matrices.
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2511_10442_b200 as fg  # noqa: E402
from paper_2511_10442_b200 import ops  # noqa: E402
from paper_2511_10442_b200.datasets import generate_associations, generate_dataset  # noqa: E402


def run(coords, off, k, d_bin, **kw):
    dev = torch.device("cuda", 0)
    c = torch.from_numpy(coords.astype(np.float32)).to(dev)
    rs = torch.from_numpy(off.astype(np.int64)).to(dev)
    n_bins = fg.compute_n_bins(int(np.diff(off).max()), k, d_bin)
    bi, so, bb, mins, widths, sc = ops.bin_by_coordinates(c, rs, d_bin, n_bins)
    idx, d2 = ops.binned_select_knn(c, rs, bi, so, bb, mins, widths, sc, k, d_bin, n_bins,
                                    kw.get("direction"), kw.get("max_r2"), kw.get("exhaustive", False),
                                    kw.get("f64", False))
    up = torch.randn(idx.shape, device=dev)
    g1 = ops.binned_select_knn_grad(up, idx, c)
    g2 = ops.binned_select_knn_grad(up, idx, c, None, True)
    torch.cuda.synchronize()
    return c, rs, idx, d2


def hd_cases():
    """The high-dimensional / float64 tile kernels (fg_knn_hd.cuh)."""
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(5)
    x10, _ = generate_dataset(3000, 10, splits=1, seed=4)
    run(x10, np.array([0, 3000], np.int64), 64, 5)
    x6, _ = generate_dataset(2000, 6, splits=2, seed=8)
    off6 = np.array([0, 900, 2000], np.int64)
    run(x6, off6, 16, 5, direction=torch.from_numpy(rng.integers(0, 4, 2000).astype(np.int8)).to(dev))
    # float64 coordinates (exact keys from the float64 values), a mask and a radius
    c64 = torch.from_numpy(x6).to(dev)
    rs = torch.from_numpy(off6).to(dev)
    nb = fg.compute_n_bins(1100, 16, 5)
    bi, so, bb, mins, widths, sc = ops.bin_by_coordinates(c64, rs, 5, nb)
    ops.binned_select_knn(c64, rs, bi, so, bb, mins, widths, sc, 16, 5, nb, None, 0.05, False, True)
    ops.binned_select_knn(c64, rs, bi, so, bb, mins, widths, sc, 100, 5, nb, None, None, False, True)
    # clustered d <= 4: the gated fallback (dense cells in Morton order, block
    # boxes, cost-ordered dispatch); the second call launches it (device hint)
    xc, _ = generate_dataset(12000, 4, splits=1, seed=2, distribution="clusters")
    for _ in range(2):
        run(xc, np.array([0, 12000], np.int64), 40, 4)
    xc3, _ = generate_dataset(6000, 3, splits=2, seed=3, distribution="clusters")
    for _ in range(2):
        run(xc3, np.array([0, 2500, 6000], np.int64), 12, 3)
    # d = 4 with d_bin = 2: the hd path with the candidate filter
    run(x6[:, :4].copy(), off6, 16, 2)
    # binning with a big cell (> 4096 points: the cluster fix-up)
    xb = np.concatenate([np.full((5000, 3), 0.25), rng.random((3000, 3))])
    run(xb, np.array([0, 8000], np.int64), 8, 3)
    torch.cuda.synchronize()


def main():
    torch.manual_seed(0)
    rng = np.random.default_rng(1)
    dev = torch.device("cuda", 0)
    # tile path (uniform, d = 4, k = 16), two splits
    x, _ = generate_dataset(6000, 4, splits=2, seed=3)
    off = np.array([0, 2500, 6000], np.int64)
    c, rs, idx, d2 = run(x, off, 16, 4)
    # GravNet on the tile-path rows
    feats = torch.randn(6000, 8, device=dev, requires_grad=True)
    d2r = d2.clone().requires_grad_(True)
    agg = ops.gravnet_aggregate(feats, idx, d2r, 10.0, [0, 1], True)
    agg.sum().backward()
    # warp-per-query kernel: float64 output, mask, radius, exhaustive
    direction = torch.from_numpy(rng.integers(0, 4, 6000).astype(np.int8)).to(dev)
    run(x, off, 16, 4, f64=True, direction=direction)
    run(x, off, 16, 4, max_r2=0.01)
    run(x, off, 9, 4, exhaustive=True)
    # d = 10, d_bin = 5 (config C shape), k = 64
    x10, _ = generate_dataset(4000, 10, splits=1, seed=4)
    run(x10, np.array([0, 4000], np.int64), 64, 5)
    # clustered data: the tile kernels decline, warp-per-query takes every query
    xc, _ = generate_dataset(5000, 4, splits=1, seed=2, distribution="clusters")
    run(xc, np.array([0, 5000], np.int64), 40, 4)
    # brute-force verifier and index_replacer
    ops.brute_knn(c, rs, 16)
    lut = torch.arange(6000, device=dev, dtype=torch.int32).flip(0).contiguous()
    ops.index_replacer(idx.clone(), lut)
    # association matrices
    asso, aoff = generate_associations(3000, 2, 6, 7, 0.2)
    fg.oc_helper(fg.Associations(asso, fg.RowSplits(aoff)))
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    if "--hd" in sys.argv:
        hd_cases()
        print("sanitize hd workload done")
    else:
        main()
