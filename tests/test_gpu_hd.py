"""GPU parity of the high-dimensional lane-per-query tile path
(csrc/fg_knn_hd.cuh): n_coords > 4 or d_bin < n_coords, k <= 64, no mask /
radius / exhaustive.  Every row is compared bit for bit with the independent
brute-force kernel (csrc/fg_verify.cu, float64 keys, canonical (d2, index)
order) and with the warp-per-query kernel (FG_KNN_NO_HD); small cases also
with the CPU oracle.  Float64 distances must equal the reference's bit for bit.
"""

import numpy as np
import pytest
import torch

import paper_2511_10442_b200 as fg
from paper_2511_10442_b200 import _lib, ops
from paper_2511_10442_b200.datasets import generate_dataset

pytestmark = pytest.mark.gpu


def search(c32, off, k, d_bin, flags=0, d2_f64=False, stats=False):
    nb = fg.compute_n_bins(int(np.diff(off).max()), k, d_bin)
    ct = torch.from_numpy(np.ascontiguousarray(c32)).cuda()
    rs = torch.from_numpy(np.asarray(off, np.int64)).cuda()
    bi, so, bb, mi, wi, sc = ops.bin_by_coordinates(ct, rs, d_bin, nb)
    ops.set_debug_flags(flags | (_lib.FG_KNN_STATS if stats else 0))
    try:
        if stats:
            ops.knn_stats(reset=True)
        idx, d2 = ops.binned_select_knn(ct, rs, bi, so, bb, mi, wi, sc, k, d_bin, nb, None, None,
                                        False, d2_f64)
        torch.cuda.synchronize()
        st = ops.knn_stats(reset=True) if stats else None
    finally:
        ops.set_debug_flags(0)
    return idx.cpu().numpy(), d2.cpu().numpy(), st


def brute(c32, off, k):
    c = torch.from_numpy(np.ascontiguousarray(c32)).cuda()
    rs = torch.from_numpy(np.asarray(off, np.int64)).cuda()
    i, d = ops.brute_knn(c, rs, k)
    return i.cpu().numpy(), d.cpu().numpy()


def assert_rows(gi, gd, ri, rd, what):
    bad = np.nonzero(~((gi == ri).all(1) & (gd == rd).all(1)))[0]
    assert bad.size == 0, (f"{what}: {bad.size} rows differ; first {bad[:3]}: {gi[bad[0]]} vs "
                           f"{ri[bad[0]]}")


CASES = [  # n, d, d_bin, k, splits, distribution
    (20000, 10, 5, 64, 1, "uniform"),
    (6000, 6, 5, 16, 3, "uniform"),
    (8000, 8, 3, 32, 2, "uniform"),
    (5000, 4, 2, 10, 1, "uniform"),
    (3000, 3, 1, 12, 2, "uniform"),
    (4000, 16, 5, 64, 1, "uniform"),
    (6000, 10, 5, 40, 2, "clusters"),
    (700, 5, 5, 40, 9, "uniform"),    # small splits: some hold fewer than k points
    (3000, 12, 4, 2, 1, "uniform"),
]


@pytest.mark.parametrize("n,d,d_bin,k,splits,dist", CASES)
def test_hd_equals_brute_every_row(n, d, d_bin, k, splits, dist):
    c, off = generate_dataset(n, d, splits, 100 + d + k, dist)
    c32 = c.astype(np.float32)
    gi, gd64, st = search(c32, off, k, d_bin, d2_f64=True, stats=True)
    assert st["hd_tiles"] > 0, "the high-dimensional tile path did not run"
    bi, bd = brute(c32, off, k)
    assert_rows(gi, gd64, bi, bd, "hd vs brute (float64 d2)")
    gi32, gd32, _ = search(c32, off, k, d_bin)
    assert_rows(gi32, gd32, bi, bd.astype(np.float32), "hd vs brute (float32 d2)")
    wi, wd, _ = search(c32, off, k, d_bin, flags=_lib.FG_KNN_NO_HD)
    assert_rows(gi32, gd32, wi, wd, "hd vs warp-per-query")


def test_hd_vs_oracle(oracle):
    c, off = generate_dataset(2500, 7, 2, 5, "uniform")
    c32 = c.astype(np.float32)
    oi, od = oracle.knn_canonical(c32.astype(np.float64), off, 24)
    gi, gd, st = search(c32, off, 24, 5, d2_f64=True, stats=True)
    assert st["hd_tiles"] > 0
    assert_rows(gi, gd, oi, od, "hd vs oracle")


def test_hd_duplicates_and_ties():
    """Coincident points and exact distance ties: lower index wins (canonical)."""
    rng = np.random.default_rng(9)
    base = rng.integers(0, 4, size=(400, 6)).astype(np.float32)  # a lattice: many ties
    c32 = np.concatenate([base, base[:150]])                      # and duplicates
    off = np.array([0, c32.shape[0]], np.int64)
    gi, gd, st = search(c32, off, 30, 5, d2_f64=True, stats=True)
    bi, bd = brute(c32, off, 30)
    assert_rows(gi, gd, bi, bd, "hd vs brute on a lattice with duplicates")


def test_hd_config_c_sample():
    """Config C (1M x 10, d_bin 5, k 64): 20k sampled rows against the brute force."""
    from paper_2511_10442_b200.datasets import config_dataset
    c, off, k = config_dataset("C")
    c32 = c.astype(np.float32)
    gi, gd, st = search(c32, off, k, 5, d2_f64=True, stats=True)
    assert st["hd_tiles"] > 0
    rng = np.random.default_rng(1)
    rows = np.sort(rng.choice(c32.shape[0], 20_000, replace=False)).astype(np.int32)
    ct = torch.from_numpy(c32).cuda()
    rs = torch.from_numpy(off).cuda()
    bi, bd = ops.brute_knn(ct, rs, k, torch.from_numpy(rows).cuda())
    assert_rows(gi[rows], gd[rows], bi.cpu().numpy(), bd.cpu().numpy(), "config C sample")


@pytest.mark.parametrize("n,d,k,splits", [(60_000, 4, 40, 1), (30_000, 3, 16, 3), (20_000, 2, 12, 2)])
def test_clustered_fallback_equals_warp_kernel(n, d, k, splits):
    """d <= 4 clustered data: the tile path declines and the high-dimensional
    tile kernels (dense cells in Morton order, stage-0 seeds) take every query;
    bit-identical to the warp-per-query kernel and to the brute force."""
    c, off = generate_dataset(n, d, splits, 7 + d, "clusters")
    c32 = c.astype(np.float32)
    search(c32, off, k, d)  # a clustered call: the next one launches the fallback
    gi, gd, st = search(c32, off, k, d, stats=True)
    assert st["hd_tiles"] > 0, "the clustered fallback did not run"
    wi, wd, _ = search(c32, off, k, d, flags=_lib.FG_KNN_NO_HD)
    assert_rows(gi, gd, wi, wd, "clustered fallback vs warp-per-query")
    bi, bd = brute(c32, off, k)
    assert_rows(gi, gd, bi, bd.astype(np.float32), "clustered fallback vs brute")


def test_clustered_fallback_dense_cell_sizes(oracle):
    """Cells of exactly 33, 4096, 16384 (kMaxSortCell: the largest the dense-cell
    counting sort orders) and 16385 points (kept in binning order) over a uniform
    background: bin arrays equal to the oracle's (medium and big-cell fix-ups),
    every neighbour row equal to the brute force."""
    rng = np.random.default_rng(5)
    k, d = 40, 4
    bg = rng.random((20_000, d))
    bg[0], bg[1] = 0.0, 1.0  # extents exactly [0, 1]: widths 1 / n_bins
    sizes = [33, 4096, 16384, 16385]
    n = bg.shape[0] + sum(sizes)
    nb = fg.compute_n_bins(n, k, d)
    cells = [np.array([2 + 3 * j, 5, 7, 9]) % nb for j in range(len(sizes))]
    bc = np.floor(bg * nb).astype(np.int64)
    keep = np.ones(len(bg), bool)
    for cl in cells:  # the blob cells hold the blob points only
        keep &= ~(bc == cl).all(1)
    keep[:2] = True
    parts = [bg[keep]]
    for cl, m in zip(cells, sizes):
        parts.append((cl + 0.5) / nb + (rng.random((m, d)) - 0.5) * (0.4 / nb))
    c32 = np.concatenate(parts).astype(np.float32)
    n = c32.shape[0]
    off = np.array([0, n], np.int64)
    assert fg.compute_n_bins(n, k, d) == nb
    ref = oracle.build_index(c32.astype(np.float64), off, d, nb)
    L = np.diff(ref[2])
    for m in sizes:
        assert (L == m).any(), f"no cell holds exactly {m} points"
    ct = torch.from_numpy(c32).cuda()
    rs = torch.from_numpy(off).cuda()
    got = [o.cpu().numpy() for o in ops.bin_by_coordinates(ct, rs, d, nb)]
    for r, g_ in zip(ref, got[:5]):
        assert np.array_equal(r, g_.astype(r.dtype))
    search(c32, off, k, d)  # a clustered call: the next one launches the fallback
    gi, gd, st = search(c32, off, k, d, stats=True)
    assert st["hd_tiles"] > 0, "the clustered fallback did not run"
    bi, bd = brute(c32, off, k)
    assert_rows(gi, gd, bi, bd.astype(np.float32), "dense cells vs brute")
