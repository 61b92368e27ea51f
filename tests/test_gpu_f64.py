"""Float64 coordinates -- the reference's own dtype (G/core.py:129) -- through
the device path: bin_by_coordinates from the float64 values
(fg_bin_by_coordinates_f64), the search with exact float64 keys from the
float64 coordinates (fg_knn_fwd_f64_ws: fp32 filter with a derived error bound,
csrc/fg_knn_hd.cuh), the brute verifier (fg_brute_knn_f64) and the backward on
float64 inputs.  Inputs are NOT float32-representable; the bar is the oracle
(C restatement, float64) bit for bit: bin arrays, neighbour indices, float64
distances; gradients to 1e-12 relative (order of the float64 sums differs).
"""

import numpy as np
import pytest
import torch

import paper_2511_10442_b200 as fg
from paper_2511_10442_b200 import _lib, ops
from paper_2511_10442_b200.datasets import generate_dataset

pytestmark = pytest.mark.gpu


def dev64(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def search64(c, off, k, d_bin=None, direction=None, max_r2=None, n_bins=None, stats=False):
    n, d = c.shape
    d_bin = d_bin or min(d, 5)
    nb = n_bins or fg.compute_n_bins(int(np.diff(off).max()), k, d_bin)
    ct = dev64(c)
    rs = torch.from_numpy(np.asarray(off, np.int64)).cuda()
    bi, so, bb, mi, wi, sc = ops.bin_by_coordinates(ct, rs, d_bin, nb)
    dr = None if direction is None else torch.from_numpy(direction.astype(np.int8)).cuda()
    ops.set_debug_flags(_lib.FG_KNN_STATS if stats else 0)
    try:
        if stats:
            ops.knn_stats(reset=True)
        idx, d2 = ops.binned_select_knn(ct, rs, bi, so, bb, mi, wi, sc, k, d_bin, nb, dr, max_r2,
                                        False, True)
        torch.cuda.synchronize()
        st = ops.knn_stats(reset=True) if stats else None
    finally:
        ops.set_debug_flags(0)
    return idx.cpu().numpy(), d2.cpu().numpy(), (bi, so, bb, mi, wi), nb, st


def assert_rows(gi, gd, oi, od, what):
    bad = np.nonzero(~((gi == oi).all(1) & (gd == od).all(1)))[0]
    assert bad.size == 0, f"{what}: {bad.size} rows differ; first {bad[:3]}: {gi[bad[0]]} vs {oi[bad[0]]}"


@pytest.mark.parametrize("n,d,k,splits,dist,seed", [
    (4000, 3, 16, 2, "uniform", 1), (5000, 4, 40, 1, "clusters", 2), (3000, 2, 9, 3, "uniform", 3),
    (3000, 6, 24, 1, "uniform", 4), (2500, 10, 64, 1, "uniform", 5), (800, 5, 7, 8, "uniform", 6),
    (2000, 4, 1, 2, "uniform", 7)])
def test_f64_search_vs_oracle(oracle, n, d, k, splits, dist, seed):
    c, off = generate_dataset(n, d, splits, seed, dist)  # float64, not float32-representable
    gi, gd, (bi, so, bb, mi, wi), nb, st = search64(c, off, k, stats=True)
    d_bin = min(d, 5)
    rb = oracle.build_index(c, off, d_bin, nb)
    assert np.array_equal(bi.cpu().numpy(), rb[0]) and np.array_equal(so.cpu().numpy(), rb[1])
    assert np.array_equal(bb.cpu().numpy(), rb[2])
    assert np.array_equal(mi.cpu().numpy(), rb[3]) and np.array_equal(wi.cpu().numpy(), rb[4])
    oi, od = oracle.knn_canonical(c, off, k, n_bins=nb)
    assert_rows(gi, gd, oi, od, "f64 search vs oracle")
    assert st["hd_tiles"] > 0


def test_f64_offset_far_from_origin(oracle):
    """Coordinates ~1e3 with neighbours ~1e-4 apart: float32 rounding (6e-5) is
    comparable to the distances -- the filter's error bound must absorb it."""
    rng = np.random.default_rng(11)
    c = 1000.0 + rng.random((3000, 3)) * 0.05
    off = np.array([0, 3000], np.int64)
    gi, gd, _, nb, _ = search64(c, off, 12)
    oi, od = oracle.knn_canonical(c, off, 12, n_bins=nb)
    assert_rows(gi, gd, oi, od, "far from origin")


def test_f64_masks_radius_and_duplicates(oracle):
    rng = np.random.default_rng(12)
    c, off = generate_dataset(3000, 4, 2, 13, "uniform")
    c[100:160] = c[50]                      # a block of coincident points
    mask = rng.integers(0, 4, size=3000).astype(np.int8)
    gi, gd, _, nb, _ = search64(c, off, 20, direction=mask)
    oi, od = oracle.knn_canonical(c, off, 20, n_bins=nb, dir_mask=mask)
    assert_rows(gi, gd, oi, od, "mask")
    gi, gd, _, nb, _ = search64(c, off, 20, max_r2=0.004)
    oi, od = oracle.knn_canonical(c, off, 20, n_bins=nb, max_radius2=0.004)
    assert_rows(gi, gd, oi, od, "max_radius2")
    cd = np.concatenate([c[:1000], c[:1000], c[:1000]])  # every point three times
    offd = np.array([0, 3000], np.int64)
    gi, gd, _, nb, _ = search64(cd, offd, 40)
    oi, od = oracle.knn_canonical(cd, offd, 40, n_bins=nb)
    assert_rows(gi, gd, oi, od, "triplicated points")


def test_f64_brute_and_backward(oracle):
    c, off = generate_dataset(2000, 5, 2, 21, "uniform")
    ct = dev64(c)
    rs = torch.from_numpy(off).cuda()
    bi, bd = ops.brute_knn(ct, rs, 17)
    oi, od = oracle.brute_canonical(c, off, 17)
    assert_rows(bi.cpu().numpy(), bd.cpu().numpy(), oi, od, "f64 brute")
    up = np.random.default_rng(3).standard_normal(oi.shape)  # float64 upstream
    g = ops.binned_select_knn_grad(dev64(up), torch.from_numpy(oi).cuda(), ct)
    assert g.dtype == torch.float64
    og = oracle.knn_backward(c, oi, up)
    np.testing.assert_allclose(g.cpu().numpy(), og, rtol=1e-12, atol=1e-13)


def test_f64_autograd_through_search(oracle):
    c, off = generate_dataset(1500, 3, 1, 31, "uniform")
    ct = dev64(c).requires_grad_(True)
    rs = torch.from_numpy(off).cuda()
    nb = fg.compute_n_bins(1500, 10, 3)
    bi, so, bb, mi, wi, sc = ops.bin_by_coordinates(ct.detach(), rs, 3, nb)
    idx, d2 = ops.binned_select_knn(ct, rs, bi, so, bb, mi, wi, sc, 10, 3, nb, None, None, False,
                                    True)
    w = torch.from_numpy(np.random.default_rng(4).standard_normal(d2.shape)).cuda()
    (d2 * w).sum().backward()
    og = oracle.knn_backward(c, idx.cpu().numpy(), w.cpu().numpy())
    np.testing.assert_allclose(ct.grad.cpu().numpy(), og, rtol=1e-12, atol=1e-13)
