"""GPU parity of binned_select_knn_grad (knn_backward, G/knn.py:135-168).

Both accumulation paths (csrc/fg_grad.cu: the default compensated atomics and
the deterministic transposed kernels) are checked against the CPU oracle's
restatement of the reference's float64 np.add.at accumulation
(oracle/fg_oracle.c orc_knn_backward) on every element, at the north_star size
too; the deterministic one for bitwise run-to-run repeatability
(pkg/tests/test_knn.py:302-309).
Tolerances: float32 output 1e-5 relative (the north_star bound), float64 output
1e-9 relative, both with an absolute floor of 1e-12 x the largest element
(elements that cancel to ~0).
"""

import numpy as np
import pytest
import torch

import paper_2511_10442_b200 as fg
from paper_2511_10442_b200 import ops
from paper_2511_10442_b200.datasets import config_dataset, generate_dataset

pytestmark = pytest.mark.gpu


def knn(coords32, offsets, k):
    n, d = coords32.shape
    d_bin = min(d, 5)
    n_bins = fg.compute_n_bins(int(np.diff(offsets).max()), k, d_bin)
    c = torch.from_numpy(coords32).cuda()
    rs = torch.from_numpy(np.asarray(offsets, np.int64)).cuda()
    bi, so, bb, mins, widths, sc = ops.bin_by_coordinates(c, rs, d_bin, n_bins)
    idx, _ = ops.binned_select_knn(c, rs, bi, so, bb, mins, widths, sc, k, d_bin, n_bins,
                                   None, None, False, False)
    return c, so, idx


def upstream(n, k, seed):
    return torch.from_numpy(np.random.default_rng(seed).standard_normal((n, k))
                            .astype(np.float32)).cuda()


def check(gpu, ref, rtol):
    np.testing.assert_allclose(gpu, ref, rtol=rtol, atol=1e-12 * np.abs(ref).max())


@pytest.mark.parametrize("n,d,k,splits", [(30_000, 3, 16, 1), (50_000, 4, 40, 3),
                                          (20_000, 7, 24, 2), (20_000, 10, 64, 1),
                                          (8_000, 4, 100, 1), (5_000, 2, 2, 4)])
def test_backward_vs_oracle(oracle, n, d, k, splits):
    coords, off = generate_dataset(n, d, splits, 300 + d + k, "uniform")
    coords = coords.astype(np.float32)
    c, so, idx = knn(coords, off, k)
    up = upstream(n, k, 7 + k)
    ref = oracle.knn_backward(coords.astype(np.float64), idx.cpu().numpy(),
                              up.cpu().numpy().astype(np.float64))
    check(ops.binned_select_knn_grad(up, idx, c, so).cpu().numpy(), ref, 1e-5)
    check(ops.binned_select_knn_grad(up, idx, c.double(), so).cpu().numpy(), ref, 1e-9)
    # the deterministic path, with and without a visiting order (identity buckets)
    check(ops.binned_select_knn_grad(up, idx, c, so, True).cpu().numpy(), ref, 1e-5)
    check(ops.binned_select_knn_grad(up, idx, c.double(), so, True).cpu().numpy(), ref, 1e-9)
    check(ops.binned_select_knn_grad(up, idx, c.double(), None, True).cpu().numpy(), ref, 1e-9)


def test_backward_bitwise_deterministic():
    coords, off, k = config_dataset("B")   # clustered: buckets with very uneven in-degree
    c, so, idx = knn(coords, off, k)
    up = upstream(len(coords), k, 35)
    outs = [ops.binned_select_knn_grad(up, idx, c, so, True) for _ in range(3)]
    outs64 = [ops.binned_select_knn_grad(up, idx, c.double(), so, True) for _ in range(3)]
    torch.cuda.synchronize()
    for o in outs[1:]:
        assert torch.equal(o, outs[0])
    for o in outs64[1:]:
        assert torch.equal(o, outs64[0])


def test_backward_edge_cases(oracle):
    dev = torch.device("cuda")
    # padded slots, self in slot 0, user-made rows with -1 holes and a k = 1 matrix
    coords = np.random.default_rng(3).random((700, 3)).astype(np.float32)
    idx = np.random.default_rng(4).integers(-1, 700, size=(700, 9)).astype(np.int32)
    idx[:, 0] = np.arange(700)
    up = np.random.default_rng(5).standard_normal((700, 9)).astype(np.float32)
    ref = oracle.knn_backward(coords.astype(np.float64), idx, up.astype(np.float64))
    c = torch.from_numpy(coords).to(dev)
    for det in (False, True):
        got = ops.binned_select_knn_grad(torch.from_numpy(up).to(dev), torch.from_numpy(idx).to(dev),
                                         c.double(), None, det).cpu().numpy()
        check(got, ref, 1e-9)
    one = ops.binned_select_knn_grad(torch.ones((700, 1), device=dev),
                                     torch.arange(700, dtype=torch.int32, device=dev)[:, None], c)
    assert torch.all(one == 0)
    # a non-finite upstream poisons exactly the vertices it touches, as in float64 numpy
    up2 = up.copy()
    up2[10, 3] = np.inf
    ref2 = oracle.knn_backward(coords.astype(np.float64), idx, up2.astype(np.float64))
    for det in (False, True):
        got2 = ops.binned_select_knn_grad(torch.from_numpy(up2).to(dev), torch.from_numpy(idx).to(dev),
                                          c.double(), None, det).cpu().numpy()
        fin = np.isfinite(ref2)
        assert np.array_equal(fin, np.isfinite(got2))
        assert np.array_equal(np.isnan(ref2), np.isnan(got2))
        check(got2[fin.all(1)], ref2[fin.all(1)], 1e-9)


def test_backward_misaligned_coords(oracle):
    """A float32 view whose storage offset is not 16-byte aligned."""
    coords = np.random.default_rng(8).random((5001, 4)).astype(np.float32)
    flat = torch.from_numpy(coords.reshape(-1)).cuda()
    c = flat[1:1 + 5000 * 4].view(5000, 4)   # offset of one float
    assert c.data_ptr() % 16 != 0
    cn = c.cpu().numpy()
    _, so, idx = knn(np.ascontiguousarray(cn), [0, 5000], 12)
    up = upstream(5000, 12, 9)
    ref = oracle.knn_backward(cn.astype(np.float64), idx.cpu().numpy(), up.cpu().numpy().astype(np.float64))
    check(ops.binned_select_knn_grad(up, idx, c, so).cpu().numpy(), ref, 1e-5)
    check(ops.binned_select_knn_grad(up, idx, c, so, True).cpu().numpy(), ref, 1e-5)


def test_north_star_backward_every_element(oracle):
    """Full size (1M x 40): every gradient element against the float64 oracle."""
    coords, off, k = config_dataset("north_star")
    c, so, idx = knn(coords, off, k)
    up = upstream(len(coords), k, 13)
    ref = oracle.knn_backward(coords.astype(np.float64), idx.cpu().numpy(),
                              up.cpu().numpy().astype(np.float64))
    check(ops.binned_select_knn_grad(up, idx, c, so).cpu().numpy(), ref, 1e-5)
    check(ops.binned_select_knn_grad(up, idx, c.double(), so).cpu().numpy(), ref, 1e-9)
    g32 = ops.binned_select_knn_grad(up, idx, c, so, True)
    g32b = ops.binned_select_knn_grad(up, idx, c, so, True)
    assert torch.equal(g32, g32b)
    check(g32.cpu().numpy(), ref, 1e-5)
    check(ops.binned_select_knn_grad(up, idx, c.double(), so, True).cpu().numpy(), ref, 1e-9)


def test_reference_api_backward_deterministic():
    """knn_backward (G/knn.py:135) through the reference-shaped API: repeatable."""
    from paper_2511_10442_b200 import knn as K
    from paper_2511_10442_b200.binning import BinningConfig, build_bin_index
    from paper_2511_10442_b200.core import PointCloud, RowSplits
    coords, off = generate_dataset(20_000, 3, 2, 35, "uniform")
    pc = PointCloud(torch.from_numpy(coords.astype(np.float32)).cuda(), RowSplits(off))
    index = build_bin_index(pc, BinningConfig(k_target=6))
    nm = K.binned_select_knn(pc, index, K.KnnOptions(k=6))
    up = np.random.default_rng(35).standard_normal(tuple(nm.dist2.shape))
    g1 = K.knn_backward(pc, nm, up)
    g2 = K.knn_backward(pc, nm, up)
    assert torch.equal(g1, g2)
