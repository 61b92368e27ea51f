"""Event sharding: every rank's share of the 64-event batch
(config D) equals the matching row slice of the single-GPU result, bit for bit
-- neighbour ids in the global numbering, distances, bin bounds, sort order --
for 2, 4 and 8 ranks (run one after another on one GPU; the ranks share no
data, so this is exactly what each GPU computes).  Reference:
G/binning.py:159-162 (global n_bins), pkg/tests/test_acceptance.py:362-383
(no index crosses a split)."""

import numpy as np
import pytest
import torch

from paper_2511_10442_b200 import ops, sharding
from paper_2511_10442_b200.datasets import config_dataset

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def full_d():
    coords, off, k = config_dataset("D")
    c = torch.from_numpy(coords).cuda()
    rs = torch.from_numpy(off).cuda()
    nb = sharding.global_n_bins(off, k, 4)
    bi, so, bb, mins, widths, sc = ops.bin_by_coordinates(c, rs, 4, nb)
    idx, d2 = ops.binned_select_knn(c, rs, bi, so, bb, mins, widths, sc, k, 4, nb, None, None,
                                    False, False)
    return coords, off, k, nb, idx.cpu().numpy(), d2.cpu().numpy(), so.cpu().numpy(), bb.cpu().numpy()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_shards_equal_single_gpu_slices(full_d, world):
    coords, off, k, nb, idx, d2, so, bb = full_d
    cells = nb ** 4
    seen = 0
    for rank in range(world):
        res = sharding.select_knn_sharded(coords, off, k, rank, world)
        sh = res.shard
        lo, hi = sh.vertex_lo, sh.vertex_hi
        assert res.n_bins == nb
        assert np.array_equal(res.idx.cpu().numpy(), idx[lo:hi])
        assert np.array_equal(res.d2.cpu().numpy(), d2[lo:hi])
        assert np.array_equal(res.sort_order.cpu().numpy() + lo, so[lo:hi])
        assert np.array_equal(res.bin_bounds.cpu().numpy() + lo,
                              bb[sh.event_lo * cells: sh.event_hi * cells + 1])
        seen += hi - lo
    assert seen == len(coords)


def test_shard_backward_equals_single_gpu(full_d):
    """Gradients stay rank-local: a shard's backward (local ids) equals the
    single-GPU gradient's rows (events are independent)."""
    coords, off, k, nb, idx, d2, so, bb = full_d
    up = torch.from_numpy(np.random.default_rng(3).standard_normal(idx.shape).astype(np.float32)).cuda()
    c = torch.from_numpy(coords).cuda()
    full = ops.binned_select_knn_grad(up, torch.from_numpy(idx).cuda(), c.double(), None, True)
    res = sharding.select_knn_sharded(coords, off, k, 1, 4)
    lo, hi = res.shard.vertex_lo, res.shard.vertex_hi
    part = ops.binned_select_knn_grad(up[lo:hi].contiguous(), sharding.local_indices(res),
                                      c[lo:hi].double(), res.sort_order, True)
    ref = full[lo:hi].cpu().numpy()
    np.testing.assert_allclose(part.cpu().numpy(), ref, rtol=1e-9, atol=1e-12 * np.abs(ref).max())
