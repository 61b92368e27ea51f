"""GPU parity of the lane-per-query tile path (csrc/fg_knn_tile.cuh).

The tile path serves float32-distance searches with every coordinate binned
(d <= 4, k <= 41, no mask / radius / exhaustive); whatever it cannot certify
goes to the warp-per-query kernel.  Both must give the canonical answer
(float64 d2 in the reference's operation order, lower index wins ties), so:
small cases against the CPU oracle bit for bit, full BASELINE sizes against the
warp-per-query kernel bit for bit (FG_KNN_NO_TILE), plus the redo fraction the
design promises on uniform data.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

import paper_2511_10442_b200 as fg  # noqa: E402
from paper_2511_10442_b200 import _lib, ops  # noqa: E402
from paper_2511_10442_b200.datasets import config_dataset, generate_dataset  # noqa: E402


def search(c32, off, k, flags=0, stats=False):
    n, d = c32.shape
    sizes = np.diff(off)
    nb = fg.compute_n_bins(int(sizes.max()), k, d)
    ct = torch.from_numpy(np.ascontiguousarray(c32)).cuda()
    rs = torch.from_numpy(np.asarray(off, np.int64)).cuda()
    bi, so, bb, mi, wi, sc = ops.bin_by_coordinates(ct, rs, d, nb)
    ops.set_debug_flags(flags | (_lib.FG_KNN_STATS if stats else 0))
    try:
        if stats:
            ops.knn_stats(reset=True)
        idx, d2 = ops.binned_select_knn(ct, rs, bi, so, bb, mi, wi, sc, k, d, nb, None, None,
                                        False, False)
        torch.cuda.synchronize()
        st = ops.knn_stats(reset=True) if stats else None
    finally:
        ops.set_debug_flags(0)
    return idx.cpu().numpy(), d2.cpu().numpy(), st


def assert_oracle(O, c32, off, k):
    oi, od = O.knn_canonical(c32.astype(np.float64), np.asarray(off, np.int64), k)
    gi, gd, st = search(c32, off, k, stats=True)
    bad = np.nonzero(~((gi == oi).all(1) & (gd == od.astype(np.float32)).all(1)))[0]
    assert bad.size == 0, (f"{bad.size} rows differ; first {bad[:3]}: gpu {gi[bad[0]]} "
                           f"oracle {oi[bad[0]]}")
    return st


@pytest.mark.parametrize("d,k,S,seed", [(4, 40, 1, 0), (4, 41, 2, 1), (4, 2, 1, 2), (3, 16, 3, 3),
                                        (3, 33, 1, 4), (2, 12, 2, 5), (2, 40, 1, 6), (1, 9, 1, 7),
                                        (4, 24, 4, 8)])
def test_tile_vs_oracle_uniform(oracle, d, k, S, seed):
    c, off = generate_dataset(12_000, d, S, seed, "uniform")
    st = assert_oracle(oracle, c.astype(np.float32), off, k)
    if d > 1:  # d = 1: 30 cells for 12k points -- the tile kernels decline (clustered rule)
        assert st["tiles"] > 0  # the tile path actually ran


def test_tile_ties_and_duplicates(oracle):
    # integer lattice: exact distance ties everywhere (tie rows go to the exact path)
    g = np.stack(np.meshgrid(*[np.arange(12)] * 4, indexing="ij"), -1).reshape(-1, 4)
    g = g[np.random.default_rng(0).permutation(len(g))].astype(np.float32)
    assert_oracle(oracle, g, [0, len(g)], 20)
    # coincident piles inside uniform background
    rng = np.random.default_rng(3)
    c = np.concatenate([np.full((500, 4), 0.5), rng.random((8000, 4)),
                        np.full((40, 4), 0.25)]).astype(np.float32)
    c = c[rng.permutation(len(c))]
    assert_oracle(oracle, c, [0, len(c)], 40)


def test_tile_clusters_and_tiny_splits(oracle):
    c, off = generate_dataset(20_000, 4, 2, 9, "clusters")
    assert_oracle(oracle, c.astype(np.float32), off, 40)
    c = np.random.default_rng(5).random((900, 4)).astype(np.float32)
    assert_oracle(oracle, c, np.array([0, 30, 30, 41, 900]), 40)  # splits smaller than k


@pytest.mark.parametrize("cfg", ["north_star", "E", "A"])
def test_tile_equals_warp_kernel_full_size(cfg):
    c, off, k = config_dataset(cfg)
    i0, d0, _ = search(c, off, k, flags=_lib.FG_KNN_NO_TILE)
    i1, d1, st = search(c, off, k, stats=True)
    assert np.array_equal(i0, i1)
    assert np.array_equal(d0.view(np.uint32), d1.view(np.uint32))
    if cfg != "A":  # uniform 1M / 500k: the tile path certifies >= 99.5% of rows
        assert st["tile_redo"] < 0.005 * len(c), st


# ---------------------------------------------------------------- fused search + GravNet
def _fused_and_pair(c32, off, k, F, reducers, incl, seed=0):
    n, d = c32.shape
    nb = fg.compute_n_bins(int(np.diff(off).max()), k, d)
    ct = torch.from_numpy(np.ascontiguousarray(c32)).cuda()
    rs = torch.from_numpy(np.asarray(off, np.int64)).cuda()
    bi, so, bb, mi, wi, sc = ops.bin_by_coordinates(ct, rs, d, nb)
    feats = torch.from_numpy(np.random.default_rng(seed).standard_normal((n, F))
                             .astype(np.float32)).cuda()
    i1, d1, a1 = ops.knn_gravnet(ct, rs, bi, so, bb, mi, wi, sc, k, d, nb, feats, 10.0, reducers,
                                 incl)
    i0, d0 = ops.binned_select_knn(ct, rs, bi, so, bb, mi, wi, sc, k, d, nb, None, None, False,
                                   False)
    a0 = ops.gravnet_aggregate(feats, i0, d0, 10.0, reducers, incl, so)
    torch.cuda.synchronize()
    return (i0, d0, a0), (i1, d1, a1), feats


@pytest.mark.parametrize("F,reducers,incl,dist", [(64, [0, 1], True, "uniform"),
                                                 (32, [1], False, "uniform"),
                                                 (8, [0], True, "uniform"), (65, [0, 1], True, "uniform"),
                                                 (64, [0, 1], True, "clusters")])
def test_fused_knn_gravnet_equals_ops(oracle, F, reducers, incl, dist):
    """Includes clustered data, where the tile path steps aside."""
    c, off = generate_dataset(20_000, 4, 2, 11, dist)
    (i0, d0, a0), (i1, d1, a1), feats = _fused_and_pair(c.astype(np.float32), off, 40, F, reducers,
                                                        incl)
    assert torch.equal(i0, i1) and torch.equal(d0, d1)
    np.testing.assert_allclose(a1.cpu().numpy(), a0.cpu().numpy(), rtol=1e-6, atol=1e-7)
    names = ["mean" if r == 0 else "max" for r in reducers]
    o = oracle.gravnet_aggregate(feats.cpu().numpy(), i1.cpu().numpy(), d1.cpu().numpy(), 10.0,
                                 tuple(names), incl)
    np.testing.assert_allclose(a1.cpu().numpy(), o, rtol=1e-5, atol=1e-6)


def test_fused_knn_gravnet_full_size_and_grad():
    c, off, k = config_dataset("E")
    (i0, d0, a0), (i1, d1, a1), feats = _fused_and_pair(c, off, k, 64, [0, 1], True)
    assert torch.equal(i0, i1) and torch.equal(d0, d1)
    np.testing.assert_allclose(a1.cpu().numpy(), a0.cpu().numpy(), rtol=1e-6, atol=1e-7)
    # autograd: the fused op's gradients = those of the two ops in sequence
    n, d = c.shape
    nb = fg.compute_n_bins(int(np.diff(off).max()), k, d)
    ct = torch.from_numpy(c[:50_000].copy()).cuda().requires_grad_(True)
    rs = torch.tensor([0, 50_000], dtype=torch.int64, device="cuda")
    f = feats[:50_000].clone().requires_grad_(True)
    bi, so, bb, mi, wi, sc = ops.bin_by_coordinates(ct.detach(), rs, d, nb)
    up = torch.randn(50_000, 128, device="cuda")
    _, d2f, af = ops.knn_gravnet(ct, rs, bi, so, bb, mi, wi, sc, k, d, nb, f, 10.0, [0, 1], True)
    (af * up).sum().backward()
    gc1, gf1 = ct.grad.clone(), f.grad.clone()
    ct.grad = None
    f.grad = None
    i2, d22 = ops.binned_select_knn(ct, rs, bi, so, bb, mi, wi, sc, k, d, nb, None, None, False,
                                    False)
    a2 = ops.gravnet_aggregate(f, i2, d22, 10.0, [0, 1], True, so)
    (a2 * up).sum().backward()
    torch.testing.assert_close(gf1, f.grad, rtol=1e-5, atol=1e-6)
    torch.testing.assert_close(gc1, ct.grad, rtol=1e-5, atol=1e-6)
