"""GPU parity at BASELINE.json sizes and through the reference backend protocol.

At full size the CPU oracle cannot run every row in seconds, so a random sample
of rows is checked exactly: the oracle runs with a DirectionMask that makes only
the sampled rows queries (roles 3) while every vertex stays a candidate (role 0)
-- the sampled rows' answers are then exactly those of the unmasked problem.
Size-independent properties (self slot, sorted rows, split isolation, gradient
sum rule) are checked on every row.
"""

import numpy as np
import pytest
import torch

import paper_2511_10442_b200 as fg
from paper_2511_10442_b200 import backend, ops
from paper_2511_10442_b200.datasets import config_dataset, generate_dataset

pytestmark = pytest.mark.gpu


def run(coords32, offsets, k, n_bins=None):
    n, d = coords32.shape
    d_bin = min(d, 5)
    if n_bins is None:
        n_bins = fg.compute_n_bins(int(np.diff(offsets).max()), k, d_bin)
    c = torch.from_numpy(coords32).cuda()
    rs = torch.from_numpy(np.asarray(offsets, np.int64)).cuda()
    bi, so, bb, mins, widths, sc = ops.bin_by_coordinates(c, rs, d_bin, n_bins)
    idx, d2 = ops.binned_select_knn(c, rs, bi, so, bb, mins, widths, sc, k, d_bin, n_bins, None,
                                    None, False, True)
    return c, rs, so, idx, d2


def sampled_oracle(oracle, coords32, offsets, k, rows):
    mask = np.zeros(len(coords32), np.int8)
    mask[rows] = 3
    oi, od = oracle.knn_canonical(coords32.astype(np.float64), offsets, k, dir_mask=mask)
    return oi[rows], od[rows]


def check_structure(idx, d2, offsets):
    n, k = idx.shape
    assert np.array_equal(idx[:, 0], np.arange(n))
    assert np.all(d2[:, 0] == 0)
    valid = idx[:, 1:] >= 0
    dd = np.where(valid, d2[:, 1:], np.inf)
    assert np.all(np.diff(dd, axis=1) >= 0)            # rows sorted by distance
    split = np.searchsorted(offsets, np.arange(n), side="right") - 1
    nb_split = np.searchsorted(offsets, np.where(valid, idx[:, 1:], 0), side="right") - 1
    assert np.all(np.where(valid, nb_split == split[:, None], True))  # no cross-split index


@pytest.mark.parametrize("cfg,sample", [("north_star", 3000), ("B", 1500), ("E", 2000),
                                        ("A", 10_000), ("D", 3000)])
def test_baseline_config_sampled_parity(oracle, cfg, sample):
    coords, off, k = config_dataset(cfg)
    _, _, _, idx, d2 = run(coords, off, k)
    idx = idx.cpu().numpy()
    d2 = d2.cpu().numpy()
    check_structure(idx, d2, off)
    if cfg == "D":  # events are independent: check rows of the first two events
        n2 = int(off[2])
        rows = np.random.default_rng(11).choice(n2, size=sample, replace=False)
        oi, od = sampled_oracle(oracle, coords[:n2], off[:3], k, rows)
    else:
        rows = np.random.default_rng(11).choice(len(coords), size=min(sample, len(coords)), replace=False)
        oi, od = sampled_oracle(oracle, coords, off, k, rows)
    bad = np.nonzero(~((idx[rows] == oi).all(1) & (d2[rows] == od).all(1)))[0]
    assert bad.size == 0, f"{cfg}: {bad.size} sampled rows differ (first row {rows[bad[0]]})"


def test_config_c_sampled_parity(oracle):
    """d=10, k=64: only 5 of 10 dims are binned (slow oracle: few rows)."""
    coords, off, k = config_dataset("C")
    _, _, _, idx, d2 = run(coords, off, k)
    rows = np.random.default_rng(12).choice(len(coords), size=60, replace=False)
    oi, od = sampled_oracle(oracle, coords, off, k, rows)
    assert np.array_equal(idx.cpu().numpy()[rows], oi)
    assert np.array_equal(d2.cpu().numpy()[rows], od)


def test_gravnet_config_e_sample(oracle):
    coords, off, k = config_dataset("E")
    _, _, _, idx, d2 = run(coords, off, k)
    feats = torch.randn(len(coords), 64, device="cuda", generator=torch.Generator("cuda").manual_seed(1))
    d2f = d2.float()
    out = ops.gravnet_aggregate(feats, idx, d2f, 10.0, [0, 1], True)
    up = torch.randn(out.shape, device="cuda", generator=torch.Generator("cuda").manual_seed(2))
    gf, gd = ops.gravnet_aggregate_grad(up, feats, idx, d2f, 10.0, [0, 1], True)
    fi, ii, di = feats.cpu().numpy(), idx.cpu().numpy(), d2f.cpu().numpy()
    o = oracle.gravnet_aggregate(fi, ii, di, 10.0)
    np.testing.assert_allclose(out.cpu().numpy(), o, rtol=1e-5, atol=1e-6)
    # gradients on the whole problem against the oracle (float64)
    ogf, ogd = oracle.gravnet_aggregate_backward(fi, ii, di, up.cpu().numpy(), 10.0)
    np.testing.assert_allclose(gd.cpu().numpy(), ogd, rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(gf.cpu().numpy(), ogf, rtol=1e-5, atol=1e-6)


def test_backend_protocol_against_oracle(oracle):
    """The reference-protocol adapter (host numpy in/out, as gridknn calls it)."""
    coords, off = generate_dataset(3000, 3, splits=2, seed=21)
    c64 = coords.astype(np.float32).astype(np.float64)
    nb = fg.compute_n_bins(1500, 9, 3)
    got = backend.build_index(c64, off, 3, nb)
    ref = oracle.build_index(c64, off, 3, nb)
    for g, r in zip(got, ref):
        assert g.dtype == r.dtype and np.array_equal(g, r)
    bi, so, bb, mins, widths = got
    oi = np.empty((3000, 9), np.int32)
    od = np.empty((3000, 9), np.float64)
    backend.binned_knn(c64, bi, so, bb, np.full(3, nb, np.int64), widths.min(axis=1), np.zeros(1, np.int8),
                       False, 0.0, False, False, 9, oi, od, 0)
    ci, cd = oracle.knn_canonical(c64, off, 9)
    assert np.array_equal(oi, ci) and np.array_equal(od, cd)
    mask = np.random.default_rng(5).integers(0, 4, 3000).astype(np.int8)
    backend.brute_knn(c64, off, mask, True, 0.01, True, 9, oi, od, 0)
    ci, cd = oracle.brute_canonical(c64, off, 9, dir_mask=mask, max_radius2=0.01)
    assert np.array_equal(oi, ci) and np.array_equal(od, cd)
