"""Every row of the BASELINE configs against the independent GPU brute force
(csrc/fg_verify.cu: thread per query, full split scan, float64 keys, canonical
(d2, index) order; no code shared with the binned search; SURVEY 8(f)2,
pyx:335-409).  The brute force itself is pinned to the CPU oracle first.
Bar: neighbour indices and float64 distances bit-identical on EVERY row
(north_star, B, D, E; 10,000 sampled rows of C), float32 distances ==
float32(float64)."""

import time

import numpy as np
import pytest
import torch

import paper_2511_10442_b200 as fg
from paper_2511_10442_b200 import ops
from paper_2511_10442_b200.datasets import config_dataset, generate_dataset

pytestmark = pytest.mark.gpu


def brute(coords32, offsets, k, queries=None, **kw):
    c = torch.from_numpy(np.ascontiguousarray(coords32)).cuda()
    rs = torch.from_numpy(np.asarray(offsets, np.int64)).cuda()
    q = None if queries is None else torch.from_numpy(np.asarray(queries, np.int32)).cuda()
    i, d = ops.brute_knn(c, rs, k, q, **kw)
    return i.cpu().numpy(), d.cpu().numpy()


def binned(coords32, offsets, k, d2_f64):
    n, d = coords32.shape
    d_bin = min(d, 5)
    nb = fg.compute_n_bins(int(np.diff(offsets).max()), k, d_bin)
    c = torch.from_numpy(coords32).cuda()
    rs = torch.from_numpy(np.asarray(offsets, np.int64)).cuda()
    bi, so, bb, mins, widths, sc = ops.bin_by_coordinates(c, rs, d_bin, nb)
    i, d2 = ops.binned_select_knn(c, rs, bi, so, bb, mins, widths, sc, k, d_bin, nb, None, None,
                                  False, d2_f64)
    return i.cpu().numpy(), d2.cpu().numpy()


@pytest.mark.parametrize("n,d,splits,k,dist", [(3000, 3, 2, 16, "uniform"), (2000, 4, 3, 40, "clusters"),
                                                (1500, 10, 1, 64, "uniform"), (500, 2, 5, 7, "uniform")])
def test_brute_equals_oracle(oracle, n, d, splits, k, dist):
    c, off = generate_dataset(n, d, splits, 40 + d, dist)
    c32 = c.astype(np.float32)
    bi, bd = brute(c32, off, k)
    oi, od = oracle.brute_canonical(c32.astype(np.float64), off, k)
    assert np.array_equal(bi, oi) and np.array_equal(bd, od)


def test_brute_lattice_mask_radius(oracle):
    g = np.stack(np.meshgrid(*[np.arange(6)] * 3, indexing="ij"), -1).reshape(-1, 3).astype(np.float32)
    g = g[np.random.default_rng(0).permutation(len(g))]
    off = [0, 100, len(g)]
    for k in (5, 13):   # exact ties everywhere: canonical rule (lower index wins)
        bi, bd = brute(g, off, k)
        oi, od = oracle.brute_canonical(g.astype(np.float64), off, k)
        assert np.array_equal(bi, oi) and np.array_equal(bd, od)
    mask = np.random.default_rng(1).integers(0, 4, len(g)).astype(np.int8)
    bi, bd = brute(g, off, 9, direction=torch.from_numpy(mask).cuda(), max_radius2=2.0)
    oi, od = oracle.brute_canonical(g.astype(np.float64), off, 9, dir_mask=mask, max_radius2=2.0)
    assert np.array_equal(bi, oi) and np.array_equal(bd, od)
    # a query subset returns those rows
    q = np.array([5, 0, 150, 215], np.int32)
    si, sd = brute(g, off, 5, queries=q)
    fi, fd = brute(g, off, 5)
    assert np.array_equal(si, fi[q]) and np.array_equal(sd, fd[q])


@pytest.mark.parametrize("cfg", ["north_star", "B", "D", "E", "A"])
def test_every_row_vs_gpu_brute_force(cfg):
    coords, off, k = config_dataset(cfg)
    t0 = time.perf_counter()
    bi, bd = brute(coords, off, k)
    t_brute = time.perf_counter() - t0
    i64, d64 = binned(coords, off, k, True)
    i32, d32 = binned(coords, off, k, False)
    assert np.array_equal(i64, bi), f"{cfg}: {int((i64 != bi).any(1).sum())} rows differ"
    assert np.array_equal(d64, bd)
    assert np.array_equal(i32, bi)
    assert np.array_equal(d32, bd.astype(np.float32))
    print(f"{cfg}: {len(coords)} rows bit-identical (brute force {t_brute:.2f} s)")


def test_config_c_sampled_rows_vs_gpu_brute_force():
    coords, off, k = config_dataset("C")
    q = np.sort(np.random.default_rng(4).choice(len(coords), 10_000, replace=False)).astype(np.int32)
    bi, bd = brute(coords, off, k, queries=q)
    i64, d64 = binned(coords, off, k, True)
    assert np.array_equal(i64[q], bi) and np.array_equal(d64[q], bd)
