"""GPU parity: the CUDA path (through the fastgraph:: ops / C ABI) against the
CPU oracle and the reference's golden vectors.

Bars (BASELINE.json north_star): bin arrays bit-identical to the reference's
build_index; neighbour indices bit-exact under the canonical rule (float64 d2,
lower index wins ties) -- and equal to the reference itself on every row whose
k-th/(k+1)-th distances are not tied; float64 distances bit-identical,
float32 distances == float32(reference d2); gradients within 1e-5 relative.
"""

import numpy as np
import pytest
import torch

from conftest import GOLDEN_CASES, golden_case

pytestmark = pytest.mark.gpu

import paper_2511_10442_b200 as fg  # noqa: E402
from paper_2511_10442_b200 import ops  # noqa: E402


def dev():
    return torch.device("cuda", 0)


def t(a, dtype=None):
    x = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        x = x.to(dtype)
    return x.to(dev())


def run_bin(coords32, offsets, d_bin, n_bins):
    out = ops.bin_by_coordinates(t(coords32, torch.float32), t(offsets, torch.int64), d_bin, n_bins)
    torch.cuda.synchronize()
    return [o.cpu().numpy() for o in out]


def run_knn(coords32, offsets, k, *, d_bin=None, n_bins=None, mask=None, max_r2=None,
            exhaustive=False, f64=True):
    c = np.ascontiguousarray(coords32, dtype=np.float32)
    n, n_c = c.shape
    off = np.asarray(offsets, dtype=np.int64)
    if d_bin is None:
        d_bin = min(n_c, 5)
    if n_bins is None:
        sizes = np.diff(off)
        n_bins = fg.compute_n_bins(int(sizes.max()) if sizes.size else 0, k, d_bin)
    ct = t(c)
    rs = t(off)
    bi, so, bb, mins, widths, sc = ops.bin_by_coordinates(ct, rs, d_bin, n_bins)
    direction = None if mask is None else t(mask, torch.int8)
    idx, d2 = ops.binned_select_knn(ct, rs, bi, so, bb, mins, widths, sc, k, d_bin, n_bins,
                                    direction, max_r2, exhaustive, f64)
    torch.cuda.synchronize()
    return idx.cpu().numpy(), d2.cpu().numpy()


def ref_sorted(idx, d2):
    """G/harness/verify.py:125-133: valid slots (self included) by (d2, idx)."""
    oi = np.full_like(idx, -1)
    od = np.zeros_like(d2)
    for v in range(idx.shape[0]):
        keep = idx[v] >= 0
        ri, rd = idx[v][keep], d2[v][keep]
        o = np.lexsort((ri, rd))
        oi[v, :ri.size] = ri[o]
        od[v, :ri.size] = rd[o]
    return oi, od


def assert_canonical(O, coords32, offsets, k, **kw):
    """GPU == oracle canonical, bitwise, float64 and float32 outputs."""
    c64 = np.asarray(coords32, dtype=np.float32).astype(np.float64)
    oi, od = O.knn_canonical(c64, offsets, k, dir_mask=kw.get("mask"),
                             max_radius2=kw.get("max_r2"))
    gi, gd = run_knn(coords32, offsets, k, **kw)
    bad = np.nonzero(~((gi == oi).all(1) & (gd == od).all(1)))[0]
    assert bad.size == 0, (f"{bad.size} rows differ; first {bad[:5]}: gpu {gi[bad[0]]} "
                           f"{gd[bad[0]]} oracle {oi[bad[0]]} {od[bad[0]]}")
    gi32, gd32 = run_knn(coords32, offsets, k, f64=False, **kw)
    assert np.array_equal(gi32, oi)
    assert np.array_equal(gd32, od.astype(np.float32))
    return gi, gd


# ---------------------------------------------------------------- binning
@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_bin_index_bitwise_vs_reference(golden, name):
    g = golden_case(golden, name)
    bi, so, bb, mins, widths, sc = run_bin(g["coords"], g["row_splits"], g["d_bin"], g["n_bins"])
    assert np.array_equal(bi, g["bin_idx"])
    assert np.array_equal(so.astype(np.int64), g["sort_order"])
    assert np.array_equal(bb.astype(np.int64), g["bin_bounds"])
    assert np.array_equal(mins, g["dim_mins"])
    assert np.array_equal(widths, g["widths"])
    n, n_c = g["coords"].shape
    assert np.array_equal(sc[:, :n_c], g["coords"][g["sort_order"]])
    assert np.all(sc[:, n_c:] == 0)


def test_bin_top_edge_and_degenerate_width():
    # T/test_binning.py:124-140
    c = np.array([[0.0, 0.0], [1.0, 1.0], [0.5, 0.5], [1.0, 0.0]], np.float32)
    bi, *_ = run_bin(c, [0, 4], 2, 6)
    assert bi[1] == 35 and bi.min() >= 0 and bi.max() < 36
    c = np.zeros((10, 2), np.float32)
    c[:, 0] = np.linspace(0.0, 1.0, 10)
    bi, so, bb, mins, widths, _ = run_bin(c, [0, 10], 2, 5)
    assert widths[0, 1] == 1.0 and np.all(bi >= 0)


def test_bin_empty_splits_and_huge_cells(oracle):
    rng = np.random.default_rng(7)
    parts = [rng.random((300, 3)), np.zeros((0, 3)), np.full((6000, 3), 0.25),
             rng.random((5000, 3)) * 0.001, np.zeros((0, 3)), rng.random((50, 3))]
    c = np.concatenate(parts).astype(np.float32)
    off = np.cumsum([0] + [len(p) for p in parts])
    ref = oracle.build_index(c.astype(np.float64), off, 3, 7)
    got = run_bin(c, off, 3, 7)
    for r, g_ in zip(ref, got[:5]):
        assert np.array_equal(r, g_.astype(r.dtype))


def test_bin_clustered_config_b_vs_oracle(oracle):
    """Config B (200k clustered points): many medium and big cells (the
    cluster-parallel big-cell fix-up) -- bin arrays equal to the oracle's."""
    from paper_2511_10442_b200.datasets import config_dataset
    c, off, k = config_dataset("B")
    nb = fg.compute_n_bins(int(np.diff(off).max()), k, 4)
    ref = oracle.build_index(c.astype(np.float64), off, 4, nb)
    got = run_bin(c, off, 4, nb)
    for r, g_ in zip(ref, got[:5]):
        assert np.array_equal(r, g_.astype(r.dtype))
    n_c = c.shape[1]
    assert np.array_equal(got[5][:, :n_c], c[ref[1]])


def test_bin_cell_edges_vs_oracle(oracle):
    """Coordinates on and one ulp either side of cell edges (the cases where the
    cell index falls back from RN(a * RN(1/w)) to the exact division), several
    n_bins (powers of two: exact quotients; odd: inexact widths), float32 and
    float64 inputs -- bin arrays equal to the oracle's."""
    rng = np.random.default_rng(11)
    for n_bins in (8, 13, 29, 64):
        edges = np.arange(n_bins + 1, dtype=np.float64) / n_bins
        base = rng.choice(edges, size=(6000, 4))
        nudge = rng.integers(-1, 2, size=base.shape)
        c32 = base.astype(np.float32)
        c32 = np.where(nudge > 0, np.nextafter(c32, np.float32(2)),
                       np.where(nudge < 0, np.nextafter(c32, np.float32(-1)), c32))
        c32[0] = 0.0
        c32[1] = 1.0
        c32 = np.concatenate([c32, rng.random((2000, 4)).astype(np.float32)])
        off = np.array([0, 3000, len(c32)], np.int64)
        ref = oracle.build_index(c32.astype(np.float64), off, 4, n_bins)
        got = run_bin(c32, off, 4, n_bins)
        for r, g_ in zip(ref, got[:5]):
            assert np.array_equal(r, g_.astype(r.dtype))
        b64 = np.where(nudge > 0, np.nextafter(base, 2.0),
                       np.where(nudge < 0, np.nextafter(base, -1.0), base))
        c64 = np.concatenate([b64, rng.random((2000, 4))])
        got64 = [o.cpu().numpy() for o in ops.bin_by_coordinates(
            t(c64, torch.float64), t(off, torch.int64), 4, n_bins)]
        ref64 = oracle.build_index(c64, off, 4, n_bins)
        for r, g_ in zip(ref64, got64[:5]):
            assert np.array_equal(r, g_.astype(r.dtype))


def test_bin_fp64_cell_kat():
    # generate_dataset(1_000_000, 4, seed=1) as f32, vertex 842094,
    # dim 3: float64 cell arithmetic gives 28 (float32 would give 27).
    from paper_2511_10442_b200.datasets import generate_dataset
    c, off = generate_dataset(1_000_000, 4, seed=1)
    c = c.astype(np.float32)
    n_bins = fg.compute_n_bins(1_000_000, 40, 4)
    bi, *_ = run_bin(c, off, 4, n_bins)
    assert (bi[842094] % n_bins) == 28


def test_index_replacer():
    x = t(np.array([[0, 2, -1], [1, -1, 3]], np.int32))
    lut = t(np.array([10, 11, 12, 13], np.int32))
    out = ops.index_replacer(x, lut).cpu().numpy()
    assert out.tolist() == [[10, 12, -1], [11, -1, 13]]


# ---------------------------------------------------------------- search
@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_knn_vs_reference_and_oracle(golden, oracle, name):
    g = golden_case(golden, name)
    k = g["k"]
    gi, gd = assert_canonical(oracle, g["coords"], g["row_splits"], k, mask=g["mask"],
                              max_r2=g["max_r2"], d_bin=g["d_bin"], n_bins=g["n_bins"])
    # against the reference itself, rows normalised the reference's way
    # (sort_neighbor_rows, G/harness/verify.py:34-44,125-133): sorted d2 rows
    # equal everywhere, indices on rows whose k-th / (k+1)-th distances are
    # not tied (G/harness/verify.py:71-96)
    si, sd = ref_sorted(gi, gd)
    assert np.array_equal(sd, g["knn_d2_sorted"])
    bk, bd = g["brute_k1_idx"], g["brute_k1_d2"]
    filled = (bk >= 0).sum(1)
    tied = (filled == k + 1) & (bd[:, k] <= bd[:, k - 1])
    assert np.array_equal(si[~tied], g["knn_idx_sorted"][~tied])


@pytest.mark.parametrize("name", ["u3", "c4", "u5", "m3"])
def test_exhaustive_rings_same_answer(golden, name):
    g = golden_case(golden, name)
    a = run_knn(g["coords"], g["row_splits"], g["k"], mask=g["mask"], max_r2=g["max_r2"])
    b = run_knn(g["coords"], g["row_splits"], g["k"], mask=g["mask"], max_r2=g["max_r2"],
                exhaustive=True)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_knn_kats():
    # T/test_knn.py:50-56 collinear
    i, d = run_knn(np.array([[0, 0], [1, 0], [4, 0]], np.float32), [0, 3], 2)
    assert i.tolist() == [[0, 1], [1, 0], [2, 1]] and d.tolist() == [[0, 1], [0, 1], [0, 9]]
    # :126-133 duplicate pair
    i, d = run_knn(np.array([[.2, .2], [.2, .2], [.9, .9]], np.float32), [0, 3], 2)
    assert i[0].tolist() == [0, 1] and i[1].tolist() == [1, 0] and d[0, 1] == 0 and d[1, 1] == 0
    # :137-144 radius boundary kept
    i, d = run_knn(np.array([[0, 0], [1, 0], [3, 0]], np.float32), [0, 3], 3, max_r2=1.0)
    assert i.tolist() == [[0, 1, -1], [1, 0, -1], [2, -1, -1]]
    # :146-152 radius 0
    i, d = run_knn(np.array([[.5, .5], [.5, .5], [.6, .5]], np.float32), [0, 3], 3, max_r2=0.0)
    assert i[0].tolist() == [0, 1, -1] and i[2].tolist() == [2, -1, -1]
    # :176-187 roles
    c = np.array([[0, 0], [.1, 0], [.2, 0], [.3, 0]], np.float32)
    i, d = run_knn(c, [0, 4], 4, mask=np.array([3, 1, 2, 3], np.int8))
    assert set(i[1].tolist()) == {1, 0, 3, -1} and 1 not in i[0, 1:] and 2 not in i[0, 1:]
    assert i[2].tolist() == [2, -1, -1, -1]
    # padding + k=1
    i, d = run_knn(np.random.default_rng(1).random((3, 2)).astype(np.float32), [0, 3], 8)
    assert np.all(i[:, 3:] == -1) and np.all(d[:, 3:] == 0) and np.all(i[:, :3] >= 0)
    i, d = run_knn(np.random.default_rng(2).random((40, 2)).astype(np.float32), [0, 40], 1)
    assert i.shape == (40, 1) and np.array_equal(i[:, 0], np.arange(40))


def test_eviction_kat_canonical():
    # compiled binned [0,1,3], compiled brute [0,3,2]; canonical [0,3,1]
    c = np.array([[0, 0], [1, 2], [2, 1], [2, 0]], np.float32)
    i, d = run_knn(c, [0, 4], 3)
    assert i[0].tolist() == [0, 3, 1] and d[0].tolist() == [0.0, 4.0, 5.0]


@pytest.mark.parametrize("k", [5, 8, 16])
def test_lattice_ties(oracle, k):
    g = np.stack(np.meshgrid(*[np.arange(8)] * 3, indexing="ij"), -1).reshape(-1, 3)
    g = g[np.random.default_rng(0).permutation(len(g))].astype(np.float32)
    assert_canonical(oracle, g, [0, len(g)], k)


def test_coincident_piles(oracle):
    rng = np.random.default_rng(3)
    c = np.concatenate([np.full((3000, 3), 0.5), rng.random((2000, 3)),
                        np.full((700, 3), 0.1)]).astype(np.float32)
    c = c[rng.permutation(len(c))]
    assert_canonical(oracle, c, [0, len(c)], 40)
    i, d = run_knn(np.full((10, 3), 0.5, np.float32), [0, 10], 4)
    assert np.all(d == 0) and np.all(i >= 0)
    assert i[7].tolist() == [7, 0, 1, 2]


def test_clustered_and_splits(oracle):
    from paper_2511_10442_b200.datasets import generate_dataset
    c, off = generate_dataset(30_000, 4, splits=3, seed=11, distribution="clusters")
    assert_canonical(oracle, c.astype(np.float32), off, 40)
    c = np.random.default_rng(4).random((600, 3)).astype(np.float32)
    off = np.array([0, 100, 100, 350, 350, 600])
    gi, _ = assert_canonical(oracle, c, off, 7)
    for s in range(5):
        blk = gi[off[s]:off[s + 1]]
        v = blk[blk >= 0]
        assert np.all((v >= off[s]) & (v < off[s + 1]))


@pytest.mark.parametrize("d,k", [(1, 5), (2, 9), (6, 8), (10, 64), (13, 12), (16, 20)])
def test_dims(oracle, d, k):
    c = np.random.default_rng(d).random((1500, d)).astype(np.float32)
    if d == 1:
        gi, gd = run_knn(c, [0, 1500], k, d_bin=1, n_bins=1)
        oi, od = oracle.brute_canonical(c.astype(np.float64), [0, 1500], k)
        assert np.array_equal(gi, oi) and np.array_equal(gd, od)
    else:
        assert_canonical(oracle, c, [0, 1500], k)


@pytest.mark.parametrize("k", [100, 300, 700])
def test_large_k(oracle, k):
    c = np.random.default_rng(k).random((3000, 3)).astype(np.float32)
    assert_canonical(oracle, c, [0, 1000, 3000], k)


def test_masks_and_radius(oracle):
    rng = np.random.default_rng(52)
    c = rng.random((2000, 3)).astype(np.float32)
    mask = rng.integers(0, 4, 2000).astype(np.int8)
    for mr2 in (None, 0.0, 0.002, 0.05):
        assert_canonical(oracle, c, [0, 900, 2000], 9, mask=mask, max_r2=mr2)


def test_brute_force_route(oracle):
    c = np.random.default_rng(9).random((800, 4)).astype(np.float32)
    cloud = fg.PointCloud(torch.from_numpy(c).cuda(), [0, 300, 800])
    nm = fg.brute_force_knn(cloud, fg.KnnOptions(k=6), d2_f64=True)
    oi, od = oracle.brute_canonical(c.astype(np.float64), [0, 300, 800], 6)
    assert np.array_equal(nm.indices.cpu().numpy(), oi)
    assert np.array_equal(nm.dist2.cpu().numpy(), od)


# ---------------------------------------------------------------- backward
def test_backward_kats():
    c = torch.tensor([[0.0], [3.0]], device=dev())
    idx = torch.tensor([[0, 1], [1, 0]], dtype=torch.int32, device=dev())
    up = torch.tensor([[0.0, 1.0], [0.0, 0.0]], device=dev())
    assert ops.binned_select_knn_grad(up, idx, c).cpu().tolist() == [[-6.0], [6.0]]
    assert ops.binned_select_knn_grad(torch.ones_like(up), idx, c).cpu().tolist() == [[-12.0], [12.0]]
    idx = torch.tensor([[0, -1], [1, -1]], dtype=torch.int32, device=dev())
    c2 = torch.tensor([[0.0, 0.0], [1.0, 1.0]], device=dev())
    assert torch.all(ops.binned_select_knn_grad(torch.ones((2, 2), device=dev()), idx, c2) == 0)


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_backward_vs_reference(golden, name):
    g = golden_case(golden, name)
    c = t(g["coords"])
    gr = ops.binned_select_knn_grad(t(g["upstream"]), t(g["knn_idx_raw"]), c).cpu().numpy()
    ref = g["grad_raw_rows"]
    np.testing.assert_allclose(gr, ref, rtol=1e-5, atol=1e-12 * np.abs(ref).max())
    c64 = c.double()
    gr64 = ops.binned_select_knn_grad(t(g["upstream"]), t(g["knn_idx_raw"]), c64).cpu().numpy()
    np.testing.assert_allclose(gr64, ref, rtol=1e-12, atol=1e-14 * np.abs(ref).max())


def test_autograd_through_select_knn(oracle):
    c = torch.rand(3000, 4, device=dev(), generator=torch.Generator(device=dev()).manual_seed(5))
    c.requires_grad_(True)
    idx, d2 = fg.select_knn(c, [0, 3000], 12)
    up = torch.randn(d2.shape, device=dev())
    (d2 * up).sum().backward()
    ref = oracle.knn_backward(c.detach().cpu().double().numpy(), idx.cpu().numpy(),
                              up.cpu().double().numpy())
    np.testing.assert_allclose(c.grad.cpu().numpy(), ref, rtol=1e-5, atol=1e-9)


# ---------------------------------------------------------------- GravNet
@pytest.mark.parametrize("red", ["mm", "mean", "max"])
@pytest.mark.parametrize("incl", [1, 0])
def test_gravnet_vs_reference(golden, oracle, red, incl):
    reducers = {"mm": ("mean", "max"), "mean": ("mean",), "max": ("max",)}[red]
    pre = f"gn_{red}_{incl}__"
    feats = golden["gn__feats"]
    idx = golden["gn__idx"]
    d2_32 = golden["gn__d2"].astype(np.float32)
    spec = fg.AggregationSpec(weight_scale=10.0, reducers=reducers, include_self=bool(incl))
    nm = fg.NeighborMatrix(t(idx), t(d2_32))
    out = fg.gravnet_aggregate(t(feats), nm, spec).cpu().numpy()
    up = golden[pre + "up"]
    gf, gd = fg.gravnet_aggregate_backward(t(feats), nm, spec, t(up))
    gf, gd = gf.cpu().numpy(), gd.cpu().numpy()
    # vs the reference (its d2 is float64; ours float32 of it)
    np.testing.assert_allclose(out, golden[pre + "out"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(gf, golden[pre + "grad_feats"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(gd, golden[pre + "grad_d2"], rtol=1e-5, atol=1e-6)
    # vs the oracle on identical float32 inputs: float64 math, tighter
    o = oracle.gravnet_aggregate(feats, idx, d2_32, 10.0, reducers, bool(incl))
    np.testing.assert_allclose(out, o, rtol=1e-6, atol=1e-7)
    ogf, ogd = oracle.gravnet_aggregate_backward(feats, idx, d2_32, up, 10.0, reducers, bool(incl))
    np.testing.assert_allclose(gf, ogf, rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(gd, ogd, rtol=1e-6, atol=1e-7)


@pytest.mark.parametrize("n,F,k", [(700, 300, 9), (400, 40, 300), (2500, 64, 40)])
def test_gravnet_wide_and_ordered(oracle, n, F, k):
    """Several feature chunks (F > 256: float64 grad_d2 partials), k > 255
    (two-byte arg-max slots), a row visit order, padding and repeated
    neighbours (one vertex in several slots of a row)."""
    rng = np.random.default_rng(n + F + k)
    feats = rng.standard_normal((n, F)).astype(np.float32)
    idx = rng.integers(0, n, (n, k)).astype(np.int32)
    idx[:, 0] = np.arange(n)
    idx[rng.random((n, k)) < 0.1] = -1
    idx[:, 0] = np.arange(n)
    d2 = np.where(idx >= 0, rng.random((n, k)) * 0.3, 0).astype(np.float32)
    d2[:, 0] = 0
    up = rng.standard_normal((n, 2 * F)).astype(np.float32)
    order = t(rng.permutation(n).astype(np.int32))
    spec = fg.AggregationSpec(weight_scale=10.0)
    nm = fg.NeighborMatrix(t(idx), t(d2))
    o = oracle.gravnet_aggregate(feats, idx, d2, 10.0)
    ogf, ogd = oracle.gravnet_aggregate_backward(feats, idx, d2, up, 10.0)
    for od in (None, order):
        out = fg.gravnet_aggregate(t(feats), nm, spec, od).cpu().numpy()
        gf, gd = fg.gravnet_aggregate_backward(t(feats), nm, spec, t(up), od)
        np.testing.assert_allclose(out, o, rtol=1e-6, atol=1e-7)
        np.testing.assert_allclose(gf.cpu().numpy(), ogf, rtol=1e-6, atol=1e-6)
        np.testing.assert_allclose(gd.cpu().numpy(), ogd, rtol=1e-6, atol=1e-6)


def test_gravnet_kats():
    # T/test_gravnet.py:40-54, 160-173
    nm = fg.NeighborMatrix(t(np.array([[0, 1], [1, 0]], np.int32)), t(np.array([[0, 1], [0, 1]], np.float32)))
    f = t(np.array([[1.0], [2.0]], np.float32))
    m = fg.gravnet_aggregate(f, nm, fg.AggregationSpec(1.0, ("mean",))).cpu().numpy()
    np.testing.assert_allclose(m[:, 0], [0.8678794411714423, 1.1839397205857212], rtol=1e-7)
    mx = fg.gravnet_aggregate(f, nm, fg.AggregationSpec(1.0, ("max",))).cpu().numpy()
    assert mx[:, 0].tolist() == [1.0, 2.0]
    idx = t(np.array([[0, 1, 2], [1, -1, -1], [2, -1, -1]], np.int32))
    nm = fg.NeighborMatrix(idx, t(np.zeros((3, 3), np.float32)))
    f = t(np.array([[0.0], [2.0], [2.0]], np.float32))
    spec = fg.AggregationSpec(1.0, ("max",))
    assert fg.gravnet_aggregate(f, nm, spec).cpu().numpy()[0, 0] == 2.0
    gf, _ = fg.gravnet_aggregate_backward(f, nm, spec, t(np.array([[1.0], [0.0], [0.0]], np.float32)))
    assert gf[1, 0].item() == 1.0 and gf[2, 0].item() == 0.0
    # no valid slot -> zeros
    nm = fg.NeighborMatrix(t(np.array([[0], [1]], np.int32)), t(np.zeros((2, 1), np.float32)))
    spec = fg.AggregationSpec(include_self=False)
    assert torch.all(fg.gravnet_aggregate(t(np.array([[1.0], [5.0]], np.float32)), nm, spec) == 0)


def test_gravnet_autograd_and_op():
    torch.manual_seed(0)
    layer = fg.GravNetOp(in_features=16, d_space=4, n_prop=8, k=10).cuda()
    x = torch.randn(2000, 16, device=dev(), requires_grad=True)
    y = layer(x, [0, 1200, 2000])
    y.square().mean().backward()
    assert x.grad is not None and torch.isfinite(x.grad).all()
    assert layer.space.weight.grad is not None and layer.space.weight.grad.abs().sum() > 0


def test_gravnet_layer_vs_oracle_chain(oracle):
    """GravNetOp (raw op, linear=False) forward and backward against the oracle
    chain: canonical kNN -> gravnet_aggregate -> its backward -> knn_backward
    (G/gravnet.py:75-150, G/knn.py:135-168), two row splits."""
    rng = np.random.default_rng(21)
    n, k, F = 6000, 12, 16
    coords = rng.random((n, 4)).astype(np.float32)
    off = np.array([0, 2500, n], np.int64)
    feats = rng.standard_normal((n, F)).astype(np.float32)
    up = rng.standard_normal((n, 2 * F)).astype(np.float32)
    layer = fg.GravNetOp(k=k, linear=False)
    c = torch.from_numpy(coords).to(dev()).requires_grad_(True)
    f = torch.from_numpy(feats).to(dev()).requires_grad_(True)
    agg, idx, d2 = layer.aggregate(c, f, off)
    (agg * torch.from_numpy(up).to(dev())).sum().backward()
    oi, od = oracle.knn_canonical(coords.astype(np.float64), off, k)
    assert np.array_equal(idx.cpu().numpy(), oi)
    od32 = od.astype(np.float32)
    assert np.array_equal(d2.detach().cpu().numpy(), od32)
    oa = oracle.gravnet_aggregate(feats, oi, od32, 10.0)
    np.testing.assert_allclose(agg.detach().cpu().numpy(), oa, rtol=1e-5, atol=1e-6)
    ogf, ogd = oracle.gravnet_aggregate_backward(feats, oi, od32, up, 10.0, ("mean", "max"), True)
    np.testing.assert_allclose(f.grad.cpu().numpy(), ogf, rtol=1e-5, atol=1e-6)
    ogc = oracle.knn_backward(coords.astype(np.float64), oi, ogd.astype(np.float32).astype(np.float64))
    np.testing.assert_allclose(c.grad.cpu().numpy(), ogc, rtol=1e-4, atol=1e-5 * np.abs(ogc).max())


def test_cpu_tensor_raises():
    with pytest.raises(fg.errors.BackendUnavailableError):
        ops.bin_by_coordinates(torch.zeros(4, 2), torch.tensor([0, 4]), 2, 5)
