"""CPU: pin the oracle (test infrastructure) to the reference.

(1) known-answer tests from the reference's own test suite (pkg/tests),
(2) golden vectors produced by running the real reference
    (tests/golden/make_golden.py), and
(3) the reference's compiled kernels themselves (oracle/_ref), when built.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_CASES, ROOT, golden_case


# ---------------------------------------------------------------- KATs
def test_n_bins_table(oracle):
    # T/test_binning.py:14-31
    table = [(1_000_000, 40, 5, 15), (100_000, 1, 5, 20), (7776, 32, 5, 6), (3375, 4, 3, 30),
             (10_000, 4, 3, 30), (100_000, 10, 3, 30), (1000, 10, 2, 30), (5, 1000, 2, 5),
             (30, 40, 2, 5), (243, 32, 5, 5), (100, 32, 2, 10), (1, 1, 2, 5), (100_000, 40, 5, 9),
             (100_000, 10, 5, 12), (10_000, 100, 4, 7)]
    for n, k, d, want in table:
        assert oracle.compute_n_bins(n, k, d) == want, (n, k, d)


def test_baseline_config_n_bins(oracle):
    want = {"A": 27, "B": 20, "north_star": 29, "C": 13, "D": 16, "E": 25}
    meta = json.load(open(os.path.join(ROOT, "tests", "golden", "datasets.json")))
    for key, nb in want.items():
        assert meta[key]["n_bins"] == nb
        m = meta[key]
        per_split = -(-m["n"] // m["splits"])
        assert oracle.compute_n_bins(per_split, m["k"], m["d_bin"]) == nb


def test_ring_kats(oracle):
    # T/test_stepper.py:55-62
    assert oracle.ring_cells([5, 5], [2, 2], 1).tolist() == [6, 7, 8, 11, 13, 16, 17, 18]
    assert oracle.ring_cells([5, 5], [0, 0], 1).tolist() == [1, 5, 6]
    assert oracle.ring_cells([5, 5], [2, 2], 0).tolist() == [12]
    assert oracle.ring_cells([3, 3], [1, 1], 5).tolist() == []


def test_knn_kats(oracle):
    # T/test_knn.py:50-56 collinear
    i, d = oracle.knn_canonical(np.array([[0, 0], [1, 0], [4, 0]], float), [0, 3], 2)
    assert i.tolist() == [[0, 1], [1, 0], [2, 1]] and d.tolist() == [[0, 1], [0, 1], [0, 9]]
    # :137-144 radius boundary kept
    i, _ = oracle.knn_canonical(np.array([[0, 0], [1, 0], [3, 0]], float), [0, 3], 3,
                                max_radius2=1.0)
    assert i.tolist() == [[0, 1, -1], [1, 0, -1], [2, -1, -1]]
    # :176-187 roles
    c = np.array([[0, 0], [.1, 0], [.2, 0], [.3, 0]], float)
    i, _ = oracle.knn_canonical(c, [0, 4], 4, dir_mask=np.array([3, 1, 2, 3], np.int8))
    assert i[2].tolist() == [2, -1, -1, -1] and set(i[1].tolist()) == {1, 0, 3, -1}


def test_eviction_kat(oracle):
    # the reference's own routes disagree under exact ties; the
    # canonical (d2, index) rule picks [0, 3, 1]
    c = np.array([[0, 0], [1, 2], [2, 1], [2, 0]], float)
    assert oracle.knn_canonical(c, [0, 4], 3)[0][0].tolist() == [0, 3, 1]
    assert oracle.knn_refslot(c, [0, 4], 3)[0][0].tolist() == [0, 1, 3]
    assert oracle.brute_refslot(c, [0, 4], 3)[0][0].tolist() == [0, 3, 2]


def test_backward_kat(oracle):
    # T/test_knn.py:253-262
    c = np.array([[0.0], [3.0]])
    idx = np.array([[0, 1], [1, 0]], np.int32)
    assert oracle.knn_backward(c, idx, np.array([[0.0, 1.0], [0.0, 0.0]])).tolist() == [[-6.0], [6.0]]
    assert oracle.knn_backward(c, idx, np.ones((2, 2))).tolist() == [[-12.0], [12.0]]
    g = oracle.knn_backward_numpy(c, idx, np.ones((2, 2)))
    assert g.tolist() == [[-12.0], [12.0]]


def test_gravnet_kats(oracle):
    # T/test_gravnet.py:40-54, 160-173
    f = np.array([[1.0], [2.0]])
    idx = np.array([[0, 1], [1, 0]], np.int32)
    d2 = np.array([[0.0, 1.0], [0.0, 1.0]])
    m = oracle.gravnet_aggregate(f, idx, d2, 1.0, ("mean",))
    np.testing.assert_allclose(m[:, 0], [0.8678794411714423, 1.1839397205857212], rtol=0, atol=1e-15)
    assert oracle.gravnet_aggregate(f, idx, d2, 1.0, ("max",))[:, 0].tolist() == [1.0, 2.0]
    f = np.array([[0.0], [2.0], [2.0]])
    idx = np.array([[0, 1, 2], [1, -1, -1], [2, -1, -1]], np.int32)
    gf, _ = oracle.gravnet_aggregate_backward(f, idx, np.zeros((3, 3)), np.array([[1.0], [0.0], [0.0]]),
                                              1.0, ("max",))
    assert gf[1, 0] == 1.0 and gf[2, 0] == 0.0


# ---------------------------------------------------------------- golden vectors
@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_oracle_build_index_vs_reference(golden, oracle, name):
    g = golden_case(golden, name)
    out = oracle.build_index(g["coords"].astype(np.float64), g["row_splits"], g["d_bin"], g["n_bins"])
    for got, key in zip(out, ("bin_idx", "sort_order", "bin_bounds", "dim_mins", "widths")):
        assert np.array_equal(got, g[key]), key


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_oracle_refslot_vs_reference(golden, oracle, name):
    """The restated slot-eviction search reproduces the reference's raw rows
    bit for bit (heap order included)."""
    g = golden_case(golden, name)
    i, d = oracle.knn_refslot(g["coords"].astype(np.float64), g["row_splits"], g["k"],
                              n_bins=g["n_bins"], d_bin=g["d_bin"], dir_mask=g["mask"],
                              max_radius2=g["max_r2"])
    assert np.array_equal(i, g["knn_idx_raw"]) and np.array_equal(d, g["knn_d2_raw"])


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_oracle_canonical_vs_reference(golden, oracle, name):
    """Canonical rows equal the reference's sorted rows (self included, G/harness/
    verify.py:34-44) in distance everywhere and in index set on untied rows."""
    g = golden_case(golden, name)
    k = g["k"]
    i, d = oracle.knn_canonical(g["coords"].astype(np.float64), g["row_splits"], k,
                                dir_mask=g["mask"], max_radius2=g["max_r2"])
    bi, bd = oracle.brute_canonical(g["coords"].astype(np.float64), g["row_splits"], k,
                                    dir_mask=g["mask"], max_radius2=g["max_r2"])
    assert np.array_equal(i, bi) and np.array_equal(d, bd)
    assert np.array_equal(np.sort(d, axis=1), np.sort(g["knn_d2_sorted"], axis=1))
    bk, bdd = g["brute_k1_idx"], g["brute_k1_d2"]
    tied = ((bk >= 0).sum(1) == k + 1) & (bdd[:, k] <= bdd[:, k - 1])
    si = np.sort(np.where(i >= 0, i, np.iinfo(np.int32).max), axis=1)
    ri = np.sort(np.where(g["knn_idx_sorted"] >= 0, g["knn_idx_sorted"], np.iinfo(np.int32).max), axis=1)
    assert np.array_equal(si[~tied], ri[~tied])


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_oracle_backward_vs_reference(golden, oracle, name):
    g = golden_case(golden, name)
    got = oracle.knn_backward(g["coords"].astype(np.float64), g["knn_idx_raw"],
                              g["upstream"].astype(np.float64))
    assert np.array_equal(got, g["grad_raw_rows"])  # same add order as np.add.at
    got2 = oracle.knn_backward_numpy(g["coords"].astype(np.float64), g["knn_idx_raw"],
                                     g["upstream"].astype(np.float64))
    assert np.array_equal(got2, g["grad_raw_rows"])


@pytest.mark.parametrize("red", ["mm", "mean", "max"])
@pytest.mark.parametrize("incl", [1, 0])
def test_oracle_gravnet_vs_reference(golden, oracle, red, incl):
    reducers = {"mm": ("mean", "max"), "mean": ("mean",), "max": ("max",)}[red]
    pre = f"gn_{red}_{incl}__"
    f = golden["gn__feats"].astype(np.float64)
    idx, d2 = golden["gn__idx"], golden["gn__d2"]
    out = oracle.gravnet_aggregate(f, idx, d2, 10.0, reducers, bool(incl))
    np.testing.assert_allclose(out, golden[pre + "out"], rtol=1e-13, atol=1e-15)
    gf, gd = oracle.gravnet_aggregate_backward(f, idx, d2, golden[pre + "up"].astype(np.float64),
                                               10.0, reducers, bool(incl))
    np.testing.assert_allclose(gf, golden[pre + "grad_feats"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(gd, golden[pre + "grad_d2"], rtol=1e-12, atol=1e-14)


def test_lattice_canonical_rule(oracle):
    """On an 8^3 lattice (massive exact ties) the canonical ring search equals a
    direct lexsort of (d2, index) per row."""
    g = np.stack(np.meshgrid(*[np.arange(8)] * 3, indexing="ij"), -1).reshape(-1, 3)
    g = g[np.random.default_rng(0).permutation(len(g))].astype(np.float64)
    for k in (5, 8, 16):
        i, d = oracle.knn_canonical(g, [0, len(g)], k)
        for v in range(0, len(g), 37):
            dd = ((g - g[v]) ** 2).sum(1)
            order = np.lexsort((np.arange(len(g)), dd))
            order = order[order != v][: k - 1]
            assert i[v, 1:].tolist() == order.tolist()


# ---------------------------------------------------------------- the reference's own kernels
def test_oracle_vs_ref_kernels(oracle):
    ref = oracle.load_ref_kernels()
    if ref is None:
        pytest.skip("oracle/_ref not built (make -C oracle ref needs /root/reference)")
    for seed, (n, d, S, k, dist) in enumerate([(1500, 3, 1, 16, "uniform"),
                                               (2000, 4, 3, 10, "clusters"),
                                               (900, 6, 2, 7, "uniform")]):
        c, off = oracle.generate_dataset(n, d, S, seed=seed, distribution=dist)
        c = c.astype(np.float32).astype(np.float64)
        db = min(d, 5)
        nb = oracle.compute_n_bins(int(np.diff(off).max()), k, db)
        a = oracle.build_index(c, off, db, nb)
        b = ref.build_index(c, off, db, nb)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))
        oi = np.empty((n, k), np.int32)
        od = np.empty((n, k))
        ref.binned_knn(c, a[0], a[1], a[2], np.full(db, nb, np.int64), a[4].min(axis=1).copy(),
                       np.zeros(1, np.int8), False, 0.0, False, False, k, oi, od, 2)
        mi, md = oracle.knn_refslot(c, off, k, n_bins=nb, threads=2)
        assert np.array_equal(oi, mi) and np.array_equal(od, md)


def test_dataset_generator_matches_reference_digests(oracle):
    """The restated generator reproduces the reference's datasets byte for byte
    (digests recorded from the reference by make_golden.py)."""
    import hashlib
    meta = json.load(open(os.path.join(ROOT, "tests", "golden", "datasets.json")))
    for key in ("A", "B", "E"):
        m = meta[key]
        c, _ = oracle.generate_dataset(m["n"], m["d"], m["splits"], m["seed"], m["distribution"])
        assert hashlib.sha256(np.ascontiguousarray(c, np.float32).tobytes()).hexdigest() == m["sha256_f32"]
