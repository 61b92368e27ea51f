"""CPU: host-side logic of the framework (no kernel launches)."""

import hashlib
import json
import os

import numpy as np
import pytest
import torch

import paper_2511_10442_b200 as fg
from paper_2511_10442_b200 import backend, datasets, errors, ops, sharding
from conftest import ROOT


def test_compute_n_bins_matches_reference_table():
    table = [(1_000_000, 40, 5, 15), (100_000, 1, 5, 20), (7776, 32, 5, 6), (3375, 4, 3, 30),
             (10_000, 4, 3, 30), (100_000, 10, 3, 30), (1000, 10, 2, 30), (5, 1000, 2, 5),
             (30, 40, 2, 5), (243, 32, 5, 5), (100, 32, 2, 10), (1, 1, 2, 5), (100_000, 40, 5, 9),
             (100_000, 10, 5, 12), (10_000, 100, 4, 7), (1_000_000, 40, 4, 29)]
    for n, k, d, want in table:
        assert fg.compute_n_bins(n, k, d) == want
    with pytest.raises(errors.BadKError):
        fg.compute_n_bins(100, 0, 2)


def test_default_bin_dims():
    assert fg.default_bin_dims(2) == 2 and fg.default_bin_dims(4) == 4
    assert fg.default_bin_dims(10) == 5
    with pytest.raises(errors.TooFewDimsError):
        fg.default_bin_dims(1)


def test_resolve_binning_validation():
    from paper_2511_10442_b200.binning import resolve_binning
    cloud = fg.PointCloud(np.random.default_rng(0).random((50, 3)), [0, 50], device="cpu")
    assert resolve_binning(cloud, fg.BinningConfig(k_target=4)) == (3, fg.compute_n_bins(50, 4, 3))
    with pytest.raises(errors.BadShapeError):
        resolve_binning(cloud, fg.BinningConfig(k_target=4, d_bin=6))
    with pytest.raises(errors.TooFewDimsError):
        resolve_binning(cloud, fg.BinningConfig(k_target=4, d_bin=1))
    with pytest.raises(errors.TooFewDimsError):
        resolve_binning(cloud, fg.BinningConfig(k_target=4, d_bin=4))
    two = fg.PointCloud(np.random.default_rng(5).random((1010, 2)), [0, 10, 1010], device="cpu")
    assert resolve_binning(two, fg.BinningConfig(k_target=1))[1] == fg.compute_n_bins(1000, 1, 2)
    assert resolve_binning(two, fg.BinningConfig(k_target=1, n_bins=7)) == (2, 7)


def test_row_splits_and_cloud_validation():
    rs = fg.RowSplits([0, 3, 3, 10])
    assert rs.n_splits == 3 and rs.n_vertices == 10 and rs.sizes().tolist() == [3, 0, 7]
    assert fg.split_of_vertex(rs, 3) == 2
    with pytest.raises(errors.BadBoundsError):
        fg.RowSplits([1, 3])
    with pytest.raises(errors.NonMonotonicError):
        fg.RowSplits([0, 5, 3])
    with pytest.raises(errors.BadShapeError):
        fg.RowSplits([0])
    with pytest.raises(errors.ShapeMismatchError):
        fg.PointCloud(np.zeros((4, 2)), [0, 3], device="cpu")
    with pytest.raises(errors.BadShapeError):
        fg.PointCloud(np.array([[0.0, np.nan]]), [0, 1], device="cpu")
    with pytest.raises(errors.BadShapeError):
        fg.DirectionMask(np.array([0, 4]))
    m = fg.DirectionMask(np.array([0, 1, 2, 3]))
    assert m.runs_query().tolist() == [False, True, False, True]
    assert m.is_candidate().tolist() == [True, False, False, True]


def test_knn_option_errors():
    from paper_2511_10442_b200.knn import _check_options
    cloud = fg.PointCloud(np.zeros((5, 2)), [0, 5], device="cpu", check_finite=False)
    for bad in (0, -1, 1.5, True, 961):
        with pytest.raises(errors.BadKError):
            _check_options(cloud, fg.KnnOptions(k=bad))
    with pytest.raises(errors.BadKError):
        _check_options(cloud, fg.KnnOptions(k=2, max_radius2=-1.0))
    with pytest.raises(errors.ShapeMismatchError):
        _check_options(cloud, fg.KnnOptions(k=2, mask=fg.DirectionMask(np.zeros(4))))


def test_aggregation_spec_validation():
    assert fg.AggregationSpec().codes == [0, 1]
    for bad in (dict(weight_scale=0.0), dict(reducers=()), dict(reducers=("median",))):
        with pytest.raises(errors.BadShapeError):
            fg.AggregationSpec(**bad)


def test_cpu_tensors_fail_loudly():
    """No CPU fallback: a CPU tensor is refused before anything runs."""
    with pytest.raises(errors.BackendUnavailableError):
        ops.bin_by_coordinates(torch.zeros(4, 2), torch.tensor([0, 4]), 2, 5)
    with pytest.raises(errors.BackendUnavailableError):
        ops.binned_select_knn_grad(torch.zeros(2, 2), torch.zeros(2, 2, dtype=torch.int32),
                                   torch.zeros(2, 2))


def test_fake_kernels_shape_inference():
    from torch._subclasses.fake_tensor import FakeTensorMode
    with FakeTensorMode():
        c = torch.empty(100, 4)
        rs = torch.empty(3, dtype=torch.int64)
        bi, so, bb, mn, wd, sc = torch.ops.fastgraph.bin_by_coordinates(c, rs, 4, 5)
        assert bi.shape == (100,) and bb.shape == (2 * 625 + 1,) and sc.shape == (100, 4)
        idx, d2 = torch.ops.fastgraph.binned_select_knn(c, rs, bi, so, bb, mn, wd, sc, 7, 4, 5,
                                                        None, None, False, False)
        assert idx.shape == (100, 7) and idx.dtype == torch.int32 and d2.dtype == torch.float32
        g = torch.ops.fastgraph.binned_select_knn_grad(d2, idx, c)
        assert g.shape == (100, 4)
        f = torch.empty(100, 16)
        out = torch.ops.fastgraph.gravnet_aggregate(f, idx, d2, 10.0, [0, 1], True)
        assert out.shape == (100, 32)
        gf, gd = torch.ops.fastgraph.gravnet_aggregate_grad(out, f, idx, d2, 10.0, [0, 1], True)
        assert gf.shape == (100, 16) and gd.shape == (100, 7)


def test_backend_ring_cells_matches_oracle(oracle):
    rng = np.random.default_rng(54)
    assert backend.ring_cells([5, 5], [2, 2], 1).tolist() == [6, 7, 8, 11, 13, 16, 17, 18]
    for _ in range(80):
        nd = int(rng.integers(1, 6))
        counts = rng.integers(1, 7, size=nd)
        center = np.array([rng.integers(0, c) for c in counts])
        radius = int(rng.integers(0, 5))
        assert backend.ring_cells(counts, center, radius).tolist() == \
            oracle.ring_cells(counts, center, radius).tolist()


def test_backend_protocol_surface():
    assert backend.NAME == "cuda"
    for name in ("build_index", "ring_cells", "binned_knn", "brute_knn"):
        assert callable(getattr(backend, name))
    off = backend._offsets_from_bin_idx(np.array([0, 1, 5, 40, 41, 130]), 36, 6)
    assert off.tolist() == [0, 3, 5, 5, 6]


def test_product_generator_matches_reference_digests():
    meta = json.load(open(os.path.join(ROOT, "tests", "golden", "datasets.json")))
    for key in ("A", "B", "north_star"):
        m = meta[key]
        c, off = datasets.generate_dataset(m["n"], m["d"], m["splits"], m["seed"], m["distribution"])
        assert hashlib.sha256(np.ascontiguousarray(c, np.float32).tobytes()).hexdigest() == m["sha256_f32"]
        assert fg.compute_n_bins(int(np.diff(off).max()), m["k"], m["d_bin"]) == m["n_bins"]


def test_sharding_event_ranges():
    off = datasets.even_row_splits(6_400, 64)
    for world in (1, 2, 4, 8, 3):
        covered = []
        for r in range(world):
            sh = sharding.shard(off, r, world)
            covered += list(range(sh.event_lo, sh.event_hi))
            assert sh.local_offsets[0] == 0 and sh.local_offsets[-1] == sh.n_vertices
            assert sh.vertex_lo == off[sh.event_lo] and sh.vertex_hi == off[sh.event_hi]
        assert covered == list(range(64))
    # n_bins is global: from the largest split of the whole batch
    assert sharding.global_n_bins(off, 40, 4) == fg.compute_n_bins(100, 40, 4)
