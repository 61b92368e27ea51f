"""GPU parity of the association matrices (csrc/fg_oc.cu) through the
reference-shaped API (paper_2511_10442_b200.ocgraph): bit-exact against the
real reference's outputs (tests/golden/reference_oc.npz), the reference's
frozen known answers and edge cases (T/test_ocgraph.py), and the oracle at a
larger size."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2511_10442_b200 as fg  # noqa: E402
from conftest import oc_case  # noqa: E402
from paper_2511_10442_b200 import _lib  # noqa: E402
from paper_2511_10442_b200.datasets import generate_associations  # noqa: E402
from paper_2511_10442_b200.errors import BadCapacityError, ShapeMismatchError  # noqa: E402


def assoc(ids, offsets):
    return fg.Associations(np.asarray(ids, dtype=np.int64), fg.RowSplits(offsets))


def test_reference_golden_all_cases(golden_oc):
    l0 = _lib.launch_count()
    for name in [str(x) for x in golden_oc["names"]]:
        c = oc_case(golden_oc, name)
        a = fg.Associations(c["asso"], fg.RowSplits(c["row_splits"]))
        u = fg.find_unique(a)
        assert np.array_equal(u.unique_idx, c["unique_idx"]), name
        assert np.array_equal(u.unique_rs_asso, c["unique_rs"]), name
        top, counts = fg.max_same_count(a, u)
        assert top == c["top"] and np.array_equal(counts, c["counts"]), name
        res = fg.oc_helper(a, u, n_maxuq=c["n_maxuq"], n_maxrs=c["n_maxrs"])
        assert np.array_equal(res.m, c["m"]), name
        assert np.array_equal(res.m_not, c["m_not"]), name
        assert res.visit_count == c["visits"], name
        res2 = fg.oc_helper(a, n_maxuq=c["n_maxuq"], n_maxrs=c["n_maxrs"], calc_m_not=False)
        assert res2.m_not is None and np.array_equal(res2.m, c["m"]), name
        assert res2.visit_count == c["visits"], name
    assert _lib.launch_count() > l0  # the CUDA kernels ran


def test_frozen_cases():
    # T/test_ocgraph.py:16-118
    assert fg.find_unique(assoc([7, 7, 3, 7, 3], [0, 5])).unique_idx.tolist() == [7, 3]
    u = fg.find_unique(assoc([-1, -1], [0, 2]))
    assert u.unique_idx.tolist() == [] and u.unique_rs_asso.tolist() == []
    u = fg.find_unique(assoc([1, 1, 1, 1], [0, 2, 4]))
    assert u.unique_idx.tolist() == [1, 1] and u.unique_rs_asso.tolist() == [0, 1]
    u = fg.find_unique(assoc([5, -1, 2, 5, -7, 2, 9], [0, 4, 7]))
    assert u.unique_idx.tolist() == [5, 2, 2, 9] and u.unique_rs_asso.tolist() == [0, 0, 1, 1]
    top, counts = fg.max_same_count(assoc([7, 7, 3, 7, 3], [0, 5]))
    assert top == 3 and counts.tolist() == [3, 2]
    assert fg.max_same_count(assoc([-1, -1], [0, 2]))[0] == 0
    m = fg.oc_helper(assoc([7, 7, 3, 7, 3], [0, 5]), n_maxuq=4, n_maxrs=5)
    assert m.m.tolist() == [[0, 1, 3, -1], [2, 4, -1, -1]]
    assert m.m_not.tolist() == [[2, 4, -1, -1, -1], [0, 1, 3, -1, -1]] and m.visit_count == 10
    m = fg.oc_helper(assoc([9, 9, 9], [0, 3]), n_maxuq=3, n_maxrs=3)
    assert m.m.tolist() == [[0, 1, 2]] and m.m_not.tolist() == [[-1, -1, -1]]
    m = fg.oc_helper(assoc([7, 7, 3, 7, 3], [0, 5]), n_maxuq=2, n_maxrs=5)
    assert m.m.tolist() == [[0, 1], [2, 4]]
    m = fg.oc_helper(assoc([7, 7, 3, 7, 3], [0, 5]))
    assert m.m.shape == (2, 3) and m.m_not.shape == (2, 5)
    assert m.m.tolist() == [[0, 1, 3], [2, 4, -1]]
    m = fg.oc_helper(assoc([7, 7, 3, 7, 3], [0, 5]), calc_m_not=False)
    assert m.m_not is None and m.visit_count == 10
    m = fg.oc_helper(assoc([7, 3, 7, 7, 3], [0, 5]), n_maxuq=5, n_maxrs=3)
    assert m.m.tolist() == [[0, 2, -1, -1, -1], [1, -1, -1, -1, -1]]
    assert m.m_not.tolist() == [[1, -1, -1], [0, 2, -1]] and m.visit_count == 6
    m = fg.oc_helper(assoc([4, -1, 4], [0, 3]))
    assert m.m.tolist() == [[0, 2]] and m.m_not.tolist() == [[1, -1, -1]]
    m = fg.oc_helper(assoc([1, 1, 8, 8, -1], [0, 2, 5]))
    assert m.unique.unique_idx.tolist() == [1, 8] and m.m.tolist() == [[0, 1], [2, 3]]
    m = fg.oc_helper(assoc([-1, -1], [0, 2]))
    assert m.m.shape[0] == 0 and m.visit_count == 0
    with pytest.raises(BadCapacityError):
        fg.oc_helper(assoc([1, 1], [0, 2]), n_maxuq=0)
    with pytest.raises(BadCapacityError):
        fg.oc_helper(assoc([1, 1], [0, 2]), n_maxrs=-2)
    with pytest.raises(ShapeMismatchError):
        fg.Associations(np.zeros(3, dtype=np.int64), fg.RowSplits([0, 4]))
    assert fg.find_unique(assoc([10 ** 12, -5], [0, 2])).unique_idx.tolist() == [10 ** 12]
    with pytest.raises(ValueError):
        fg.oc_helper(assoc([1, 1], [0, 2])).m[0, 0] = 5


def test_large_batch_vs_oracle(oracle):
    # 8 events x 25k vertices, 20 objects each, ids = representative vertex ids
    asso, off = generate_associations(200_000, 8, 20, 4242, 0.25)
    a = fg.Associations(asso, fg.RowSplits(off))
    res = fg.oc_helper(a)
    ui, ur, cnt = oracle.find_unique(asso, off)
    assert np.array_equal(res.unique.unique_idx, ui) and np.array_equal(res.unique.unique_rs_asso, ur)
    m, mn, v = oracle.oc_helper(asso, off, ui, ur, int(cnt.max()), int(np.diff(off).max()))
    assert np.array_equal(res.m, m) and np.array_equal(res.m_not, mn) and res.visit_count == v
    # a window cap cutting every split, and a member cap below the counts
    res = fg.oc_helper(a, n_maxuq=100, n_maxrs=10_000)
    m, mn, v = oracle.oc_helper(asso, off, ui, ur, 100, 10_000)
    assert np.array_equal(res.m, m) and np.array_equal(res.m_not, mn) and res.visit_count == v


def test_many_objects_grid_y_loop(oracle):
    # > 65535 objects: the object axis of the grid loops
    n = 140_000
    asso = np.arange(n, dtype=np.int64) // 2
    off = np.array([0, n], dtype=np.int64)
    a = fg.Associations(asso, fg.RowSplits(off))
    res = fg.oc_helper(a, n_maxrs=64, calc_m_not=True)
    assert res.unique.n_unique == n // 2
    ui, ur, _ = oracle.find_unique(asso, off)
    m, mn, v = oracle.oc_helper(asso, off, ui, ur, 2, 64)
    assert np.array_equal(res.m, m) and np.array_equal(res.m_not, mn) and res.visit_count == v


def test_caller_objects_validated_and_counted():
    """a caller-supplied object list is checked on the host (the
    reference raises OutOfRangeError through RowSplits.bounds, G/core.py:80-84)
    and counted like the reference's max_same_count (G/ocgraph.py:137-149),
    including ids the fresh table does not hold (negative background ids)."""
    asso = np.array([-1, 3, 3, -1, 5, 7, -1, 7], np.int64)
    a = fg.Associations(asso, fg.RowSplits([0, 4, 8]))
    bad = fg.UniqueObjects(np.array([3, 7]), np.array([0, 2]))
    with pytest.raises(fg.errors.OutOfRangeError):
        fg.oc_helper(a, bad)
    with pytest.raises(fg.errors.OutOfRangeError):
        fg.max_same_count(a, fg.UniqueObjects(np.array([3]), np.array([-1])))
    top, counts = fg.max_same_count(a, fg.UniqueObjects(np.array([3, -1, 7, 9]),
                                                        np.array([0, 0, 1, 1])))
    assert counts.tolist() == [2, 2, 2, 0] and top == 2
