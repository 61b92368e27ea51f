"""CPU: the association-matrix oracle (oracle/oracle.py find_unique /
oc_helper) and the association generator, pinned to the reference: its
frozen known answers (T/test_ocgraph.py) and golden vectors made by running
the real gridknn.ocgraph (tests/golden/make_golden_oc.py)."""

import numpy as np
import pytest

from conftest import oc_case
from paper_2511_10442_b200.datasets import generate_associations


def resolve_caps(c, counts):
    sizes = np.diff(c["row_splits"])
    uq = c["n_maxuq"] if c["n_maxuq"] is not None else max(1, int(counts.max()) if counts.size else 0)
    rs = c["n_maxrs"] if c["n_maxrs"] is not None else max(1, int(sizes.max()) if sizes.size else 0)
    return uq, rs


def test_oc_kats(oracle):
    # T/test_ocgraph.py:16-36 (find_unique) and :59-118 (oc_helper frozen cases)
    ui, ur, cnt = oracle.find_unique([7, 7, 3, 7, 3], [0, 5])
    assert ui.tolist() == [7, 3] and ur.tolist() == [0, 0] and cnt.tolist() == [3, 2]
    ui, ur, _ = oracle.find_unique([5, -1, 2, 5, -7, 2, 9], [0, 4, 7])
    assert ui.tolist() == [5, 2, 2, 9] and ur.tolist() == [0, 0, 1, 1]
    ui, ur, _ = oracle.find_unique([1, 1, 1, 1], [0, 2, 4])
    assert ui.tolist() == [1, 1] and ur.tolist() == [0, 1]
    m, mn, v = oracle.oc_helper([7, 7, 3, 7, 3], [0, 5], [7, 3], [0, 0], 4, 5)
    assert m.tolist() == [[0, 1, 3, -1], [2, 4, -1, -1]]
    assert mn.tolist() == [[2, 4, -1, -1, -1], [0, 1, 3, -1, -1]] and v == 10
    m, mn, v = oracle.oc_helper([7, 3, 7, 7, 3], [0, 5], [7, 3], [0, 0], 5, 3)
    assert m.tolist() == [[0, 2, -1, -1, -1], [1, -1, -1, -1, -1]]
    assert mn.tolist() == [[1, -1, -1], [0, 2, -1]] and v == 6


def test_oc_oracle_vs_reference_golden(oracle, golden_oc):
    names = [str(x) for x in golden_oc["names"]]
    assert len(names) >= 50
    for name in names:
        c = oc_case(golden_oc, name)
        ui, ur, cnt = oracle.find_unique(c["asso"], c["row_splits"])
        assert np.array_equal(ui, c["unique_idx"]) and np.array_equal(ur, c["unique_rs"]), name
        assert np.array_equal(cnt, c["counts"]), name
        uq, rs = resolve_caps(c, cnt)
        assert (uq, rs) == (c["cap_uq"], c["cap_rs"]), name
        m, mn, v = oracle.oc_helper(c["asso"], c["row_splits"], ui, ur, uq, rs)
        assert np.array_equal(m, c["m"]) and np.array_equal(mn, c["m_not"]), name
        assert v == c["visits"], name


@pytest.mark.parametrize("name", ["brute0", "brute5", "crit3", "crit17", "big"])
def test_association_generator_matches_reference(golden_oc, name):
    c = oc_case(golden_oc, name)
    if name.startswith("brute"):
        seed = int(name[5:])
        rng = np.random.default_rng(seed)
        n = int(rng.integers(10, 400))
        splits = int(rng.integers(1, 5))
        n = max(n, splits)
        asso, off = generate_associations(n, splits, int(rng.integers(1, 12)), seed)
    else:
        # criterion-5 trials: replay the trial parameter stream
        rng = np.random.default_rng(5000)
        params = {}
        for trial in range(40):
            n = int(rng.integers(20, 2000))
            splits = int(rng.integers(1, 5))
            n_obj = int(rng.integers(1, 51))
            bg = float(rng.random() * 0.5)
            if trial % 3 == 0:
                rng.integers(1, 30)
                rng.integers(1, n + 5)
            params[f"crit{trial}"] = (n, splits, n_obj, 5000 + trial, bg)
        params["big"] = (10_000, 3, 10, 5095, 0.3)
        n, splits, n_obj, seed, bg = params[name]
        asso, off = generate_associations(n, splits, n_obj, seed, bg)
    assert np.array_equal(asso, c["asso"]) and np.array_equal(off, c["row_splits"])
