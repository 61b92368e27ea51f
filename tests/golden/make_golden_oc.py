"""Golden vectors for the association matrices, made by the REAL reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_oc.py

Imports gridknn from /root/reference/pkg/src (ocgraph is pure Python/numpy,
no compiled kernels involved) and records, for association batches drawn with
the reference's own generator (the T/test_ocgraph.py and criterion-5 patterns
of T/test_acceptance.py:230-283), the inputs and find_unique / max_same_count /
oc_helper outputs into tests/golden/reference_oc.npz.  The file travels to the
GPU box; /root/reference does not.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"


def main():
    sys.path.insert(0, REF_SRC)
    import gridknn as g  # noqa: E402
    from gridknn.harness.datasets import generate_associations  # noqa: E402

    out = {}
    cases = []
    # T/test_ocgraph.py::test_matches_brute_enumeration pattern (seeds 0-7)
    for seed in range(8):
        rng = np.random.default_rng(seed)
        n = int(rng.integers(10, 400))
        splits = int(rng.integers(1, 5))
        n = max(n, splits)
        n_obj = int(rng.integers(1, 12))
        uq = int(rng.integers(1, 20))
        rs_cap = int(rng.integers(1, n + 10))
        cases.append((f"brute{seed}", n, splits, n_obj, seed, 0.2, uq, rs_cap))
    # criterion-5 pattern (T/test_acceptance.py:230-250), bounded output sizes
    rng = np.random.default_rng(5000)
    for trial in range(40):
        n = int(rng.integers(20, 2000))
        splits = int(rng.integers(1, 5))
        n_obj = int(rng.integers(1, 51))
        bg = float(rng.random() * 0.5)
        explicit = trial % 3 == 0
        uq = int(rng.integers(1, 30)) if explicit else None
        rs_cap = int(rng.integers(1, n + 5)) if explicit else None
        cases.append((f"crit{trial}", n, splits, n_obj, 5000 + trial, bg, uq, rs_cap))
    cases.append(("big", 10_000, 3, 10, 5095, 0.3, None, None))
    cases.append(("empty_splits", 50, 1, 3, 77, 0.2, None, None))

    for name, n, splits, n_obj, seed, bg, uq, rs_cap in cases:
        a = generate_associations(n, splits=splits, n_objects=n_obj, seed=seed,
                                  background_frac=bg)
        asso = np.asarray(a.asso_idx)
        offsets = np.asarray(a.row_splits.offsets)
        if name == "empty_splits":  # empty rows are legal (T/test_binning.py:177-181)
            offsets = np.array([0, 0, 20, 20, 50, 50], dtype=np.int64)
            a = g.Associations(asso, g.RowSplits(offsets))
        uniq = g.find_unique(a)
        top, counts = g.max_same_count(a, uniq)
        res = g.oc_helper(a, uniq, n_maxuq=uq, n_maxrs=rs_cap)
        res_nm = g.oc_helper(a, uniq, n_maxuq=uq, n_maxrs=rs_cap, calc_m_not=False)
        assert np.array_equal(res.m, res_nm.m) and res_nm.visit_count == res.visit_count
        pre = f"{name}__"
        out[pre + "asso"] = asso
        out[pre + "row_splits"] = offsets
        out[pre + "caps"] = np.array([-1 if uq is None else uq, -1 if rs_cap is None else rs_cap,
                                      res.m.shape[1], res.m_not.shape[1], res.visit_count, top],
                                     dtype=np.int64)
        out[pre + "unique_idx"] = uniq.unique_idx
        out[pre + "unique_rs"] = uniq.unique_rs_asso
        out[pre + "counts"] = counts
        out[pre + "m"] = res.m
        out[pre + "m_not"] = res.m_not
    out["names"] = np.array([c[0] for c in cases])
    path = os.path.join(HERE, "reference_oc.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes,", len(cases), "cases")


if __name__ == "__main__":
    main()
