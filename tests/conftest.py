import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O  # test infrastructure only
    O.lib()
    return O


GOLDEN_CASES = ["u3", "c4", "u2", "u5", "u8", "u10", "m3", "r4"]


def golden_case(g, name):
    pre = f"{name}__"
    meta = g[pre + "meta"]
    k, d_bin, n_bins, use_mask, mr2 = int(meta[0]), int(meta[1]), int(meta[2]), int(meta[3]), \
        float(meta[4])
    return {
        "coords": g[pre + "coords"],
        "row_splits": g[pre + "row_splits"],
        "k": k, "d_bin": d_bin, "n_bins": n_bins,
        "mask": g[pre + "mask"] if use_mask else None,
        "max_r2": None if mr2 < 0 else mr2,
        **{key: g[pre + key] for key in ("bin_idx", "sort_order", "bin_bounds", "dim_mins",
                                           "widths", "knn_idx_raw", "knn_d2_raw",
                                           "knn_idx_sorted", "knn_d2_sorted", "brute_k1_idx",
                                           "brute_k1_d2", "upstream", "grad_raw_rows")},
    }


GOLDEN_OC = os.path.join(ROOT, "tests", "golden", "reference_oc.npz")


@pytest.fixture(scope="session")
def golden_oc():
    return np.load(GOLDEN_OC)


def oc_case(g, name):
    """One association batch + the reference's find_unique / oc_helper outputs
    (tests/golden/make_golden_oc.py)."""
    pre = f"{name}__"
    caps = g[pre + "caps"]
    return {
        "asso": g[pre + "asso"], "row_splits": g[pre + "row_splits"],
        "n_maxuq": None if caps[0] < 0 else int(caps[0]),
        "n_maxrs": None if caps[1] < 0 else int(caps[1]),
        "cap_uq": int(caps[2]), "cap_rs": int(caps[3]), "visits": int(caps[4]),
        "top": int(caps[5]),
        **{key: g[pre + key] for key in ("unique_idx", "unique_rs", "counts", "m", "m_not")},
    }
