"""CPU: the C-ABI library loads and exports exactly what include/*.h declares;
argument validation happens before any launch (so it is testable without a
GPU) and maps onto the reference's error types."""

import ctypes
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2511_10442_b200 import _lib, errors

HEADER = os.path.join(ROOT, "include", "fastgraph_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fg_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    assert declared_symbols() == sorted(_lib.EXPORTS)
    for name in declared_symbols():
        assert getattr(L, name) is not None
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = sorted(set(re.findall(r" T (fg_\w+)", out)))
    assert exported == declared_symbols()


def test_library_is_built_for_sm_100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_abi_version_and_error_strings():
    L = _lib.load()
    assert L.fg_abi_version() == 3
    assert L.fg_error_string(0) == b"ok"
    assert b"k must be" in L.fg_error_string(-1)


def test_validation_before_launch():
    L = _lib.load()
    n = ctypes.c_size_t(0)
    assert L.fg_bin_workspace_size(1000, 1, 4, 29, ctypes.byref(n)) == 0 and n.value > 29 ** 4 * 4
    assert L.fg_bin_workspace_size(1000, 1, 6, 29, ctypes.byref(n)) == -3
    def knn(n=10, n_c=4, S=1, d_bin=4, nb=5, k=5, r2=0.0, flags=0):
        return L.fg_knn_fwd(None, None, None, None, None, None, None, n, n_c, S, d_bin, nb, k,
                            None, r2, flags, None, None, None)

    assert knn(k=0) == -1                 # BadK
    assert knn(k=961) == -1
    assert knn(d_bin=6) == -3             # d_bin outside [1, 5]
    assert knn(n_c=3, d_bin=4) == -3      # d_bin > n_coords
    assert knn(n_c=17) == -6              # too many dims
    assert knn(r2=-1.0, flags=0x2) == -7  # negative radius
    assert knn() == -5                    # NULL pointers
    def knn_ws(ws_bytes, n=10, n_c=4, k=5):
        return L.fg_knn_fwd_ws(None, None, None, None, None, None, None, n, n_c, 1, 4, 5, k,
                               None, 0.0, 0, None, None, None, ws_bytes, None)
    assert knn_ws(0, k=0) == -1
    assert knn_ws(0) == -5
    # the tile paths need scratch (d <= 4 tiles; high-dimensional tiles for n_c > 4,
    # k <= 64); the warp-per-query kernel (here k > 64) needs none
    assert L.fg_knn_workspace_size(1000, 4, 1, 4, 29, 40, 0, ctypes.byref(n)) == 0 and n.value > 4000
    assert L.fg_knn_workspace_size(1000, 5, 1, 4, 29, 40, 0, ctypes.byref(n)) == 0 and n.value > 4000
    assert L.fg_knn_workspace_size(1000, 5, 1, 4, 29, 80, 0, ctypes.byref(n)) == 0 and n.value == 0
    assert L.fg_knn_f64_workspace_size(1000, 5, 1, 4, 29, 40, 0, ctypes.byref(n)) == 0 and n.value > 4000
    def knn64(n=10, k=5):
        return L.fg_knn_fwd_f64_ws(None, None, None, None, None, None, None, None, n, 4, 1, 4, 5, k,
                                   None, 0.0, 0, None, None, None, 0, None)
    assert knn64(k=0) == -1 and knn64() == -5
    assert L.fg_knn_workspace_size(1000, 4, 1, 4, 29, 40, _lib.FG_KNN_NO_TILE,
                                   ctypes.byref(n)) == 0 and n.value == 0
    # fused search + GravNet: float32 distances only, reducers validated before any launch
    red = (ctypes.c_int32 * 2)(0, 1)
    def kg(flags=0, k=40, n_feats=64, scale=10.0, reducers=red, n_red=2):
        return L.fg_knn_gravnet_fwd_ws(None, None, None, None, None, None, None, 10, 4, 1, 4, 5, k,
                                       flags, None, n_feats, scale, reducers, n_red, 1, None, None,
                                       None, None, 0, None)
    assert kg(flags=_lib.FG_KNN_D2_F64) == -2
    assert kg(k=0) == -1
    assert kg(scale=0.0) == -2
    assert kg(n_red=5) == -2
    assert kg() == -5  # NULL pointers
    # association matrices: capacities checked first, then pointers
    assert L.fg_oc_matrices(None, None, 1, None, None, 3, 0, 5, 10, None, None, None, None, 0,
                            None) == -8
    assert L.fg_oc_matrices(None, None, 1, None, None, 3, 4, 5, 10, None, None, None, None, 0,
                            None) == -5
    assert L.fg_oc_unique_workspace_size(1000, ctypes.byref(n)) == 0 and n.value > 16 * 1000
    assert L.fg_oc_matrices_workspace_size(10, 5000, ctypes.byref(n)) == 0 and n.value >= 120
    for rc, exc in ((-8, errors.BadCapacityError), (-1, errors.BadKError), (-3, errors.TooFewDimsError),
                    (-6, errors.BadShapeError), (-7, errors.BadKError)):
        with pytest.raises(exc):
            _lib.check(rc)


def test_oracle_is_not_linked_into_the_product():
    """The product path never touches oracle/: no import, no symbol."""
    pkg = os.path.join(ROOT, "paper_2511_10442_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py") or f.endswith(".cu") or f.endswith(".cuh"):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
    out = subprocess.run(["nm", "-D", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "orc_" not in out
