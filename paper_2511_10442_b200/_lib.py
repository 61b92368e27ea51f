"""ctypes binding of the C ABI (``include/fastgraph_b200.h``).

The product path has exactly one implementation: the sm_100a kernels in
``libfastgraph_b200.so``.  If the library is missing this module raises
``BackendUnavailableError`` -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os

from .errors import (BackendUnavailableError, BadCapacityError, BadKError, BadShapeError, GridKnnError,
                     ShapeMismatchError, TooFewDimsError)

PKG = os.path.dirname(os.path.abspath(__file__))
# FG_LIB_PATH selects an experimental build of the same ABI (benchmarking only)
LIB_PATH = os.environ.get("FG_LIB_PATH") or os.path.join(PKG, "libfastgraph_b200.so")

FG_KNN_USE_DIRECTION = 0x1
FG_KNN_USE_MAX_R2 = 0x2
FG_KNN_EXHAUSTIVE = 0x4
FG_KNN_D2_F64 = 0x8
FG_KNN_STATS = 0x100
FG_KNN_NO_TILE = 0x200
FG_KNN_FUSED_EPI = 0x800
FG_KNN_NO_HD = 0x1000
FG_KNN_FORCE_HD = 0x2000
FG_BWD_F64 = 0x1
FG_BWD_DETERMINISTIC = 0x2
FG_BWD_X64 = 0x4
FG_BWD_G64 = 0x8
FG_REDUCE_MEAN = 0
FG_REDUCE_MAX = 1

# every symbol include/fastgraph_b200.h declares
EXPORTS = (
    "fg_bin_workspace_size", "fg_bin_by_coordinates", "fg_index_replacer", "fg_knn_fwd",
    "fg_knn_bwd_workspace_size", "fg_knn_bwd", "fg_gravnet_fwd",
    "fg_gravnet_bwd_workspace_size", "fg_gravnet_bwd", "fg_error_string", "fg_abi_version",
    "fg_launch_count", "fg_knn_stats", "fg_knn_workspace_size", "fg_knn_fwd_ws",
    "fg_knn_gravnet_fwd_ws", "fg_oc_unique_workspace_size", "fg_oc_find_unique",
    "fg_oc_matrices_workspace_size", "fg_oc_matrices", "fg_brute_knn",
    "fg_bin_by_coordinates_f64", "fg_knn_f64_workspace_size", "fg_knn_fwd_f64_ws",
    "fg_brute_knn_f64",
)

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_U32 = ctypes.c_uint32
_D = ctypes.c_double
_SZ = ctypes.POINTER(ctypes.c_size_t)

_SIGS = {
    "fg_bin_workspace_size": ([_I64, _I32, _I32, _I32, _SZ], ctypes.c_int),
    "fg_bin_by_coordinates": ([_P, _I64, _I32, _P, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _P,
                               ctypes.c_size_t, _P], ctypes.c_int),
    "fg_bin_by_coordinates_f64": ([_P, _I64, _I32, _P, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P,
                                   _P, ctypes.c_size_t, _P], ctypes.c_int),
    "fg_knn_f64_workspace_size": ([_I64, _I32, _I32, _I32, _I32, _I32, _U32, _SZ], ctypes.c_int),
    "fg_knn_fwd_f64_ws": ([_P, _P, _P, _P, _P, _P, _P, _P, _I64, _I32, _I32, _I32, _I32, _I32, _P,
                           _D, _U32, _P, _P, _P, ctypes.c_size_t, _P], ctypes.c_int),
    "fg_index_replacer": ([_P, _I64, _P, _I64, _P], ctypes.c_int),
    "fg_knn_fwd": ([_P, _P, _P, _P, _P, _P, _P, _I64, _I32, _I32, _I32, _I32, _I32, _P, _D, _U32,
                    _P, _P, _P], ctypes.c_int),
    "fg_knn_workspace_size": ([_I64, _I32, _I32, _I32, _I32, _I32, _U32, _SZ], ctypes.c_int),
    "fg_knn_fwd_ws": ([_P, _P, _P, _P, _P, _P, _P, _I64, _I32, _I32, _I32, _I32, _I32, _P, _D,
                       _U32, _P, _P, _P, ctypes.c_size_t, _P], ctypes.c_int),
    "fg_knn_gravnet_fwd_ws": ([_P, _P, _P, _P, _P, _P, _P, _I64, _I32, _I32, _I32, _I32, _I32,
                               _U32, _P, _I32, _D, _P, _I32, _I32, _P, _P, _P, _P,
                               ctypes.c_size_t, _P], ctypes.c_int),
    "fg_knn_bwd_workspace_size": ([_I64, _I32, _I32, _SZ], ctypes.c_int),
    "fg_knn_bwd": ([_P, _I64, _I32, _P, _I32, _P, _P, _P, _I32, _P, ctypes.c_size_t, _P],
                   ctypes.c_int),
    "fg_gravnet_fwd": ([_P, _I64, _I32, _P, _P, _I32, _D, _P, _I32, _I32, _P, _P, _P],
                       ctypes.c_int),
    "fg_gravnet_bwd_workspace_size": ([_I64, _I32, _I32, _SZ], ctypes.c_int),
    "fg_gravnet_bwd": ([_P, _I64, _I32, _P, _P, _I32, _D, _P, _I32, _I32, _P, _P, _P, _P, _P,
                        ctypes.c_size_t, _P], ctypes.c_int),
    "fg_oc_unique_workspace_size": ([_I64, _SZ], ctypes.c_int),
    "fg_oc_find_unique": ([_P, _I64, _P, _I32, _P, _P, _P, _P, _P, ctypes.c_size_t, _P],
                          ctypes.c_int),
    "fg_oc_matrices_workspace_size": ([_I64, _I64, _SZ], ctypes.c_int),
    "fg_oc_matrices": ([_P, _P, _I32, _P, _P, _I64, _I64, _I64, _I64, _P, _P, _P, _P,
                        ctypes.c_size_t, _P], ctypes.c_int),
    "fg_brute_knn_f64": ([_P, _I64, _I32, _P, _I32, _P, _I64, _P, _D, _U32, _I32, _P, _P, _P],
                         ctypes.c_int),
    "fg_brute_knn": ([_P, _I64, _I32, _P, _I32, _P, _I64, _P, _D, _U32, _I32, _P, _P, _P],
                     ctypes.c_int),
    "fg_error_string": ([ctypes.c_int], ctypes.c_char_p),
    "fg_abi_version": ([], ctypes.c_int),
    "fg_launch_count": ([], ctypes.c_uint64),
    "fg_knn_stats": ([_P, _I32, _I32], ctypes.c_int),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load the CUDA library (raises BackendUnavailableError when absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise BackendUnavailableError(
            f"{path} is missing: build it with `python -m paper_2511_10442_b200._build` "
            "(there is no CPU fallback)")
    try:
        L = ctypes.CDLL(path)
    except OSError as exc:  # pragma: no cover - depends on the host
        raise BackendUnavailableError(f"cannot load {path}: {exc}") from exc
    for name, (args, res) in _SIGS.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res
    _lib = L
    return L


def check(rc: int, what: str = "") -> None:
    """Map an fg_status / cudaError_t to the reference's exception types."""
    if rc == 0:
        return
    msg = load().fg_error_string(rc).decode()
    if what:
        msg = f"{what}: {msg}"
    if rc == -1 or rc == -7:
        raise BadKError(msg)
    if rc == -3:
        raise TooFewDimsError(msg)
    if rc in (-2, -6, -9):
        raise BadShapeError(msg)
    if rc == -4:
        raise ShapeMismatchError(msg)
    if rc == -8:
        raise BadCapacityError(msg)
    raise GridKnnError(f"{msg} (code {rc})")


def size_out(fn, *args) -> int:
    n = ctypes.c_size_t(0)
    check(fn(*args, ctypes.byref(n)), fn.__name__)
    return int(n.value)


def launch_count() -> int:
    return int(load().fg_launch_count())
