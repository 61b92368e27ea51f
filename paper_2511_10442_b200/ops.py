"""torch.library registration of the FastGraph op surface (namespace
``fastgraph``) over the C ABI of ``libfastgraph_b200.so``.

Ops (all CUDA, all enqueued on torch's current stream, no host sync):

* ``fastgraph::bin_by_coordinates(coords, row_splits, d_bin, n_bins)``
    -> (bin_idx i64[N], sort_order i32[N], bin_bounds i32[S*n_bins^d_bin+1],
        dim_mins f64[S,d_bin], widths f64[S,d_bin], sorted_coords f32[N,4*ceil(d/4)])
    replaces build_bin_index -> build_index (G/binning.py:136-170, pyx:66-139).
* ``fastgraph::index_replacer(to_be_replaced, replacements)``
    out = replacements[x] for x >= 0 (pyx:262's implicit sort_order lookup).
* ``fastgraph::binned_select_knn(coords, row_splits, <index tensors>, K, d_bin,
  n_bins, direction, max_radius2, exhaustive, d2_f64)`` -> (idx i32[N,K], d2[N,K])
    replaces binned_select_knn -> binned_knn (G/knn.py:82-115, pyx:188-329);
    differentiable w.r.t. ``coords`` (backward = binned_select_knn_grad).
* ``fastgraph::binned_select_knn_grad(grad_d2, idx, coords)`` -> grad_coords
    replaces knn_backward (G/knn.py:135-168).
* ``fastgraph::gravnet_aggregate(feats, idx, d2, weight_scale, reducers,
  include_self)`` -> out[N, F*len(reducers)], differentiable w.r.t. feats, d2
    replaces G/gravnet.py:75-97; backward ``gravnet_aggregate_grad``
    replaces G/gravnet.py:100-150.

Every op has a fake (meta) implementation, so it traces under torch.compile /
FakeTensor without running the kernels.  There is no CPU implementation: a
CPU tensor raises BackendUnavailableError.
"""

from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import torch
from torch import Tensor

from . import _lib
from .errors import BackendUnavailableError, BadShapeError, ShapeMismatchError

_LIB_NS = "fastgraph"
_DEBUG_FLAGS = 0  # OR-ed into fg_knn_fwd flags (diagnostics only, see set_debug_flags)


def set_debug_flags(flags: int) -> None:
    """Diagnostics: e.g. ``set_debug_flags(_lib.FG_KNN_STATS)`` makes every search
    launch count its events (read them with ``knn_stats()``)."""
    global _DEBUG_FLAGS
    _DEBUG_FLAGS = int(flags)


def knn_stats(reset: bool = True) -> dict:
    names = ("queries", "regions", "chunks", "appends", "compactions", "spec_fail", "exact_epi",
             "rows", "tiles", "tile_candidates", "tile_redo", "tile_fail", "tile_expanded",
             "tile_evaluated", "hd_tiles", "hd_chunks", "hd_stages", "hd_max_tile_cycles", "hd_cuts")
    buf = (ctypes.c_uint64 * len(names))()
    _lib.check(_lib.load().fg_knn_stats(ctypes.cast(buf, ctypes.c_void_p), len(names), int(reset)))
    return dict(zip(names, [int(x) for x in buf]))


def _order(order: Optional[Tensor], n: int, device) -> Optional[Tensor]:
    """Validated int32 device copy of an optional row visit order."""
    if order is None:
        return None
    if order.numel() != n:
        raise ShapeMismatchError(f"order covers {order.numel()} rows, there are {n}")
    return order.to(device=device, dtype=torch.int32).contiguous()


def _p(t: Optional[Tensor]):
    if t is None or t.numel() == 0:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _stream(t: Tensor):
    return ctypes.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _require_cuda(*ts: Tensor) -> None:
    for t in ts:
        if t is not None and t.device.type != "cuda":
            raise BackendUnavailableError(
                "fastgraph ops run on CUDA tensors only (no CPU fallback); got "
                f"a {t.device.type} tensor")


def coord_stride(n_coords: int) -> int:
    return 4 * ((n_coords + 3) // 4)


def _ws(nbytes: int, device) -> Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


# ---------------------------------------------------------------- binning
@torch.library.custom_op(f"{_LIB_NS}::bin_by_coordinates", mutates_args=())
def bin_by_coordinates(coords: Tensor, row_splits: Tensor, d_bin: int,
                       n_bins: int) -> tuple[Tensor, Tensor, Tensor, Tensor, Tensor, Tensor]:
    _require_cuda(coords)
    L = _lib.load()
    dev = coords.device
    if coords.dim() != 2:
        raise BadShapeError("coords must be 2-d (n_vertices, n_coords)")
    # float64 coordinates (the reference's dtype) are binned from their float64
    # values: every array bit-identical to the reference for any finite input
    x64 = coords.dtype == torch.float64
    coords = coords.contiguous() if x64 else coords.to(torch.float32).contiguous()
    rs = row_splits.to(device=dev, dtype=torch.int64).contiguous()
    n, n_c = coords.shape
    S = rs.numel() - 1
    total = int(n_bins) ** int(d_bin)
    bin_idx = torch.empty(n, dtype=torch.int64, device=dev)
    sort_order = torch.empty(n, dtype=torch.int32, device=dev)
    bounds = torch.empty(S * total + 1, dtype=torch.int32, device=dev)
    mins = torch.empty((S, d_bin), dtype=torch.float64, device=dev)
    widths = torch.empty((S, d_bin), dtype=torch.float64, device=dev)
    sorted_coords = torch.empty((n, coord_stride(n_c)), dtype=torch.float32, device=dev)
    nbytes = _lib.size_out(L.fg_bin_workspace_size, n, S, d_bin, n_bins)
    ws = _ws(nbytes, dev)
    fn = L.fg_bin_by_coordinates_f64 if x64 else L.fg_bin_by_coordinates
    _lib.check(fn(_p(coords), n, n_c, _p(rs), S, d_bin, n_bins, _p(bin_idx), _p(sort_order),
                  _p(bounds), _p(mins), _p(widths), _p(sorted_coords), _p(ws), ws.numel(),
                  _stream(coords)), "bin_by_coordinates")
    return bin_idx, sort_order, bounds, mins, widths, sorted_coords


@bin_by_coordinates.register_fake
def _bin_fake(coords, row_splits, d_bin, n_bins):
    n, n_c = coords.shape
    S = row_splits.shape[0] - 1
    total = int(n_bins) ** int(d_bin)
    e = coords.new_empty
    return (e(n, dtype=torch.int64), e(n, dtype=torch.int32), e(S * total + 1, dtype=torch.int32),
            e((S, d_bin), dtype=torch.float64), e((S, d_bin), dtype=torch.float64),
            e((n, coord_stride(n_c)), dtype=torch.float32))


@torch.library.custom_op(f"{_LIB_NS}::index_replacer", mutates_args=())
def index_replacer(to_be_replaced: Tensor, replacements: Tensor) -> Tensor:
    _require_cuda(to_be_replaced, replacements)
    out = to_be_replaced.to(torch.int32).contiguous().clone()
    rep = replacements.to(torch.int32).contiguous()
    _lib.check(_lib.load().fg_index_replacer(_p(out), out.numel(), _p(rep), rep.numel(),
                                             _stream(out)), "index_replacer")
    return out


@index_replacer.register_fake
def _ir_fake(to_be_replaced, replacements):
    return torch.empty_like(to_be_replaced, dtype=torch.int32)


# ---------------------------------------------------------------- search
@torch.library.custom_op(f"{_LIB_NS}::binned_select_knn", mutates_args=())
def binned_select_knn(coords: Tensor, row_splits: Tensor, bin_idx: Tensor, sort_order: Tensor,
                      bin_bounds: Tensor, dim_mins: Tensor, widths: Tensor,
                      sorted_coords: Tensor, K: int, d_bin: int, n_bins: int,
                      direction: Optional[Tensor] = None,
                      max_radius2: Optional[float] = None, exhaustive: bool = False,
                      d2_f64: bool = False) -> tuple[Tensor, Tensor]:
    _require_cuda(coords, sorted_coords)
    L = _lib.load()
    dev = sorted_coords.device
    n, n_c = coords.shape
    rs = row_splits.to(device=dev, dtype=torch.int64).contiguous()
    S = rs.numel() - 1
    flags = 0
    dir_t = None
    if direction is not None:
        if direction.numel() != n:
            raise ShapeMismatchError(f"direction covers {direction.numel()} vertices, cloud has {n}")
        dir_t = direction.to(device=dev, dtype=torch.int8).contiguous()
        flags |= _lib.FG_KNN_USE_DIRECTION
    if max_radius2 is not None:
        flags |= _lib.FG_KNN_USE_MAX_R2
    if exhaustive:
        flags |= _lib.FG_KNN_EXHAUSTIVE
    if d2_f64:
        flags |= _lib.FG_KNN_D2_F64
    flags |= _DEBUG_FLAGS
    idx = torch.empty((n, K), dtype=torch.int32, device=dev)
    d2 = torch.empty((n, K), dtype=torch.float64 if d2_f64 else torch.float32, device=dev)
    if coords.dtype == torch.float64:
        # exact float64 keys from the float64 coordinates (fg_knn_fwd_f64_ws)
        x = coords.detach().to(dev).contiguous()
        nbytes = _lib.size_out(L.fg_knn_f64_workspace_size, n, n_c, S, d_bin, n_bins, K, flags)
        ws = _ws(nbytes, dev)
        _lib.check(L.fg_knn_fwd_f64_ws(_p(x), _p(sorted_coords), _p(sort_order), _p(bin_idx),
                                       _p(bin_bounds), _p(rs), _p(dim_mins), _p(widths), n, n_c,
                                       S, d_bin, n_bins, K, _p(dir_t),
                                       float(max_radius2 or 0.0), flags, _p(idx), _p(d2), _p(ws),
                                       ws.numel(), _stream(sorted_coords)),
                   "binned_select_knn (float64 coordinates)")
        return idx, d2
    nbytes = _lib.size_out(L.fg_knn_workspace_size, n, n_c, S, d_bin, n_bins, K, flags)
    ws = _ws(nbytes, dev)
    _lib.check(L.fg_knn_fwd_ws(_p(sorted_coords), _p(sort_order), _p(bin_idx), _p(bin_bounds),
                               _p(rs), _p(dim_mins), _p(widths), n, n_c, S, d_bin, n_bins, K,
                               _p(dir_t), float(max_radius2 or 0.0), flags, _p(idx), _p(d2),
                               _p(ws), ws.numel(), _stream(sorted_coords)), "binned_select_knn")
    return idx, d2


@binned_select_knn.register_fake
def _knn_fake(coords, row_splits, bin_idx, sort_order, bin_bounds, dim_mins, widths,
              sorted_coords, K, d_bin, n_bins, direction=None, max_radius2=None,
              exhaustive=False, d2_f64=False):
    n = coords.shape[0]
    return (coords.new_empty((n, K), dtype=torch.int32),
            coords.new_empty((n, K), dtype=torch.float64 if d2_f64 else torch.float32))


@torch.library.custom_op(f"{_LIB_NS}::binned_select_knn_grad", mutates_args=())
def binned_select_knn_grad(grad_d2: Tensor, idx: Tensor, coords: Tensor,
                           order: Optional[Tensor] = None, deterministic: bool = False) -> Tensor:
    _require_cuda(grad_d2, idx, coords)
    L = _lib.load()
    n, n_c = coords.shape
    k = idx.shape[1]
    if grad_d2.shape != idx.shape:
        raise ShapeMismatchError(f"upstream shape {tuple(grad_d2.shape)} != neighbour shape "
                                 f"{tuple(idx.shape)}")
    if idx.shape[0] != n:
        raise ShapeMismatchError(f"neighbours cover {idx.shape[0]} vertices, cloud has {n}")
    # float64 inputs keep their dtype (terms formed as numpy forms them); the
    # deterministic kernel takes float32 inputs
    x64 = coords.dtype == torch.float64 and not deterministic
    g64 = grad_d2.dtype == torch.float64 and not deterministic
    c = coords.contiguous() if x64 else coords.to(torch.float32).contiguous()
    g = grad_d2.contiguous() if g64 else grad_d2.to(torch.float32).contiguous()
    ix = idx.to(torch.int32).contiguous()
    out_f64 = coords.dtype == torch.float64
    grad = torch.empty((n, n_c), dtype=torch.float64 if out_f64 else torch.float32,
                       device=coords.device)
    ws = _ws(_lib.size_out(L.fg_knn_bwd_workspace_size, n, n_c, k), coords.device)
    od = _order(order, n, coords.device)
    flags = (_lib.FG_BWD_F64 if out_f64 else 0) | (_lib.FG_BWD_DETERMINISTIC if deterministic else 0)
    flags |= (_lib.FG_BWD_X64 if x64 else 0) | (_lib.FG_BWD_G64 if g64 else 0)
    _lib.check(L.fg_knn_bwd(_p(c), n, n_c, _p(ix), k, _p(g), _p(od), _p(grad), flags,
                            _p(ws), ws.numel(), _stream(c)), "binned_select_knn_grad")
    return grad


@binned_select_knn_grad.register_fake
def _knn_grad_fake(grad_d2, idx, coords, order=None, deterministic=False):
    return torch.empty_like(coords)


def _knn_setup(ctx, inputs, output):
    # inputs[3] = sort_order: the backward visits rows in spatial order
    ctx.save_for_backward(inputs[0], output[0], inputs[3])
    ctx.coords_dtype = inputs[0].dtype


def _knn_backward(ctx, grad_idx, grad_d2):
    coords, idx, order = ctx.saved_tensors
    if grad_d2 is None:
        g = None
    else:
        g = binned_select_knn_grad(grad_d2, idx, coords, order).to(ctx.coords_dtype)
    return (g,) + (None,) * 14


binned_select_knn.register_autograd(_knn_backward, setup_context=_knn_setup)


# ---------------------------------------------------------------- GravNet
def _check_red(reducers: Sequence[int]) -> Tensor:
    return torch.tensor(list(reducers), dtype=torch.int32)


@torch.library.custom_op(f"{_LIB_NS}::gravnet_aggregate", mutates_args=())
def gravnet_aggregate(feats: Tensor, idx: Tensor, d2: Tensor, weight_scale: float,
                      reducers: list[int], include_self: bool,
                      order: Optional[Tensor] = None) -> Tensor:
    """``order`` (optional): row visit order, e.g. the bin index's sort_order."""
    _require_cuda(feats, idx, d2)
    n, F = feats.shape
    k = idx.shape[1]
    f = feats.to(torch.float32).contiguous()
    ix = idx.to(torch.int32).contiguous()
    dd = d2.to(torch.float32).contiguous()
    red = _check_red(reducers)
    od = _order(order, n, feats.device)
    out = torch.empty((n, F * red.numel()), dtype=torch.float32, device=feats.device)
    _lib.check(_lib.load().fg_gravnet_fwd(_p(f), n, F, _p(ix), _p(dd), k, float(weight_scale),
                                          ctypes.c_void_p(red.data_ptr()), red.numel(),
                                          int(include_self), _p(od), _p(out),
                                          _stream(f)),
               "gravnet_aggregate")
    return out


@gravnet_aggregate.register_fake
def _gn_fake(feats, idx, d2, weight_scale, reducers, include_self, order=None):
    return feats.new_empty((feats.shape[0], feats.shape[1] * len(reducers)), dtype=torch.float32)


@torch.library.custom_op(f"{_LIB_NS}::gravnet_aggregate_grad", mutates_args=())
def gravnet_aggregate_grad(grad_out: Tensor, feats: Tensor, idx: Tensor, d2: Tensor,
                           weight_scale: float, reducers: list[int], include_self: bool,
                           order: Optional[Tensor] = None) -> tuple[Tensor, Tensor]:
    _require_cuda(grad_out, feats, idx, d2)
    L = _lib.load()
    n, F = feats.shape
    k = idx.shape[1]
    red = _check_red(reducers)
    if tuple(grad_out.shape) != (n, F * red.numel()):
        raise ShapeMismatchError(f"upstream shape {tuple(grad_out.shape)} != {(n, F * red.numel())}")
    f = feats.to(torch.float32).contiguous()
    ix = idx.to(torch.int32).contiguous()
    dd = d2.to(torch.float32).contiguous()
    up = grad_out.to(torch.float32).contiguous()
    od = _order(order, n, feats.device)
    gf = torch.empty((n, F), dtype=torch.float32, device=feats.device)
    gd = torch.empty((n, k), dtype=torch.float32, device=feats.device)
    ws = _ws(_lib.size_out(L.fg_gravnet_bwd_workspace_size, n, F, k), feats.device)
    _lib.check(L.fg_gravnet_bwd(_p(f), n, F, _p(ix), _p(dd), k, float(weight_scale),
                                ctypes.c_void_p(red.data_ptr()), red.numel(), int(include_self),
                                _p(od), _p(up), _p(gf), _p(gd), _p(ws), ws.numel(),
                                _stream(f)),
               "gravnet_aggregate_grad")
    return gf, gd


@gravnet_aggregate_grad.register_fake
def _gn_grad_fake(grad_out, feats, idx, d2, weight_scale, reducers, include_self, order=None):
    return (torch.empty_like(feats, dtype=torch.float32),
            torch.empty_like(d2, dtype=torch.float32))


def _gn_setup(ctx, inputs, output):
    feats, idx, d2, scale, reducers, include_self, order = inputs
    ctx.save_for_backward(feats, idx, d2, order)
    ctx.args = (scale, list(reducers), include_self)
    ctx.dtypes = (feats.dtype, d2.dtype)


def _gn_backward(ctx, grad_out):
    feats, idx, d2, order = ctx.saved_tensors
    scale, reducers, include_self = ctx.args
    gf, gd = gravnet_aggregate_grad(grad_out, feats, idx, d2, scale, reducers, include_self, order)
    return gf.to(ctx.dtypes[0]), None, gd.to(ctx.dtypes[1]), None, None, None, None


gravnet_aggregate.register_autograd(_gn_backward, setup_context=_gn_setup)


# ---------------------------------------------------------------- fused search + GravNet
@torch.library.custom_op(f"{_LIB_NS}::knn_gravnet", mutates_args=())
def knn_gravnet(coords: Tensor, row_splits: Tensor, bin_idx: Tensor, sort_order: Tensor,
                bin_bounds: Tensor, dim_mins: Tensor, widths: Tensor, sorted_coords: Tensor,
                K: int, d_bin: int, n_bins: int, feats: Tensor, weight_scale: float,
                reducers: list[int], include_self: bool) -> tuple[Tensor, Tensor, Tensor]:
    """binned_select_knn (float32 distances) + gravnet_aggregate of its rows
    (the GravNetOp forward): -> (idx, d2, aggregated
    features) from one C-ABI call, differentiable w.r.t. coords and feats."""
    _require_cuda(coords, sorted_coords, feats)
    L = _lib.load()
    dev = sorted_coords.device
    n, n_c = coords.shape
    if feats.shape[0] != n:
        raise ShapeMismatchError(f"{feats.shape[0]} feature rows for {n} vertices")
    rs = row_splits.to(device=dev, dtype=torch.int64).contiguous()
    S = rs.numel() - 1
    F = feats.shape[1]
    f = feats.to(torch.float32).contiguous()
    red = _check_red(reducers)
    flags = _DEBUG_FLAGS
    idx = torch.empty((n, K), dtype=torch.int32, device=dev)
    d2 = torch.empty((n, K), dtype=torch.float32, device=dev)
    agg = torch.empty((n, F * red.numel()), dtype=torch.float32, device=dev)
    nbytes = _lib.size_out(L.fg_knn_workspace_size, n, n_c, S, d_bin, n_bins, K, flags)
    ws = _ws(nbytes, dev)
    _lib.check(L.fg_knn_gravnet_fwd_ws(
        _p(sorted_coords), _p(sort_order), _p(bin_idx), _p(bin_bounds), _p(rs), _p(dim_mins),
        _p(widths), n, n_c, S, d_bin, n_bins, K, flags, _p(f), F, float(weight_scale),
        ctypes.c_void_p(red.data_ptr()), red.numel(), int(include_self), _p(idx), _p(d2),
        _p(agg), _p(ws), ws.numel(), _stream(sorted_coords)), "knn_gravnet")
    return idx, d2, agg


@knn_gravnet.register_fake
def _kg_fake(coords, row_splits, bin_idx, sort_order, bin_bounds, dim_mins, widths, sorted_coords,
             K, d_bin, n_bins, feats, weight_scale, reducers, include_self):
    n = coords.shape[0]
    return (coords.new_empty((n, K), dtype=torch.int32),
            coords.new_empty((n, K), dtype=torch.float32),
            feats.new_empty((n, feats.shape[1] * len(reducers)), dtype=torch.float32))


def _kg_setup(ctx, inputs, output):
    coords, order, feats = inputs[0], inputs[3], inputs[11]
    ctx.save_for_backward(coords, output[0], output[1], feats, order)
    ctx.args = (inputs[12], list(inputs[13]), inputs[14])
    ctx.dtypes = (coords.dtype, feats.dtype)


def _kg_backward(ctx, grad_idx, grad_d2, grad_agg):
    coords, idx, d2, feats, order = ctx.saved_tensors
    scale, reducers, include_self = ctx.args
    gd, gf = grad_d2, None
    if grad_agg is not None:
        gf, gd_agg = gravnet_aggregate_grad(grad_agg, feats, idx, d2, scale, reducers,
                                            include_self, order)
        gd = gd_agg if gd is None else gd + gd_agg
        gf = gf.to(ctx.dtypes[1])
    gc = None if gd is None else binned_select_knn_grad(gd, idx, coords, order).to(ctx.dtypes[0])
    return (gc,) + (None,) * 10 + (gf, None, None, None)


knn_gravnet.register_autograd(_kg_backward, setup_context=_kg_setup)


# ---------------------------------------------------------------- brute force (verifier)
@torch.library.custom_op(f"{_LIB_NS}::brute_knn", mutates_args=())
def brute_knn(coords: Tensor, row_splits: Tensor, K: int, queries: Optional[Tensor] = None,
              direction: Optional[Tensor] = None,
              max_radius2: Optional[float] = None) -> tuple[Tensor, Tensor]:
    """Brute-force exact kNN (pyx:335-409, G/knn.py:118-132) with its own
    kernel (csrc/fg_verify.cu, no code shared with the binned search): ->
    (idx i32 [Q, K], d2 f64 [Q, K]) for the rows ``queries`` (default all),
    canonical (d2, index) order."""
    _require_cuda(coords)
    L = _lib.load()
    dev = coords.device
    n, n_c = coords.shape
    x64 = coords.dtype == torch.float64
    c = coords.contiguous() if x64 else coords.to(torch.float32).contiguous()
    rs = row_splits.to(device=dev, dtype=torch.int64).contiguous()
    q = None if queries is None else queries.to(device=dev, dtype=torch.int32).contiguous()
    nq = n if q is None else q.numel()
    flags = 0
    dr = None
    if direction is not None:
        flags |= _lib.FG_KNN_USE_DIRECTION
        dr = direction.to(device=dev, dtype=torch.int8).contiguous()
    if max_radius2 is not None:
        flags |= _lib.FG_KNN_USE_MAX_R2
    idx = torch.empty((nq, K), dtype=torch.int32, device=dev)
    d2 = torch.empty((nq, K), dtype=torch.float64, device=dev)
    fn = L.fg_brute_knn_f64 if x64 else L.fg_brute_knn
    _lib.check(fn(_p(c), n, n_c, _p(rs), rs.numel() - 1, _p(q), nq, _p(dr),
                  float(max_radius2 or 0.0), flags, K, _p(idx), _p(d2), _stream(c)), "brute_knn")
    return idx, d2


@brute_knn.register_fake
def _brute_fake(coords, row_splits, K, queries=None, direction=None, max_radius2=None):
    nq = coords.shape[0] if queries is None else queries.shape[0]
    return (coords.new_empty((nq, K), dtype=torch.int32),
            coords.new_empty((nq, K), dtype=torch.float64))


# ---------------------------------------------------------------- association matrices
# Object counts are data dependent (the result size is read back once), so these
# two are plain functions over the C ABI rather than traceable torch.library ops.
def oc_find_unique(asso: Tensor, row_splits: Tensor):
    """find_unique + max_same_count (G/ocgraph.py:114-149) on the device.

    asso i64[N] (negative = background), row_splits i64[S+1] ->
    (unique_idx i64[U], unique_rs i64[U], counts i64[U], max_count int)."""
    _require_cuda(asso, row_splits)
    a = asso.to(torch.int64).contiguous()
    rs = row_splits.to(device=a.device, dtype=torch.int64).contiguous()
    n, S = a.numel(), rs.numel() - 1
    if S < 1:
        raise BadShapeError("row_splits needs at least 2 entries")
    L = _lib.load()
    ws = _ws(_lib.size_out(L.fg_oc_unique_workspace_size, n), a.device)
    uidx = torch.empty(max(n, 1), dtype=torch.int64, device=a.device)
    urs = torch.empty_like(uidx)
    cnt = torch.empty_like(uidx)
    summary = torch.empty(2, dtype=torch.int64, device=a.device)
    _lib.check(L.fg_oc_find_unique(_p(a), n, _p(rs), S, _p(uidx), _p(urs), _p(cnt), _p(summary),
                                   _p(ws), ws.numel(), _stream(a)), "find_unique")
    n_u, top = (int(x) for x in summary.cpu())
    return uidx[:n_u], urs[:n_u], cnt[:n_u], top


def oc_matrices(asso: Tensor, row_splits: Tensor, unique_idx: Tensor, unique_rs: Tensor,
                n_maxuq: int, n_maxrs: int, max_window: int, calc_m_not: bool = True):
    """oc_helper's M / M-not rows (G/ocgraph.py:152-202) on the device ->
    (m i64[U, n_maxuq], m_not i64[U, n_maxrs] or None, visits i64[1] device)."""
    _require_cuda(asso, row_splits, unique_idx, unique_rs)
    a = asso.to(torch.int64).contiguous()
    rs = row_splits.to(device=a.device, dtype=torch.int64).contiguous()
    ui = unique_idx.to(device=a.device, dtype=torch.int64).contiguous()
    ur = unique_rs.to(device=a.device, dtype=torch.int64).contiguous()
    if ui.numel() != ur.numel():
        raise BadShapeError("unique ids and splits must be equally long")
    n_u = ui.numel()
    L = _lib.load()
    if n_maxuq < 1 or n_maxrs < 1:  # validated by the library before any launch
        _lib.check(L.fg_oc_matrices(None, None, 1, None, None, 0, int(n_maxuq), int(n_maxrs), 0,
                                    None, None, None, None, 0, None), "oc_helper")
    ws = _ws(_lib.size_out(L.fg_oc_matrices_workspace_size, n_u, int(max_window)), a.device)
    m = torch.empty((n_u, int(n_maxuq)), dtype=torch.int64, device=a.device)
    m_not = torch.empty((n_u, int(n_maxrs)), dtype=torch.int64, device=a.device) if calc_m_not else None
    visits = torch.empty(1, dtype=torch.int64, device=a.device)
    _lib.check(L.fg_oc_matrices(_p(a), _p(rs), rs.numel() - 1, _p(ui), _p(ur), n_u, int(n_maxuq),
                                int(n_maxrs), int(max_window), _p(m), _p(m_not), _p(visits), _p(ws),
                                ws.numel(), _stream(a)), "oc_helper")
    return m, m_not, visits
