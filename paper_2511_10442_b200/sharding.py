"""Event-parallel sharding of a multi-event batch across ranks.

Row splits (events) are independent -- no query crosses a split
(T/test_acceptance.py:362-383) -- so each rank owns one contiguous range of
events and runs the whole path on it with NO collective in the data path.
The only global quantity is n_bins, which the reference takes from the
LARGEST split of the whole batch (G/binning.py:159-162); every rank computes
it from the (host) row splits, so each rank's bin_bounds slice equals the
matching slice of the single-GPU index.  Neighbour indices are emitted in the
global numbering (local id + the rank's vertex offset).  torch.distributed is
used only to gather per-rank timings and checksums.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .binning import compute_n_bins, default_bin_dims


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    event_lo: int
    event_hi: int
    vertex_lo: int
    vertex_hi: int
    local_offsets: np.ndarray  # row splits of this shard, starting at 0

    @property
    def n_vertices(self) -> int:
        return self.vertex_hi - self.vertex_lo

    @property
    def n_events(self) -> int:
        return self.event_hi - self.event_lo


def event_range(n_events: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, as-even-as-possible event ranges (first n % world ranks get
    one more)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"bad rank/world {rank}/{world}")
    base, rem = divmod(n_events, world)
    lo = rank * base + min(rank, rem)
    hi = lo + base + (1 if rank < rem else 0)
    return lo, hi


def shard(offsets, rank: int, world: int) -> Shard:
    off = np.asarray(offsets, dtype=np.int64)
    e0, e1 = event_range(off.size - 1, rank, world)
    v0, v1 = int(off[e0]), int(off[e1])
    return Shard(rank, world, e0, e1, v0, v1, off[e0:e1 + 1] - v0)


def global_n_bins(offsets, k: int, n_coords: int, d_bin: int | None = None) -> int:
    sizes = np.diff(np.asarray(offsets, dtype=np.int64))
    d_bin = d_bin or default_bin_dims(n_coords)
    return compute_n_bins(int(sizes.max()) if sizes.size else 0, k, d_bin)


@dataclass
class ShardResult:
    """One rank's slice of the batch's neighbour matrix, in the GLOBAL vertex
    numbering: ``idx[i]`` is the row of global vertex ``shard.vertex_lo + i``
    and holds global neighbour ids (-1 padding kept)."""
    shard: Shard
    idx: "object"           # torch int32 (n_local, k), global ids
    d2: "object"            # torch float32/float64 (n_local, k)
    sort_order: "object"    # torch int32 (n_local,), LOCAL ids (for the backward)
    bin_bounds: "object"    # torch int32, this shard's slice of the global bounds
    n_bins: int


def select_knn_sharded(coords, offsets, k: int, rank: int, world: int, *, device=None,
                       d_bin: int | None = None, d2_f64: bool = False) -> ShardResult:
    """The rank's share of binned_select_knn over a multi-event batch.

    ``coords``: the WHOLE batch (host numpy or a tensor) or only this rank's
    rows (len == its vertex count); ``offsets``: the whole batch's row splits.
    Bins the rank's contiguous event range with the batch's global n_bins
    (G/binning.py:159-162) and searches it; every index is shifted by the
    shard's first vertex, so the result is exactly the corresponding row slice
    of the single-GPU result (tests/test_gpu_shard.py).  No collective."""
    import torch
    from . import ops
    off = np.asarray(offsets, dtype=np.int64)
    sh = shard(off, rank, world)
    n_c = int(coords.shape[1])
    d_bin = d_bin or default_bin_dims(n_c)
    n_bins = global_n_bins(off, k, n_c, d_bin)
    device = device or torch.device("cuda", torch.cuda.current_device())
    total = int(off[-1])
    local = coords[sh.vertex_lo:sh.vertex_hi] if int(coords.shape[0]) == total and total != sh.n_vertices \
        else coords
    if int(local.shape[0]) != sh.n_vertices:
        raise ValueError(f"coords has {coords.shape[0]} rows: expected the batch ({total}) or "
                         f"this shard ({sh.n_vertices})")
    c = local if isinstance(local, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(local))
    c = c.to(device=device, dtype=torch.float32).contiguous()
    rs = torch.from_numpy(sh.local_offsets).to(device)
    bi, so, bb, mins, widths, sc = ops.bin_by_coordinates(c, rs, d_bin, n_bins)
    idx, d2 = ops.binned_select_knn(c, rs, bi, so, bb, mins, widths, sc, k, d_bin, n_bins, None,
                                    None, False, d2_f64)
    if sh.vertex_lo:
        idx = torch.where(idx >= 0, idx + sh.vertex_lo, idx)
    return ShardResult(sh, idx, d2, so, bb, n_bins)


def local_indices(res: ShardResult):
    """The shard's neighbour matrix in its local numbering (for its backward)."""
    import torch
    idx = res.idx
    return torch.where(idx >= 0, idx - res.shard.vertex_lo, idx) if res.shard.vertex_lo else idx


def gather_floats(values, group=None):
    """all_gather a short list of floats (timings, checksums) across ranks;
    returns a (world, len) numpy array.  Works on gloo (CPU) and nccl."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return np.asarray([values], dtype=np.float64)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else \
        torch.device("cpu")
    t = torch.tensor(list(values), dtype=torch.float64, device=dev)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    return torch.stack(out).cpu().numpy()
