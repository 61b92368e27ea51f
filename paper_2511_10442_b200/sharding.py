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
