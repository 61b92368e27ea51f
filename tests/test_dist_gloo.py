"""CPU, world_size 2 over gloo: the multi-GPU host path (event sharding by row
splits, global n_bins, all-gather of per-rank timings/checksums).  The data
path has no collective; only statistics are gathered."""

import os
import socket

import numpy as np
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2511_10442_b200 import datasets, sharding
    coords, off = datasets.generate_dataset(6_400, 4, 64, seed=5)
    sh = sharding.shard(off, rank, world)
    nb = sharding.global_n_bins(off, 40, 4)
    local = coords[sh.vertex_lo:sh.vertex_hi]
    checksum = float(np.float64(local.sum()))
    stats = sharding.gather_floats([float(rank), float(sh.n_events), float(nb), checksum])
    out[rank] = stats.tolist()
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharding_over_gloo():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    from paper_2511_10442_b200 import datasets
    coords, off = datasets.generate_dataset(6_400, 4, 64, seed=5)
    for r in range(world):
        rows = np.asarray(out[r])
        assert rows.shape == (world, 4)
        assert rows[:, 0].tolist() == [0.0, 1.0]
        assert rows[:, 1].sum() == 64            # every event owned exactly once
        assert len(set(rows[:, 2])) == 1         # same global n_bins on every rank
        assert np.isclose(rows[:, 3].sum(), coords.sum())
