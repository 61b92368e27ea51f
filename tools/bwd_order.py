"""Experiment: backward row visiting order -- binning order (cells row-major) vs
cell Morton order vs 2x2x2xL cell blocks -- CUDA events, L2 flushed per call.
python tools/bwd_order.py [cfg]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2511_10442_b200 import ops
from paper_2511_10442_b200.datasets import config_dataset
from paper_2511_10442_b200.binning import compute_n_bins

cfg = sys.argv[1] if len(sys.argv) > 1 else "north_star"
c, off, k = config_dataset(cfg)
n, d = c.shape
db = min(d, 5)
nb = compute_n_bins(int(np.diff(off).max()), k, db)
ct = torch.from_numpy(c).cuda(); rs = torch.from_numpy(off).cuda()
bi, so, bb, mi, wi, sc = ops.bin_by_coordinates(ct, rs, db, nb)
idx, d2 = ops.binned_select_knn(ct, rs, bi, so, bb, mi, wi, sc, k, db, nb, None, None, False, False)
up = torch.randn(n, k, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
# cell coordinates of every sorted position
cell = bi[so.long()]  # flat cell of the vertex at each sorted position
cc = []
rem = cell.clone()
for _ in range(db):
    cc.append(rem % nb)
    rem = rem // nb
cc = cc[::-1]  # cc[0] = lead dim
def morton(coords, bits=6):
    key = torch.zeros_like(coords[0])
    for b in range(bits):
        for j, x in enumerate(coords):
            key |= ((x >> b) & 1) << (b * len(coords) + j)
    return key
orders = {"binning (row-major cells)": so}
pos = torch.arange(n, device="cuda")
key_m = morton(cc)
orders["cell Morton"] = so[torch.argsort(key_m * n + pos)]
# blocks of 2 in the first d-1 dims, whole last-dim columns (the tile path's blocks)
blk = torch.zeros_like(cc[0])
for x in cc[:-1]:
    blk = blk * ((nb + 1) // 2) + (x >> 1)
key_b = (blk * nb + cc[-1]) * (1 << (db - 1))
sub = torch.zeros_like(cc[0])
for x in cc[:-1]:
    sub = sub * 2 + (x & 1)
orders["2^(d-1) blocks x last-dim column"] = so[torch.argsort((key_b + sub) * n + pos)]
for name, od in orders.items():
    ts = []
    for i in range(14):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); g = ops.binned_select_knn_grad(up, idx, ct, od.int().contiguous(), False); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ts = ts[2:]
    print(cfg, f"{name:40s} bwd ms min {min(ts):.3f} median {sorted(ts)[len(ts) // 2]:.3f}", flush=True)
