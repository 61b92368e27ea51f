"""Time gravnet_aggregate forward / backward (CUDA events, min of reps) on config E."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2511_10442_b200 import ops
from paper_2511_10442_b200.datasets import config_dataset
from paper_2511_10442_b200.binning import compute_n_bins
c, off, k = config_dataset("E")
n, d = c.shape
nb = compute_n_bins(int(np.diff(off).max()), k, d)
ct = torch.from_numpy(c).cuda(); rs = torch.from_numpy(off).cuda()
bi, so, bb, mi, wi, sc = ops.bin_by_coordinates(ct, rs, d, nb)
idx, d2 = ops.binned_select_knn(ct, rs, bi, so, bb, mi, wi, sc, k, d, nb, None, None, False, False)
g = torch.Generator(device="cuda").manual_seed(0)
f = torch.randn(n, 64, device="cuda", generator=g)
ua = torch.randn(n, 128, device="cuda", generator=g)
def t(fn):
    ts = []
    for i in range(6):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts)
out = ops.gravnet_aggregate(f, idx, d2, 10.0, [0, 1], True, so)
tf = t(lambda: ops.gravnet_aggregate(f, idx, d2, 10.0, [0, 1], True, so))
tb = t(lambda: ops.gravnet_aggregate_grad(ua, f, idx, d2, 10.0, [0, 1], True, so))
print("gravnet fwd ms %.3f bwd ms %.3f checksum %.6f" % (tf, tb, float(out.double().sum())))
