"""Time binned_select_knn_grad (CUDA events, min of reps) for FG_LIB_PATH."""
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
nb = compute_n_bins(int(np.diff(off).max()), k, d)
ct = torch.from_numpy(c).cuda(); rs = torch.from_numpy(off).cuda()
bi, so, bb, mi, wi, sc = ops.bin_by_coordinates(ct, rs, d, nb)
idx, d2 = ops.binned_select_knn(ct, rs, bi, so, bb, mi, wi, sc, k, d, nb, None, None, False, False)
up = torch.randn(n, k, device="cuda")
ref = ops.binned_select_knn_grad(up, idx, ct, so).double()
ts = []
for i in range(8):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); g = ops.binned_select_knn_grad(up, idx, ct, so); e1.record()
    torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
print(cfg, "bwd ms min %.3f median %.3f" % (min(ts), sorted(ts)[len(ts)//2]))
