"""One backward call (transposed path) on a config, for ncu launch lists."""
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
nb = compute_n_bins(int(np.diff(off).max()), k, min(d, 5))
ct = torch.from_numpy(c).cuda(); rs = torch.from_numpy(off).cuda()
bi, so, bb, mi, wi, sc = ops.bin_by_coordinates(ct, rs, min(d, 5), nb)
idx, d2 = ops.binned_select_knn(ct, rs, bi, so, bb, mi, wi, sc, k, min(d, 5), nb, None, None, False, False)
up = torch.randn(n, k, device="cuda")
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
g = ops.binned_select_knn_grad(up, idx, ct, so, True)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
