"""Minimal initcheck repro: the sanitizer workload's first tile-path call."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2511_10442_b200 as fg
from paper_2511_10442_b200 import _lib, ops
from paper_2511_10442_b200.datasets import generate_dataset

flags = int(sys.argv[1]) if len(sys.argv) > 1 else 0
x, _ = generate_dataset(6000, 4, splits=2, seed=3)
off = np.array([0, 2500, 6000], np.int64)
c = torch.from_numpy(x.astype(np.float32)).cuda()
rs = torch.from_numpy(off).cuda()
nb = fg.compute_n_bins(3500, 16, 4)
bi, so, bb, mins, widths, sc = ops.bin_by_coordinates(c, rs, 4, nb)
ops.set_debug_flags(flags | _lib.FG_KNN_STATS)
ops.knn_stats(reset=True)
idx, d2 = ops.binned_select_knn(c, rs, bi, so, bb, mins, widths, sc, 16, 4, nb, None, None, False, False)
torch.cuda.synchronize()
print(ops.knn_stats(reset=True))
