"""Time binned_select_knn_grad (CUDA events) -- transposed path and the atomic
fallback -- with L2 flushed before each call: python tools/time_bwd.py [cfg]."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2511_10442_b200 import ops
from paper_2511_10442_b200.datasets import config_dataset
from paper_2511_10442_b200.binning import compute_n_bins
for cfg in (sys.argv[1:] or ["north_star"]):
    c, off, k = config_dataset(cfg)
    n, d = c.shape
    nb = compute_n_bins(int(np.diff(off).max()), k, min(d, 5))
    ct = torch.from_numpy(c).cuda(); rs = torch.from_numpy(off).cuda()
    bi, so, bb, mi, wi, sc = ops.bin_by_coordinates(ct, rs, min(d, 5), nb)
    idx, d2 = ops.binned_select_knn(ct, rs, bi, so, bb, mi, wi, sc, k, min(d, 5), nb, None, None,
                                    False, False)
    up = torch.randn(n, k, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for det in (False, True):
        ts = []
        for i in range(12):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); g = ops.binned_select_knn_grad(up, idx, ct, so, det); e1.record()
            torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        ts = ts[2:]
        print(cfg, "deterministic" if det else "atomic", "bwd ms min %.3f median %.3f"
              % (min(ts), sorted(ts)[len(ts) // 2]), flush=True)
