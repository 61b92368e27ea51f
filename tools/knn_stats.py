"""Diagnostics: per-query search statistics of the forward kernel on the
BASELINE configs (regions, candidate chunks, appends, compactions, ...)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2511_10442_b200 import _lib, ops
from paper_2511_10442_b200.datasets import config_dataset
from paper_2511_10442_b200.binning import compute_n_bins

for cfg in sys.argv[1:] or ["north_star", "B", "E", "A"]:
    c, off, k = config_dataset(cfg)
    n, d = c.shape
    d_bin = min(d, 5)
    nb = compute_n_bins(int(np.diff(off).max()), k, d_bin)
    ct = torch.from_numpy(c).cuda(); rs = torch.from_numpy(off).cuda()
    bi, so, bb, mi, wi, sc = ops.bin_by_coordinates(ct, rs, d_bin, nb)
    ops.set_debug_flags(_lib.FG_KNN_STATS)
    ops.knn_stats(reset=True)
    ops.binned_select_knn(ct, rs, bi, so, bb, mi, wi, sc, k, d_bin, nb, None, None, False, False)
    torch.cuda.synchronize()
    st = ops.knn_stats(reset=True)
    ops.set_debug_flags(0)
    q = max(st["queries"], 1)
    print(cfg, {kk: round(v / q, 3) for kk, v in st.items()}, "per query; cand slots/q =",
          round(32 * st["chunks"] / q, 1))
