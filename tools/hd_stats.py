"""Search time + counters of the high-dimensional tile path vs the warp-per-query
kernel on a BASELINE config: python tools/hd_stats.py C [B ...]"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2511_10442_b200 as fg
from paper_2511_10442_b200 import _lib, ops
from paper_2511_10442_b200.datasets import config_dataset

for cfg in sys.argv[1:] or ["C"]:
    c, off, k = config_dataset(cfg)
    n, d = c.shape
    d_bin = min(d, 5)
    nb = fg.compute_n_bins(int(np.diff(off).max()), k, d_bin)
    ct = torch.from_numpy(c).cuda(); rs = torch.from_numpy(off).cuda()
    bi, so, bb, mi, wi, sc = ops.bin_by_coordinates(ct, rs, d_bin, nb)
    for name, fl in (("default", 0), ("force_hd", _lib.FG_KNN_FORCE_HD), ("no_hd", _lib.FG_KNN_NO_HD)):
        if cfg == "C" and name == "no_hd" and "--all" not in sys.argv:
            continue
        ops.set_debug_flags(fl | _lib.FG_KNN_STATS)
        ops.knn_stats(reset=True)
        ts = []
        for i in range(3):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            ops.binned_select_knn(ct, rs, bi, so, bb, mi, wi, sc, k, d_bin, nb, None, None, False, False)
            e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        st = ops.knn_stats(reset=True)
        ops.set_debug_flags(0)
        keep = {kk: (v if kk == "hd_max_tile_cycles" or kk.startswith("slow") else v // 3) for kk, v in st.items() if v}
        print(cfg, name, "ms", [round(t, 3) for t in ts], keep, flush=True)
