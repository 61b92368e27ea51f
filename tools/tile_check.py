"""Tile path vs warp-per-query path on the BASELINE configs: bit-exact rows,
per-path search time (CUDA events), tile statistics."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2511_10442_b200 import _lib, ops
from paper_2511_10442_b200.datasets import config_dataset, generate_dataset
from paper_2511_10442_b200.binning import compute_n_bins


def run(c, off, k, flags, reps=5):
    n, d = c.shape
    d_bin = min(d, 5)
    nb = compute_n_bins(int(np.diff(off).max()), k, d_bin)
    ct = torch.from_numpy(c).cuda(); rs = torch.from_numpy(off).cuda()
    bi, so, bb, mi, wi, sc = ops.bin_by_coordinates(ct, rs, d_bin, nb)
    ops.set_debug_flags(flags)
    out = ops.binned_select_knn(ct, rs, bi, so, bb, mi, wi, sc, k, d_bin, nb, None, None, False, False)
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); ops.binned_select_knn(ct, rs, bi, so, bb, mi, wi, sc, k, d_bin, nb, None, None,
                                           False, False); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ops.set_debug_flags(flags | _lib.FG_KNN_STATS); ops.knn_stats(reset=True)
    ops.binned_select_knn(ct, rs, bi, so, bb, mi, wi, sc, k, d_bin, nb, None, None, False, False)
    torch.cuda.synchronize()
    st = ops.knn_stats(reset=True)
    ops.set_debug_flags(0)
    return out[0].cpu().numpy(), out[1].cpu().numpy(), min(ts), st


cases = []
for name in (sys.argv[1:] or ["north_star", "E", "A", "D", "B"]):
    if name == "small":
        for seed in range(6):
            rng = np.random.default_rng(seed)
            n = int(rng.integers(2000, 30000)); d = int(rng.integers(1, 5)); S = int(rng.integers(1, 5))
            k = int(rng.integers(2, 42))
            c, off = generate_dataset(n, d, S, seed, "uniform" if seed % 2 else "clusters")
            cases.append((f"small{seed} n={n} d={d} S={S} k={k}", c.astype(np.float32), off, k))
    else:
        c, off, k = config_dataset(name)
        cases.append((name, c, off, k))
for name, c, off, k in cases:
    i0, d0, t0, s0 = run(c, off, k, _lib.FG_KNN_NO_TILE)
    i1, d1, t1, s1 = run(c, off, k, 0)
    same = np.array_equal(i0, i1) and np.array_equal(d0.view(np.uint32), d1.view(np.uint32))
    bad = int((i0 != i1).any(1).sum())
    q = max(s1["tiles"], 1)
    print(f"{name}: exact={same} bad_rows={bad} warp_ms={t0:.3f} tile_ms={t1:.3f} "
          f"tiles={s1['tiles']} cand/tile={s1['tile_candidates']/q:.0f} redo={s1['tile_redo']} "
          f"({100*s1['tile_redo']/len(c):.3f}%) tile_fail={s1['tile_fail']} expanded={s1['tile_expanded']} "
          f"eval/tile={s1['tile_evaluated']/q:.0f}", flush=True)
