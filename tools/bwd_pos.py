"""Backward locality experiment (tools/micro/bwd_pos.cu) on the north_star rows:
library backward vs position-indexed accumulation with slots in distance order,
sorted in-kernel, or pre-sorted by position.  Timing only."""
import ctypes
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_2511_10442_b200 as fg
from paper_2511_10442_b200 import ops
from paper_2511_10442_b200.datasets import config_dataset

lib = ctypes.CDLL("tools/micro/libbwd_pos.so")
lib.bwd_pos.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p,
                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
c, off, k = config_dataset("north_star")
n, d = c.shape
ct = torch.from_numpy(c).cuda(); rs = torch.from_numpy(off).cuda()
nb = fg.compute_n_bins(n, k, d)
bi, so, bb, mi, wi, sc = ops.bin_by_coordinates(ct, rs, d, nb)
idx, d2 = ops.binned_select_knn(ct, rs, bi, so, bb, mi, wi, sc, k, d, nb, None, None, False, False)
g = torch.randn(n, k, device="cuda")
inv = torch.empty(n, dtype=torch.int32, device="cuda")
inv[so.long()] = torch.arange(n, dtype=torch.int32, device="cuda")
rows = idx[so.long()]
pm = torch.where(rows >= 0, inv[rows.clamp(min=0).long()], torch.full_like(rows, -1)).contiguous()
gm = g[so.long()].contiguous()
ps, order = torch.sort(torch.where(pm[:, 1:] >= 0, pm[:, 1:], torch.full_like(pm[:, 1:], 2**31 - 1)), dim=1)
pm_sorted = torch.cat([pm[:, :1], torch.where(ps == 2**31 - 1, torch.full_like(ps, -1), ps)], 1).contiguous()
gm_sorted = torch.cat([gm[:, :1], torch.gather(gm[:, 1:], 1, order)], 1).contiguous()
hi = torch.zeros(n, 4, device="cuda"); lo = torch.zeros(n, 4, device="cuda")
st = torch.cuda.current_stream().cuda_stream

def timeit(fn, reps=10):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return round(min(ts), 4), round(float(np.median(ts)), 4)

def pos(variant, P, G):
    def f():
        hi.zero_(); lo.zero_()
        lib.bwd_pos(ctypes.c_void_p(sc.data_ptr()), n, ctypes.c_void_p(P.data_ptr()), k,
                    ctypes.c_void_p(G.data_ptr()), ctypes.c_void_p(hi.data_ptr()),
                    ctypes.c_void_p(lo.data_ptr()), variant, ctypes.c_void_p(st))
    return f

print("library backward (atomic, ids)", timeit(lambda: ops.binned_select_knn_grad(g, idx, ct, so)))
print("library backward (deterministic)", timeit(lambda: ops.binned_select_knn_grad(g, idx, ct, so, True)))
print("positions, distance order", timeit(pos(0, pm, gm)))
print("positions, in-kernel sort", timeit(pos(1, pm, gm)))
print("positions, pre-sorted", timeit(pos(0, pm_sorted, gm_sorted)))
# check: position-indexed sums equal the library's (same terms, any order)
pos(0, pm, gm)(); torch.cuda.synchronize()
gp = (hi.double() + lo.double())
ref = ops.binned_select_knn_grad(g, idx, ct, so).double()
out = torch.empty_like(gp); out[so.long()] = gp
print("max rel diff vs library", float(((out - ref).abs() / ref.abs().clamp(min=1e-6)).max()))
