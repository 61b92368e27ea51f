"""Time the association matrices (find_unique + oc_helper) on a D-like batch:
64 events x 100k vertices, 50 objects per event (generate_associations), with
CUDA events on the launching stream; the oracle (numpy restatement of
G/ocgraph.py) on a 4-event sample for the CPU side.  Development tool."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2511_10442_b200 import ops  # noqa: E402
from paper_2511_10442_b200.datasets import generate_associations  # noqa: E402

S, PER, OBJ = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (64, 100_000, 50)))
asso, off = generate_associations(S * PER, S, OBJ, 11, 0.2)
a = torch.from_numpy(asso).cuda()
rs = torch.from_numpy(off).cuda()
window = int(np.diff(off).max())


def step():
    ui, ur, cnt, top = ops.oc_find_unique(a, rs)
    return ui, ur, ops.oc_matrices(a, rs, ui, ur, max(1, top), window, window, True)


for _ in range(3):
    step()
torch.cuda.synchronize()
ui, ur, cnt, top = ops.oc_find_unique(a, rs)
ts_u, ts_m = [], []
for _ in range(10):
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    ui, ur, cnt, top = ops.oc_find_unique(a, rs)
    e1.record()
    m, mn, v = ops.oc_matrices(a, rs, ui, ur, max(1, top), window, window, True)
    e2.record()
    torch.cuda.synchronize()
    ts_u.append(e0.elapsed_time(e1))
    ts_m.append(e1.elapsed_time(e2))
n_u = ui.numel()
wbytes = n_u * (max(1, top) + window) * 8
tm = min(ts_m)
print(f"S={S} per={PER} objects={n_u} n_maxuq={top} window={window}")
print(f"find_unique ms min {min(ts_u):.3f} (includes the 16-byte summary read-back)")
print(f"matrices ms min {tm:.3f}  output {wbytes/1e9:.2f} GB -> {wbytes/tm/1e6:.0f} GB/s")
sys.path.insert(0, ".")
from oracle import oracle as O  # noqa: E402  (CPU reference restatement, timing only)
sub = off[:5]
t0 = time.perf_counter()
u2, r2, c2 = O.find_unique(asso[:sub[-1]], sub)
O.oc_helper(asso[:sub[-1]], sub, u2, r2, int(c2.max()), window)
dt = time.perf_counter() - t0
print(f"oracle (numpy, 1 thread) on 4 of {S} events: {dt:.2f} s -> ~{dt * S / 4:.1f} s for the batch")
