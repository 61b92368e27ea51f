"""Dev tool: kernel timeline of the bench's back-to-back e2e loop (torch.profiler).

    python tools/e2e_prof.py B [n_steps]

Runs bin -> search -> backward with pinned host copies on side streams exactly as
bench.py's e2e block does, then prints per-step wall (CUDA events) and the
kernels/copies of the profiled steps sorted by start time, so a step that is
slower back to back than alone shows where the time goes.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2511_10442_b200 import ops  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "B"
n_steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
dev = torch.device("cuda", 0)
coords_np, off_np, k, n_bins, _, _ = bench.workload(cfg, 0, 1)
n, d = coords_np.shape
d_bin = min(d, 5)
up_np = np.random.default_rng(1).standard_normal((n, k)).astype(np.float32)
rs = torch.from_numpy(off_np).to(dev)
stream = torch.cuda.current_stream(dev)
s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
h_c = torch.from_numpy(coords_np).pin_memory()
h_u = torch.from_numpy(up_np).pin_memory()
d_c, d_u = torch.empty_like(h_c, device=dev), torch.empty_like(h_u, device=dev)
h_out = None


def e2e_step(join):
    global h_out
    ev_first, ev_late = torch.cuda.Event(), torch.cuda.Event()
    s_h2d.wait_stream(stream)
    with torch.cuda.stream(s_h2d):
        d_c.copy_(h_c, non_blocking=True)
        ev_first.record(s_h2d)
        d_u.copy_(h_u, non_blocking=True)
        ev_late.record(s_h2d)
    stream.wait_event(ev_first)
    bi, so, bb, mins, widths, sc = ops.bin_by_coordinates(d_c, rs, d_bin, n_bins)
    idx, d2 = ops.binned_select_knn(d_c, rs, bi, so, bb, mins, widths, sc, k, d_bin, n_bins,
                                    None, None, False, False)
    ev_fwd = torch.cuda.Event()
    ev_fwd.record(stream)
    stream.wait_event(ev_late)
    g = ops.binned_select_knn_grad(d_u, idx, d_c, so, False)
    ev_bwd = torch.cuda.Event()
    ev_bwd.record(stream)
    outs = [idx, d2, g]
    if h_out is None:
        h_out = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in outs]
    with torch.cuda.stream(s_d2h):
        s_d2h.wait_event(ev_fwd)
        h_out[0].copy_(idx, non_blocking=True)
        h_out[1].copy_(d2, non_blocking=True)
        s_d2h.wait_event(ev_bwd)
        h_out[2].copy_(g, non_blocking=True)
    for o in outs:
        o.record_stream(s_d2h)
    if join:
        stream.wait_stream(s_d2h)


def pipelined(m, marks=None):
    done = []
    for it in range(m):
        if it >= 2:
            stream.wait_event(done[it - 2])
        if marks is not None:
            ev0 = torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            marks.append(ev0)
        e2e_step(False)
        ev = torch.cuda.Event()
        ev.record(s_d2h)
        done.append(ev)
    stream.wait_stream(s_d2h)


for _ in range(3):
    e2e_step(True)
torch.cuda.synchronize()
for mode in ("alone", "pipelined"):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    if mode == "alone":
        for _ in range(n_steps):
            e2e_step(True)
            torch.cuda.synchronize()
    else:
        pipelined(n_steps)
    e1.record(stream)
    e1.synchronize()
    print(f"{cfg} {mode}: {e0.elapsed_time(e1) / n_steps:.3f} ms/step", flush=True)
for rep in range(3):
    marks = []
    import time as _t
    h0 = _t.perf_counter()
    pipelined(n_steps, marks)
    h1 = _t.perf_counter()
    end = torch.cuda.Event(enable_timing=True)
    end.record(stream)
    end.synchronize()
    marks.append(end)
    print("pipelined per-step ms:", [round(marks[i].elapsed_time(marks[i + 1]), 3) for i in range(len(marks) - 1)],
          f"host enqueue {1e3 * (h1 - h0):.2f} ms", flush=True)

from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    pipelined(n_steps)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
evs.sort(key=lambda e: e.time_range.start)
t0 = evs[0].time_range.start if evs else 0
for e in evs:
    print(f"{(e.time_range.start - t0) / 1000:9.3f} ms  {e.time_range.elapsed_us() / 1000:8.3f} ms  "
          f"{e.name[:90]}")
cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU
       and ("Synchronize" in e.name or "cudaMalloc" in e.name or "cudaFree" in e.name
            or "Memcpy" in e.name)]
for e in cpu[:40]:
    print("CPU", f"{(e.time_range.start - t0) / 1000:9.3f} ms {e.time_range.elapsed_us() / 1000:8.3f} ms", e.name)
