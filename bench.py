#!/usr/bin/env python
"""Benchmark of the hot path: bin_by_coordinates -> binned_select_knn forward ->
backward (BASELINE.json metric: N=1M, d=4, k=40, fwd+bwd; % of HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config north_star|A|B|C|D|E]
    python -m torch.distributed.run --nproc-per-node N ... bench.py --gpus N   (N > 1)
    python bench.py --impl reference     (the reference's own CPU path, rank 0)

Workload (default ``north_star``): one step = one pass of the path over one
event of 1,000,000 uniform points in [0,1)^4 (the reference's generator,
seed 3 + rank, cast to float32), k = 40, fixed upstream gradient for the
backward.  Multi-GPU = event sharding by row splits, one event per GPU (weak
scaling), no collective in the data path; timings are all-gathered and the
max over ranks is reported.  Inputs are resident in HBM when the timed region
starts; L2 is flushed (256 MiB write) before every step.  ``e2e`` repeats the
measurement with pinned HOST buffers and the host<->device copies inside the
timed region (copy streams overlap the compute: upstream gradients go in
while the search runs, the neighbour matrix comes back while the backward runs),
timed over steps run back to back like a training loop (``latency_ms_per_step``
= one step alone, outputs on the host before the next starts).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "binned kNN graph-build ms & queries/s, N=1M d=4 k=40, fwd+bwd; % HBM roofline"

# reference candidate counts C_total (the reference algorithm at
# the reference n_bins), used in the algorithmic byte model.
C_TOTAL = {"A": 8.6e5, "B": 3.68e9, "north_star": 7.47e8, "C": 1.81e11, "D": 4.51e9,
           "E": 3.31e8}


# query sample for the CPU reference where its full search would take minutes+
REF_QUERY_FRAC = {"C": 0.002, "D": 0.1}


def algorithmic_bytes(n, d, k, c_total):
    """B_fwd = 4Nd + 4d*C_total + 8Nk; B_bwd = 8Nk + 8Ndk + 8Nd."""
    b_fwd = 4 * n * d + 4 * d * c_total + 8 * n * k
    b_bwd = 8 * n * k + 8 * n * d * k + 8 * n * d
    return b_fwd, b_bwd


def load_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


SEARCH_KERNELS = ("k_tiles", "k_tile_search", "k_tile_finish", "k_knn_fwd")


def load_traffic(config):
    """dram bytes per search call (its kernels) from the committed ncu captures."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            data = json.load(fh)[config]
        got = [data[k]["dram_bytes_per_launch"] for k in SEARCH_KERNELS if k in data]
        return float(sum(got)) if got else None
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed loop runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.FIELDS,
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                return
            self._stop.wait(0.05)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def workload(config, rank, world):
    from paper_2511_10442_b200.datasets import CONFIGS, generate_dataset
    n, d, splits, k, dist, seed = CONFIGS[config]
    if config == "D":
        # strong scaling: the 64-event batch is sharded by row splits
        from paper_2511_10442_b200 import sharding
        coords, off = generate_dataset(n, d, splits, seed, dist)
        sh = sharding.shard(off, rank, world)
        n_bins = sharding.global_n_bins(off, k, d)
        c = coords[sh.vertex_lo:sh.vertex_hi].astype(np.float32)
        return c, sh.local_offsets, k, n_bins, "strong", \
            f"D: 64 events x 100k points (events {sh.event_lo}..{sh.event_hi - 1} on rank {rank})"
    # weak scaling: one event per GPU
    coords, off = generate_dataset(n, d, splits, seed + rank, dist)
    from paper_2511_10442_b200.binning import compute_n_bins, default_bin_dims
    n_bins = compute_n_bins(int(np.diff(off).max()), k, default_bin_dims(d))
    desc = {"north_star": "north_star: 1 event x 1,000,000 uniform points per GPU, d=4, k=40",
            "A": "A: 10k points d=3 k=16", "B": "B: 200k clustered points d=4 k=40",
            "C": "C: 1M points d=10 k=64", "E": "E: 500k points d=4 k=40"}[config]
    return coords.astype(np.float32), off, k, n_bins, "weak", desc


def cpu_reference_step(coords32, offsets, k, n_bins, bwd_rows=100_000, seed=0,
                       query_frac=1.0):
    """One step of the reference's own CPU path on this host: build_index +
    binned_knn over ALL queries (oracle/_ref = the reference's compiled
    _binned_cy kernels, all host threads) + knn_backward (the oracle's
    restatement of the reference's numpy np.add.at code, 1 core) on a sample of
    rows, extrapolated linearly (the backward has no per-call fixed cost).
    Returns (seconds for the full workload, details)."""
    from oracle import oracle as O  # cpu_baseline leg only
    ref = O.load_ref_kernels()
    kind = "reference" if ref is not None else "port"
    c64 = coords32.astype(np.float64)
    n, n_c = c64.shape
    d_bin = min(n_c, 5)
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(seed)
    mask = None
    if query_frac < 1.0:  # configs whose full CPU search takes hours (C): query sample
        mask = np.zeros(n, np.int8)  # role 0: candidate only
        mask[rng.choice(n, size=max(1, int(n * query_frac)), replace=False)] = 3

    def run(m):
        t0 = time.perf_counter()
        if ref is not None:
            bi, so, bb, mins, widths = ref.build_index(c64, offsets, d_bin, n_bins)
            oi = np.empty((n, k), np.int32)
            od = np.empty((n, k), np.float64)
            ref.binned_knn(c64, bi, so, bb, np.full(d_bin, n_bins, np.int64),
                           widths.min(axis=1).copy(), np.zeros(1, np.int8) if m is None else m,
                           m is not None, 0.0, False, False, k, oi, od, threads)
        else:
            oi, od = O.knn_refslot(c64, offsets, k, n_bins=n_bins, dir_mask=m, threads=threads)
        return time.perf_counter() - t0, oi

    if mask is None:
        t_fwd, out_i = run(None)
    else:  # fixed per-vertex cost measured with zero queries, query cost scaled
        t_zero, _ = run(np.zeros(n, np.int8))
        t_s, out_i = run(mask)
        t_fwd = t_zero + max(t_s - t_zero, 0.0) / query_frac
        sel = np.nonzero(mask == 3)[0]
        out_i = out_i.copy()
        out_i[np.setdiff1d(np.arange(n), sel)] = out_i[sel[0]]  # bwd rows use real neighbours
    rows = rng.choice(n, size=min(bwd_rows, n), replace=False)
    up = rng.standard_normal((len(rows), k))
    t0 = time.perf_counter()
    O.knn_backward_numpy(c64, out_i[rows], up, rows)
    t_bwd = (time.perf_counter() - t0) * (n / len(rows))
    total = t_fwd + t_bwd
    return total, {"kind": kind, "cores": threads, "t_fwd_s": t_fwd, "t_bwd_s": t_bwd,
                   "sample": (f"fwd: build_index + binned_knn over "
                              + (f"all {n} queries" if mask is None else
                                 f"a {query_frac:.0%} query sample (fixed per-vertex cost timed "
                                 f"separately, query cost x{1 / query_frac:.0f})")
                              + f" (reference compiled _binned_cy, {threads} threads); bwd: numpy "
                              f"knn_backward on {len(rows)} rows x{n / len(rows):.0f} (1 core)")}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    coords, off, k, n_bins, scaling, desc = workload(args.config, 0, 1)
    n = coords.shape[0]
    times = []
    det = None
    for s_ in range(max(args.warmup, 0) + args.steps):
        tt, det = cpu_reference_step(coords, off, k, n_bins, seed=100 + s_,
                                     query_frac=REF_QUERY_FRAC.get(args.config, 1.0))
        if s_ >= args.warmup:
            times.append(tt)
    t = float(np.mean(times))
    value = n / t
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "queries/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": scaling,
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": desc, "n_points": n, "k": k, "n_bins": n_bins},
            "cpu_baseline": {"value": value, "unit": "queries/s", "cores": det["cores"],
                             "kind": det["kind"], "sample": det["sample"]},
            "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="north_star", choices=["north_star", "A", "B", "C", "D", "E"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-flush", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    import paper_2511_10442_b200 as fg
    from paper_2511_10442_b200 import _lib, ops, sharding
    _lib.load()

    coords_np, off_np, k, n_bins, scaling, desc = workload(args.config, rank, world)
    n, d = coords_np.shape
    d_bin = min(d, 5)
    rng = np.random.default_rng(1000 + rank)
    up_np = rng.standard_normal((n, k)).astype(np.float32)
    coords = torch.from_numpy(coords_np).to(dev)
    rs = torch.from_numpy(off_np).to(dev)
    up = torch.from_numpy(up_np).to(dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    gravnet = args.config == "E"  # config E: the GravNetOp layer on top of the search
    if gravnet:
        n_feat = 64
        feats = torch.from_numpy(rng.standard_normal((n, n_feat)).astype(np.float32)).to(dev)
        up_agg = torch.from_numpy(rng.standard_normal((n, 2 * n_feat)).astype(np.float32)).to(dev)

    def step(c, u, f=None, ua=None):
        """One pass of the path; returns outputs and the phase events."""
        evs = []

        def mark():
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            evs.append(e)

        bi, so, bb, mins, widths, sc = ops.bin_by_coordinates(c, rs, d_bin, n_bins)
        mark()
        if gravnet:  # GravNetOp layer: the fused search + aggregation, then its backward
            idx, d2, agg = ops.knn_gravnet(c, rs, bi, so, bb, mins, widths, sc, k, d_bin, n_bins,
                                           f, 10.0, [0, 1], True)
            mark()
            gf, gd = ops.gravnet_aggregate_grad(ua, f, idx, d2, 10.0, [0, 1], True, so)
            mark()
            g = ops.binned_select_knn_grad(gd, idx, c, so)
            return (idx, d2, g, agg, gf), evs
        idx, d2 = ops.binned_select_knn(c, rs, bi, so, bb, mins, widths, sc, k, d_bin, n_bins,
                                        None, None, False, False)
        mark()
        g = ops.binned_select_knn_grad(u, idx, c, so)
        return (idx, d2, g), evs

    # warm-up: at least W steps and at least 1.5 s of work, so the SM clocks have
    # left their idle state before anything is timed
    t_warm = time.perf_counter()
    it = 0
    while it < max(args.warmup, 3) or time.perf_counter() - t_warm < 1.5:
        step(coords, up, feats if gravnet else None, up_agg if gravnet else None)
        torch.cuda.synchronize()
        it += 1
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()

    sampler = ClockSampler(int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[0])
                           if os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")[0].isdigit()
                           else local)
    launches0 = _lib.launch_count()
    names = (["bin_by_coordinates", "knn_gravnet_fwd", "gravnet_bwd", "knn_bwd"] if gravnet
             else ["bin_by_coordinates", "knn_fwd", "knn_bwd"])
    t_step = 0.0
    t_phase = [0.0] * len(names)
    with sampler:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for _ in range(args.steps):
            if not args.no_flush:
                flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e3 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _, evs = step(coords, up, feats if gravnet else None, up_agg if gravnet else None)
            e3.record(stream)
            e3.synchronize()
            t_step += e0.elapsed_time(e3)
            marks = [e0] + evs + [e3]
            for i in range(len(names)):
                t_phase[i] += marks[i].elapsed_time(marks[i + 1])
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = _lib.launch_count() - launches0
    clocks = sampler.summary()

    # e2e through the public API with pinned host buffers: every step copies its
    # inputs in and every output back inside the timed region.  The copies run
    # on their own streams and overlap the compute the way a user pipeline
    # would: coordinates (+ features) first, the upstream gradients while the
    # search runs; the forward outputs go back while the backward runs.
    e2e = None
    if not args.no_e2e:
        s_h2d = torch.cuda.Stream(dev)
        s_d2h = torch.cuda.Stream(dev)
        h_first = [torch.from_numpy(coords_np).pin_memory()]
        h_late = [torch.from_numpy(up_np).pin_memory()] if not gravnet else [up_agg.cpu().pin_memory()]
        if gravnet:
            h_first.append(feats.cpu().pin_memory())
        d_first = [torch.empty_like(h, device=dev) for h in h_first]
        d_late = [torch.empty_like(h, device=dev) for h in h_late]

        def e2e_step(h_out=None, join=True):
            ev_first = torch.cuda.Event()
            ev_late = torch.cuda.Event()
            s_h2d.wait_stream(stream)
            with torch.cuda.stream(s_h2d):
                for d_, h_ in zip(d_first, h_first):
                    d_.copy_(h_, non_blocking=True)
                ev_first.record(s_h2d)
                for d_, h_ in zip(d_late, h_late):
                    d_.copy_(h_, non_blocking=True)
                ev_late.record(s_h2d)
            stream.wait_event(ev_first)
            c = d_first[0]
            bi, so, bb, mins, widths, sc = ops.bin_by_coordinates(c, rs, d_bin, n_bins)
            if gravnet:
                idx, d2, agg = ops.knn_gravnet(c, rs, bi, so, bb, mins, widths, sc, k, d_bin,
                                               n_bins, d_first[1], 10.0, [0, 1], True)
                fwd_outs = [idx, d2, agg]
            else:
                idx, d2 = ops.binned_select_knn(c, rs, bi, so, bb, mins, widths, sc, k, d_bin,
                                                n_bins, None, None, False, False)
                fwd_outs = [idx, d2]
            ev_fwd = torch.cuda.Event()
            ev_fwd.record(stream)
            stream.wait_event(ev_late)
            if gravnet:
                gf, gd = ops.gravnet_aggregate_grad(d_late[0], d_first[1], idx, d2, 10.0, [0, 1],
                                                    True, so)
                bwd_outs = [ops.binned_select_knn_grad(gd, idx, c, so), gf]
            else:
                bwd_outs = [ops.binned_select_knn_grad(d_late[0], idx, c, so)]
            ev_bwd = torch.cuda.Event()
            ev_bwd.record(stream)
            outs = fwd_outs + bwd_outs
            if h_out is not None:
                with torch.cuda.stream(s_d2h):
                    s_d2h.wait_event(ev_fwd)
                    for h_, o_ in zip(h_out[:len(fwd_outs)], fwd_outs):
                        h_.copy_(o_, non_blocking=True)
                    s_d2h.wait_event(ev_bwd)
                    for h_, o_ in zip(h_out[len(fwd_outs):], bwd_outs):
                        h_.copy_(o_, non_blocking=True)
                for o_ in outs:  # the caching allocator must not recycle them early
                    o_.record_stream(s_d2h)
                if join:
                    stream.wait_stream(s_d2h)
            return outs

        outs = e2e_step()
        torch.cuda.synchronize()
        h_out = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in outs]
        e2e_steps = max(1, min(args.steps, 10))
        # latency: each step on its own (its outputs back on the host before the
        # next one starts)
        t_lat = 0.0
        for it in range(e2e_steps + 1):
            if not args.no_flush:
                flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            e2e_step(h_out)
            e1.record(stream)  # after stream.wait_stream(s_d2h): all copies done
            e1.synchronize()
            if it > 0:  # first iteration warms the pinned paths
                t_lat += e0.elapsed_time(e1)
        lat_ms = t_lat / e2e_steps
        # throughput: the steps back to back, as a training loop runs them -- step
        # i's outputs stream back while step i+1's inputs arrive and it computes
        # (every step still copies all its inputs in and all its outputs out)
        # (at most two steps in flight: step i waits for step i-2's copies, so
        # the caching allocator recycles output blocks instead of growing)
        def pipelined(n_steps):
            done = []
            for it in range(n_steps):
                if it >= 2:
                    stream.wait_event(done[it - 2])
                if not args.no_flush:
                    flush.zero_()
                e2e_step(h_out, join=False)
                ev = torch.cuda.Event()
                ev.record(s_d2h)
                done.append(ev)
            stream.wait_stream(s_d2h)

        pipelined(3)  # warm-up: the allocator's blocks for two steps in flight
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        pipelined(e2e_steps)
        e1.record(stream)
        e1.synchronize()
        e2e_ms = e0.elapsed_time(e1) / e2e_steps
        h2d = sum(h.numel() * h.element_size() for h in h_first + h_late)
        d2h = sum(h.numel() * h.element_size() for h in h_out)
        e2e = [e2e_ms, h2d, d2h, lat_ms]

    per_rank = [t_step / args.steps, n, e2e[0] if e2e else 0.0, e2e[3] if e2e else 0.0] + \
        [t / args.steps for t in t_phase]
    allr = sharding.gather_floats(per_rank)
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return 0
    ms = float(allr[:, 0].max())
    total_q = float(allr[:, 1].sum())
    phase = {nm: float(allr[0, 4 + i]) for i, nm in enumerate(names)}
    value = total_q / (ms * 1e-3)
    peak, peak_src = load_peak()
    c_total = C_TOTAL[args.config]
    if args.config == "D":
        c_total = C_TOTAL["D"] * (n / 6_400_000)
    b_fwd, b_bwd = algorithmic_bytes(n, d, k, c_total)
    if gravnet:  # B_agg = (8Nk + 4NkF + 8NF) + (8NF + 8Nk + 8NkF + 4Nk)
        F = 64
        b_bwd += (8 * n * k + 4 * n * k * F + 8 * n * F) + (8 * n * F + 8 * n * k + 8 * n * k * F + 4 * n * k)
    t_knn_ms = phase["knn_gravnet_fwd" if gravnet else "knn_fwd"]
    b_phase = b_fwd
    if gravnet:  # the fused op also does the aggregation forward: 8Nk + 4NkF + 8NF
        b_phase += 8 * n * k + 4 * n * k * 64 + 8 * n * 64
    achieved = b_phase / (t_knn_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference generate_dataset, seed per rank, cast to float32)",
        "config": {"workload": desc, "n_points_per_gpu": n, "d": d, "k": k, "n_bins": n_bins,
                   "d_bin": d_bin, "events": world if scaling == "weak" else 64,
                   "l2": "no flush" if args.no_flush else "flushed (256 MiB write) before every step",
                   "precision": "fp32 distance filter, float64 exact epilogue / gradient sums"},
        "breakdown_ms": phase,
        "roofline": {"bound": "hbm",
                     "kernel": ("knn_gravnet (k_tiles + k_tile_search + k_tile_finish + redo, then"
                                " the aggregation)") if gravnet else
                               "binned_select_knn (k_tiles + k_tile_search + k_tile_finish + "
                               "k_knn_fwd redo)",
                     "note": "achieved = the reference algorithm's bytes (SURVEY 8(d)) / time; "
                             "frac > 1 means the kernels serve those candidate reads from "
                             "L2/shared memory: traffic is what they take from DRAM",
                     "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": load_traffic(args.config),
                     "peak_source": peak_src,
                     "bytes_model": "SURVEY 8(d) B_fwd = 4Nd + 4d*C_total + 8Nk "
                                    f"(C_total={c_total:.3g}) per launch"
                                    + (" + GravNet fwd 8Nk + 4NkF + 8NF (fused)" if gravnet else ""),
                     "step_frac": (b_fwd + b_bwd) / (ms * 1e-3) / 1e9 / peak},
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if e2e:
        e2e_ms = float(allr[:, 2].max())
        line["e2e"] = {"value": total_q / (e2e_ms * 1e-3), "unit": "queries/s",
                       "h2d_bytes_per_step": int(e2e[1]), "d2h_bytes_per_step": int(e2e[2]),
                       "ms_per_step": e2e_ms,
                       "mode": "steps back to back (step i's outputs copy back while step i+1's "
                               "inputs arrive and it computes); every step moves all its bytes",
                       "latency_ms_per_step": float(allr[:, 3].max())}
    if world == 1 and not args.no_cpu_baseline:
        try:
            tt, det = cpu_reference_step(coords_np, off_np, k, n_bins,
                                         query_frac=REF_QUERY_FRAC.get(args.config, 1.0))
            line["cpu_baseline"] = {"value": n / tt, "unit": "queries/s", "cores": det["cores"],
                                    "kind": det["kind"], "sample": det["sample"]}
        except Exception as exc:  # the baseline must not kill the GPU number
            line["cpu_baseline"] = {"value": None, "unit": "queries/s", "cores": os.cpu_count(),
                                    "kind": "unavailable", "sample": repr(exc)}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
