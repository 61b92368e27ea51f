#!/usr/bin/env python
"""Benchmark of the hot path: bin_by_coordinates -> binned_select_knn forward ->
backward (BASELINE.json metric: N=1M, d=4, k=40, fwd+bwd; % of HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config north_star|A|B|C|D|E]
    python bench.py --impl reference     (the reference's own CPU path, rank 0)

``--gpus N > 1`` without a torchrun environment re-launches this script under
``torch.distributed.run`` with N ranks (one per GPU, NCCL, 127.0.0.1).

Workload (default ``north_star``): one step = one pass of the path over one
event of 1,000,000 uniform points in [0,1)^4 (the reference's generator,
seed 3 + rank, cast to float32), k = 40, fixed upstream gradient for the
backward.  Multi-GPU = event sharding by row splits, one event per GPU (weak
scaling, ``value`` = all ranks' queries / max-over-ranks step time), no
collective in the data path.  Every run also reports ``strong_scaling``: the
64-event batch of config D sharded by row splits over the N ranks (global
n_bins, global neighbour ids), T_N (max over ranks) against T_1 (the whole
batch on rank 0's GPU alone) on the same batch.

Inputs are resident in HBM when the timed region starts; L2 is flushed (256 MiB
write) before every step.  ``e2e`` repeats the measurement with pinned HOST
buffers and the host<->device copies inside the timed region, steps back to
back like a training loop (``latency_ms_per_step`` = one step alone).
"""

from __future__ import annotations

import argparse
import json
import os
import socket
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

# query sample per reference step (DirectionMask: sample rows are queries, every
# vertex stays a candidate, so the per-query cost is the full problem's)
REF_QUERY_FRAC = {"north_star": 1.0, "A": 1.0, "B": 1.0, "C": 0.002, "D": 0.1, "E": 1.0}

SEARCH_KERNELS = ("k_tiles", "k_tile_search", "k_tile_finish", "k_knn_fwd", "k_hd_tiles",
                  "k_hd_search")

DESC = {"north_star": "north_star: 1 event x 1,000,000 uniform points per GPU, d=4, k=40",
        "A": "A: 10k points d=3 k=16", "B": "B: 200k clustered points d=4 k=40",
        "C": "C: 1M points d=10 k=64", "E": "E: 500k points d=4 k=40 + GravNet (F=64)",
        "D": "D: 64 events x 100k points d=4 k=40, row splits sharded over the ranks"}


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


def load_fp32_peak():
    """Measured FP32 CUDA-core peak (tools/micro/fp32_peak.cu, FFMA2) on this pool."""
    path = os.path.join(ROOT, "profiles", "r2", "fp32_peak.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["ffma2_tflops"]), "measured (profiles/r2/fp32_peak.json, FFMA2 loop)"
    except Exception:
        return 74.4, "fallback (148 SMs x 128 FMA/clk x 2 x 1.965 GHz)"


def load_traffic(config):
    """DRAM bytes per search call (its kernels) from the committed ncu captures."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            data = json.load(fh)[config]
        got = [data[k]["dram_bytes_per_launch"] for k in SEARCH_KERNELS if k in data]
        return float(sum(got)) if got else None
    except Exception:
        return None


class ClockSampler:
    """SM clocks + throttle reasons sampled through NVML every millisecond while
    the timed loop runs (nvidia-smi fallback)."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.sm, self.mx, self.reasons = [], [], set()
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
            self._nvml = pynvml
        except Exception:
            self._nvml = None

    def _sample(self):
        if self._nvml is not None:
            p = self._nvml
            self.sm.append(float(p.nvmlDeviceGetClockInfo(self._h, p.NVML_CLOCK_SM)))
            self.mx.append(float(p.nvmlDeviceGetMaxClockInfo(self._h, p.NVML_CLOCK_SM)))
            r = p.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            for name, const in self.REASONS:
                if r & getattr(p, const):
                    self.reasons.add(name)
            return
        out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=clocks.sm,clocks.max.sm,"
                              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip().split(",")
        self.sm.append(float(out[0]))
        self.mx.append(float(out[1]))
        for i, (name, _) in enumerate(self.REASONS):
            if out[2 + i].strip().lower().startswith("active"):
                self.reasons.add(name)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                return
            self._stop.wait(0.001)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": max(self.mx),
                "reasons": sorted(self.reasons), "samples": len(self.sm),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def workload(config, rank, world):
    """-> (coords f32 (local rows), local row splits, k, n_bins, scaling, desc)."""
    from paper_2511_10442_b200.datasets import CONFIGS, generate_dataset
    n, d, splits, k, dist, seed = CONFIGS[config]
    if config == "D":  # strong scaling: the 64-event batch is sharded by row splits
        from paper_2511_10442_b200 import sharding
        coords, off = generate_dataset(n, d, splits, seed, dist)
        sh = sharding.shard(off, rank, world)
        n_bins = sharding.global_n_bins(off, k, d)
        c = coords[sh.vertex_lo:sh.vertex_hi].astype(np.float32)
        return c, sh.local_offsets, k, n_bins, "strong", DESC["D"]
    coords, off = generate_dataset(n, d, splits, seed + rank, dist)
    from paper_2511_10442_b200.binning import compute_n_bins, default_bin_dims
    n_bins = compute_n_bins(int(np.diff(off).max()), k, default_bin_dims(d))
    return coords.astype(np.float32), off, k, n_bins, "weak", DESC[config]


def config_keys(config, n, d, k, n_bins, events, flushed):
    """The workload description shared by both arms (same keys)."""
    return {"workload": DESC[config], "n_points_per_gpu": n, "d": d, "k": k, "n_bins": n_bins,
            "d_bin": min(d, 5), "events": events,
            "l2": ("GPU arm: L2 flushed (256 MiB write) before every step; CPU reference arm: "
                   "no flush") if flushed else "no flush"}


def cpu_reference_step(coords32, offsets, k, n_bins, query_frac=1.0, bwd_rows=100_000, seed=0):
    """One step of the reference's own CPU path on this host: build_index over
    the whole event + binned_knn over all queries (or, where the full search
    takes minutes, a DirectionMask query sample: sample = role 3, the rest stay
    candidates with role 0, so the per-query work is the full problem's) on all
    host threads (oracle/_ref = the reference's compiled _binned_cy kernels),
    then the reference's numpy knn_backward (np.add.at, 1 core) over a random
    sample of bwd_rows rows.  Returns (seconds, queries/s, details): the rate is
    1 / (fwd s per query + bwd s per row), both measured in this step -- no time
    is extrapolated."""
    from oracle import oracle as O  # cpu_baseline / reference leg only
    ref = O.load_ref_kernels()
    kind = "reference" if ref is not None else "port"
    c64 = coords32.astype(np.float64)
    n, n_c = c64.shape
    d_bin = min(n_c, 5)
    threads = os.cpu_count() or 1
    rng = np.random.default_rng(seed)
    if query_frac < 1.0:
        q_rows = np.sort(rng.choice(n, size=max(1, int(n * query_frac)), replace=False))
        mask = np.zeros(n, np.int8)
        mask[q_rows] = 3
    else:
        q_rows, mask = np.arange(n), None
    t0 = time.perf_counter()
    if ref is not None:
        bi, so, bb, mins, widths = ref.build_index(c64, offsets, d_bin, n_bins)
        oi = np.empty((n, k), np.int32)
        od = np.empty((n, k), np.float64)
        ref.binned_knn(c64, bi, so, bb, np.full(d_bin, n_bins, np.int64), widths.min(axis=1).copy(),
                       np.zeros(1, np.int8) if mask is None else mask, mask is not None, 0.0, False,
                       False, k, oi, od, threads)
    else:
        oi, od = O.knn_refslot(c64, offsets, k, n_bins=n_bins, dir_mask=mask, threads=threads)
    t_fwd = time.perf_counter() - t0
    rows = np.sort(rng.choice(q_rows, size=min(bwd_rows, len(q_rows)), replace=False))
    up = rng.standard_normal((len(rows), k))
    t1 = time.perf_counter()
    O.knn_backward_numpy(c64, oi[rows], up, rows)
    t_bwd = time.perf_counter() - t1
    rate = 1.0 / (t_fwd / len(q_rows) + t_bwd / len(rows))
    sample = (f"fwd: build_index over all {n} points + binned_knn over "
              + (f"all {n} queries" if mask is None else
                 f"{len(q_rows)} sampled queries (DirectionMask: sample = role 3, rest = role 0 "
                 "candidates)")
              + f" (reference compiled _binned_cy, {threads} threads); bwd: numpy knn_backward "
              f"(np.add.at, 1 core) over {len(rows)} sampled rows; rate = 1 / (fwd s/query + "
              "bwd s/row), both measured in the step")
    return t_fwd + t_bwd, rate, {"kind": kind, "cores": threads, "t_fwd_s": t_fwd,
                                 "t_bwd_s": t_bwd, "fwd_queries": int(len(q_rows)),
                                 "bwd_rows": int(len(rows)), "sample": sample}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    coords, off, k, n_bins, scaling, desc = workload(args.config, 0, 1)
    n, d = coords.shape
    frac = REF_QUERY_FRAC.get(args.config, 1.0)
    times, fwd_t, bwd_t, det = [], [], [], None
    for s_ in range(max(args.warmup, 0) + args.steps):
        tt, rate, det = cpu_reference_step(coords, off, k, n_bins, frac, seed=100 + s_)
        if s_ >= args.warmup:
            times.append(tt)
            fwd_t.append(det["t_fwd_s"] / det["fwd_queries"])
            bwd_t.append(det["t_bwd_s"] / det["bwd_rows"])
    value = 1.0 / (float(np.mean(fwd_t)) + float(np.mean(bwd_t)))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "queries/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": float(np.mean(times)) * 1e3, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generate_dataset)",
            # same keys and values as the GPU arm's line (weak scaling: one event
            # per GPU; the host's rate is per query, so it covers N events alike)
            "config": config_keys(args.config, n, d, k, n_bins,
                                  max(args.gpus, 1) if scaling == "weak" else len(off) - 1,
                                  not args.no_flush),
            "per_step": {"fwd_queries": det["fwd_queries"], "bwd_rows": det["bwd_rows"],
                         "us_per_query_fwd": float(np.mean(fwd_t)) * 1e6,
                         "us_per_row_bwd": float(np.mean(bwd_t)) * 1e6},
            "cpu_baseline": {"value": value, "unit": "queries/s", "cores": det["cores"],
                             "kind": det["kind"], "sample": det["sample"]},
            "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def spawn(args):
    """--gpus N > 1 outside torchrun: re-launch under torch.distributed.run."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible", file=sys.stderr)
        return 2
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def timed_steps(step, n_steps, warmup, stream, flush=None, world=1):
    """Warm-up, then n_steps steps bracketed by barrier + synchronize, each timed
    with CUDA events on ``stream``; returns (mean ms per step, phase ms list)."""
    import torch
    import torch.distributed as dist
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    tot, phases = 0.0, None
    for _ in range(n_steps):
        if flush is not None:
            flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        marks = step()
        e1.record(stream)
        e1.synchronize()
        tot += e0.elapsed_time(e1)
        if marks:
            m = [e0] + marks + [e1]
            ph = [m[i].elapsed_time(m[i + 1]) for i in range(len(m) - 1)]
            phases = ph if phases is None else [a + b for a, b in zip(phases, ph)]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    return tot / n_steps, [p / n_steps for p in phases] if phases else []


def strong_scaling(args, rank, world, dev, flush):
    """Config D (64 events x 100k, d=4, k=40) sharded by row splits: T_N = max
    over ranks of one step of the rank's share; T_1 = the whole batch on rank 0's
    GPU alone.  Same batch, same global n_bins, global neighbour ids."""
    import torch
    import torch.distributed as dist
    from paper_2511_10442_b200 import ops, sharding
    from paper_2511_10442_b200.datasets import CONFIGS, generate_dataset
    n, d, splits, k, distn, seed = CONFIGS["D"]
    coords, off = generate_dataset(n, d, splits, seed, distn)
    coords = coords.astype(np.float32)
    nb = sharding.global_n_bins(off, k, d)
    stream = torch.cuda.current_stream(dev)
    steps = max(1, min(args.steps, 5))
    gen = torch.Generator(device=dev)
    gen.manual_seed(77)

    def make_step(lo, hi, offs):
        c = torch.from_numpy(coords[lo:hi]).to(dev)
        rs = torch.from_numpy(np.asarray(offs, np.int64)).to(dev)
        up = torch.randn((hi - lo, k), generator=gen, device=dev)

        def step():
            bi, so, bb, mins, widths, sc = ops.bin_by_coordinates(c, rs, min(d, 5), nb)
            idx, d2 = ops.binned_select_knn(c, rs, bi, so, bb, mins, widths, sc, k, min(d, 5), nb,
                                            None, None, False, False)
            ops.binned_select_knn_grad(up, idx, c, so)
            return []
        return step

    sh = sharding.shard(off, rank, world)
    t_n, _ = timed_steps(make_step(sh.vertex_lo, sh.vertex_hi, sh.local_offsets), steps, 2, stream,
                         flush, world)
    t_all = sharding.gather_floats([t_n, float(sh.n_events)])
    t1 = None
    if world == 1:
        t1 = t_n
    else:
        if rank == 0:
            t1, _ = timed_steps(make_step(0, n, off), steps, 2, stream, flush, 1)
        dist.barrier()
    if rank != 0:
        return None
    tn = float(t_all[:, 0].max())
    return {"workload": "D: 64 events x 100,000 uniform points, d=4, k=40, fwd+bwd; row splits "
                        "sharded over the ranks (contiguous event ranges), global n_bins, no "
                        "collective in the data path",
            "n_gpus": world, "steps": steps, "t1_ms": t1, "tn_ms": tn,
            "speedup_t1_over_tn": t1 / tn, "events_per_rank": [int(x) for x in t_all[:, 1]],
            "t_rank_ms": [float(x) for x in t_all[:, 0]],
            "note": "T_1 = the whole batch on rank 0's GPU alone (same process, same batch)"}


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
    ap.add_argument("--no-strong", action="store_true", help="skip the config-D strong-scaling block")
    ap.add_argument("--deterministic", action="store_true",
                    help="bitwise-repeatable backward (FG_BWD_DETERMINISTIC)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn(args)

    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

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
    flush = None if args.no_flush else torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    det = args.deterministic

    gravnet = args.config == "E"  # config E: the GravNetOp layer on top of the search
    if gravnet:
        n_feat = 64
        feats = torch.from_numpy(rng.standard_normal((n, n_feat)).astype(np.float32)).to(dev)
        up_agg = torch.from_numpy(rng.standard_normal((n, 2 * n_feat)).astype(np.float32)).to(dev)

    def run_path(c, u, f=None, ua=None, marks=None):
        """One pass of the path; ``marks`` collects phase events."""
        def mark():
            if marks is not None:
                e = torch.cuda.Event(enable_timing=True)
                e.record(stream)
                marks.append(e)

        bi, so, bb, mins, widths, sc = ops.bin_by_coordinates(c, rs, d_bin, n_bins)
        mark()
        if gravnet:  # GravNetOp layer: search + aggregation, then its backward
            idx, d2, agg = ops.knn_gravnet(c, rs, bi, so, bb, mins, widths, sc, k, d_bin, n_bins,
                                           f, 10.0, [0, 1], True)
            mark()
            gf, gd = ops.gravnet_aggregate_grad(ua, f, idx, d2, 10.0, [0, 1], True, so)
            mark()
            g = ops.binned_select_knn_grad(gd, idx, c, so, det)
            return [idx, d2, agg], [g, gf]
        idx, d2 = ops.binned_select_knn(c, rs, bi, so, bb, mins, widths, sc, k, d_bin, n_bins,
                                        None, None, False, False)
        mark()
        g = ops.binned_select_knn_grad(u, idx, c, so, det)
        return [idx, d2], [g]

    names = (["bin_by_coordinates", "knn_gravnet_fwd", "gravnet_bwd", "knn_bwd"] if gravnet
             else ["bin_by_coordinates", "knn_fwd", "knn_bwd"])

    def step():
        marks = []
        run_path(coords, up, feats if gravnet else None, up_agg if gravnet else None, marks)
        return marks

    # warm-up: at least W (>= 3) steps and 1.5 s of work, so the SM clocks have left idle
    t_warm = time.perf_counter()
    it = 0
    while it < max(args.warmup, 3) or time.perf_counter() - t_warm < 1.5:
        step()
        torch.cuda.synchronize()
        it += 1
    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")[local:local + 1]
    sampler = ClockSampler(int(vis[0]) if vis and vis[0].isdigit() else local)
    launches0 = _lib.launch_count()
    with sampler:
        t_step, t_phase = timed_steps(step, args.steps, 0, stream, flush, world)
    launches = _lib.launch_count() - launches0
    clocks = sampler.summary()

    # e2e through the public API with pinned host buffers: every step copies its
    # inputs in and every output back inside the timed region.  The copies run
    # on their own streams and overlap the compute the way a user pipeline
    # would: coordinates (+ features) first, the upstream gradients while the
    # search runs; the forward outputs go back while the backward runs.
    e2e = None
    e2e_reps = []
    if not args.no_e2e:
        s_h2d = torch.cuda.Stream(dev)
        s_d2h = torch.cuda.Stream(dev)
        copy_streams = [s_h2d, s_d2h]  # replaced per timed repetition (see below)
        h_first = [torch.from_numpy(coords_np).pin_memory()]
        h_late = [torch.from_numpy(up_np).pin_memory()] if not gravnet else [up_agg.cpu().pin_memory()]
        if gravnet:
            h_first.append(feats.cpu().pin_memory())
        d_first = [torch.empty_like(h, device=dev) for h in h_first]
        d_late = [torch.empty_like(h, device=dev) for h in h_late]

        def e2e_step(h_out=None, join=True):
            s_h2d, s_d2h = copy_streams
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
                bwd_outs = [ops.binned_select_knn_grad(gd, idx, c, so, det), gf]
            else:
                bwd_outs = [ops.binned_select_knn_grad(d_late[0], idx, c, so, det)]
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
                # no record_stream: the caller keeps the outputs alive until `stream`
                # has waited for their copies (join below, or pipelined()'s window),
                # so the caching allocator recycles blocks in stream order without
                # polling copy-stream events
                if join:
                    stream.wait_stream(s_d2h)
            return outs

        outs = e2e_step()
        torch.cuda.synchronize()
        h_out = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in outs]
        e2e_steps = max(1, min(args.steps, 10))
        t_lat = 0.0
        for it in range(e2e_steps + 1):  # one step alone: outputs on the host before the next
            if flush is not None:
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

        # steps back to back, at most two in flight (step i waits for step i-2's
        # copies, so the caching allocator recycles output blocks)
        def pipelined(n_steps):
            done, alive = [], []
            for it in range(n_steps):
                if it >= 2:
                    stream.wait_event(done[it - 2])
                    alive.pop(0)  # step it-2's outputs: their copies are ordered before `stream` now
                if flush is not None:
                    flush.zero_()
                alive.append(e2e_step(h_out, join=False))
                ev = torch.cuda.Event()
                ev.record(copy_streams[1])
                done.append(ev)
            stream.wait_stream(copy_streams[1])
            alive.clear()

        # back to back: three timed repetitions, each on fresh copy streams after
        # >= 0.3 s of warm-up in that mode; the median is reported and every
        # repetition listed (single runs were seen 1.6x slower than the rest:
        # 10.5 vs 6.6 ms at north_star, 14 vs 4 ms at B -- copies serialised)
        reps = []
        for rep in range(3):
            copy_streams[:] = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
            t_w = time.perf_counter()
            while True:
                pipelined(3)
                torch.cuda.synchronize()
                if time.perf_counter() - t_w >= 0.3:
                    break
            if world > 1:
                dist.barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pipelined(e2e_steps)
            e1.record(stream)
            e1.synchronize()
            reps.append(e0.elapsed_time(e1) / e2e_steps)
        e2e_ms = float(np.median(reps))
        h2d = sum(h.numel() * h.element_size() for h in h_first + h_late)
        d2h = sum(h.numel() * h.element_size() for h in h_out)
        e2e = [e2e_ms, h2d, d2h, lat_ms]
        e2e_reps = reps

    per_rank = [t_step, n, e2e[0] if e2e else 0.0, e2e[3] if e2e else 0.0] + list(t_phase)
    allr = sharding.gather_floats(per_rank)
    strong = None if args.no_strong else strong_scaling(args, rank, world, dev, flush)
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
    compulsory = 4 * n * d + 8 * n * k  # coords in, idx + d2 out
    if gravnet:  # the op also does the aggregation forward: 8Nk + 4NkF + 8NF
        b_phase += 8 * n * k + 4 * n * k * 64 + 8 * n * 64
        compulsory += 4 * n * 64 + 4 * n * 128
    achieved = b_phase / (t_knn_ms * 1e-3) / 1e9
    traffic = load_traffic(args.config)
    if d > 4:  # config C: the search is FP32 compute, not bytes (3 d C_total flops)
        fpk, fpk_src = load_fp32_peak()
        flops = 3.0 * d * c_total
        ach = flops / (t_knn_ms * 1e-3) / 1e12
        roof = {"bound": "fp32", "kernel": "binned_select_knn (k_hd_tiles + k_hd_search: lane-per-"
                                          "query tiles, FADD2/FFMA2 over broadcast candidates)",
                "achieved": ach, "peak": fpk, "unit": "TFLOP/s", "frac": ach / fpk,
                "frac_kind": "model: SURVEY 8(d) 3*d*C_total fp32 flops (the reference algorithm's "
                             "candidate count) / measured search time",
                "flops_model": f"3 * d * C_total = 3 * {d} * {c_total:.3g}",
                "peak_source": fpk_src, "traffic": traffic,
                "compulsory_bytes": compulsory,
                "binding": "SM issue / latency (ncu: IPC ~1.1-1.5 at 6 warps/SM, the per-lane "
                           "buffers' shared memory bounds occupancy; profiles/r2/)",
                "hbm_model_frac": achieved / peak}
        b_phase = None
    else:
        roof = None
    if roof is None:
      roof = {"bound": "hbm",
            "kernel": ("knn_gravnet (k_tiles + k_tile_search + k_tile_finish + redo, then the "
                       "aggregation)") if gravnet else
                      "binned_select_knn (k_tiles + k_tile_search + k_tile_finish + k_knn_fwd redo)",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "frac_kind": "model: SURVEY 8(d) algorithmic bytes (counts the reference algorithm's "
                         "candidate reads, which these kernels serve from L2/shared memory) / "
                         "measured time; not a DRAM measurement",
            "bytes_model": "B_fwd = 4Nd + 4d*C_total + 8Nk "
                           f"(C_total={c_total:.3g}) per launch"
                           + (" + GravNet fwd 8Nk + 4NkF + 8NF" if gravnet else ""),
            "compulsory_bytes": compulsory,
            "compulsory_frac": compulsory / (t_knn_ms * 1e-3) / 1e9 / peak,
            "traffic": traffic,
            "dram_frac": (traffic / (t_knn_ms * 1e-3) / 1e9 / peak) if traffic else None,
            "traffic_source": "ncu dram__bytes_read+write of the search kernels "
                              "(profiles/ncu_summary.json, same build)",
            "binding": "SM instruction issue / latency (ncu: k_tile_search and k_tile_finish "
                       "SM throughput ~70%, DRAM < 15%; profiles/)",
            "peak_source": peak_src,
            "step_frac_model": (b_fwd + b_bwd) / (ms * 1e-3) / 1e9 / peak}
      if d > 4 or d_bin < d:
          roof["kernel"] = "binned_select_knn (k_hd_tiles + k_hd_search)"
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference generate_dataset, seed per rank, cast to float32)",
        # the same config keys and values as the reference arm's line
        "config": config_keys(args.config, n, d, k, n_bins,
                              world if scaling == "weak" else 64, not args.no_flush),
        "precision": "fp32 distance filter, float64 exact epilogue / gradient terms",
        "backward_mode": "deterministic transposed" if det else
                         "compensated fp32x4 atomics (pipelined stream kernel for d = 4)",
        "breakdown_ms": phase,
        "roofline": roof,
        "gpu_launches": int(launches),
        "clocks": clocks,
    }
    if strong:
        line["strong_scaling"] = strong
    if e2e:
        e2e_ms = float(allr[:, 2].max())
        line["e2e"] = {"value": total_q / (e2e_ms * 1e-3), "unit": "queries/s",
                       "h2d_bytes_per_step": int(e2e[1]), "d2h_bytes_per_step": int(e2e[2]),
                       "ms_per_step": e2e_ms,
                       "mode": "steps back to back (step i's outputs copy back while step i+1's "
                               "inputs arrive and it computes); every step moves all its bytes",
                       "latency_ms_per_step": float(allr[:, 3].max()),
                       "repetitions_ms_per_step": [round(float(x), 4) for x in e2e_reps],
                       "statistic": "median of 3 timed repetitions (rank 0's list; max over ranks of the median)"}
    if world == 1 and not args.no_cpu_baseline:
        try:
            tt, rate, det_ = cpu_reference_step(coords_np, off_np, k, n_bins,
                                                REF_QUERY_FRAC.get(args.config, 1.0))
            line["cpu_baseline"] = {"value": rate, "unit": "queries/s", "cores": det_["cores"],
                                    "kind": det_["kind"], "sample": det_["sample"]}
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
