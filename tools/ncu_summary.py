"""Summarise ncu full captures (details + raw CSV exports) into
profiles/ncu_summary.json:  python tools/ncu_summary.py CONFIG KERNEL:PREFIX ...
where gpurun_out/PREFIX.details.csv and PREFIX.raw.csv exist."""
import csv, json, os, sys

DETAILS = ["Duration", "Executed Ipc Active", "Executed Instructions", "Registers Per Thread",
           "Theoretical Occupancy", "Achieved Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate",
           "DRAM Throughput", "Memory Throughput", "L2 Cache Throughput",
           "Compute (SM) Throughput", "Warp Cycles Per Issued Instruction",
           "Avg. Active Threads Per Warp", "Dynamic Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def summarise(prefix):
    out = {}
    with open(prefix + ".details.csv") as fh:
        rows = list(csv.reader(fh))
    hdr = next(r for r in rows if r and r[0] == "ID")
    ki, mi, ui, vi = (hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"),
                      hdr.index("Metric Value"))
    for r in rows:
        if len(r) > vi and r[mi] in DETAILS:
            out["kernel"] = r[ki]
            out[r[mi]] = f"{r[vi]} {r[ui]}".strip()
    with open(prefix + ".raw.csv") as fh:
        raw = list(csv.reader(fh))
    h, u, v = raw[0], raw[1], raw[2]
    dram = 0.0
    for name in RAW:
        if name in h:
            i = h.index(name)
            out[name] = f"{v[i]} {u[i]}".strip()
            if name.startswith("dram__bytes"):
                dram += float(v[i].replace(",", "")) * UNIT.get(u[i], 1)
    out["dram_bytes_per_launch"] = dram
    return out


if __name__ == "__main__":
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = os.path.join(root, "profiles", "ncu_summary.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    cfg = sys.argv[1]
    data.setdefault(cfg, {})
    for spec in sys.argv[2:]:
        kern, prefix = spec.split(":")
        data[cfg][kern] = summarise(os.path.join(root, "gpurun_out", prefix))
    json.dump(data, open(path, "w"), indent=1)
    print(json.dumps({k: {kk: vv.get("Duration"), } for k, vv in data[cfg].items()} if False else
                     {kk: vv.get("Duration") for kk, vv in data[cfg].items()}))
