"""Aggregate an ncu SASS source export of k_hd_search by code region
(cut_lane, eval_chunk, scan_spans, seed, stages, epilogue ...).
usage: python tools/region_prof.py <sass.csv> <cubin> <mangled kernel substring>"""
import collections, re, subprocess, sys

src = open("paper_2511_10442_b200/csrc/fg_knn_hd.cuh").read().splitlines()


def find(pat):
    return next(i + 1 for i, l in enumerate(src) if pat in l)


marks = [("helpers", 1)]
for name, pat in [("cut_lane", "__device__ __noinline__ int cut_lane"),
                  ("seed_bound", "__device__ __forceinline__ float seed_bound"),
                  ("eval_chunk", "__device__ __forceinline__ void eval_chunk"),
                  ("scan_spans", "__device__ __forceinline__ void scan_spans"),
                  ("search_setup", "k_hd_search(const __grid_constant__"),
                  ("stages", "---- staged region growth"),
                  ("epilogue(hd)", "---- epilogue, one row at a time"),
                  ("k_abs", "static __global__ void k_abs_bound")]:
    try:
        marks.append((name, find(pat)))
    except StopIteration:
        pass
marks.sort(key=lambda x: x[1])
out = subprocess.run(["python", "tools/sass_lines.py", *sys.argv[1:4], "100000"],
                     capture_output=True, text=True).stdout.splitlines()
agg, st = collections.Counter(), collections.Counter()
for l in out[1:]:
    m = re.match(r"\s*([\d.]+)M\s+([\d.]+)%\s+stall\s+([\d.]+)%\s+(\S+)", l)
    if not m:
        continue
    loc = m.group(4).split("<")[0]
    f, ln = loc.split(":")[0], int(loc.split(":")[1])
    name = f
    if f == "fg_knn_hd.cuh":
        for nm, start in marks:
            if ln >= start:
                name = nm
    agg[name] += float(m.group(1))
    st[name] += float(m.group(3))
tot = sum(agg.values())
print(f"total {tot:.1f}M warp instructions")
for k, v in agg.most_common():
    print(f"{k:28s} {v:8.1f}M {100 * v / tot:5.1f}%  stall {st[k]:.1f}%")
