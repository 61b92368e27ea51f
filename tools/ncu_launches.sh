# per-launch device times of one bench step (cold-cache, serialised: compare shares)
CFG=${1:-north_star}
OUT=${2:-launches}
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$OUT.csv python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-strong > /dev/null 2>&1
python - "$OUT" <<'PY'
import csv, sys, collections
rows = list(csv.reader(open(f"gpurun_out/{sys.argv[1]}.csv")))
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hd = rows[h]; ki = hd.index("Kernel Name"); vi = hd.index("Metric Value")
agg = collections.OrderedDict()
for r in rows[h + 1:]:
    agg.setdefault(r[ki][:70], []).append(float(r[vi].replace(",", "")))
for k, v in agg.items():
    print(f"{k:70s} n={len(v):3d} last_us={v[-1] / 1000:10.2f}")
PY
