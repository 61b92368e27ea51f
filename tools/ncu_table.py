"""Summarise an ncu --csv metrics log: one line per launch, metrics as columns.
usage: python tools/ncu_table.py LOG.csv [name-filter]"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
flt = sys.argv[2] if len(sys.argv) > 2 else ""
h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hd = rows[h]
ii, ki, mi, vi = hd.index("ID"), hd.index("Kernel Name"), hd.index("Metric Name"), hd.index("Metric Value")
launch = OrderedDict()
names = []
for r in rows[h + 1:]:
    if len(r) <= vi or flt not in r[ki]:
        continue
    key = (r[ii], r[ki].split("(")[0][:48])
    launch.setdefault(key, OrderedDict())[r[mi]] = r[vi]
    if r[mi] not in names:
        names.append(r[mi])
short = [n.replace("gpu__time_duration.sum", "us").replace("dram__bytes_read.sum", "dramR_MB")
         .replace("dram__bytes_write.sum", "dramW_MB")
         .replace("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%")
         .replace("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram%")
         .replace("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%")[:12] for n in names]
print(f"{'kernel':50s}" + "".join(f"{s:>12s}" for s in short))
for (i, k), m in launch.items():
    out = []
    for n in names:
        v = float(m.get(n, "nan").replace(",", ""))
        if n == "gpu__time_duration.sum":
            v /= 1000
        elif n.startswith("dram__bytes"):
            v /= 1e6
        out.append(f"{v:12.1f}")
    print(f"{k:50s}" + "".join(out))
