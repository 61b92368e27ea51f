"""Hottest SASS lines of an ncu source export (stall samples), with totals per
stall reason: python tools/sass_hot.py gpurun_out/X.sass.csv [N]"""
import csv
import sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
h = next(i for i, r in enumerate(rows) if r and "Source" in r)
hd = rows[h]
src = hd.index("Source")
samp = next(i for i, c in enumerate(hd) if c.startswith("Warp Stall Sampling (All"))
stall_cols = [i for i, c in enumerate(hd) if c.startswith("stall_") or "Stall" in c and i != samp]
lines = []
for r in rows[h + 1:]:
    if len(r) <= samp:
        continue
    try:
        v = float(r[samp] or 0)
    except ValueError:
        continue
    lines.append((v, r))
tot = sum(v for v, _ in lines) or 1
print("total samples", tot)
for v, r in sorted(lines, key=lambda x: -x[0])[:n]:
    print(f"{100 * v / tot:5.1f}%  {r[0]:>6s}  {r[src][:90]}")
ie = hd.index("Instructions Executed") if "Instructions Executed" in hd else None
if ie is not None:
    from collections import Counter
    ops = Counter()
    tot_i = 0
    for v, r in lines:
        try:
            c = int(r[ie] or 0)
        except ValueError:
            continue
        tot_i += c
        op = r[src].split()[0] if not r[src].strip().startswith("@") else r[src].split()[1]
        ops[op.split(".")[0]] += c
    print("executed warp instructions", tot_i)
    for op, c in ops.most_common(25):
        print(f"  {op:10s} {c:12d} {100 * c / tot_i:5.1f}%")
