"""Stall reasons per code region of an ncu source export (--page source
--print-source sass), regions = instruction blocks by execution count."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
ia = h.index("Source"); ie = h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ri = [h.index(c) for c in reasons]
L = []
for r in rows[2:]:
    if len(r) <= ie or not r[ie].isdigit():
        continue
    L.append((r[ia].strip(), int(r[ie]), [int(r[i]) if r[i].isdigit() else 0 for i in ri]))
tot = sum(sum(x[2]) for x in L)
blocks = collections.defaultdict(lambda: [0, 0, [0] * len(reasons), ""])
for s, n, st in L:
    k = round(n / 2e4) if n else -1
    b = blocks[k]
    b[0] += 1; b[1] += n; b[3] = b[3] or s[:40]
    for j, v in enumerate(st): b[2][j] += v
for k in sorted(blocks, key=lambda k: -sum(blocks[k][2]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 10]:
    c, n, st, s0 = blocks[k]
    top = sorted(zip(reasons, st), key=lambda x: -x[1])[:5]
    print(f"exec~{k*2e4/1e6:6.2f}M n={c:4d} instr={n/1e6:7.1f}M samples={100*sum(st)/tot:5.1f}%  " +
          " ".join(f"{r[6:]}={100*v/max(sum(st),1):.0f}%" for r, v in top))
