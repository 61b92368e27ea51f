"""Attribute an ncu SASS source export (instructions executed, stall samples)
to CUDA source lines via nvdisasm -g of the same build's cubin.
usage: python tools/sass_lines.py <ncu .sass.csv> <cubin> <mangled kernel substring> [N]"""
import collections, csv, re, subprocess, sys

prof_csv, cubin, kern = sys.argv[1:4]
N = int(sys.argv[4]) if len(sys.argv) > 4 else 40
lines = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith("//----") and kern in l)
end = next((i for i in range(start + 1, len(lines)) if lines[i].startswith("//----")), len(lines))
cur, ins = None, []
for l in lines[start:end]:
    m = re.search(r'//## File ".*/(\S+)", line (\d+)(?: inlined at ".*/(\S+)", line (\d+))?', l)
    if m:
        cur = f"{m.group(1)}:{m.group(2)}" + (f"<{m.group(3)}:{m.group(4)}" if m.group(3) else "")
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((m.group(2).strip(), cur))
rows = list(csv.reader(open(prof_csv)))
h = rows[1]
ia, ie = h.index("Source"), h.index("Instructions Executed")
isamp = h.index("Warp Stall Sampling (All Samples)")
prof = [(r[ia].strip(), int(r[ie]) if r[ie].isdigit() else 0, int(r[isamp]) if r[isamp].isdigit() else 0)
        for r in rows[2:] if len(r) > ie]
ok = sum(1 for a, b in zip(ins, prof) if a[0].split()[0] == b[0].split()[0])
print(f"sass {len(ins)} profiled {len(prof)} opcode matches {ok}")
agg, samp = collections.Counter(), collections.Counter()
for (txt, src), (ptxt, n, st) in zip(ins, prof):
    agg[src] += n
    samp[src] += st
tot, ts = sum(agg.values()) or 1, sum(samp.values()) or 1
for src, n in agg.most_common(N):
    print(f"{n / 1e6:8.1f}M {100 * n / tot:5.1f}%  stall {100 * samp[src] / ts:5.1f}%  {src}")
