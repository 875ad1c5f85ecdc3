"""Warp-stall samples of one kernel by CUDA source line: ncu SASS-page CSV (--print-source=sass)
joined with `nvdisasm -g -c` line info of the same cubin.
usage: stall_by_line.py SASS_CSV DISASM_TXT MANGLED_KERNEL_NAME [top]"""
import collections
import csv
import re
import sys

sass_csv, dis, fn = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
ia, isamp, iex = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
samples = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        samples.append((int(r[ia], 16), float(r[isamp] or 0), float((r[iex] or "0").replace(",", ""))))
    except ValueError:
        pass
seen = {}
for a, s, e in samples:  # the CSV repeats rows
    seen[a] = (s, e)
base = min(seen)
# line info: walk the function's text section
lines = {}
cur = None
infn = False
for ln in open(dis):
    if ln.startswith(".text."):
        infn = ln.strip().rstrip(":") == ".text." + fn
        continue
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        lines[int(m.group(1), 16)] = cur
agg = collections.defaultdict(lambda: [0.0, 0.0])
for a, (s, e) in seen.items():
    key = lines.get(a - base, "?")
    agg[key][0] += s
    agg[key][1] += e
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
print(f"{len(seen)} instrs, {tot:.0f} samples, {toti:.0f} warp-instrs executed")
for k, (s, e) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{100 * s / tot:5.1f}% samp {100 * e / toti:5.1f}% inst  {k}")
