"""Per-kernel device time / DRAM bytes of the LAST launch of each kernel in an ncu CSV launch list."""
import collections
import csv
import sys

for f in sys.argv[1:]:
    rows = list(csv.reader(open(f)))
    hdr, agg = None, collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("mmmcu::", "")[:16]
            agg.setdefault((d["ID"], name), []).append((d["Metric Name"], d["Metric Value"], d["Metric Unit"]))
    last = {}
    for (i, n), v in agg.items():
        last[n] = v
    out = []
    sc = {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "ns": 1e-3, "us": 1, "ms": 1e3}
    bs = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}
    for n, v in last.items():
        dd = {m: (float(x.replace(",", "")), u) for m, x, u in v}
        t = dd["gpu__time_duration.sum"]
        s = f"{n}={t[0] * sc[t[1]]:.1f}us"
        if "dram__bytes_read.sum" in dd:
            rd, wr = dd["dram__bytes_read.sum"], dd["dram__bytes_write.sum"]
            s += f" r{rd[0] * bs[rd[1]]:.0f}w{wr[0] * bs[wr[1]]:.0f}MB"
        out.append(s)
    print(f.split("/")[-1][:-4].ljust(26), "  ".join(out))
