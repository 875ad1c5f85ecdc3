"""Summarise an ncu launch list (gpu__time_duration.sum per launch) of one bench run:
per-kernel launch count, total and average device time, share of the timed step."""
import collections
import csv
import sys


def main(path, last=None):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name", "gpu__time_duration.sum") == "gpu__time_duration.sum":
                data.append(d)
    if last:
        data = data[-int(last):]
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("void ", "")[:48]
        agg[name][0] += 1
        agg[name][1] += float(d["Metric Value"]) * scale[d["Metric Unit"]]
    tot = sum(v[1] for v in agg.values())
    print(f"{len(data)} launches, {tot / 1000:.3f} ms total (ncu: cold caches, serialised)")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:48s} n={n:5d} total={t / 1000:9.3f} ms share={t / tot * 100:5.1f}% avg={t / n:9.2f} us")


if __name__ == "__main__":
    main(*sys.argv[1:])
