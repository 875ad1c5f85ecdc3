"""Top SASS instructions by warp-stall samples from `ncu -i X.ncu-rep --page source --csv
--print-source=sass` output (what the profile says the kernel waits on)."""
import csv
import sys


def main(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    i_src, i_all = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    data = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        try:
            data.append((float(r[i_all]), r[0][-5:], r[i_src].strip()[:90]))
        except ValueError:
            pass
    tot = sum(d[0] for d in data) or 1.0
    print(f"{len(data)} instructions, {tot:.0f} samples")
    for v, a, s in sorted(data, reverse=True)[: int(top)]:
        print(f"{v / tot * 100:5.1f}%  {a}  {s}")


if __name__ == "__main__":
    main(*sys.argv[1:])
