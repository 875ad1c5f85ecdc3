"""Regenerate the committed evidence under profiles/ from a tools/capture_evidence.sh run
(gpurun_out/r01_launches.csv, r01_cell_full.ncu-rep, r01_k2tc_sparse.ncu-rep, r01_bench.json):

    gpurun -- ./tools/capture_evidence.sh   # on the GPU box
    python tools/make_profiles.py 450      # here

    python tools/make_profiles.py <launches per bench step>
"""
import csv
import json
import shutil
import subprocess
import sys

PER_STEP = int(sys.argv[1]) if len(sys.argv) > 1 else 450
G = "gpurun_out/"


def launch_list():
    rows = list(csv.reader(open(G + "r01_launches.csv")))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    data = [dict(zip(hdr, r)) for r in rows[hi + 1:] if len(r) == len(hdr)]
    ids = set(sorted({int(d["ID"]) for d in data})[-PER_STEP:])
    keep = [d for d in data if int(d["ID"]) in ids]
    with open("profiles/r01_launches_step.csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"])
        for d in keep:
            w.writerow([d["ID"], d["Kernel Name"].split("(")[0], d["Metric Name"], d["Metric Unit"], d["Metric Value"]])
    agg = {}
    tu = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    bu = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    for d in keep:
        k = d["Kernel Name"].split("(")[0].replace("void ", "")
        a = agg.setdefault(k, {"n": set(), "us": 0.0, "rd": 0.0, "wr": 0.0})
        a["n"].add(d["ID"])
        v = float(d["Metric Value"])
        if d["Metric Name"] == "gpu__time_duration.sum":
            a["us"] += v * tu[d["Metric Unit"]]
        elif "read" in d["Metric Name"]:
            a["rd"] += v * bu[d["Metric Unit"]]
        else:
            a["wr"] += v * bu[d["Metric Unit"]]
    tot = sum(a["us"] for a in agg.values())
    out = ["# r01 launch list: one timed bench step (75 sweep cells, AUTO), ncu --metrics "
           "gpu__time_duration.sum,dram__bytes_{read,write}.sum --clock-control none",
           "# (cold caches, serialised launches: compare SHARES with the bench's CUDA-event times, not absolute times)",
           f"{len(ids)} launches, {tot / 1000:.3f} ms total"]
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["us"]):
        n = len(a["n"])
        out.append(f"{k:30s} n={n:4d} total={a['us'] / 1000:8.3f} ms share={a['us'] / tot * 100:5.1f}% "
                   f"avg={a['us'] / n:8.2f} us  dram_read={a['rd'] / n:7.1f} MB/launch dram_write={a['wr'] / n:6.1f} MB/launch")
    open("profiles/r01_launches_summary.txt", "w").write("\n".join(out) + "\n")
    print("\n".join(out))
    tc = agg.get("mmmcu::k2_tc<1>") or agg.get("k2_tc<1>")
    return tc and (tc["rd"] + tc["wr"]) / len(tc["n"])


def ncu_block(rep, kernel_regex, title):
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv", "-k", "regex:" + kernel_regex],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(det.splitlines()))
    if len(rows) < 2:
        return [f"## {title}: not captured"]
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    first = rows[1][0]
    keys = ["Duration", "Elapsed Cycles", "Memory Throughput", "DRAM Throughput", "L2 Hit Rate", "L2 Cache Throughput",
            "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "No Eligible",
            "Registers Per Thread", "Dynamic Shared Memory Per Block", "Achieved Occupancy"]
    out, seen = [f"## {title}"], set()
    for r in rows[1:]:
        if r[0] != first:
            continue
        m = r[ix["Metric Name"]]
        if m in keys and m not in seen:
            seen.add(m)
            out.append(f"  {m:40s} {r[ix['Metric Value']]:>14s} {r[ix['Metric Unit']]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "-k", "regex:" + kernel_regex],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) > 2:
        for i, k in enumerate(rr[0]):
            if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
                     "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"):
                out.append(f"  {k:40s} {rr[2][i]:>14s} {rr[1][i]}")
    return out


def ncu_summaries():
    out = ["# r01 ncu --set full --clock-control none --import-source on: one AUTO multiply of a 4096^3 sweep cell "
           "(tools/tc_profile.py <zA> <zB> <bw> 0)"]
    rep = G + "r01_cell_full.ncu-rep"
    for rx, t in (("k2_tc", "k2_tc<true> (fp16 split, CTA pairs), dense cell zA=zB=0.6 bw=8"),
                  ("k1_pass", "k1_pass, dense cell"), ("k1_pack_auto", "k1_pack_auto, dense cell"),
                  ("k1_csr", "k1_csr<uint16_t>, dense cell")):
        out += ncu_block(rep, rx, t)
    out += ncu_block(G + "r01_k2tc_sparse.ncu-rep", "k2_tc", "k2_tc<true>, sparse-k cell zA=0.6 zB=0.95 bw=16")
    open("profiles/r01_ncu_cell.txt", "w").write("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    tc_bytes = launch_list()
    ncu_summaries()
    if tc_bytes:
        json.dump({"k2_tc": {"bytes_per_launch": round(tc_bytes * 1e6),
                             "source": "r01: dram__bytes_read.sum + dram__bytes_write.sum averaged over the 75 K2-TC "
                                       "launches of one timed sweep step (profiles/r01_launches_summary.txt); "
                                       "algorithmic bytes per cell, 4*(MK + K_live*N + MN), are 201 MB"}},
                  open("profiles/traffic.json", "w"), indent=2)
    shutil.copy(G + "r01_bench.json", "profiles/r01_bench.json")
