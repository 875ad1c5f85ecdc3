"""Write the r02 evidence under profiles/ from this round's gpurun_out captures:
  r02_launches.csv (ncu launch list of a bench run) -> r02_launches_step.csv + r02_launches_summary.txt
  r02_k2tc_dense / r02_k2tc_sparse / r02_k1_chain / r02_k2simt_cfg4 .ncu-rep -> r02_ncu_*.txt
  r02_bench.json -> r02_bench.json (the last line)
  dbg2_tdprof.log / cpu_engines.log -> r02_tdprof.txt / r02_cpu_engines.txt

    python tools/make_profiles_r02.py <launches per bench step>"""
import collections
import csv
import json
import subprocess
import sys

PER_STEP = int(sys.argv[1]) if len(sys.argv) > 1 else 300
G = "gpurun_out/"
P = "profiles/"
TU = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
BU = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}


def launches():
    rows = list(csv.reader(open(G + "r02_launches.csv")))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr = rows[hi]
    data = [dict(zip(hdr, r)) for r in rows[hi + 1:] if len(r) == len(hdr)]
    ids = sorted({int(d["ID"]) for d in data})
    # the timed step = the last PER_STEP launches of the mmmcu kernels
    mm = [i for i in ids if any(d["ID"] == str(i) and "mmmcu::" in d["Kernel Name"] for d in data[:0])]
    keep_ids = set(ids[-PER_STEP:])
    keep = [d for d in data if int(d["ID"]) in keep_ids]
    with open(P + "r02_launches_step.csv", "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"])
        for d in keep:
            w.writerow([d["ID"], d["Kernel Name"].split("(")[0], d["Metric Name"], d["Metric Unit"], d["Metric Value"]])
    agg = collections.OrderedDict()
    for d in keep:
        k = d["Kernel Name"].split("(")[0].replace("void ", "")
        a = agg.setdefault(k, {"n": set(), "us": 0.0, "rd": 0.0, "wr": 0.0})
        a["n"].add(d["ID"])
        v = float(d["Metric Value"].replace(",", ""))
        if d["Metric Name"] == "gpu__time_duration.sum":
            a["us"] += v * TU[d["Metric Unit"]]
        elif d["Metric Name"] == "dram__bytes_read.sum":
            a["rd"] += v * BU[d["Metric Unit"]]
        elif d["Metric Name"] == "dram__bytes_write.sum":
            a["wr"] += v * BU[d["Metric Unit"]]
    tot = sum(a["us"] for a in agg.values())
    with open(P + "r02_launches_summary.txt", "w") as f:
        f.write("# r02 launch list: one timed bench step (75 sweep cells, AUTO), ncu --metrics gpu__time_duration.sum,"
                "dram__bytes_{read,write}.sum --clock-control none\n# (cold caches, serialised launches: compare SHARES "
                "with the bench's CUDA-event times, not absolute times)\n")
        f.write(f"{len(keep_ids)} launches, {tot / 1000:.3f} ms total\n")
        for k, a in sorted(agg.items(), key=lambda x: -x[1]["us"]):
            n = len(a["n"])
            f.write(f"{k[:30]:30s} n={n:4d} total={a['us'] / 1000:8.3f} ms share={100 * a['us'] / tot:5.1f}% "
                    f"avg={a['us'] / n:8.2f} us  dram_read={a['rd'] / n:7.1f} MB/launch dram_write={a['wr'] / n:6.1f} MB/launch\n")
    print(open(P + "r02_launches_summary.txt").read())


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]


def ncu_summary(rep, out, title):
    raw = subprocess.run(["ncu", "-i", G + rep + ".ncu-rep", "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    with open(P + out, "w") as f:
        f.write(f"# {title}\n# ncu --set full --clock-control none (gpurun_out/{rep}.ncu-rep)\n")
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            u = dict(zip(hdr, units))
            f.write(f"\n{d['Kernel Name'][:90]}\n")
            for k in KEYS:
                if k in d and d[k] != "":
                    f.write(f"  {k:65s} {d[k]:>14s} {u.get(k, '')}\n")
            st = [(float(d[h].replace(",", "")), h) for h in hdr
                  if "pcsamp_warps_issue_stalled" in h and not h.endswith("not_issued") and d[h] not in ("", "n/a")]
            tot = sum(v for v, _ in st) or 1.0
            f.write("  stall reasons (pc samples): " + ", ".join(
                f"{h.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.0f}%"
                for v, h in sorted(st, reverse=True)[:7]) + "\n")
    print(open(P + out).read())


if __name__ == "__main__":
    launches()
    ncu_summary("r02_k2tc_dense", "r02_ncu_k2tc_dense.txt", "K2-TC on the dense sweep cell zA=0.6 zB=0.6 bw=8 (tools/tc_profile.py)")
    ncu_summary("r02_k2tc_sparse", "r02_ncu_k2tc_sparse.txt", "K2-TC on the sparse-k sweep cell zA=0.6 zB=0.95 bw=32")
    ncu_summary("r02_k1_chain", "r02_ncu_k1_chain.txt", "K1 chain (k1_pass, k1_fin, k1_pack_auto) on the cell zA=0.6 zB=0.6 bw=8")
    ncu_summary("r02_k2simt_cfg4", "r02_ncu_k2simt_cfg4.txt", "K2-SIMT (k2_simt2<16>) on configs[3] (skinny 64x12288x49152): FP32 pipe")
    d = json.loads(open(G + "r02_bench.json").read().strip().splitlines()[-1])
    json.dump(d, open(P + "r02_bench.json", "w"), indent=1)
    for src, dst in (("r02_tdprof.log", "r02_tdprof.txt"), ("cpu_engines.log", "r02_cpu_engines.txt")):
        try:
            open(P + dst, "w").write(open(G + src).read())
        except OSError:
            pass
