#!/usr/bin/env python
"""Benchmark of the masked fp32 matmul hot path (BASELINE.json metric: useful GFLOP/s of masked
fp32 matmul at 60-95% zeros, % of roofline, 1/2/4/8 GPUs).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload sweep|cfg1|cfg3|cfg4|cfg5]

One STEP = one pass of the hot path — K1 preprocessing (A/B sparsity maps, index lists,
pattern codes, exact counters) + K2 masked multiply (C += A*B) — over every cell of the
workload, inputs resident in HBM.  The default workload is BASELINE.json configs[1]: the
4096^3 fp32 sparsity sweep, zA x zB in {.6,.7,.8,.9,.95}^2 x B block width {8,16,32}
(75 cells), uniform[-1,1] values, i.i.d. Bernoulli masks (seeded synthetic data).

Multi-GPU (--gpus N: one process per GPU, re-launched under torchrun when WORLD_SIZE is not
set; NCCL): the default workload becomes configs[4] with STRONG scaling — one 32768 x 8192 A
whose rows are partitioned across the ranks by mmmcu_shard_rows (each rank generates its own
rows), B generated on rank 0 and broadcast ONCE with NCCL before timing (broadcast_ms) — and
each rank computes its own C rows; timing is max over ranks.  The N=1 sweep line also carries
the 1-GPU configs[4] value (cfg5_1gpu) as the same-workload reference of the scaling run.

value     = Σ 2*lane_fma_ops over all ranks / step time     (useful GFLOP/s)
e2e       = the same metric end to end through the public API with host operands: per step the
            H2D of every distinct A / B of the step and of C (pinned, overlapped with the cells
            already computing) and the D2H of C inside the timed region; per_call: the one-call
            mmmcu_multiply_host path (every operand copied per cell)
roofline  = K2 (dominant kernel) useful TFLOP/s vs the measured FP32 SIMT peak; plus the
            BASELINE roofline time fraction Σ max(flops/P_fp32, bytes/BW_hbm) / Σ (K1+K2)
cpu_baseline = the reference's CPU path (oracle/_ref: SPEC preprocess_a (ABlockIndex) /
            preprocess_b and the leaf-blocked multiply_parallel over the
            reference's compiled KernelTable) on a bounded row sample, all host cores
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ZS = (0.6, 0.7, 0.8, 0.9, 0.95)
BWS = (8, 16, 32)
T90 = 1.2815515655446004  # Φ^-1(0.90)
T95 = 1.6448536269514722  # Φ^-1(0.95)


# ---------------------------------------------------------------------------- workloads
def workload_cells(name):
    """Cells: (label, M, K, N, A spec, B spec).  spec = dict(value_kind, sigma, thresh, mask_kind, p, block)."""
    uni = dict(value_kind=0, sigma=1.0, thresh=0.0)
    if name == "sweep":
        cells = []
        for zA in ZS:
            for zB in ZS:
                for bw in BWS:
                    cells.append((f"zA{zA}_zB{zB}_bw{bw}", 4096, 4096, 4096,
                                  dict(uni, mask_kind=1, p=zA, block=1, key=("A", zA)),
                                  dict(uni, mask_kind=2, p=zB, block=bw, key=("B", zB, bw))))
        return cells
    if name == "cfg1":
        return [("cfg1", 1024, 1024, 1024, dict(uni, mask_kind=1, p=0.8, block=1, key=("A", 0.8)),
                 dict(uni, mask_kind=2, p=0.8, block=16, key=("B", 0.8, 16)))]
    if name == "cfg3":
        return [("cfg3", 2048, 16384, 4096, dict(value_kind=2, sigma=1.0, thresh=T90, mask_kind=0, p=0.0, block=1,
                                                 key=("A3",)),
                 dict(value_kind=1, sigma=0.02, thresh=0.0, mask_kind=2, p=0.9, block=32, key=("B3",)))]
    if name == "cfg4":
        return [("cfg4", 64, 12288, 49152, dict(value_kind=2, sigma=1.0, thresh=T95, mask_kind=0, p=0.0, block=1,
                                                key=("A4",)),
                 dict(value_kind=1, sigma=0.02, thresh=0.0, mask_kind=2, p=0.85, block=16, key=("B4",)))]
    if name == "cfg5":
        return [("cfg5", 32768, 8192, 8192, dict(uni, mask_kind=1, p=0.85, block=1, key=("A5",)),
                 dict(uni, mask_kind=2, p=0.85, block=16, key=("B5",)))]
    raise SystemExit(f"unknown workload {name}")


def seed_of(key, base=20240220):
    """Stable per-matrix seed (identical on every rank and in the reference arm)."""
    import hashlib

    d = hashlib.blake2b(f"{base}:{key!r}".encode(), digest_size=8).digest()
    return int.from_bytes(d, "little")


# ---------------------------------------------------------------------------- helpers
class ClockSampler:
    """SM clock and clock-event-reason sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []
        self.nvml = None

    @staticmethod
    def _power_mw(pynvml, h):
        # instantaneous board power (nvmlDeviceGetPowerUsage is a ~1 s average, useless for a
        # 0.1 s timed region); None when the field is not available
        try:
            fid = getattr(pynvml, "NVML_FI_DEV_POWER_INSTANT", 186)
            v = pynvml.nvmlDeviceGetFieldValues(h, [fid])[0]
            if v.nvmlReturn == 0:
                return float(v.value.uiVal)
        except Exception:  # noqa: BLE001
            pass
        return None

    def start(self):
        # NVML in a thread (5 ms period; the timed region of a sweep step is ~0.2 s, too short
        # for nvidia-smi's start-up); nvidia-smi -lms as the fallback
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.nvml = (pynvml, h)
            self.samples, self.run = [], True

            def loop():
                while self.run:
                    try:
                        self.samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                                             pynvml.nvmlDeviceGetCurrentClocksEventReasons(h),
                                             self._power_mw(pynvml, h)))
                    except Exception:  # noqa: BLE001
                        pass
                    time.sleep(0.005)

            self.t = threading.Thread(target=loop, daemon=True)
            self.t.start()
            while not self.samples:  # sampling is live before the timed region starts
                time.sleep(0.001)
            self.samples.clear()
            return
        except Exception:  # noqa: BLE001
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
                 "--format=csv,noheader,nounits", "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nvml is not None:
            self.run = False
            self.t.join(timeout=1)
            pynvml, h = self.nvml
            try:
                mx = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            except Exception:  # noqa: BLE001
                mx = None
            sm = [float(c) for c, _, _ in self.samples]
            reasons = {name for _, bits, _ in self.samples for bit, name in self.REASONS.items()
                       if bits & bit and name != "gpu_idle"}
            # board power beside the clocks: K2-TC runs at the power limit, which is what holds the
            # SM clock below its maximum (the reason bit is not set in every 5 ms sample)
            pw = [float(p) / 1e3 for _, _, p in self.samples if p is not None]
            try:
                lim = float(pynvml.nvmlDeviceGetEnforcedPowerLimit(h)) / 1e3
            except Exception:  # noqa: BLE001
                lim = None
            return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                    "samples": len(sm), "source": "nvml", "power_w": round(float(np.median(pw)), 1) if pw else None,
                    "power_w_max": round(max(pw), 1) if pw else None, "power_limit_w": lim,
                    "power_source": "NVML_FI_DEV_POWER_INSTANT" if pw else None}
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.06)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=1)
        sm, mx, reasons = [], None, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 3:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
                bits = int(parts[2], 16)
            except ValueError:
                continue
            for bit, name in self.REASONS.items():
                if bits & bit and name != "gpu_idle":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    hbm, src = 6650.0, "fallback (B200_PROFILING.md)"
    if os.path.exists(path):
        try:
            hbm = float(json.load(open(path))["hbm_gbs"])
            src = "measured (MEASURED_PEAKS.json)"
        except (KeyError, ValueError):
            pass
    return hbm, src


def measured_bf16():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return float(json.load(open(path))["bf16_tflops"])
    except (OSError, KeyError, ValueError):
        return None


def probe_fp32_peak(device):
    import ctypes

    so = os.path.join(ROOT, "tools", "_lib", "libfp32probe.so")
    if not os.path.exists(so):
        return 74.45, "analytic (148 SM x 128 x 2 x 1.965 GHz; probe not built)"
    lib = ctypes.CDLL(so)
    lib.probe_fp32_tflops.restype = ctypes.c_double
    lib.probe_fp32_tflops.argtypes = [ctypes.c_int, ctypes.c_int]
    v = lib.probe_fp32_tflops(device, 20000)
    if v <= 0:
        return 74.45, "analytic (probe failed)"
    return v, "measured live (tools/probe/fp32_probe.cu: FFMA chains, 8x256 threads/SM)"


# ----------------------------------------------------------------------------- setup
def shard_cells(cells, rank, world):
    """Strong scaling: every cell's A/C rows are partitioned across the
    ranks with mmmcu_shard_rows; rank r gets rows [r0, r1) of the SAME job.  Returns cells
    with per-rank M plus each cell's first global row."""
    import paper_2402_14118_b200 as mmm

    out = []
    for (label, M, K, N, sa, sb) in cells:
        r0, r1 = mmm.shard_rows(M, world, rank)
        out.append((label, r1 - r0, K, N, dict(sa, row0=r0), sb))
    return out


def make_inputs(cells, ctx, rank, world, torch, dist, device):
    """Generate this rank's A rows locally (row-offset generator: the rows of the full matrix)
    and B on rank 0, broadcast once with NCCL.  Returns dicts of tensors."""
    import paper_2402_14118_b200 as mmm

    As, Bs = {}, {}
    bcast_ms = 0.0
    for (_, M, K, N, sa, sb) in cells:
        ka = sa["key"]
        if ka not in As:
            lda = mmm.round_up(K, 64)
            t = torch.empty((max(M, 1), lda), dtype=torch.float32, device=device)
            mmm.generate(t, seed=seed_of(ka), value_kind=sa["value_kind"], sigma=sa["sigma"], thresh=sa["thresh"],
                         mask_kind=sa["mask_kind"], p=sa["p"], block=sa["block"], cols=K, row0=sa.get("row0", 0),
                         ctx=ctx)
            As[ka] = t[:M, :K]
        kb = sb["key"]
        if kb not in Bs:
            ldb = mmm.round_up(N, 64)
            t = torch.empty((K, ldb), dtype=torch.float32, device=device)
            if rank == 0:
                mmm.generate(t, seed=seed_of(kb), value_kind=sb["value_kind"], sigma=sb["sigma"], thresh=sb["thresh"],
                             mask_kind=sb["mask_kind"], p=sb["p"], block=sb["block"], cols=N, ctx=ctx)
            Bs[kb] = t
    if world > 1:
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for kb in sorted(Bs, key=str):
            dist.broadcast(Bs[kb], src=0)  # NCCL over NVLink: B is broadcast once
        e1.record()
        torch.cuda.synchronize()
        bcast_ms = e0.elapsed_time(e1)
    for kb in list(Bs):
        N = [c[3] for c in cells if c[5]["key"] == kb][0]
        Bs[kb] = Bs[kb][:, :N]
    torch.cuda.synchronize()
    return As, Bs, bcast_ms


TC_TM, TC_TN = 128, 192  # K2-TC C tile (k2_tc.cuh)


def tc_executed_flops(M, b, torch):
    """Tensor-core flops K2-TC executes on a cell (fp16 split, AUTO's TC path): per 192-column
    tile, ceil(live k / 16) MMA steps of 3 fp16 MMAs (hi/lo split) of 128 x 192 x 16, for every
    128-row tile."""
    K, N = b.shape
    nt = (N + TC_TN - 1) // TC_TN
    nz = torch.zeros((K, nt * TC_TN), dtype=torch.bool, device=b.device)
    nz[:, :N] = b != 0
    live = nz.view(K, nt, TC_TN).any(dim=2).sum(dim=0)  # live k per tile
    steps = int(((live + 15) // 16).sum().item())
    return steps * ((M + TC_TM - 1) // TC_TM) * 3 * 2 * TC_TM * TC_TN * 16


def cell_stats(cells, As, Bs, ctx, torch):
    """Per cell: useful flops (2*lane_fma_ops), algorithmic bytes, counters, the K2 path AUTO
    takes and, for K2-TC, the tensor-core flops it executes (setup, untimed)."""
    stats = []
    for (label, M, K, N, sa, sb) in cells:
        a, b = As[sa["key"]], Bs[sb["key"]]
        ctx.preprocess(a, b)
        cnt = ctx.planned_counters()
        c = torch.zeros((M, N), dtype=torch.float32, device=a.device)
        ctx.multiply(c, a, b, want_counters=False)
        path = {5: "k2_tc", 3: "k2_simt2<8>", 4: "k2_simt2<16>"}.get(ctx.last_algo(), str(ctx.last_algo()))
        k_live = int((a != 0).any(dim=0).sum().item())
        algo_bytes = 4 * (M * K + k_live * N + M * N)
        stats.append(dict(label=label, flops=2 * cnt.lane_fma_ops, bytes=algo_bytes, k_live=k_live,
                          lane_fma_ops=cnt.lane_fma_ops, M=M, K=K, N=N, path=path,
                          tc_flops=tc_executed_flops(M, b, torch) if path == "k2_tc" else 0))
        del c
    return stats


def run_step(cells, As, Bs, Cs, ctx, torch, events=None):
    for t, (label, M, K, N, sa, sb) in enumerate(cells):
        a, b = As[sa["key"]], Bs[sb["key"]]
        c = Cs[(M, N)]
        if events is not None:
            events[t][0].record()
        ctx.preprocess(a, b)
        if events is not None:
            events[t][1].record()
        ctx.multiply(c, a, b, want_counters=False)
        if events is not None:
            events[t][2].record()


class CellStreams:
    """The step's cells dealt round-robin to S contexts, each on its own CUDA stream (the
    package's MmmStreams): cells are independent jobs, so the HBM-bound K1 chain of one cell
    runs on the SMs K2-TC leaves free (it takes the fewest CTA pairs that keep its number of
    rounds) and in the tail round of another cell's tensor-bound K2 (measured on the sweep:
    22.9 -> 21.5 ms/step with 2 streams).  Every stream owns its plans (context) and its C."""

    def __init__(self, n, cells, device, torch):
        import paper_2402_14118_b200 as mmm

        self.n = n
        self.pool = mmm.MmmStreams(n, device.index or 0)
        self.Cs = []
        for _ in range(n):
            cs = {}
            for (_, M, K, N, sa, sb) in cells:
                if (M, N) not in cs:
                    cs[(M, N)] = torch.zeros((M, mmm.round_up(N, 64)), dtype=torch.float32, device=device)[:, :N]
            self.Cs.append(cs)

    def fork(self):
        self.pool.fork()

    def join(self):
        self.pool.join()

    def step(self, cells, As, Bs):
        for t, (label, M, K, N, sa, sb) in enumerate(cells):
            s = t % self.n
            self.pool.submit(self.Cs[s][(M, N)], As[sa["key"]], Bs[sb["key"]], stream=s)


def quick_measure(workload, ctx, torch, device, steps, warmup):
    """Device-timed value of another workload on this GPU (the N=1 reference point of the
    multi-GPU configs[4] run): same step definition, CUDA events, inputs freed afterwards."""
    cells = workload_cells(workload)
    As, Bs, _ = make_inputs(cells, ctx, 0, 1, torch, None, device)
    Cs = {}
    for (_, M, K, N, sa, sb) in cells:
        if (M, N) not in Cs:
            import paper_2402_14118_b200 as mmm

            Cs[(M, N)] = torch.zeros((M, mmm.round_up(N, 64)), dtype=torch.float32, device=device)[:, :N]
    stats = cell_stats(cells, As, Bs, ctx, torch)
    for _ in range(warmup):
        run_step(cells, As, Bs, Cs, ctx, torch)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        run_step(cells, As, Bs, Cs, ctx, torch)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    flops = float(sum(x["flops"] for x in stats))
    del As, Bs, Cs
    torch.cuda.empty_cache()
    return {"workload": workload, "value": round(flops / (ms * 1e-3) / 1e9, 2), "unit": "GFLOP/s",
            "ms_per_step": round(ms, 4), "steps": steps, "warmup": warmup,
            "paths": sorted({x["path"] for x in stats})}


def count_launches(cells):
    # per cell (AUTO): K1 = k1_pass (A and B tiles) + k1_fin (plan totals, range guard, path
    # choice, CSR tile prefix) + k1_pack_auto (the chosen B pack and A's CSR in one persistent
    # launch); K2 = k2_simt2_any + k2_tc (gated on the device: one runs, the other exits at
    # entry).  (profiles/r02_launches_summary.txt: 375 kernel launches per 75-cell step.)
    return 5 * len(cells)


# ---------------------------------------------------------------------------- CPU leg
def ref_build():
    from oracle import oracle as orc  # cpu_baseline leg only

    v4 = orc.ref_so_path().endswith("_v4.so")
    return "-O3 -fopenmp " + ("-march=x86-64-v4: AVX-512 host" if v4 else "-march=x86-64-v3: AVX2 host")


def ref_engines(orc):
    """The two reference-kind CPU engines (oracle/_ref/ref_driver.cpp): the SPEC multiply with
    the ABlockIndex-driven A traversal, and with the Fig. 4 per-element A branch (SPEC.md:304
    keeps both)."""
    return {"ablock_index": orc.ref_multiply_mmm, "fig4_branch": orc.ref_multiply_parallel}


def pick_ref_engine(orc, A, B, threads, rows=64):
    """The faster engine on a calibration sample (the baseline is the reference path at its
    best on this host): returns (name, fn, rate flop/s)."""
    best = None
    for name, fn in ref_engines(orc).items():
        C = np.zeros((rows, B.shape[1]), np.float32)
        fn(C, np.ascontiguousarray(A[:rows]), B, workers=threads)  # warm
        C[:] = 0
        cnt = fn(C, np.ascontiguousarray(A[:rows]), B, workers=threads)
        rate = 2 * cnt["lane_fma_ops"] / max(cnt["multiply_ns"], 1) * 1e9
        if best is None or rate > best[2]:
            best = (name, fn, rate)
    return best


def cpu_reference_sample(cells, host_A, host_B, budget_s, threads, stats):
    """The reference CPU path on a bounded row sample of every cell (oracle/_ref).

    Per cell: rows [0, r) with r sized so the whole sample takes ~budget_s; preprocessing of
    B (done once per B by the reference path) is amortised in proportion to the rows run.
    The engine is the faster of the two reference-kind engines on the middle cell."""
    from oracle import oracle as orc  # cpu_baseline leg only

    orc.ref_lib()
    # calibrate on the middle cell
    mid = len(cells) // 2
    lab, M, K, N, sa, sb = cells[mid]
    t0 = time.perf_counter()
    engine, fn, rate = pick_ref_engine(orc, host_A[sa["key"]], host_B[sb["key"]], threads)
    per_cell_s = budget_s / len(cells)
    flops_total, time_total, rows_total = 0.0, 0.0, 0
    for i, (lab, M, K, N, sa, sb) in enumerate(cells):
        A = host_A[sa["key"]]
        B = host_B[sb["key"]]
        flops_per_row = stats[i]["flops"] / M
        rows = int(min(M, max(8, per_cell_s * rate / max(flops_per_row, 1.0))))
        C = np.zeros((rows, B.shape[1]), np.float32)
        cnt = fn(C, np.ascontiguousarray(A[:rows]), B, workers=threads)
        flops_total += 2 * cnt["lane_fma_ops"]
        time_total += (cnt["multiply_ns"] + cnt["preprocess_ns"] * rows / M) * 1e-9
        rows_total += rows
    return flops_total / time_total / 1e9, rows_total, time.perf_counter() - t0, engine


def host_copies(cells, As, Bs):
    host_A = {k: v.cpu().numpy() for k, v in As.items()}
    host_B = {k: np.ascontiguousarray(v.cpu().numpy()) for k, v in Bs.items()}
    # A views carry the padded leading dimension: keep the logical K columns contiguous
    host_A = {k: np.ascontiguousarray(v) for k, v in host_A.items()}
    return host_A, host_B


# -------------------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="",
                    help="sweep (configs[1]; the N=1 default) | cfg1 | cfg3 | cfg4 | cfg5 (the N>1 default: "
                         "strong scaling, one 32768-row A partitioned across the ranks)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-per-call", action="store_true", help="e2e: skip the per-call mmmcu_multiply_host number")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of CPU work for cpu_baseline")
    ap.add_argument("--e2e-steps", type=int, default=0, help="0 = same as --steps")
    ap.add_argument("--per-cell", default="", help="write per-cell timings (JSON) to this path")
    ap.add_argument("--no-cfg5-ref", action="store_true", help="N=1: skip the 1-GPU configs[4] reference line")
    ap.add_argument("--streams", type=int, default=0,
                    help="contexts / CUDA streams the step's cells are dealt to (0 = 2 for multi-cell workloads, else 1)")
    args = ap.parse_args()
    warmup = max(args.warmup, 3)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch under torchrun (the driver may also launch us that way)
        import socket

        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        raise SystemExit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world} (launch one rank per GPU)")
    if not args.workload:
        args.workload = "sweep" if world == 1 else "cfg5"
    cells = workload_cells(args.workload)
    strong = world > 1
    if strong:
        cells = shard_cells(cells, rank, world)
    metric = "useful GFLOP/s of masked fp32 matmul (60-95% zeros)"
    cfg = {"workload": {"sweep": "configs[1]: 4096^3 fp32 sparsity sweep, zA x zB in {.6,.7,.8,.9,.95}^2 x "
                                  "B block width {8,16,32} (75 cells), uniform[-1,1], i.i.d. Bernoulli masks",
                        "cfg1": "configs[0]: 1024^3, zA=zB=0.8, bw 16",
                        "cfg3": "configs[2]: MLP down-projection 2048x16384x4096, A=ReLU(G-t) 90% zeros, "
                                "B~N(0,0.02) 32-wide blocks kept p=0.1",
                        "cfg4": "configs[3]: skinny decode 64x12288x49152, A ReLU 95% zeros, B 16-wide blocks kept 0.15",
                        "cfg5": "configs[4]: 32768x8192x8192 per GPU, 0.85/0.85, bw 16"}[args.workload],
           "cells": len(cells), "rows_per_gpu": cells[0][1],
           "shard": ("A/C rows partitioned across the ranks (mmmcu_shard_rows, strong scaling: the same job at "
                     "every N), B generated on rank 0 and NCCL-broadcast once before timing (broadcast_ms)")
           if strong else "one GPU, whole job",
           "step": "K1 (preprocess_a + preprocess_b: masks, index lists, codes, B operand pack) + K2 (C += A*B) "
                   "for every cell",
           "l2": "inputs larger than L2 per cell (A+B+C >= 126 MB for the sweep; A is shared by the 15 cells of "
                 "one zA, B by the 5 cells of one (zB, bw), each cell is one preprocess + multiply)",
           "streams": "the step's cells are dealt round-robin to 2 contexts on 2 CUDA streams (--streams; independent "
                    "cells overlap one cell's HBM-bound K1 with another's tensor-bound K2); 1 = one stream",
           "global_batch": sum(c[1] for c in cells) // max(len(cells), 1) * world if not strong
           else workload_cells(args.workload)[0][1],
           "parallelism": f"dp{world} (A/C row shards)"}

    if args.impl == "reference":
        return run_reference_arm(args, cells, cfg, metric, world, rank, warmup)

    import torch
    import torch.distributed as dist

    import paper_2402_14118_b200 as mmm

    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)
    ctx = mmm.MmmContext(local)
    As, Bs, bcast_ms = make_inputs(cells, ctx, rank, world, torch, dist, device)
    Cs = {}
    for (_, M, K, N, sa, sb) in cells:
        if (M, N) not in Cs:
            Cs[(M, N)] = torch.zeros((M, mmm.round_up(N, 64)), dtype=torch.float32, device=device)[:, :N]
    stats = cell_stats(cells, As, Bs, ctx, torch)
    fp32_peak, fp32_src = probe_fp32_peak(local)
    hbm_peak, hbm_src = measured_peaks()

    # ---- device-timed steps: the step's cells on `streams` contexts / streams (CellStreams)
    nl = args.streams if args.streams > 0 else (2 if len(cells) >= 2 else 1)
    nl = max(1, min(nl, len(cells)))
    cstreams = CellStreams(nl, cells, device, torch)
    cfg["streams_used"] = nl
    main = torch.cuda.current_stream(device)
    cstreams.fork()
    for _ in range(warmup):
        cstreams.step(cells, As, Bs)
    cstreams.join()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record(main)
    cstreams.fork()
    for k in range(args.steps):
        cstreams.step(cells, As, Bs)
    cstreams.join()
    s1.record(main)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    total_ms = s0.elapsed_time(s1)
    # ---- per-cell K1 / K2 times (diagnostic pass, one stream, after the timed region: the
    # per-kernel breakdown, the K2 path table and roofline.tensor come from here)
    dsteps = max(1, min(args.steps, 3))
    ev = [[[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in cells] for _ in range(dsteps)]
    run_step(cells, As, Bs, Cs, ctx, torch)
    for k in range(dsteps):
        run_step(cells, As, Bs, Cs, ctx, torch, events=ev[k])
    torch.cuda.synchronize()
    # the same step with WorkCounters returned by every multiply (the C++ drop-in's default:
    # k1_counters + a stream synchronisation per cell), one stream, device events
    cw0, cw1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cw0.record()
    for (label, M, K, N, sa, sb) in cells:
        a_, b_ = As[sa["key"]], Bs[sb["key"]]
        ctx.preprocess(a_, b_)
        ctx.multiply(Cs[(M, N)], a_, b_, want_counters=True)
    cw1.record()
    torch.cuda.synchronize()
    counters_ms = cw0.elapsed_time(cw1)
    k1_ms = np.zeros(len(cells))
    k2_ms = np.zeros(len(cells))
    for k in range(dsteps):
        for t in range(len(cells)):
            k1_ms[t] += ev[k][t][0].elapsed_time(ev[k][t][1]) / dsteps
            k2_ms[t] += ev[k][t][1].elapsed_time(ev[k][t][2]) / dsteps
    flops_rank = float(sum(s["flops"] for s in stats))
    step_ms_local = total_ms / args.steps  # this rank's step (the roofline below is rank-local)
    if world > 1:
        tt = torch.tensor([total_ms, flops_rank], dtype=torch.float64, device=device)
        mx = tt.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(tt, op=dist.ReduceOp.SUM)
        total_ms, flops_all = float(mx[0]), float(tt[1])
    else:
        flops_all = flops_rank
    ms_per_step = total_ms / args.steps
    value = flops_all / (ms_per_step * 1e-3) / 1e9

    # ---- roofline (rank-local; K2 is the dominant kernel)
    k2_flops = sum(s["flops"] for s in stats)
    k2_time = float(k2_ms.sum()) * 1e-3
    achieved_tf = k2_flops / k2_time / 1e12
    paths = {}
    for i, s_ in enumerate(stats):
        paths.setdefault(s_["path"], [0, 0.0])
        paths[s_["path"]][0] += 1
        paths[s_["path"]][1] += float(k2_ms[i])
    dominant = max(paths, key=lambda p: paths[p][1])
    tc_ms = sum(float(k2_ms[i]) for i, s_ in enumerate(stats) if s_["path"] == "k2_tc")
    tc_exec = sum(s_["tc_flops"] for s_ in stats)
    bf16 = measured_bf16()
    tensor = None
    if tc_ms > 0:
        tensor = {"kernel": "k2_tc", "executed_tflops": round(tc_exec / (tc_ms * 1e-3) / 1e12, 1),
                  "peak_tflops": round(bf16, 1) if bf16 else None,
                  "peak_source": "fp16 dense = measured bf16 (MEASURED_PEAKS.json, same kind::f16 rate)" if bf16 else None,
                  "frac": round(tc_exec / (tc_ms * 1e-3) / 1e12 / bf16, 4) if bf16 else None,
                  "def": "fp16-split MMAs the kernel issues (3 per live-k step of 16 per 128x192 tile) / K2-TC time"}
    t_roof = sum(max(s["flops"] / (fp32_peak * 1e12), s["bytes"] / (hbm_peak * 1e9)) for s in stats)
    t_meas = step_ms_local * 1e-3  # the timed step (cells overlapped across the streams)
    t_serial = float((k1_ms + k2_ms).sum()) * 1e-3  # the same cells one after the other on one stream
    hbm_bytes = sum(s["bytes"] for s in stats)
    useful = {"achieved": round(achieved_tf, 3), "peak": round(fp32_peak, 2), "unit": "TFLOP/s",
              "frac": round(achieved_tf / fp32_peak, 4), "peak_source": fp32_src,
              "def": "BASELINE useful FLOPs (2 x surviving products) / K2 device time, against the FP32 SIMT peak"}
    traffic, traffic_src = None, None
    try:  # dram__bytes_read.sum + dram__bytes_write.sum per launch, from the committed ncu capture
        tr = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")))
        if dominant in tr:
            traffic, traffic_src = tr[dominant]["bytes_per_launch"], tr[dominant]["source"]
    except (OSError, ValueError, KeyError):
        pass
    common = {"kernel": dominant, "traffic": traffic, "traffic_source": traffic_src,
              "paths": {p: {"cells": v[0], "k2_ms": round(v[1], 4)} for p, v in paths.items()},
              "useful": useful, "time_frac": round(t_roof / t_meas, 4),
              "time_frac_def": "BASELINE: Σ_cells max(useful_flops/P_fp32, algo_bytes/BW_hbm) / device time of the timed step",
              "streams": nl, "serial_ms_per_step": round(t_serial * 1e3, 4),
              "serial_with_counters_ms_per_step": round(counters_ms, 4),
              "serial_def": "K1 + K2 of every cell on ONE stream with CUDA events per cell (diagnostic pass after the "
                            "timed region); k1_ms_per_step, k2_ms_per_step, paths and tensor come from it",
              "hbm_peak_gbs": hbm_peak, "hbm_peak_source": hbm_src,
              "hbm_achieved_gbs": round(hbm_bytes / t_meas / 1e9, 1),
              "k1_ms_per_step": round(float(k1_ms.sum()), 4), "k2_ms_per_step": round(float(k2_ms.sum()), 4)}
    # SURVEY.md §8(d) roofline: per cell T_roof = max(useful flops / P_fp32, algorithmic bytes /
    # BW_hbm); achieved = useful TFLOP/s over the device time of the step (K1 + K2), peak = the
    # rate the roofline allows for the same cells (flops / Σ T_roof), so frac = Σ T_roof / Σ T.
    # The tensor-pipe view of K2-TC (executed fp16-split MMAs vs the bf16 peak) is kept as
    # roofline.tensor, the K2-only useful rate as roofline.useful.
    total_flops = float(sum(x["flops"] for x in stats))
    roofline = {"bound": "fp32+hbm", "achieved": round(total_flops / t_meas / 1e12, 3),
                "peak": round(total_flops / t_roof / 1e12, 3), "unit": "TFLOP/s",
                "frac": round(t_roof / t_meas, 4),
                "def": "SURVEY.md §8(d): per cell max(2*lane_fma_ops / P_fp32, 4*(MK + K_live*N + MN) / BW_hbm); "
                       "achieved = useful FLOPs / device time of the timed step (K1 + K2 of every cell, CUDA events "
                       "around the step); peak = useful FLOPs / Σ roofline times",
                "peak_fp32_tflops": round(fp32_peak, 2), "peak_fp32_source": fp32_src, "tensor": tensor, **common}

    # ---- e2e through the host-buffer public API
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, cells, As, Bs, ctx, torch, dist, world, device, stats)

    # ---- CPU baseline (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            host_A, host_B = host_copies(cells, As, Bs)
            threads = os.cpu_count() or 1
            v, rows, wall, engine = cpu_reference_sample(cells, host_A, host_B, args.cpu_budget, threads, stats)
            from oracle import oracle as orc
            cpu = {"value": round(v, 3), "unit": "GFLOP/s", "cores": orc.ref_lib().ref_max_threads(),
                   "kind": "reference",
                   "sample": f"{rows} A rows spread over the {len(cells)} cells (each cell's leading rows), full B "
                             f"preprocessing amortised per row; {wall:.1f} s wall; oracle/_ref = the SPEC multiply_parallel "
                             f"(preprocess_a/b, then per non-zero a_ik the reference's compiled KernelTable over B row k) with "
                             f"the faster A traversal on this host ({engine}: ABlockIndex or the Fig. 4 branch), "
                             f"{ref_build()}"}
        except Exception as e:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "GFLOP/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {type(e).__name__}: {e}"}

    # ---- the 1-GPU point of the multi-GPU workload (configs[4]), so the N>1 lines of the
    # scaling run have a same-workload N=1 reference
    cfg5_1gpu = None
    if world == 1 and args.workload == "sweep" and not args.no_cfg5_ref:
        cfg5_1gpu = quick_measure("cfg5", ctx, torch, device, max(3, args.steps // 4), 3)

    if args.per_cell and rank == 0:
        json.dump([dict(s, k1_ms=float(k1_ms[i]), k2_ms=float(k2_ms[i])) for i, s in enumerate(stats)],
                  open(args.per_cell, "w"), indent=1)

    if rank == 0:
        line = {
            "metric": metric, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps,
            "warmup": warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded counter-hash generator, device side)",
            "config": cfg,
            "roofline": roofline,
            "e2e": e2e, "cpu_baseline": cpu, "clocks": clk, "gpu_launches": count_launches(cells) * args.steps,
            "broadcast_ms": round(bcast_ms, 3),
            **({"cfg5_1gpu": cfg5_1gpu} if cfg5_1gpu else {}),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(args, cells, As, Bs, ctx, torch, dist, world, device, stats):
    """The same metric end to end through the public Python API with HOST operands: every step
    copies each distinct A and B of the step (and C) from pinned host memory to the device
    (a copy stream, one event per operand, so the copies overlap the cells already computing),
    runs K1 + K2 of every cell (MmmContext.preprocess / multiply_mmm), and reads C back.
    Wall clock around whole steps.  A second number, per_call, times mmmcu_multiply_host (the
    one-call C ABI host path: H2D A, B, C + K1 + K2 + D2H C per cell, synchronous)."""
    import paper_2402_14118_b200 as mmm

    steps = args.e2e_steps or args.steps
    flops = float(sum(s["flops"] for s in stats))
    # Host-path cell order: the step needs each distinct A (5) and B (15) once.  Their copies are
    # queued interleaved (A0 B0 A1 B1 ... then the remaining B's) and the cells run in the order
    # their two operands have both arrived, so the computable cells grow as i*j with the first
    # copies and the later copies (one 64 MiB B per 5 cells) hide behind the compute (device
    # order: 41 ms per step, the first A's cells waiting for all 15 B's).  Same cells, same
    # bytes per step.
    a_keys = list(dict.fromkeys(c[4]["key"] for c in cells))
    b_keys = list(dict.fromkeys(c[5]["key"] for c in cells))
    pos = {}
    for i in range(max(len(a_keys), len(b_keys))):
        for ks in (a_keys, b_keys):
            if i < len(ks):
                pos[ks[i]] = len(pos)
    order = sorted(range(len(cells)), key=lambda i: (max(pos[cells[i][4]["key"]], pos[cells[i][5]["key"]]), i))
    cells = [cells[i] for i in order]

    def pinned_like(t):  # host copy of a device operand (its padded base layout), pinned
        base = t if t.is_contiguous() else t.as_strided((t.shape[0], t.stride(0)), (t.stride(0), 1))
        return base.cpu().pin_memory()

    # Two sets of device operand buffers (step parity): the H2D copies of step i+1 run while
    # step i computes, so a step costs max(copies, compute) instead of copies + the last cells.
    NB = 2
    host, dev, host_out = {}, [dict() for _ in range(NB)], [dict() for _ in range(NB)]
    for (_, M, K, N, sa, sb) in cells:
        for key, t in ((sa["key"], As[sa["key"]]), (sb["key"], Bs[sb["key"]])):
            if key not in host:
                host[key] = pinned_like(t)
                for d in dev:
                    d[key] = torch.empty_like(host[key], device=device)
        if ("C", M, N) not in host:
            host[("C", M, N)] = torch.zeros((M, mmm.round_up(N, 64)), dtype=torch.float32).pin_memory()
            for d, ho in zip(dev, host_out):
                d[("C", M, N)] = torch.empty_like(host[("C", M, N)], device=device)
                ho[("C", M, N)] = torch.empty_like(host[("C", M, N)]).pin_memory()
    h2d = int(sum(v.numel() * 4 for v in host.values()))
    d2h = int(sum(v.numel() * 4 for k, v in host.items() if k[0] == "C"))
    copy_stream = torch.cuda.Stream(device)
    main = torch.cuda.current_stream(device)
    done = [None] * NB  # per buffer set: the event after the D2H of the last step that used it

    def step(i):
        s = i % NB
        d = dev[s]
        if done[s] is not None:
            done[s].synchronize()  # host: at most NB steps in flight (and host_out[s] was read back)
        ready = {}
        with torch.cuda.stream(copy_stream):  # H2D in first-use order, one event per operand
            for (_, M, K, N, sa, sb) in cells:
                for key in (("C", M, N), sa["key"], sb["key"]):
                    if key not in ready:
                        d[key].copy_(host[key], non_blocking=True)
                        ev = torch.cuda.Event()
                        ev.record(copy_stream)
                        ready[key] = ev
        for (_, M, K, N, sa, sb) in cells:
            for key in (("C", M, N), sa["key"], sb["key"]):
                main.wait_event(ready[key])
            a, b = d[sa["key"]][:M, :K], d[sb["key"]][:K, :N]
            ctx.preprocess(a, b)
            ctx.multiply(d[("C", M, N)][:M, :N], a, b, want_counters=False)
        for k in host:
            if k[0] == "C":
                host_out[s][k].copy_(d[k], non_blocking=True)  # D2H of the step's result
        ev = torch.cuda.Event()
        ev.record(main)
        done[s] = ev

    step(0)  # warm-up
    torch.cuda.synchronize(device)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for i in range(steps):
        step(i)
    torch.cuda.synchronize(device)
    el = time.perf_counter() - t0
    fl = flops
    if world > 1:
        tt = torch.tensor([el, flops], dtype=torch.float64, device=device)
        mx = tt.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(tt, op=dist.ReduceOp.SUM)
        el, fl = float(mx[0]), float(tt[1])
    out = {"value": round(fl / (el / steps) / 1e9, 2), "unit": "GFLOP/s", "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": d2h, "steps": steps,
           "path": "public Python API with host operands: per step, H2D of each distinct A and B of the step and of "
                   "C (pinned, copy stream; two sets of device buffers, so the copies of step i+1 overlap the cells of "
                   "step i), preprocess + multiply_mmm of every cell, D2H of C; wall clock over all steps, device idle "
                   "at both ends"}
    # the one-call host path of the C ABI (mmmcu_multiply_host), every operand copied per cell
    if world == 1 and not args.no_per_call:
        host_A = {k: host[k].numpy() for k in As}
        host_B = {k: host[k].numpy() for k in Bs}
        hc = {k: host[k][:, : k[2]].numpy() for k in host if k[0] == "C"}
        del dev[1:]

        def step_call():
            for (_, M, K, N, sa, sb) in cells:
                mmm.multiply_host(hc[("C", M, N)], host_A[sa["key"]][:, :K], host_B[sb["key"]][:, :N], ctx=ctx)

        step_call()
        t0 = time.perf_counter()
        n_call = max(1, min(steps, 2))
        for _ in range(n_call):
            step_call()
        el2 = time.perf_counter() - t0
        out["per_call"] = {"value": round(flops / (el2 / n_call) / 1e9, 2), "unit": "GFLOP/s", "steps": n_call,
                           "h2d_bytes_per_step": int(sum(host_A[c[4]["key"]][:, :c[2]].nbytes + host_B[c[5]["key"]].nbytes
                                                         + hc[("C", c[1], c[3])].nbytes for c in cells)),
                           "d2h_bytes_per_step": int(sum(hc[("C", c[1], c[3])].nbytes for c in cells)),
                           "path": "mmmcu_multiply_host per cell (H2D A, B, C, K1, K2, D2H C, synchronous)"}
    return out


def run_reference_arm(args, cells, cfg, metric, world, rank, warmup):
    """--impl reference: the reference's own CPU path (oracle/_ref) on this box's host cores."""
    if rank != 0:
        return
    from oracle import oracle as orc  # reference arm: the reference CPU path

    if not orc.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libmmmref.so was not built "
                                                              "(needs /root/reference at build time)"}))
        return
    threads = os.cpu_count() or 1
    # inputs: the same cells, generated on the host by the oracle generator (same formulas,
    # bit-identical to the device generator for these modes), only the sampled rows of A
    budget = max(2.0, min(args.cpu_budget, 120.0 / max(args.steps + warmup, 1)))
    vals = []
    host_B = {}
    rows_used = 0
    # the faster of the two reference-kind engines on the middle cell (pick_ref_engine)
    lab, M, K, N, sa, sb = cells[len(cells) // 2]
    Bm = orc.gen_iid(K, N, seed_of(sb["key"]), value_kind=sb["value_kind"], sigma=sb["sigma"], thresh=sb["thresh"],
                     mask_kind=sb["mask_kind"], p=sb["p"], block=sb["block"], ld=(N + 63) // 64 * 64)
    Am = orc.gen_iid(64, K, seed_of(sa["key"]), value_kind=sa["value_kind"], sigma=sa["sigma"], thresh=sa["thresh"],
                     mask_kind=sa["mask_kind"], p=sa["p"], block=sa["block"])
    engine, ref_fn, _ = pick_ref_engine(orc, Am, Bm, threads)
    for k in range(warmup + args.steps):
        flops_total, time_total = 0.0, 0.0
        rows_used = 0
        for i, (lab, M, K, N, sa, sb) in enumerate(cells):
            if sb["key"] not in host_B:
                host_B[sb["key"]] = orc.gen_iid(K, N, seed_of(sb["key"]), value_kind=sb["value_kind"],
                                                sigma=sb["sigma"], thresh=sb["thresh"], mask_kind=sb["mask_kind"],
                                                p=sb["p"], block=sb["block"], ld=(N + 63) // 64 * 64)
            rows = max(8, int(budget / len(cells) * 2e9 / max(2 * K * N * (1 - sa["p"]) * (1 - sb["p"]), 1)))
            rows = min(rows, M)
            A = orc.gen_iid(rows, K, seed_of(sa["key"]), value_kind=sa["value_kind"], sigma=sa["sigma"],
                            thresh=sa["thresh"], mask_kind=sa["mask_kind"], p=sa["p"], block=sa["block"])
            C = np.zeros((rows, host_B[sb["key"]].shape[1]), np.float32)
            cnt = ref_fn(C, A, host_B[sb["key"]], workers=threads)
            flops_total += 2 * cnt["lane_fma_ops"]
            time_total += (cnt["multiply_ns"] + cnt["preprocess_ns"] * rows / M) * 1e-9
            rows_used += rows
        if k >= warmup:
            vals.append(flops_total / time_total / 1e9)
    v = float(np.median(vals))
    line = {"impl": "reference", "metric": metric, "value": round(v, 3), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": warmup, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (seeded counter-hash generator, host side)", "config": cfg,
            "cpu_baseline": {"value": round(v, 3), "unit": "GFLOP/s", "cores": orc.ref_lib().ref_max_threads(),
                             "kind": "reference",
                             "sample": f"per step {rows_used} A rows over {len(cells)} cells (full B preprocessing "
                                       f"amortised per row); the SPEC multiply_parallel over the reference's compiled "
                                       f"KernelTable with the faster A traversal on this host ({engine}), "
                                       f"{ref_build()}; median of {args.steps} steps"},
            "e2e": {"value": round(v, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
