"""The SPEC bench-cli on the GPU path (paper_2402_14118_b200/_lib/mmm-cuda; SPEC.md bench-cli:
subcommands gen / bench / sweep / verify / analyze, the BenchRecord CSV header, exit codes 0 ok,
1 verification failure, 2 usage error, 3 I/O error).  Usage errors are caught before any device
work, so they are checked on CPU; the rest runs on the B200 through the C ABI."""
import csv
import os
import subprocess

import numpy as np
import pytest

from paper_2402_14118_b200 import _native as N

EXE = os.path.join(os.path.dirname(N.LIB_PATH), "mmm-cuda")
HEADER = ("algo,n,a_sparsity,b_sparsity,structure_b,dtype,workers,trial,preprocess_ns,multiply_ns,total_ns,"
          "kernel_invocations,lane_fma_ops,rows_skipped,regions_skipped,checksum").split(",")


def run(*args, timeout=300):
    if not os.path.exists(EXE):
        pytest.skip("mmm-cuda not built")
    return subprocess.run([EXE, *args], capture_output=True, text=True, timeout=timeout)


def test_usage_errors_exit_2():
    assert run().returncode == 2
    assert run("--help").returncode == 0
    assert run("frobnicate").returncode == 2
    assert run("bench", "--n").returncode == 2          # flag without a value
    assert run("gen", "--rows", "x").returncode == 2    # not an integer


@pytest.mark.gpu
def test_gen_analyze_bench_verify(tmp_path):
    a, b = str(tmp_path / "a.mmmb"), str(tmp_path / "b.mmmb")
    r = run("gen", "--rows", "1024", "--cols", "1024", "--structure", "random", "--sparsity", "0.8", "--seed", "7",
            "--out", a)
    assert r.returncode == 0, r.stderr
    assert abs(float(r.stdout.split("measured sparsity")[1]) - 0.8) < 0.01  # SPEC cmd_gen example
    r = run("gen", "--rows", "1024", "--cols", "1024", "--structure", "block_random", "--sparsity", "0.8",
            "--block-len", "16", "--seed", "8", "--out", b)
    assert r.returncode == 0, r.stderr
    r2 = run("gen", "--rows", "1024", "--cols", "1024", "--structure", "block_random", "--sparsity", "0.8",
             "--block-len", "16", "--seed", "8", "--out", str(tmp_path / "b2.mmmb"))
    assert open(b, "rb").read() == open(str(tmp_path / "b2.mmmb"), "rb").read()  # determinism
    r = run("analyze", "--matrix", b)
    assert r.returncode == 0, r.stderr
    z16 = float([ln for ln in r.stdout.splitlines() if "fraction 16" in ln][0].split()[-1])
    assert abs(z16 - 0.8) < 0.02  # 16-wide blocks zeroed with p = 0.8
    out = str(tmp_path / "bench.csv")
    r = run("bench", "--a", a, "--b", b, "--algo", "all", "--trials", "3", "--out", out)
    assert r.returncode == 0, r.stderr
    rows = list(csv.reader(open(out)))
    assert rows[0] == HEADER
    recs = rows[1:]
    algos = {x[0] for x in recs}
    assert algos == {"mmm", "mmm_exact", "mmm_tc", "mmm_tc32", "dense", "cublas"}
    med = {x[0]: x for x in recs if x[7] == "median"}
    assert len(med) == 6
    # the exact path and multiply_simple give the oracle's bits: equal checksums
    assert med["mmm_exact"][15] == med["dense"][15]
    # exact counters are identical across the masked variants
    assert len({med[k][12] for k in ("mmm", "mmm_exact", "mmm_tc", "mmm_tc32")}) == 1
    for x in recs:
        assert float(x[10]) >= float(x[9])  # total_ns >= multiply_ns
    r = run("verify", "--a", a, "--b", b)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "mmm_exact  max rel error 0.000e+00" in r.stdout
    r = run("verify", "--a", a, "--b", b, "--tolerance", "0")
    assert r.returncode == 1  # negative control: the tensor-core paths are not bit-exact
    assert run("bench", "--a", a, "--b", str(tmp_path / "missing.mmmb")).returncode == 3


@pytest.mark.gpu
def test_sweep_small(tmp_path):
    out = str(tmp_path / "sweep.csv")
    r = run("sweep", "--n", "512", "--grid-step", "0.5", "--trials", "1", "--out", out)
    assert r.returncode == 0, r.stderr
    rows = list(csv.DictReader(open(out)))
    assert len(rows) == 9
    one = [x for x in rows if float(x["a_sparsity"]) == 1.0 and float(x["b_sparsity"]) == 1.0][0]
    assert float(one["lane_fma_ops_per_n3"]) == 0.0  # SPEC cmd_sweep example: cell (1, 1)
