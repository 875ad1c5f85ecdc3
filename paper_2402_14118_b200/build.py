"""In-tree build of the CUDA library (sm_100a) and of the oracle (test infrastructure).

    python -m paper_2402_14118_b200.build          # libmmmcu.so (+ oracle, + oracle/_ref)

The library is compiled straight with nvcc (-gencode arch=compute_100a,code=sm_100a
-lineinfo) into paper_2402_14118_b200/_lib/ so it travels with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _run(cmd, cwd=None):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=cwd)


def build_lib(verbose_ptxas: bool = False) -> str:
    out_dir = os.path.join(HERE, "_lib")
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, "libmmmcu.so")
    srcs = [os.path.join(HERE, "csrc", f) for f in ("mmmcu.cu", "mmmcu_group.cu", "mmmcu_io.cu")]
    cmd = [NVCC, *GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
           "-I", os.path.join(ROOT, "include"), "-o", out, *srcs, "-ldl"]
    if verbose_ptxas:
        cmd.insert(1, "-Xptxas=-v")
    _run(cmd)
    return out


def build_cli() -> str:
    """The SPEC bench-cli on the GPU path (cli/mmm_cuda.cpp -> _lib/mmm-cuda), linked against
    libmmmcu.so (C ABI) and cuBLAS (the dense comparator only)."""
    out = os.path.join(HERE, "_lib", "mmm-cuda")
    cuda = os.path.dirname(os.path.dirname(NVCC))
    _run(["g++", "-O2", "-std=c++17", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(cuda, "include"),
          os.path.join(HERE, "cli", "mmm_cuda.cpp"), "-L", os.path.join(HERE, "_lib"), "-L", os.path.join(cuda, "lib64"),
          "-lmmmcu", "-lcublas", "-lcudart", "-Wl,-rpath,$ORIGIN", "-o", out])
    return out


def build_probe() -> str:
    """FP32 peak probe used by bench.py for the SIMT roofline denominator (tools/, not product)."""
    out_dir = os.path.join(ROOT, "tools", "_lib")
    os.makedirs(out_dir, exist_ok=True)
    out = os.path.join(out_dir, "libfp32probe.so")
    _run([NVCC, *GENCODE, "-O3", "-Xcompiler", "-fPIC", "-shared", "-o", out,
          os.path.join(ROOT, "tools", "probe", "fp32_probe.cu")])
    return out


def build_dropin_test() -> str:
    """C++ drop-in check (tests/cpp/dropin_test.cpp) against the reference's own headers; only
    where /root/reference exists (the binary then travels with the repo snapshot)."""
    ref_inc = "/root/reference/proj/include"
    out = os.path.join(HERE, "_lib", "dropin_test")
    if not os.path.isdir(ref_inc):
        return ""
    _run(["g++", "-std=c++20", "-O2", "-I", ref_inc, "-I", os.path.join(ROOT, "include"),
          os.path.join(ROOT, "tests", "cpp", "dropin_test.cpp"), "-L", os.path.join(HERE, "_lib"), "-lmmmcu",
          "-Wl,-rpath,$ORIGIN", "-o", out])
    return out


def build_oracle() -> None:
    env_make = ["make", "-C", os.path.join(ROOT, "oracle")]
    _run(env_make)
    if os.path.isdir("/root/reference/proj"):
        _run(env_make + ["ref"])


def main(argv=None):
    build_lib()
    build_cli()
    build_probe()
    build_dropin_test()
    build_oracle()


if __name__ == "__main__":
    main(sys.argv[1:])
