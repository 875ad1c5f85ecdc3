"""CPU-side checks of the drop-in boundary: the C-ABI library builds, loads, and exports every
symbol include/mmmcu.h declares; host-only logic and error mapping work without a GPU."""
import ctypes
import os
import re

import pytest

from paper_2402_14118_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "mmmcu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mmmcu_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_header_symbols():
    lib = N.load()
    names = header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), f"libmmmcu.so does not export {name}"
    bound = {n for n, _, _ in N.SIGNATURES}
    assert set(names) == bound, set(names) ^ bound
    assert lib.mmmcu_abi_version() == 1


def test_algo_constants_match_header():
    # the Python mirror's algorithm ids are the C ABI's mmmcu_algo enum values
    src = open(os.path.join(ROOT, "include", "mmmcu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    enum = {k: int(v) for k, v in re.findall(r"\bMMMCU_ALGO_([A-Z0-9_]+)\s*=\s*(\d+)", src)}
    assert enum["TC"] == 5 and enum["TC32"] == 6
    for name, value in enum.items():
        assert getattr(N, "ALGO_" + name) == value, name


def test_no_device_fails_loudly_without_fallback():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    lib = N.load()
    h = ctypes.c_void_p()
    st = lib.mmmcu_ctx_create(0, ctypes.byref(h))
    assert st == N.ERR_NO_DEVICE
    assert b"no CUDA device" in lib.mmmcu_last_error(None)
    import paper_2402_14118_b200 as mmm

    with pytest.raises(mmm.NoDeviceError):
        mmm.MmmContext(0)


def test_lane_validation_matches_reference():
    # KernelTable<float>::build errors (kernel_table.cpp:66-72) before any device work
    lib = N.load()
    assert lib.mmmcu_validate_lane(None, N.Lane(8, 17, 1)) == N.ERR_INVALID_ARG
    assert b"pattern size must lie in [1, 16], got 17" in lib.mmmcu_last_error(None)
    assert lib.mmmcu_validate_lane(None, N.Lane(3, 8, 1)) == N.ERR_INVALID_ARG
    assert b"unsupported lane configuration: group width 3 for f32" in lib.mmmcu_last_error(None)
    assert lib.mmmcu_validate_lane(None, N.Lane(8, 8, 0)) == N.ERR_INVALID_ARG
    # every valid lane config has a GPU path (the lane-general kernels, kgen.cuh)
    for lane in ((4, 8, 1), (1, 16, 1), (2, 8, 4), (64, 1, 1), (8, 8, 1)):
        assert lib.mmmcu_validate_lane(None, N.Lane(*lane)) == N.OK, lane
    # KernelTable<double>::build (kernel_table.cpp:69-72 with dtype_name f64)
    assert lib.mmmcu_validate_lane_t(None, N.F64, N.Lane(3, 8, 1)) == N.ERR_INVALID_ARG
    assert b"unsupported lane configuration: group width 3 for f64" in lib.mmmcu_last_error(None)
    assert lib.mmmcu_validate_lane_t(None, N.F64, N.Lane(4, 8, 1)) == N.OK
    assert lib.mmmcu_validate_lane_t(None, 7, N.Lane(4, 8, 1)) == N.ERR_UNSUPPORTED  # no such dtype


@pytest.mark.parametrize("M,world", [(32768, 1), (32768, 2), (32768, 8), (1000, 3), (7, 8)])
def test_shard_rows_partition(M, world):
    import paper_2402_14118_b200 as mmm

    spans = [mmm.shard_rows(M, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == M
    for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
        assert a1 == b0 and a0 <= a1
    assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    with pytest.raises(ValueError):
        mmm.shard_rows(M, world, world)
