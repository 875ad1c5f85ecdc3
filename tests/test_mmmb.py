"""MMMB interchange files (matrix_io.hpp:11-49) through the C ABI.

The header checks run without a GPU (mmmcu_mmmb_peek parses on the host); loading into and
saving from device memory is covered by the gpu-marked tests.  The files are written here
byte by byte from the format description, and the golden MMMB bytes the reference's own
write_matrix produced (tests/golden/reference_golden.npz) must load unchanged.
"""
import struct

import numpy as np
import pytest

import paper_2402_14118_b200 as mmm


def write_mmmb(path, a, dtype_code=0, version=1, magic=b"MMMB", truncate=0):
    body = a.astype(np.float32 if dtype_code == 0 else np.float64).tobytes()
    data = magic + struct.pack("<IIQQ", version, dtype_code, a.shape[0], a.shape[1]) + body
    with open(path, "wb") as f:
        f.write(data[: len(data) - truncate] if truncate else data)


def test_peek_and_errors(tmp_path):
    a = np.arange(12, dtype=np.float32).reshape(3, 4)
    p = tmp_path / "a.mmmb"
    write_mmmb(p, a)
    assert mmm.mmmb_peek(str(p)) == ("f32", 3, 4)
    write_mmmb(p, a, dtype_code=1)
    assert mmm.mmmb_peek(str(p)) == ("f64", 3, 4)
    write_mmmb(p, a, magic=b"XXXX")
    with pytest.raises(mmm.api.BadFormatError):
        mmm.mmmb_peek(str(p))
    write_mmmb(p, a, version=2)
    with pytest.raises(mmm.api.BadFormatError):
        mmm.mmmb_peek(str(p))
    write_mmmb(p, a, dtype_code=7)
    with pytest.raises(mmm.api.BadFormatError):
        mmm.mmmb_peek(str(p))
    p.write_bytes(b"MMMB\x01\x00")
    with pytest.raises(mmm.api.TruncatedFileError):
        mmm.mmmb_peek(str(p))
    with pytest.raises(mmm.api.FileIoError):
        mmm.mmmb_peek(str(tmp_path / "missing.mmmb"))


def test_golden_reference_file_header(golden, tmp_path):
    # bytes written by the reference's own write_matrix (gen_golden.py)
    keys = [k for k in golden.files if "mmmb" in k.lower()]
    if not keys:
        pytest.skip("no MMMB golden bytes")
    p = tmp_path / "g.mmmb"
    p.write_bytes(golden[keys[0]].tobytes())
    dt, r, c = mmm.mmmb_peek(str(p))
    assert dt == "f32" and r > 0 and c > 0


@pytest.mark.gpu
def test_load_save_roundtrip_device(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    rng = np.random.default_rng(1)
    a = rng.uniform(-1, 1, (37, 101)).astype(np.float32)
    a[a < 0.3] = 0
    p = tmp_path / "a.mmmb"
    write_mmmb(p, a)
    t = mmm.mmmb_load(str(p))
    assert t.shape == (37, 101) and t.stride(0) == 128
    full = t.as_strided((37, 128), (128, 1)).cpu().numpy()
    assert np.array_equal(full[:, :101].view(np.uint32), a.view(np.uint32))
    assert (full[:, 101:] == 0).all()  # Matrix padding rebuilt
    q = tmp_path / "b.mmmb"
    mmm.mmmb_save(str(q), t)
    assert q.read_bytes() == p.read_bytes()
    write_mmmb(p, a, dtype_code=1)
    with pytest.raises(mmm.UnsupportedError):
        mmm.mmmb_load(str(p))
    write_mmmb(p, a, truncate=20)
    with pytest.raises(mmm.api.TruncatedFileError):
        mmm.mmmb_load(str(p))


@pytest.mark.gpu
def test_reference_written_file_loads_on_device(golden, tmp_path):
    # the identity the reference's write_matrix wrote (gen_golden.py) lands on the device as is
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    p = tmp_path / "eye.mmmb"
    p.write_bytes(golden["mmmb_eye4"].tobytes())
    t = mmm.mmmb_load(str(p))
    assert np.array_equal(t.cpu().numpy(), np.eye(4, dtype=np.float32) * np.float32(1.5))
