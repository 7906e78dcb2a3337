"""Quantized tensor files (write/read_quantized_tensor, quantize.hpp:405-474)
against the UNMODIFIED reference reader and writer (oracle/_ref): a file
written by libhalo_b200 reads back in the reference with the same code values
and scales, and a reference-written file reads into the same device code
bytes.  Host-side only (no GPU needed)."""
import numpy as np
import pytest
import torch


@pytest.fixture(scope="module")
def H():
    from paper_2501_02625_b200 import halo
    return halo


def _codes(orc, fmt, gran, rows=24, cols=40, seed=5):
    a = orc.bf16_round(orc.randn(rows, cols, seed))
    a[:, 3] *= 30
    vals, scales = orc.quantize(a, fmt, gran)
    return vals, scales, orc.codes_to_bytes(vals, fmt)


@pytest.mark.parametrize("fmt", [0, 1, 2])
@pytest.mark.parametrize("gran", [0, 1, 2])
def test_our_file_reads_in_the_reference(H, orc, tmp_path, fmt, gran):
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built")
    vals, scales, dev = _codes(orc, fmt, gran)
    path = tmp_path / "q.halt"
    H.write_quantized_tensor(path, torch.from_numpy(dev.copy()), torch.from_numpy(scales), fmt, gran)
    rv, rs, rf, rg = orc.ref_read_quantized(path)
    assert (rf, rg) == (fmt, gran)
    assert np.array_equal(rv, vals) and np.array_equal(rs, scales)
    # and back through our reader: the same device bytes
    codes, sc, f, g = H.read_quantized_tensor(path)
    assert (f, g) == (fmt, gran)
    assert np.array_equal(codes.numpy().view(np.uint8), dev.view(np.uint8))
    assert np.array_equal(sc.numpy(), scales)


@pytest.mark.parametrize("fmt", [0, 1, 2])
def test_reference_file_reads_here(H, orc, tmp_path, fmt):
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built")
    vals, scales, dev = _codes(orc, fmt, 0, seed=9)
    path = tmp_path / "r.halt"
    orc.ref_write_quantized(path, vals, scales, fmt, 0)
    codes, sc, f, g = H.read_quantized_tensor(path)
    assert (f, g) == (fmt, 0)
    assert np.array_equal(codes.numpy().view(np.uint8), dev.view(np.uint8))
    assert np.array_equal(sc.numpy(), scales)
    # byte-identical files from both writers
    mine = tmp_path / "m.halt"
    H.write_quantized_tensor(mine, torch.from_numpy(dev.copy()), torch.from_numpy(scales), fmt, 0)
    assert mine.read_bytes() == path.read_bytes()


def test_io_errors(H, orc, tmp_path):
    from paper_2501_02625_b200._lib import HaloIOError
    with pytest.raises(HaloIOError):
        H.read_quantized_tensor(tmp_path / "missing.halt")
    bad = tmp_path / "bad.halt"
    bad.write_bytes(b"NOPE" + bytes(40))
    with pytest.raises(HaloIOError):
        H.read_quantized_tensor(bad)
    vals, scales, dev = _codes(orc, 0, 0)
    good = tmp_path / "g.halt"
    H.write_quantized_tensor(good, torch.from_numpy(dev.copy()), torch.from_numpy(scales), 0, 0)
    trunc = tmp_path / "t.halt"
    trunc.write_bytes(good.read_bytes()[:-5])
    with pytest.raises(HaloIOError):
        H.read_quantized_tensor(trunc)
    # an FP8 file whose code is off the E4M3 grid
    if orc.ref_available():
        v = np.full((2, 2), 1.0, np.float32)
        v[0, 0] = 1.0625  # between 1.0 and 1.125
        off = tmp_path / "off.halt"
        orc.ref_write_quantized(off, v, np.ones(1, np.float32), 1, 0)
        with pytest.raises(HaloIOError):
            H.read_quantized_tensor(off)
    with pytest.raises(HaloIOError):  # scale count vs granularity
        H.write_quantized_tensor(tmp_path / "x.halt", torch.zeros(3, 4, dtype=torch.int8), torch.ones(2), 0, 0)
