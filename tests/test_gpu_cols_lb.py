"""The single-kernel large-block left transform (csrc/fwht_cols_lb.cu, 512 <=
B <= 4096: one strip of B rows x W columns per CTA, one smem exchange)
against the C oracle: rotated and plain codes + scales (phase A + phase B,
every format, bf16 and fp32 inputs, several strips in both directions,
padded token blocks) and the fp32 transform-only mode (K4-left), bit-exact.
Reference: halo_linear.hpp:393-399 (error_path), hadamard.hpp:136-177,
205-216 (transform_left), quantize.hpp:244-280."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2501_02625_b200 import halo
    return halo


@pytest.fixture(scope="module")
def orc():
    from oracle import oracle
    return oracle


def _codes(t):
    return t.cpu().numpy().view(np.uint8)


@pytest.mark.parametrize("block", [512, 1024, 2048, 4096])
@pytest.mark.parametrize("dtype", ["bf16", "f32"])
@pytest.mark.parametrize("fmt", [0, 1, 2])
def test_left_large_block_codes_bitexact(H, orc, block, dtype, fmt):
    E = 32768 if (dtype == "bf16" and block >= 1024) else 16384  # strip elements
    W = E // block
    b, n = 2 * block - 37, 4 * W           # two token blocks (the second padded), four column strips
    rng = np.random.default_rng(block + 7 * fmt)
    e = rng.standard_normal((b, n)).astype(np.float32) * 1e-3
    e[b // 3, :] *= 40.0                    # an outlier token row
    e[:, 1] *= 9.0                          # and an outlier column
    if dtype == "bf16":
        e = orc.bf16_round(e)
        t = torch.from_numpy(e).cuda().to(torch.bfloat16)
    else:
        t = torch.from_numpy(e).cuda()
    cr, sr, cp, sp = H.left_rotate_quantize(t, had_block=block, fmt=fmt)
    bp = H.padded_batch(b, block)
    assert bp == 2 * block
    pad = np.zeros((bp, n), np.float32)
    pad[:b] = e
    wr, wsr = orc.quantize(orc.fwht_cols(pad, block), fmt)
    wp, wsp = orc.quantize(e, fmt)
    torch.cuda.synchronize()
    assert sr.item() == wsr[0] and sp.item() == wsp[0]
    assert np.array_equal(_codes(cr), orc.codes_to_bytes(wr, fmt).view(np.uint8))
    assert np.array_equal(_codes(cp), orc.codes_to_bytes(wp, fmt).view(np.uint8))


@pytest.mark.parametrize("block", [512, 1024, 2048, 4096])
def test_left_large_block_transform_bitexact(H, orc, block):
    """transform_left on fp32 (the non-fused HALO-2 backward, B > 256):
    in place and into a separate buffer, rows_out < rows_pad."""
    W = 16384 // block
    rows, n = 2 * block, 2 * W
    f = np.random.default_rng(block).standard_normal((rows, n)).astype(np.float32)
    want = orc.fwht_cols(f, block)
    t = torch.from_numpy(f).cuda()
    assert np.array_equal(H.transform_left(t, block).cpu().numpy(), want)
    assert np.array_equal(H.transform_left(t, block, rows_out=rows - 100).cpu().numpy(), want[:rows - 100])


def test_left_large_block_nonstrip_width_falls_back(H, orc):
    """cols not a multiple of the strip width keep the two-kernel path."""
    block, b, n = 1024, 1000, 48   # bf16 strip width at B = 1024 is 32
    e = orc.bf16_round(np.random.default_rng(5).standard_normal((b, n)).astype(np.float32))
    cr, sr, cp, sp = H.left_rotate_quantize(torch.from_numpy(e).cuda().to(torch.bfloat16), had_block=block)
    pad = np.zeros((block, n), np.float32)
    pad[:b] = e
    wr, wsr = orc.quantize(orc.fwht_cols(pad, block), 0)
    torch.cuda.synchronize()
    assert sr.item() == wsr[0]
    assert np.array_equal(_codes(cr), orc.codes_to_bytes(wr, 0).view(np.uint8))


def test_left_large_block_nonfinite_flagged(H):
    """An Inf in E_Y reaches the absmax word and the context's error flag
    (had_block = 0 over 2048 tokens: B = 2048 on the token axis)."""
    layer = H.HaloLinearLayer(torch.randn(16, 64, device="cuda"), H.halo2(0, 0))
    ctx = H.SavedContext()
    layer.forward(torch.randn(2048, 64, device="cuda"), ctx)
    ctx.check()
    e = torch.zeros((2048, 16), device="cuda")
    e[7, 3] = float("inf")
    layer.backward(ctx, e)
    with pytest.raises(H._lib.HaloNumericError):
        ctx.check()
