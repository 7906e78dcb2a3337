"""FP6 E3M2 on the tcgen05 tensor cores (per-tensor).

The reference emulates FP6 E3M2 (round_minifloat(x, 2, -2, 28),
quantize.hpp:138-150, 164-166) and multiplies dequantized codes in double
(:377-379).  B200 multiplies E3M2 natively (kind::f8f6f4): device codes are
one per byte with the E3M2 bits in 7:2.  Codes and scales are bit-exact with
the oracle (tests/test_gpu_kernels.py and test_gpu_layer.py run fmt=2); here
the GEMM's operand decoding is pinned exhaustively and the accumulation
checked against fp64.
"""
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


@pytest.mark.parametrize("a_kmajor,b_kmajor", [(True, True), (False, True), (True, False), (False, False)])
def test_fp6_gemm_every_code_pair(H, orc, a_kmajor, b_kmajor):
    """C[i, j] = v(i) * v(j) for all 64 x 64 E3M2 codes, exactly."""
    K = 64
    A = np.zeros((64, K), np.uint8)
    B = np.zeros((64, K), np.uint8)
    A[:, 5] = np.arange(64, dtype=np.uint8) << 2
    B[:, 5] = np.arange(64, dtype=np.uint8) << 2
    t = orc.e3m2_table().astype(np.float64)
    want = np.outer(t, t).astype(np.float32)
    one = torch.ones(1, device="cuda")
    Ad = torch.from_numpy(A if a_kmajor else np.ascontiguousarray(A.T)).cuda()
    Bd = torch.from_numpy(B if b_kmajor else np.ascontiguousarray(B.T)).cuda()
    got = H.qmatmul(Ad, Bd, one, one, a_kmajor=a_kmajor, b_kmajor=b_kmajor, fmt=2).cpu().numpy()
    assert np.array_equal(got, want)
    # the device decode used by the tests agrees with the oracle grid
    codes = torch.arange(64, dtype=torch.int32, device="cuda").to(torch.uint8) << 2
    assert np.array_equal(H.fp6_decode(codes).cpu().numpy(), orc.e3m2_table())


@pytest.mark.parametrize("M,N,K", [(256, 256, 1024), (300, 200, 512)])
def test_fp6_gemm_vs_fp64(H, orc, M, N, K):
    rng = np.random.default_rng(M + K)
    A = (rng.integers(0, 64, size=(M, K)) << 2).astype(np.uint8)
    B = (rng.integers(0, 64, size=(N, K)) << 2).astype(np.uint8)
    t = orc.e3m2_table().astype(np.float64)
    sa, sb = np.float32(0.03), np.float32(0.0007)
    want = ((t[A >> 2] * np.float64(sa)).astype(np.float32).astype(np.float64) @
            (t[B >> 2] * np.float64(sb)).astype(np.float32).astype(np.float64).T)
    got = H.qmatmul(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), torch.tensor([sa], device="cuda"),
                    torch.tensor([sb], device="cuda"), fmt=2).cpu().numpy()
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert rel < 1e-6, rel


def test_fp6_golden_values(H):
    """test_quantize.cpp:73-79: FP6 30 -> 28 (saturation); per-tensor scale
    float(absmax / 28)."""
    a = torch.tensor([[30.0, -30.0, 1.0, 0.0] * 4], device="cuda")
    codes, scale = H.rotate_quantize(a, fmt=2, rotate=False, scale=torch.ones(1, device="cuda"))
    v = H.fp6_decode(codes).cpu().numpy()
    assert v[0, 0] == 28.0 and v[0, 1] == -28.0 and v[0, 2] == 1.0 and v[0, 3] == 0.0
    codes, scale = H.rotate_quantize(a, fmt=2, rotate=False)
    assert scale.item() == np.float32(30.0 / 28.0)



def test_fp6_wire_format_pack_unpack(H, orc):
    """The packed FP6 payload of the HQ-FSDP gather (hqfsdp.hpp:36-49: 4 codes
    in 3 bytes): layout c0 | c1<<6 | c2<<12 | c3<<18 little-endian, restated
    in numpy; unpack(pack(codes)) == codes; 0.375 of the BF16 bytes."""
    from paper_2501_02625_b200 import fsdp
    a = orc.bf16_round(orc.randn(64, 256, 13))
    codes, _ = H.rotate_quantize(torch.from_numpy(a).cuda().to(torch.bfloat16), 256, fmt=2)
    packed = H.fp6_pack(codes)
    c6 = (codes.cpu().numpy().view(np.uint8).reshape(-1, 4).astype(np.uint32) >> 2)
    word = c6[:, 0] | (c6[:, 1] << 6) | (c6[:, 2] << 12) | (c6[:, 3] << 18)
    want = np.stack([word & 0xFF, (word >> 8) & 0xFF, (word >> 16) & 0xFF], 1).astype(np.uint8).reshape(-1)
    assert np.array_equal(packed.cpu().numpy(), want)
    back = H.fp6_unpack(packed, codes.numel())
    assert torch.equal(back, codes.view(torch.uint8).reshape(-1))
    assert packed.numel() == fsdp.code_payload_bytes(fsdp.FP6_E3M2, codes.numel())
    assert packed.numel() / (2 * codes.numel()) == 0.375


# ------------------------------------------------------------------ MXFP6
# NumericFormat::MxFp6E3M2 with Granularity::mx (the only pairing the
# reference accepts, quantize.hpp:247-250): power-of-two scales per 1 x 32
# block, E3M2 codes; every layer product is the reference's dequantized
# double matmul (deq_gemm, opt-in), bit-exact.

@pytest.mark.parametrize("block", [-1, 32, 256])
def test_mx_quantizer_matches_oracle(H, orc, block):
    a = orc.randn(48, 512, 3)
    a[:, 5] *= 300
    a[7, :64] = 0.0
    a = orc.bf16_round(a)  # the device input is bf16: keep the oracle's identical
    codes, scales = H.rotate_quantize_mx(torch.from_numpy(a).cuda().to(torch.bfloat16), block, rotate=block >= 0)
    x = orc.fwht_rows(a, block) if block >= 0 else a
    want_c, want_s = orc.quantize(x, 3, 4)
    assert np.array_equal(scales.cpu().numpy().reshape(-1), want_s)
    assert np.array_equal(codes.cpu().numpy(), orc.codes_to_bytes(want_c, 3))
    # quantize(transpose(E)) -- the gradient path's operand
    e = orc.bf16_round(orc.randn(96, 64, 5, 1e-3))
    tc, ts = H.rotate_quantize_mx(torch.from_numpy(e).cuda().to(torch.bfloat16), transpose=True)
    wc, ws = orc.quantize(np.ascontiguousarray(e.T), 3, 4)
    assert np.array_equal(ts.cpu().numpy().reshape(-1), ws)
    assert np.array_equal(tc.cpu().numpy(), orc.codes_to_bytes(wc, 3))


@pytest.mark.parametrize("level", [0, 1, 2])
@pytest.mark.parametrize("block", [0, 64])
def test_mxfp6_layer_matches_reference(H, orc, level, block):
    """The unmodified reference HaloLinearLayer with halo{level}(MxFp6E3M2,
    Granularity::mx()): Y, E_X, grad_W bit-exact; counters as the reference
    (the gradient path quantizes transpose(E_Y) itself: e += 1)."""
    H.allow_dequantized_products(True)
    b, m, n = 96, 256, 128
    X = orc.bf16_round(orc.randn(b, m, 1))
    X[:, 3] *= 40
    X = orc.bf16_round(X)
    W = orc.bf16_round(orc.randn(n, m, 2, 1 / 16))
    E = orc.bf16_round(orc.randn(b, n, 3, 1e-3))
    want = orc.ref_linear(level, 3, block, X, W, E, gran=4)
    layer = H.HaloLinearLayer(torch.from_numpy(W).cuda().to(torch.bfloat16),
                              getattr(H, f"halo{level}")(H.MXFP6_E3M2, block, H.GRAN_MX), out_dtype=torch.float32)
    ctx = H.SavedContext()
    y = layer.forward(torch.from_numpy(X).cuda().to(torch.bfloat16), ctx)
    back = layer.backward(ctx, torch.from_numpy(E).cuda().to(torch.bfloat16))
    ctx.check()
    xq, sx, wq, sw = ctx.saved(layer)
    assert np.array_equal(xq.cpu().numpy(), orc.codes_to_bytes(want["xq"], 3))
    assert sx[0].item() == want["sx"] and sw[0].item() == want["sw"]
    assert np.array_equal(y.cpu().numpy(), want["Y"])
    assert np.array_equal(back.e_x.cpu().numpy(), want["EX"])
    assert np.array_equal(back.grad_w.cpu().numpy(), want["GW"])
    c = layer.counters()
    assert (c.x, c.w, c.e) == (1, 1, 2)


def test_mxfp6_rules(H):
    W = torch.zeros(128, 256, dtype=torch.bfloat16, device="cuda")
    H.allow_dequantized_products(True)
    with pytest.raises(ValueError):  # mxfp6 needs mx granularity
        H.HaloLinearLayer(W, H.halo2(H.MXFP6_E3M2, 256))
    with pytest.raises(ValueError):  # mx granularity needs mxfp6
        H.HaloLinearLayer(W, H.halo2(H.FP6_E3M2, 256, H.GRAN_MX))
    with pytest.raises(ValueError):  # per-tensor quantizers refuse mxfp6
        H.rotate_quantize(W, 256, fmt=H.MXFP6_E3M2)
