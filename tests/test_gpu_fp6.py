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
