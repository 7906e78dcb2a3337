"""Hadamard blocks of 12·2^k and 20·2^k elements (hadamard.hpp:62-129, the
reference's Paley bases) on the device (csrc/fwht_base.cu), checked bit for
bit against the UNMODIFIED reference library (oracle/_ref, built from
/root/reference): its transforms, its quantizer on those transforms, and its
HaloLinearLayer at HALO-1/2.  Both orientations are exercised: H for
transform_right / transform_left, H^T for transform_right_ht / the error
path's transform_left_h.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H(orc):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built")
    from paper_2501_02625_b200 import halo
    return halo


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t.to(dtype) if dtype is not None else t


def make(orc, rows, cols, seed, std=1.0):
    a = orc.randn(rows, cols, seed, std)
    a[:, 1] *= 30.0
    return orc.bf16_round(a)


def test_paley_bases_match_reference(H, orc):
    """The device's base matrices (Paley I over GF(11) / GF(19)) are the
    reference's tables: transform of the identity, both orientations."""
    for m, cols in ((12, 48), (20, 80), (24, 48), (40, 80)):  # rows of whole blocks, 16-multiple length
        eye = np.zeros((m, cols), np.float32)
        eye[np.arange(m), np.arange(m)] = 1.0
        got = H.transform_right(dev(eye), had_block=m).cpu().numpy()
        assert np.array_equal(got, orc.ref_fwht_rows(eye, m)), m


@pytest.mark.parametrize("rows,cols,block", [(16, 96, 48), (8, 384, 384), (12, 640, 320), (5, 1280, 0),
                                             (9, 3072, 768)])
def test_transforms_base_dims(H, orc, rows, cols, block):
    a = orc.randn(rows, cols, 5 + rows)
    B = block or cols
    got = H.transform_right(dev(a), had_block=block).cpu().numpy()
    assert np.array_equal(got, orc.ref_fwht_rows(a, B))
    at = orc.randn(cols, rows * 8, 9)  # token-axis (left) transform over `cols` rows
    got_l = H.transform_left(dev(at), had_block=block).cpu().numpy()
    assert np.array_equal(got_l, orc.ref_fwht_cols(at, B))


@pytest.mark.parametrize("rows,cols,block", [(16, 96, 48), (37, 384, 0), (20, 640, 320), (8, 3072, 0)])
@pytest.mark.parametrize("fmt", [0, 1])
def test_rotate_quantize_base_dims(H, orc, rows, cols, block, fmt):
    a = make(orc, rows, cols, 11 + rows)
    codes, scale = H.rotate_quantize(dev(a, torch.bfloat16), had_block=block, fmt=fmt)
    want_codes, want_s = orc.ref_quantize(orc.ref_fwht_rows(a, block or cols), fmt)
    torch.cuda.synchronize()
    assert scale.item() == want_s[0]
    assert np.array_equal(codes.cpu().numpy().view(np.uint8), orc.codes_to_bytes(want_codes, fmt).view(np.uint8))


@pytest.mark.parametrize("b,n,block", [(48, 64, 0), (150, 32, 0), (96, 48, 48), (300, 16, 320)])
def test_left_rotate_quantize_base_dims(H, orc, b, n, block):
    """K2: (H_b pad(E))_Q -- transform_left_h, the H^T orientation of the
    row transform applied down each column (halo_linear.hpp:393-399)."""
    e = make(orc, b, n, 3 + b, 1e-3)
    cr, sr, cp, sp = H.left_rotate_quantize(dev(e, torch.bfloat16), had_block=block, fmt=0)
    bp = H.padded_batch(b, block)
    pad = np.zeros((bp, n), np.float32)
    pad[:b] = e
    rot = orc.ref_fwht_rows(np.ascontiguousarray(pad.T), block or bp, ht=True).T  # H pad(E)
    wr, wsr = orc.ref_quantize(np.ascontiguousarray(rot), 0)
    wp, wsp = orc.ref_quantize(e, 0)
    torch.cuda.synchronize()
    assert sr.item() == wsr[0] and sp.item() == wsp[0]
    assert np.array_equal(cr.cpu().numpy(), orc.codes_to_bytes(wr, 0))
    assert np.array_equal(cp.cpu().numpy(), orc.codes_to_bytes(wp, 0))


@pytest.mark.parametrize("level,b,m,n,block", [(2, 160, 384, 96, 0), (2, 100, 640, 64, 320), (1, 77, 384, 48, 0),
                                               (2, 48, 96, 32, 48)])
def test_layer_base_dims_matches_reference_library(H, orc, level, b, m, n, block):
    X = make(orc, b, m, 21)
    W = orc.bf16_round(orc.randn(n, m, 22, 1.0 / np.sqrt(m)))
    E = orc.bf16_round(orc.randn(b, n, 23, 1e-3))
    want = orc.ref_linear(level, 0, block, X, W, E)
    layer = H.HaloLinearLayer(dev(W, torch.bfloat16), H.scheme_from_string(f"halo{level}", 0, block),
                              out_dtype=torch.float32, grad_dtype=torch.float32)
    ctx = H.SavedContext()
    y = layer.forward(dev(X, torch.bfloat16), ctx)
    back = layer.backward(ctx, dev(E, torch.bfloat16))
    torch.cuda.synchronize()
    assert np.array_equal(y.cpu().numpy(), want["Y"])
    assert np.array_equal(back.e_x.cpu().numpy(), want["EX"])
    assert np.array_equal(back.grad_w.cpu().numpy(), want["GW"])
