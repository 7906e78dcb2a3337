"""The C restatement against the reference compiled from /root/reference
(oracle/_ref/libhalo_ref.so): bit-exact on randomized cases.  Skipped where
the prebuilt reference library is absent."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def O(orc):
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built (no /root/reference here)")
    return orc


@pytest.mark.parametrize("level", [0, 1, 2])
@pytest.mark.parametrize("fmt", [0, 1, 2])
@pytest.mark.parametrize("block,b,m,n", [(0, 64, 128, 32), (32, 96, 64, 48), (16, 30, 32, 16), (0, 60, 64, 16)])
def test_layer_bitexact(O, level, fmt, block, b, m, n):
    seed = 1000 + 7 * level + 3 * fmt + b
    X = O.bf16_round(O.ref_randn(b, m, seed))
    X[:, 1] *= 40
    W = O.bf16_round(O.ref_randn(n, m, seed + 1, 1 / np.sqrt(m)))
    E = O.bf16_round(O.ref_randn(b, n, seed + 2, 1e-3))
    r = O.ref_linear(level, fmt, block, X, W, E)
    o = O.linear(level, fmt, block, X, W, E)
    for k in ("Y", "EX", "GW", "xq", "wq"):
        assert np.array_equal(r[k], o[k]), k
    assert r["sx"] == o["sx"] and r["sw"] == o["sw"]


def _seq_double_product(a, b):
    """sum_k a[:, k] * b[k, :] in double, k ascending (tensor.hpp:127-144)."""
    acc = np.zeros((a.shape[0], b.shape[1]), np.float64)
    for k in range(a.shape[1]):
        acc += a[:, k:k + 1] * b[k:k + 1, :]
    return acc.astype(np.float32)


@pytest.mark.parametrize("fmt", [0, 1])
def test_row_granularity_backward_is_dequantized_double_product(O, fmt):
    """What csrc/deq_gemm.cu restates: with Granularity::row the reference's
    E and G products dequantize each operand to float (double(code) * scale,
    quantize.hpp:283-294) and accumulate in double, k ascending
    (quantize.hpp:377-379); E_Y^T carries E_Y's row scales as column scales
    (transpose_quantized, :297-334).  HALO-0 (no rotations) isolates it."""
    b, m, n = 40, 64, 48
    X = O.bf16_round(O.ref_randn(b, m, 71))
    W = O.bf16_round(O.ref_randn(n, m, 72, 1 / np.sqrt(m)))
    E = O.bf16_round(O.ref_randn(b, n, 73, 1e-3))
    r = O.ref_linear(0, fmt, 0, X, W, E, gran=1)
    deq = lambda c, s: (c.astype(np.float64) * s[:, None].astype(np.float64)).astype(np.float32).astype(np.float64)
    xq, sx = O.ref_quantize(X, fmt, gran=1)
    wq, sw = O.ref_quantize(W, fmt, gran=1)
    eq, se = O.ref_quantize(E, fmt, gran=1)
    assert np.array_equal(r["EX"], _seq_double_product(deq(eq, se), deq(wq, sw)))
    assert np.array_equal(r["GW"], _seq_double_product(deq(eq, se).T, deq(xq, sx)))


@pytest.mark.parametrize("fmt", [0, 1])
def test_column_granularity_is_dequantized_double_product(O, fmt):
    """Granularity::column (quantize.hpp:73-132): one scale per column, all
    three products dequantized double matmuls; E_Y^T's column scales become
    row scales (transpose_quantized :317-320).  HALO-0 isolates it."""
    b, m, n = 24, 32, 40
    X = O.bf16_round(O.ref_randn(b, m, 81))
    W = O.bf16_round(O.ref_randn(n, m, 82, 1 / np.sqrt(m)))
    E = O.bf16_round(O.ref_randn(b, n, 83, 1e-3))
    r = O.ref_linear(0, fmt, 0, X, W, E, gran=2)
    deq = lambda c, s: (c.astype(np.float64) * s[None, :].astype(np.float64)).astype(np.float32).astype(np.float64)
    xq, sx = O.ref_quantize(X, fmt, gran=2)
    wq, sw = O.ref_quantize(W, fmt, gran=2)
    eq, se = O.ref_quantize(E, fmt, gran=2)
    assert sx.shape == (m,) and se.shape == (n,)
    assert np.array_equal(r["Y"], _seq_double_product(deq(xq, sx), deq(wq, sw).T))
    assert np.array_equal(r["EX"], _seq_double_product(deq(eq, se), deq(wq, sw)))
    assert np.array_equal(r["GW"], _seq_double_product(deq(eq, se).T, deq(xq, sx)))


@pytest.mark.parametrize("block", [2, 8, 64, 256, 1024])
def test_transforms(O, block):
    a = O.ref_randn(8, 1024, block)
    assert np.array_equal(O.fwht_rows(a, block), O.ref_fwht_rows(a, block))
    assert np.array_equal(O.fwht_rows(a, block), O.ref_fwht_rows(a, block, ht=True))  # H == H^T for 2^n
    c = O.ref_randn(1024, 8, block + 1)
    assert np.array_equal(O.fwht_cols(c, block), O.ref_fwht_cols(c, block))


def test_round_code_random(O):
    rng = np.random.default_rng(3)
    xs = np.concatenate([rng.normal(0, 60, 20000), np.arange(-130, 130) + 0.5, rng.normal(0, 300, 20000)])
    for fmt in (0, 1):
        for x in xs:
            assert O.orc().orc_round_code(float(x), fmt) == O.ref_round_code(float(x), fmt)


def test_fsdp_gather_matches_single_process(O):
    # test_hqfsdp.cpp:98-125 semantics: 50 random weights per world size
    rng = np.random.default_rng(11)
    for world in (1, 2, 4, 8):
        for rep in range(10):
            rows = 3 + int(rng.integers(0, 38))
            cols = 16 if rep % 2 == 0 else 32
            W = O.ref_randn(rows, cols, 50 * world + rep)
            fmt = 1 if rep % 5 == 0 else 0
            codes, scale, _ = O.ref_fsdp_gather(world, W, fmt, rep % 4 != 3)
            padded = (rows + world - 1) // world * world
            P = np.zeros((padded, cols), np.float32)
            P[:rows] = W
            want, s = O.quantize(O.fwht_rows(P, cols) if rep % 4 != 3 else P, fmt)
            assert np.array_equal(codes, want) and scale == s[0]


def test_mxfp6_quantizer(O):
    """NumericFormat::MxFp6E3M2 under Granularity::mx (the only pairing the
    reference accepts, quantize.hpp:247-250): power-of-two scale per 1 x 32
    block (:224-232), E3M2 codes -- the restatement against the reference,
    incl. an absmax exactly at 28 * 2^k, all-zero blocks and ragged cols."""
    for cols in (64, 80):
        a = O.bf16_round(O.randn(40, cols, 31))
        a[3, :] = 28.0 * 4      # m / 2^e == 28 exactly: no bump
        a[5, :32] = 0.0         # all-zero block -> scale 1
        a[:, 7] *= 1e-20
        got = O.quantize(a, 3, 4)
        want = O.ref_quantize(a, 3, 4)
        assert np.array_equal(got[1], want[1]) and np.array_equal(got[0], want[0])
        s = want[1][want[1] != 1.0]
        assert np.all(np.frexp(s)[0] == 0.5)  # powers of two
    with pytest.raises(ValueError):
        O.ref_quantize(a, 3, 0)  # mxfp6 needs mx granularity
