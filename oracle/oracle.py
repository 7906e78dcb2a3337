"""TEST INFRASTRUCTURE ONLY — numpy/ctypes front-end for the CPU checkers.

Two libraries sit behind this module:

* ``_build/libhalo_oracle.so`` — the plain-C restatement (halo_oracle.c).
* ``_ref/libhalo_ref.so`` — the UNMODIFIED reference headers behind an
  ``extern "C"`` shim (ref_shim.cpp), built in this container from
  /root/reference and shipped prebuilt to the GPU box.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg import this module.  The product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libhalo_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libhalo_ref.so")

INT8, FP8_E4M3, FP6_E3M2, MXFP6_E3M2 = 0, 1, 2, 3

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i8p = np.ctypeslib.ndpointer(np.int8, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i64 = C.c_int64
_ll = C.c_longlong


def build():
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class _Scheme(C.Structure):
    _fields_ = [("level", C.c_int), ("fmt", C.c_int), ("block", C.c_int64)]


_orc = None
_ref = None


def orc():
    """The C restatement (always available once built)."""
    global _orc
    if _orc is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = C.CDLL(ORACLE_SO)
        L.orc_is_supported_hadamard_dim.argtypes = [_i64]
        L.orc_next_supported_hadamard_dim.argtypes = [_i64]
        L.orc_next_supported_hadamard_dim.restype = _i64
        L.orc_fwht_rows.argtypes = [_f32p, _i64, _i64, _i64]
        L.orc_fwht_cols.argtypes = [_f32p, _i64, _i64, _i64]
        L.orc_round_code.argtypes = [C.c_double, C.c_int]
        L.orc_round_code.restype = C.c_double
        L.orc_tensor_scale.argtypes = [_f32p, _i64, C.c_int, C.POINTER(C.c_int)]
        L.orc_tensor_scale.restype = C.c_float
        L.orc_quantize.argtypes = [_f32p, _i64, _i64, C.c_int, C.c_int, C.c_int, _f32p, _f32p]
        L.orc_codes_to_int8.argtypes = [_f32p, _i64, _i8p]
        L.orc_codes_to_e4m3.argtypes = [_f32p, _i64, _u8p]
        L.orc_e4m3_to_float.argtypes = [C.c_uint8]
        L.orc_e4m3_to_float.restype = C.c_float
        L.orc_qmatmul_i8.argtypes = [_i8p, _i8p, _i64, _i64, _i64, C.c_int, C.c_int,
                                     C.c_float, C.c_float, C.c_void_p, C.c_void_p]
        L.orc_qmatmul_deq.argtypes = [_f32p, _f32p, _i64, _i64, _i64, C.c_int, C.c_int,
                                      C.c_float, C.c_float, _f32p]
        L.orc_linear_forward.argtypes = [C.POINTER(_Scheme), _i64, _i64, _i64, _f32p, _f32p,
                                         _f32p, _f32p, C.POINTER(C.c_float), _f32p,
                                         C.POINTER(C.c_float)]
        L.orc_linear_backward.argtypes = [C.POINTER(_Scheme), _i64, _i64, _i64, _f32p,
                                          C.c_float, _f32p, C.c_float, _f32p, _f32p, _f32p,
                                          _f32p, C.POINTER(C.c_float), _f32p,
                                          C.POINTER(C.c_float)]
        L.orc_padded_batch.argtypes = [C.POINTER(_Scheme), _i64]
        L.orc_padded_batch.restype = _i64
        L.orc_time_linear.argtypes = [C.POINTER(_Scheme), _i64, _i64, _i64, C.c_uint64]
        L.orc_time_linear.restype = C.c_double
        L.orc_randn.argtypes = [_f32p, _i64, C.c_uint64, C.c_double]
        _orc = L
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The reference itself (headers compiled unmodified)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            if os.path.isdir("/root/reference/proj/include/halo"):
                build()
            else:
                raise RuntimeError("oracle/_ref/libhalo_ref.so missing and no reference to build from")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_is_supported_hadamard_dim.argtypes = [_ll]
        L.ref_next_supported_hadamard_dim.argtypes = [_ll]
        L.ref_next_supported_hadamard_dim.restype = _ll
        for f in (L.ref_fwht_rows, L.ref_fwht_rows_ht, L.ref_fwht_cols):
            f.argtypes = [_f32p, _ll, _ll, _ll]
        L.ref_round_code.argtypes = [C.c_double, C.c_int]
        L.ref_round_code.restype = C.c_double
        L.ref_quantize.argtypes = [_f32p, _ll, _ll, C.c_int, C.c_int, C.c_int, _f32p, _f32p]
        L.ref_qmatmul.argtypes = [_f32p, _f32p, _ll, _ll, _ll, C.c_int, C.c_int, C.c_float,
                                  C.c_float, _f32p]
        L.ref_linear.argtypes = [C.c_int, C.c_int, _ll, _ll, _ll, _ll, _f32p, _f32p, _f32p, _f32p,
                                 _f32p, _f32p, _f32p, C.POINTER(C.c_float), _f32p,
                                 C.POINTER(C.c_float)]
        L.ref_linear_g.argtypes = [C.c_int, C.c_int, _ll, C.c_int] + L.ref_linear.argtypes[3:]
        L.ref_fsdp_gather.argtypes = [_ll, _f32p, _ll, _ll, C.c_int, C.c_int, _f32p,
                                      C.POINTER(C.c_float), _f64p]
        L.ref_reduce_scatter.argtypes = [_ll, _f32p, _ll, _ll, _f32p]
        L.ref_randn.argtypes = [_f32p, _ll, C.c_ulonglong, C.c_double]
        L.ref_inject_outliers.argtypes = [_f32p, _ll, _ll, _i64p, _ll, C.c_double, C.c_int]
        L.ref_time_linear.argtypes = [C.c_int, C.c_int, _ll, _ll, _ll, _ll, C.c_int]
        L.ref_time_linear.restype = C.c_double
        _ref = L
    return _ref


def _chk(lib, rc):
    if rc != 0:
        msg = lib.ref_last_error().decode() if hasattr(lib, "ref_last_error") else ""
        exc = {1: ValueError, 2: ArithmeticError, 3: RuntimeError}.get(rc, RuntimeError)
        raise exc(msg)


def f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def bf16_round(a):
    """Round float32 values to bfloat16 (RNE) and return them as float32."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


# ----------------------------------------------------------- restatement --

def fwht_rows(a, block):
    out = f32(a).copy()
    orc().orc_fwht_rows(out, out.shape[0], out.shape[1], block)
    return out


def fwht_cols(a, block):
    out = f32(a).copy()
    orc().orc_fwht_cols(out, out.shape[0], out.shape[1], block)
    return out


def _groups(gran, rows, cols):
    return 1 if gran == 0 else rows if gran == 1 else cols if gran == 2 else rows * ((cols + 31) // 32)


def quantize(a, fmt=INT8, gran=0, scales=None):
    """gran: 0 tensor, 1 row, 2 column, 4 mx (1 x 32 blocks along rows)."""
    a = f32(a)
    rows, cols = a.shape
    groups = _groups(gran, rows, cols)
    s = np.zeros(groups, np.float32) if scales is None else f32(np.atleast_1d(scales)).copy()
    codes = np.zeros_like(a)
    orc().orc_quantize(a, rows, cols, fmt, gran, 0 if scales is None else 1, s, codes)
    return codes, s


def e3m2_table():
    """Value of every 6-bit OCP E3M2 code (bias 3, no inf/NaN): the grid of
    round_minifloat(x, 2, -2, 28) (quantize.hpp:138-150, 164-166)."""
    c = np.arange(64)
    e = (c >> 2) & 7
    m = c & 3
    v = np.where(e == 0, m * 0.0625, (1 + m / 4.0) * 2.0 ** (e - 3))
    return np.where(c & 0x20, -v, v).astype(np.float32)


def codes_to_bytes(codes, fmt):
    """Code values -> the device's code bytes (INT8 two's complement, OCP
    E4M3, and for FP6 the E3M2 code shifted into bits 7:2)."""
    codes = f32(codes)
    if fmt == INT8:
        out = np.empty(codes.shape, np.int8)
        orc().orc_codes_to_int8(codes, codes.size, out)
    elif fmt in (FP6_E3M2, MXFP6_E3M2):
        table = e3m2_table()
        lut = {}
        for c in range(63, -1, -1):  # 0.0 -> code 0 (the reference's +0)
            lut[float(table[c])] = c
        flat = np.array([lut[float(v) if v != 0 else 0.0] for v in codes.ravel()], np.uint8)
        out = (flat << 2).astype(np.uint8).reshape(codes.shape)
    else:
        out = np.empty(codes.shape, np.uint8)
        orc().orc_codes_to_e4m3(codes, codes.size, out)
    return out


def e4m3_table():
    return np.array([orc().orc_e4m3_to_float(i) for i in range(256)], np.float32)


def qmatmul_i8(A, B, a_kmajor=True, b_kmajor=True, sa=1.0, sb=1.0, M=None, N=None, K=None):
    """Returns (int32 accumulators, float output). A/B int8 arrays."""
    A = np.ascontiguousarray(A, np.int8)
    B = np.ascontiguousarray(B, np.int8)
    if M is None:
        M, K = A.shape if a_kmajor else A.shape[::-1]
        N = B.shape[0] if b_kmajor else B.shape[1]
    acc = np.zeros((M, N), np.int32)
    out = np.zeros((M, N), np.float32)
    orc().orc_qmatmul_i8(A, B, M, N, K, int(a_kmajor), int(b_kmajor), sa, sb,
                         acc.ctypes.data, out.ctypes.data)
    return acc, out


def qmatmul_deq(A, B, a_kmajor, b_kmajor, sa, sb):
    A, B = f32(A), f32(B)
    M, K = A.shape if a_kmajor else A.shape[::-1]
    N = B.shape[0] if b_kmajor else B.shape[1]
    out = np.zeros((M, N), np.float32)
    orc().orc_qmatmul_deq(A, B, M, N, K, int(a_kmajor), int(b_kmajor), sa, sb, out)
    return out


def scheme(level, fmt=INT8, block=0):
    return _Scheme(level, fmt, block)


def padded_batch(level, fmt, block, b):
    s = scheme(level, fmt, block)
    return orc().orc_padded_batch(C.byref(s), b)


def linear(level, fmt, block, X, W, EY):
    """Restated HaloLinearLayer forward+backward. Returns a dict."""
    X, W, EY = f32(X), f32(W), f32(EY)
    b, m = X.shape
    n = W.shape[0]
    s = scheme(level, fmt, block)
    bp = orc().orc_padded_batch(C.byref(s), b)
    Y = np.zeros((b, n), np.float32)
    xq = np.zeros((b, m), np.float32)
    wq = np.zeros((n, m), np.float32)
    sx, sw = C.c_float(), C.c_float()
    orc().orc_linear_forward(C.byref(s), b, m, n, X, W, Y, xq, C.byref(sx), wq, C.byref(sw))
    EX = np.zeros((b, m), np.float32)
    GW = np.zeros((n, m), np.float32)
    ehq = np.zeros((bp, n), np.float32)
    eq = np.zeros((b, n), np.float32)
    seh, se = C.c_float(), C.c_float()
    orc().orc_linear_backward(C.byref(s), b, m, n, xq, sx.value, wq, sw.value, EY, EX, GW, ehq,
                              C.byref(seh), eq, C.byref(se))
    return dict(Y=Y, EX=EX, GW=GW, xq=xq, sx=sx.value, wq=wq, sw=sw.value, ehq=ehq,
                seh=seh.value, eq=eq, se=se.value)


def randn(rows, cols, seed, stddev=1.0):
    out = np.zeros((rows, cols), np.float32)
    orc().orc_randn(out, rows * cols, seed, stddev)
    return out


def time_linear(level, fmt, block, b, m, n, seed=1):
    s = scheme(level, fmt, block)
    return orc().orc_time_linear(C.byref(s), b, m, n, seed)


# ------------------------------------------------------------- reference --

def ref_fwht_rows(a, block, ht=False):
    out = f32(a).copy()
    L = ref()
    _chk(L, (L.ref_fwht_rows_ht if ht else L.ref_fwht_rows)(out, out.shape[0], out.shape[1], block))
    return out


def ref_fwht_cols(a, block):
    out = f32(a).copy()
    L = ref()
    _chk(L, L.ref_fwht_cols(out, out.shape[0], out.shape[1], block))
    return out


def ref_quantize(a, fmt=INT8, gran=0, scales=None):
    a = f32(a)
    rows, cols = a.shape
    groups = _groups(gran, rows, cols)
    s = np.zeros(groups, np.float32) if scales is None else f32(np.atleast_1d(scales)).copy()
    codes = np.zeros_like(a)
    L = ref()
    _chk(L, L.ref_quantize(a, rows, cols, fmt, gran, 0 if scales is None else 1, s, codes))
    return codes, s


def ref_round_code(x, fmt):
    return ref().ref_round_code(float(x), fmt)


def ref_qmatmul(A, B, transpose_b, fmt, sa, sb):
    A, B = f32(A), f32(B)
    M, K = A.shape
    N = B.shape[0] if transpose_b else B.shape[1]
    out = np.zeros((M, N), np.float32)
    L = ref()
    _chk(L, L.ref_qmatmul(A, B, M, N, K, int(transpose_b), fmt, sa, sb, out))
    return out


def ref_linear(level, fmt, block, X, W, EY, gran=0):
    """The reference HaloLinearLayer forward+backward (gran 1 = Granularity::row():
    per-row scales, dequantized double products, quantize.hpp:377-379);
    sx / sw are the first scale of each operand."""
    X, W, EY = f32(X), f32(W), f32(EY)
    b, m = X.shape
    n = W.shape[0]
    Y = np.zeros((b, n), np.float32)
    EX = np.zeros((b, m), np.float32)
    GW = np.zeros((n, m), np.float32)
    xq = np.zeros((b, m), np.float32)
    wq = np.zeros((n, m), np.float32)
    sx, sw = C.c_float(), C.c_float()
    L = ref()
    _chk(L, L.ref_linear_g(level, fmt, block, gran, b, m, n, X, W, EY, Y, EX, GW, xq, C.byref(sx), wq,
                           C.byref(sw)))
    return dict(Y=Y, EX=EX, GW=GW, xq=xq, sx=sx.value, wq=wq, sw=sw.value)


def ref_fsdp_gather(world, W, fmt=INT8, hadamard=True):
    W = f32(W)
    rows, cols = W.shape
    padded = (rows + world - 1) // world * world
    codes = np.zeros((padded, cols), np.float32)
    scale = C.c_float()
    absmax = np.zeros(world, np.float64)
    L = ref()
    _chk(L, L.ref_fsdp_gather(world, W, rows, cols, fmt, int(hadamard), codes, C.byref(scale),
                              absmax))
    return codes, scale.value, absmax


def ref_reduce_scatter(grads):
    grads = f32(grads)
    world, rows, cols = grads.shape
    shard_rows = (rows + world - 1) // world
    out = np.zeros((world, shard_rows, cols), np.float32)
    L = ref()
    _chk(L, L.ref_reduce_scatter(world, grads, rows, cols, out))
    return out


def ref_randn(rows, cols, seed, stddev=1.0):
    out = np.zeros((rows, cols), np.float32)
    ref().ref_randn(out, rows * cols, seed, stddev)
    return out


def ref_inject_outliers(a, channels, mag, axis_rows=False):
    out = f32(a).copy()
    ch = np.ascontiguousarray(channels, np.int64)
    L = ref()
    _chk(L, L.ref_inject_outliers(out, out.shape[0], out.shape[1], ch, len(ch), mag,
                                  int(axis_rows)))
    return out


def ref_time_linear(level, fmt, block, b, m, n, threads=1):
    return ref().ref_time_linear(level, fmt, block, b, m, n, threads)


def ref_write_quantized(path, codes, scales, fmt, gran=0):
    """The reference's write_quantized_tensor (quantize.hpp:405-430)."""
    codes, scales = f32(codes), f32(np.atleast_1d(scales))
    L = ref()
    L.ref_write_quantized.argtypes = [C.c_char_p, C.c_int, C.c_int, _ll, _ll, _f32p, _f32p, _ll]
    _chk(L, L.ref_write_quantized(str(path).encode(), fmt, gran, codes.shape[0], codes.shape[1], codes, scales,
                                  scales.size))


def ref_read_quantized(path):
    """The reference's read_quantized_tensor (quantize.hpp:432-474) ->
    (codes as float values, scales, fmt, granularity kind)."""
    L = ref()
    L.ref_read_quantized_info.argtypes = [C.c_char_p] + [C.POINTER(C.c_int)] * 2 + [C.POINTER(_ll)] * 3
    L.ref_read_quantized.argtypes = [C.c_char_p, _f32p, _f32p]
    f, g = C.c_int(), C.c_int()
    r, c, n = _ll(), _ll(), _ll()
    _chk(L, L.ref_read_quantized_info(str(path).encode(), C.byref(f), C.byref(g), C.byref(r), C.byref(c),
                                      C.byref(n)))
    codes = np.zeros((r.value, c.value), np.float32)
    scales = np.zeros(n.value, np.float32)
    _chk(L, L.ref_read_quantized(str(path).encode(), codes, scales))
    return codes, scales, f.value, g.value


def ref_rmsnorm(x, gain, e):
    """The reference's rmsnorm_forward / _backward / rmsnorm_gain_gradient
    (rmsnorm.hpp:27-100) -> (y, dx, dgain); x, e [rows x dim], gain [dim]."""
    x, e, gain = f32(x), f32(e), f32(np.asarray(gain).reshape(1, -1))
    rows, dim = x.shape
    y = np.zeros_like(x)
    dx = np.zeros_like(x)
    dg = np.zeros((1, dim), np.float32)
    L = ref()
    L.ref_rmsnorm.argtypes = [_f32p, _f32p, _f32p, _ll, _ll, _f32p, _f32p, _f32p]
    _chk(L, L.ref_rmsnorm(x, gain, e, rows, dim, y, dx, dg))
    return y, dx, dg[0]
