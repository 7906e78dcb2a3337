"""Python mirror of the reference HALO operator API over libhalo_b200.so.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/halo):

=====================================  ======================================
reference                              here
=====================================  ======================================
``halo0/halo1/halo2`` (:81-106),       ``halo0/halo1/halo2``,
``scheme_from_string`` (:117-152)      ``scheme_from_string``
``build_spec`` dims (hadamard:69-93)   ``is_supported_hadamard_dim``,
                                       ``next_supported_hadamard_dim``
``quantize(transform_right(a))``       ``rotate_quantize``
``quantize(transform_left_h(pad(e)))`` ``left_rotate_quantize``
``transform_right`` / ``_left``        ``transform_right`` / ``transform_left``
``qmatmul`` (quantize:339-380)         ``qmatmul``
``HaloLinearLayerT`` (:227-462)        ``HaloLinearLayer``
``SavedContextT`` (:207-216)           ``SavedContext``
``BackwardResultT`` (:220-225)         ``BackwardResult``
``QuantCallCounters`` (:161-164)       ``Counters`` via ``layer.counters()``
=====================================  ======================================

Tensors are CUDA torch tensors (bf16 or fp32 inputs); torch is only the
allocator and the stream provider.  Every op launches the sm_100a kernels
of the shared library on ``torch.cuda.current_stream()``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import (DTYPE_BF16, DTYPE_F32, FMT_FP6_E3M2, FMT_FP8_E4M3, FMT_INT8, FMT_MXFP6_E3M2, OUT_BF16, OUT_F32, OUT_S32,
                   Counters, Scheme, check, lib)

INT8 = FMT_INT8
FP8_E4M3 = FMT_FP8_E4M3
FP6_E3M2 = FMT_FP6_E3M2
MXFP6_E3M2 = FMT_MXFP6_E3M2

_DT = {torch.float32: DTYPE_F32, torch.bfloat16: DTYPE_BF16}


GRAN_TENSOR, GRAN_ROW, GRAN_COLUMN, GRAN_MX = 0, 1, 2, 4  # halo_b200.h HALO_GRAN_*


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def _dt(t):
    if t.dtype not in _DT:
        raise ValueError(f"unsupported dtype {t.dtype}: bf16 or fp32 expected")
    return _DT[t.dtype]


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("HALO device path: tensors must live on a CUDA device")
        if t is not None and not t.is_contiguous():
            raise ValueError("HALO device path: tensors must be contiguous (row-major)")


def code_dtype(fmt):
    return torch.int8 if fmt == INT8 else torch.uint8


def fp6_decode(codes: torch.Tensor) -> torch.Tensor:
    """Values of device FP6 E3M2 code bytes (E3M2 in bits 7:2), fp32."""
    c = (codes.to(torch.int32) >> 2) & 0x3F
    e = (c >> 2) & 7
    m = (c & 3).to(torch.float32)
    v = torch.where(e == 0, m * 0.0625, (1 + m / 4) * torch.exp2((e - 3).to(torch.float32)))
    return torch.where((c & 0x20) != 0, -v, v)


# ------------------------------------------------------------------ schemes

def scheme_from_string(id: str, fmt: int = INT8, had_block: int = 0) -> Scheme:
    s = Scheme()
    check(lib().halo_scheme_from_string(id.encode(), fmt, had_block, C.byref(s)))
    return s


def halo0(fmt=INT8, had_block=0, granularity=GRAN_TENSOR):
    s = scheme_from_string("halo0", fmt, had_block)
    s.granularity = granularity  # halo_linear.hpp:81-106 take a Granularity
    return s


def halo1(fmt=INT8, had_block=0, granularity=GRAN_TENSOR):
    s = scheme_from_string("halo1", fmt, had_block)
    s.granularity = granularity  # halo_linear.hpp:81-106 take a Granularity
    return s


def halo2(fmt=INT8, had_block=0, granularity=GRAN_TENSOR):
    s = scheme_from_string("halo2", fmt, had_block)
    s.granularity = granularity  # halo_linear.hpp:81-106 take a Granularity
    return s


def is_supported_hadamard_dim(d: int) -> bool:
    return bool(lib().halo_is_supported_hadamard_dim(d))


def next_supported_hadamard_dim(d: int) -> int:
    return int(lib().halo_next_supported_hadamard_dim(d))


def padded_batch(b: int, had_block: int) -> int:
    return int(lib().halo_padded_batch(b, had_block))


# --------------------------------------------------------------- primitives

def rotate_quantize(a: torch.Tensor, had_block: int = 0, fmt: int = INT8, scale: torch.Tensor | None = None,
                    rotate: bool = True, out: torch.Tensor | None = None):
    """``quantize(transform_right(a, spec), fmt, tensor, scales)`` fused.

    Returns ``(codes, scale)``: codes int8 (INT8) or uint8 OCP-E4M3 bytes of
    the same shape, scale a 1-element fp32 CUDA tensor.  ``scale`` supplied ->
    used verbatim (quantize.hpp:259-266)."""
    _need_cuda(a, scale)
    rows, cols = a.shape
    codes = torch.empty((rows, cols), dtype=code_dtype(fmt), device=a.device) if out is None else out
    if tuple(codes.shape) != (rows, cols) or codes.element_size() != 1 or not codes.is_contiguous():
        raise ValueError("rotate_quantize: out must be a contiguous (rows x cols) code buffer")
    s_out = scale.clone() if scale is not None else torch.empty(1, dtype=torch.float32, device=a.device)
    check(lib().halo_rotate_quantize(_ptr(a), _dt(a), rows, cols, had_block if rotate else -1, fmt,
                                     _ptr(scale), _ptr(codes), _ptr(s_out), _stream()))
    return codes, s_out


def rotate_quantize_mx(a: torch.Tensor, had_block: int = 0, rotate: bool = True, transpose: bool = False):
    """``quantize([transform_right](a), mxfp6_e3m2, Granularity::mx())``:
    E3M2 codes (bits 7:2) and power-of-two scales per 1 x 32 block along rows
    (quantize.hpp:224-232), scales shaped [rows, ceil(cols/32)].  transpose:
    quantize ``a.T`` itself (halo_linear.hpp:427-431; no rotation)."""
    _need_cuda(a)
    a = a.contiguous()
    rows, cols = (a.shape[1], a.shape[0]) if transpose else a.shape
    codes = torch.empty((rows, cols), dtype=torch.uint8, device=a.device)
    scales = torch.empty((rows, (cols + 31) // 32), dtype=torch.float32, device=a.device)
    blk = -1 if (transpose or not rotate) else had_block
    check(lib().halo_rotate_quantize_mx(_ptr(a), _dt(a), rows, cols, blk, int(transpose), _ptr(codes), _ptr(scales),
                                        _stream()))
    return codes, scales


def rotate_quantize_rows(a: torch.Tensor, had_block: int = 0, fmt: int = INT8, rotate: bool = True):
    """``quantize(transform_right(a), fmt, Granularity::row())``: codes and one
    scale per row (``rows`` fp32).  cols must be a multiple of 256."""
    _need_cuda(a)
    rows, cols = a.shape
    codes = torch.empty((rows, cols), dtype=code_dtype(fmt), device=a.device)
    s_out = torch.empty(rows, dtype=torch.float32, device=a.device)
    check(lib().halo_rotate_quantize_rows(_ptr(a), _dt(a), rows, cols, had_block if rotate else -1, fmt, _ptr(codes),
                                          _ptr(s_out), _stream()))
    return codes, s_out


def qmatmul_scaled(a: torch.Tensor, b: torch.Tensor, scale_a: torch.Tensor, scale_b: torch.Tensor, *,
                   a_kmajor: bool = True, b_kmajor: bool = True, fmt: int = INT8, out: str = "f32") -> torch.Tensor:
    """qmatmul with per-row scales on the non-contracted dims: ``scale_a`` has 1
    or M entries (rows of C), ``scale_b`` 1 or N entries (columns of C)."""
    _need_cuda(a, b, scale_a, scale_b)
    M, K = a.shape if a_kmajor else a.shape[::-1]
    N, Kb = b.shape if b_kmajor else b.shape[::-1]
    if K != Kb:
        raise ValueError("qmatmul_scaled: inner dimensions disagree")
    kind = {"f32": OUT_F32, "bf16": OUT_BF16}[out]
    c = torch.empty((M, N), dtype=torch.float32 if kind == OUT_F32 else torch.bfloat16, device=a.device)
    check(lib().halo_qmatmul_scaled(fmt, _ptr(a), int(a_kmajor), _ptr(b), int(b_kmajor), M, N, K, _ptr(scale_a),
                                    int(scale_a.numel() > 1), _ptr(scale_b), int(scale_b.numel() > 1), _ptr(c), kind,
                                    _stream()))
    return c


def rotate_absmax(a: torch.Tensor, had_block: int = 0, rotate: bool = True) -> torch.Tensor:
    _need_cuda(a)
    out = torch.empty(1, dtype=torch.float32, device=a.device)
    check(lib().halo_rotate_absmax(_ptr(a), _dt(a), a.shape[0], a.shape[1], had_block if rotate else -1,
                                   _ptr(out), _stream()))
    return out


def left_rotate_quantize(e: torch.Tensor, had_block: int = 0, fmt: int = INT8, plain: bool = True):
    """HALO-2 error operands: ``(codes_rot[b_pad x n], scale_rot, codes_plain[b x n], scale_plain)``."""
    _need_cuda(e)
    b, n = e.shape
    bp = padded_batch(b, had_block)
    cr = torch.empty((bp, n), dtype=code_dtype(fmt), device=e.device)
    cp = torch.empty((b, n), dtype=code_dtype(fmt), device=e.device) if plain else None
    sr = torch.empty(1, dtype=torch.float32, device=e.device)
    sp = torch.empty(1, dtype=torch.float32, device=e.device)
    check(lib().halo_left_rotate_quantize(_ptr(e), _dt(e), b, n, had_block, fmt, _ptr(cr), _ptr(sr), _ptr(cp),
                                          _ptr(sp), _stream()))
    return cr, sr, cp, sp


def transform_right(a: torch.Tensor, had_block: int = 0, out_dtype=torch.float32) -> torch.Tensor:
    _need_cuda(a)
    if a.dtype != torch.float32:
        raise ValueError("transform_right takes fp32 input")
    out = torch.empty(a.shape, dtype=out_dtype, device=a.device)
    check(lib().halo_transform_right(_ptr(a), _ptr(out), _DT[out_dtype], a.shape[0], a.shape[1], had_block,
                                     _stream()))
    return out


def transform_left(a: torch.Tensor, had_block: int = 0, rows_out: int | None = None) -> torch.Tensor:
    _need_cuda(a)
    if a.dtype != torch.float32:
        raise ValueError("transform_left takes fp32 input")
    rows_pad, cols = a.shape
    rows_out = rows_pad if rows_out is None else rows_out
    out = torch.empty((rows_out, cols), dtype=torch.float32, device=a.device) if rows_out != rows_pad \
        else torch.empty_like(a)
    if rows_out != rows_pad:
        work = a.clone()
        check(lib().halo_transform_left(_ptr(work), _ptr(work), rows_pad, rows_out, cols, had_block, _stream()))
        out.copy_(work[:rows_out])
        return out
    check(lib().halo_transform_left(_ptr(a), _ptr(out), rows_pad, rows_out, cols, had_block, _stream()))
    return out


def qmatmul(a: torch.Tensor, b: torch.Tensor, scale_a: torch.Tensor, scale_b: torch.Tensor, *,
            a_kmajor: bool = True, b_kmajor: bool = True, fmt: int = INT8, out: str = "f32",
            had_block: int | None = None, transposed: bool = False, n_valid: int | None = None) -> torch.Tensor:
    """``qmatmul`` (quantize.hpp:339-380) on device codes; with ``had_block``
    the result is also right-transformed along N in the GEMM epilogue.

    A is ``[M, K]`` (a_kmajor) or ``[K, M]``; B is ``[N, K]`` (b_kmajor, the
    reference's transpose_b) or ``[K, N]``.  out: "f32", "bf16" or "s32"
    (raw int32 accumulators)."""
    _need_cuda(a, b, scale_a, scale_b)
    M, K = a.shape if a_kmajor else a.shape[::-1]
    N, Kb = b.shape if b_kmajor else b.shape[::-1]
    if K != Kb:
        raise ValueError("qmatmul: inner dimensions disagree")
    kind = {"f32": OUT_F32, "bf16": OUT_BF16, "s32": OUT_S32}[out]
    dt = {OUT_F32: torch.float32, OUT_BF16: torch.bfloat16, OUT_S32: torch.int32}[kind]
    if had_block is None:
        c = torch.empty((M, N), dtype=dt, device=a.device)
        check(lib().halo_qmatmul(fmt, _ptr(a), int(a_kmajor), _ptr(b), int(b_kmajor), M, N, K, _ptr(scale_a),
                                 _ptr(scale_b), _ptr(c), kind, _stream()))
        return c
    # qmatmul -> transform_right along N, fused in the GEMM epilogue;
    # transposed: C^T[:n_valid] (the HALO-2 error path's layout)
    nv = N if n_valid is None else n_valid
    c = torch.empty((nv, M) if transposed else (M, N), dtype=dt, device=a.device)
    check(lib().halo_qmatmul_rotate(fmt, _ptr(a), int(a_kmajor), _ptr(b), int(b_kmajor), M, N, K, _ptr(scale_a),
                                    _ptr(scale_b), _ptr(c), kind, had_block, int(transposed), nv, _stream()))
    return c


def allow_dequantized_products(on: bool = True):
    """Opt in to row / column granularity layers, whose contracted-dim scales
    make the reference multiply dequantized values in double
    (quantize.hpp:377-379): served bit-exactly on the FP64 pipe (deq_gemm),
    off the tensor-core path.  Process-wide; off by default."""
    check(lib().halo_allow_dequantized_products(1 if on else 0))


# ------------------------------------------------------ FP6 wire format

def fp6_pack(codes: torch.Tensor) -> torch.Tensor:
    """Device E3M2 codes (bits 7:2 of a byte each) -> the packed FP6 payload
    (3 bytes per 4 codes, hqfsdp.hpp:36-49), uint8 [numel * 3/4]."""
    _need_cuda(codes)
    c = codes.contiguous().view(torch.uint8).reshape(-1)
    out = torch.empty(c.numel() // 4 * 3, dtype=torch.uint8, device=c.device)
    check(lib().halo_fp6_pack(_ptr(c), _ptr(out), c.numel(), _stream()))
    return out


def fp6_unpack(packed: torch.Tensor, n: int) -> torch.Tensor:
    """The packed FP6 payload -> n device codes (uint8, E3M2 in bits 7:2)."""
    _need_cuda(packed)
    out = torch.empty(n, dtype=torch.uint8, device=packed.device)
    check(lib().halo_fp6_unpack(_ptr(packed.contiguous()), _ptr(out), n, _stream()))
    return out


# ------------------------------------------------------ quantized tensor files

def write_quantized_tensor(path: str, codes: torch.Tensor, scales: torch.Tensor, fmt: int = INT8,
                           granularity: int = GRAN_TENSOR):
    """write_quantized_tensor (quantize.hpp:405-430): the reference's HALT
    file of device codes (any device; copied to the host) and their scales."""
    c = codes.detach().contiguous().cpu()
    sc = scales.detach().float().contiguous().cpu()
    rows, cols = c.shape
    check(lib().halo_quantized_tensor_write(str(path).encode(), fmt, granularity, rows, cols, c.data_ptr(),
                                            sc.data_ptr(), sc.numel()))


def read_quantized_tensor(path: str, device=None):
    """read_quantized_tensor (quantize.hpp:432-474) -> (codes, scales, fmt,
    granularity) in the device code layout (on `device` if given)."""
    f, g = C.c_int32(), C.c_int32()
    r, c, n = C.c_int64(), C.c_int64(), C.c_int64()
    p = str(path).encode()
    check(lib().halo_quantized_tensor_info(p, C.byref(f), C.byref(g), C.byref(r), C.byref(c), C.byref(n)))
    fmt = f.value
    if fmt not in (INT8, FP8_E4M3, FP6_E3M2):
        raise _lib.HaloIOError("read_quantized_tensor: format has no device code layout")
    codes = torch.empty((r.value, c.value), dtype=code_dtype(fmt))
    scales = torch.empty(n.value, dtype=torch.float32)
    check(lib().halo_quantized_tensor_read(p, codes.data_ptr(), scales.data_ptr()))
    if device is not None:
        codes, scales = codes.to(device), scales.to(device)
    return codes, scales, fmt, g.value


# -------------------------------------------------------------------- layer

class SavedContext:
    """SavedContextT (halo_linear.hpp:207-216): owns (XH)_Q, (WH)_Q and scales
    in device memory.  No full-precision copy of X is kept."""

    def __init__(self):
        h = C.c_void_p()
        check(lib().halo_ctx_create(C.byref(h)))
        self._h = h

    def __del__(self):
        h = getattr(self, "_h", None)
        try:
            if h and _lib._lib is not None:
                _lib._lib.halo_ctx_destroy(h)
        except Exception:  # interpreter shutdown
            pass
        self._h = None

    def saved(self, layer: "HaloLinearLayer"):
        """Views of (xq, sx, wq, sw) as torch tensors (copies)."""
        xq, sx, wq, sw = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        b = C.c_int64()
        check(lib().halo_ctx_saved(self._h, C.byref(xq), C.byref(sx), C.byref(wq), C.byref(sw), C.byref(b)))
        dt = code_dtype(layer.fmt)
        g = layer.scheme.granularity
        nb = (layer.in_features + 31) // 32
        nsx = b.value if g == GRAN_ROW else layer.in_features if g == GRAN_COLUMN else b.value * nb if g == GRAN_MX else 1
        nsw = (layer.out_features if g == GRAN_ROW else layer.in_features if g == GRAN_COLUMN
               else layer.out_features * nb if g == GRAN_MX else 1)
        return (_from_ptr(xq.value, (b.value, layer.in_features), dt),
                _from_ptr(sx.value, (nsx,), torch.float32),
                _from_ptr(wq.value, (layer.out_features, layer.in_features), dt),
                _from_ptr(sw.value, (nsw,), torch.float32))

    def error_operands(self, layer: "HaloLinearLayer"):
        ehq, seh, eq, se = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        bp = C.c_int64()
        check(lib().halo_ctx_error_operands(self._h, C.byref(ehq), C.byref(seh), C.byref(eq), C.byref(se),
                                            C.byref(bp)))
        dt = code_dtype(layer.fmt)
        b = layer._last_b
        g = layer.scheme.granularity
        # scale vectors: per token (ROW), per output column (COLUMN), else one
        n_se = b if g == GRAN_ROW else layer.out_features if g == GRAN_COLUMN else 1
        n_seh = bp.value if g == GRAN_ROW else layer.out_features if g == GRAN_COLUMN else 1
        out = {"eq": _from_ptr(eq.value, (b, layer.out_features), dt),
               "se": _from_ptr(se.value, (n_se,), torch.float32)}
        if layer.scheme.E.left:
            out["ehq"] = _from_ptr(ehq.value, (bp.value, layer.out_features), dt)
            out["seh"] = _from_ptr(seh.value, (n_seh,), torch.float32)
        return out

    def share_scratch(self, owner: "SavedContext | None"):
        """Use `owner`'s backward scratch (halo_ctx_share_scratch): contexts
        whose backwards run one after another share one set of buffers."""
        check(lib().halo_ctx_share_scratch(self._h, owner._h if owner is not None else None))
        self._scratch_owner = owner  # keep it alive

    def check(self):
        """Synchronise and raise HaloNumericError for non-finite inputs."""
        check(lib().halo_ctx_check(self._h, _stream()))


def _from_ptr(ptr, shape, dtype):
    """Copy `numel` elements at a device address into a fresh tensor."""
    numel = 1
    for s in shape:
        numel *= s
    out = torch.empty(shape, dtype=dtype, device="cuda")
    check(lib().halo_device_copy(_ptr(out), C.c_void_p(ptr), numel * out.element_size(), _stream()))
    return out


@dataclass
class BackwardResult:
    """BackwardResultT (halo_linear.hpp:220-225)."""
    e_x: torch.Tensor
    grad_w: torch.Tensor | None


class HaloLinearLayer:
    """HaloLinearLayerT (halo_linear.hpp:227-462) on the B200.

    ``w`` is the (out x in) weight, bf16 or fp32, on a CUDA device; the layer
    keeps a reference (not a copy) and re-rotates/re-quantizes it at every
    forward, as the reference does (:295-297).  Errors mirror the
    reference: ValueError for std::invalid_argument, HaloNumericError for
    numeric_error."""

    def __init__(self, w: torch.Tensor, scheme: Scheme, out_dtype=torch.bfloat16, grad_dtype=torch.float32):
        _need_cuda(w)
        self.w = w
        self.scheme = scheme
        self.fmt = scheme.format_x
        self.out_dtype = out_dtype
        self.grad_dtype = grad_dtype
        self._last_b = 0
        h = C.c_void_p()
        check(lib().halo_linear_create(C.byref(scheme), _ptr(w), _dt(w), w.shape[0], w.shape[1], C.byref(h)))
        self._h = h
        self._qweight = None

    def __del__(self):
        h = getattr(self, "_h", None)
        try:
            if h and _lib._lib is not None:
                _lib._lib.halo_linear_destroy(h)
        except Exception:  # interpreter shutdown
            pass
        self._h = None

    @property
    def in_features(self):
        return self.w.shape[1]

    @property
    def out_features(self):
        return self.w.shape[0]

    def set_weight(self, w: torch.Tensor):
        _need_cuda(w)
        if tuple(w.shape) != (self.out_features, self.in_features):
            raise ValueError("halo layer: weight shape mismatch")
        self.w = w
        check(lib().halo_linear_set_weight(self._h, _ptr(w), _dt(w)))

    def set_qweight(self, codes: torch.Tensor | None, scale: torch.Tensor | None):
        """Use gathered / frozen (WH)_Q codes instead of quantizing W."""
        if codes is not None:
            _need_cuda(codes, scale)
        self._qweight = (codes, scale)
        check(lib().halo_linear_set_qweight(self._h, _ptr(codes), _ptr(scale)))

    def set_qweight_sharded(self, parts, scale: torch.Tensor | None, keepalive=None):
        """(WH)_Q as row shards read in place by the GEMMs (HQ-FSDP without
        the all-gather): `parts` are device addresses (ints, e.g. local or
        IPC-opened peer buffers) or tensors of out_features/len(parts) rows
        each.  None reverts."""
        if parts is None:
            self._qweight = (None, None)
            check(lib().halo_linear_set_qweight_sharded(self._h, None, 0, None))
            return
        ptrs = [p.data_ptr() if isinstance(p, torch.Tensor) else int(p) for p in parts]
        arr = (C.c_void_p * len(ptrs))(*ptrs)
        self._qweight = (tuple(parts), scale, keepalive)
        check(lib().halo_linear_set_qweight_sharded(self._h, arr, len(ptrs), _ptr(scale)))

    def set_grad_scatter(self, recv, rank: int):
        """Fuse the HQ-FSDP gradient reduce-scatter into the G GEMM: `recv`
        are the ranks' receive-buffer addresses ([world][rows/world][in]
        fp32 each); backward then returns grad_w None and stores this rank's
        fp32 partial rows into their owners' slots.  None reverts."""
        if recv is None:
            self._scatter = None
            check(lib().halo_linear_set_grad_scatter(self._h, None, 0, 0))
            return
        arr = (C.c_void_p * len(recv))(*[int(r) for r in recv])
        check(lib().halo_linear_set_grad_scatter(self._h, arr, len(recv), rank))
        self._scatter = tuple(recv)

    def forward(self, x: torch.Tensor, ctx: SavedContext) -> torch.Tensor:
        _need_cuda(x)
        if x.dim() != 2 or x.shape[1] != self.in_features:
            raise ValueError("halo layer: input feature dim mismatch")
        b = x.shape[0]
        y = torch.empty((b, self.out_features), dtype=self.out_dtype, device=x.device)
        check(lib().halo_linear_forward(self._h, _ptr(x), _dt(x), b, _ptr(y), _DT[self.out_dtype], ctx._h,
                                        _stream()))
        self._last_b = b
        ctx._layer_b = b
        return y

    def forward_residual(self, x: torch.Tensor, ctx: SavedContext, res: torch.Tensor) -> torch.Tensor:
        """res + forward(x) with the add in the GEMM epilogue (bf16 output,
        out_features % 256 == 0): identical to ``res + self.forward(x, ctx)``
        for a bf16 layer."""
        _need_cuda(x)
        if x.dim() != 2 or x.shape[1] != self.in_features:
            raise ValueError("halo layer: input feature dim mismatch")
        b = x.shape[0]
        if res.dtype != torch.bfloat16 or tuple(res.shape) != (b, self.out_features) or not res.is_contiguous():
            raise ValueError("forward_residual: res must be a contiguous bf16 (b x out_features) tensor")
        y = torch.empty((b, self.out_features), dtype=torch.bfloat16, device=x.device)
        check(lib().halo_linear_forward_residual(self._h, _ptr(x), _dt(x), b, _ptr(res), _ptr(y), ctx._h, _stream()))
        self._last_b = b
        ctx._layer_b = b
        return y

    def forward_shared(self, src: SavedContext, ctx: SavedContext) -> torch.Tensor:
        """forward() on the X already quantized in ``src`` (another layer's
        context with the same in_features and X quantizer): the gate/up pattern
        of a Llama MLP quantizes X once.  Identical results to forward(x)."""
        b = src._layer_b
        y = torch.empty((b, self.out_features), dtype=self.out_dtype, device=self.w.device)
        check(lib().halo_linear_forward_shared(self._h, src._h, ctx._h, _ptr(y), _DT[self.out_dtype], _stream()))
        self._last_b = b
        ctx._layer_b = b
        ctx._shared_src = src  # keep the borrowed codes alive
        return y

    def forward_shared_swiglu(self, src: SavedContext, ctx: SavedContext, g: torch.Tensor):
        """forward_shared() of the up projection with the SwiGLU product in
        the GEMM epilogue: returns (u, h = silu(g) * u), both bf16, h
        identical to halo_swiglu_forward(g, u).  out_features % 256 == 0."""
        b = src._layer_b
        if g.dtype != torch.bfloat16 or tuple(g.shape) != (b, self.out_features) or not g.is_contiguous():
            raise ValueError("forward_shared_swiglu: g must be a contiguous bf16 (b x out_features) tensor")
        u = torch.empty((b, self.out_features), dtype=torch.bfloat16, device=self.w.device)
        h = torch.empty_like(u)
        check(lib().halo_linear_forward_shared_swiglu(self._h, src._h, ctx._h, _ptr(g), _ptr(u), _ptr(h), _stream()))
        self._last_b = b
        ctx._layer_b = b
        ctx._shared_src = src
        return u, h

    def backward(self, ctx: SavedContext, e_y: torch.Tensor, need_grad_w: bool = True,
                 e_x_dtype=None, e_x_add: torch.Tensor = None) -> BackwardResult:
        """e_x_add (bf16, b x in_features): return e_x_add + E_X instead of
        E_X (halo_linear_backward_acc: the add fused into the K4 store)."""
        _need_cuda(e_y)
        b = getattr(ctx, "_layer_b", None)
        if b is None:
            raise ValueError("halo layer: backward without forward context")
        if e_y.dim() != 2 or e_y.shape[0] != b or e_y.shape[1] != self.out_features:
            raise ValueError("halo layer: upstream error shape mismatch")
        ex_dt = e_x_dtype or self.out_dtype
        e_x = torch.empty((b, self.in_features), dtype=ex_dt, device=e_y.device)
        scatter = getattr(self, "_scatter", None) is not None
        g = torch.empty((self.out_features, self.in_features), dtype=self.grad_dtype, device=e_y.device) \
            if need_grad_w and not scatter else None
        if e_x_add is not None:
            if e_x_add.dtype != torch.bfloat16 or tuple(e_x_add.shape) != (b, self.in_features) or \
                    not e_x_add.is_contiguous() or ex_dt != torch.bfloat16:
                raise ValueError("backward: e_x_add must be a contiguous bf16 (b x in_features) tensor, e_x bf16")
            check(lib().halo_linear_backward_acc(self._h, ctx._h, _ptr(e_y), _dt(e_y), _ptr(e_x_add), _ptr(e_x),
                                                 _DT[ex_dt], _ptr(g), _DT[self.grad_dtype], _stream()))
        else:
            check(lib().halo_linear_backward(self._h, ctx._h, _ptr(e_y), _dt(e_y), _ptr(e_x), _DT[ex_dt], _ptr(g),
                                             _DT[self.grad_dtype], _stream()))
        return BackwardResult(e_x, g)

    def export_inference_weights(self, path: str | None = None):
        """(WH)_Q codes and scale (halo_linear.hpp:332-338); with `path`, also
        written as the reference's quantized tensor file (quantize.hpp:405-430)."""
        codes = torch.empty((self.out_features, self.in_features), dtype=code_dtype(self.fmt), device=self.w.device)
        rows = self.scheme.granularity == GRAN_ROW
        scale = torch.empty(self.out_features if rows else 1, dtype=torch.float32, device=self.w.device)
        check(lib().halo_linear_export_inference_weights(self._h, _ptr(codes), _ptr(scale), _stream()))
        if path is not None:
            write_quantized_tensor(path, codes, scale, self.fmt, GRAN_ROW if rows else GRAN_TENSOR)
        return codes, scale

    def counters(self) -> Counters:
        c = Counters()
        check(lib().halo_linear_counters(self._h, C.byref(c)))
        return c

    def reset_counters(self):
        check(lib().halo_linear_reset_counters(self._h))


class PeftHaloLinear:
    """HaloLinearLayerT's PEFT form (halo_linear.hpp:236-250, 272-283, 311-319,
    441-455): W is frozen and quantized once, (WH)_Q at construction; the
    forward is ``(XH)_Q (WH)_Q^T + (X U^T) V^T`` and the backward
    ``E_X = H_b (H_b^T E_Y)_Q (WH)_Q H_m^T + (E_Y V) U`` with the LoRA
    gradients ``grad_V = E_Y^T (X U^T)``, ``grad_U = (E_Y V)^T X``.  The
    quantized products run on the device path (scheme "halo-peft": F:M, E:LR);
    the rank-r LoRA products are plain working-precision matmuls (torch /
    cuBLAS), as the reference computes them in double."""

    def __init__(self, w: torch.Tensor, u: torch.Tensor, v: torch.Tensor, fmt: int = INT8, had_block: int = 0,
                 out_dtype=torch.bfloat16):
        if u.shape[1] != w.shape[1] or v.shape[0] != w.shape[0] or u.shape[0] != v.shape[1]:
            raise ValueError("halo layer: U/V shapes must be r x m and n x r")
        self.layer = HaloLinearLayer(w, scheme_from_string("halo-peft", fmt, had_block), out_dtype=out_dtype)
        self.u, self.v = u, v
        self.out_dtype = out_dtype

    @property
    def lora_rank(self):
        return self.u.shape[0]

    def forward(self, x: torch.Tensor, ctx: SavedContext) -> torch.Tensor:
        y = self.layer.forward(x, ctx)
        ctx._peft_x = x  # SavedContextT keeps x for the LoRA gradients (:271)
        if self.lora_rank > 0:
            y = (y.float() + (x.float() @ self.u.float().t()) @ self.v.float().t()).to(self.out_dtype)
        return y

    def backward(self, ctx: SavedContext, e_y: torch.Tensor):
        """Returns (e_x, grad_u, grad_v)."""
        e_x = self.layer.backward(ctx, e_y, need_grad_w=False).e_x
        x = ctx._peft_x.float()
        ey = e_y.float()
        ev = ey @ self.v.float()  # b x r
        if self.lora_rank > 0:
            e_x = (e_x.float() + ev @ self.u.float()).to(e_x.dtype)
        grad_v = ey.t() @ (x @ self.u.float().t())
        grad_u = ev.t() @ x
        return e_x, grad_u, grad_v

    def export_inference_weights(self):
        return self.layer.export_inference_weights()

    def counters(self) -> Counters:
        return self.layer.counters()
