"""ctypes binding of libhalo_b200.so (include/halo_b200.h).

The shared library is built in-tree (``make -C paper_2501_02625_b200``) and is
the only compute path: there is no CPU or PyTorch fallback.  Importing this
module on a machine where the library is missing raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# HALO_B200_LIB: an alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("HALO_B200_LIB") or os.path.join(HERE, "libhalo_b200.so")

HALO_OK = 0
HALO_ERR_INVALID_ARGUMENT = 1
HALO_ERR_NUMERIC = 2
HALO_ERR_LOGIC = 3
HALO_ERR_CUDA = 4
HALO_ERR_NCCL = 5
HALO_ERR_IO = 6

FMT_INT8 = 0
FMT_FP8_E4M3 = 1
FMT_FP6_E3M2 = 2  # one E3M2 code per byte, in bits 7:2 (the tcgen05 kind::f8f6f4 operand form)
FMT_MXFP6_E3M2 = 3  # E3M2 codes as FP6, power-of-two scale (quantize.hpp:224-232)
DTYPE_F32 = 0
DTYPE_BF16 = 1
OUT_F32, OUT_BF16, OUT_S32 = 0, 1, 2


class HaloNumericError(ArithmeticError):
    """numeric_error (tensor.hpp:22-24): a non-finite value reached a quantizer."""


class HaloLogicError(RuntimeError):
    """std::logic_error (hqfsdp.hpp:246-259: missing / stale scales)."""


class HaloIOError(RuntimeError):
    """io_error (tensor_io.hpp:25-27): tensor file open / format / truncation."""


class HaloNcclError(RuntimeError):
    """A failed NCCL call of the HQ-FSDP data plane."""


class HaloCudaError(RuntimeError):
    pass


class Placement(C.Structure):
    _fields_ = [("left", C.c_uint8), ("middle", C.c_uint8), ("right", C.c_uint8), ("pad_", C.c_uint8)]

    def __str__(self):  # halo_linear.hpp:38-47
        s = ("L" if self.left else "") + ("M" if self.middle else "") + ("R" if self.right else "")
        return s or "O"


class Scheme(C.Structure):
    _fields_ = [
        ("F", Placement), ("E", Placement), ("G", Placement),
        ("format_x", C.c_int32), ("format_w", C.c_int32), ("format_e", C.c_int32),
        ("granularity", C.c_int32),
        ("quantize_f", C.c_int32), ("quantize_e", C.c_int32), ("quantize_g", C.c_int32),
        ("peft", C.c_int32),
        ("had_block", C.c_int64),
        ("name", C.c_char * 16),
    ]

    def __str__(self):  # halo_linear.hpp:154-159
        if self.name:
            return self.name.decode()
        return f"F:{self.F};E:{self.E};G:{self.G}"


class Counters(C.Structure):
    _fields_ = [("x", C.c_int64), ("w", C.c_int64), ("e", C.c_int64)]


PROFILE_CLASSES = ("k1_rows_fwht_quant", "k2_cols_fwht_quant", "k3_gemm", "k4_unrotate", "glue")


class Profile(C.Structure):
    _fields_ = [("launches", C.c_int64 * 5), ("ms", C.c_double * 5), ("work", C.c_double * 5)]

    def as_dict(self):
        return {name: {"launches": int(self.launches[i]), "ms": float(self.ms[i]), "work": float(self.work[i])}
                for i, name in enumerate(PROFILE_CLASSES)}


_lib = None

_vp = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C {HERE}` (or __graft_entry__.build()); "
            "there is no CPU fallback for the HALO device path")
    L = C.CDLL(LIB_PATH)
    L.halo_abi_version.restype = C.c_int
    L.halo_last_error.restype = C.c_char_p
    L.halo_is_supported_hadamard_dim.argtypes = [_i64]
    L.halo_next_supported_hadamard_dim.argtypes = [_i64]
    L.halo_next_supported_hadamard_dim.restype = _i64
    L.halo_padded_batch.argtypes = [_i64, _i64]
    L.halo_padded_batch.restype = _i64
    L.halo_scheme_from_string.argtypes = [C.c_char_p, _i32, _i64, C.POINTER(Scheme)]
    L.halo_rotate_quantize.argtypes = [_vp, _i32, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _vp]
    L.halo_rotate_absmax.argtypes = [_vp, _i32, _i64, _i64, _i64, _vp, _vp]
    L.halo_left_rotate_quantize.argtypes = [_vp, _i32, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _vp]
    L.halo_transform_right.argtypes = [_vp, _vp, _i32, _i64, _i64, _i64, _vp]
    L.halo_transform_left.argtypes = [_vp, _vp, _i64, _i64, _i64, _i64, _vp]
    L.halo_qmatmul.argtypes = [_i32, _vp, _i32, _vp, _i32, _i64, _i64, _i64, _vp, _vp, _vp, _i32, _vp]
    L.halo_qmatmul_rotate.argtypes = [_i32, _vp, _i32, _vp, _i32, _i64, _i64, _i64, _vp, _vp, _vp, _i32, _i64, _i32,
                                      _i64, _vp]
    L.halo_rotate_quantize_rows.argtypes = [_vp, _i32, _i64, _i64, _i64, _i32, _vp, _vp, _vp]
    L.halo_qmatmul_scaled.argtypes = [_i32, _vp, _i32, _vp, _i32, _i64, _i64, _i64, _vp, _i32, _vp, _i32, _vp, _i32,
                                      _vp]
    L.halo_linear_forward_shared.argtypes = [_vp, _vp, _vp, _vp, _i32, _vp]
    L.halo_linear_forward_shared_swiglu.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp]
    L.halo_linear_forward_shared_swiglu.restype = C.c_int
    L.halo_linear_forward_residual.argtypes = [_vp, _vp, _i32, _i64, _vp, _vp, _vp, _vp]
    L.halo_linear_forward_residual.restype = C.c_int
    L.halo_linear_backward_acc.argtypes = [_vp, _vp, _vp, _i32, _vp, _vp, _i32, _vp, _i32, _vp]
    L.halo_linear_backward_acc.restype = C.c_int
    L.halo_linear_create.argtypes = [C.POINTER(Scheme), _vp, _i32, _i64, _i64, C.POINTER(_vp)]
    L.halo_linear_destroy.argtypes = [_vp]
    L.halo_linear_set_weight.argtypes = [_vp, _vp, _i32]
    L.halo_linear_set_qweight.argtypes = [_vp, _vp, _vp]
    L.halo_ctx_create.argtypes = [C.POINTER(_vp)]
    L.halo_ctx_destroy.argtypes = [_vp]
    L.halo_linear_forward.argtypes = [_vp, _vp, _i32, _i64, _vp, _i32, _vp, _vp]
    L.halo_linear_backward.argtypes = [_vp, _vp, _vp, _i32, _vp, _i32, _vp, _i32, _vp]
    L.halo_linear_export_inference_weights.argtypes = [_vp, _vp, _vp, _vp]
    L.halo_linear_counters.argtypes = [_vp, C.POINTER(Counters)]
    L.halo_linear_reset_counters.argtypes = [_vp]
    L.halo_ctx_saved.argtypes = [_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp),
                                 C.POINTER(_i64)]
    L.halo_ctx_error_operands.argtypes = [_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp),
                                          C.POINTER(_vp), C.POINTER(_i64)]
    L.halo_ctx_check.argtypes = [_vp, _vp]
    L.halo_device_copy.argtypes = [_vp, _vp, _i64, _vp]
    L.halo_swiglu_forward.argtypes = [_vp, _vp, _vp, _i64, _vp]
    L.halo_swiglu_backward.argtypes = [_vp, _vp, _vp, _vp, _vp, _i64, _vp]
    L.halo_swiglu_backward_absmax.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp]
    L.halo_swiglu_forward_absmax.argtypes = [_vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp]
    L.halo_swiglu_forward_absmax.restype = C.c_int
    L.halo_add.argtypes = [_vp, _vp, _vp, _i32, _i64, _vp]
    L.halo_linear_set_qweight_sharded.argtypes = [_vp, C.POINTER(_vp), _i32, _vp]
    L.halo_peer_alloc.argtypes = [_i64, C.POINTER(_vp)]
    L.halo_peer_free.argtypes = [_vp]
    L.halo_ipc_handle.argtypes = [_vp, C.c_char_p]
    L.halo_ipc_open.argtypes = [C.c_char_p, C.POINTER(_vp)]
    L.halo_ipc_close.argtypes = [_vp]
    L.halo_peer_sync.argtypes = [C.POINTER(_vp), _i32, _i32, C.c_uint32, _vp, _vp, _vp]
    L.halo_linear_set_grad_scatter.argtypes = [_vp, C.POINTER(_vp), _i32, _i32]
    L.halo_rotate_quantize_amax.argtypes = [_vp, _i32, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _vp]
    L.halo_rotate_quantize_amax.restype = C.c_int
    L.halo_reduce_scatter_shard.argtypes = [_vp, _i32, _i64, _i64, _vp, _i32, _vp]
    for fn in ("halo_linear_set_qweight_sharded", "halo_peer_alloc", "halo_peer_free", "halo_ipc_handle",
               "halo_ipc_open", "halo_ipc_close", "halo_peer_sync", "halo_linear_set_grad_scatter",
               "halo_reduce_scatter_shard"):
        getattr(L, fn).restype = C.c_int
    L.halo_adamw_step.argtypes = [_vp, _i32, _vp, _i32, _vp, _vp, _i64] + [C.c_double] * 7 + [_vp]
    L.halo_adamw_step.restype = C.c_int
    L.halo_rmsnorm_forward.argtypes = [_vp, _vp, _vp, _i32, _vp, _i64, _i64, _i32, C.c_double, _vp]
    L.halo_rmsnorm_backward.argtypes = [_vp, _vp, _i32, _vp, _vp, _vp, _vp, _i64, _i64, _i32, _vp]
    L.halo_add_rmsnorm_forward.argtypes = [_vp, _vp, _vp, _vp, _vp, _vp, _i64, _i64, C.c_double, _vp]
    L.halo_rmsnorm_backward_res.argtypes = [_vp, _vp, _i32, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _vp]
    L.halo_rope_qkv.argtypes = [_vp, _vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32, _vp]
    for fn in ("halo_rmsnorm_forward", "halo_rmsnorm_backward", "halo_rope_qkv", "halo_add_rmsnorm_forward",
               "halo_rmsnorm_backward_res"):
        getattr(L, fn).restype = C.c_int
    L.halo_rotate_quantize_mx.argtypes = [_vp, _i32, _i64, _i64, _i64, _i32, _vp, _vp, _vp]
    L.halo_rotate_quantize_mx.restype = C.c_int
    L.halo_ctx_share_scratch.argtypes = [_vp, _vp]
    L.halo_ctx_share_scratch.restype = C.c_int
    L.halo_allow_dequantized_products.argtypes = [_i32]
    L.halo_allow_dequantized_products.restype = C.c_int
    L.halo_fp6_pack.argtypes = [_vp, _vp, _i64, _vp]
    L.halo_fp6_unpack.argtypes = [_vp, _vp, _i64, _vp]
    L.halo_fp6_pack.restype = C.c_int
    L.halo_fp6_unpack.restype = C.c_int
    L.halo_fsdp_get_unique_id.argtypes = [_vp]
    L.halo_fsdp_create.argtypes = [_vp, _i32, _i32, C.POINTER(_vp)]
    L.halo_fsdp_destroy.argtypes = [_vp]
    L.halo_fsdp_world.argtypes = [_vp, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]
    L.halo_fsdp_quantized_all_gather.argtypes = [_vp, _vp, _i32, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _vp]
    L.halo_fsdp_backward_regather.argtypes = [_vp, _vp, _i32, _i64, _i64, _i64, _i32, _vp, _vp, _vp, _vp, _vp]
    L.halo_fsdp_reduce_scatter.argtypes = [_vp, _vp, _i32, _i64, _i64, _vp, _vp]
    L.halo_fsdp_all_reduce_mean.argtypes = [_vp, _vp, _i32, _i64, _vp]
    for fn in ("halo_fsdp_get_unique_id", "halo_fsdp_create", "halo_fsdp_destroy", "halo_fsdp_world",
               "halo_fsdp_quantized_all_gather", "halo_fsdp_backward_regather", "halo_fsdp_reduce_scatter",
               "halo_fsdp_all_reduce_mean"):
        getattr(L, fn).restype = C.c_int
    L.halo_quantized_tensor_write.argtypes = [C.c_char_p, _i32, _i32, _i64, _i64, _vp, _vp, _i64]
    L.halo_quantized_tensor_info.argtypes = [C.c_char_p] + [C.POINTER(C.c_int32)] * 2 + [C.POINTER(_i64)] * 3
    L.halo_quantized_tensor_read.argtypes = [C.c_char_p, _vp, _vp]
    for fn in ("halo_quantized_tensor_write", "halo_quantized_tensor_info", "halo_quantized_tensor_read"):
        getattr(L, fn).restype = C.c_int
    L.halo_profile_enable.argtypes = [C.c_int]
    L.halo_profile_read.argtypes = [C.POINTER(Profile)]
    for fn in ("halo_swiglu_forward", "halo_swiglu_backward", "halo_swiglu_backward_absmax", "halo_add", "halo_profile_enable",
               "halo_profile_read"):
        getattr(L, fn).restype = C.c_int
    for fn in ("halo_scheme_from_string", "halo_rotate_quantize", "halo_rotate_absmax",
               "halo_left_rotate_quantize", "halo_transform_right", "halo_transform_left",
               "halo_qmatmul", "halo_qmatmul_rotate", "halo_rotate_quantize_rows", "halo_qmatmul_scaled",
               "halo_linear_forward_shared", "halo_linear_create", "halo_linear_destroy", "halo_linear_set_weight", "halo_linear_set_qweight", "halo_ctx_create", "halo_ctx_destroy", "halo_linear_forward",
               "halo_linear_backward", "halo_linear_export_inference_weights", "halo_linear_counters",
               "halo_linear_reset_counters", "halo_ctx_saved", "halo_ctx_error_operands",
               "halo_ctx_check", "halo_device_copy"):
        getattr(L, fn).restype = C.c_int
    if L.halo_abi_version() != 1:
        raise ImportError("libhalo_b200.so ABI version mismatch")
    _lib = L
    return L


def check(rc: int):
    """Map halo_status to the reference's exception classes."""
    if rc == HALO_OK:
        return
    msg = lib().halo_last_error().decode(errors="replace")
    if rc == HALO_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == HALO_ERR_NUMERIC:
        raise HaloNumericError(msg)
    if rc == HALO_ERR_IO:
        raise HaloIOError(msg)
    if rc == HALO_ERR_NCCL:
        raise HaloNcclError(msg)
    if rc == HALO_ERR_LOGIC:
        raise HaloLogicError(msg)
    raise HaloCudaError(msg)


# Every exported symbol declared in include/halo_b200.h (checked by tests).
EXPORTS = (
    "halo_abi_version", "halo_last_error", "halo_is_supported_hadamard_dim",
    "halo_next_supported_hadamard_dim", "halo_scheme_from_string", "halo_rotate_quantize",
    "halo_rotate_absmax", "halo_left_rotate_quantize", "halo_padded_batch", "halo_transform_right",
    "halo_transform_left", "halo_qmatmul", "halo_qmatmul_rotate", "halo_rotate_quantize_rows",
    "halo_qmatmul_scaled", "halo_linear_forward_shared", "halo_linear_forward_shared_swiglu",
    "halo_linear_forward_residual", "halo_linear_backward_acc",
    "halo_linear_create", "halo_linear_destroy",
    "halo_linear_set_weight", "halo_linear_set_qweight", "halo_ctx_create", "halo_ctx_destroy",
    "halo_linear_forward", "halo_linear_backward", "halo_linear_export_inference_weights",
    "halo_linear_counters", "halo_linear_reset_counters", "halo_ctx_saved",
    "halo_ctx_error_operands", "halo_ctx_check", "halo_device_copy", "halo_swiglu_forward",
    "halo_swiglu_backward", "halo_swiglu_backward_absmax", "halo_add", "halo_profile_enable",
    "halo_profile_read", "halo_linear_set_qweight_sharded", "halo_peer_alloc", "halo_peer_free",
    "halo_ipc_handle", "halo_ipc_open", "halo_ipc_close", "halo_peer_sync", "halo_linear_set_grad_scatter",
    "halo_reduce_scatter_shard", "halo_rotate_quantize_amax", "halo_swiglu_forward_absmax",
    "halo_adamw_step", "halo_rmsnorm_forward", "halo_rmsnorm_backward", "halo_rope_qkv",
    "halo_add_rmsnorm_forward", "halo_rmsnorm_backward_res", "halo_quantized_tensor_write", "halo_quantized_tensor_info", "halo_quantized_tensor_read",
    "halo_fsdp_get_unique_id", "halo_fsdp_create", "halo_fsdp_destroy", "halo_fsdp_world",
    "halo_fsdp_quantized_all_gather", "halo_fsdp_backward_regather", "halo_fsdp_reduce_scatter",
    "halo_fsdp_all_reduce_mean", "halo_fp6_pack", "halo_fp6_unpack",
    "halo_allow_dequantized_products", "halo_rotate_quantize_mx", "halo_ctx_share_scratch",
)
