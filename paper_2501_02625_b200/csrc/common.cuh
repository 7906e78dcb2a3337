// common.cuh — shared device helpers (sm_100a only).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "quant_round.cuh"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "paper_2501_02625_b200 targets sm_100a only"
#endif

namespace halo_b200 {

enum Fmt : int { FMT_INT8 = 0, FMT_E4M3 = 1, FMT_E3M2 = 2 };
enum DType : int { DT_F32 = 0, DT_BF16 = 1 };

// error flag bits written by kernels into the per-call status word
enum : unsigned { ERRF_NONFINITE = 1u };

struct DevFlags {
    unsigned* err;  // device word, OR-ed by kernels
};

__device__ __forceinline__ float load_elem(const float* p) { return *p; }
__device__ __forceinline__ float load_elem(const __nv_bfloat16* p) { return __bfloat162float(*p); }

// 8 consecutive elements -> fp32 registers (16 B for bf16, 32 B for fp32)
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float v[8]) {
    const uint4 r = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        v[2 * i] = __uint_as_float(w[i] << 16);
        v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
}
__device__ __forceinline__ void load8(const float* p, float v[8]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

__device__ __forceinline__ void store8(float* p, const float v[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float v[8]) {
    uint4 r;
    r.x = pack_bf16x2(v[0], v[1]);
    r.y = pack_bf16x2(v[2], v[3]);
    r.z = pack_bf16x2(v[4], v[5]);
    r.w = pack_bf16x2(v[6], v[7]);
    *reinterpret_cast<uint4*>(p) = r;
}

template <int FMT>
__device__ __forceinline__ uint8_t quant1(float x, float s, float inv) {
    if constexpr (FMT == FMT_INT8) return (uint8_t)quant_int8(x, s, inv);
    else if constexpr (FMT == FMT_E3M2) return (uint8_t)(quant_e3m2(x, s, inv) << 2);  // MMA operand byte
    else return quant_e4m3(x, s, inv);
}

// 8 codes -> one 8-byte store
template <int FMT>
__device__ __forceinline__ void quant_store8(uint8_t* p, const float v[8], float s, float inv) {
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) lo |= (uint32_t)quant1<FMT>(v[i], s, inv) << (8 * i);
#pragma unroll
    for (int i = 0; i < 4; ++i) hi |= (uint32_t)quant1<FMT>(v[4 + i], s, inv) << (8 * i);
    *reinterpret_cast<uint2*>(p) = make_uint2(lo, hi);
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// absmax of non-negative floats via the integer order of their bit patterns
// SwiGLU glue (the Llama MLP's activation; not part of the reference path).
// Every rounding is spelled out so the fused kernels (K1 swiglu-absmax, K2
// swiglu-absmax) and the stand-alone glue kernels produce identical bits.
// sigmoid(g) = 1 / (1 + exp(-g)) on the SFU (ex2.approx, rcp.approx: one
// MUFU op each; the SwiGLU GEMM epilogue runs this per element)
__device__ __forceinline__ float swiglu_sigmoid(float g) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(__fadd_rn(1.0f, __expf(-g))));
    return r;
}
// h = silu(g) * u
__device__ __forceinline__ float swiglu_fwd1(float g, float u) {
    return __fmul_rn(__fmul_rn(g, swiglu_sigmoid(g)), u);
}
// du = dh * silu(g);  dg = dh * u * s * (1 + g * (1 - s)),  s = sigmoid(g)
__device__ __forceinline__ void swiglu_bwd1(float dh, float g, float u, float& dg, float& du) {
    const float s = swiglu_sigmoid(g);
    du = __fmul_rn(__fmul_rn(dh, g), s);
    dg = __fmul_rn(__fmul_rn(__fmul_rn(dh, u), s), __fmaf_rn(g, __fadd_rn(1.0f, -s), 1.0f));
}

__device__ __forceinline__ void atomic_absmax(unsigned* slot, float v) {
    atomicMax(slot, __float_as_uint(v));
}

// branch-free non-finite test: all exponent bits set
__device__ __forceinline__ uint32_t nonfinite_bits(float x) {
    return (uint32_t)((__float_as_uint(x) & 0x7f800000u) == 0x7f800000u);
}
__device__ __forceinline__ bool finite8(const float v[8]) {
    uint32_t bad = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) bad |= nonfinite_bits(v[i]);
    return bad == 0;
}

// raw 8-element vectors: loads are issued before any arithmetic so a warp
// keeps several 16-32 B requests in flight
template <typename T>
struct Raw8;
template <>
struct Raw8<__nv_bfloat16> {
    uint4 r;
    __device__ __forceinline__ void load(const __nv_bfloat16* p) { r = __ldg(reinterpret_cast<const uint4*>(p)); }
    __device__ __forceinline__ void zero() { r = make_uint4(0, 0, 0, 0); }
    __device__ __forceinline__ void get(float v[8]) const {
        const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            v[2 * i] = __uint_as_float(w[i] << 16);
            v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        }
    }
};
template <>
struct Raw8<float> {
    float4 a, b;
    __device__ __forceinline__ void load(const float* p) {
        a = __ldg(reinterpret_cast<const float4*>(p));
        b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    }
    __device__ __forceinline__ void zero() { a = b = make_float4(0.f, 0.f, 0.f, 0.f); }
    __device__ __forceinline__ void get(float v[8]) const {
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    }
};

// scale and its reciprocal from the device absmax word (or a supplied scale)
__device__ __forceinline__ void resolve_scale(const unsigned* absmax_bits, const float* supplied, int fmt,
                                              float* s_out, float* inv_out) {
    float s;
    if (supplied) s = *supplied;
    else s = scale_from_absmax(__uint_as_float(*absmax_bits), fmt);
    *s_out = s;
    *inv_out = 1.0f / s;
}

}  // namespace halo_b200
