// glue.cu — the elementwise glue between HALO linears in a Llama MLP block
// (down(silu(gate(x)) * up(x))): SwiGLU forward / backward and a residual
// add.  HBM-streaming, 16 B vector loads, grid-stride over 148 x k CTAs.
//
// The reference's toy block uses silu between fc1 and fc2 (model.hpp:77-96,
// 169-171, 193-195); the Llama MLP gates it with a second projection.
#include "common.cuh"
#include "sm100.cuh"
#include "halo_internal.h"

namespace halo_b200 {


// H = silu(G) * U, all bf16, n % 8 == 0
__global__ void __launch_bounds__(256) k_swiglu_fwd(const __nv_bfloat16* __restrict__ G,
                                                    const __nv_bfloat16* __restrict__ U,
                                                    __nv_bfloat16* __restrict__ H, int64_t n) {
    pdl_wait();
    pdl_trigger();
    // two 8-element groups per thread and trip (one grid stride apart): four
    // 16 B loads in flight before any math
    const int64_t half = (int64_t)gridDim.x * blockDim.x * 8;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; i < n; i += 2 * half) {
        const int64_t i2 = i + half;
        float g[8], u[8], g2[8], u2[8], h[8];
        load8(G + i, g);
        load8(U + i, u);
        if (i2 < n) {
            load8(G + i2, g2);
            load8(U + i2, u2);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) h[j] = swiglu_fwd1(g[j], u[j]);
        store8(H + i, h);
        if (i2 < n) {
#pragma unroll
            for (int j = 0; j < 8; ++j) h[j] = swiglu_fwd1(g2[j], u2[j]);
            store8(H + i2, h);
        }
    }
}

// dU = dH * silu(G); dG = dH * U * s * (1 + G * (1 - s)),  s = sigmoid(G)
__global__ void __launch_bounds__(256) k_swiglu_bwd(const __nv_bfloat16* __restrict__ dH,
                                                    const __nv_bfloat16* __restrict__ G,
                                                    const __nv_bfloat16* __restrict__ U,
                                                    __nv_bfloat16* __restrict__ dG, __nv_bfloat16* __restrict__ dU,
                                                    int64_t n) {
    pdl_wait();
    pdl_trigger();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; i < n; i += stride) {
        float dh[8], g[8], u[8], dg[8], du[8];
        load8(dH + i, dh);
        load8(G + i, g);
        load8(U + i, u);
#pragma unroll
        for (int j = 0; j < 8; ++j) swiglu_bwd1(dh[j], g[j], u[j], dg[j], du[j]);
        store8(dG + i, dg);
        store8(dU + i, du);
    }
}

// out = a + b (bf16 or fp32 elements, computed in fp32)
template <typename T>
__global__ void __launch_bounds__(256) k_add(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out,
                                             int64_t n) {
    pdl_wait();
    pdl_trigger();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 8;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 8; i < n; i += stride) {
        float x[8], y[8];
        load8(a + i, x);
        load8(b + i, y);
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] += y[j];
        store8(out + i, x);
    }
}

// HQ-FSDP reduce-scatter, owner side (hqfsdp.hpp:271-300): out[i] =
// T(sum_w double(recv[w][i]) / world), accumulated in double in rank order
template <typename T>
__global__ void __launch_bounds__(256) k_rank_mean(const float* __restrict__ recv, int world, int64_t n,
                                                   T* __restrict__ out) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
        double acc[4] = {0.0, 0.0, 0.0, 0.0};
        for (int w = 0; w < world; ++w) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(recv + (int64_t)w * n + i));
            acc[0] += (double)v.x;
            acc[1] += (double)v.y;
            acc[2] += (double)v.z;
            acc[3] += (double)v.w;
        }
        float r[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) r[j] = (float)(acc[j] / (double)world);
        if constexpr (sizeof(T) == 4) {
            *reinterpret_cast<float4*>(out + i) = make_float4(r[0], r[1], r[2], r[3]);
        } else {
            *reinterpret_cast<uint2*>(out + i) = make_uint2(pack_bf16x2(r[0], r[1]), pack_bf16x2(r[2], r[3]));
        }
    }
}


// INT8 contractions longer than the s32 TMEM accumulator can hold exactly
// (K*127^2 >= 2^31): K slices of raw s32 accumulators summed in int64, as the
// reference accumulates (quantize.hpp:358-371), then its double epilogue
// float(double(acc) * (double(sa) * double(sb))) (:370).
__global__ void __launch_bounds__(256) k_acc_s64(const int* __restrict__ part, long long* __restrict__ acc,
                                                 int64_t n, int first) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
        acc[i] = (first ? 0LL : acc[i]) + (long long)part[i];
}

template <typename T>
__global__ void __launch_bounds__(256) k_epi_s64(const long long* __restrict__ acc, const float* __restrict__ sa,
                                                 const float* __restrict__ sb, T* __restrict__ out, int64_t n) {
    const double ss = (double)*sa * (double)*sb;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const float c = (float)((double)acc[i] * ss);
        if constexpr (sizeof(T) == 4) out[i] = c;
        else out[i] = __float2bfloat16_rn(c);
    }
}

static unsigned ew_grid(int64_t n) {
    int64_t want = (n / 8 + 255) / 256;
    const int64_t cap = (int64_t)num_sms() * 8;
    if (want > cap) want = cap;
    if (want < 1) want = 1;
    return (unsigned)want;
}

void run_swiglu_fwd(const void* G, const void* U, void* H, int64_t n, cudaStream_t st) {
    launch_pdl(k_swiglu_fwd, dim3(ew_grid(n)), dim3(256), 0, st, static_cast<const __nv_bfloat16*>(G),
               static_cast<const __nv_bfloat16*>(U), static_cast<__nv_bfloat16*>(H), n);
}

void run_swiglu_bwd(const void* dH, const void* G, const void* U, void* dG, void* dU, int64_t n, cudaStream_t st) {
    launch_pdl(k_swiglu_bwd, dim3(ew_grid(n)), dim3(256), 0, st, static_cast<const __nv_bfloat16*>(dH),
               static_cast<const __nv_bfloat16*>(G), static_cast<const __nv_bfloat16*>(U),
               static_cast<__nv_bfloat16*>(dG), static_cast<__nv_bfloat16*>(dU), n);
}

void run_add(const void* a, const void* b, void* out, int dtype, int64_t n, cudaStream_t st) {
    if (dtype == DT_BF16)
        launch_pdl(k_add<__nv_bfloat16>, dim3(ew_grid(n)), dim3(256), 0, st, static_cast<const __nv_bfloat16*>(a),
                   static_cast<const __nv_bfloat16*>(b), static_cast<__nv_bfloat16*>(out), n);
    else
        launch_pdl(k_add<float>, dim3(ew_grid(n)), dim3(256), 0, st, static_cast<const float*>(a),
                   static_cast<const float*>(b), static_cast<float*>(out), n);
}

void run_rank_mean(const float* recv, int world, int64_t n, void* out, int dtype, cudaStream_t st) {
    const unsigned grid = ew_grid(n * 2);
    if (dtype == DT_BF16)
        k_rank_mean<__nv_bfloat16><<<grid, 256, 0, st>>>(recv, world, n, static_cast<__nv_bfloat16*>(out));
    else
        k_rank_mean<float><<<grid, 256, 0, st>>>(recv, world, n, static_cast<float*>(out));
}

void run_acc_s64(const int* part, long long* acc, int64_t n, int first, cudaStream_t st) {
    k_acc_s64<<<ew_grid(n * 8), 256, 0, st>>>(part, acc, n, first);
}

void run_epi_s64(const long long* acc, const float* sa, const float* sb, void* out, int dtype, int64_t n,
                 cudaStream_t st) {
    if (dtype == DT_BF16)
        k_epi_s64<__nv_bfloat16><<<ew_grid(n * 8), 256, 0, st>>>(acc, sa, sb, static_cast<__nv_bfloat16*>(out), n);
    else
        k_epi_s64<float><<<ew_grid(n * 8), 256, 0, st>>>(acc, sa, sb, static_cast<float*>(out), n);
}

// HQ-FSDP helpers: stale-scale flag (hqfsdp.hpp:256-259) and the 1/world
// of the gradient mean after a reduce-scatter (:288-292)
__global__ void k_flag_neq(const float* a, const float* b, unsigned* flag) {
    if (!(*a == *b)) atomicOr(flag, 1u);
}
void run_flag_neq(const float* a, const float* b, unsigned* flag, cudaStream_t st) { k_flag_neq<<<1, 1, 0, st>>>(a, b, flag); }

template <typename T>
__global__ void __launch_bounds__(256) k_scale_mul(T* p, int64_t n, float k) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        if constexpr (sizeof(T) == 4) p[i] = p[i] * k;
        else p[i] = __float2bfloat16_rn(__bfloat162float(p[i]) * k);
    }
}
void run_scale_mul(void* buf, int dtype, int64_t n, float k, cudaStream_t st) {
    if (n <= 0) return;
    if (dtype == DT_BF16) k_scale_mul<__nv_bfloat16><<<ew_grid(n * 8), 256, 0, st>>>(static_cast<__nv_bfloat16*>(buf), n, k);
    else k_scale_mul<float><<<ew_grid(n * 8), 256, 0, st>>>(static_cast<float*>(buf), n, k);
}

// FP6 E3M2 wire format (the HQ-FSDP gather payload, hqfsdp.hpp:36-49: four
// codes in three bytes): group g of 4 device codes (E3M2 in bits 7:2 of one
// byte each) -> 24-bit little-endian word c0 | c1 << 6 | c2 << 12 | c3 << 18.
// One thread packs / unpacks 8 groups (32 codes <-> 24 bytes).
__global__ void __launch_bounds__(256) k_fp6_pack(const uint8_t* __restrict__ codes, uint8_t* __restrict__ packed,
                                                  int64_t groups) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += stride) {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(codes + 4 * g);
        const uint32_t v = ((w >> 2) & 0x3Fu) | (((w >> 10) & 0x3Fu) << 6) | (((w >> 18) & 0x3Fu) << 12) |
                           (((w >> 26) & 0x3Fu) << 18);
        uint8_t* o = packed + 3 * g;
        o[0] = (uint8_t)v;
        o[1] = (uint8_t)(v >> 8);
        o[2] = (uint8_t)(v >> 16);
    }
}
__global__ void __launch_bounds__(256) k_fp6_unpack(const uint8_t* __restrict__ packed, uint8_t* __restrict__ codes,
                                                    int64_t groups) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += stride) {
        const uint8_t* i = packed + 3 * g;
        const uint32_t v = (uint32_t)i[0] | ((uint32_t)i[1] << 8) | ((uint32_t)i[2] << 16);
        const uint32_t w = ((v & 0x3Fu) << 2) | (((v >> 6) & 0x3Fu) << 10) | (((v >> 12) & 0x3Fu) << 18) |
                           (((v >> 18) & 0x3Fu) << 26);
        *reinterpret_cast<uint32_t*>(codes + 4 * g) = w;
    }
}
void run_fp6_pack(const uint8_t* codes, uint8_t* packed, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    k_fp6_pack<<<ew_grid(n * 2), 256, 0, st>>>(codes, packed, n / 4);
}
void run_fp6_unpack(const uint8_t* packed, uint8_t* codes, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    k_fp6_unpack<<<ew_grid(n * 2), 256, 0, st>>>(packed, codes, n / 4);
}

void retain_async_pool() {
    static thread_local int done_dev = -1;
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d == done_dev) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, d) == cudaSuccess) {
        uint64_t keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done_dev = d;
}

}  // namespace halo_b200
