// adamw.cu — AdamWT::step (trainer.hpp:104-160) over a device-resident,
// row-sharded master (HQ-FSDP: every rank updates only its own rows, the
// reference's train_fsdp optimizer over `masters`, hqfsdp.hpp:340-411).
//
// Per element, in IEEE double exactly as the reference writes it (:141-150):
//   m = b1*m + (1-b1)*g ; v = b2*v + (1-b2)*g*g
//   w = w - lr_t * ((m/bc1) / (sqrt(v/bc2) + eps) + wd*w)
// lr_t, bc1 = 1-b1^t, bc2 = 1-b2^t are computed once per step on the host
// (:127-131).  The state is stored in fp32 (the reference keeps double), the
// master in bf16 or fp32: w is rounded double -> float -> T (the reference's
// static_cast<T> for T = float, then RNE to bf16).  Compiled with
// --fmad=false: no contraction, so a host restatement reproduces every bit.
// HBM-bound streaming kernel: 4 elements per thread and trip, 16 B / 8 B
// vector accesses, grid of 8 CTAs per SM.
#include "common.cuh"
#include "halo_internal.h"
#include "sm100.cuh"

namespace halo_b200 {

namespace {

template <typename T>
__device__ __forceinline__ void ld4(const T* p, float (&o)[4]);
template <>
__device__ __forceinline__ void ld4<float>(const float* p, float (&o)[4]) {
    const float4 f = __ldg(reinterpret_cast<const float4*>(p));
    o[0] = f.x; o[1] = f.y; o[2] = f.z; o[3] = f.w;
}
template <>
__device__ __forceinline__ void ld4<__nv_bfloat16>(const __nv_bfloat16* p, float (&o)[4]) {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(p));
    o[0] = __uint_as_float(u.x << 16);
    o[1] = __uint_as_float(u.x & 0xFFFF0000u);
    o[2] = __uint_as_float(u.y << 16);
    o[3] = __uint_as_float(u.y & 0xFFFF0000u);
}

template <typename T>
__device__ __forceinline__ void st4(T* p, const float (&o)[4]);
template <>
__device__ __forceinline__ void st4<float>(float* p, const float (&o)[4]) {
    *reinterpret_cast<float4*>(p) = make_float4(o[0], o[1], o[2], o[3]);
}
template <>
__device__ __forceinline__ void st4<__nv_bfloat16>(__nv_bfloat16* p, const float (&o)[4]) {
    *reinterpret_cast<uint2*>(p) = make_uint2(pack_bf16x2(o[0], o[1]), pack_bf16x2(o[2], o[3]));
}

template <typename PT, typename GT>
__global__ void __launch_bounds__(256) k_adamw(PT* __restrict__ p, const GT* __restrict__ g, float* __restrict__ m,
                                               float* __restrict__ v, int64_t n, double lr, double b1, double b2,
                                               double eps, double wd, double bc1, double bc2) {
    const double c1 = 1.0 - b1, c2 = 1.0 - b2;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
        float w4[4], g4[4], m4[4], v4[4];
        ld4<PT>(p + i, w4);
        ld4<GT>(g + i, g4);
        ld4<float>(m + i, m4);
        ld4<float>(v + i, v4);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const double gk = (double)g4[j];
            const double mk = b1 * (double)m4[j] + c1 * gk;
            const double vk = b2 * (double)v4[j] + c2 * gk * gk;
            m4[j] = (float)mk;
            v4[j] = (float)vk;
            const double mh = mk / bc1;
            const double vh = vk / bc2;
            const double wk = (double)w4[j];
            w4[j] = (float)(wk - lr * (mh / (sqrt(vh) + eps) + wd * wk));
        }
        st4<PT>(p + i, w4);
        st4<float>(m + i, m4);
        st4<float>(v + i, v4);
    }
}

template <typename PT, typename GT>
void launch(void* p, const void* g, float* m, float* v, int64_t n, double lr, double b1, double b2, double eps,
            double wd, double bc1, double bc2, cudaStream_t st) {
    int64_t want = (n / 4 + 255) / 256;
    const int64_t cap = (int64_t)num_sms() * 8;
    if (want > cap) want = cap;
    if (want < 1) want = 1;
    k_adamw<PT, GT><<<(unsigned)want, 256, 0, st>>>(static_cast<PT*>(p), static_cast<const GT*>(g), m, v, n, lr, b1,
                                                    b2, eps, wd, bc1, bc2);
}

}  // namespace

void run_adamw(void* p, int p_dtype, const void* g, int g_dtype, float* m, float* v, int64_t n, double lr, double b1,
               double b2, double eps, double wd, double bc1, double bc2, cudaStream_t st) {
    if (p_dtype == DT_BF16 && g_dtype == DT_BF16)
        launch<__nv_bfloat16, __nv_bfloat16>(p, g, m, v, n, lr, b1, b2, eps, wd, bc1, bc2, st);
    else if (p_dtype == DT_BF16)
        launch<__nv_bfloat16, float>(p, g, m, v, n, lr, b1, b2, eps, wd, bc1, bc2, st);
    else if (g_dtype == DT_BF16)
        launch<float, __nv_bfloat16>(p, g, m, v, n, lr, b1, b2, eps, wd, bc1, bc2, st);
    else
        launch<float, float>(p, g, m, v, n, lr, b1, b2, eps, wd, bc1, bc2, st);
}

}  // namespace halo_b200
