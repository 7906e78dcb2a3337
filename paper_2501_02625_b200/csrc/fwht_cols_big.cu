// fwht_cols_big.cu — K2 for large Hadamard blocks along the token axis,
// sm_100a: 512 <= B <= 16384 (the reference's default had_block = 0 pads the
// tokens to b_pad and transforms all of them: B = b_pad).
//
// Reference: error_path, halo_linear.hpp:393-399 — (H_b pad(E_Y))_Q with
// transform_left (hadamard.hpp:205-216): the row transform of
// hadamard.hpp:136-177 down each column, stages len = 1, 2, ..., B/2 over the
// row index, one normalising multiply; plus (E_Y)_Q for G (:371).
// Bit-exact: the same fp32 butterflies in the same order.
//
// Two kernels split the LB row-index bits 8 + (LB - 8):
//   lo: a 4-warp CTA owns a 256-row x 32-column tile, runs stages len =
//       1..128 (row bits 0..7: 4 in registers, one smem exchange, 4 more)
//       and writes the partial transform to an fp32 scratch tensor; it also
//       reduces the plain absmax of the raw input (for (E_Y)_Q).
//   hi: a warp owns one residue r (row mod 256) of one B-block and 32
//       columns: lane c loads the 2^(LB-8) rows r + 256 i of its column
//       (coalesced 128 B per row), runs stages len = 256..B/2, then either
//       reduces the rotated absmax (last stage as |u|+|v|) or normalises and
//       quantizes (one byte per lane and row: a 32 B sector per warp store).
// The plain codes come from the generic plain quantizer.
#include "common.cuh"
#include "halo_internal.h"
#include "sm100.cuh"


namespace halo_b200 {

namespace {

__device__ __forceinline__ float cb_max3nan(float a, float b, float c) {
    float r;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ void cb_bfly(float2& a, float2& b) {
    const float2 x = a, y = b;
    a = __fadd2_rn(x, y);
    b = __fadd2_rn(x, make_float2(-y.x, -y.y));
}

template <typename InT>
__device__ __forceinline__ void cb_load4(const InT* p, bool ok, float2& a, float2& b) {
    if constexpr (sizeof(InT) == 2) {
        uint2 r = make_uint2(0, 0);
        if (ok) r = __ldg(reinterpret_cast<const uint2*>(p));
        a = make_float2(__uint_as_float(r.x << 16), __uint_as_float(r.x & 0xFFFF0000u));
        b = make_float2(__uint_as_float(r.y << 16), __uint_as_float(r.y & 0xFFFF0000u));
    } else {
        float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
        if (ok) r = __ldg(reinterpret_cast<const float4*>(p));
        a = make_float2(r.x, r.y);
        b = make_float2(r.z, r.w);
    }
}

// stages len = 1..128 of 256-row tiles; out: fp32 [rows_pad x cols]
template <typename InT>
__global__ void __launch_bounds__(128) k_cols_lo(const InT* __restrict__ in, int64_t b, int64_t rows_pad, int64_t cols,
                                                 float* __restrict__ out, unsigned* amax_plain, unsigned* err) {
    __shared__ __align__(16) float4 X4[256 * 8];
    pdl_wait();
    pdl_trigger();
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int cg = l & 7, q = 4 * w + (l >> 3);
    const int64_t ct = (cols + 31) / 32, rt = rows_pad / 256;
    float am_p = 0.f;
    for (int64_t tile = blockIdx.x; tile < ct * rt; tile += gridDim.x) {
        const int64_t r0 = (tile / ct) * 256, c0 = (tile % ct) * 32;
        const int64_t col = c0 + 4 * cg;
        const bool cok = col < cols;
        const int64_t row1 = r0 + 16 * q;
        float2 v[16][2];
#pragma unroll
        for (int m = 0; m < 16; ++m) cb_load4<InT>(in + (row1 + m) * cols + col, cok && row1 + m < b, v[m][0], v[m][1]);
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            am_p = cb_max3nan(am_p, fabsf(v[m][0].x), fabsf(v[m][0].y));
            am_p = cb_max3nan(am_p, fabsf(v[m][1].x), fabsf(v[m][1].y));
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int h = 1 << t;
#pragma unroll
            for (int m = 0; m < 16; ++m)
                if ((m & h) == 0) {
                    cb_bfly(v[m][0], v[m + h][0]);
                    cb_bfly(v[m][1], v[m + h][1]);
                }
        }
#pragma unroll
        for (int m = 0; m < 16; ++m) X4[(16 * q + m) * 8 + cg] = make_float4(v[m][0].x, v[m][0].y, v[m][1].x, v[m][1].y);
        __syncthreads();
        float2 u[16][2];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const float4 f = X4[(16 * i + q) * 8 + cg];
            u[i][0] = make_float2(f.x, f.y);
            u[i][1] = make_float2(f.z, f.w);
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int h = 1 << t;
#pragma unroll
            for (int i = 0; i < 16; ++i)
                if ((i & h) == 0) {
                    cb_bfly(u[i][0], u[i + h][0]);
                    cb_bfly(u[i][1], u[i + h][1]);
                }
        }
        if (cok) {
#pragma unroll
            for (int i = 0; i < 16; ++i)
                *reinterpret_cast<float4*>(out + (r0 + 16 * i + q) * cols + col) =
                    make_float4(u[i][0].x, u[i][0].y, u[i][1].x, u[i][1].y);
        }
    }
    if (amax_plain) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) am_p = cb_max3nan(am_p, __shfl_xor_sync(0xffffffffu, am_p, o), 0.f);
        if (l == 0) {
            atomic_absmax(amax_plain, fabsf(am_p));
            if (!(am_p <= 3.402823466e38f)) atomicOr(err, ERRF_NONFINITE);
        }
    }
}

// stages len = 256..B/2 (row bits 8..LB-1), then absmax (MODE 0) or codes (MODE 1)
template <int LBH, int FMT, int MODE>
__global__ void __launch_bounds__(128) k_cols_hi(const float* __restrict__ buf, int64_t rows_pad, int64_t cols,
                                                 float norm, unsigned* amax, const float* supplied,
                                                 uint8_t* __restrict__ codes, unsigned* err, float* scale_out,
                                                 float* __restrict__ xout, int64_t rows_out) {
    constexpr int R = 1 << LBH;
    constexpr bool FOLD = ((LBH + 8) % 2) == 0;
    pdl_wait();
    pdl_trigger();
    float s = 1.f, inv = 1.f, h = 0.f;
    if constexpr (MODE == 1) {
        resolve_scale(amax, supplied, FMT, &s, &inv);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            if (scale_out) *scale_out = s;
            if (!supplied && *amax >= 0x7f800000u) atomicOr(err, ERRF_NONFINITE);
        }
        if (FOLD) {
            s = s / norm;  // exact power-of-two rescale
            inv = inv * norm;
        }
        h = half_margin(s);
    }
    const int lane = threadIdx.x & 31;
    const int64_t strips = (cols + 31) / 32, blocks = rows_pad / (R * 256);
    const int64_t tasks = blocks * 256 * strips;
    const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    float am = 0.f;
    for (int64_t task = warp0; task < tasks; task += nwarps) {
        // consecutive warps: consecutive strips of the same residue (row)
        const int64_t strip = task % strips, rest = task / strips;
        const int64_t resid = rest % 256, blk = rest / 256;
        const int64_t c = strip * 32 + lane;
        if (c >= cols) continue;
        const int64_t row0 = blk * (R * 256) + resid;
        float v[R];
#pragma unroll
        for (int i = 0; i < R; ++i) v[i] = __ldg(buf + (row0 + 256 * (int64_t)i) * cols + c);
#pragma unroll
        for (int t = 0; t < LBH; ++t) {
            const int hh = 1 << t;
            const bool last = MODE == 0 && t == LBH - 1;
#pragma unroll
            for (int i = 0; i < R; ++i)
                if ((i & hh) == 0) {
                    const float a = v[i], b2 = v[i + hh];
                    if (last) {
                        am = cb_max3nan(am, fabsf(a) + fabsf(b2), 0.f);
                    } else {
                        v[i] = __fadd_rn(a, b2);
                        v[i + hh] = __fadd_rn(a, -b2);
                    }
                }
        }
        if constexpr (MODE == 2) {  // transform only (K4-left): normalised fp32, rows < rows_out kept
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const int64_t row = row0 + 256 * (int64_t)i;
                if (row < rows_out) xout[row * cols + c] = __fmul_rn(v[i], norm);
            }
        }
        if constexpr (MODE == 1) {
#pragma unroll
            for (int i = 0; i < R; ++i) {
                const float x = FOLD ? v[i] : __fmul_rn(v[i], norm);
                uint8_t code;
                if constexpr (FMT == FMT_INT8) {
                    uint32_t slow;
                    code = quant_int8_try_r(x, s, inv, h, slow);
                    if (slow) code = (uint8_t)quant_int8(x, s, inv);
                } else if constexpr (FMT == FMT_E3M2) {
                    code = (uint8_t)(quant_e3m2(x, s, inv) << 2);
                } else {
                    code = quant_e4m3(x, s, inv);
                }
                codes[(row0 + 256 * (int64_t)i) * cols + c] = code;
            }
        }
    }
    if constexpr (MODE == 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) am = cb_max3nan(am, __shfl_xor_sync(0xffffffffu, am, o), 0.f);
        am *= norm;  // monotone: max(fl(|x| * norm)) == fl(max|x| * norm)
        if (lane == 0) {
            atomic_absmax(amax, fabsf(am));
            if (!(am <= 3.402823466e38f)) atomicOr(err, ERRF_NONFINITE);
        }
    }
}

template <int LBH, int FMT, int MODE>
void cb_hi(const float* buf, int64_t rows_pad, int64_t cols, float norm, unsigned* amax, const float* sup,
           uint8_t* codes, unsigned* err, float* sout, cudaStream_t st, float* xout = nullptr, int64_t rows_out = 0) {
    auto kern = k_cols_hi<LBH, FMT, MODE>;
    const int64_t tasks = rows_pad / 256 * ((cols + 31) / 32);
    int64_t grid = (tasks + 3) / 4;
    const int64_t cap = (int64_t)num_sms() * 16;
    if (grid > cap) grid = cap;
    launch_pdl(kern, dim3((unsigned)(grid < 1 ? 1 : grid)), dim3(128), 0, st, buf, rows_pad, cols, norm, amax, sup,
               codes, err, sout, xout, rows_out);
}

template <int LBH>
void cb_hi_dispatch(int mode, int fmt, const float* buf, int64_t rows_pad, int64_t cols, float norm, unsigned* amax,
                    const float* sup, uint8_t* codes, unsigned* err, float* sout, cudaStream_t st, float* xout,
                    int64_t rows_out) {
    if (mode == 2) cb_hi<LBH, 0, 2>(buf, rows_pad, cols, norm, amax, sup, codes, err, sout, st, xout, rows_out);
    else if (mode == 0) cb_hi<LBH, 0, 0>(buf, rows_pad, cols, norm, amax, sup, codes, err, sout, st);
    else if (fmt == FMT_INT8) cb_hi<LBH, FMT_INT8, 1>(buf, rows_pad, cols, norm, amax, sup, codes, err, sout, st);
    else if (fmt == FMT_E3M2) cb_hi<LBH, FMT_E3M2, 1>(buf, rows_pad, cols, norm, amax, sup, codes, err, sout, st);
    else cb_hi<LBH, FMT_E4M3, 1>(buf, rows_pad, cols, norm, amax, sup, codes, err, sout, st);
}

}  // namespace

// K2 modes 0 (absmax) / 1 (quantize) / 2 (transform, fp32 in -> fp32 out,
// rows < rows_out: K4-left) for 512 <= B <= 16384 (B = 2^k,
// rows_pad a multiple of B, cols % 4 == 0).  The plain operand: absmax in
// mode 0 (from the raw input), codes in mode 1 through run_plain.
bool cols_big(int mode, int fmt, int in_dtype, const void* in, int64_t b, int64_t rows_pad, int64_t cols, int64_t B,
              unsigned* ar, unsigned* ap, const float* sr, const float* sp, uint8_t* cr, uint8_t* cp, unsigned* err,
              float* sro, float* spo, cudaStream_t st, float* xout, int64_t rows_out) {
    if (mode > 2 || B < 512 || B > 16384 || (B & (B - 1)) || rows_pad % B || cols % 4) return false;
    if (mode == 2 && (in_dtype != DT_F32 || !xout)) return false;
    if ((uintptr_t)in % (in_dtype == DT_BF16 ? 8 : 16)) return false;
    // stream-ordered scratch for the partial transform: no sharing between
    // streams or calls, returned to the pool after the last reader
    float* buf = nullptr;
    retain_async_pool();
    if (cudaMallocAsync(reinterpret_cast<void**>(&buf), (size_t)rows_pad * (size_t)cols * sizeof(float), st) !=
        cudaSuccess)
        return false;
    int lb = 0;
    while ((int64_t(1) << lb) < B) ++lb;
    {
        const int64_t tiles = (rows_pad / 256) * ((cols + 31) / 32);
        const int64_t cap = (int64_t)num_sms() * 4;
        const unsigned grid = (unsigned)(tiles < cap ? tiles : cap);
        unsigned* plain_amax = (mode == 0 && !sp && ap) ? ap : nullptr;
        if (in_dtype == DT_BF16)
            launch_pdl(k_cols_lo<__nv_bfloat16>, dim3(grid), dim3(128), 0, st, static_cast<const __nv_bfloat16*>(in), b,
                       rows_pad, cols, buf, plain_amax, err);
        else
            launch_pdl(k_cols_lo<float>, dim3(grid), dim3(128), 0, st, static_cast<const float*>(in), b, rows_pad, cols,
                       buf, plain_amax, err);
    }
    const float norm = hadamard_norm(B);
    switch (lb) {
    case 9: cb_hi_dispatch<1>(mode, fmt, buf, rows_pad, cols, norm, ar, sr, cr, err, sro, st, xout, rows_out); break;
    case 10: cb_hi_dispatch<2>(mode, fmt, buf, rows_pad, cols, norm, ar, sr, cr, err, sro, st, xout, rows_out); break;
    case 11: cb_hi_dispatch<3>(mode, fmt, buf, rows_pad, cols, norm, ar, sr, cr, err, sro, st, xout, rows_out); break;
    case 12: cb_hi_dispatch<4>(mode, fmt, buf, rows_pad, cols, norm, ar, sr, cr, err, sro, st, xout, rows_out); break;
    case 13: cb_hi_dispatch<5>(mode, fmt, buf, rows_pad, cols, norm, ar, sr, cr, err, sro, st, xout, rows_out); break;
    default: cb_hi_dispatch<6>(mode, fmt, buf, rows_pad, cols, norm, ar, sr, cr, err, sro, st, xout, rows_out); break;
    }
    if (mode == 1 && cp) run_plain(in, in_dtype, b * cols, 1, fmt, ap, sp, cp, err, spo, st);
    cudaFreeAsync(buf, st);
    return true;
}

}  // namespace halo_b200
