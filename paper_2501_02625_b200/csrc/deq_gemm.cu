// Granularity::row backward products (halo_linear.hpp:381-439 with
// scheme.granularity = row).  Per-row scales of (WH)_Q and of E_Y's codes sit
// on the CONTRACTED dim of the E and G products, so one rescale of an integer
// accumulator cannot reproduce them; the reference dequantizes each operand
// to T = float (double(code) * scale rounded to float, quantize.hpp:283-294)
// and multiplies in double, k ascending per output (qmatmul :377-379,
// tensor.hpp:127-144 / matmul_nt_acc / matmul_tn_acc).
//
// This kernel restates exactly that: the products of two floats are exact in
// double, the accumulation runs k = 0..K-1 sequentially per output element in
// double (one DFMA of an exact product == the reference's add), and the
// result is rounded once to float -- bit-exact with the reference for any
// shapes.  It runs on the FP64 pipe (the tensor cores have no double
// accumulate of dequantized floats); the row-granularity backward is a
// parity path, the HALO tensor-granularity GEMMs in gemm_sm100.cu are the
// throughput path.
//
// Operand views: A(i,k) = deq(a[i*a_si + k*a_sk], as[i*as_si + k*as_sk]),
// B(k,j) = deq(b[k*b_sk + j*b_sj], bs[k*bs_sk + j*bs_sj]); one of each scale
// stride pair is 0 (per-row / per-column scales) -- so the transposed views
// the backward needs (E^T for G, transpose_quantized :297-334) are strides,
// not copies.
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"
#include "halo_internal.h"
#include "quant_round.cuh"
#include "sm100.cuh"

namespace halo_b200 {
namespace {

constexpr int DG_TM = 8, DG_TN = 4, DG_BM = 16 * DG_TM, DG_BN = 16 * DG_TN, DG_BK = 32, DG_THREADS = 256;

template <int FMT>
__device__ __forceinline__ float code_value(uint8_t c) {
    if (FMT == FMT_INT8) return (float)(int8_t)c;
    if (FMT == FMT_E3M2) return e3m2_to_float((uint8_t)(c >> 2));  // bits 7:2 (MXFP6 codes)
    const float mag = e4m3_mag(c & 0x7Fu);
    return (c & 0x80u) ? -mag : mag;
}

// deq (quantize.hpp:289): static_cast<float>(double(code) * double(scale)),
// kept as the double the reference's matmul_acc widens it to
template <int FMT>
__device__ __forceinline__ double deq(uint8_t c, float s) {
    return (double)__double2float_rn(__dmul_rn((double)code_value<FMT>(c), (double)s));
}

struct DeqView {
    const uint8_t* codes;
    const float* scale;
    int64_t s0, s1;    // element strides (row index, k) for A; (k, col index) for B
    int64_t ss0, ss1;  // scale strides, same index pair
    int sh0, sh1;      // the scale index uses (index >> sh): 5 for the 32-wide MX blocks (quantize.hpp:129)
};

// 128 x 64 output tile per CTA, 8 x 4 per thread (rows tr + 16 r, columns
// tc + 16 c): 12 LDS.64 feed 32 DFMA per k step, and two CTAs fit an SM so
// one's operand staging overlaps the other's DFMAs.  Operands are
// dequantized once per tile element into shared memory as doubles.
template <int FMT>
__global__ void __launch_bounds__(DG_THREADS, 2) k_deq_gemm(DeqView A, DeqView B, float* __restrict__ C, int64_t M,
                                                        int64_t N, int64_t K, int64_t ldc) {
    __shared__ double As[DG_BK][DG_BM];
    __shared__ double Bs[DG_BK][DG_BN];
    const int tid = threadIdx.x;
    const int64_t i0 = (int64_t)blockIdx.y * DG_BM, j0 = (int64_t)blockIdx.x * DG_BN;
    const int tr = tid / 16, tc = tid % 16;
    double acc[DG_TM][DG_TN];
#pragma unroll
    for (int r = 0; r < DG_TM; ++r)
#pragma unroll
        for (int c = 0; c < DG_TN; ++c) acc[r][c] = 0.0;
    pdl_wait();
    for (int64_t k0 = 0; k0 < K; k0 += DG_BK) {
        // the operand tiles, the fastest index following the operand's
        // unit stride so loads coalesce
#pragma unroll
        for (int e = 0; e < (DG_BM * DG_BK) / DG_THREADS; ++e) {
            const int idx = tid + e * DG_THREADS;
            int ii, kk;
            if (A.s1 == 1) { kk = idx % DG_BK; ii = idx / DG_BK; } else { ii = idx % DG_BM; kk = idx / DG_BM; }
            const int64_t gi = i0 + ii, gk = k0 + kk;
            double v = 0.0;
            if (gi < M && gk < K)
                v = deq<FMT>(A.codes[gi * A.s0 + gk * A.s1], A.scale[(gi >> A.sh0) * A.ss0 + (gk >> A.sh1) * A.ss1]);
            As[kk][ii] = v;
        }
#pragma unroll
        for (int e = 0; e < (DG_BN * DG_BK) / DG_THREADS; ++e) {
            const int idx = tid + e * DG_THREADS;
            int jj, kk;
            if (B.s1 == 1) { jj = idx % DG_BN; kk = idx / DG_BN; } else { kk = idx % DG_BK; jj = idx / DG_BK; }
            const int64_t gj = j0 + jj, gk = k0 + kk;
            double w = 0.0;
            if (gj < N && gk < K)
                w = deq<FMT>(B.codes[gk * B.s0 + gj * B.s1], B.scale[(gk >> B.sh0) * B.ss0 + (gj >> B.sh1) * B.ss1]);
            Bs[kk][jj] = w;
        }
        __syncthreads();
        const int kn = (int)(K - k0 < DG_BK ? K - k0 : DG_BK);
        for (int kk = 0; kk < kn; ++kk) {  // k ascending: the reference's order
            double a[DG_TM], b[DG_TN];
#pragma unroll
            for (int r = 0; r < DG_TM; ++r) a[r] = As[kk][tr + 16 * r];
#pragma unroll
            for (int c = 0; c < DG_TN; ++c) b[c] = Bs[kk][tc + 16 * c];
#pragma unroll
            for (int r = 0; r < DG_TM; ++r)
#pragma unroll
                for (int c = 0; c < DG_TN; ++c) acc[r][c] = __fma_rn(a[r], b[c], acc[r][c]);
        }
        __syncthreads();
    }
    pdl_trigger();
#pragma unroll
    for (int r = 0; r < DG_TM; ++r) {
        const int64_t i = i0 + tr + 16 * r;
        if (i >= M) continue;
#pragma unroll
        for (int c = 0; c < DG_TN; ++c) {
            const int64_t j = j0 + tc + 16 * c;
            if (j < N) C[i * ldc + j] = __double2float_rn(acc[r][c]);
        }
    }
}

// pad_rows (halo_linear.hpp:393-395) into fp32: rows [b, b_pad) are zero
template <typename InT>
__global__ void k_pad_f32(const InT* __restrict__ in, float* __restrict__ out, int64_t nin, int64_t nout) {
    pdl_wait();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nout; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = i < nin ? (float)in[i] : 0.f;
    pdl_trigger();
}

// Granularity::column quantization (quantize.hpp:202-280, group_of = j):
// absmax per column, scale = absmax / format_max (1 for an all-zero
// column), codes by the exact quantizers.  One thread per column and a chunk
// of DG_RCH rows per CTA row: warps read 32 consecutive columns (coalesced).
constexpr int DG_RCH = 64;

template <typename InT>
__global__ void __launch_bounds__(256) k_col_absmax(const InT* __restrict__ in, int64_t rows, int64_t cols,
                                                   unsigned* __restrict__ amax, unsigned* err) {
    pdl_wait();
    const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (j < cols) {
        const int64_t r0 = (int64_t)blockIdx.y * DG_RCH;
        const int64_t r1 = r0 + DG_RCH < rows ? r0 + DG_RCH : rows;
        float m = 0.f;
        uint32_t bad = 0;
        for (int64_t r = r0; r < r1; ++r) {
            const float v = (float)in[r * cols + j];
            bad |= nonfinite_bits(v);
            m = fmaxf(m, fabsf(v));
        }
        atomic_absmax(&amax[j], m);
        if (bad) atomicOr(err, ERRF_NONFINITE);
    }
    pdl_trigger();
}

template <typename InT, int FMT>
__global__ void __launch_bounds__(256) k_col_quant(const InT* __restrict__ in, int64_t rows, int64_t cols,
                                                  const unsigned* __restrict__ amax, float* __restrict__ scales,
                                                  uint8_t* __restrict__ codes) {
    pdl_wait();
    const int64_t j = (int64_t)blockIdx.x * 256 + threadIdx.x;
    if (j < cols) {
        float s, inv;
        resolve_scale(&amax[j], nullptr, FMT, &s, &inv);
        if (blockIdx.y == 0) scales[j] = s;
        const int64_t r0 = (int64_t)blockIdx.y * DG_RCH;
        const int64_t r1 = r0 + DG_RCH < rows ? r0 + DG_RCH : rows;
        for (int64_t r = r0; r < r1; ++r) codes[r * cols + j] = quant1<FMT>((float)in[r * cols + j], s, inv);
    }
    pdl_trigger();
}

template <typename InT>
static void col_quant_launch(int fmt, const InT* in, int64_t rows, int64_t cols, unsigned* amax, float* scales,
                             uint8_t* codes, unsigned* err, cudaStream_t st) {
    const dim3 grid((unsigned)((cols + 255) / 256), (unsigned)((rows + DG_RCH - 1) / DG_RCH));
    launch_pdl(k_col_absmax<InT>, grid, dim3(256), 0, st, in, rows, cols, amax, err);
    if (fmt == FMT_INT8)
        launch_pdl(k_col_quant<InT, FMT_INT8>, grid, dim3(256), 0, st, in, rows, cols, (const unsigned*)amax, scales,
                   codes);
    else
        launch_pdl(k_col_quant<InT, FMT_E4M3>, grid, dim3(256), 0, st, in, rows, cols, (const unsigned*)amax, scales,
                   codes);
}

}  // namespace

void pad_rows_f32(const void* in, int in_dtype, int64_t b, int64_t b_pad, int64_t cols, float* out, cudaStream_t st) {
    const int64_t nout = b_pad * cols;
    if (nout <= 0) return;
    const unsigned grid = (unsigned)((nout + 255) / 256 < 148 * 16 ? (nout + 255) / 256 : 148 * 16);
    if (in_dtype == DT_BF16)
        launch_pdl(k_pad_f32<__nv_bfloat16>, dim3(grid), dim3(256), 0, st, static_cast<const __nv_bfloat16*>(in), out,
                   b * cols, nout);
    else
        launch_pdl(k_pad_f32<float>, dim3(grid), dim3(256), 0, st, static_cast<const float*>(in), out, b * cols, nout);
}

bool deq_gemm(int fmt, const uint8_t* a, const float* as, int64_t a_si, int64_t a_sk, int64_t as_si, int64_t as_sk,
              const uint8_t* b, const float* bs, int64_t b_sk, int64_t b_sj, int64_t bs_sk, int64_t bs_sj, float* c,
              int64_t M, int64_t N, int64_t K, int64_t ldc, cudaStream_t st, int a_sh_i, int a_sh_k, int b_sh_k,
              int b_sh_j) {
    fmt = code_format(fmt);
    if (fmt != FMT_INT8 && fmt != FMT_E4M3 && fmt != FMT_E3M2) return false;
    if (M <= 0 || N <= 0) return true;
    const DeqView A{a, as, a_si, a_sk, as_si, as_sk, a_sh_i, a_sh_k}, B{b, bs, b_sk, b_sj, bs_sk, bs_sj, b_sh_k, b_sh_j};
    const dim3 grid((unsigned)((N + DG_BN - 1) / DG_BN), (unsigned)((M + DG_BM - 1) / DG_BM));
    if (fmt == FMT_INT8)
        launch_pdl(k_deq_gemm<FMT_INT8>, grid, dim3(DG_THREADS), 0, st, A, B, c, M, N, K, ldc);
    else if (fmt == FMT_E3M2)
        launch_pdl(k_deq_gemm<FMT_E3M2>, grid, dim3(DG_THREADS), 0, st, A, B, c, M, N, K, ldc);
    else
        launch_pdl(k_deq_gemm<FMT_E4M3>, grid, dim3(DG_THREADS), 0, st, A, B, c, M, N, K, ldc);
    return cudaPeekAtLastError() == cudaSuccess;
}

// Granularity::mx quantization of NumericFormat::MxFp6E3M2 (quantize.hpp:
// 202-280): per 1 x 32 block along each row, absmax (exact), power-of-two
// scale by the MX rule (:224-232: e = ilogb(m/28), +1 if m/2^e > 28, >= -126;
// 1 for an all-zero block), codes round_code(x / s, Fp6E3M2) by the exact
// E3M2 quantizer, stored in bits 7:2.  The input is a strided view
// in[r * rs + c * cs] (cs != 1: quantize(transpose(E_Y)), :427-431); one
// thread per block, threads of a warp on consecutive blocks.
template <typename InT>
__global__ void __launch_bounds__(256) k_mx_quant(const InT* __restrict__ in, int64_t rows, int64_t cols, int64_t rs,
                                                 int64_t cs, uint8_t* __restrict__ codes, float* __restrict__ scales,
                                                 unsigned* err) {
    const int64_t nb = (cols + 31) / 32;
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= rows * nb) return;
    // consecutive threads: consecutive rows of one block column when the
    // view is transposed (coalesced reads), consecutive blocks of a row
    // otherwise
    int64_t r, cb;
    if (cs != 1) { r = g % rows; cb = g / rows; } else { r = g / nb; cb = g % nb; }
    const int64_t c0 = cb * 32, cn = cols - c0 < 32 ? cols - c0 : 32;
    float v[32];
    float m = 0.f;
    uint32_t bad = 0;
#pragma unroll
    for (int t = 0; t < 32; ++t) {
        v[t] = t < cn ? (float)in[r * rs + (c0 + t) * cs] : 0.f;
        bad |= nonfinite_bits(v[t]);
        m = fmaxf(m, fabsf(v[t]));
    }
    if (bad) atomicOr(err, ERRF_NONFINITE);
    double sd;
    if (m == 0.f) {
        sd = 1.0;
    } else {
        const double md = (double)m;
        int e = ilogb(md / 28.0);
        if (md / ldexp(1.0, e) > 28.0) ++e;
        if (e < -126) e = -126;
        sd = ldexp(1.0, e);
    }
    const float s = (float)sd, inv = (float)(1.0 / sd);  // exact: a power of two
    scales[r * nb + cb] = s;
    uint8_t* o = codes + r * cols + c0;
#pragma unroll
    for (int t = 0; t < 32; ++t)
        if (t < cn) o[t] = (uint8_t)(quant_e3m2(v[t], s, inv) << 2);
}

bool mx_quantize(int in_dtype, const void* in, int64_t rows, int64_t cols, int64_t rs, int64_t cs, uint8_t* codes,
                 float* scales, unsigned* err, cudaStream_t st) {
    if (rows <= 0 || cols <= 0) return true;
    const int64_t n = rows * ((cols + 31) / 32);
    const unsigned grid = (unsigned)((n + 255) / 256);
    if (in_dtype == DT_BF16)
        k_mx_quant<__nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(in), rows, cols, rs, cs,
                                                        codes, scales, err);
    else
        k_mx_quant<float><<<grid, 256, 0, st>>>(static_cast<const float*>(in), rows, cols, rs, cs, codes, scales, err);
    return cudaPeekAtLastError() == cudaSuccess;
}

bool col_quantize(int fmt, int in_dtype, const void* in, int64_t rows, int64_t cols, unsigned* amax, float* scales,
                  uint8_t* codes, unsigned* err, cudaStream_t st) {
    if (fmt != FMT_INT8 && fmt != FMT_E4M3) return false;
    if (rows <= 0 || cols <= 0) return true;
    cudaMemsetAsync(amax, 0, (size_t)cols * sizeof(unsigned), st);
    if (in_dtype == DT_BF16)
        col_quant_launch(fmt, static_cast<const __nv_bfloat16*>(in), rows, cols, amax, scales, codes, err, st);
    else
        col_quant_launch(fmt, static_cast<const float*>(in), rows, cols, amax, scales, codes, err, st);
    return cudaPeekAtLastError() == cudaSuccess;
}

}  // namespace halo_b200
