// fwht_base.cu — Hadamard blocks of 12·2^k and 20·2^k elements (the
// reference's Kronecker bases, hadamard.hpp:62-129), sm_100a.
//
// Reference: transform_row, hadamard.hpp:136-177 with base_dim m = 12 / 20:
// Sylvester stages len = 1, 2, ..., blocks/2 over the 2^k sub-blocks of m
// elements (butterflies of whole sub-blocks), then every sub-block times the
// m x m base matrix (out[j] = sum_l blk[l] * base[l][j], accumulated in
// order over l; transpose_base: base[j][l]), then one normalising multiply.
// The bases are the Paley type-I matrices H = I + S (S the bordered
// Jacobsthal matrix of GF(11) / GF(19)), built here on the host; the
// construction reproduces the reference's tables entry for entry
// (tests/test_gpu_base_dims.py checks it against oracle/_ref).
//
// One CTA owns one vector of the block dimension (<= 20480 elements) in
// shared memory: a pass per Sylvester stage, the base products, then
// absmax / quantize / transform.  Column (token-axis) transforms run on a
// transposed copy.  This is the compatibility path for the non-power-of-two
// dims; power-of-two blocks take fwht3 / fwht_big / fwht_cols*.
#include "common.cuh"
#include "halo_internal.h"
#include "sm100.cuh"

#include <mutex>
#include <vector>

namespace halo_b200 {

namespace {

__constant__ int8_t c_base12[144];
__constant__ int8_t c_base20[400];

// Paley type I: q prime (11 or 19), m = q + 1
void paley(int q, std::vector<int8_t>& out) {
    const int m = q + 1;
    auto chi = [q](int a) {
        a = ((a % q) + q) % q;
        if (a == 0) return 0;
        int r = 1;
        for (int e = 0; e < (q - 1) / 2; ++e) r = (r * a) % q;  // Euler's criterion
        return r == 1 ? 1 : -1;
    };
    out.assign((size_t)m * m, 0);
    for (int i = 0; i < m; ++i)
        for (int j = 0; j < m; ++j) {
            int s;
            if (i == 0) s = j == 0 ? 0 : 1;
            else if (j == 0) s = -1;
            else s = chi(j - i);
            out[(size_t)i * m + j] = (int8_t)((i == j ? 1 : 0) + s);
        }
}

bool base_tables_ready() {
    static std::once_flag once;
    static bool ok = false;
    std::call_once(once, [] {
        std::vector<int8_t> b12, b20;
        paley(11, b12);
        paley(19, b20);
        ok = cudaMemcpyToSymbol(c_base12, b12.data(), 144) == cudaSuccess &&
             cudaMemcpyToSymbol(c_base20, b20.data(), 400) == cudaSuccess;
    });
    return ok;
}

__device__ __forceinline__ float bs_max3nan(float a, float b, float c) {
    float r;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

template <typename InT>
__device__ __forceinline__ float bs_ld(const InT* p) {
    if constexpr (sizeof(InT) == 2) return __bfloat162float(*p);
    else return *p;
}

// MODE 0 absmax, 1 quantize (codes), 2 transform (fp32 / bf16 out)
template <typename InT, int FMT, int MODE, typename OutT>
__global__ void __launch_bounds__(256) k_rows_base(const InT* __restrict__ in, int64_t nvec, int L, int m, int ht,
                                                   float norm, unsigned* amax, const float* supplied,
                                                   uint8_t* __restrict__ codes, OutT* __restrict__ out,
                                                   unsigned* err, float* scale_out) {
    extern __shared__ float bsm[];
    float* X = bsm;      // L floats
    float* Y = bsm + L;  // L floats
    pdl_wait();
    pdl_trigger();
    const int8_t* base = m == 12 ? c_base12 : c_base20;
    float s = 1.f, inv = 1.f;
    if constexpr (MODE == 1) {
        resolve_scale(amax, supplied, FMT, &s, &inv);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            if (scale_out) *scale_out = s;
            if (!supplied && *amax >= 0x7f800000u) atomicOr(err, ERRF_NONFINITE);
        }
    }
    const int nb = L / m;
    float am = 0.f;
    for (int64_t v = blockIdx.x; v < nvec; v += gridDim.x) {
        const InT* src = in + v * L;
        for (int i = threadIdx.x; i < L; i += blockDim.x) X[i] = bs_ld(src + i);
        __syncthreads();
        // Sylvester stages over sub-blocks (hadamard.hpp:139-151)
        for (int len = 1; len < nb; len *= 2) {
            for (int e = threadIdx.x; e < (nb / 2) * m; e += blockDim.x) {
                const int pair = e / m, l = e - pair * m;
                const int i = (pair / len) * 2 * len + pair % len;  // first sub-block of the pair
                const float x = X[i * m + l], y = X[(i + len) * m + l];
                X[i * m + l] = __fadd_rn(x, y);
                X[(i + len) * m + l] = __fadd_rn(x, -y);
            }
            __syncthreads();
        }
        // base products (hadamard.hpp:152-172), sequential over l
        for (int e = threadIdx.x; e < L; e += blockDim.x) {
            const int k = e / m, j = e - k * m;
            const float* blk = X + k * m;
            float acc = 0.f;
            for (int l = 0; l < m; ++l) {
                const int b = ht ? base[j * m + l] : base[l * m + j];
                acc = __fadd_rn(acc, b > 0 ? blk[l] : -blk[l]);
            }
            Y[e] = __fmul_rn(acc, norm);  // the normalising multiply (:174-176)
        }
        __syncthreads();
        for (int i = threadIdx.x; i < L; i += blockDim.x) {
            const float y = Y[i];
            const int64_t e = v * L + i;
            if constexpr (MODE == 0) {
                am = bs_max3nan(am, fabsf(y), 0.f);
            } else if constexpr (MODE == 1) {
                uint8_t c;
                if constexpr (FMT == FMT_INT8) c = (uint8_t)quant_int8(y, s, inv);
                else if constexpr (FMT == FMT_E3M2) c = (uint8_t)(quant_e3m2(y, s, inv) << 2);
                else c = quant_e4m3(y, s, inv);
                codes[e] = c;
            } else {
                if constexpr (sizeof(OutT) == 4) out[e] = y;
                else out[e] = __float2bfloat16_rn(y);
            }
        }
        __syncthreads();
    }
    if constexpr (MODE == 0) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) am = bs_max3nan(am, __shfl_xor_sync(0xffffffffu, am, o), 0.f);
        if ((threadIdx.x & 31) == 0) {
            atomic_absmax(amax, fabsf(am));
            if (!(am <= 3.402823466e38f)) atomicOr(err, ERRF_NONFINITE);
        }
    }
}

// tiled transpose with zero rows past `valid` (pad): out[c][r] = in[r][c]
template <typename T>
__global__ void k_transpose(const T* __restrict__ in, int64_t rows, int64_t valid, int64_t cols, T* __restrict__ out) {
    __shared__ T tile[32][33];
    const int64_t r0 = (int64_t)blockIdx.y * 32, c0 = (int64_t)blockIdx.x * 32;
    pdl_wait();
    pdl_trigger();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        T v = static_cast<T>(0.0f);
        if (r < valid && c < cols) v = in[r * cols + c];
        tile[i][threadIdx.x] = v;
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (c < cols && r < rows) out[c * rows + r] = tile[threadIdx.x][i];
    }
}

template <typename T>
void transpose(const void* in, int64_t rows, int64_t valid, int64_t cols, void* out, cudaStream_t st) {
    dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
    launch_pdl(k_transpose<T>, grid, dim3(32, 8), 0, st, static_cast<const T*>(in), rows, valid, cols,
               static_cast<T*>(out));
}

thread_local int t_transpose_base = 0;

template <typename InT, typename OutT>
void rb_launch(int mode, int fmt, const InT* in, int64_t n, int L, int m, int ht, unsigned* amax, const float* sup,
               uint8_t* codes, OutT* out, unsigned* err, float* sout, cudaStream_t st) {
    const size_t smem = (size_t)2 * L * sizeof(float);
    const int64_t nvec = n / L;
    const int64_t cap = (int64_t)num_sms() * (smem > 100000 ? 1 : 2);
    const unsigned grid = (unsigned)(nvec < cap ? nvec : cap);
    const float norm = (float)(1.0 / sqrt((double)L));
#define HALO_RB(F, M)                                                                                             \
    {                                                                                                             \
        auto k = k_rows_base<InT, F, M, OutT>;                                                                    \
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);                          \
        launch_pdl(k, dim3(grid), dim3(256), smem, st, in, nvec, L, m, ht, norm, amax, sup, codes, out, err, sout); \
    }
    if (mode == 0) HALO_RB(0, 0)
    else if (mode == 2) HALO_RB(0, 2)
    else if (fmt == FMT_INT8) HALO_RB(FMT_INT8, 1)
    else if (fmt == FMT_E3M2) HALO_RB(FMT_E3M2, 1)
    else HALO_RB(FMT_E4M3, 1)
#undef HALO_RB
}

}  // namespace

BaseScope::BaseScope(bool transpose_base) { t_transpose_base = transpose_base ? 1 : 0; }
BaseScope::~BaseScope() { t_transpose_base = 0; }

int base_dim_of(int64_t B) {
    if (B < 12) return 0;
    int64_t odd = B;
    while (odd % 2 == 0) odd /= 2;
    if (odd == 3 && B % 12 == 0) return 12;
    if (odd == 5 && B % 20 == 0) return 20;
    return 0;
}

// rows: K1 (modes 0/1, bf16 or fp32 in) and K4-right (mode 2, fp32 in) for
// B = 12·2^k / 20·2^k <= 20480; the transform orientation comes from the
// enclosing BaseScope (H for transform_right, H^T for transform_right_ht)
bool rows_base(int mode, int fmt, int in_dtype, const void* in, int64_t n, int64_t B, unsigned* amax,
               const float* sup, uint8_t* codes, void* out, int out_dtype, unsigned* err, float* sout,
               cudaStream_t st) {
    const int m = base_dim_of(B);
    if (!m || B > 20480 || n % B || !base_tables_ready()) return false;
    if (mode == 2 && in_dtype != DT_F32) return false;
    const int ht = t_transpose_base;
    if (mode == 2) {
        if (out_dtype == DT_BF16)
            rb_launch<float, __nv_bfloat16>(2, fmt, static_cast<const float*>(in), n, (int)B, m, ht, amax, sup, codes,
                                            static_cast<__nv_bfloat16*>(out), err, sout, st);
        else
            rb_launch<float, float>(2, fmt, static_cast<const float*>(in), n, (int)B, m, ht, amax, sup, codes,
                                    static_cast<float*>(out), err, sout, st);
    } else if (in_dtype == DT_BF16) {
        rb_launch<__nv_bfloat16, float>(mode, fmt, static_cast<const __nv_bfloat16*>(in), n, (int)B, m, ht, amax, sup,
                                        codes, nullptr, err, sout, st);
    } else {
        rb_launch<float, float>(mode, fmt, static_cast<const float*>(in), n, (int)B, m, ht, amax, sup, codes, nullptr,
                                err, sout, st);
    }
    return true;
}

// cols: K2 (modes 0/1 over the token axis, rows >= b zero) and K4-left
// (mode 2) by transposing to rows, running rows_base, transposing back
bool cols_base(int mode, int fmt, int in_dtype, const void* in, int64_t b, int64_t rows_pad, int64_t cols, int64_t B,
               unsigned* ar, unsigned* ap, const float* sr, const float* sp, uint8_t* cr, uint8_t* cp, unsigned* err,
               float* sro, float* spo, cudaStream_t st, float* xout, int64_t rows_out) {
    const int m = base_dim_of(B);
    if (!m || B > 20480 || rows_pad % B || !base_tables_ready()) return false;
    if (mode == 2 && (in_dtype != DT_F32 || !xout)) return false;
    const size_t esz = in_dtype == DT_BF16 ? 2 : 4;
    const int64_t n = rows_pad * cols;
    // stream-ordered scratch (transposed copies), freed after use
    void *t_in = nullptr, *t_out = nullptr;
    retain_async_pool();
    if (cudaMallocAsync(&t_in, (size_t)n * (mode == 2 ? 4 : esz), st) != cudaSuccess) return false;
    if (cudaMallocAsync(&t_out, (size_t)n * (mode == 2 ? 4 : 1), st) != cudaSuccess) {
        cudaFreeAsync(t_in, st);
        return false;
    }
    struct Release {
        void *a, *b;
        cudaStream_t s;
        ~Release() {
            cudaFreeAsync(a, s);
            cudaFreeAsync(b, s);
        }
    } release{t_in, t_out, st};
    if (esz == 2) transpose<__nv_bfloat16>(in, rows_pad, b, cols, t_in, st);
    else transpose<float>(in, rows_pad, b, cols, t_in, st);
    if (mode == 2) {
        rows_base(2, fmt, DT_F32, t_in, n, B, nullptr, nullptr, nullptr, t_out, DT_F32, err, nullptr, st);
        // back to [rows_out x cols] (rows past rows_out dropped: take_rows)
        transpose<float>(t_out, cols, cols, rows_pad, t_in, st);
        cudaMemcpy2DAsync(xout, (size_t)cols * 4, t_in, (size_t)cols * 4, (size_t)cols * 4, (size_t)rows_out,
                          cudaMemcpyDeviceToDevice, st);
        return true;
    }
    if (mode == 0) {
        rows_base(0, fmt, in_dtype, t_in, n, B, ar, nullptr, nullptr, nullptr, 0, err, nullptr, st);
        if (ap && !sp) run_plain(in, in_dtype, b * cols, 0, fmt, ap, nullptr, nullptr, err, nullptr, st);
        return true;
    }
    rows_base(1, fmt, in_dtype, t_in, n, B, ar, sr, static_cast<uint8_t*>(t_out), nullptr, 0, err, sro, st);
    transpose<uint8_t>(t_out, cols, cols, rows_pad, cr, st);
    if (cp) run_plain(in, in_dtype, b * cols, 1, fmt, ap, sp, cp, err, spo, st);
    return true;
}

}  // namespace halo_b200
