// fwht_quant.cu — K1 / K2 / K4: fused blockwise fast Walsh–Hadamard
// transform + absmax + RTN quantize, HBM-streaming, sm_100a.
//
// Reference semantics (paths relative to /root/reference/proj/include/halo):
//   * butterfly order and normalisation: hadamard.hpp:136-177 — stages with
//     stride len = 1, 2, 4, ... (u+v, u-v in fp32), then ONE multiply by
//     float(1/sqrt(double(B))).  Every element sees the same sequence of fp32
//     operations as in the reference, so results are bit-identical;
//   * right transform A*H (transform_right, :194-197) along the contiguous
//     dim; left transform H*A (transform_left_h, :213-216) along rows;
//   * blockwise extension I_{d/B} (x) H_B; B == d is the reference verbatim;
//   * per-tensor scale float(double(absmax)/fmax) (quantize.hpp:202-239),
//     codes round_code(x/s) (quantize.hpp:275) — see quant_round.cuh.
//
// A per-tensor scale needs the global absmax before any code can be written,
// so every quantizing op is two launches on one stream: phase A (transform +
// absmax -> atomicMax on a device word) and phase B (transform again +
// quantize + store).  Phase B re-reads the bf16 input; for tensors below
// ~60 MB the second read hits the 126 MB L2.  No host synchronisation: the
// scale is derived on the device from the absmax word.
//
// K1 (rows, B <= 256): one warp per 256-element chunk, 8 contiguous elements
//   per lane (one 16 B load), stages 1,2,4 in registers, 8..128 via
//   shfl.xor 1..16.  Grid-stride over chunks.
// The production kernels for 8 <= B <= 256 (rows) and B <= 256 (columns)
// live in fwht2.cu; this file keeps the warp-shuffle row kernel for B < 8
// and a CTA-per-segment shared-memory kernel for B > 256 (parity / sweep).
#include <cstdlib>

#include "common.cuh"
#include "halo_internal.h"

#include <type_traits>

namespace halo_b200 {

enum Mode : int { MODE_ABSMAX = 0, MODE_QUANT = 1, MODE_XFORM = 2 };

// ------------------------------------------------------------------ warp --
// v[0..7] = elements lane*8 .. lane*8+7 of a 256-element chunk.
// LOGB >= 0: block size fixed at compile time; LOGB < 0: runtime `lb`.
template <int LOGB>
__device__ __forceinline__ void fwht_warp(float v[8], int lane, int lb_rt) {
    const int lb = LOGB >= 0 ? LOGB : lb_rt;
#pragma unroll
    for (int len = 1; len < 8; len <<= 1) {
        if (len < (1 << lb)) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if ((i & len) == 0) {
                    const float x = v[i], y = v[i + len];
                    v[i] = x + y;
                    v[i + len] = x - y;
                }
            }
        }
    }
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        if ((8 << j) < (1 << lb)) {
            const int m = 1 << j;
            const bool upper = (lane & m) != 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const float o = __shfl_xor_sync(0xffffffffu, v[i], m);
                v[i] = upper ? (o - v[i]) : (v[i] + o);
            }
        }
    }
}

// K1 / K4-right.  n_elems = rows*cols, cols % 16 == 0, B | cols.
template <typename InT, int LOGB, int FMT, int MODE, typename OutT>
__global__ void __launch_bounds__(256) k_rows_small(const InT* __restrict__ in, int64_t n_elems, int lb, float norm,
                                                    unsigned* absmax, const float* supplied,
                                                    uint8_t* __restrict__ codes, OutT* __restrict__ out,
                                                    unsigned* err, float* scale_out) {
    const int lane = threadIdx.x & 31;
    const int64_t warp0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nchunks = (n_elems + 255) >> 8;
    float s = 1.f, inv = 1.f;
    if constexpr (MODE == MODE_QUANT) {
        resolve_scale(absmax, supplied, FMT, &s, &inv);
        if (scale_out && blockIdx.x == 0 && threadIdx.x == 0) *scale_out = s;
    }
    float amax = 0.f;
    bool ok = true;
    for (int64_t c = warp0; c < nchunks; c += nwarps) {
        const int64_t base = (c << 8) + lane * 8;
        const bool active = base < n_elems;
        float v[8];
        if (active) {
            load8(in + base, v);
        } else {
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = 0.f;
        }
        fwht_warp<LOGB>(v, lane, lb);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] *= norm;
        if constexpr (MODE == MODE_ABSMAX) {
            ok = ok && finite8(v);
#pragma unroll
            for (int i = 0; i < 8; ++i) amax = fmaxf(amax, fabsf(v[i]));
        } else if constexpr (MODE == MODE_QUANT) {
            if (active) quant_store8<FMT>(codes + base, v, s, inv);
        } else {
            if (active) store8(out + base, v);
        }
    }
    if constexpr (MODE == MODE_ABSMAX) {
        amax = warp_max(amax);
        const unsigned bad = __any_sync(0xffffffffu, !ok);
        if (lane == 0) {
            atomic_absmax(absmax, amax);
            if (bad) atomicOr(err, ERRF_NONFINITE);
        }
    }
}

// ------------------------------------------------------- large blocks (>256)
// Generic shared-memory butterfly: a CTA holds `lanes` independent
// B-element segments: segment l element i lives at
//   base + l * lane_stride + i * elem_stride   (global)
// and at tile[i * lanes + l] (shared).  Stage order as the reference.
template <typename InT, int FMT, int MODE, typename OutT>
__global__ void __launch_bounds__(256) k_generic(const InT* in, int64_t nseg_major, int64_t nseg_minor,
                                                 int64_t B, int lanes, int64_t major_stride,
                                                 int64_t lane_stride, int64_t elem_stride, int64_t valid_elems,
                                                 int64_t valid_lanes, float norm, unsigned* absmax,
                                                 const float* supplied, uint8_t* codes, OutT* out,
                                                 int64_t out_elems, unsigned* err, float* scale_out) {
    extern __shared__ __align__(16) float tile[];
    const int tid = threadIdx.x;
    float s = 1.f, inv = 1.f;
    if constexpr (MODE == MODE_QUANT) {
        resolve_scale(absmax, supplied, FMT, &s, &inv);
        if (scale_out && blockIdx.x == 0 && threadIdx.x == 0) *scale_out = s;
    }
    float amax = 0.f;
    bool ok = true;
    const int64_t ngroups = nseg_major * ((nseg_minor + lanes - 1) / lanes);
    for (int64_t gi = blockIdx.x; gi < ngroups; gi += gridDim.x) {
        const int64_t maj = gi / ((nseg_minor + lanes - 1) / lanes);
        const int64_t lane0 = (gi % ((nseg_minor + lanes - 1) / lanes)) * lanes;
        const int64_t base = maj * major_stride;
        const int64_t total = B * lanes;
        for (int64_t p = tid; p < total; p += blockDim.x) {
            const int l = (int)(p % lanes);
            const int64_t i = p / lanes;
            const int64_t gl = lane0 + l;
            const int64_t ge = maj * B + i;
            float v = 0.f;
            if (gl < valid_lanes && ge < valid_elems) v = load_elem(in + base + gl * lane_stride + i * elem_stride);
            tile[i * lanes + l] = v;
        }
        __syncthreads();
        for (int64_t len = 1; len < B; len <<= 1) {
            for (int64_t p = tid; p < (B / 2) * lanes; p += blockDim.x) {
                const int l = (int)(p % lanes);
                const int64_t pi = p / lanes;
                const int64_t i = (pi / len) * 2 * len + (pi % len);
                const float x = tile[i * lanes + l], y = tile[(i + len) * lanes + l];
                tile[i * lanes + l] = x + y;
                tile[(i + len) * lanes + l] = x - y;
            }
            __syncthreads();
        }
        for (int64_t p = tid; p < total; p += blockDim.x) {
            const int l = (int)(p % lanes);
            const int64_t i = p / lanes;
            const int64_t gl = lane0 + l;
            const int64_t ge = maj * B + i;
            const float v = tile[i * lanes + l] * norm;
            if (gl >= valid_lanes) continue;
            const int64_t off = base + gl * lane_stride + i * elem_stride;
            if constexpr (MODE == MODE_ABSMAX) {
                ok = ok && isfinite(v);
                amax = fmaxf(amax, fabsf(v));
            } else if constexpr (MODE == MODE_QUANT) {
                codes[off] = quant1<FMT>(v, s, inv);
            } else {
                if (ge < out_elems) out[off] = (OutT)v;
            }
        }
        __syncthreads();
    }
    if constexpr (MODE == MODE_ABSMAX) {
        __shared__ float red[8];
        __shared__ int redbad;
        if (tid == 0) redbad = 0;
        __syncthreads();
        amax = warp_max(amax);
        if (!ok) atomicOr(&redbad, 1);
        if ((tid & 31) == 0) red[tid >> 5] = amax;
        __syncthreads();
        if (tid == 0) {
            float m = 0.f;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) m = fmaxf(m, red[w]);
            atomic_absmax(absmax, m);
            if (redbad) atomicOr(err, ERRF_NONFINITE);
        }
    }
}

// plain (un-rotated) absmax / quantize, for HALO-0 and the plain E_Y path
template <typename InT, int FMT, int MODE>
__global__ void __launch_bounds__(256) k_plain(const InT* __restrict__ in, int64_t n_elems, unsigned* absmax,
                                               const float* supplied, uint8_t* __restrict__ codes,
                                               unsigned* err, float* scale_out) {
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    float s = 1.f, inv = 1.f;
    if constexpr (MODE == MODE_QUANT) {
        resolve_scale(absmax, supplied, FMT, &s, &inv);
        if (scale_out && blockIdx.x == 0 && threadIdx.x == 0) *scale_out = s;
    }
    float amax = 0.f;
    bool ok = true;
    for (int64_t v0 = t0 * 8; v0 < n_elems; v0 += nt * 8) {
        float v[8];
        load8(in + v0, v);
        if constexpr (MODE == MODE_ABSMAX) {
            ok = ok && finite8(v);
#pragma unroll
            for (int i = 0; i < 8; ++i) amax = fmaxf(amax, fabsf(v[i]));
        } else {
            quant_store8<FMT>(codes + v0, v, s, inv);
        }
    }
    if constexpr (MODE == MODE_ABSMAX) {
        amax = warp_max(amax);
        const unsigned bad = __any_sync(0xffffffffu, !ok);
        if ((threadIdx.x & 31) == 0) {
            atomic_absmax(absmax, amax);
            if (bad) atomicOr(err, ERRF_NONFINITE);
        }
    }
}

// ============================================================ launchers ==

static int g_num_sms = 0;
int num_sms() {
    if (!g_num_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_num_sms <= 0) g_num_sms = 148;
    }
    return g_num_sms;
}

static int ilog2i(int64_t v) {
    int l = 0;
    while ((int64_t(1) << l) < v) ++l;
    return l;
}

float hadamard_norm(int64_t B) { return (float)(1.0 / sqrt((double)B)); }

static unsigned grid_cap(int64_t want, int per_sm) {
    const int64_t cap = (int64_t)num_sms() * per_sm;
    if (want > cap) want = cap;
    if (want < 1) want = 1;
    return (unsigned)want;
}

// ---- right transform over the contiguous dim (K1 / K4-right) -----------
template <typename InT, int FMT, int MODE, typename OutT>
static void launch_rows_small(int logb, const InT* in, int64_t n, float norm, unsigned* amax, const float* sup,
                              uint8_t* codes, OutT* out, unsigned* err, float* sout, cudaStream_t st) {
    const unsigned blocks = grid_cap(((n + 255) / 256 + 7) / 8, 8);
    k_rows_small<InT, -1, FMT, MODE, OutT><<<blocks, 256, 0, st>>>(in, n, logb, norm, amax, sup, codes, out, err, sout);
}

template <typename InT, int FMT, int MODE, typename OutT>
static void launch_generic(const InT* in, int64_t nseg_major, int64_t nseg_minor, int64_t B, int lanes,
                           int64_t major_stride, int64_t lane_stride, int64_t elem_stride, int64_t valid_elems,
                           int64_t valid_lanes, float norm, unsigned* amax, const float* sup, uint8_t* codes,
                           OutT* out, int64_t out_elems, unsigned* err, float* sout, cudaStream_t st) {
    const size_t smem = (size_t)B * lanes * sizeof(float);
    auto kern = k_generic<InT, FMT, MODE, OutT>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int64_t groups = nseg_major * ((nseg_minor + lanes - 1) / lanes);
    kern<<<grid_cap(groups, 2), 256, smem, st>>>(in, nseg_major, nseg_minor, B, lanes, major_stride, lane_stride,
                                                 elem_stride, valid_elems, valid_lanes, norm, amax, sup, codes, out,
                                                 out_elems, err, sout);
}

template <typename InT, typename OutT, bool XF>
static void rows_dispatch(int mode, int fmt, const InT* in, int64_t rows, int64_t cols, int64_t B,
                          unsigned* amax, const float* sup, uint8_t* codes, OutT* out, unsigned* err, float* sout,
                          cudaStream_t st);

// quantizing modes: any input dtype; no output tensor
template <typename InT>
static void rows_quant(int mode, int fmt, const InT* in, int64_t rows, int64_t cols, int64_t B, unsigned* amax,
                       const float* sup, uint8_t* codes, unsigned* err, float* sout, cudaStream_t st) {
    rows_dispatch<InT, float, false>(mode, fmt, in, rows, cols, B, amax, sup, codes, (float*)nullptr, err, sout, st);
}

template <typename InT, typename OutT, bool XF>
static void rows_dispatch(int mode, int fmt, const InT* in, int64_t rows, int64_t cols, int64_t B,
                          unsigned* amax, const float* sup, uint8_t* codes, OutT* out, unsigned* err, float* sout,
                          cudaStream_t st) {
    const int64_t n = rows * cols;
    const float norm = hadamard_norm(B);
    if (B <= 256) {
        const int lb = ilog2i(B);
        if constexpr (XF) {
            launch_rows_small<InT, 0, MODE_XFORM, OutT>(lb, in, n, norm, amax, sup, codes, out, err, sout, st);
        } else {
            if (mode == MODE_ABSMAX) launch_rows_small<InT, 0, MODE_ABSMAX, OutT>(lb, in, n, norm, amax, sup, codes, out, err, sout, st);
            else if (fmt == FMT_INT8) launch_rows_small<InT, FMT_INT8, MODE_QUANT, OutT>(lb, in, n, norm, amax, sup, codes, out, err, sout, st);
            else if (fmt == FMT_E3M2) launch_rows_small<InT, FMT_E3M2, MODE_QUANT, OutT>(lb, in, n, norm, amax, sup, codes, out, err, sout, st);
            else launch_rows_small<InT, FMT_E4M3, MODE_QUANT, OutT>(lb, in, n, norm, amax, sup, codes, out, err, sout, st);
        }
        return;
    }
    // segments are contiguous B-element runs, one per CTA iteration
    const int64_t nseg = n / B;
#define HALO_G(F, M) launch_generic<InT, F, M, OutT>(in, nseg, 1, B, 1, B, 0, 1, n, 1, norm, amax, sup, codes, out, n, err, sout, st)
    if constexpr (XF) {
        HALO_G(0, MODE_XFORM);
    } else {
        if (mode == MODE_ABSMAX) HALO_G(0, MODE_ABSMAX);
        else if (fmt == FMT_INT8) HALO_G(FMT_INT8, MODE_QUANT);
        else if (fmt == FMT_E3M2) HALO_G(FMT_E3M2, MODE_QUANT);
        else HALO_G(FMT_E4M3, MODE_QUANT);
    }
#undef HALO_G
}

// ---- left transform over rows (K2 / K4-left) ----------------------------
template <typename InT>
static void plain_dispatch(int mode, int fmt, const InT* in, int64_t n, unsigned* amax, const float* sup,
                           uint8_t* codes, unsigned* err, float* sout, cudaStream_t st) {
    const unsigned blocks = grid_cap((n / 8 + 255) / 256, 8);
    if (mode == MODE_ABSMAX) k_plain<InT, 0, MODE_ABSMAX><<<blocks, 256, 0, st>>>(in, n, amax, sup, codes, err, sout);
    else if (fmt == FMT_INT8) k_plain<InT, FMT_INT8, MODE_QUANT><<<blocks, 256, 0, st>>>(in, n, amax, sup, codes, err, sout);
    else if (fmt == FMT_E3M2) k_plain<InT, FMT_E3M2, MODE_QUANT><<<blocks, 256, 0, st>>>(in, n, amax, sup, codes, err, sout);
    else k_plain<InT, FMT_E4M3, MODE_QUANT><<<blocks, 256, 0, st>>>(in, n, amax, sup, codes, err, sout);
}

template <typename InT>
static void cols_dispatch(int mode, int fmt, const InT* in, int64_t b, int64_t rows_pad, int64_t cols, int64_t B,
                          unsigned* ar, unsigned* ap, const float* sr, const float* sp, uint8_t* cr, uint8_t* cp,
                          float* out, int64_t rows_out, unsigned* err, float* sro, float* spo, cudaStream_t st) {
    const float norm = hadamard_norm(B);
    // large B: segments run down a column (element stride = cols); `lanes`
    // adjacent columns share a CTA.  The un-rotated E_Y path is k_plain.
    int lanes = (int)(32768 / B);
    if (lanes < 1) lanes = 1;
    if (lanes > cols) lanes = (int)cols;
    const int64_t nmaj = rows_pad / B;
#define HALO_G(F, M) launch_generic<InT, F, M, float>(in, nmaj, cols, B, lanes, B * cols, 1, cols, b, cols, norm, ar, sr, cr, out, rows_out, err, sro, st)
    if (mode == MODE_ABSMAX) {
        HALO_G(0, MODE_ABSMAX);
        if (ap) plain_dispatch<InT>(MODE_ABSMAX, fmt, in, b * cols, ap, sp, cp, err, spo, st);
    } else if (mode == MODE_XFORM) {
        if constexpr (std::is_same<InT, float>::value) HALO_G(0, MODE_XFORM);
    } else {
        if (fmt == FMT_INT8) HALO_G(FMT_INT8, MODE_QUANT);
        else if (fmt == FMT_E3M2) HALO_G(FMT_E3M2, MODE_QUANT);
        else HALO_G(FMT_E4M3, MODE_QUANT);
        if (cp) plain_dispatch<InT>(MODE_QUANT, fmt, in, b * cols, ap, sp, cp, err, spo, st);
    }
#undef HALO_G
}

// ============================================================ internal API

void run_rows(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t B, int mode, int fmt,
              unsigned* amax, const float* sup, uint8_t* codes, void* out, int out_dtype, unsigned* err,
              float* scale_out, cudaStream_t st) {
    fmt = code_format(fmt);
    // production kernels: fwht3.cu (B <= 256; TMA-staged v4, or v3 with
    // direct loads), then fwht2.cu (8 <= B <= 256); this file keeps the
    // generic paths for the remaining block sizes.  HALO_K1_VERSION=2 / 3
    // pins an older kernel (A/B measurements).
    if (base_dim_of(B)) {  // 12·2^k / 20·2^k blocks: the only path for them
        rows_base(mode, fmt, in_dtype, in, rows * cols, B, amax, sup, codes, out, out_dtype, err, scale_out, st);
        return;
    }
    const int ver = k1_version();
    const bool aligned = ((uintptr_t)in % 32 == 0) && ((uintptr_t)codes % 32 == 0) && ((uintptr_t)out % 16 == 0);
    if (ver >= 3 && aligned &&
        rows_v3(mode, fmt, in_dtype, in, rows * cols, B, amax, sup, codes, out, out_dtype, err, scale_out, st))
        return;
    if (rows_lb(mode, fmt, in_dtype, in, rows * cols, B, amax, sup, codes, out, out_dtype, err, scale_out, st))
        return;
    if (rows_big(mode, fmt, in_dtype, in, rows * cols, B, amax, sup, codes, out, out_dtype, err, scale_out, st))
        return;
    if (rows_v2(mode, fmt, in_dtype, in, rows * cols, B, amax, sup, codes, out, out_dtype, err, scale_out, st))
        return;
    if (mode != MODE_XFORM) {
        if (in_dtype == DT_BF16) rows_quant<__nv_bfloat16>(mode, fmt, static_cast<const __nv_bfloat16*>(in), rows, cols, B, amax, sup, codes, err, scale_out, st);
        else rows_quant<float>(mode, fmt, static_cast<const float*>(in), rows, cols, B, amax, sup, codes, err, scale_out, st);
        return;
    }
    // transform-only (K4): fp32 GEMM output in, fp32 or bf16 out
    auto p = static_cast<const float*>(in);
    if (out_dtype == DT_BF16) rows_dispatch<float, __nv_bfloat16, true>(mode, fmt, p, rows, cols, B, amax, sup, codes, static_cast<__nv_bfloat16*>(out), err, scale_out, st);
    else rows_dispatch<float, float, true>(mode, fmt, p, rows, cols, B, amax, sup, codes, static_cast<float*>(out), err, scale_out, st);
}

void run_cols(const void* in, int in_dtype, int64_t b, int64_t rows_pad, int64_t cols, int64_t B, int mode, int fmt,
              unsigned* amax_rot, unsigned* amax_plain, const float* sup_rot, const float* sup_plain,
              uint8_t* codes_rot, uint8_t* codes_plain, float* out, int64_t rows_out, unsigned* err,
              float* scale_rot_out, float* scale_plain_out, cudaStream_t st) {
    fmt = code_format(fmt);
    if (base_dim_of(B)) {
        cols_base(mode, fmt, in_dtype, in, b, rows_pad, cols, B, amax_rot, amax_plain, sup_rot, sup_plain, codes_rot,
                  codes_plain, err, scale_rot_out, scale_plain_out, st, out, rows_out);
        return;
    }
    if (mode != MODE_XFORM && k1_version() >= 3 &&
        cols_v3(mode, fmt, in_dtype, in, b, rows_pad, cols, B, amax_rot, amax_plain, sup_rot, sup_plain, codes_rot,
                codes_plain, err, scale_rot_out, scale_plain_out, st))
        return;
    if (cols_lb(mode, fmt, in_dtype, in, b, rows_pad, cols, B, amax_rot, amax_plain, sup_rot, sup_plain, codes_rot,
                codes_plain, err, scale_rot_out, scale_plain_out, st, out, rows_out))
        return;
    if (cols_big(mode, fmt, in_dtype, in, b, rows_pad, cols, B, amax_rot, amax_plain, sup_rot, sup_plain, codes_rot,
                 codes_plain, err, scale_rot_out, scale_plain_out, st, out, rows_out))
        return;
    if (cols_v2(mode, fmt, in_dtype, in, b, rows_pad, cols, B, amax_rot, amax_plain, sup_rot, sup_plain, codes_rot,
                codes_plain, out, rows_out, err, scale_rot_out, scale_plain_out, st))
        return;
    if (in_dtype == DT_BF16)
        cols_dispatch<__nv_bfloat16>(mode, fmt, static_cast<const __nv_bfloat16*>(in), b, rows_pad, cols, B, amax_rot,
                                     amax_plain, sup_rot, sup_plain, codes_rot, codes_plain, out, rows_out, err,
                                     scale_rot_out, scale_plain_out, st);
    else
        cols_dispatch<float>(mode, fmt, static_cast<const float*>(in), b, rows_pad, cols, B, amax_rot, amax_plain,
                             sup_rot, sup_plain, codes_rot, codes_plain, out, rows_out, err, scale_rot_out,
                             scale_plain_out, st);
}

void run_plain(const void* in, int in_dtype, int64_t n, int mode, int fmt, unsigned* amax, const float* sup,
               uint8_t* codes, unsigned* err, float* scale_out, cudaStream_t st) {
    fmt = code_format(fmt);
    if (in_dtype == DT_BF16)
        plain_dispatch<__nv_bfloat16>(mode, fmt, static_cast<const __nv_bfloat16*>(in), n, amax, sup, codes, err, scale_out, st);
    else
        plain_dispatch<float>(mode, fmt, static_cast<const float*>(in), n, amax, sup, codes, err, scale_out, st);
}

}  // namespace halo_b200
