// fwht_big.cu — K1 / K4 for large Hadamard blocks, sm_100a: the right-hand
// blockwise FWHT with B = 2^LB, 512 <= B <= 16384 (the reference's
// full-dimension transform when had_block = 0, e.g. B = in_features = 4096),
// fused with the per-tensor absmax (phase A), the quantizer (phase B) or the
// bare transform (K4 un-rotation).
//
// Reference: transform_row, hadamard.hpp:136-177 with base_dim 1 (stages
// len = 1, 2, 4, ..., B/2 over the whole row, one normalising multiply by
// float(1/sqrt(B))); codes by quantize.hpp:244-280 (quant_round.cuh).
// Bit-exact: the same fp32 butterflies in the same stage order.
//
// Layout: a 256-thread CTA owns a tile of T = max(B, 4096) contiguous
// elements (T/B whole blocks) in shared memory as fp32 (16-64 KB).  The LB
// stage bits are processed four at a time ("radix-16 rounds"): in round r a
// thread holds the 16 elements whose index differs only in bits
// [4r, 4r+4), runs those four stages in registers and writes them back.
// Round 0 reads straight from global (16 contiguous elements per thread),
// the last round of an absmax pass reduces |u|+|v| instead of writing back,
// and the quantize / transform passes end with one coalesced sweep over the
// tile.  Stage order across rounds is increasing, as the reference's.
#include "common.cuh"
#include "halo_internal.h"
#include "sm100.cuh"

namespace halo_b200 {

namespace {

enum : int { BG_ABSMAX = 0, BG_QUANT = 1, BG_XFORM = 2 };
constexpr int BG_THREADS = 256;

__device__ __forceinline__ float bg_max3nan(float a, float b, float c) {
    float r;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

template <typename InT>
__device__ __forceinline__ void bg_load16(const InT* p, float (&v)[16]) {
    if constexpr (sizeof(InT) == 2) {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(p));
        const uint4 b = __ldg(reinterpret_cast<const uint4*>(p) + 1);
        const uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            v[2 * i] = __uint_as_float(w[i] << 16);
            v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(p) + i);
            v[4 * i] = q.x;
            v[4 * i + 1] = q.y;
            v[4 * i + 2] = q.z;
            v[4 * i + 3] = q.w;
        }
    }
}

// stages over the W low bits of the 16-slot register index (slot j <-> index
// bits), in increasing order; `abs_last`: the final stage of the whole
// transform becomes the exact absmax max(|u+v|, |u-v|) = |u| + |v|
template <int W, bool ABS_LAST>
__device__ __forceinline__ void bg_stages(float (&v)[16], float& amax) {
#pragma unroll
    for (int t = 0; t < W; ++t) {
        const int h = 1 << t;
        const bool last = ABS_LAST && t == W - 1;
#pragma unroll
        for (int j = 0; j < (1 << W); ++j) {
            if ((j & h) == 0) {
                const float a = v[j], b = v[j + h];
                if (last) {
                    amax = bg_max3nan(amax, fabsf(a) + fabsf(b), 0.f);
                } else {
                    v[j] = __fadd_rn(a, b);
                    v[j + h] = __fadd_rn(a, -b);
                }
            }
        }
    }
}

template <int FMT, bool SUP>
struct BgQuant {
    float s, inv, h;
    float2 ilo2, ihi2;
    __device__ __forceinline__ void init(const unsigned* amax, const float* supplied, float fold, float* scale_out) {
        resolve_scale(amax, supplied, FMT, &s, &inv);
        if (scale_out && blockIdx.x == 0 && threadIdx.x == 0) *scale_out = s;
        s = s / fold;  // exact power-of-two rescale (1 when not folded)
        inv = inv * fold;
        h = half_margin(s);
        if (FMT != FMT_INT8) e4m3_brackets(inv, ilo2, ihi2);
    }
    // 4 values -> code word (certified fast path, exact fallback)
    __device__ __forceinline__ uint32_t q4(float4 x) const {
        if constexpr (FMT == FMT_INT8) {
            const float xs[4] = {x.x, x.y, x.z, x.w};
            uint32_t w = 0;
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                uint32_t slow;
                uint8_t c = quant_int8_try_r(xs[i], s, inv, h, slow);
                if (slow) c = (uint8_t)quant_int8(xs[i], s, inv);
                w |= (uint32_t)c << (8 * i);
            }
            return w;
        } else if constexpr (FMT == FMT_E3M2) {
            return e3m2x4_fast(make_float2(x.x, x.y), make_float2(x.z, x.w), ilo2, ihi2, s);
        } else {
            uint32_t bad = 0;
            return e4m3x4_fast(make_float2(x.x, x.y), make_float2(x.z, x.w), ilo2, ihi2, s, bad);
        }
    }
};

template <int LB, typename InT, int FMT, int MODE, bool SUP, typename OutT>
__global__ void __launch_bounds__(BG_THREADS)
    k_rows_big(const InT* __restrict__ in, int64_t n, float norm, unsigned* amax_word, const float* supplied,
               uint8_t* __restrict__ codes, OutT* __restrict__ out, unsigned* err, float* scale_out) {
    constexpr int B = 1 << LB;
    constexpr int T = B > 4096 ? B : 4096;  // tile: whole blocks, >= one group per thread
    constexpr int GROUPS = T / 16;
    constexpr int ROUNDS = (LB + 3) / 4;
    constexpr bool FOLD = (LB % 2) == 0;
    extern __shared__ __align__(16) float S[];
    pdl_wait();
    pdl_trigger();

    BgQuant<FMT, SUP> q;
    if constexpr (MODE == BG_QUANT) {
        q.init(amax_word, supplied, FOLD ? norm : 1.f, scale_out);
        if (blockIdx.x == 0 && threadIdx.x == 0 && !SUP && *amax_word >= 0x7f800000u) atomicOr(err, ERRF_NONFINITE);
    }
    float amax = 0.f;
    const int64_t tiles = (n + T - 1) / T;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const InT* src = in + tile * T;
        // the last tile may hold fewer (whole) blocks
        const int te = (int)((n - tile * T) < T ? (n - tile * T) : T);
        // ---- round 0: bits [0, 4) from global, 16 contiguous elements
#pragma unroll
        for (int g = threadIdx.x; g < GROUPS; g += BG_THREADS) {
            if (g * 16 >= te) break;
            float v[16];
            bg_load16<InT>(src + g * 16, v);
            bg_stages<4, false>(v, amax);
            float4* d = reinterpret_cast<float4*>(S + g * 16);
#pragma unroll
            for (int i = 0; i < 4; ++i) d[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
        __syncthreads();
        // ---- rounds 1..: bits [4r, 4r + w)
#pragma unroll
        for (int r = 1; r < ROUNDS; ++r) {
            const int s = 4 * r;
            const int w = (LB - s) < 4 ? (LB - s) : 4;
            const bool last = r == ROUNDS - 1;
            const int per = te >> w;  // groups of 2^w elements
#pragma unroll 1
            for (int g = threadIdx.x; g < per; g += BG_THREADS) {
                const int base = (g & ((1 << s) - 1)) | ((g >> s) << (s + w));
                float v[16];
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (j < (1 << w)) v[j] = S[base + (j << s)];
                if (MODE == BG_ABSMAX && last) {
                    switch (w) {
                    case 1: bg_stages<1, true>(v, amax); break;
                    case 2: bg_stages<2, true>(v, amax); break;
                    case 3: bg_stages<3, true>(v, amax); break;
                    default: bg_stages<4, true>(v, amax); break;
                    }
                } else {
                    switch (w) {
                    case 1: bg_stages<1, false>(v, amax); break;
                    case 2: bg_stages<2, false>(v, amax); break;
                    case 3: bg_stages<3, false>(v, amax); break;
                    default: bg_stages<4, false>(v, amax); break;
                    }
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (j < (1 << w)) S[base + (j << s)] = v[j];
                }
            }
            __syncthreads();
        }
        // ---- final sweep: normalise, then codes / transformed values
        if constexpr (MODE != BG_ABSMAX) {
            const float4* S4 = reinterpret_cast<const float4*>(S);
#pragma unroll 4
            for (int i = threadIdx.x; i < te / 4; i += BG_THREADS) {
                float4 x = S4[i];
                if (MODE == BG_XFORM || !FOLD) {
                    x.x = __fmul_rn(x.x, norm);
                    x.y = __fmul_rn(x.y, norm);
                    x.z = __fmul_rn(x.z, norm);
                    x.w = __fmul_rn(x.w, norm);
                }
                const int64_t e = tile * T + (int64_t)i * 4;
                if constexpr (MODE == BG_QUANT) {
                    reinterpret_cast<uint32_t*>(codes + e)[0] = q.q4(x);
                } else if constexpr (sizeof(OutT) == 4) {
                    *reinterpret_cast<float4*>(out + e) = x;
                } else {
                    *reinterpret_cast<uint2*>(out + e) = make_uint2(pack_bf16x2(x.x, x.y), pack_bf16x2(x.z, x.w));
                }
            }
            __syncthreads();  // the next tile's round 0 overwrites S
        }
    }
    if constexpr (MODE == BG_ABSMAX) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) amax = bg_max3nan(amax, __shfl_xor_sync(0xffffffffu, amax, o), 0.f);
        amax *= norm;  // monotone: max(fl(|x| * norm)) == fl(max|x| * norm)
        if ((threadIdx.x & 31) == 0) {
            atomic_absmax(amax_word, fabsf(amax));
            if (!(amax <= 3.402823466e38f)) atomicOr(err, ERRF_NONFINITE);
        }
    }
}

template <int LB, typename InT, int FMT, int MODE, bool SUP, typename OutT>
void bg_launch(const InT* in, int64_t n, unsigned* amax, const float* sup, uint8_t* codes, OutT* out, unsigned* err,
               float* sout, cudaStream_t st) {
    constexpr int B = 1 << LB;
    constexpr int T = B > 4096 ? B : 4096;
    const size_t smem = (size_t)T * sizeof(float);
    auto kern = k_rows_big<LB, InT, FMT, MODE, SUP, OutT>;
    static int per_sm = 0;
    if (!per_sm) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BG_THREADS, smem);
        if (per_sm < 1) per_sm = 1;
    }
    const int64_t tiles = (n + T - 1) / T;
    const int64_t cap = (int64_t)num_sms() * per_sm;
    const unsigned grid = (unsigned)(tiles < cap ? (tiles < 1 ? 1 : tiles) : cap);
    launch_pdl(kern, dim3(grid), dim3(BG_THREADS), smem, st, in, n, hadamard_norm(B), amax, sup, codes, out, err, sout);
}

template <int LB>
void bg_dispatch(int mode, int fmt, int in_dtype, const void* in, int64_t n, unsigned* amax, const float* sup,
                 uint8_t* codes, void* out, int out_dtype, unsigned* err, float* sout, cudaStream_t st) {
    using bf = __nv_bfloat16;
    if (mode == BG_XFORM) {
        auto p = static_cast<const float*>(in);
        if (out_dtype == DT_BF16) bg_launch<LB, float, 0, BG_XFORM, false, bf>(p, n, amax, sup, codes, static_cast<bf*>(out), err, sout, st);
        else bg_launch<LB, float, 0, BG_XFORM, false, float>(p, n, amax, sup, codes, static_cast<float*>(out), err, sout, st);
        return;
    }
#define HALO_BGQ(T, F)                                                                                          \
    {                                                                                                           \
        if (sup) bg_launch<LB, T, F, BG_QUANT, true, float>(p, n, amax, sup, codes, nullptr, err, sout, st);    \
        else bg_launch<LB, T, F, BG_QUANT, false, float>(p, n, amax, sup, codes, nullptr, err, sout, st);       \
    }
#define HALO_BG(T)                                                                                              \
    {                                                                                                           \
        auto p = static_cast<const T*>(in);                                                                     \
        if (mode == BG_ABSMAX) bg_launch<LB, T, 0, BG_ABSMAX, false, float>(p, n, amax, sup, codes, nullptr, err, sout, st); \
        else if (fmt == FMT_INT8) HALO_BGQ(T, FMT_INT8)                                                         \
        else if (fmt == FMT_E3M2) HALO_BGQ(T, FMT_E3M2)                                                         \
        else HALO_BGQ(T, FMT_E4M3)                                                                              \
    }
    if (in_dtype == DT_BF16) HALO_BG(bf) else HALO_BG(float)
#undef HALO_BG
#undef HALO_BGQ
}

}  // namespace

// modes 0 absmax / 1 quantize / 2 transform (fp32 in); 512 <= B <= 16384,
// B a power of two; n a multiple of B and 32 / 16 B aligned operands.
bool rows_big(int mode, int fmt, int in_dtype, const void* in, int64_t n, int64_t B, unsigned* amax, const float* sup,
              uint8_t* codes, void* out, int out_dtype, unsigned* err, float* sout, cudaStream_t st) {
    if (B < 512 || B > 16384 || (B & (B - 1))) return false;
    if (n % B) return false;
    if (mode == BG_XFORM && in_dtype != DT_F32) return false;
    if ((uintptr_t)in % 32 || (uintptr_t)codes % 16 || (uintptr_t)out % 16) return false;
    int lb = 0;
    while ((int64_t(1) << lb) < B) ++lb;
    switch (lb) {
    case 9: bg_dispatch<9>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    case 10: bg_dispatch<10>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    case 11: bg_dispatch<11>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    case 12: bg_dispatch<12>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    case 13: bg_dispatch<13>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    default: bg_dispatch<14>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    }
    return true;
}

}  // namespace halo_b200
