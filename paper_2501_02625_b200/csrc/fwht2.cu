// fwht2.cu — K1/K2/K4 production kernels for Hadamard blocks B <= 256.
//
// Same arithmetic as fwht_quant.cu (reference stage order len = 1, 2, 4, ...
// in fp32, one normalising multiply, hadamard.hpp:136-177) with far fewer
// instructions per element:
//   * no warp shuffles: a block of 256 is split into "low" index bits held
//     in one thread's registers and "high" bits reached after ONE shared-
//     memory exchange, so every butterfly is a register add/sub;
//   * the absmax pass skips the last butterfly stage: max(|u+v|, |u-v|) is
//     fl(|u|+|v|) exactly (rounding is sign-symmetric), and the normalising
//     multiply is applied once to the maximum (monotone rounding);
//   * for B = 4^k the norm 2^-k is folded exactly into the quantizer scale
//     (x*2^-k / s == x / (s*2^k) bit for bit);
//   * the fast quantizers of quant_round.cuh (exact fallback near midpoints).
//
// K1 (rows): a warp processes 4 segments of 256 contiguous elements per
//   iteration.  Coalesced 16 B loads give lane l elements 8l..8l+7 of each
//   segment (stages 1,2,4 in registers); an XOR-swizzled, conflict-free
//   transpose through shared memory gives lane (k, i) elements i + 8j,
//   j = 0..31, of segment k (stages 8..128 in registers).  Codes are staged
//   through shared memory into 16 B stores.
// K2 (cols): a CTA owns a 256-row x 64-column tile.  Warp w loads rows
//   32w..32w+31 (lane = column pair, 128 B coalesced per row), runs stages
//   1..16 in registers (and emits the un-rotated E_Y codes on the way), parks
//   the tile in shared memory, then every thread takes rows r + 32k,
//   k = 0..7, for stages 32, 64, 128.  Row-contiguous stores throughout.
#include "common.cuh"
#include "halo_internal.h"

#include <type_traits>

namespace halo_b200 {

enum : int { V2_ABSMAX = 0, V2_QUANT = 1, V2_XFORM = 2 };

// candidate code + slow flag (branch-free), and the exact path out of line
template <int FMT>
__device__ __forceinline__ uint8_t qtry(float x, float inv, uint32_t& slow) {
    if constexpr (FMT == FMT_INT8) return quant_int8_try(x, inv, slow);
    else return quant_e4m3_try(x, inv, slow);
}
template <int FMT>
__device__ __noinline__ uint8_t qexact(float x, float s, float inv) {
    if constexpr (FMT == FMT_INT8) return (uint8_t)quant_int8(x, s, inv);
    else return quant_e4m3(x, s, inv);
}

__device__ __forceinline__ void bfly(float& a, float& b) {
    const float x = a, y = b;
    a = x + y;
    b = x - y;
}

// quantizer scale with the normalisation folded in (FOLD: norm is 2^-k)
__device__ __forceinline__ void quant_scale(const unsigned* amax, const float* sup, int fmt, bool fold, float norm,
                                            float* s_q, float* inv_q, float* scale_out) {
    float s, inv;
    resolve_scale(amax, sup, fmt, &s, &inv);
    if (scale_out && blockIdx.x == 0 && threadIdx.x == 0) *scale_out = s;
    if (fold) {
        s = s / norm;  // exact: power-of-two rescale
        inv = inv * norm;
    }
    *s_q = s;
    *inv_q = inv;
}

// ===================================================================== K1
constexpr int R_SEG_PAD = 272;  // bytes per segment in the code staging buffer

template <typename InT, int FMT, int MODE, typename OutT>
__global__ void __launch_bounds__(256) k_rows_v2(const InT* __restrict__ in, int64_t n, int lb, float norm, int fold,
                                                 unsigned* absmax, const float* supplied, uint8_t* __restrict__ codes,
                                                 OutT* __restrict__ out, unsigned* err, float* scale_out) {
    __shared__ __align__(16) float xs[8][4 * 256];
    __shared__ __align__(16) uint8_t cs[8][4 * R_SEG_PAD];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int B = 1 << lb;
    float s = 1.f, inv = 1.f;
    if constexpr (MODE == V2_QUANT) quant_scale(absmax, supplied, FMT, fold, norm, &s, &inv, scale_out);
    float amax = 0.f;
    bool ok = true;
    float* X = xs[w];
    const int kk = l >> 3, il = l & 7;
    const int64_t nchunks = (n + 1023) >> 10;
    const int64_t cstride = (int64_t)gridDim.x * 8;
    // software pipeline: the next chunk's four 16/32 B loads are in flight
    // while the current chunk is transformed
    Raw8<InT> cur[4], nxt[4];
    auto load_chunk = [&](Raw8<InT>(&r)[4], int64_t cc) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int64_t e0 = (cc << 10) + k * 256 + l * 8;
            if (cc < nchunks && e0 < n) r[k].load(in + e0);
            else r[k].zero();
        }
    };
    int64_t c0 = (int64_t)blockIdx.x * 8 + w;
    load_chunk(cur, c0);
    for (int64_t c = c0; c < nchunks; c += cstride) {
        const int64_t base = c << 10;
        load_chunk(nxt, c + cstride);
        float v[4][8];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            cur[k].get(v[k]);
            cur[k] = nxt[k];
            if constexpr (MODE == V2_ABSMAX) ok = ok & finite8(v[k]);
            // low stages: len 1, 2, 4 within the lane's 8 contiguous elements
#pragma unroll
            for (int len = 1; len < 8; len <<= 1) {
                if (len < B) {
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                        if ((i & len) == 0) bfly(v[k][i], v[k][i + len]);
                }
            }
            // transpose: element e = 8l + i  ->  lane (k, i), slot j = l
#pragma unroll
            for (int i = 0; i < 8; ++i) X[k * 256 + i * 32 + ((((l >> 2) ^ i) & 7) << 2) + (l & 3)] = v[k][i];
        }
        __syncwarp();
        float u[32];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const float4 f = *reinterpret_cast<const float4*>(&X[kk * 256 + il * 32 + (((q ^ il) & 7) << 2)]);
            u[4 * q] = f.x;
            u[4 * q + 1] = f.y;
            u[4 * q + 2] = f.z;
            u[4 * q + 3] = f.w;
        }
        __syncwarp();
        // high stages: len = 8 << t  <->  bit t of j
        bool done = false;
#pragma unroll
        for (int t = 0; t < 5; ++t) {
            const int len = 8 << t, jl = 1 << t;
            if (len < B) {
                if (MODE == V2_ABSMAX && 2 * len == B) {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if ((j & jl) == 0) amax = fmaxf(amax, fabsf(u[j]) + fabsf(u[j + jl]));
                    done = true;
                } else {
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if ((j & jl) == 0) bfly(u[j], u[j + jl]);
                }
            }
        }
        if constexpr (MODE == V2_ABSMAX) {
            if (!done) {
#pragma unroll
                for (int j = 0; j < 32; ++j) amax = fmaxf(amax, fabsf(u[j]));
            }
        } else if constexpr (MODE == V2_QUANT) {
            uint8_t* C = cs[w];
            uint32_t mask = 0;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                if (!fold) u[j] *= norm;
                uint32_t sl;
                C[kk * R_SEG_PAD + il + 8 * j] = qtry<FMT>(u[j], inv, sl);
                mask |= sl << j;
            }
            if (__any_sync(0xffffffffu, mask != 0)) {
                // ~0.02% of elements sit near a midpoint: exact path, out of
                // the unrolled loop, through a lane-private scratch (X is free)
#pragma unroll
                for (int j = 0; j < 32; ++j) X[l * 32 + j] = u[j];
                while (mask) {
                    const int j = __ffs(mask) - 1;
                    mask &= mask - 1;
                    C[kk * R_SEG_PAD + il + 8 * j] = qexact<FMT>(X[l * 32 + j], s, inv);
                }
            }
            __syncwarp();
            const int64_t e0 = base + kk * 256 + il * 32;
            const uint4* src = reinterpret_cast<const uint4*>(C + kk * R_SEG_PAD + il * 32);
            if (e0 + 32 <= n) {
                uint4* dst = reinterpret_cast<uint4*>(codes + e0);
                dst[0] = src[0];
                dst[1] = src[1];
            } else {
                for (int i = 0; i < 32 && e0 + i < n; ++i) codes[e0 + i] = C[kk * R_SEG_PAD + il * 32 + i];
            }
            __syncwarp();
        } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                const int64_t e = base + kk * 256 + il + 8 * j;
                if (e < n) out[e] = (OutT)(u[j] * norm);
            }
        }
    }
    if constexpr (MODE == V2_ABSMAX) {
        amax = warp_max(amax) * norm;  // monotone: max(fl(|x| * norm)) == fl(max|x| * norm)
        const unsigned bad = __any_sync(0xffffffffu, !ok);
        if (l == 0) {
            atomic_absmax(absmax, amax);
            if (bad) atomicOr(err, ERRF_NONFINITE);
        }
    }
}

// ===================================================================== K2
constexpr int C_COLS = 64;
constexpr size_t C_SMEM = (256 * C_COLS + 256 * 16) * sizeof(float);

template <typename T>
struct Raw2;
template <>
struct Raw2<__nv_bfloat16> {
    uint32_t r;
    __device__ __forceinline__ void load(const __nv_bfloat16* p) { r = __ldg(reinterpret_cast<const unsigned int*>(p)); }
    __device__ __forceinline__ void zero() { r = 0; }
    __device__ __forceinline__ void get(float& a, float& b) const {
        a = __uint_as_float(r << 16);
        b = __uint_as_float(r & 0xFFFF0000u);
    }
};
template <>
struct Raw2<float> {
    float2 r;
    __device__ __forceinline__ void load(const float* p) { r = __ldg(reinterpret_cast<const float2*>(p)); }
    __device__ __forceinline__ void zero() { r = make_float2(0.f, 0.f); }
    __device__ __forceinline__ void get(float& a, float& b) const {
        a = r.x;
        b = r.y;
    }
};

template <typename InT, int FMT, int MODE>
__global__ void __launch_bounds__(256, 2) k_cols_v2(const InT* in, int64_t b, int64_t rows_pad, int64_t cols, int lb,
                                                 float norm, int fold, unsigned* amax_r, unsigned* amax_p,
                                                 const float* sup_r, const float* sup_p, uint8_t* __restrict__ codes_r,
                                                 uint8_t* __restrict__ codes_p, float* out, int64_t rows_out,
                                                 unsigned* err, float* sro, float* spo) {
    extern __shared__ __align__(16) float T[];  // [256][64] tile + [256][16] exact-path scratch
    float* scratch = T + 256 * C_COLS;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int B = 1 << lb;
    float s_r = 1.f, i_r = 1.f, s_p = 1.f, i_p = 1.f;
    if constexpr (MODE == V2_QUANT) {
        quant_scale(amax_r, sup_r, FMT, fold, norm, &s_r, &i_r, sro);
        quant_scale(amax_p, sup_p, FMT, false, 1.f, &s_p, &i_p, spo);
    }
    float am_r = 0.f, am_p = 0.f;
    bool ok = true;
    const int64_t ct = (cols + C_COLS - 1) / C_COLS, rt = (rows_pad + 255) / 256;
    // One tile = 256 rows x 64 columns.  Interior tiles (the common case:
    // b, rows_pad multiples of 256, cols a multiple of 64) run without any
    // bounds checks; edge tiles take the checked instantiation.
    auto run = [&](auto edge_tag, int64_t r0, int64_t c0) {
        constexpr bool EDGE = decltype(edge_tag)::value;
        const int64_t gc = c0 + 2 * l;
        const bool cok = !EDGE || gc < cols;
        const int64_t row1 = r0 + 32 * w;  // first phase-1 row of this warp
        // ---- phase 1: rows row1 + i, stages 1..16 in registers
        float a[32], bb[32];
        {
            Raw2<InT> raw[32];
            const InT* p = in + row1 * cols + gc;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                if (!EDGE || (cok && row1 + i < b)) raw[i].load(p);
                else raw[i].zero();
                p += cols;
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) raw[i].get(a[i], bb[i]);
        }
        if constexpr (MODE == V2_ABSMAX) {
            uint32_t bad = 0;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                bad |= nonfinite_bits(a[i]) | nonfinite_bits(bb[i]);
                am_p = fmaxf(am_p, fmaxf(fabsf(a[i]), fabsf(bb[i])));
            }
            ok = ok & (bad == 0);
        } else if constexpr (MODE == V2_QUANT) {
            // codes of the un-rotated E_Y (the G operand); the warp vote is
            // outside every lane-dependent branch
            uint32_t ma = 0, mb = 0;
            if (codes_p) {
                uint8_t* q = codes_p + row1 * cols + gc;
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    uint32_t s1, s2;
                    const uint32_t ca = qtry<FMT>(a[i], i_p, s1);
                    const uint32_t cb2 = qtry<FMT>(bb[i], i_p, s2);
                    if (!EDGE || (cok && row1 + i < b)) {
                        ma |= s1 << i;
                        mb |= s2 << i;
                        *reinterpret_cast<uint16_t*>(q) = (uint16_t)(ca | (cb2 << 8));
                    }
                    q += cols;
                }
            }
            if (__any_sync(0xffffffffu, (ma | mb) != 0)) {  // rare, warp-uniform exact path
#pragma unroll
                for (int i = 0; i < 32; ++i) {
                    const int64_t gr = row1 + i;
                    if ((ma >> i) & 1u) codes_p[gr * cols + gc] = qexact<FMT>(a[i], s_p, i_p);
                    if ((mb >> i) & 1u) codes_p[gr * cols + gc + 1] = qexact<FMT>(bb[i], s_p, i_p);
                }
            }
        }
#pragma unroll
        for (int t = 0; t < 5; ++t) {
            const int len = 1 << t;
            if (len < B) {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if ((i & len) == 0) {
                        bfly(a[i], a[i + len]);
                        bfly(bb[i], bb[i + len]);
                    }
            }
        }
        float* Tw = T + (32 * w) * C_COLS + 2 * l;
#pragma unroll
        for (int i = 0; i < 32; ++i) *reinterpret_cast<float2*>(Tw + i * C_COLS) = make_float2(a[i], bb[i]);
        __syncthreads();
        // ---- phase 2: rows r + 32k (r = 4w + g), stages 32, 64, 128
#pragma unroll
        for (int g = 0; g < 4; ++g) {
            const int rl = 4 * w + g;
            float x[8], y[8];
            const float* Tr = T + rl * C_COLS + 2 * l;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float2 f = *reinterpret_cast<const float2*>(Tr + 32 * k * C_COLS);
                x[k] = f.x;
                y[k] = f.y;
            }
            bool done = false;
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const int len = 32 << t, kl = 1 << t;
                if (len < B) {
                    if (MODE == V2_ABSMAX && 2 * len == B) {
#pragma unroll
                        for (int k = 0; k < 8; ++k)
                            if ((k & kl) == 0)
                                am_r = fmaxf(am_r, fmaxf(fabsf(x[k]) + fabsf(x[k + kl]), fabsf(y[k]) + fabsf(y[k + kl])));
                        done = true;
                    } else {
#pragma unroll
                        for (int k = 0; k < 8; ++k)
                            if ((k & kl) == 0) {
                                bfly(x[k], x[k + kl]);
                                bfly(y[k], y[k + kl]);
                            }
                    }
                }
            }
            const int64_t row2 = r0 + rl;  // phase-2 rows: row2 + 32k
            (void)row2;  // unused by the absmax instantiations
            if constexpr (MODE == V2_ABSMAX) {
                if (!done) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) am_r = fmaxf(am_r, fmaxf(fabsf(x[k]), fabsf(y[k])));
                }
            } else if constexpr (MODE == V2_QUANT) {
                uint32_t m = 0;
                uint8_t* q = codes_r + row2 * cols + gc;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (!fold) {
                        x[k] *= norm;
                        y[k] *= norm;
                    }
                    uint32_t s1, s2;
                    const uint32_t cx = qtry<FMT>(x[k], i_r, s1);
                    const uint32_t cy = qtry<FMT>(y[k], i_r, s2);
                    if (!EDGE || (cok && row2 + 32 * k < rows_pad)) {
                        m |= (s1 << k) | (s2 << (k + 8));
                        *reinterpret_cast<uint16_t*>(q) = (uint16_t)(cx | (cy << 8));
                    }
                    q += 32 * cols;
                }
                if (__any_sync(0xffffffffu, m != 0)) {  // rare: exact path via scratch
                    float* S = scratch + threadIdx.x * 16;
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        S[k] = x[k];
                        S[k + 8] = y[k];
                    }
                    while (m) {
                        const int qq = __ffs(m) - 1;
                        m &= m - 1;
                        const int64_t gr = row2 + 32 * (qq & 7);
                        codes_r[gr * cols + gc + (qq >> 3)] = qexact<FMT>(S[qq], s_r, i_r);
                    }
                }
            } else {
                float* o = out + row2 * cols + gc;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    if (!EDGE || (cok && row2 + 32 * k < rows_out))
                        *reinterpret_cast<float2*>(o) = make_float2(x[k] * norm, y[k] * norm);
                    o += 32 * cols;
                }
            }
        }
        __syncthreads();
    };
    for (int64_t tile = blockIdx.x; tile < ct * rt; tile += gridDim.x) {
        const int64_t r0 = (tile / ct) * 256, c0 = (tile % ct) * C_COLS;
        const int64_t rlim = MODE == V2_XFORM ? rows_out : (b < rows_pad ? b : rows_pad);
        const bool interior = (r0 + 256 <= rlim) && (r0 + 256 <= rows_pad) && (c0 + C_COLS <= cols);
        if (interior) run(std::false_type{}, r0, c0);
        else run(std::true_type{}, r0, c0);
    }
    if constexpr (MODE == V2_ABSMAX) {
        am_r = warp_max(am_r) * norm;
        am_p = warp_max(am_p);
        const unsigned bad = __any_sync(0xffffffffu, !ok);
        if (l == 0) {
            atomic_absmax(amax_r, am_r);
            atomic_absmax(amax_p, am_p);
            if (bad) atomicOr(err, ERRF_NONFINITE);
        }
    }
}

// ============================================================ launchers

static int lg2(int64_t v) {
    int l = 0;
    while ((int64_t(1) << l) < v) ++l;
    return l;
}

static unsigned cap_grid(int64_t want, int per_sm) {
    const int64_t cap = (int64_t)num_sms() * per_sm;
    if (want > cap) want = cap;
    if (want < 1) want = 1;
    return (unsigned)want;
}

template <typename InT, int FMT, int MODE, typename OutT>
static void rows_v2_launch(const InT* in, int64_t n, int64_t B, unsigned* amax, const float* sup, uint8_t* codes,
                           OutT* out, unsigned* err, float* sout, cudaStream_t st) {
    const int lb = lg2(B);
    const float norm = hadamard_norm(B);
    const int fold = (lb % 2) == 0;
    const unsigned grid = cap_grid(((n + 1023) / 1024 + 7) / 8, 5);
    k_rows_v2<InT, FMT, MODE, OutT><<<grid, 256, 0, st>>>(in, n, lb, norm, fold, amax, sup, codes, out, err, sout);
}

bool rows_v2(int mode, int fmt, int in_dtype, const void* in, int64_t n, int64_t B, unsigned* amax, const float* sup,
             uint8_t* codes, void* out, int out_dtype, unsigned* err, float* sout, cudaStream_t st) {
    if (B < 8 || B > 256) return false;
    if (mode == V2_QUANT && fmt == FMT_E3M2) return false;  // FP6: fwht3.cu / generic kernels
    if (mode == V2_XFORM) {
        if (in_dtype != DT_F32) return false;
        auto p = static_cast<const float*>(in);
        if (out_dtype == DT_BF16)
            rows_v2_launch<float, 0, V2_XFORM, __nv_bfloat16>(p, n, B, amax, sup, codes, static_cast<__nv_bfloat16*>(out), err, sout, st);
        else
            rows_v2_launch<float, 0, V2_XFORM, float>(p, n, B, amax, sup, codes, static_cast<float*>(out), err, sout, st);
        return true;
    }
#define HALO_R2(T)                                                                                                 \
    {                                                                                                              \
        auto p = static_cast<const T*>(in);                                                                        \
        if (mode == V2_ABSMAX) rows_v2_launch<T, 0, V2_ABSMAX, float>(p, n, B, amax, sup, codes, nullptr, err, sout, st); \
        else if (fmt == FMT_INT8) rows_v2_launch<T, FMT_INT8, V2_QUANT, float>(p, n, B, amax, sup, codes, nullptr, err, sout, st); \
        else rows_v2_launch<T, FMT_E4M3, V2_QUANT, float>(p, n, B, amax, sup, codes, nullptr, err, sout, st);      \
    }
    if (in_dtype == DT_BF16) HALO_R2(__nv_bfloat16) else HALO_R2(float)
#undef HALO_R2
    return true;
}

template <typename InT, int FMT, int MODE>
static void cols_v2_launch(const InT* in, int64_t b, int64_t rows_pad, int64_t cols, int64_t B, unsigned* ar,
                           unsigned* ap, const float* sr, const float* sp, uint8_t* cr, uint8_t* cp, float* out,
                           int64_t rows_out, unsigned* err, float* sro, float* spo, cudaStream_t st) {
    const int lb = lg2(B);
    const float norm = hadamard_norm(B);
    const int fold = (lb % 2) == 0;
    auto kern = k_cols_v2<InT, FMT, MODE>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C_SMEM);
        attr = true;
    }
    const int64_t tiles = ((cols + C_COLS - 1) / C_COLS) * ((rows_pad + 255) / 256);
    kern<<<cap_grid(tiles, 3), 256, C_SMEM, st>>>(in, b, rows_pad, cols, lb, norm, fold, ar, ap, sr, sp, cr, cp, out,
                                                  rows_out, err, sro, spo);
}

bool cols_v2(int mode, int fmt, int in_dtype, const void* in, int64_t b, int64_t rows_pad, int64_t cols, int64_t B,
             unsigned* ar, unsigned* ap, const float* sr, const float* sp, uint8_t* cr, uint8_t* cp, float* out,
             int64_t rows_out, unsigned* err, float* sro, float* spo, cudaStream_t st) {
    if (B > 256 || cols % 2) return false;
    if (mode == V2_QUANT && fmt == FMT_E3M2) return false;  // FP6: fwht_cols3.cu / generic kernels
    if (mode == V2_XFORM) {
        if (in_dtype != DT_F32) return false;
        cols_v2_launch<float, 0, V2_XFORM>(static_cast<const float*>(in), b, rows_pad, cols, B, ar, ap, sr, sp, cr, cp,
                                           out, rows_out, err, sro, spo, st);
        return true;
    }
#define HALO_C2(T)                                                                                                       \
    {                                                                                                                    \
        auto p = static_cast<const T*>(in);                                                                              \
        if (mode == V2_ABSMAX) cols_v2_launch<T, 0, V2_ABSMAX>(p, b, rows_pad, cols, B, ar, ap, sr, sp, cr, cp, out, rows_out, err, sro, spo, st); \
        else if (fmt == FMT_INT8) cols_v2_launch<T, FMT_INT8, V2_QUANT>(p, b, rows_pad, cols, B, ar, ap, sr, sp, cr, cp, out, rows_out, err, sro, spo, st); \
        else cols_v2_launch<T, FMT_E4M3, V2_QUANT>(p, b, rows_pad, cols, B, ar, ap, sr, sp, cr, cp, out, rows_out, err, sro, spo, st); \
    }
    if (in_dtype == DT_BF16) HALO_C2(__nv_bfloat16) else HALO_C2(float)
#undef HALO_C2
    return true;
}

}  // namespace halo_b200
