// fwht_cols3.cu — K2, third generation: left (token-axis) blockwise FWHT of
// the output gradient E_Y [b x n] fused with the HALO-2 dual quantization,
// sm_100a.
//
// Reference: error_path, halo_linear.hpp:381-411 — (H_b pad(E_Y))_Q for the
// E GEMM (:393-399) and the un-rotated (E_Y)_Q for the G GEMM (:371, shared
// with the gradient path :433); transform_left, hadamard.hpp:205-216 (the
// row transform of hadamard.hpp:136-177 applied down each column, stages
// len = 1, 2, 4, ... over the row index, one normalising multiply); codes by
// quantize.hpp:244-280 (quant_round.cuh).  Bit-exact with the reference.
//
// Layout: a 4-warp CTA owns a 256-row x 32-column tile (every code store
// of a warp covers whole 32 B sectors: 8 lanes x 4 codes per row; narrower
// strips measured 3x slower from partial-sector writes).  Phase 1: thread
// (column group cg = lane & 7, row group q = 4*warp + lane/8) loads rows
// 16q + m, m = 0..15, four columns each (8 B), emits the plain codes, and
// runs row-bit stages len = 1..8 in registers.  Column pairs share a
// register pair, so every butterfly is an FADD2 (no scalar stage at all,
// unlike the row kernel).  One fp32 exchange through 32 KB of shared memory
// (row-major, 128 B rows, conflict-free) hands thread (cg, mm) rows
// 16i + mm, i = 0..15, for stages len = 16..128; small CTAs keep 4 of them
// per SM so the two barriers per tile overlap across CTAs.  Absmax passes skip the last stage
// (max(|u+v|,|u-v|) = |u|+|v| exactly) and propagate NaN.
#include "common.cuh"
#include "halo_internal.h"
#include "sm100.cuh"

#include <cstdlib>
#include <cstring>
#include <type_traits>

namespace halo_b200 {

namespace {

__device__ __forceinline__ float2 c3_add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 c3_sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 c3_mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ void c3_bfly(float2& a, float2& b) {
    const float2 x = a, y = b;
    a = c3_add2(x, y);
    b = c3_sub2(x, y);
}
__device__ __forceinline__ float c3_max3nan(float a, float b, float c) {
    float r;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ float c3_fmax3(float a, float b, float c) { return fmaxf(fmaxf(a, b), c); }
__device__ __forceinline__ uint32_t c3_pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

// 4 consecutive columns of one row -> two float2
template <typename InT>
__device__ __forceinline__ void c3_load4(const InT* p, bool ok, float2& a, float2& b);
template <>
__device__ __forceinline__ void c3_load4<__nv_bfloat16>(const __nv_bfloat16* p, bool ok, float2& a, float2& b) {
    uint2 r = make_uint2(0, 0);
    if (ok) r = __ldg(reinterpret_cast<const uint2*>(p));
    a = make_float2(__uint_as_float(r.x << 16), __uint_as_float(r.x & 0xFFFF0000u));
    b = make_float2(__uint_as_float(r.y << 16), __uint_as_float(r.y & 0xFFFF0000u));
}
template <>
__device__ __forceinline__ void c3_load4<float>(const float* p, bool ok, float2& a, float2& b) {
    float4 r = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ok) r = __ldg(reinterpret_cast<const float4*>(p));
    a = make_float2(r.x, r.y);
    b = make_float2(r.z, r.w);
}

template <int FMT>
__device__ __noinline__ uint32_t c3_exact4(float2 a, float2 b, float s, float inv) {
    if constexpr (FMT == FMT_INT8)
        return c3_pack4((uint8_t)quant_int8(a.x, s, inv), (uint8_t)quant_int8(a.y, s, inv),
                        (uint8_t)quant_int8(b.x, s, inv), (uint8_t)quant_int8(b.y, s, inv));
    else if constexpr (FMT == FMT_E3M2)
        return c3_pack4(quant_e3m2(a.x, s, inv) << 2, quant_e3m2(a.y, s, inv) << 2, quant_e3m2(b.x, s, inv) << 2,
                        quant_e3m2(b.y, s, inv) << 2);
    else
        return c3_pack4(quant_e4m3(a.x, s, inv), quant_e4m3(a.y, s, inv), quant_e4m3(b.x, s, inv),
                        quant_e4m3(b.y, s, inv));
}

template <int FMT>
__device__ __forceinline__ bool c3_group_slow(float2 a, float2 b, float s, float inv, float h) {
    const float x[4] = {a.x, a.y, b.x, b.y};
    bool slow = false;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        uint32_t sl;
        if constexpr (FMT == FMT_INT8) (void)quant_int8_try_r(x[i], s, inv, h, sl);
        else sl = 1;  // E4M3: the bracket test is per word; redo the group exactly
        slow |= sl != 0;
    }
    return slow;
}

// rare exact path, out of line: the caller parks the lane's values in a
// local array only when the warp vote fired, so the hot loop keeps no
// local-memory traffic and stays small in the instruction cache
template <int FMT>
__device__ __noinline__ void c3_fix(const float4* v, int cnt, uint32_t valid, uint8_t* dst, int64_t stride, float s,
                                    float inv, float h) {
    for (int g = 0; g < cnt; ++g) {
        if (!((valid >> g) & 1u)) continue;
        const float2 a = make_float2(v[g].x, v[g].y), c = make_float2(v[g].z, v[g].w);
        if (c3_group_slow<FMT>(a, c, s, inv, h)) *reinterpret_cast<uint32_t*>(dst + g * stride) = c3_exact4<FMT>(a, c, s, inv);
    }
}

template <int FMT, bool SUP>
struct Quant {
    float s, inv, thr;
    float2 inv2, nsm2, ilo2, ihi2;
    __device__ __forceinline__ void init(const unsigned* amax, const float* supplied, float fold_norm,
                                         float* scale_out, unsigned* err) {
        resolve_scale(amax, supplied, FMT, &s, &inv);
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            if (scale_out) *scale_out = s;
            if (!supplied && *amax >= 0x7f800000u) atomicOr(err, ERRF_NONFINITE);
        }
        s = s / fold_norm;  // exact power-of-two rescale (1 when not folded)
        inv = inv * fold_norm;
        inv2 = make_float2(inv, inv);
        nsm2 = make_float2(-s, -s);
        thr = FMT == FMT_INT8 ? half_margin(s) : 0.5f;
        if (FMT != FMT_INT8) e4m3_brackets(inv, ilo2, ihi2);
    }
    // 4 values -> code word; running maximum of the certification residual
    // (INT8: quant_int8_try_r; slow path when it reaches thr)
    __device__ __forceinline__ uint32_t q4(float2 a, float2 c, float& dmax) const {
        if constexpr (FMT == FMT_INT8) {
            const float2 m2 = make_float2(kRoundMagic, kRoundMagic);
            const float2 ta = __ffma2_rn(a, inv2, m2), tc = __ffma2_rn(c, inv2, m2);
            const float2 qa = c3_sub2(ta, m2), qc = c3_sub2(tc, m2);
            const float2 ra = __ffma2_rn(qa, nsm2, a), rc = __ffma2_rn(qc, nsm2, c);
            float m = c3_fmax3(c3_fmax3(0.f, fabsf(ra.x), fabsf(ra.y)), fabsf(rc.x), fabsf(rc.y));
            if (SUP)  // |q| <= 127 maps below thr, |q| >= 128 above it
                m = fmaxf(m, c3_fmax3(c3_fmax3(0.f, fabsf(qa.x), fabsf(qa.y)), fabsf(qc.x), fabsf(qc.y)) * (thr / 127.5f));
            // uncertified group: decide its 4 codes exactly right here
            if (!(m < thr)) return c3_exact4<FMT>(a, c, s, inv);
            return c3_pack4(__float_as_uint(ta.x), __float_as_uint(ta.y), __float_as_uint(tc.x), __float_as_uint(tc.y));
        } else if constexpr (FMT == FMT_E3M2) {
            return e3m2x4_fast(a, c, ilo2, ihi2, s);
        } else {
            uint32_t bad = 0;
            const uint32_t w = e4m3x4_fast(a, c, ilo2, ihi2, s, bad);
            dmax = bad ? 1.0f : dmax;
            return w;
        }
    }
};

enum : int { C3_ABSMAX = 0, C3_QUANT = 1 };
constexpr int C3_COLS = 32, C3_ROWS = 256;  // one CTA tile
constexpr int C3_WARPS = 4;
constexpr size_t C3_SMEM = (size_t)C3_ROWS * C3_COLS * sizeof(float);  // 32 KB fp32 exchange
constexpr int C3_STAGE = C3_ROWS * C3_COLS * 2;                         // 16 KB bf16 TMA stage
constexpr int C3_TS = 1;                                                // TMA ring depth (bf16)

}  // namespace

// TS > 0 (bf16 input): the CTA's tiles stream through a TS-deep ring of
// 16 KB shared-memory stages filled by TMA (box 32 columns x 256 rows, rows
// past b and columns past `cols` zero-filled by the copy engine); thread 0
// refills a stage right after the tile's first exchange barrier, when every
// thread has read it, so the next tiles' HBM latency hides behind compute.
template <int LB, typename InT, int FMT, int MODE, bool SUP_R, bool SUP_P, int TS>
__global__ void __launch_bounds__(128, 4)
    k_cols_v3(const __grid_constant__ CUtensorMap tm, const InT* __restrict__ in, int64_t b, int64_t rows_pad, int64_t cols, float norm, unsigned* amax_r,
              unsigned* amax_p, const float* sup_r, const float* sup_p, uint8_t* __restrict__ codes_r,
              uint8_t* __restrict__ codes_p, unsigned* err, float* sro, float* spo) {
    constexpr bool FOLD = (LB % 2) == 0;
    constexpr int P1 = LB < 4 ? LB : 4;  // row bits handled in phase 1
    constexpr int P2 = LB > 4 ? LB - 4 : 0;
    extern __shared__ __align__(128) float4 X4[];  // [256 rows][8 float4], then the TMA stages
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int cg = l & 7, q = 4 * w + (l >> 3);  // 4-column group, row group
    uint8_t* const stg = reinterpret_cast<uint8_t*>(X4) + C3_SMEM;
    uint64_t* const bars = reinterpret_cast<uint64_t*>(stg + (TS > 0 ? TS : 0) * C3_STAGE);
    pdl_wait();  // launched with PDL: the predecessor's writes are visible past this point
    pdl_trigger();
    Quant<FMT, SUP_R> qr;
    Quant<FMT, SUP_P> qp;
    if constexpr (MODE == C3_QUANT) {
        qr.init(amax_r, sup_r, FOLD ? norm : 1.f, sro, err);
        if (codes_p) qp.init(amax_p, sup_p, 1.f, spo, err);
    }
    const float2 norm2 = make_float2(norm, norm);
    float am_r = 0.f, am_p = 0.f;
    const int64_t ct = (cols + C3_COLS - 1) / C3_COLS, rt = (rows_pad + C3_ROWS - 1) / C3_ROWS;

    // rotated codes of 16 groups held in x[i] (rows row0 + i*rstep), then
    // the rare exact fix-up out of line
    auto emit_rot = [&](auto edge_tag, float2 (&x)[16][2], int64_t row0, int rstep, int64_t col, bool cok) {
        constexpr bool EDGE = decltype(edge_tag)::value;
        float dmax = 0.f;
        uint32_t valid = 0xFFFFu;
        uint8_t* o = codes_r + row0 * cols + col;
        const int64_t st = (int64_t)rstep * cols;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            if (!FOLD) {
                x[i][0] = c3_mul2(x[i][0], norm2);
                x[i][1] = c3_mul2(x[i][1], norm2);
            }
            const uint32_t wd = qr.q4(x[i][0], x[i][1], dmax);
            const bool ok = !EDGE || (cok && row0 + (int64_t)i * rstep < rows_pad);
            if (EDGE && !ok) valid &= ~(1u << i);
            if (ok) *reinterpret_cast<uint32_t*>(o) = wd;
            o += st;
        }
        if (__any_sync(0xffffffffu, !(dmax < qr.thr))) {
            if (!(dmax < qr.thr)) {
                float4 tmp[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) tmp[i] = make_float4(x[i][0].x, x[i][0].y, x[i][1].x, x[i][1].y);
                c3_fix<FMT>(tmp, 16, valid, codes_r + row0 * cols + col, st, qr.s, qr.inv, qr.thr);
            }
        }
    };

    // TMA ring: refill stage s with tile `next` once every thread has read it
    auto refill = [&](int s, int64_t next) {
        if constexpr (TS > 0) {
            if (threadIdx.x == 0 && next >= 0) {
                mbar_expect_tx(&bars[s], C3_STAGE);
                tma_load_2d(stg + s * C3_STAGE, &tm, &bars[s], (int)((next % ct) * C3_COLS),
                            (int)((next / ct) * C3_ROWS));
            }
        }
    };
    auto run = [&](auto edge_tag, int64_t r0, int64_t c0, int s, int64_t next) {
        constexpr bool EDGE = decltype(edge_tag)::value;
        const int64_t col = c0 + 4 * cg;
        const bool cok = !EDGE || col < cols;
        const int64_t row1 = r0 + 16 * q;
        (void)cok;  // unused by some instantiations
        (void)row1;
        // ---------------- phase 1: rows 16q + m
        float2 v[16][2];
        if constexpr (TS > 0) {
            const uint8_t* p = stg + s * C3_STAGE + (16 * q) * (C3_COLS * 2) + cg * 8;
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const uint2 r = *reinterpret_cast<const uint2*>(p + m * (C3_COLS * 2));
                v[m][0] = make_float2(__uint_as_float(r.x << 16), __uint_as_float(r.x & 0xFFFF0000u));
                v[m][1] = make_float2(__uint_as_float(r.y << 16), __uint_as_float(r.y & 0xFFFF0000u));
            }
        } else {
            const InT* p = in + row1 * cols + col;
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                c3_load4<InT>(p, !EDGE || (cok && row1 + m < b), v[m][0], v[m][1]);
                p += cols;
            }
        }
        if constexpr (MODE == C3_ABSMAX) {
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                am_p = c3_max3nan(am_p, fabsf(v[m][0].x), fabsf(v[m][0].y));
                am_p = c3_max3nan(am_p, fabsf(v[m][1].x), fabsf(v[m][1].y));
            }
        } else {
            if (codes_p) {
                float dmax = 0.f;
                uint32_t valid = 0xFFFFu;
                uint8_t* o = codes_p + row1 * cols + col;
#pragma unroll
                for (int m = 0; m < 16; ++m) {
                    const uint32_t wd = qp.q4(v[m][0], v[m][1], dmax);
                    const bool ok = !EDGE || (cok && row1 + m < b);
                    if (EDGE && !ok) valid &= ~(1u << m);
                    if (ok) *reinterpret_cast<uint32_t*>(o) = wd;
                    o += cols;
                }
                if (__any_sync(0xffffffffu, !(dmax < qp.thr))) {
                    if (!(dmax < qp.thr)) {
                        float4 tmp[16];
#pragma unroll
                        for (int m = 0; m < 16; ++m) tmp[m] = make_float4(v[m][0].x, v[m][0].y, v[m][1].x, v[m][1].y);
                        c3_fix<FMT>(tmp, 16, valid, codes_p + row1 * cols + col, cols, qp.s, qp.inv, qp.thr);
                    }
                }
            }
        }
#pragma unroll
        for (int t = 0; t < P1; ++t) {
            const int h = 1 << t;
            const bool last = MODE == C3_ABSMAX && P2 == 0 && t == P1 - 1;
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                if ((m & h) == 0) {
                    if (last) {
                        am_r = c3_max3nan(am_r, fabsf(v[m][0].x) + fabsf(v[m + h][0].x),
                                          fabsf(v[m][0].y) + fabsf(v[m + h][0].y));
                        am_r = c3_max3nan(am_r, fabsf(v[m][1].x) + fabsf(v[m + h][1].x),
                                          fabsf(v[m][1].y) + fabsf(v[m + h][1].y));
                    } else {
                        c3_bfly(v[m][0], v[m + h][0]);
                        c3_bfly(v[m][1], v[m + h][1]);
                    }
                }
            }
        }
        if constexpr (MODE == C3_ABSMAX && LB == 0) {
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                am_r = c3_max3nan(am_r, fabsf(v[m][0].x), fabsf(v[m][0].y));
                am_r = c3_max3nan(am_r, fabsf(v[m][1].x), fabsf(v[m][1].y));
            }
        }
        if constexpr (P2 == 0) {
            if constexpr (TS > 0) {
                __syncthreads();  // stage s fully read
                refill(s, next);
            }
            if constexpr (MODE == C3_QUANT) emit_rot(edge_tag, v, row1, 1, col, cok);
        } else {
            // ---------------- exchange (fp32, row-major [256][64])
#pragma unroll
            for (int m = 0; m < 16; ++m)
                X4[(16 * q + m) * 8 + cg] = make_float4(v[m][0].x, v[m][0].y, v[m][1].x, v[m][1].y);
            __syncthreads();
            refill(s, next);  // stage s fully read (phase 1 precedes the barrier)
            // ---------------- phase 2: thread (cg, mm = q) takes rows 16i + mm
            float2 u[16][2];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                const float4 f = X4[(16 * i + q) * 8 + cg];
                u[i][0] = make_float2(f.x, f.y);
                u[i][1] = make_float2(f.z, f.w);
            }
            __syncthreads();  // the next tile's exchange overwrites X4
#pragma unroll
            for (int t = 0; t < P2; ++t) {
                const int h = 1 << t;
                const bool last = MODE == C3_ABSMAX && t == P2 - 1;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    if ((i & h) == 0) {
                        if (last) {
                            am_r = c3_max3nan(am_r, fabsf(u[i][0].x) + fabsf(u[i + h][0].x),
                                              fabsf(u[i][0].y) + fabsf(u[i + h][0].y));
                            am_r = c3_max3nan(am_r, fabsf(u[i][1].x) + fabsf(u[i + h][1].x),
                                              fabsf(u[i][1].y) + fabsf(u[i + h][1].y));
                        } else {
                            c3_bfly(u[i][0], u[i + h][0]);
                            c3_bfly(u[i][1], u[i + h][1]);
                        }
                    }
                }
            }
            if constexpr (MODE == C3_QUANT) emit_rot(edge_tag, u, r0 + q, 16, col, cok);
        }
    };

    const int64_t ntiles = ct * rt;
    if constexpr (TS > 0) {
        if (threadIdx.x == 0) {
            tma_prefetch_desc(&tm);
            for (int s = 0; s < TS; ++s) mbar_init(&bars[s], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            for (int s = 0; s < TS; ++s) {
                const int64_t t = blockIdx.x + (int64_t)s * gridDim.x;
                refill(s, t < ntiles ? t : -1);
            }
        }
        __syncthreads();
    }
    int it = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int64_t r0 = (tile / ct) * C3_ROWS, c0 = (tile % ct) * C3_COLS;
        const bool interior = r0 + C3_ROWS <= b && r0 + C3_ROWS <= rows_pad && c0 + C3_COLS <= cols;
        int s = 0;
        int64_t next = -1;
        if constexpr (TS > 0) {
            s = it % TS;
            mbar_wait(&bars[s], (uint32_t)(it / TS) & 1u);
            const int64_t nt = tile + (int64_t)TS * gridDim.x;
            next = nt < ntiles ? nt : -1;
        }
        if (interior) run(std::false_type{}, r0, c0, s, next);
        else run(std::true_type{}, r0, c0, s, next);
    }
    if constexpr (MODE == C3_ABSMAX) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            am_r = c3_max3nan(am_r, __shfl_xor_sync(0xffffffffu, am_r, o), 0.f);
            am_p = c3_max3nan(am_p, __shfl_xor_sync(0xffffffffu, am_p, o), 0.f);
        }
        am_r *= norm;  // monotone: max(fl(|x| * norm)) == fl(max|x| * norm)
        if (l == 0) {
            atomic_absmax(amax_r, fabsf(am_r));
            if (amax_p) atomic_absmax(amax_p, fabsf(am_p));
            if (!(am_r <= 3.402823466e38f) || !(am_p <= 3.402823466e38f)) atomicOr(err, ERRF_NONFINITE);
        }
    }
}

// ------------------------------------------------------------------ K2 + SwiGLU backward
// Phase A of K2 for both MLP input projections, fused with the SwiGLU
// backward glue: dG, dU are computed from (dH, G, U) on the fly
// (swiglu_bwd1, the exact formula of the stand-alone glue kernel), stored in
// bf16 for K2's quantize passes, and the rotated and plain absmax words of
// both come out of the same pass — one read of dH, G, U replaces the glue
// kernel plus two K2 absmax passes over dG and dU.

// rotated + plain absmax of one 256 x 32 tile held as thread (cg, q)'s rows
// 16q + m (phase 1 layout of k_cols_v3)
template <int LB>
__device__ __forceinline__ void c3_tile_absmax(float2 (&v)[16][2], float4* X4, int q, int cg, float& am_r, float& am_p) {
    constexpr int P1 = LB < 4 ? LB : 4;
    constexpr int P2 = LB > 4 ? LB - 4 : 0;
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        am_p = c3_max3nan(am_p, fabsf(v[m][0].x), fabsf(v[m][0].y));
        am_p = c3_max3nan(am_p, fabsf(v[m][1].x), fabsf(v[m][1].y));
    }
#pragma unroll
    for (int t = 0; t < P1; ++t) {
        const int h = 1 << t;
        const bool last = P2 == 0 && t == P1 - 1;
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            if ((m & h) == 0) {
                if (last) {
                    am_r = c3_max3nan(am_r, fabsf(v[m][0].x) + fabsf(v[m + h][0].x), fabsf(v[m][0].y) + fabsf(v[m + h][0].y));
                    am_r = c3_max3nan(am_r, fabsf(v[m][1].x) + fabsf(v[m + h][1].x), fabsf(v[m][1].y) + fabsf(v[m + h][1].y));
                } else {
                    c3_bfly(v[m][0], v[m + h][0]);
                    c3_bfly(v[m][1], v[m + h][1]);
                }
            }
        }
    }
    if constexpr (LB == 0) {
#pragma unroll
        for (int m = 0; m < 16; ++m) {
            am_r = c3_max3nan(am_r, fabsf(v[m][0].x), fabsf(v[m][0].y));
            am_r = c3_max3nan(am_r, fabsf(v[m][1].x), fabsf(v[m][1].y));
        }
    }
    if constexpr (P2 > 0) {
#pragma unroll
        for (int m = 0; m < 16; ++m)
            X4[(16 * q + m) * 8 + cg] = make_float4(v[m][0].x, v[m][0].y, v[m][1].x, v[m][1].y);
        __syncthreads();
        float2 w[16][2];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const float4 f = X4[(16 * i + q) * 8 + cg];
            w[i][0] = make_float2(f.x, f.y);
            w[i][1] = make_float2(f.z, f.w);
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < P2; ++t) {
            const int h = 1 << t;
            const bool last = t == P2 - 1;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                if ((i & h) == 0) {
                    if (last) {
                        am_r = c3_max3nan(am_r, fabsf(w[i][0].x) + fabsf(w[i + h][0].x), fabsf(w[i][0].y) + fabsf(w[i + h][0].y));
                        am_r = c3_max3nan(am_r, fabsf(w[i][1].x) + fabsf(w[i + h][1].x), fabsf(w[i][1].y) + fabsf(w[i + h][1].y));
                    } else {
                        c3_bfly(w[i][0], w[i + h][0]);
                        c3_bfly(w[i][1], w[i + h][1]);
                    }
                }
            }
        }
    }
}

__device__ __forceinline__ void c3_unpack(const uint2 (&pk)[16], float2 (&v)[16][2]) {
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        v[m][0] = make_float2(__uint_as_float(pk[m].x << 16), __uint_as_float(pk[m].x & 0xFFFF0000u));
        v[m][1] = make_float2(__uint_as_float(pk[m].y << 16), __uint_as_float(pk[m].y & 0xFFFF0000u));
    }
}

template <int LB>
__global__ void __launch_bounds__(128, 3)
    k_cols_swiglu_absmax(const __nv_bfloat16* __restrict__ dH, const __nv_bfloat16* __restrict__ G,
                         const __nv_bfloat16* __restrict__ U, __nv_bfloat16* __restrict__ dG,
                         __nv_bfloat16* __restrict__ dU, int64_t b, int64_t rows_pad, int64_t cols, float norm,
                         unsigned* am_gr, unsigned* am_gp, unsigned* am_ur, unsigned* am_up, unsigned* err) {
    extern __shared__ __align__(128) float4 X4[];
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int cg = l & 7, q = 4 * w + (l >> 3);
    float gr = 0.f, gp = 0.f, ur = 0.f, up = 0.f;
    const int64_t ct = (cols + C3_COLS - 1) / C3_COLS, rt = (rows_pad + C3_ROWS - 1) / C3_ROWS;
    for (int64_t tile = blockIdx.x; tile < ct * rt; tile += gridDim.x) {
        const int64_t r0 = (tile / ct) * C3_ROWS, c0 = (tile % ct) * C3_COLS;
        const int64_t col = c0 + 4 * cg;
        const bool cok = col < cols;
        const int64_t row1 = r0 + 16 * q;
        uint2 pg[16], pu[16];
        {
            const int64_t off = row1 * cols + col;
            const uint2* ph = reinterpret_cast<const uint2*>(dH + off);
            const uint2* pgi = reinterpret_cast<const uint2*>(G + off);
            const uint2* pui = reinterpret_cast<const uint2*>(U + off);
            uint2* og = reinterpret_cast<uint2*>(dG + off);
            uint2* ou = reinterpret_cast<uint2*>(dU + off);
            const int64_t st = cols / 4;  // uint2 per row
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const bool ok = cok && row1 + m < b;
                uint2 rh = make_uint2(0, 0), rg = rh, ru = rh;
                if (ok) {
                    rh = __ldg(ph + m * st);
                    rg = __ldg(pgi + m * st);
                    ru = __ldg(pui + m * st);
                }
                const uint32_t hw[2] = {rh.x, rh.y}, gw[2] = {rg.x, rg.y}, uw[2] = {ru.x, ru.y};
                uint32_t dgw[2], duw[2];
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    float g0, g1, u0, u1;
                    swiglu_bwd1(__uint_as_float(hw[j] << 16), __uint_as_float(gw[j] << 16), __uint_as_float(uw[j] << 16), g0, u0);
                    swiglu_bwd1(__uint_as_float(hw[j] & 0xFFFF0000u), __uint_as_float(gw[j] & 0xFFFF0000u),
                                __uint_as_float(uw[j] & 0xFFFF0000u), g1, u1);
                    dgw[j] = pack_bf16x2(g0, g1);
                    duw[j] = pack_bf16x2(u0, u1);
                }
                pg[m] = make_uint2(dgw[0], dgw[1]);
                pu[m] = make_uint2(duw[0], duw[1]);
                if (ok) {
                    og[m * st] = pg[m];
                    ou[m * st] = pu[m];
                }
            }
        }
        {
            float2 v[16][2];
            c3_unpack(pg, v);
            c3_tile_absmax<LB>(v, X4, q, cg, gr, gp);
        }
        {
            float2 v[16][2];
            c3_unpack(pu, v);
            c3_tile_absmax<LB>(v, X4, q, cg, ur, up);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        gr = c3_max3nan(gr, __shfl_xor_sync(0xffffffffu, gr, o), 0.f);
        gp = c3_max3nan(gp, __shfl_xor_sync(0xffffffffu, gp, o), 0.f);
        ur = c3_max3nan(ur, __shfl_xor_sync(0xffffffffu, ur, o), 0.f);
        up = c3_max3nan(up, __shfl_xor_sync(0xffffffffu, up, o), 0.f);
    }
    gr *= norm;  // monotone: max(fl(|x| * norm)) == fl(max|x| * norm)
    ur *= norm;
    if (l == 0) {
        atomic_absmax(am_gr, fabsf(gr));
        atomic_absmax(am_gp, fabsf(gp));
        atomic_absmax(am_ur, fabsf(ur));
        atomic_absmax(am_up, fabsf(up));
        constexpr float F = 3.402823466e38f;
        if (!(gr <= F) || !(gp <= F) || !(ur <= F) || !(up <= F))
            atomicOr(err, ERRF_NONFINITE);
    }
}

namespace {

template <int LB, typename InT, int FMT, int MODE, bool SR, bool SP, int TS>
void c3_go(const CUtensorMap& tm, const InT* in, int64_t b, int64_t rows_pad, int64_t cols, unsigned* ar, unsigned* ap,
           const float* sr, const float* sp, uint8_t* cr, uint8_t* cp, unsigned* err, float* sro, float* spo,
           cudaStream_t st) {
    auto kern = k_cols_v3<LB, InT, FMT, MODE, SR, SP, TS>;
    const size_t smem = C3_SMEM + (size_t)TS * C3_STAGE + (TS > 0 ? 8 * TS : 0);
    static int per_sm = 0;
    if (!per_sm) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * C3_WARPS, smem);
        if (per_sm < 1) per_sm = 1;
    }
    const int64_t tiles = ((cols + C3_COLS - 1) / C3_COLS) * ((rows_pad + C3_ROWS - 1) / C3_ROWS);
    const int64_t cap = (int64_t)num_sms() * per_sm;
    const unsigned grid = (unsigned)(tiles < cap ? tiles : cap);
    launch_pdl(kern, dim3(grid), dim3(32 * C3_WARPS), smem, st, tm, in, b, rows_pad, cols, hadamard_norm(int64_t(1) << LB),
               ar, ap, sr, sp, cr, cp, err, sro, spo);
}

inline bool c3_use_tma() {
    static const int v = [] {
        const char* e = getenv("HALO_K2_TMA");
        return e ? atoi(e) : 1;
    }();
    return v != 0;
}

template <int LB, typename InT, int FMT, int MODE, bool SR, bool SP>
void c3_launch(const InT* in, int64_t b, int64_t rows_pad, int64_t cols, unsigned* ar, unsigned* ap, const float* sr,
               const float* sp, uint8_t* cr, uint8_t* cp, unsigned* err, float* sro, float* spo, cudaStream_t st) {
    CUtensorMap tm;
    if constexpr (sizeof(InT) == 2) {
        // TMA ring: row pitch a multiple of 16 B, 16 B aligned base
        if (c3_use_tma() && cols % 8 == 0 && (uintptr_t)in % 16 == 0 &&
            encode_2d_plain(&tm, 1, in, (uint64_t)cols, (uint64_t)b, (uint64_t)cols * 2, C3_COLS, C3_ROWS)) {
            c3_go<LB, InT, FMT, MODE, SR, SP, C3_TS>(tm, in, b, rows_pad, cols, ar, ap, sr, sp, cr, cp, err, sro, spo, st);
            return;
        }
    }
    memset(&tm, 0, sizeof(tm));
    c3_go<LB, InT, FMT, MODE, SR, SP, 0>(tm, in, b, rows_pad, cols, ar, ap, sr, sp, cr, cp, err, sro, spo, st);
}

template <int LB>
void c3_dispatch(int mode, int fmt, int in_dtype, const void* in, int64_t b, int64_t rows_pad, int64_t cols,
                 unsigned* ar, unsigned* ap, const float* sr, const float* sp, uint8_t* cr, uint8_t* cp,
                 unsigned* err, float* sro, float* spo, cudaStream_t st) {
#define HALO_C3Q(T, F) c3_launch<LB, T, F, C3_QUANT, false, false>(p, b, rows_pad, cols, ar, ap, sr, sp, cr, cp, err, sro, spo, st);
#define HALO_C3(T)                                                                                                 \
    {                                                                                                              \
        auto p = static_cast<const T*>(in);                                                                        \
        if (mode == C3_ABSMAX) c3_launch<LB, T, 0, C3_ABSMAX, false, false>(p, b, rows_pad, cols, ar, ap, sr, sp, cr, cp, err, sro, spo, st); \
        else if (fmt == FMT_INT8) HALO_C3Q(T, FMT_INT8)                                                            \
        else if (fmt == FMT_E3M2) HALO_C3Q(T, FMT_E3M2)                                                            \
        else HALO_C3Q(T, FMT_E4M3)                                                                                 \
    }
    if (in_dtype == DT_BF16) HALO_C3(__nv_bfloat16) else HALO_C3(float)
#undef HALO_C3
#undef HALO_C3Q
}

}  // namespace

// K2 v3: modes 0 (absmax) / 1 (quantize); B = 2^k <= 256; cols % 4 == 0.
bool cols_v3(int mode, int fmt, int in_dtype, const void* in, int64_t b, int64_t rows_pad, int64_t cols, int64_t B,
             unsigned* ar, unsigned* ap, const float* sr, const float* sp, uint8_t* cr, uint8_t* cp, unsigned* err,
             float* sro, float* spo, cudaStream_t st) {
    if (mode > 1 || B < 1 || B > 256 || (B & (B - 1)) || cols % 4) return false;
    if (sr || sp) return false;  // supplied scales: fwht2.cu (the HALO-2 layer never supplies them here)
    if ((uintptr_t)in % (in_dtype == DT_BF16 ? 8 : 16) || (uintptr_t)cr % 4 || (uintptr_t)cp % 4) return false;
    int lb = 0;
    while ((int64_t(1) << lb) < B) ++lb;
    switch (lb) {
    case 0: c3_dispatch<0>(mode, fmt, in_dtype, in, b, rows_pad, cols, ar, ap, sr, sp, cr, cp, err, sro, spo, st); break;
    case 1: c3_dispatch<1>(mode, fmt, in_dtype, in, b, rows_pad, cols, ar, ap, sr, sp, cr, cp, err, sro, spo, st); break;
    case 2: c3_dispatch<2>(mode, fmt, in_dtype, in, b, rows_pad, cols, ar, ap, sr, sp, cr, cp, err, sro, spo, st); break;
    case 3: c3_dispatch<3>(mode, fmt, in_dtype, in, b, rows_pad, cols, ar, ap, sr, sp, cr, cp, err, sro, spo, st); break;
    case 4: c3_dispatch<4>(mode, fmt, in_dtype, in, b, rows_pad, cols, ar, ap, sr, sp, cr, cp, err, sro, spo, st); break;
    case 5: c3_dispatch<5>(mode, fmt, in_dtype, in, b, rows_pad, cols, ar, ap, sr, sp, cr, cp, err, sro, spo, st); break;
    case 6: c3_dispatch<6>(mode, fmt, in_dtype, in, b, rows_pad, cols, ar, ap, sr, sp, cr, cp, err, sro, spo, st); break;
    case 7: c3_dispatch<7>(mode, fmt, in_dtype, in, b, rows_pad, cols, ar, ap, sr, sp, cr, cp, err, sro, spo, st); break;
    default: c3_dispatch<8>(mode, fmt, in_dtype, in, b, rows_pad, cols, ar, ap, sr, sp, cr, cp, err, sro, spo, st); break;
    }
    return true;
}

// K2 phase A for the MLP's gate and up projections fused with the SwiGLU
// backward: dG, dU (bf16, [b x cols]) written, absmax words (rotated over
// blocks of B rows of the b_pad-padded token axis, and plain) of both.
bool cols_swiglu_absmax(const void* dh, const void* g, const void* u, void* dg, void* du, int64_t b, int64_t rows_pad,
                        int64_t cols, int64_t B, unsigned* gr, unsigned* gp, unsigned* ur, unsigned* up, unsigned* err,
                        cudaStream_t st) {
    if (B < 1 || B > 256 || (B & (B - 1)) || cols % 4) return false;
    for (const void* p : {dh, g, u, (const void*)dg, (const void*)du})
        if ((uintptr_t)p % 8) return false;
    int lb = 0;
    while ((int64_t(1) << lb) < B) ++lb;
    const int64_t tiles = ((cols + C3_COLS - 1) / C3_COLS) * ((rows_pad + C3_ROWS - 1) / C3_ROWS);
    auto go = [&](auto kern) {
        static int per_sm = 0;
        if (!per_sm) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C3_SMEM);
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * C3_WARPS, C3_SMEM);
            if (per_sm < 1) per_sm = 1;
        }
        const int64_t cap = (int64_t)num_sms() * per_sm;
        kern<<<(unsigned)(tiles < cap ? tiles : cap), 32 * C3_WARPS, C3_SMEM, st>>>(
            static_cast<const __nv_bfloat16*>(dh), static_cast<const __nv_bfloat16*>(g),
            static_cast<const __nv_bfloat16*>(u), static_cast<__nv_bfloat16*>(dg), static_cast<__nv_bfloat16*>(du), b,
            rows_pad, cols, hadamard_norm(B), gr, gp, ur, up, err);
    };
    switch (lb) {
    case 0: go(k_cols_swiglu_absmax<0>); break;
    case 1: go(k_cols_swiglu_absmax<1>); break;
    case 2: go(k_cols_swiglu_absmax<2>); break;
    case 3: go(k_cols_swiglu_absmax<3>); break;
    case 4: go(k_cols_swiglu_absmax<4>); break;
    case 5: go(k_cols_swiglu_absmax<5>); break;
    case 6: go(k_cols_swiglu_absmax<6>); break;
    case 7: go(k_cols_swiglu_absmax<7>); break;
    default: go(k_cols_swiglu_absmax<8>); break;
    }
    return true;
}

}  // namespace halo_b200
