// fwht_cols_lb.cu — K2 for large Hadamard blocks along the token axis,
// 512 <= B <= 4096, one kernel per phase and no fp32 scratch round trip.
//
// Reference: error_path, halo_linear.hpp:393-399 — (H_b pad(E_Y))_Q with
// transform_left (hadamard.hpp:205-216): the row transform of
// hadamard.hpp:136-177 run down each column, stages len = 1, 2, ..., B/2 over
// the row index, then one normalising multiply; plus the plain (E_Y)_Q for G
// (:371).  The same fp32 butterflies in the same order: bit-exact.
//
// A CTA owns a STRIP: one B-row block of W = E / B adjacent columns
// (E = 32768 elements for bf16 input, 16384 for fp32), so the whole column
// transform of the strip is resident on chip:
//   * cp.async (16 B, L2 only) stages the strip in 64-row groups, one group
//     per 65-row slot (the spare row staggers the banks: conflict-free
//     round-1 reads; TMA cannot place boxes off 128 B boundaries), rows past
//     b zero-filled by the copy;
//   * round 1: thread (g, cp) holds rows 64g .. 64g+63 of column pair cp (64
//     float2 in registers) and runs row bits 0..5 (stages 1..32) as FADD2;
//     the plain absmax / plain codes come from the raw values here;
//   * one fp32 exchange through an XOR-swizzled buffer (bank-optimal for both
//     access patterns, tools/lb_banks.py) — the only smem round trip;
//   * round 2: thread (j, q) holds rows 64i + j (i < B/64) of C2 = 64/(B/64)
//     column pairs and runs row bits 6..LB-1; the last stage feeds the
//     absmax as |u|+|v| (phase A), or the values are normalised and
//     quantized (phase B), or stored (transform-only, K4-left);
//   * the next strip's copies are issued as soon as round 1 has read the
//     stage, so their HBM latency hides behind the exchange and round 2.
// One persistent CTA per SM (~226 KB of shared memory for bf16).
#include <cstdlib>

#include "common.cuh"
#include "halo_internal.h"
#include "sm100.cuh"

namespace halo_b200 {

namespace {

__device__ __forceinline__ float2 lb_add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 lb_sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ void lb_bfly(float2& a, float2& b) {
    const float2 x = a, y = b;
    a = lb_add2(x, y);
    b = lb_sub2(x, y);
}
__device__ __forceinline__ float lb_max3nan(float a, float b, float c) {
    float r;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
// 16-byte global -> shared copy, zero-filled when !ok (rows past b)
__device__ __forceinline__ void lb_cp16(void* dst, const void* src, bool ok) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void lb_cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void lb_cp_wait() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ float lb_fmax3(float a, float b, float c) { return fmaxf(fmaxf(a, b), c); }
__device__ __forceinline__ uint32_t lb_pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

template <int FMT>
__device__ __forceinline__ uint32_t lb_exact4(float2 a, float2 b, float s, float inv) {
    if constexpr (FMT == FMT_INT8)
        return lb_pack4((uint8_t)quant_int8(a.x, s, inv), (uint8_t)quant_int8(a.y, s, inv),
                        (uint8_t)quant_int8(b.x, s, inv), (uint8_t)quant_int8(b.y, s, inv));
    else if constexpr (FMT == FMT_E3M2)
        return lb_pack4(quant_e3m2(a.x, s, inv) << 2, quant_e3m2(a.y, s, inv) << 2, quant_e3m2(b.x, s, inv) << 2,
                        quant_e3m2(b.y, s, inv) << 2);
    else
        return lb_pack4(quant_e4m3(a.x, s, inv), quant_e4m3(a.y, s, inv), quant_e4m3(b.x, s, inv),
                        quant_e4m3(b.y, s, inv));
}

// certified quantizer for 4 values (the K1/K2 scheme, quant_round.cuh); a
// supplied scale may saturate INT8 codes, so |q| joins the certification
// maximum (sup_k = thr / 127.5 maps |q| <= 127 below thr, >= 128 above it)
template <int FMT>
struct LbQuant {
    float s = 1.f, inv = 1.f, thr = 0.5f, sup_k = 0.f;
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
        sup_k = supplied ? thr / 127.5f : 0.f;
        if (FMT != FMT_INT8) e4m3_brackets(inv, ilo2, ihi2);
    }
    // fast code word of 4 values, branch-free; `slow` is set when the INT8
    // word is not certified (a group is exact iff its maximum < thr)
    __device__ __forceinline__ uint32_t q4(float2 a, float2 c, bool& slow) const {
        if constexpr (FMT == FMT_INT8) {
            const float2 m2 = make_float2(kRoundMagic, kRoundMagic);
            const float2 ta = __ffma2_rn(a, inv2, m2), tc = __ffma2_rn(c, inv2, m2);
            const float2 qa = lb_sub2(ta, m2), qc = lb_sub2(tc, m2);
            const float2 ra = __ffma2_rn(qa, nsm2, a), rc = __ffma2_rn(qc, nsm2, c);
            float m = lb_fmax3(lb_fmax3(0.f, fabsf(ra.x), fabsf(ra.y)), fabsf(rc.x), fabsf(rc.y));
            m = fmaxf(m, lb_fmax3(lb_fmax3(0.f, fabsf(qa.x), fabsf(qa.y)), fabsf(qc.x), fabsf(qc.y)) * sup_k);
            slow = !(m < thr);
            return lb_pack4(__float_as_uint(ta.x), __float_as_uint(ta.y), __float_as_uint(tc.x),
                            __float_as_uint(tc.y));
        } else if constexpr (FMT == FMT_E3M2) {
            return e3m2x4_fast(a, c, ilo2, ihi2, s);
        } else {
            uint32_t bad = 0;
            return e4m3x4_fast(a, c, ilo2, ihi2, s, bad);
        }
    }
    // the exact word of a group whose fast word is not certified (INT8 only;
    // the minifloat fast paths are exact)
    __device__ __forceinline__ uint32_t exact(float2 a, float2 c) const { return lb_exact4<FMT>(a, c, s, inv); }
};

enum : int { LB_ABSMAX = 0, LB_QUANT = 1, LB_XFORM = 2 };

template <int LB, typename InT>
struct LbCfg {
    static constexpr int B = 1 << LB;
    static constexpr int ES = (int)sizeof(InT);
    // elements per strip: wide rows pay (32-column bf16 strips run the
    // B = 1024 op 1.3-1.5x faster than 16-column ones, 16 vs 8 columns at
    // B = 2048 1.3x: profiles/r02k_ab_left_strip_width.txt), so bf16 takes
    // 32 K-element strips (one CTA per SM) from B = 1024 on
    static constexpr int E = (ES == 2 && LB >= 10) ? 32768 : 16384;
    static constexpr int W = E / B;                    // columns per strip
    static constexpr int NCP = W / 2;                  // column pairs
    static constexpr int NT = E / 128;                 // 64 float2 per thread
    static constexpr int R2B = LB - 6;                 // row bits of round 2
    static constexpr int R2 = 1 << R2B;
    static constexpr int C2 = 64 / R2;                 // column pairs per thread in round 2
    static constexpr int NQ = NCP / C2;
    static constexpr int NBOX = B / 64;
    static constexpr int ROWB = W * ES;                // staged row bytes
    static constexpr int BOX_STRIDE = 65 * ROWB;       // 64 rows + one stagger row
    static constexpr int STG_BYTES = (NBOX * BOX_STRIDE + 127) / 128 * 128;
    static constexpr int RB = 4 * W;                   // exchange row bytes (fp32)
    static constexpr int INL = RB >= 128 ? 0 : (RB == 64 ? 1 : (RB == 32 ? 2 : 3));  // log2(rows per 128 B)
    static constexpr int XCH_BYTES = E * 4;
    static constexpr int CPR = ROWB / 16;              // 16 B copies per staged row
    static constexpr int NCOPY = E * ES / 16 / NT;     // copies per thread and strip
    static constexpr size_t SMEM = (size_t)STG_BYTES + XCH_BYTES;
    static constexpr int CTAS = SMEM <= 112 * 1024 ? 2 : 1;  // resident CTAs per SM
    static_assert(NQ >= 1 && NT * 64 * 2 == E && NT % 32 == 0, "strip geometry");
    static_assert(ROWB >= 16 && ROWB % 16 == 0 && (E * ES / 16) % NT == 0, "16 B staging copies");
};

// byte offset of float2 slot (row r, column pair cp) in the exchange: XOR of
// the 16-byte chunk bits with row bits outside the 128 B line
template <int RB, int INL>
__device__ __forceinline__ uint32_t lb_swz(uint32_t r, uint32_t cp) {
    const uint32_t f = (((r >> 6) << (RB == 16 ? 0 : 1)) ^ (r >> INL)) & 7u;
    return (r * RB + 8u * cp) ^ (f << 4);
}
// The hot loops split lb_swz(64 a + b, cp) into a per-thread part XOR a
// compile-time part: 64 a RB has no bits below 1024 (RB >= 16), b RB + 8 cp
// has none at or above it, and the XOR term only touches bits 4..6, so
//   lb_swz(64 a + b, cp) = (64 a RB) ^ ((b RB + 8 cp) ^ (f << 4)),
//   f = ((a << k) ^ (b >> INL)) & 7   (k = 0 for RB = 16, else 1;
//   64 a >> INL is a multiple of 8 for INL <= 3).
template <int RB, int INL>
__device__ __forceinline__ uint32_t lb_hi(uint32_t a) {  // row block a: 64 a RB ^ (a-part of f)
    return (64u * RB * a) ^ ((((a << (RB == 16 ? 0 : 1)) & 7u)) << 4);
}
template <int RB, int INL>
__device__ __forceinline__ uint32_t lb_lo(uint32_t b, uint32_t cp) {  // row b < 64, pair cp
    return (b * RB + 8u * cp) ^ (((b >> INL) & 7u) << 4);
}

template <int LB, typename InT, int MODE, int FMT>
__global__ void __launch_bounds__(LbCfg<LB, InT>::NT, LbCfg<LB, InT>::CTAS)
    k_cols_lb(const InT* __restrict__ in, int64_t b, int64_t rows_pad, int64_t cols, float norm,
              unsigned* amax_r, unsigned* amax_p, const float* sup_r, const float* sup_p,
              uint8_t* __restrict__ codes_r, uint8_t* __restrict__ codes_p, unsigned* err, float* sro, float* spo,
              float* __restrict__ xout, int64_t rows_out) {
    using C = LbCfg<LB, InT>;
    constexpr bool FOLD = (LB % 2) == 0;  // norm = 2^-LB/2 folds into the scale
    extern __shared__ __align__(128) uint8_t smem[];
    uint8_t* const stg = smem;
    uint8_t* const xch = smem + C::STG_BYTES;
    const int t = threadIdx.x;
    const int64_t ncs = cols / C::W;
    const int64_t nstrips = (rows_pad / C::B) * ncs;
    pdl_wait();
    pdl_trigger();
    LbQuant<FMT> qr, qp;
    if constexpr (MODE == LB_QUANT) {
        qr.init(amax_r, sup_r, FOLD ? norm : 1.f, sro, err);
        if (codes_p) qp.init(amax_p, sup_p, 1.f, spo, err);
    }
    const float2 norm2 = make_float2(norm, norm);
    // stage strip s: copy k covers row k / CPR, 16-byte chunk k % CPR
    auto issue = [&](int64_t s) {
        if (s < nstrips) {
            const int64_t rb = s / ncs, cs = s % ncs;
            const InT* src0 = in + (rb * C::B) * cols + cs * C::W;
#pragma unroll
            for (int i = 0; i < C::NCOPY; ++i) {
                const int k = t + i * C::NT;
                const int r = k / C::CPR, c = k % C::CPR;
                const bool ok = rb * C::B + r < b;
                lb_cp16(stg + (r >> 6) * C::BOX_STRIDE + (r & 63) * C::ROWB + 16 * c,
                        ok ? (const void*)(src0 + (int64_t)r * cols + c * (16 / C::ES)) : (const void*)in, ok);
            }
        }
        lb_cp_commit();
    };
    issue(blockIdx.x);

    const int cp1 = t % C::NCP, g1 = t / C::NCP;  // round 1: rows 64 g1 + j, pair cp1
    const int q2 = t % C::NQ, j2 = t / C::NQ;     // round 2: rows 64 i + j2, pairs q2*C2 + c
    float am_r = 0.f, am_p = 0.f;
    for (int64_t s = blockIdx.x; s < nstrips; s += gridDim.x) {
        const int64_t rb = s / ncs, cs = s % ncs;
        const int64_t row0 = rb * C::B, col0 = cs * C::W;
        lb_cp_wait();
        __syncthreads();  // every thread's copies of this strip have landed
        // ---------------- round 1
        float2 v[64];
        {
            const uint8_t* p = stg + g1 * C::BOX_STRIDE + cp1 * 2 * C::ES;
#pragma unroll
            for (int j = 0; j < 64; ++j) {
                if constexpr (C::ES == 2) {
                    const uint32_t r = *reinterpret_cast<const uint32_t*>(p + j * C::ROWB);
                    v[j] = make_float2(__uint_as_float(r << 16), __uint_as_float(r & 0xFFFF0000u));
                } else {
                    v[j] = *reinterpret_cast<const float2*>(p + j * C::ROWB);
                }
            }
        }
        if constexpr (MODE == LB_ABSMAX) {
            if (amax_p) {
#pragma unroll
                for (int j = 0; j < 64; ++j) am_p = lb_max3nan(am_p, fabsf(v[j].x), fabsf(v[j].y));
            }
        } else if constexpr (MODE == LB_QUANT) {
            if (codes_p) {  // plain codes of the real rows: two rows per 4-code word
                const int64_t r1 = row0 + 64 * g1;
                const int64_t left = b - r1;
                const int nvalid = left >= 64 ? 64 : (left > 0 ? (int)left : 0);
                uint8_t* o = codes_p + r1 * cols + col0 + 2 * cp1;
                auto put = [&](int j, uint32_t w) {
                    if (j < nvalid) *reinterpret_cast<uint16_t*>(o + j * cols) = (uint16_t)(w & 0xFFFFu);
                    if (j + 1 < nvalid) *reinterpret_cast<uint16_t*>(o + (j + 1) * cols) = (uint16_t)(w >> 16);
                };
                uint32_t mask = 0;  // groups whose fast word is not certified
                if (nvalid == 64) {
                    uint8_t* oo = o;
#pragma unroll
                    for (int j = 0; j < 64; j += 2) {
                        bool sl = false;
                        const uint32_t w = qp.q4(v[j], v[j + 1], sl);
                        *reinterpret_cast<uint16_t*>(oo) = (uint16_t)(w & 0xFFFFu);
                        *reinterpret_cast<uint16_t*>(oo + cols) = (uint16_t)(w >> 16);
                        oo += 2 * cols;
                        mask |= (uint32_t)sl << (j / 2);
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 64; j += 2) {
                        bool sl = false;
                        put(j, qp.q4(v[j], v[j + 1], sl));
                        mask |= (uint32_t)sl << (j / 2);
                    }
                }
                if (FMT == FMT_INT8 && __any_sync(0xffffffffu, mask != 0)) {
                    if (mask) {  // ties (bf16 data hits exact midpoints) or saturation
                        float4 tmp[32];  // local memory on this path only
#pragma unroll
                        for (int j = 0; j < 64; j += 2) tmp[j / 2] = make_float4(v[j].x, v[j].y, v[j + 1].x, v[j + 1].y);
                        while (mask) {
                            const int g = __ffs(mask) - 1;
                            mask &= mask - 1;
                            put(2 * g, qp.exact(make_float2(tmp[g].x, tmp[g].y), make_float2(tmp[g].z, tmp[g].w)));
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int tt = 0; tt < 6; ++tt) {
            const int h = 1 << tt;
#pragma unroll
            for (int j = 0; j < 64; ++j)
                if ((j & h) == 0) lb_bfly(v[j], v[j + h]);
        }
        __syncthreads();  // the stage is read (and the previous strip's outputs copied out)
        issue(s + gridDim.x);
        {
            // per-thread base ^ per-j constant (see lb_hi / lb_lo)
            const uint32_t base = lb_hi<C::RB, C::INL>(g1) ^ (8u * cp1);
#pragma unroll
            for (int j = 0; j < 64; ++j)
                *reinterpret_cast<float2*>(xch + (base ^ lb_lo<C::RB, C::INL>(j, 0))) = v[j];
        }
        __syncthreads();
        // ---------------- round 2
        float2 u[C::R2][C::C2];
        const uint32_t base2 = lb_lo<C::RB, C::INL>(j2, q2 * C::C2);
#pragma unroll
        for (int i = 0; i < C::R2; ++i) {
            if constexpr (C::C2 == 1) {
                u[i][0] = *reinterpret_cast<const float2*>(xch + (base2 ^ lb_hi<C::RB, C::INL>(i)));
            } else {
#pragma unroll
                for (int c = 0; c < C::C2; c += 2) {
                    const float4 f =
                        *reinterpret_cast<const float4*>(xch + (base2 ^ lb_hi<C::RB, C::INL>(i) ^ (8u * c)));
                    u[i][c] = make_float2(f.x, f.y);
                    u[i][c + 1] = make_float2(f.z, f.w);
                }
            }
        }
#pragma unroll
        for (int tt = 0; tt < C::R2B; ++tt) {
            const int h = 1 << tt;
            const bool last = MODE == LB_ABSMAX && tt == C::R2B - 1;
#pragma unroll
            for (int i = 0; i < C::R2; ++i)
                if ((i & h) == 0) {
#pragma unroll
                    for (int c = 0; c < C::C2; ++c) {
                        if (last) {
                            am_r = lb_max3nan(am_r, fabsf(u[i][c].x) + fabsf(u[i + h][c].x),
                                              fabsf(u[i][c].y) + fabsf(u[i + h][c].y));
                        } else {
                            lb_bfly(u[i][c], u[i + h][c]);
                        }
                    }
                }
        }
        if constexpr (MODE == LB_ABSMAX) continue;
        __syncthreads();  // every thread has read the exchange
        if constexpr (MODE == LB_QUANT) {
            // rotated codes into the exchange area as dense [B][W] bytes
#pragma unroll
            for (int i = 0; i < C::R2; ++i)
#pragma unroll
                for (int c = 0; c < C::C2; ++c)
                    if (!FOLD) u[i][c] = __fmul2_rn(u[i][c], norm2);
            // word k of row 64i + j2 (4 codes: C2 >= 2), or rows i, i+1 (C2 == 1)
            auto putr = [&](int i, int c, uint32_t w) {
                if constexpr (C::C2 == 1) {
                    *reinterpret_cast<uint16_t*>(xch + (64 * i + j2) * C::W + 2 * q2) = (uint16_t)(w & 0xFFFFu);
                    *reinterpret_cast<uint16_t*>(xch + (64 * (i + 1) + j2) * C::W + 2 * q2) = (uint16_t)(w >> 16);
                } else {
                    *reinterpret_cast<uint32_t*>(xch + (64 * i + j2) * C::W + 2 * (q2 * C::C2 + c)) = w;
                }
            };
            constexpr int IS = C::C2 == 1 ? 2 : 1, CS = C::C2 == 1 ? 1 : 2;
            constexpr int NGC = C::C2 == 1 ? 1 : C::C2 / 2;  // groups per row step
            uint32_t mask = 0;
#pragma unroll
            for (int i = 0; i < C::R2; i += IS)
#pragma unroll
                for (int c = 0; c < C::C2; c += CS) {
                    bool sl = false;
                    putr(i, c, C::C2 == 1 ? qr.q4(u[i][0], u[i + IS - 1][0], sl) : qr.q4(u[i][c], u[i][c + CS - 1], sl));
                    mask |= (uint32_t)sl << ((i / IS) * NGC + c / CS);
                }
            if (FMT == FMT_INT8 && __any_sync(0xffffffffu, mask != 0)) {
                if (mask) {  // local memory on this path only
                    float4 tmp[32];
#pragma unroll
                    for (int i = 0; i < C::R2; i += IS)
#pragma unroll
                        for (int c = 0; c < C::C2; c += CS) {
                            const float2 a = C::C2 == 1 ? u[i][0] : u[i][c];
                            const float2 d = C::C2 == 1 ? u[i + IS - 1][0] : u[i][c + CS - 1];
                            tmp[(i / IS) * NGC + c / CS] = make_float4(a.x, a.y, d.x, d.y);
                        }
                    while (mask) {
                        const int g = __ffs(mask) - 1;
                        mask &= mask - 1;
                        putr((g / NGC) * IS, (g % NGC) * CS,
                             qr.exact(make_float2(tmp[g].x, tmp[g].y), make_float2(tmp[g].z, tmp[g].w)));
                    }
                }
            }
            __syncthreads();
            // copy out: every row of the padded block (ehq keeps rows_pad rows)
            constexpr int CH = C::W >= 16 ? 16 : C::W;  // bytes per chunk
            constexpr int CPR = C::W / CH;
#pragma unroll 4
            for (int k = t; k < C::B * CPR; k += C::NT) {
                const int r = k / CPR, c = k % CPR;
                uint8_t* dst = codes_r + (row0 + r) * cols + col0 + c * CH;
                const uint8_t* src = xch + r * C::W + c * CH;
                if constexpr (CH == 16) *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
                else if constexpr (CH == 8) *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(src);
                else *reinterpret_cast<uint32_t*>(dst) = *reinterpret_cast<const uint32_t*>(src);
            }
        } else {  // LB_XFORM: normalised fp32 back into the (swizzled) exchange, rows < rows_out out
#pragma unroll
            for (int i = 0; i < C::R2; ++i)
#pragma unroll
                for (int c = 0; c < C::C2; ++c)
                    *reinterpret_cast<float2*>(xch + (base2 ^ lb_hi<C::RB, C::INL>(i) ^ (8u * c))) =
                        __fmul2_rn(u[i][c], norm2);
            __syncthreads();
            constexpr int CPR = C::W / 4;  // 16-byte chunks per row
#pragma unroll 4
            for (int k = t; k < C::B * CPR; k += C::NT) {
                const int r = k / CPR, c = k % CPR;
                if (row0 + r < rows_out)
                    *reinterpret_cast<float4*>(xout + (row0 + r) * cols + col0 + 4 * c) =
                        *reinterpret_cast<const float4*>(xch + lb_swz<C::RB, C::INL>(r, 2 * c));
            }
        }
        // the next strip's round 1 writes nothing to the exchange before its
        // first barrier, which also orders these copy-out reads
    }
    if constexpr (MODE == LB_ABSMAX) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            am_r = lb_max3nan(am_r, __shfl_xor_sync(0xffffffffu, am_r, o), 0.f);
            am_p = lb_max3nan(am_p, __shfl_xor_sync(0xffffffffu, am_p, o), 0.f);
        }
        am_r *= norm;  // monotone: max(fl(|x| * norm)) == fl(max|x| * norm)
        if ((t & 31) == 0) {
            atomic_absmax(amax_r, fabsf(am_r));
            if (amax_p) atomic_absmax(amax_p, fabsf(am_p));
            if (!(am_r <= 3.402823466e38f) || !(am_p <= 3.402823466e38f)) atomicOr(err, ERRF_NONFINITE);
        }
    }
}

template <int LB, typename InT, int MODE, int FMT>
void lb_go(const InT* in, int64_t b, int64_t rows_pad, int64_t cols, unsigned* ar, unsigned* ap,
           const float* sr, const float* sp, uint8_t* cr, uint8_t* cp, unsigned* err, float* sro, float* spo,
           float* xout, int64_t rows_out, cudaStream_t st) {
    using C = LbCfg<LB, InT>;
    auto kern = k_cols_lb<LB, InT, MODE, FMT>;
    static bool init = false;
    if (!init) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
        init = true;
    }
    const int64_t strips = (rows_pad / C::B) * (cols / C::W);
    const int64_t cap = (int64_t)num_sms() * C::CTAS;
    const unsigned grid = (unsigned)(strips < cap ? strips : cap);
    launch_pdl(kern, dim3(grid < 1 ? 1 : grid), dim3(C::NT), C::SMEM, st, in, b, rows_pad, cols,
               hadamard_norm(C::B), ar, ap, sr, sp, cr, cp, err, sro, spo, xout, rows_out);
}

template <int LB, typename InT>
void lb_mode(int mode, int fmt, const InT* in, int64_t b, int64_t rows_pad, int64_t cols, unsigned* ar,
             unsigned* ap, const float* sr, const float* sp, uint8_t* cr, uint8_t* cp, unsigned* err, float* sro,
             float* spo, float* xout, int64_t rows_out, cudaStream_t st) {
#define HALO_LB(M, F) lb_go<LB, InT, M, F>(in, b, rows_pad, cols, ar, ap, sr, sp, cr, cp, err, sro, spo, xout, rows_out, st)
    if (mode == LB_ABSMAX) HALO_LB(LB_ABSMAX, FMT_INT8);
    else if (mode == LB_XFORM) {
        if constexpr (sizeof(InT) == 4) HALO_LB(LB_XFORM, FMT_INT8);
    } else if (fmt == FMT_INT8) HALO_LB(LB_QUANT, FMT_INT8);
    else if (fmt == FMT_E3M2) HALO_LB(LB_QUANT, FMT_E3M2);
    else HALO_LB(LB_QUANT, FMT_E4M3);
#undef HALO_LB
}

bool lb_enabled() {
    static const bool on = [] {
        const char* e = getenv("HALO_K2_LB");
        return !(e && e[0] == '0');
    }();
    return on;
}

}  // namespace

// K2 modes 0 (absmax of the rotated and, with ap, the plain operand) /
// 1 (rotated codes for rows_pad rows + plain codes for b rows) / 2
// (transform only: fp32 in, normalised fp32 rows < rows_out out, in place
// allowed) for 512 <= B <= 4096.  Returns false (caller falls back) for
// shapes it does not cover: cols not a multiple of the strip width, or
// rows that are not 16-byte aligned.
bool cols_lb(int mode, int fmt, int in_dtype, const void* in, int64_t b, int64_t rows_pad, int64_t cols, int64_t B,
             unsigned* ar, unsigned* ap, const float* sr, const float* sp, uint8_t* cr, uint8_t* cp, unsigned* err,
             float* sro, float* spo, cudaStream_t st, float* xout, int64_t rows_out) {
    if (!lb_enabled() || mode > 2 || B < 512 || B > 4096 || (B & (B - 1)) || rows_pad % B || b <= 0) return false;
    if (mode == LB_XFORM && (in_dtype != DT_F32 || !xout)) return false;
    const int es = in_dtype == DT_BF16 ? 2 : 4;
    const int64_t W = ((es == 2 && B >= 1024) ? 32768 : 16384) / B;  // LbCfg::W
    if (cols % W || (uintptr_t)in % 16 || (cols * es) % 16) return false;
    if (mode == LB_QUANT && ((uintptr_t)cr % 16 || (cp && (uintptr_t)cp % 4))) return false;
    if (mode == LB_XFORM && (uintptr_t)xout % 16) return false;
    if (mode == LB_ABSMAX && sp) ap = nullptr;  // supplied plain scale: no plain absmax
    int lb = 0;
    while ((int64_t(1) << lb) < B) ++lb;
#define HALO_LBT(L)                                                                                                  \
    if (es == 2)                                                                                                     \
        lb_mode<L, __nv_bfloat16>(mode, fmt, static_cast<const __nv_bfloat16*>(in), b, rows_pad, cols, ar, ap, sr, sp, cr, cp, err, sro, spo, xout,    \
                                  rows_out, st);                                                                     \
    else                                                                                                             \
        lb_mode<L, float>(mode, fmt, static_cast<const float*>(in), b, rows_pad, cols, ar, ap, sr, sp, cr, cp, err, sro, spo, xout, rows_out, st);
    switch (lb) {
    case 9: HALO_LBT(9) break;
    case 10: HALO_LBT(10) break;
    case 11: HALO_LBT(11) break;
    default: HALO_LBT(12) break;
    }
#undef HALO_LBT
    return true;
}

}  // namespace halo_b200
