// fwht3.cu — K1 / K4-right, third generation: right (row) blockwise FWHT for
// Hadamard blocks B = 2^LB <= 256, fused with absmax (phase A), quantize
// (phase B) or a plain transformed store (K4-right), sm_100a.
//
// Arithmetic is the reference's, bit for bit (hadamard.hpp:136-177): stages
// len = 1, 2, 4, ... in fp32 add/sub, one normalising multiply by
// float(1/sqrt(double(B))) (folded exactly into the quantizer scale when
// B = 4^k).  Codes follow quantize.hpp:244-280 via quant_round.cuh.
//
// What changed against fwht2.cu (issue-bound at ~30 thread instructions per
// element): the block size is a template parameter (no runtime stage
// branches) and the work is laid out for sm_100a's packed fp32 pipe:
//   * phase 1: lane holds 32 CONTIGUOUS elements (two 256-bit loads,
//     LDG.E.ENL2.256); stage 1 is scalar, stages 2..16 are FADD2 pairs;
//   * one XOR-swizzled, conflict-free smem exchange (8 STS.128 + 8 LDS.128
//     per lane) turns the 8 lanes of a 256-element segment from
//     "block p of 32" into "chunk r of 4 contiguous elements of every block";
//   * phase 2: stages 32..128 as FADD2 pairs across the 8 chunks;
//   * quantize in pairs: q = RNE(x*inv) by one FFMA2 with the 1.5*2^23
//     magic, certified by the once-rounded residual x - q*s (FFMA2;
//     quant_round.cuh quant_int8_try_r); a running FMNMX3 of |residual|
//     decides the rare exact path once per 32 elements (inputs within ~2^-22
//     of a rounding midpoint), 4 contiguous codes are packed
//     with 3 PRMT and written as one 32-bit store (8 lanes x 4 B = full
//     32 B sectors per segment);
//   * absmax: the last stage is skipped (max(|u+v|,|u-v|) = |u|+|v|
//     exactly), a NaN-propagating FMNMX3 carries non-finite inputs into the
//     absmax word (every FWHT output of a block containing Inf/NaN is
//     non-finite), so no separate finiteness pass is needed.
#include <cstdlib>

#include "common.cuh"
#include "halo_internal.h"
#include "sm100.cuh"

namespace halo_b200 {

namespace {

__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ void bfly2(float2& a, float2& b) {
    const float2 x = a, y = b;
    a = add2(x, y);
    b = sub2(x, y);
}
__device__ __forceinline__ float fmax3(float a, float b, float c) { return fmaxf(fmaxf(a, b), c); }
__device__ __forceinline__ float max3nan(float a, float b, float c) {
    float r;
    asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// 32 contiguous inputs -> 16 float2 (pair k = elements 2k, 2k+1)
template <typename InT>
struct Load32;
template <>
struct Load32<__nv_bfloat16> {
    uint32_t r[16];
    __device__ __forceinline__ void load(const __nv_bfloat16* p, bool lo_ok, bool hi_ok) {
        const uint32_t* q = reinterpret_cast<const uint32_t*>(p);
        if (lo_ok)
            asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                         : "l"(q));
        else
            for (int i = 0; i < 8; ++i) r[i] = 0;
        if (hi_ok)
            asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                           "=r"(r[15])
                         : "l"(q + 8));
        else
            for (int i = 8; i < 16; ++i) r[i] = 0;
    }
    __device__ __forceinline__ void get(float2 (&v)[16]) const {
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = make_float2(__uint_as_float(r[k] << 16), __uint_as_float(r[k] & 0xFFFF0000u));
    }
};
template <>
struct Load32<float> {
    float r[32];
    __device__ __forceinline__ void ld8(const float* p, int o) {
        asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r[o]), "=f"(r[o + 1]), "=f"(r[o + 2]), "=f"(r[o + 3]), "=f"(r[o + 4]), "=f"(r[o + 5]),
                       "=f"(r[o + 6]), "=f"(r[o + 7])
                     : "l"(p));
    }
    __device__ __forceinline__ void load(const float* p, bool lo_ok, bool hi_ok) {
        if (lo_ok) {
            ld8(p, 0);
            ld8(p + 8, 8);
        } else {
            for (int i = 0; i < 16; ++i) r[i] = 0.f;
        }
        if (hi_ok) {
            ld8(p + 16, 16);
            ld8(p + 24, 24);
        } else {
            for (int i = 16; i < 32; ++i) r[i] = 0.f;
        }
    }
    __device__ __forceinline__ void get(float2 (&v)[16]) const {
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = make_float2(r[2 * k], r[2 * k + 1]);
    }
};

// 4 codes (low bytes of the magic-rounded fp32 words) -> one word
__device__ __forceinline__ uint32_t pack4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    return __byte_perm(__byte_perm(a, b, 0x0040), __byte_perm(c, d, 0x0040), 0x5410);
}

}  // namespace

template <int FMT>
__device__ __noinline__ uint32_t exact4(float2 a, float2 b, float s, float inv) {
    if constexpr (FMT == FMT_INT8)
        return pack4((uint8_t)quant_int8(a.x, s, inv), (uint8_t)quant_int8(a.y, s, inv), (uint8_t)quant_int8(b.x, s, inv),
                     (uint8_t)quant_int8(b.y, s, inv));
    else if constexpr (FMT == FMT_E3M2)
        return pack4(quant_e3m2(a.x, s, inv) << 2, quant_e3m2(a.y, s, inv) << 2, quant_e3m2(b.x, s, inv) << 2,
                     quant_e3m2(b.y, s, inv) << 2);
    else
        return pack4(quant_e4m3(a.x, s, inv), quant_e4m3(a.y, s, inv), quant_e4m3(b.x, s, inv), quant_e4m3(b.y, s, inv));
}

// does any of these 4 elements need the exact path?  (re-derived in the
// rare slow branch with the same criteria as the hot loop)
template <int FMT, bool SUP>
__device__ __forceinline__ bool group_slow(float2 a, float2 b, float s, float inv, float h) {
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

enum : int { V3_ABSMAX = 0, V3_QUANT = 1, V3_XFORM = 2, V3_ABSMAX_ROWS = 3, V3_QUANT_ROWS = 4 };
// per-row scale modes (Granularity::row, quantize.hpp:73-132): one absmax
// word / scale per row of `cols` elements (cols a multiple of 256, so every
// 256-element segment of a lane lies in one row)
template <int MODE> __host__ __device__ constexpr bool v3_abs() { return MODE == V3_ABSMAX || MODE == V3_ABSMAX_ROWS; }
template <int MODE> __host__ __device__ constexpr bool v3_q() { return MODE == V3_QUANT || MODE == V3_QUANT_ROWS; }
template <int MODE> __host__ __device__ constexpr bool v3_rows() { return MODE == V3_ABSMAX_ROWS || MODE == V3_QUANT_ROWS; }


// ------------------------------------------------------------------ core
// One warp iteration = one chunk of 1024 elements = 4 segments of 256; lane
// l = (segment k = l>>3, part p = l&7) enters with the 32 contiguous inputs
// base + 256k + 32p + 0..31 (pair i = elements 2i, 2i+1).  B <= 32: every
// stage runs in phase 1 and the lane owns those 32 outputs; B >= 64: the
// exchange gives the lane chunk p (4 contiguous elements) of every 32-block
// of its segment.
template <int LB, int FMT, int MODE, bool SUP, typename OutT>
struct RowsCore {
    static constexpr bool FOLD = (LB % 2) == 0;  // norm = 2^-LB/2 folds into the scale
    static constexpr int P1 = LB < 5 ? LB : 5;   // stages in phase 1
    static constexpr bool X2 = LB > 5;           // phase 2 needed
    static constexpr int P2 = X2 ? LB - 5 : 0;   // stages in phase 2

    float s = 1.f, inv = 1.f, norm = 1.f, amax = 0.f;
    float thr = 0.5f;  // slow-path threshold on the running residual maximum
    float2 inv2, magic2, norm2, nsm2, ilo2, ihi2;
    int64_t cols = 0;                  // row length (per-row modes)
    unsigned* amax_rows = nullptr;     // V3_ABSMAX_ROWS: one absmax word per row
    const float* row_scale = nullptr;  // V3_QUANT_ROWS: per-row scales (k_row_scales)

    // per-row modes: the scale of the row holding element e0
    __device__ __forceinline__ void row_setup(int64_t e0) {
        if constexpr (MODE == V3_QUANT_ROWS) {
            s = __ldg(row_scale + e0 / cols);
            // any inv near 1/s works: candidates are certified against s
            inv = FMT == FMT_INT8 ? __fdividef(1.0f, s) : __frcp_rn(s);
            if (FOLD) {
                s = s / norm;
                inv = inv * norm;
            }
            inv2 = make_float2(inv, inv);
            nsm2 = make_float2(-s, -s);
            if (FMT == FMT_INT8) thr = half_margin(s);
            else e4m3_brackets(inv, ilo2, ihi2);
        }
    }
    // per-row absmax: reduce the lane's segment maximum over the 8 lanes of
    // the segment (lanes 8k..8k+7), one atomic per segment and chunk
    __device__ __forceinline__ void row_flush(int64_t e0, unsigned* err) {
        if constexpr (MODE == V3_ABSMAX_ROWS) {
            float m = amax;
#pragma unroll
            for (int o = 4; o > 0; o >>= 1) m = max3nan(m, __shfl_xor_sync(0xffffffffu, m, o), 0.f);
            m *= norm;
            if ((threadIdx.x & 7) == 0) {
                atomic_absmax(amax_rows + e0 / cols, fabsf(m));
                if (!(m <= 3.402823466e38f)) atomicOr(err, ERRF_NONFINITE);
            }
            amax = 0.f;
        }
    }

    __device__ __forceinline__ void init(const unsigned* absmax, const float* supplied, float nrm, unsigned* err,
                                         float* scale_out) {
        norm = nrm;
        if constexpr (MODE == V3_QUANT) {
            resolve_scale(absmax, supplied, FMT, &s, &inv);
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                if (scale_out) *scale_out = s;
                if (!SUP && (*absmax >= 0x7f800000u)) atomicOr(err, ERRF_NONFINITE);
            }
            if (FOLD) {
                s = s / norm;  // exact power-of-two rescale
                inv = inv * norm;
            }
        }
        inv2 = make_float2(inv, inv);
        magic2 = make_float2(kRoundMagic, kRoundMagic);
        nsm2 = make_float2(-s, -s);
        if (FMT == FMT_INT8) thr = half_margin(s);
        else e4m3_brackets(inv, ilo2, ihi2);
        norm2 = make_float2(norm, norm);
    }

    // phase 1: stages len = 1 .. min(B, 32)/2 in registers
    __device__ __forceinline__ void phase1(float2 (&v)[16]) {
        if constexpr (P1 >= 1) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                if (v3_abs<MODE>() && LB == 1) {
                    amax = max3nan(amax, fabsf(v[i].x) + fabsf(v[i].y), 0.f);
                } else {
                    const float a = v[i].x, b = v[i].y;
                    v[i] = make_float2(a + b, a - b);
                }
            }
        }
#pragma unroll
        for (int t = 1; t < P1; ++t) {
            const int h = 1 << (t - 1);  // pair-index distance for len = 2^t
            const bool last = v3_abs<MODE>() && !X2 && (t == LB - 1);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                if ((i & h) == 0) {
                    if (last) amax = max3nan(amax, fabsf(v[i].x) + fabsf(v[i + h].x), fabsf(v[i].y) + fabsf(v[i + h].y));
                    else bfly2(v[i], v[i + h]);
                }
            }
        }
        if constexpr (v3_abs<MODE>() && LB == 0) {
#pragma unroll
            for (int i = 0; i < 16; ++i) amax = max3nan(amax, fabsf(v[i].x), fabsf(v[i].y));
        }
    }

    // 4 contiguous outputs (a = elements 0,1; c = 2,3) -> code word; running
    // fast-path residual maximum in dmax
    __device__ __forceinline__ uint32_t quant4(float2& a, float2& c, float& dmax) const {
        if (!FOLD) {
            a = mul2(a, norm2);
            c = mul2(c, norm2);
        }
        if constexpr (FMT == FMT_INT8) {
            // candidate q = RNE(x*inv) by the magic add, certified by the
            // once-rounded residual x - q*s (quant_int8_try_r)
            const float2 ta = __ffma2_rn(a, inv2, magic2), tc = __ffma2_rn(c, inv2, magic2);
            const float2 qa = sub2(ta, magic2), qc = sub2(tc, magic2);
            const float2 ra = __ffma2_rn(qa, nsm2, a), rc = __ffma2_rn(qc, nsm2, c);
            float m = fmax3(fmax3(0.f, fabsf(ra.x), fabsf(ra.y)), fabsf(rc.x), fabsf(rc.y));
            if (SUP)  // |q| <= 127 (the clamp) maps below thr, |q| >= 128 above it
                m = fmaxf(m, fmax3(fmax3(0.f, fabsf(qa.x), fabsf(qa.y)), fabsf(qc.x), fabsf(qc.y)) * (thr / 127.5f));
            // uncertified group (within ~2^-22 of a midpoint, or clamped):
            // decide its 4 codes exactly right here (divergent but rare)
            if (!(m < thr)) return exact4<FMT>(a, c, s, inv);
            return pack4(__float_as_uint(ta.x), __float_as_uint(ta.y), __float_as_uint(tc.x), __float_as_uint(tc.y));
        } else if constexpr (FMT == FMT_E3M2) {
            return e3m2x4_fast(a, c, ilo2, ihi2, s);
        } else {
            uint32_t bad = 0;
            const uint32_t w = e4m3x4_fast(a, c, ilo2, ihi2, s, bad);
            dmax = bad ? 1.0f : dmax;
            return w;
        }
    }

    // B = 512 / 1024 (LB 9, 10): a segment is NP = 16 / 32 lanes (two / one
    // per warp chunk); one exchange through the warp's 4 KB gives lane pp
    // the CW = 2 / 1 elements at offset CW*pp of every 32-block of its
    // segment (slot pp*NP + (q ^ pp): conflict-free both ways), then the
    // block-index bits run as FADD2 pairs -- one exchange where the generic
    // large-block kernel needs a round per 3 bits.
    __device__ __forceinline__ void finish_wide(float2 (&v)[16], int64_t base, int64_t n, float4* S,
                                                uint8_t* __restrict__ codes, OutT* __restrict__ out) {
        constexpr int NP = 1 << (LB - 5);
        const int l = threadIdx.x & 31;
        const int kk = l / NP, pp = l % NP;
        const int64_t sb = base + (int64_t)kk * (NP * 32);  // segment base
        float2 U[16];  // LB 9: U[b] = elements 32b + 2pp + {0,1}; LB 10: U[j] = (32j + pp, 32(j+16) + pp)
        if constexpr (LB == 9) {
            float2* T = reinterpret_cast<float2*>(S) + kk * 256;
#pragma unroll
            for (int q = 0; q < 16; ++q) T[pp * 16 + (q ^ pp)] = v[q];
            __syncwarp();
#pragma unroll
            for (int b = 0; b < 16; ++b) U[b] = T[b * 16 + (pp ^ b)];
            __syncwarp();
        } else {
            float* T = reinterpret_cast<float*>(S);
#pragma unroll
            for (int q = 0; q < 16; ++q) {
                T[pp * 32 + ((2 * q) ^ pp)] = v[q].x;
                T[pp * 32 + ((2 * q + 1) ^ pp)] = v[q].y;
            }
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 16; ++j) U[j] = make_float2(T[j * 32 + (pp ^ j)], T[(j + 16) * 32 + (pp ^ (j + 16))]);
            __syncwarp();
        }
        // phase 2: block-index bit t <-> stage len = 32 << t
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int h = 1 << t;
            const bool last = v3_abs<MODE>() && LB == 9 && t == 3;
#pragma unroll
            for (int b = 0; b < 16; ++b)
                if ((b & h) == 0) {
                    if (last) amax = max3nan(amax, fabsf(U[b].x) + fabsf(U[b + h].x), fabsf(U[b].y) + fabsf(U[b + h].y));
                    else bfly2(U[b], U[b + h]);
                }
        }
        if constexpr (LB == 10) {  // len = 512: the two halves of each U
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                if constexpr (v3_abs<MODE>()) {
                    amax = max3nan(amax, fabsf(U[j].x) + fabsf(U[j].y), 0.f);
                } else {
                    const float a = U[j].x, c = U[j].y;
                    U[j] = make_float2(a + c, a - c);
                }
            }
        }
        // element offset (within the segment) of value w (0/1) of U[i]
        auto off = [&](int i, int w) -> int64_t { return LB == 9 ? 32 * i + 2 * pp + w : 32 * (i + 16 * w) + pp; };
        if constexpr (v3_q<MODE>()) {
            float dmax = 0.f;
            uint32_t wd[8];
#pragma unroll
            for (int g = 0; g < 8; ++g) wd[g] = quant4(U[2 * g], U[2 * g + 1], dmax);
            if (__any_sync(0xffffffffu, !(dmax < thr))) {
                if (!(dmax < thr)) {
#pragma unroll
                    for (int g = 0; g < 8; ++g)
                        if (group_slow<FMT, SUP>(U[2 * g], U[2 * g + 1], s, inv, thr))
                            wd[g] = exact4<FMT>(U[2 * g], U[2 * g + 1], s, inv);
                }
            }
            if (sb < n) {
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    const uint32_t w = wd[g];
                    if constexpr (LB == 9) {  // bytes 0,1 -> block 2g; 2,3 -> block 2g+1
                        *reinterpret_cast<uint16_t*>(codes + sb + off(2 * g, 0)) = (uint16_t)(w & 0xFFFFu);
                        *reinterpret_cast<uint16_t*>(codes + sb + off(2 * g + 1, 0)) = (uint16_t)(w >> 16);
                    } else {  // bytes: U[2g].x, U[2g].y, U[2g+1].x, U[2g+1].y
                        codes[sb + off(2 * g, 0)] = (uint8_t)(w & 0xFFu);
                        codes[sb + off(2 * g, 1)] = (uint8_t)((w >> 8) & 0xFFu);
                        codes[sb + off(2 * g + 1, 0)] = (uint8_t)((w >> 16) & 0xFFu);
                        codes[sb + off(2 * g + 1, 1)] = (uint8_t)(w >> 24);
                    }
                }
            }
        } else if constexpr (MODE == V3_XFORM) {
            if (sb < n) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const float2 a = mul2(U[i], norm2);
                    if constexpr (LB == 9) {
                        if constexpr (sizeof(OutT) == 4) *reinterpret_cast<float2*>(out + sb + off(i, 0)) = a;
                        else *reinterpret_cast<uint32_t*>(out + sb + off(i, 0)) = pack_bf16x2(a.x, a.y);
                    } else {
                        if constexpr (sizeof(OutT) == 4) {
                            out[sb + off(i, 0)] = a.x;
                            out[sb + off(i, 1)] = a.y;
                        } else {
                            out[sb + off(i, 0)] = __float2bfloat16_rn(a.x);
                            out[sb + off(i, 1)] = __float2bfloat16_rn(a.y);
                        }
                    }
                }
            }
        }
    }

    // everything after phase 1 (all 32 lanes of the warp call this together)
    __device__ __forceinline__ void finish(float2 (&v)[16], int64_t base, int64_t n, int k, int p, float4* S,
                                           uint8_t* __restrict__ codes, OutT* __restrict__ out) {
        if constexpr (LB == 9 || LB == 10) {
            finish_wide(v, base, n, S, codes, out);
        } else if constexpr (!X2) {
            const int64_t e0 = base + k * 256 + p * 32;
            if constexpr (v3_q<MODE>()) {
                float dmax = 0.f;
                uint32_t wd[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) wd[q] = quant4(v[2 * q], v[2 * q + 1], dmax);
                if (__any_sync(0xffffffffu, !(dmax < thr))) {
                    if (!(dmax < thr)) {
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            if (group_slow<FMT, SUP>(v[2 * q], v[2 * q + 1], s, inv, thr))
                                wd[q] = exact4<FMT>(v[2 * q], v[2 * q + 1], s, inv);
                    }
                }
                if (e0 < n) {
                    uint32_t* d = reinterpret_cast<uint32_t*>(codes + e0);
                    if (e0 + 32 <= n) {
                        asm volatile("st.global.v8.u32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(d), "r"(wd[0]),
                                     "r"(wd[1]), "r"(wd[2]), "r"(wd[3]), "r"(wd[4]), "r"(wd[5]), "r"(wd[6]), "r"(wd[7])
                                     : "memory");
                    } else {
                        *reinterpret_cast<uint4*>(d) = make_uint4(wd[0], wd[1], wd[2], wd[3]);
                    }
                }
            } else if constexpr (MODE == V3_XFORM) {
                if (e0 < n) {
                    const int cnt = (e0 + 32 <= n) ? 4 : 2;  // 8-element groups
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        if (g < cnt) {
                            float2 o[4];
#pragma unroll
                            for (int m = 0; m < 4; ++m) o[m] = mul2(v[4 * g + m], norm2);
                            if constexpr (sizeof(OutT) == 4) {
                                float4* d = reinterpret_cast<float4*>(out + e0 + 8 * g);
                                d[0] = make_float4(o[0].x, o[0].y, o[1].x, o[1].y);
                                d[1] = make_float4(o[2].x, o[2].y, o[3].x, o[3].y);
                            } else {
                                *reinterpret_cast<uint4*>(out + e0 + 8 * g) =
                                    make_uint4(pack_bf16x2(o[0].x, o[0].y), pack_bf16x2(o[1].x, o[1].y),
                                               pack_bf16x2(o[2].x, o[2].y), pack_bf16x2(o[3].x, o[3].y));
                            }
                        }
                    }
                }
            }
        } else {
            // ---------------- exchange: (block p, chunk q) -> slot 8p + (q ^ p) of segment k
            float4* T = S + k * 64;
#pragma unroll
            for (int q = 0; q < 8; ++q)
                T[p * 8 + (q ^ p)] = make_float4(v[2 * q].x, v[2 * q].y, v[2 * q + 1].x, v[2 * q + 1].y);
            __syncwarp();
            float2 u[8][2];
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const float4 f = T[b * 8 + (p ^ b)];
                u[b][0] = make_float2(f.x, f.y);
                u[b][1] = make_float2(f.z, f.w);
            }
            __syncwarp();
            // ---------------- phase 2: len = 32 << t  <->  block-index bit t
#pragma unroll
            for (int t = 0; t < P2; ++t) {
                const int h = 1 << t;
                const bool last = v3_abs<MODE>() && (t == P2 - 1);
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    if ((b & h) == 0) {
                        if (last) {
                            amax = max3nan(amax, fabsf(u[b][0].x) + fabsf(u[b + h][0].x),
                                           fabsf(u[b][0].y) + fabsf(u[b + h][0].y));
                            amax = max3nan(amax, fabsf(u[b][1].x) + fabsf(u[b + h][1].x),
                                           fabsf(u[b][1].y) + fabsf(u[b + h][1].y));
                        } else {
                            bfly2(u[b][0], u[b + h][0]);
                            bfly2(u[b][1], u[b + h][1]);
                        }
                    }
                }
            }
            // lane's outputs: elements base + 256k + 32b + 4p + 0..3
            const int64_t e0 = base + k * 256 + 4 * p;
            if constexpr (v3_q<MODE>()) {
                float dmax = 0.f;
                uint32_t* dst = reinterpret_cast<uint32_t*>(codes + e0);
                if (base + 1024 <= n) {  // interior chunk: no per-group bounds
#pragma unroll
                    for (int b = 0; b < 8; ++b) dst[8 * b] = quant4(u[b][0], u[b][1], dmax);
                } else {
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        const uint32_t wd = quant4(u[b][0], u[b][1], dmax);
                        if (e0 + 32 * b < n) dst[8 * b] = wd;
                    }
                }
                if (__any_sync(0xffffffffu, !(dmax < thr))) {
                    if (!(dmax < thr)) {
                        // rare: re-store the groups the fast path cannot certify
#pragma unroll
                        for (int b = 0; b < 8; ++b)
                            if (group_slow<FMT, SUP>(u[b][0], u[b][1], s, inv, thr) && e0 + 32 * b < n)
                                *reinterpret_cast<uint32_t*>(codes + e0 + 32 * b) = exact4<FMT>(u[b][0], u[b][1], s, inv);
                    }
                }
            } else if constexpr (MODE == V3_XFORM) {
                // the optional bf16 addend (see below): all 8 loads in flight first
                uint2 addq[8];
                if constexpr (sizeof(OutT) == 2) {
                    if (codes) {
#pragma unroll
                        for (int b = 0; b < 8; ++b)
                            addq[b] = e0 + 32 * b < n ? __ldg(reinterpret_cast<const uint2*>(codes) + (e0 + 32 * b) / 4)
                                                      : make_uint2(0u, 0u);
                    }
                }
#pragma unroll
                for (int b = 0; b < 8; ++b) {
                    if (e0 + 32 * b < n) {
                        const float2 a = mul2(u[b][0], norm2), c = mul2(u[b][1], norm2);
                        if constexpr (sizeof(OutT) == 4) {
                            *reinterpret_cast<float4*>(out + e0 + 32 * b) = make_float4(a.x, a.y, c.x, c.y);
                        } else {
                            uint2 o = make_uint2(pack_bf16x2(a.x, a.y), pack_bf16x2(c.x, c.y));
                            if (codes) {
                                // XFORM: `codes` carries an optional bf16 addend
                                // (rows_xform_add): out = RN(add + RN(value)),
                                // a bf16 tensor add of the transformed output
                                const uint2 q = addq[b];
                                o.x = pack_bf16x2(__uint_as_float(q.x << 16) + __uint_as_float(o.x << 16),
                                                  __uint_as_float(q.x & 0xFFFF0000u) + __uint_as_float(o.x & 0xFFFF0000u));
                                o.y = pack_bf16x2(__uint_as_float(q.y << 16) + __uint_as_float(o.y << 16),
                                                  __uint_as_float(q.y & 0xFFFF0000u) + __uint_as_float(o.y & 0xFFFF0000u));
                            }
                            *reinterpret_cast<uint2*>(out + e0 + 32 * b) = o;
                        }
                    }
                }
            }
        }
    }

    __device__ __forceinline__ void reduce(unsigned* absmax, unsigned* err) {
        if constexpr (MODE == V3_ABSMAX) {
            // warp max (NaN-propagating), then the normalising multiply once:
            // max(fl(|x| * norm)) == fl(max|x| * norm) (monotone rounding)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) amax = max3nan(amax, __shfl_xor_sync(0xffffffffu, amax, o), 0.f);
            amax *= norm;
            if ((threadIdx.x & 31) == 0) {
                atomic_absmax(absmax, fabsf(amax));
                if (!(amax <= 3.402823466e38f)) atomicOr(err, ERRF_NONFINITE);
            }
        }
    }
};

// ------------------------------------------------ v3: direct 256-bit loads
template <int LB, typename InT, int FMT, int MODE, bool SUP, typename OutT>
__global__ void __launch_bounds__(256) k_rows_v3(const InT* __restrict__ in, int64_t n, int64_t cols, float norm,
                                                 unsigned* absmax, const float* supplied, uint8_t* __restrict__ codes,
                                                 OutT* __restrict__ out, unsigned* err, float* scale_out) {
    __shared__ __align__(16) float4 xs[8][4 * 64];  // per warp: 4 segments x 64 float4 slots
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int k = l >> 3, p = l & 7;
    RowsCore<LB, FMT, MODE, SUP, OutT> core;
    core.init(absmax, supplied, norm, err, scale_out);
    core.cols = cols;
    core.amax_rows = absmax;
    core.row_scale = supplied;
    const int64_t nchunks = (n + 1023) >> 10;
    const int64_t cstride = (int64_t)gridDim.x * 8;
    const int lane_off = k * 256 + p * 32;
    Load32<InT> cur, nxt;
    auto load_chunk = [&](Load32<InT>& r, int64_t cc) {
        const int64_t e0 = (cc << 10) + lane_off;
        r.load(in + e0, e0 < n, e0 + 16 < n);
    };
    const int64_t c0 = (int64_t)blockIdx.x * 8 + w;
    if (c0 < nchunks) load_chunk(cur, c0);
    for (int64_t c = c0; c < nchunks; c += cstride) {
        float2 v[16];
        cur.get(v);
        if (c + cstride < nchunks) load_chunk(nxt, c + cstride);
        const int64_t seg0 = (c << 10) + k * 256;  // this lane's 256-element segment
        core.row_setup(seg0);
        core.phase1(v);
        core.finish(v, c << 10, n, k, p, xs[w], codes, out);
        core.row_flush(seg0, err);
        cur = nxt;
    }
    core.reduce(absmax, err);
}

// ------------------------------------- v4: TMA-staged (128 B swizzled) input
// Each warp streams its chunks through a private S-deep ring of smem stages
// filled by cp.async.bulk.tensor (one elected lane, mbarrier complete_tx), so
// the bytes in flight do not cost registers: 4 warps/CTA x S stages x 2 KB.
// The tensor map views the input as rows of 128 B; the 128 B swizzle makes
// the lanes' 16 B reads conflict-free.
template <typename InT>
struct V4Cfg {
    static constexpr int ROW_ELEMS = 128 / sizeof(InT);       // 64 bf16 / 32 fp32
    static constexpr int CHUNK_ROWS = 1024 / ROW_ELEMS;       // 16 / 32
    static constexpr int STAGE_BYTES = 1024 * sizeof(InT);    // 2 / 4 KB
    static constexpr int STAGES = sizeof(InT) == 2 ? 2 : 3;
    static constexpr int WARPS = 4;
    static constexpr int XCH_BYTES = 4096;                    // exchange, per warp
    static constexpr size_t SMEM = 1024 + (size_t)WARPS * (STAGES * STAGE_BYTES + XCH_BYTES) + WARPS * STAGES * 8;
};

template <typename InT>
__device__ __forceinline__ void v4_read(const uint8_t* stage, int k, int p, float2 (&v)[16]) {
    if constexpr (sizeof(InT) == 2) {
        const int row = 4 * k + (p >> 1);
        const uint8_t* r = stage + row * 128;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint4 q = *reinterpret_cast<const uint4*>(r + ((((p & 1) * 4 + j) ^ (row & 7)) << 4));
            const uint32_t wv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int m = 0; m < 4; ++m)
                v[4 * j + m] = make_float2(__uint_as_float(wv[m] << 16), __uint_as_float(wv[m] & 0xFFFF0000u));
        }
    } else {
        const int row = 8 * k + p;
        const uint8_t* r = stage + row * 128;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float4 q = *reinterpret_cast<const float4*>(r + ((j ^ (row & 7)) << 4));
            v[2 * j] = make_float2(q.x, q.y);
            v[2 * j + 1] = make_float2(q.z, q.w);
        }
    }
}

template <int LB, typename InT, int FMT, int MODE, bool SUP, typename OutT>
__global__ void __launch_bounds__(128) k_rows_v4(const __grid_constant__ CUtensorMap tm, int64_t n, int64_t cols, float norm,
                                                 unsigned* absmax, const float* supplied,
                                                 uint8_t* __restrict__ codes, OutT* __restrict__ out, unsigned* err,
                                                 float* scale_out) {
    using C = V4Cfg<InT>;
    extern __shared__ uint8_t smem_raw[];
    // 1024 B alignment for the 128 B swizzle, by pointer arithmetic on the
    // __shared__ array so every access stays an LDS/STS (not a generic LD/ST)
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int k = l >> 3, p = l & 7;
    uint8_t* stages = smem + w * C::STAGES * C::STAGE_BYTES;
    float4* xch = reinterpret_cast<float4*>(smem + C::WARPS * C::STAGES * C::STAGE_BYTES + w * C::XCH_BYTES);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::WARPS * (C::STAGES * C::STAGE_BYTES + C::XCH_BYTES)) +
                     w * C::STAGES;

    const int64_t nchunks = (n + 1023) >> 10;
    const int64_t G = (int64_t)gridDim.x * C::WARPS;
    const int64_t c0 = (int64_t)blockIdx.x * C::WARPS + w;
    if (l == 0) {
        if (w == 0) tma_prefetch_desc(&tm);
        for (int s = 0; s < C::STAGES; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // everything above overlaps the previous kernel's tail (PDL)
    pdl_wait();
    pdl_trigger();
    if (l == 0) {
        for (int s = 0; s < C::STAGES; ++s) {
            const int64_t c = c0 + s * G;
            if (c < nchunks) {
                mbar_expect_tx(&bars[s], C::STAGE_BYTES);
                tma_load_2d(stages + s * C::STAGE_BYTES, &tm, &bars[s], 0, (int)(c * C::CHUNK_ROWS));
            }
        }
    }
    __syncwarp();
    RowsCore<LB, FMT, MODE, SUP, OutT> core;
    core.init(absmax, supplied, norm, err, scale_out);
    core.cols = cols;
    core.amax_rows = absmax;
    core.row_scale = supplied;
    int i = 0;
    for (int64_t c = c0; c < nchunks; c += G, ++i) {
        const int s = i % C::STAGES;
        mbar_wait(&bars[s], (uint32_t)(i / C::STAGES) & 1u);
        float2 v[16];
        v4_read<InT>(stages + s * C::STAGE_BYTES, k, p, v);
        const int64_t seg0 = (c << 10) + k * 256;  // this lane's 256-element segment
        core.row_setup(seg0);
        core.phase1(v);  // consumes every loaded value: the stage's reads are complete
        __syncwarp();
        if (l == 0) {
            const int64_t cn = c + C::STAGES * G;
            if (cn < nchunks) {
                // no proxy fence: the stage's generic-proxy reads completed
                // (their values fed phase 1) before the async-proxy refill
                mbar_expect_tx(&bars[s], C::STAGE_BYTES);
                tma_load_2d(stages + s * C::STAGE_BYTES, &tm, &bars[s], 0, (int)(cn * C::CHUNK_ROWS));
            }
        }
        core.finish(v, c << 10, n, k, p, xch, codes, out);
        core.row_flush(seg0, err);
    }
    core.reduce(absmax, err);
}

// ------------------------------- large blocks: 512 <= B <= 8192 (LB 9..13)
// A 256-thread CTA owns a tile of 8192 contiguous elements (8192 / B whole
// blocks), fp32 in 32 KB of shared memory.  Stage bits are processed in
// increasing order, the reference's (hadamard.hpp:140-176):
//   * bits 0..4 in registers exactly as RowsCore's phase 1 (thread t holds
//     elements 32t .. 32t+31);
//   * then rounds of up to 3 bits: a thread takes 8 float4 slots -- 4
//     consecutive elements (bits 0-1, four independent columns, so every
//     butterfly is an FADD2) x the 2^k values of the round's bits -- with
//     consecutive lanes on consecutive slots (conflict-free LDS.128 /
//     STS.128; the phase-1 write goes through an XOR swizzle of the slot's low
//     3 bits with bits 3-5), runs the k stages, writes back;
//   * the last round does not write back: it quantizes (4 codes -> one 32-bit
//     store, lanes on consecutive words), reduces the absmax (skipping the
//     last stage: max(|u+v|,|u-v|) = |u|+|v| exactly) or stores the
//     transformed values.
// One barrier per round.  Replaces the radix-16 scalar kernel of
// fwht_big.cu for these block sizes.
namespace {
constexpr int BG2_TILE = 8192;
__device__ __forceinline__ int bg2_phys(int q) { return q ^ ((q >> 3) & 7); }

template <int LB, int LO>
struct Bg2Round {
    static constexpr int K = (LB - LO) < 3 ? (LB - LO) : 3;
    static constexpr bool LAST = LO + K >= LB;
    // slot of (thread t, s = 0..7): round bits v = s & (2^K - 1), group g = s >> K
    __device__ __forceinline__ static int slot(int t, int s) {
        const int v = s & ((1 << K) - 1), g = s >> K;
        const int rest = t + 256 * g;                 // 11 - K bits: slot bits [0, LO-2) then [LO-2+K, 11)
        const int low = rest & ((1 << (LO - 2)) - 1);
        const int high = rest >> (LO - 2);
        return low | (v << (LO - 2)) | (high << (LO - 2 + K));
    }
};
}  // namespace


// rounds LO, LO+3, ... (compile-time recursion); the last one emits
template <int LB, int LO, int FMT, int MODE, bool SUP, typename OutT>
__device__ __forceinline__ void bg2_rounds(float4* S, int t, int64_t base, int64_t n,
                                           RowsCore<LB, FMT, MODE, SUP, OutT>& core, uint8_t* __restrict__ codes,
                                           OutT* __restrict__ out) {
    using R = Bg2Round<LB, LO>;
    float2 a[8], c[8];  // slot s: elements 0,1 in a[s], 2,3 in c[s]
    int q[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        q[s] = R::slot(t, s);
        const float4 f = S[bg2_phys(q[s])];
        a[s] = make_float2(f.x, f.y);
        c[s] = make_float2(f.z, f.w);
    }
#pragma unroll
    for (int b = 0; b < R::K; ++b) {
        const int h = 1 << b;
        const bool last_stage = v3_abs<MODE>() && R::LAST && b == R::K - 1;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
            if ((s & h) == 0) {
                if (last_stage) {
                    core.amax = max3nan(core.amax, fabsf(a[s].x) + fabsf(a[s + h].x), fabsf(a[s].y) + fabsf(a[s + h].y));
                    core.amax = max3nan(core.amax, fabsf(c[s].x) + fabsf(c[s + h].x), fabsf(c[s].y) + fabsf(c[s + h].y));
                } else {
                    bfly2(a[s], a[s + h]);
                    bfly2(c[s], c[s + h]);
                }
            }
        }
    }
    if constexpr (!R::LAST) {
#pragma unroll
        for (int s = 0; s < 8; ++s) S[bg2_phys(q[s])] = make_float4(a[s].x, a[s].y, c[s].x, c[s].y);
        __syncthreads();
        bg2_rounds<LB, LO + 3>(S, t, base, n, core, codes, out);
    } else {
        if constexpr (v3_q<MODE>()) {
            float dmax = 0.f;
            uint32_t wd[8];
#pragma unroll
            for (int s = 0; s < 8; ++s) wd[s] = core.quant4(a[s], c[s], dmax);
            if (__any_sync(0xffffffffu, !(dmax < core.thr))) {
                if (!(dmax < core.thr)) {
#pragma unroll
                    for (int s = 0; s < 8; ++s)
                        if (group_slow<FMT, SUP>(a[s], c[s], core.s, core.inv, core.thr))
                            wd[s] = exact4<FMT>(a[s], c[s], core.s, core.inv);
                }
            }
#pragma unroll
            for (int s = 0; s < 8; ++s) *reinterpret_cast<uint32_t*>(codes + base + 4 * q[s]) = wd[s];
        } else if constexpr (MODE == V3_XFORM) {
#pragma unroll
            for (int s = 0; s < 8; ++s) {
                const float2 x = mul2(a[s], core.norm2), y = mul2(c[s], core.norm2);
                if constexpr (sizeof(OutT) == 4)
                    *reinterpret_cast<float4*>(out + base + 4 * q[s]) = make_float4(x.x, x.y, y.x, y.y);
                else
                    *reinterpret_cast<uint2*>(out + base + 4 * q[s]) = make_uint2(pack_bf16x2(x.x, x.y), pack_bf16x2(y.x, y.y));
            }
        }
    }
}

template <int LB, typename InT, int FMT, int MODE, bool SUP, typename OutT>
__global__ void __launch_bounds__(256) k_rows_lb(const InT* __restrict__ in, int64_t n, float norm, unsigned* absmax,
                                                 const float* supplied, uint8_t* __restrict__ codes,
                                                 OutT* __restrict__ out, unsigned* err, float* scale_out) {
    __shared__ __align__(16) float4 S[BG2_TILE / 4];
    const int t = threadIdx.x;
    RowsCore<LB, FMT, MODE, SUP, OutT> core;
    core.init(absmax, supplied, norm, err, scale_out);
    const int64_t ntiles = n / BG2_TILE;
    // the next tile's global loads are issued before this tile's rounds so
    // their latency hides behind the shared-memory work
    Load32<InT> cur, nxt;
    if (blockIdx.x < ntiles) cur.load(in + (int64_t)blockIdx.x * BG2_TILE + 32 * t, true, true);
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t base = tile * BG2_TILE;
        // ---- bits 0..4 in registers
        float2 v[16];
        cur.get(v);
        if (tile + gridDim.x < ntiles) nxt.load(in + (tile + gridDim.x) * BG2_TILE + 32 * t, true, true);
        core.phase1(v);
        __syncthreads();  // the previous tile's last round has read its slots
#pragma unroll
        for (int j = 0; j < 8; ++j)
            S[bg2_phys(8 * t + j)] = make_float4(v[2 * j].x, v[2 * j].y, v[2 * j + 1].x, v[2 * j + 1].y);
        __syncthreads();
        bg2_rounds<LB, 5>(S, t, base, n, core, codes, out);
        cur = nxt;
    }
    core.reduce(absmax, err);
}

// ------------------------------------------ SwiGLU forward + K1 phase A
// h = silu(g) * u (swiglu_fwd1, the glue kernel's exact formula), rounded to
// bf16 and written out for K1's quantize pass, and in the same pass the
// absmax of (h H) for the down projection's per-tensor scale (phase A with
// B = 256): one read of g and u replaces the glue kernel's and phase A's.
__global__ void __launch_bounds__(128) k_swiglu_absmax(const __grid_constant__ CUtensorMap tmg,
                                                       const __grid_constant__ CUtensorMap tmu, int64_t n, float norm,
                                                       __nv_bfloat16* __restrict__ h, unsigned* absmax, unsigned* err) {
    using C = V4Cfg<__nv_bfloat16>;
    constexpr int SB = 2 * C::STAGE_BYTES;  // g chunk + u chunk
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int k = l >> 3, p = l & 7;
    uint8_t* stages = smem + w * C::STAGES * SB;
    float4* xch = reinterpret_cast<float4*>(smem + C::WARPS * C::STAGES * SB + w * C::XCH_BYTES);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::WARPS * (C::STAGES * SB + C::XCH_BYTES)) + w * C::STAGES;
    const int64_t nchunks = n >> 10;
    const int64_t G = (int64_t)gridDim.x * C::WARPS;
    const int64_t c0 = (int64_t)blockIdx.x * C::WARPS + w;
    if (l == 0) {
        if (w == 0) {
            tma_prefetch_desc(&tmg);
            tma_prefetch_desc(&tmu);
        }
        for (int s = 0; s < C::STAGES; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    pdl_wait();
    pdl_trigger();
    auto issue = [&](int s, int64_t c) {
        mbar_expect_tx(&bars[s], SB);
        tma_load_2d(stages + s * SB, &tmg, &bars[s], 0, (int)(c * C::CHUNK_ROWS));
        tma_load_2d(stages + s * SB + C::STAGE_BYTES, &tmu, &bars[s], 0, (int)(c * C::CHUNK_ROWS));
    };
    if (l == 0)
        for (int s = 0; s < C::STAGES; ++s)
            if (c0 + s * G < nchunks) issue(s, c0 + s * G);
    __syncwarp();
    RowsCore<8, 0, V3_ABSMAX, false, float> core;
    core.init(absmax, nullptr, norm, err, nullptr);
    int i = 0;
    for (int64_t c = c0; c < nchunks; c += G, ++i) {
        const int s = i % C::STAGES;
        mbar_wait(&bars[s], (uint32_t)(i / C::STAGES) & 1u);
        float2 vg[16], vu[16];
        v4_read<__nv_bfloat16>(stages + s * SB, k, p, vg);
        v4_read<__nv_bfloat16>(stages + s * SB + C::STAGE_BYTES, k, p, vu);
        // h in bf16 (what the unfused path quantizes), stored and transformed
        uint32_t hw[16];
        float2 v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            hw[j] = pack_bf16x2(swiglu_fwd1(vg[j].x, vu[j].x), swiglu_fwd1(vg[j].y, vu[j].y));
            v[j] = make_float2(__uint_as_float(hw[j] << 16), __uint_as_float(hw[j] & 0xFFFF0000u));
        }
        // every loaded value is consumed above: the stage's reads are done
        __syncwarp();
        if (l == 0 && c + C::STAGES * G < nchunks) issue(s, c + C::STAGES * G);
        uint4* dst = reinterpret_cast<uint4*>(h + (c << 10) + k * 256 + p * 32);
#pragma unroll
        for (int j = 0; j < 4; ++j) dst[j] = make_uint4(hw[4 * j], hw[4 * j + 1], hw[4 * j + 2], hw[4 * j + 3]);
        core.phase1(v);
        core.finish(v, c << 10, n, k, p, xch, nullptr, (float*)nullptr);
    }
    core.reduce(absmax, err);
}

// h = swiglu(g, u) (bf16, n elements) and the rotated absmax of h (B = 256)
bool swiglu_absmax(const void* g, const void* u, void* h, int64_t n, int64_t cols, unsigned* amax, unsigned* err,
                   cudaStream_t st) {
    using C = V4Cfg<__nv_bfloat16>;
    if (n % 1024 || cols % 256 || (uintptr_t)g % 16 || (uintptr_t)u % 16 || (uintptr_t)h % 16) return false;
    CUtensorMap tg, tu;
    if (!encode_2d_sw128(&tg, 1, g, C::ROW_ELEMS, n / C::ROW_ELEMS, C::CHUNK_ROWS) ||
        !encode_2d_sw128(&tu, 1, u, C::ROW_ELEMS, n / C::ROW_ELEMS, C::CHUNK_ROWS))
        return false;
    const size_t smem = 1024 + (size_t)C::WARPS * (C::STAGES * 2 * C::STAGE_BYTES + C::XCH_BYTES) + C::WARPS * C::STAGES * 8;
    static int per_sm = 0;
    if (!per_sm) {
        cudaFuncSetAttribute(k_swiglu_absmax, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_swiglu_absmax, 32 * C::WARPS, smem);
        if (per_sm < 1) per_sm = 1;
    }
    int64_t want = (n / 1024 + C::WARPS - 1) / C::WARPS;
    const int64_t cap = (int64_t)num_sms() * per_sm;
    if (want > cap) want = cap;
    launch_pdl(k_swiglu_absmax, dim3((unsigned)(want < 1 ? 1 : want)), dim3(32 * C::WARPS), smem, st, tg, tu, n,
               hadamard_norm(256), static_cast<__nv_bfloat16*>(h), amax, err);
    return true;
}

// ============================================================ launcher

namespace {

template <typename K>
unsigned v3_grid(K kern, int64_t n) {
    static int per_sm = 0;
    if (!per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
        if (per_sm < 1) per_sm = 1;
    }
    int64_t want = ((n + 1023) / 1024 + 7) / 8;
    const int64_t cap = (int64_t)num_sms() * per_sm;
    if (want > cap) want = cap;
    if (want < 1) want = 1;
    return (unsigned)want;
}

}  // namespace

// HALO_K1_WIDE=0: B = 512 / 1024 through the generic large-block kernel (A/B)
bool wide_enabled() {
    static const bool on = [] {
        const char* e = getenv("HALO_K1_WIDE");
        return !(e && e[0] == '0');
    }();
    return on;
}

int k1_version() {
    static const int ver = [] {
        const char* e = getenv("HALO_K1_VERSION");
        return e ? atoi(e) : 4;
    }();
    return ver;
}

namespace {

template <int LB, typename InT, int FMT, int MODE, bool SUP, typename OutT>
void launch_v3(const InT* in, int64_t n, unsigned* amax, const float* sup, uint8_t* codes, OutT* out, unsigned* err,
               float* sout, cudaStream_t st, int64_t cols = 256) {
    const float norm = hadamard_norm(int64_t(1) << LB);
    using C = V4Cfg<InT>;
    if (k1_version() >= 4 && n % C::ROW_ELEMS == 0 && (uintptr_t)in % 16 == 0) {
        CUtensorMap tm;
        if (encode_2d_sw128(&tm, sizeof(InT) == 4 ? 0 : 1, in, C::ROW_ELEMS, n / C::ROW_ELEMS, C::CHUNK_ROWS)) {
            auto kern = k_rows_v4<LB, InT, FMT, MODE, SUP, OutT>;
            static int per_sm = 0;
            if (!per_sm) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * C::WARPS, C::SMEM);
                if (per_sm < 1) per_sm = 1;
            }
            int64_t want = ((n + 1023) / 1024 + C::WARPS - 1) / C::WARPS;
            const int64_t cap = (int64_t)num_sms() * per_sm;
            if (want > cap) want = cap;
            launch_pdl(kern, dim3((unsigned)(want < 1 ? 1 : want)), dim3(32 * C::WARPS), C::SMEM, st, tm, n, cols, norm,
                       amax, sup, codes, out, err, sout);
            return;
        }
    }
    auto kern = k_rows_v3<LB, InT, FMT, MODE, SUP, OutT>;
    kern<<<v3_grid(kern, n), 256, 0, st>>>(in, n, cols, norm, amax, sup, codes, out, err, sout);
}

template <int LB>
void dispatch_v3(int mode, int fmt, int in_dtype, const void* in, int64_t n, unsigned* amax, const float* sup,
                 uint8_t* codes, void* out, int out_dtype, unsigned* err, float* sout, cudaStream_t st) {
    using bf = __nv_bfloat16;
    if (mode == V3_XFORM) {
        const float* p = static_cast<const float*>(in);
        if (out_dtype == DT_BF16) launch_v3<LB, float, 0, V3_XFORM, false, bf>(p, n, amax, sup, codes, static_cast<bf*>(out), err, sout, st);
        else launch_v3<LB, float, 0, V3_XFORM, false, float>(p, n, amax, sup, codes, static_cast<float*>(out), err, sout, st);
        return;
    }
#define HALO_V3(T)                                                                                                       \
    {                                                                                                                    \
        auto p = static_cast<const T*>(in);                                                                              \
        if (mode == V3_ABSMAX) launch_v3<LB, T, 0, V3_ABSMAX, false, float>(p, n, amax, sup, codes, nullptr, err, sout, st); \
        else if (fmt == FMT_INT8) {                                                                                      \
            if (sup) launch_v3<LB, T, FMT_INT8, V3_QUANT, true, float>(p, n, amax, sup, codes, nullptr, err, sout, st);  \
            else launch_v3<LB, T, FMT_INT8, V3_QUANT, false, float>(p, n, amax, sup, codes, nullptr, err, sout, st);     \
        } else if (fmt == FMT_E3M2) {                                                                                    \
            if (sup) launch_v3<LB, T, FMT_E3M2, V3_QUANT, true, float>(p, n, amax, sup, codes, nullptr, err, sout, st);  \
            else launch_v3<LB, T, FMT_E3M2, V3_QUANT, false, float>(p, n, amax, sup, codes, nullptr, err, sout, st);     \
        } else {                                                                                                         \
            if (sup) launch_v3<LB, T, FMT_E4M3, V3_QUANT, true, float>(p, n, amax, sup, codes, nullptr, err, sout, st);  \
            else launch_v3<LB, T, FMT_E4M3, V3_QUANT, false, float>(p, n, amax, sup, codes, nullptr, err, sout, st);     \
        }                                                                                                                \
    }
    if (in_dtype == DT_BF16) HALO_V3(bf) else HALO_V3(float)
#undef HALO_V3
}

}  // namespace

namespace {

template <int LB>
void dispatch_rows_v3(int mode, int fmt, int in_dtype, const void* in, int64_t n, int64_t cols, unsigned* amax_rows,
                      const float* row_scales, uint8_t* codes, unsigned* err, cudaStream_t st) {
#define HALO_VR(T)                                                                                                 \
    {                                                                                                              \
        auto p = static_cast<const T*>(in);                                                                        \
        if (mode == 0) launch_v3<LB, T, 0, V3_ABSMAX_ROWS, false, float>(p, n, amax_rows, nullptr, nullptr, nullptr, err, nullptr, st, cols); \
        else if (fmt == FMT_INT8) launch_v3<LB, T, FMT_INT8, V3_QUANT_ROWS, false, float>(p, n, nullptr, row_scales, codes, nullptr, err, nullptr, st, cols); \
        else launch_v3<LB, T, FMT_E4M3, V3_QUANT_ROWS, false, float>(p, n, nullptr, row_scales, codes, nullptr, err, nullptr, st, cols); \
    }
    if (in_dtype == DT_BF16) HALO_VR(__nv_bfloat16) else HALO_VR(float)
#undef HALO_VR
}

__global__ void k_row_scales(const unsigned* amax, int64_t rows, int fmt, float* scales, unsigned* err) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= rows) return;
    const unsigned w = amax[r];
    if (w >= 0x7f800000u) atomicOr(err, ERRF_NONFINITE);
    scales[r] = scale_from_absmax(__uint_as_float(w), fmt);  // compute_scales, quantize.hpp:202-239
}

}  // namespace

// Granularity::row (one scale per row, quantize.hpp:73-132): phase A
// per-row rotated absmax words, per-row scales, phase B quantize with the
// row's scale.  cols a multiple of 256; B = 2^lb <= 256.
bool rows_v3_per_row(int fmt, int in_dtype, const void* in, int64_t rows, int64_t cols, int64_t B,
                     unsigned* amax_rows, float* row_scales, uint8_t* codes, unsigned* err, cudaStream_t st) {
    if (cols % 256 || B < 1 || B > 256 || (B & (B - 1))) return false;
    if ((uintptr_t)in % 32 || (uintptr_t)codes % 32) return false;
    const int64_t n = rows * cols;
    int lb = 0;
    while ((int64_t(1) << lb) < B) ++lb;
    cudaMemsetAsync(amax_rows, 0, rows * sizeof(unsigned), st);
    for (int mode = 0; mode < 2; ++mode) {
        if (mode == 1) k_row_scales<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(amax_rows, rows, fmt, row_scales, err);
        switch (lb) {
        case 0: dispatch_rows_v3<0>(mode, fmt, in_dtype, in, n, cols, amax_rows, row_scales, codes, err, st); break;
        case 1: dispatch_rows_v3<1>(mode, fmt, in_dtype, in, n, cols, amax_rows, row_scales, codes, err, st); break;
        case 2: dispatch_rows_v3<2>(mode, fmt, in_dtype, in, n, cols, amax_rows, row_scales, codes, err, st); break;
        case 3: dispatch_rows_v3<3>(mode, fmt, in_dtype, in, n, cols, amax_rows, row_scales, codes, err, st); break;
        case 4: dispatch_rows_v3<4>(mode, fmt, in_dtype, in, n, cols, amax_rows, row_scales, codes, err, st); break;
        case 5: dispatch_rows_v3<5>(mode, fmt, in_dtype, in, n, cols, amax_rows, row_scales, codes, err, st); break;
        case 6: dispatch_rows_v3<6>(mode, fmt, in_dtype, in, n, cols, amax_rows, row_scales, codes, err, st); break;
        case 7: dispatch_rows_v3<7>(mode, fmt, in_dtype, in, n, cols, amax_rows, row_scales, codes, err, st); break;
        default: dispatch_rows_v3<8>(mode, fmt, in_dtype, in, n, cols, amax_rows, row_scales, codes, err, st); break;
        }
    }
    return true;
}


// ------------------------------------------------------- large-block launcher
namespace {
template <int LB, typename InT, int FMT, int MODE, bool SUP, typename OutT>
void launch_lb(const InT* in, int64_t n, unsigned* amax, const float* sup, uint8_t* codes, OutT* out, unsigned* err,
               float* sout, cudaStream_t st) {
    auto kern = k_rows_lb<LB, InT, FMT, MODE, SUP, OutT>;
    static int per_sm = 0;
    if (!per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
        if (per_sm < 1) per_sm = 1;
    }
    int64_t grid = n / BG2_TILE;
    const int64_t cap = (int64_t)num_sms() * per_sm;
    if (grid > cap) grid = cap;
    kern<<<(unsigned)(grid < 1 ? 1 : grid), 256, 0, st>>>(in, n, hadamard_norm(int64_t(1) << LB), amax, sup, codes, out,
                                                          err, sout);
}

template <int LB>
void dispatch_lb(int mode, int fmt, int in_dtype, const void* in, int64_t n, unsigned* amax, const float* sup,
                 uint8_t* codes, void* out, int out_dtype, unsigned* err, float* sout, cudaStream_t st) {
    using bf = __nv_bfloat16;
    if (mode == V3_XFORM) {
        const float* p = static_cast<const float*>(in);
        if (out_dtype == DT_BF16) launch_lb<LB, float, 0, V3_XFORM, false, bf>(p, n, amax, sup, codes, static_cast<bf*>(out), err, sout, st);
        else launch_lb<LB, float, 0, V3_XFORM, false, float>(p, n, amax, sup, codes, static_cast<float*>(out), err, sout, st);
        return;
    }
#define HALO_LB(T)                                                                                                        \
    {                                                                                                                     \
        auto p = static_cast<const T*>(in);                                                                               \
        if (mode == V3_ABSMAX) launch_lb<LB, T, 0, V3_ABSMAX, false, float>(p, n, amax, sup, codes, nullptr, err, sout, st); \
        else if (fmt == FMT_INT8) {                                                                                       \
            if (sup) launch_lb<LB, T, FMT_INT8, V3_QUANT, true, float>(p, n, amax, sup, codes, nullptr, err, sout, st);   \
            else launch_lb<LB, T, FMT_INT8, V3_QUANT, false, float>(p, n, amax, sup, codes, nullptr, err, sout, st);      \
        } else if (fmt == FMT_E3M2) {                                                                                     \
            if (sup) launch_lb<LB, T, FMT_E3M2, V3_QUANT, true, float>(p, n, amax, sup, codes, nullptr, err, sout, st);   \
            else launch_lb<LB, T, FMT_E3M2, V3_QUANT, false, float>(p, n, amax, sup, codes, nullptr, err, sout, st);      \
        } else {                                                                                                          \
            if (sup) launch_lb<LB, T, FMT_E4M3, V3_QUANT, true, float>(p, n, amax, sup, codes, nullptr, err, sout, st);   \
            else launch_lb<LB, T, FMT_E4M3, V3_QUANT, false, float>(p, n, amax, sup, codes, nullptr, err, sout, st);      \
        }                                                                                                                 \
    }
    if (in_dtype == DT_BF16) HALO_LB(bf) else HALO_LB(float)
#undef HALO_LB
}
}  // namespace

// B = 2^lb, 9 <= lb <= 13, n a multiple of 8192, 32 B aligned operands.
// HALO_K1_LB=0 keeps the older radix-16 kernel (fwht_big.cu) for A/B runs.
bool rows_lb(int mode, int fmt, int in_dtype, const void* in, int64_t n, int64_t B, unsigned* amax, const float* sup,
             uint8_t* codes, void* out, int out_dtype, unsigned* err, float* sout, cudaStream_t st) {
    static const bool on = [] {
        const char* e = getenv("HALO_K1_LB");
        return !(e && e[0] == '0');
    }();
    if (!on || B < 512 || B > 8192 || (B & (B - 1)) || n % BG2_TILE) return false;
    if (mode == V3_XFORM && in_dtype != DT_F32) return false;
    if ((uintptr_t)in % 32 || (uintptr_t)codes % 16 || (uintptr_t)out % 16) return false;
    int lb = 0;
    while ((int64_t(1) << lb) < B) ++lb;
    switch (lb) {
    case 9: dispatch_lb<9>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    case 10: dispatch_lb<10>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    case 11: dispatch_lb<11>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    case 12: dispatch_lb<12>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    default: dispatch_lb<13>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    }
    return true;
}

// B = 2^lb with lb in [0, 10]; n a multiple of 16 (and of B).  B = 512 / 1024
// (RowsCore::finish_wide) only for whole 1024-element chunks.
// K4 (transform-only, fp32 in, bf16 out) with a bf16 addend fused into the
// store: out = RN_bf16(add + RN_bf16(H-rotated in)).  Only the exchange path
// of the row kernels (B = 64 .. 256) implements it; false = not handled.
bool rows_xform_add(const float* in, int64_t n, int64_t B, const void* add, void* out, cudaStream_t st) {
    if (B != 64 && B != 128 && B != 256) return false;
    if (n % 16 || (uintptr_t)in % 32 || (uintptr_t)add % 32 || (uintptr_t)out % 16) return false;
    return rows_v3(V3_XFORM, 0, DT_F32, in, n, B, nullptr, nullptr,
                   const_cast<uint8_t*>(static_cast<const uint8_t*>(add)), out, DT_BF16, nullptr, nullptr, st);
}

bool rows_v3(int mode, int fmt, int in_dtype, const void* in, int64_t n, int64_t B, unsigned* amax, const float* sup,
             uint8_t* codes, void* out, int out_dtype, unsigned* err, float* sout, cudaStream_t st) {
    if (n % 16 || B < 1 || B > 1024 || (B & (B - 1))) return false;
    if (B > 256 && (n % 1024 || !wide_enabled())) return false;
    if (mode == V3_XFORM && in_dtype != DT_F32) return false;
    int lb = 0;
    while ((int64_t(1) << lb) < B) ++lb;
    switch (lb) {
    case 0: dispatch_v3<0>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    case 1: dispatch_v3<1>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    case 2: dispatch_v3<2>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    case 3: dispatch_v3<3>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    case 4: dispatch_v3<4>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    case 5: dispatch_v3<5>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    case 6: dispatch_v3<6>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    case 7: dispatch_v3<7>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    case 8: dispatch_v3<8>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    case 9: dispatch_v3<9>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    default: dispatch_v3<10>(mode, fmt, in_dtype, in, n, amax, sup, codes, out, out_dtype, err, sout, st); break;
    }
    return true;
}

}  // namespace halo_b200
