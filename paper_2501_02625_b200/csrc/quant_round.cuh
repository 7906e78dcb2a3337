// quant_round.cuh — bit-exact RTN quantizers for the fused kernels.
//
// The reference computes every code as round_code(double(x) / double(s))
// (quantize.hpp:275) with nearbyint (ties to even) in double precision.  A
// double division per element would cap the fused kernels far below HBM
// speed, so the device path works in fp32 and then *proves* the result:
//
//   1. candidate q0 = RNE(x * (1/s)) in fp32 — within one grid step of the
//      true RNE(x/s) because the fp32 quotient is off by < 2^-22 relative;
//   2. the sign of  x - mid * s  for the midpoints between q0 and its grid
//      neighbours is computed with ONE rounding by fmaf (mid * s is exact in
//      the fma), so it is the sign of the exact real residual;
//   3. the candidate moves one step if the true quotient lies beyond a
//      midpoint, and an exact tie picks the even code (ties-to-even).
//
// The double path (x/s correctly rounded to double, then nearbyint) equals
// the exact real RNE(x/s) here: a non-tie quotient of two floats sits at
// least 2^-32 (relative) away from every half-integer / minifloat midpoint,
// far above the 2^-53 double rounding error.  So both paths compute the same
// function; tests/test_round_cpu.py checks this header against the oracle on
// 10^8 inputs including every midpoint.  Valid for scales s >= 2^-100 (the
// fma residual must not underflow; any realistic tensor).
//
// These functions are __host__ __device__ so the CPU test compiles exactly
// the code the kernels run.
#pragma once

#include <stdint.h>
#include <math.h>
#include <string.h>

#if defined(__CUDACC__)
#define HALO_HD __host__ __device__ __forceinline__
#else
#define HALO_HD inline
#endif

namespace halo_b200 {

HALO_HD uint32_t f2u(float f) {
#if defined(__CUDA_ARCH__)
    return __float_as_uint(f);
#else
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
#endif
}
HALO_HD float u2f(uint32_t u) {
#if defined(__CUDA_ARCH__)
    return __uint_as_float(u);
#else
    float f;
    memcpy(&f, &u, 4);
    return f;
#endif
}

// ---------------------------------------------------------------- INT8 ----
// quantize.hpp:154-161: nearbyint, clamp to +-127 (-128 never produced).
HALO_HD int8_t quant_int8(float x, float s, float inv_s) {
    const float q0 = rintf(x * inv_s);
    if (q0 >= 128.0f) return 127;   // true RNE >= 127 after a one-step fix
    if (q0 <= -128.0f) return -127;
    float q = q0;
    const float hi = fmaf(-(q0 + 0.5f), s, x);  // sign(x/s - (q0 + 1/2))
    const float lo = fmaf(-(q0 - 0.5f), s, x);  // sign(x/s - (q0 - 1/2))
    if (hi > 0.0f) {
        q = q0 + 1.0f;
    } else if (hi == 0.0f) {
        q = (((int)q0 & 1) == 0) ? q0 : q0 + 1.0f;  // tie -> even
    } else if (lo < 0.0f) {
        q = q0 - 1.0f;
    } else if (lo == 0.0f) {
        q = (((int)q0 & 1) == 0) ? q0 : q0 - 1.0f;
    }
    if (q > 127.0f) q = 127.0f;
    if (q < -127.0f) q = -127.0f;
    return (int8_t)(int)q;
}

// ---------------------------------------------------------------- E4M3 ----
// quantize.hpp:138-150, 162-163: round_minifloat(x, 3 mantissa bits,
// min_exp -6, saturate 448); zero is +0 (the "+ 0.0" at :149).
// Encoding: OCP E4M3 (bias 7, S.1111.111 is NaN and never produced).

HALO_HD int ilog2_pos(float v) {  // floor(log2(v)) for a finite v > 0
    int e;
    frexpf(v, &e);
    return e - 1;
}

// grid spacing of the binade holding v (v >= 0)
HALO_HD float e4m3_step(float v) {
    int e = (v > 0.0f) ? ilog2_pos(v) : -6;
    if (e < -6) e = -6;
    return ldexpf(1.0f, e - 3);
}

// encode a non-negative grid value (<= 448) as the 7 magnitude bits
HALO_HD uint8_t e4m3_bits_pos(float v) {
    if (v == 0.0f) return 0;
    int e = ilog2_pos(v);
    if (e < -6) return (uint8_t)(int)(v * 512.0f);  // subnormal: m * 2^-9
    const int mant = (int)((ldexpf(v, -e) - 1.0f) * 8.0f);
    return (uint8_t)(((e + 7) << 3) | mant);
}

HALO_HD uint8_t quant_e4m3(float x, float s, float inv_s) {
    const float a = fabsf(x);
    const float y = a * inv_s;                 // approximate quotient
    float q0;
    if (y >= 464.0f) {
        q0 = 480.0f;                            // beyond saturation; fixed below
    } else {
        const float st = e4m3_step(y);
        q0 = rintf(y / st) * st;               // exact: st is a power of two
    }
    float q = q0;
    // upward: midpoint between q0 and the next grid value
    const float up = e4m3_step(q0);
    const float mid_up = q0 + 0.5f * up;
    const float r_up = fmaf(-mid_up, s, a);
    if (r_up > 0.0f) {
        q = q0 + up;
    } else if (r_up == 0.0f) {
        // tie: the grid neighbour with the even code wins
        q = (e4m3_bits_pos(q0 > 448.0f ? 448.0f : q0) & 1) ? q0 + up : q0;
    } else if (q0 > 0.0f) {
        // downward: spacing below q0 halves when q0 opens a binade
        float dn = up;
        if (q0 <= 448.0f && ldexpf(1.0f, ilog2_pos(q0)) == q0 && ilog2_pos(q0) > -6) dn = 0.5f * up;
        const float mid_dn = q0 - 0.5f * dn;
        const float r_dn = fmaf(-mid_dn, s, a);
        if (r_dn < 0.0f) {
            q = q0 - dn;
        } else if (r_dn == 0.0f) {
            const float lowv = q0 - dn;
            q = (e4m3_bits_pos(lowv) & 1) ? q0 : lowv;
        }
    }
    if (q > 448.0f) q = 448.0f;
    const uint8_t mag = e4m3_bits_pos(q);
    return (mag != 0 && x < 0.0f) ? (uint8_t)(mag | 0x80) : mag;
}

// ---------------------------------------------------------- FP6 E3M2 ----
// quantize.hpp:138-150, 164-166: round_minifloat(x, 2 mantissa bits, min_exp
// -2, saturate 28); zero is +0.  Code: OCP E3M2 (bias 3, no inf/NaN),
// S.EEE.MM in the low 6 bits.  Device tensors hold the code shifted left by
// two (bits 7:2 of the byte), the layout tcgen05 kind::f8f6f4 reads FP6
// operands in (measured: tools/fp6_probe.py).
HALO_HD float e3m2_step(float v) {
    int e = (v > 0.0f) ? ilog2_pos(v) : -2;
    if (e < -2) e = -2;
    return ldexpf(1.0f, e - 2);
}
HALO_HD uint8_t e3m2_bits_pos(float v) {  // grid value (<= 28) -> 5 magnitude bits
    if (v == 0.0f) return 0;
    const int e = ilog2_pos(v);
    if (e < -2) return (uint8_t)(int)(v * 16.0f);  // subnormal: m * 2^-4
    const int mant = (int)((ldexpf(v, -e) - 1.0f) * 4.0f);
    return (uint8_t)(((e + 3) << 2) | mant);
}
// 6-bit code of round_code(x / s, Fp6E3M2) (low-aligned)
HALO_HD uint8_t quant_e3m2(float x, float s, float inv_s) {
    const float a = fabsf(x);
    const float y = a * inv_s;
    float q0;
    if (y >= 31.0f) {
        q0 = 32.0f;  // beyond saturation; fixed below
    } else {
        const float st = e3m2_step(y);
        q0 = rintf(y / st) * st;
    }
    float q = q0;
    const float up = e3m2_step(q0);
    const float mid_up = q0 + 0.5f * up;
    const float r_up = fmaf(-mid_up, s, a);
    if (r_up > 0.0f) {
        q = q0 + up;
    } else if (r_up == 0.0f) {
        q = (e3m2_bits_pos(q0 > 28.0f ? 28.0f : q0) & 1) ? q0 + up : q0;
    } else if (q0 > 0.0f) {
        float dn = up;
        if (q0 <= 28.0f && ldexpf(1.0f, ilog2_pos(q0)) == q0 && ilog2_pos(q0) > -2) dn = 0.5f * up;
        const float mid_dn = q0 - 0.5f * dn;
        const float r_dn = fmaf(-mid_dn, s, a);
        if (r_dn < 0.0f) {
            q = q0 - dn;
        } else if (r_dn == 0.0f) {
            const float lowv = q0 - dn;
            q = (e3m2_bits_pos(lowv) & 1) ? q0 : lowv;
        }
    }
    if (q > 28.0f) q = 28.0f;
    const uint8_t mag = e3m2_bits_pos(q);
    return (mag != 0 && x < 0.0f) ? (uint8_t)(mag | 0x20) : mag;
}
HALO_HD float e3m2_to_float(uint8_t c) {  // low-aligned code
    const int e = (c >> 2) & 7, m = c & 3;
    const float v = e == 0 ? (float)m * 0.0625f : (1.0f + (float)m * 0.25f) * ldexpf(1.0f, e - 3);
    return (c & 0x20) ? -v : v;
}

// ------------------------------------------------------------ fast paths --
// Same functions, cheaper common case: when y = x * inv sits closer than
// kFastMargin (below) to the rounded grid value, the true quotient is
// strictly nearer to that grid value than to any other, so the candidate is
// the exact RNE result.  Near a midpoint the exact fma-checked path above
// decides.  Rounding to an integer uses the
// 1.5 * 2^23 trick: y + 12582912 rounds y to nearest-even in fp32.
constexpr float kRoundMagic = 12582912.0f;

// Fast-path acceptance margin, in grid steps.  The candidate q is certified
// when |y - q| < kFastMargin.  Error budget of y against the true quotient
// Q = x/s (|Q| <= 127.5 for INT8, the scaled E4M3 mantissa z < 16): inv =
// RN(1/s) contributes |Q| * 2^-24 <= 7.6e-6, the rounding of y = RN(x*inv)
// (absent when ptxas contracts it into an FFMA) another 7.6e-6 and the
// residual y - q 2^-25; 0.5 - 0.49998 = 2e-5 covers the sum, so |Q - q| < 0.5
// and q = RNE(Q).  Inputs within 2e-5 steps of a midpoint (4e-5 of them)
// take the exact fma-checked path.
constexpr float kFastMargin = 0.49998f;

HALO_HD int8_t quant_int8_fast(float x, float s, float inv_s) {
    const float y = x * inv_s;
    const float t = y + kRoundMagic;
    const float q = t - kRoundMagic;
    if (fabsf(y - q) < kFastMargin && fabsf(q) <= 127.0f) return (int8_t)(int)q;
    return quant_int8(x, s, inv_s);
}

HALO_HD uint8_t quant_e4m3_fast(float x, float s, float inv_s) {
    const float a = fabsf(x);
    const float y = a * inv_s;
    uint8_t code;
    if (y >= 448.0f) {
        code = 0x7E;  // every quotient >= 448*(1-2^-22) rounds (or saturates) to 448
    } else {
        // binade of y (normal fp32 here), clamped to the E4M3 minimum -6
        int e = (y >= 0.015625f) ? (int)((f2u(y) >> 23) & 0xFF) - 127 : -6;
        const float z = y * u2f((uint32_t)(127 + 3 - e) << 23);  // exact: y / step, in [0, 16)
        const float t = z + kRoundMagic;
        const float qz = t - kRoundMagic;
        if (!(fabsf(z - qz) < kFastMargin)) return quant_e4m3(x, s, inv_s);
        code = (uint8_t)(((e + 7) << 3) + (int)qz - 8);  // also right when qz == 16 (next binade)
    }
    return (code != 0 && x < 0.0f) ? (uint8_t)(code | 0x80) : code;
}

// Branch-free candidates for the vectorised kernels: return the fast-path
// code and flag inputs that need the exact path.  Kernels collect the flags
// into a mask and take the (rare, warp-uniform) exact loop only when a flag
// is set, which keeps the hot loop free of per-element branches.
HALO_HD uint8_t quant_int8_try(float x, float inv_s, uint32_t& slow) {
    const float y = x * inv_s;
    const float t = y + kRoundMagic;
    const float q = t - kRoundMagic;
    slow = (uint32_t)!(fabsf(y - q) < kFastMargin && fabsf(q) <= 127.0f);
    return (uint8_t)(f2u(t) & 0xFFu);  // two's complement low byte of the integer q
}

HALO_HD uint8_t quant_e4m3_try(float x, float inv_s, uint32_t& slow) {
    const float a = fabsf(x);
    const float y = a * inv_s;
    const bool sat = y >= 448.0f;
    const int e = (y >= 0.015625f) ? (int)((f2u(y) >> 23) & 0xFF) - 127 : -6;
    const float z = sat ? 0.0f : y * u2f((uint32_t)(127 + 3 - e) << 23);
    const float t = z + kRoundMagic;
    const float qz = t - kRoundMagic;
    slow = (uint32_t)(!sat && !(fabsf(z - qz) < kFastMargin));
    const uint32_t code = sat ? 0x7Eu : (uint32_t)(((e + 7) << 3) + (int)qz - 8);
    return (uint8_t)((code != 0 && x < 0.0f) ? (code | 0x80u) : code);
}

// Residual-certified INT8 candidate (the vectorised kernels' fast path).
// q is any integer near x/s (here RNE of x*inv, however y was rounded); the
// residual r = fma(-q, s, x) is x - q*s rounded once, so |r| < h with
// h = half_margin(s) = RN(0.5 * s * (1 - 2^-22)) proves |x - q*s| < s/2,
// i.e. q = RNE(x/s) with no tie.  Only inputs within ~2^-22 of a midpoint
// (plus |q| > 127, which needs the clamp) fall to the exact path: ~100x
// fewer than the |y - q| < kFastMargin test above.
HALO_HD float half_margin(float s) { return (0.5f * s) * (1.0f - 2.384185791015625e-07f); }

HALO_HD uint8_t quant_int8_try_r(float x, float s, float inv_s, float h, uint32_t& slow) {
    const float t = x * inv_s + kRoundMagic;
    const float q = t - kRoundMagic;
    const float r = fmaf(-q, s, x);
    slow = (uint32_t)!(fabsf(r) < h && fabsf(q) <= 127.0f);
    return (uint8_t)(f2u(t) & 0xFFu);
}

#if defined(__CUDACC__)
// Fast E4M3 for 4 values (device only).  The hardware F2FP
// (cvt.rn.satfinite.e4m3x2.f32) rounds to nearest-even with saturation at
// 448, exactly the reference's round_minifloat (quantize.hpp:138-150,
// 162-163) applied to its argument.  It is applied to x*inv_lo and x*inv_hi,
// where inv_lo/hi = RN(RN(1/s) * (1 -+ 2^-21)) bracket 1/s tightly enough
// that x*inv_lo <= x/s <= x*inv_hi (relative slack 2^-21 against <= 2^-22
// of rounding), so equal codes prove the code of the exact quotient by
// monotonicity -- subnormal and saturating ranges included; where they
// differ, one fma decides (e4m3x4_fast below).  The hardware
// encodes a negative value that rounds to zero as 0x80; the reference adds
// +0.0 (quantize.hpp:149), so such bytes become 0x00.
__device__ __forceinline__ uint32_t e4m3_word(float2 a, float2 c) {
    uint32_t w;
    asm("{\n\t.reg .b16 lo, hi;\n\t"
        "cvt.rn.satfinite.e4m3x2.f32 lo, %2, %1;\n\t"
        "cvt.rn.satfinite.e4m3x2.f32 hi, %4, %3;\n\t"
        "mov.b32 %0, {lo, hi};\n\t}"
        : "=r"(w)
        : "f"(a.x), "f"(a.y), "f"(c.x), "f"(c.y));
    return w;
}
// magnitude of an E4M3 code 0..0x7E
__device__ __forceinline__ float e4m3_mag(uint32_t b) {
    const uint32_t e = b >> 3, m = b & 7u;
    return e ? __uint_as_float(((e + 120u) << 23) | (m << 20)) : (float)m * 0.001953125f;
}
// Exact E4M3 codes of x[i]/s for 4 values (bit-exact with round_code):
// when the two bracketed conversions disagree on a byte, the codes are the
// two grid neighbours of the quotient and the sign of x - mid*s (one fma,
// exact sign) picks the side; an exact tie takes the even code.  `bad` is
// kept for the callers' slow-path plumbing and stays 0.
__device__ __forceinline__ uint32_t e4m3x4_fast(float2 a, float2 c, float2 inv_lo2, float2 inv_hi2, float s,
                                                uint32_t& bad) {
    const uint32_t wl = e4m3_word(__fmul2_rn(a, inv_lo2), __fmul2_rn(c, inv_lo2));
    const uint32_t wh = e4m3_word(__fmul2_rn(a, inv_hi2), __fmul2_rn(c, inv_hi2));
    uint32_t w = wl;
    const uint32_t diff = wl ^ wh;
    if (diff) {
        const float xs[4] = {a.x, a.y, c.x, c.y};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if ((diff >> (8 * i)) & 0xFFu) {
                const uint32_t bl = (wl >> (8 * i)) & 0x7Fu, bh = (wh >> (8 * i)) & 0x7Fu;  // adjacent magnitudes
                const float mid = 0.5f * (e4m3_mag(bl) + e4m3_mag(bh));
                const float r = fmaf(-mid, s, fabsf(xs[i]));
                const uint32_t pick = r > 0.f ? bh : (r < 0.f ? bl : ((bl & 1u) ? bh : bl));
                w = (w & ~(0x7Fu << (8 * i))) | (pick << (8 * i));
            }
        }
    }
    (void)bad;
    const uint32_t nz = ((w & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) & 0x80808080u;  // bytes with a nonzero magnitude
    return w & (nz | 0x7F7F7F7Fu);
}
// E3M2 counterpart of e4m3_word / e4m3x4_fast: the hardware F2FP
// (cvt.rn.satfinite.e3m2x2.f32, RNE, saturating at 28) on the bracketed
// quotients, one fma per disagreeing byte, +0 for zero magnitudes; returns
// the 4 codes shifted into bits 7:2 of their bytes (the MMA operand form).
__device__ __forceinline__ uint32_t e3m2_word(float2 a, float2 c) {
    uint32_t w;
    asm("{\n\t.reg .b16 lo, hi;\n\t"
        "cvt.rn.satfinite.e3m2x2.f32 lo, %2, %1;\n\t"
        "cvt.rn.satfinite.e3m2x2.f32 hi, %4, %3;\n\t"
        "mov.b32 %0, {lo, hi};\n\t}"
        : "=r"(w)
        : "f"(a.x), "f"(a.y), "f"(c.x), "f"(c.y));
    return w;
}
__device__ __forceinline__ float e3m2_mag(uint32_t b) {  // magnitude code 0..0x1F
    const uint32_t e = b >> 2, m = b & 3u;
    return e ? __uint_as_float(((e + 124u) << 23) | (m << 21)) : (float)m * 0.0625f;
}
__device__ __forceinline__ uint32_t e3m2x4_fast(float2 a, float2 c, float2 inv_lo2, float2 inv_hi2, float s) {
    const uint32_t wl = e3m2_word(__fmul2_rn(a, inv_lo2), __fmul2_rn(c, inv_lo2));
    const uint32_t wh = e3m2_word(__fmul2_rn(a, inv_hi2), __fmul2_rn(c, inv_hi2));
    uint32_t w = wl;
    const uint32_t diff = wl ^ wh;
    if (diff) {
        const float xs[4] = {a.x, a.y, c.x, c.y};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if ((diff >> (8 * i)) & 0xFFu) {
                const uint32_t bl = (wl >> (8 * i)) & 0x1Fu, bh = (wh >> (8 * i)) & 0x1Fu;
                const float mid = 0.5f * (e3m2_mag(bl) + e3m2_mag(bh));
                const float r = fmaf(-mid, s, fabsf(xs[i]));
                const uint32_t pick = r > 0.f ? bh : (r < 0.f ? bl : ((bl & 1u) ? bh : bl));
                w = (w & ~(0x1Fu << (8 * i))) | (pick << (8 * i));
            }
        }
    }
    const uint32_t nz = ((w & 0x1F1F1F1Fu) + 0x1F1F1F1Fu) & 0x20202020u;  // bytes with a nonzero magnitude
    return (w & (nz | 0x1F1F1F1Fu)) << 2;
}
__device__ __forceinline__ void e4m3_brackets(float inv, float2& lo2, float2& hi2) {
    const float lo = __fmul_rn(inv, 1.0f - 4.76837158203125e-07f), hi = __fmul_rn(inv, 1.0f + 4.76837158203125e-07f);
    lo2 = make_float2(lo, lo);
    hi2 = make_float2(hi, hi);
}
#endif

// decode for the dequantize / epilogue paths
HALO_HD float e4m3_to_float(uint8_t b) {
    const int e = (b >> 3) & 0xF, m = b & 7;
    const float v = e == 0 ? (float)m * ldexpf(1.0f, -9) : (1.0f + (float)m * 0.125f) * ldexpf(1.0f, e - 7);
    return (b & 0x80) ? -v : v;
}

// quantize.hpp:234 / hqfsdp.hpp:172-177: s = float(double(absmax)/fmax),
// 1.0 for an all-zero tensor.
HALO_HD float scale_from_absmax(float absmax, int fmt) {
    if (absmax == 0.0f) return 1.0f;
    const double fmax = fmt == 0 ? 127.0 : fmt == 1 ? 448.0 : 28.0;  // format_max, quantize.hpp:53-63
    return (float)((double)absmax / fmax);
}

}  // namespace halo_b200
