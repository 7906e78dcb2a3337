/*
 * halo_oracle.c — TEST INFRASTRUCTURE ONLY (see halo_oracle.h).
 *
 * Plain-C restatement of the reference HALO hot path.  Every function cites
 * the reference lines it restates (paths relative to /root/reference/proj/
 * include/halo/).  Build: oracle/Makefile (gcc -O2 -ffp-contract=off, no
 * fast-math: the butterflies and the quantizer divisions must be IEEE exact).
 */
#include "halo_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ---------------------------------------------------------------- dims -- */

/* hadamard.hpp:69-85 */
int orc_is_supported_hadamard_dim(int64_t d) {
    if (d < 1) return 0;
    int64_t odd = d;
    int twos = 0;
    while (odd % 2 == 0) { odd /= 2; ++twos; }
    if (odd == 1) return 1;
    if (odd == 3 && twos >= 2) return 1;
    if (odd == 5 && twos >= 2) return 1;
    return 0;
}

/* hadamard.hpp:87-93 */
int64_t orc_next_supported_hadamard_dim(int64_t d) {
    if (d < 1) d = 1;
    while (!orc_is_supported_hadamard_dim(d)) ++d;
    return d;
}

/* ----------------------------------------------------------- transforms -- */

/* hadamard.hpp:136-177, pow2 path (base_dim == 1): butterflies with stride
 * len = 1, 2, 4, ... (u+v, u-v in working precision, :140-153), then one
 * multiply by T(1/sqrt(double(d))) (:174-176).  Applied per B-segment. */
static void fwht_segment(float* row, int64_t B) {
    for (int64_t len = 1; len < B; len *= 2) {
        for (int64_t i = 0; i < B; i += 2 * len) {
            for (int64_t b = 0; b < len; ++b) {
                const float x = row[i + b];
                const float y = row[i + b + len];
                row[i + b] = x + y;
                row[i + b + len] = x - y;
            }
        }
    }
    const float norm = (float)(1.0 / sqrt((double)B));
    for (int64_t j = 0; j < B; ++j) row[j] *= norm;
}

/* Only power-of-two blocks are restated (the base-12/20 Kronecker factors of
 * hadamard.hpp:20-58 are outside this path); other sizes leave A untouched. */
static int pow2(int64_t b) { return b > 0 && (b & (b - 1)) == 0; }

void orc_fwht_rows(float* a, int64_t rows, int64_t cols, int64_t block) {
    if (!pow2(block) || cols % block) return;
    for (int64_t r = 0; r < rows; ++r)
        for (int64_t s = 0; s < cols; s += block)
            fwht_segment(a + r * cols + s, block);
}

/* hadamard.hpp:205-216: left = transpose(right(transpose(A))).  For a
 * power-of-two block the H^T / H variants coincide (base_dim 1). */
void orc_fwht_cols(float* a, int64_t rows, int64_t cols, int64_t block) {
    if (!pow2(block) || rows % block) return;
    float* col = (float*)malloc(sizeof(float) * (size_t)block);
    for (int64_t s = 0; s < rows; s += block) {
        for (int64_t c = 0; c < cols; ++c) {
            for (int64_t i = 0; i < block; ++i) col[i] = a[(s + i) * cols + c];
            fwht_segment(col, block);
            for (int64_t i = 0; i < block; ++i) a[(s + i) * cols + c] = col[i];
        }
    }
    free(col);
}

/* ------------------------------------------------------------- quantize -- */

/* quantize.hpp:53-63 */
static double format_max(int fmt) {
    switch (fmt) {
    case ORC_INT8: return 127.0;
    case ORC_FP8_E4M3: return 448.0;
    case ORC_FP6_E3M2: return 28.0;
    case ORC_MXFP6_E3M2: return 28.0;
    }
    return 0.0;
}

/* quantize.hpp:138-150 */
static double round_minifloat(double x, int mant_bits, int min_exp, double max_val) {
    if (x == 0.0) return 0.0;
    const double a = fabs(x);
    int e = ilogb(a);
    if (e < min_exp) e = min_exp;
    const double step = ldexp(1.0, e - mant_bits);
    double q = nearbyint(a / step) * step;
    if (q > max_val) q = max_val;
    return copysign(q, x) + 0.0;
}

/* quantize.hpp:152-180 */
double orc_round_code(double x, int fmt) {
    switch (fmt) {
    case ORC_INT8: {
        double q = nearbyint(x);
        if (q > 127.0) q = 127.0;
        if (q < -127.0) q = -127.0;
        return q + 0.0;
    }
    case ORC_FP8_E4M3: return round_minifloat(x, 3, -6, 448.0);
    case ORC_FP6_E3M2:
    case ORC_MXFP6_E3M2: return round_minifloat(x, 2, -2, 28.0);
    }
    return x;
}

/* quantize.hpp:219-237: the scale of one group from its absmax; MX formats
 * take the smallest power of two keeping absmax / s <= fmax (:224-232) */
static float group_scale(double m, int fmt) {
    if (m == 0.0) return 1.0f;
    if (fmt == ORC_MXFP6_E3M2) {
        const double fmax = format_max(fmt);
        int e = ilogb(m / fmax);
        if (m / ldexp(1.0, e) > fmax) ++e;
        if (e < -126) e = -126;
        return (float)ldexp(1.0, e);
    }
    return (float)(m / format_max(fmt));
}

/* quantize.hpp:202-239, per-tensor group */
float orc_tensor_scale(const float* a, int64_t n, int fmt, int* nonfinite) {
    double m = 0.0;
    int bad = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (!isfinite(a[i])) bad = 1;
        const double v = fabs((double)a[i]);
        if (v > m) m = v;
    }
    if (nonfinite) *nonfinite = bad;
    return group_scale(m, fmt);
}

/* quantize.hpp:244-280 (+ compute_scales :202-239 for row / column groups) */
/* group_count / group_of (quantize.hpp:110-132): tensor 0, row 1, column 2,
 * mx 4 (32 consecutive elements along each row) */
static int64_t mx_blocks(int64_t cols) { return (cols + 31) / 32; }
static int64_t group_count(int gran, int64_t rows, int64_t cols) {
    return gran == 0 ? 1 : gran == 1 ? rows : gran == 2 ? cols : rows * mx_blocks(cols);
}
static int64_t group_of(int gran, int64_t cols, int64_t i, int64_t j) {
    return gran == 0 ? 0 : gran == 1 ? i : gran == 2 ? j : i * mx_blocks(cols) + j / 32;
}

void orc_quantize(const float* a, int64_t rows, int64_t cols, int fmt, int gran,
                  int supplied, float* scales, float* codes) {
    if (!supplied) {
        const int64_t groups = group_count(gran, rows, cols);
        double* absmax = (double*)calloc((size_t)groups, sizeof(double));
        for (int64_t i = 0; i < rows; ++i)
            for (int64_t j = 0; j < cols; ++j) {
                const int64_t g = group_of(gran, cols, i, j);
                const double v = fabs((double)a[i * cols + j]);
                if (v > absmax[g]) absmax[g] = v;
            }
        for (int64_t g = 0; g < groups; ++g)
            scales[g] = group_scale(absmax[g], fmt);
        free(absmax);
    }
    for (int64_t i = 0; i < rows; ++i)
        for (int64_t j = 0; j < cols; ++j) {
            const int64_t g = group_of(gran, cols, i, j);
            const double s = scales[g];
            codes[i * cols + j] = (float)orc_round_code((double)a[i * cols + j] / s, fmt);
        }
}

void orc_codes_to_int8(const float* codes, int64_t n, int8_t* out) {
    for (int64_t i = 0; i < n; ++i) out[i] = (int8_t)codes[i];
}

/* OCP E4M3 (bias 7, no inf, S.1111.111 = NaN): encodes an exact grid value */
void orc_codes_to_e4m3(const float* codes, int64_t n, uint8_t* out) {
    for (int64_t i = 0; i < n; ++i) {
        const double v = codes[i];
        if (v == 0.0) { out[i] = 0; continue; }
        const uint8_t sign = v < 0 ? 0x80 : 0;
        const double a = fabs(v);
        int e = ilogb(a);
        uint8_t bits;
        if (e < -6) {
            bits = (uint8_t)(a / ldexp(1.0, -9));           /* subnormal: m * 2^-9 */
        } else {
            const int mant = (int)((a / ldexp(1.0, e) - 1.0) * 8.0);
            bits = (uint8_t)(((e + 7) << 3) | mant);
        }
        out[i] = sign | bits;
    }
}

float orc_e4m3_to_float(uint8_t b) {
    const int sign = b & 0x80;
    const int e = (b >> 3) & 0xF;
    const int m = b & 7;
    double v = e == 0 ? m * ldexp(1.0, -9) : (1.0 + m / 8.0) * ldexp(1.0, e - 7);
    return (float)(sign ? -v : v);
}

/* ------------------------------------------------------------- qmatmul -- */

/* quantize.hpp:350-375 */
void orc_qmatmul_i8(const int8_t* A, const int8_t* B, int64_t M, int64_t N, int64_t K,
                    int a_kmajor, int b_kmajor, float sa, float sb, int32_t* acc, float* out) {
    const double ss = (double)sa * (double)sb;
    int64_t* row = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
    for (int64_t i = 0; i < M; ++i) {
        memset(row, 0, sizeof(int64_t) * (size_t)N);
        for (int64_t k = 0; k < K; ++k) {
            const int64_t av = a_kmajor ? A[i * K + k] : A[k * M + i];
            if (av == 0) continue;
            if (b_kmajor) {
                for (int64_t j = 0; j < N; ++j) row[j] += av * B[j * K + k];
            } else {
                const int8_t* brow = B + k * N;
                for (int64_t j = 0; j < N; ++j) row[j] += av * brow[j];
            }
        }
        for (int64_t j = 0; j < N; ++j) {
            if (acc) acc[i * N + j] = (int32_t)row[j];
            if (out) out[i * N + j] = (float)((double)row[j] * ss);
        }
    }
    free(row);
}

/* quantize.hpp:377-379 -> dequantize :282-294 -> matmul(_nt) Accum::Double
 * tensor.hpp:126-160 */
void orc_qmatmul_deq(const float* A, const float* B, int64_t M, int64_t N, int64_t K,
                     int a_kmajor, int b_kmajor, float sa, float sb, float* out) {
    double* row = (double*)malloc(sizeof(double) * (size_t)N);
    for (int64_t i = 0; i < M; ++i) {
        memset(row, 0, sizeof(double) * (size_t)N);
        for (int64_t k = 0; k < K; ++k) {
            const float ca = a_kmajor ? A[i * K + k] : A[k * M + i];
            const double av = (double)(float)((double)ca * (double)sa);
            for (int64_t j = 0; j < N; ++j) {
                const float cb = b_kmajor ? B[j * K + k] : B[k * N + j];
                row[j] += av * (double)(float)((double)cb * (double)sb);
            }
        }
        for (int64_t j = 0; j < N; ++j) out[i * N + j] = (float)row[j];
    }
    free(row);
}

/* ---------------------------------------------------------------- layer -- */

static int64_t blk(const orc_scheme* s, int64_t d) { return s->block ? s->block : d; }

int64_t orc_padded_batch(const orc_scheme* s, int64_t b) {
    if (s->block) return (b + s->block - 1) / s->block * s->block;
    return orc_next_supported_hadamard_dim(b); /* halo_linear.hpp:395 */
}

static void to_i8(const float* c, int64_t n, int8_t* o) { orc_codes_to_int8(c, n, o); }

/* one quantized product in the reference's two numeric paths */
static void qmm(const orc_scheme* s, const float* A, const float* B, int64_t M, int64_t N,
                int64_t K, int a_kmajor, int b_kmajor, float sa, float sb, float* out) {
    if (s->fmt == ORC_INT8) {
        int8_t* ia = (int8_t*)malloc((size_t)(M * K));
        int8_t* ib = (int8_t*)malloc((size_t)(N * K));
        to_i8(A, M * K, ia);
        to_i8(B, N * K, ib);
        orc_qmatmul_i8(ia, ib, M, N, K, a_kmajor, b_kmajor, sa, sb, NULL, out);
        free(ia);
        free(ib);
    } else {
        orc_qmatmul_deq(A, B, M, N, K, a_kmajor, b_kmajor, sa, sb, out);
    }
}

/* halo_linear.hpp:267-303 (placement_F none or M) */
void orc_linear_forward(const orc_scheme* s, int64_t b, int64_t m, int64_t n,
                        const float* X, const float* W, float* Y,
                        float* xq, float* sx, float* wq, float* sw) {
    float* xt = (float*)malloc(sizeof(float) * (size_t)(b * m));
    float* wt = (float*)malloc(sizeof(float) * (size_t)(n * m));
    memcpy(xt, X, sizeof(float) * (size_t)(b * m));
    memcpy(wt, W, sizeof(float) * (size_t)(n * m));
    if (s->level >= 1) { /* placement_F == {M}: :292-296 */
        orc_fwht_rows(xt, b, m, blk(s, m));
        orc_fwht_rows(wt, n, m, blk(s, m));
    }
    orc_quantize(xt, b, m, s->fmt, 0, 0, sx, xq);
    orc_quantize(wt, n, m, s->fmt, 0, 0, sw, wq);
    qmm(s, xq, wq, b, n, m, 1, 1, *sx, *sw, Y); /* qmatmul(xq, wq, true) :299 */
    free(xt);
    free(wt);
}

/* halo_linear.hpp:305-439 */
void orc_linear_backward(const orc_scheme* s, int64_t b, int64_t m, int64_t n,
                         const float* xq, float sx, const float* wq, float sw,
                         const float* EY, float* EX, float* GW,
                         float* ehq, float* seh, float* eq, float* se) {
    /* plain E_Y quantization, shared by E (halo0/1) and G (all levels):
     * plain_error_operand :368-376 */
    orc_quantize(EY, b, n, s->fmt, 0, 0, se, eq);

    /* ---- error path :381-413 ---- */
    if (s->level == 2) { /* placement_E = {L, R} */
        const int64_t bp = orc_padded_batch(s, b);
        float* pad = (float*)calloc((size_t)(bp * n), sizeof(float)); /* pad_rows :397 */
        memcpy(pad, EY, sizeof(float) * (size_t)(b * n));
        orc_fwht_cols(pad, bp, n, s->block ? s->block : bp);   /* transform_left_h :399 */
        float* eh = ehq ? ehq : (float*)malloc(sizeof(float) * (size_t)(bp * n));
        float sh;
        orc_quantize(pad, bp, n, s->fmt, 0, 0, &sh, eh);
        if (seh) *seh = sh;
        float* prod = (float*)malloc(sizeof(float) * (size_t)(bp * m));
        qmm(s, eh, wq, bp, m, n, 1, 0, sh, sw, prod);          /* qmatmul(eq, wq) :401 */
        orc_fwht_cols(prod, bp, m, s->block ? s->block : bp);  /* transform_left :406 */
        memcpy(EX, prod, sizeof(float) * (size_t)(b * m));    /* take_rows :408 */
        orc_fwht_rows(EX, b, m, blk(s, m));                   /* transform_right_ht :411 */
        free(prod);
        free(pad);
        if (!ehq) free(eh);
    } else {
        qmm(s, eq, wq, b, m, n, 1, 0, *se, sw, EX);            /* :403 */
        if (s->level == 1) orc_fwht_rows(EX, b, m, blk(s, m)); /* :410-411 */
    }

    /* ---- gradient path :418-439: qmatmul(transpose_quantized(eq), xq) ---- */
    qmm(s, eq, xq, n, m, b, 0, 0, *se, sx, GW);
    if (s->level >= 1) orc_fwht_rows(GW, n, m, blk(s, m));     /* :436-437 */
}

/* ------------------------------------------------------------------ rng -- */

/* std::mt19937_64 (the standard fixes the sequence), tensor.hpp:398-431 */
typedef struct { uint64_t mt[312]; int idx; double spare; int has_spare; } orc_rng;

static void rng_seed(orc_rng* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
    r->has_spare = 0;
}

static uint64_t rng_bits(orc_rng* r) {
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
        }
        r->idx = 0;
    }
    uint64_t y = r->mt[r->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

static double rng_uniform(orc_rng* r) { return (double)(rng_bits(r) >> 11) * 0x1.0p-53; }

static double rng_normal(orc_rng* r) {
    if (r->has_spare) { r->has_spare = 0; return r->spare; }
    const double u1 = 1.0 - rng_uniform(r);
    const double u2 = rng_uniform(r);
    const double rad = sqrt(-2.0 * log(u1));
    const double a = 2.0 * 3.14159265358979323846 * u2;
    r->spare = rad * sin(a);
    r->has_spare = 1;
    return rad * cos(a);
}

/* tensor.hpp:433-439 */
void orc_randn(float* out, int64_t n, uint64_t seed, double stddev) {
    orc_rng r;
    rng_seed(&r, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = (float)(rng_normal(&r) * stddev);
}

/* ------------------------------------------------------------ baseline -- */

double orc_time_linear(const orc_scheme* s, int64_t b, int64_t m, int64_t n, uint64_t seed) {
    const int64_t bp = orc_padded_batch(s, b);
    float* X = malloc(sizeof(float) * (size_t)(b * m));
    float* W = malloc(sizeof(float) * (size_t)(n * m));
    float* EY = malloc(sizeof(float) * (size_t)(b * n));
    float* Y = malloc(sizeof(float) * (size_t)(b * n));
    float* xq = malloc(sizeof(float) * (size_t)(b * m));
    float* wq = malloc(sizeof(float) * (size_t)(n * m));
    float* EX = malloc(sizeof(float) * (size_t)(b * m));
    float* GW = malloc(sizeof(float) * (size_t)(n * m));
    float* eq = malloc(sizeof(float) * (size_t)(b * n));
    float* ehq = malloc(sizeof(float) * (size_t)(bp * n));
    orc_randn(X, b * m, seed, 1.0);
    orc_randn(W, n * m, seed + 1, 1.0 / sqrt((double)m));
    orc_randn(EY, b * n, seed + 2, 1e-3);
    float sx, sw, se, seh;
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    orc_linear_forward(s, b, m, n, X, W, Y, xq, &sx, wq, &sw);
    orc_linear_backward(s, b, m, n, xq, sx, wq, sw, EY, EX, GW, ehq, &seh, eq, &se);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    free(X); free(W); free(EY); free(Y); free(xq); free(wq); free(EX); free(GW); free(eq); free(ehq);
    return (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
}
