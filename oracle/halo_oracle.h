/*
 * halo_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference HALO hot path (arxiv 2501.02625, reference
 * at /root/reference/proj/include/halo/*.hpp) in plain C.  It is the checker
 * for the CUDA path; nothing in the product (paper_2501_02625_b200/) links,
 * imports or executes it.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may call it.
 *
 * Parity is pinned two ways:
 *   1. against the reference headers themselves, compiled unmodified into
 *      oracle/_ref/libhalo_ref.so by oracle/Makefile (tests/test_oracle_vs_ref.py);
 *   2. against golden vectors generated from that build
 *      (tests/golden/make_golden.py -> tests/golden/*.npz) and the pinned
 *      values of the reference's own Catch2 tests (tests/test_oracle_golden.py).
 *
 * Block-size extension: every transform takes a power-of-two block B that
 * divides the transformed dimension; the transform is I_{d/B} (x) H_B.  With
 * B == d it is exactly the reference's full-dimension transform.
 */
#ifndef HALO_ORACLE_H
#define HALO_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* format ids follow NumericFormat (quantize.hpp:22-29) */
enum { ORC_INT8 = 0, ORC_FP8_E4M3 = 1, ORC_FP6_E3M2 = 2, ORC_MXFP6_E3M2 = 3 };

/* hadamard.hpp:69-93 */
int orc_is_supported_hadamard_dim(int64_t d);
int64_t orc_next_supported_hadamard_dim(int64_t d);

/* Right transform A <- A (I (x) H_B), rows x cols row-major, in place.
 * hadamard.hpp:136-177 (transform_row, pow2 path) applied to every
 * contiguous B-element segment of every row. */
void orc_fwht_rows(float* a, int64_t rows, int64_t cols, int64_t block);

/* Left transform A <- (I (x) H_B) A over the row index, in place.
 * hadamard.hpp:205-216 (transform_left/_left_h: transpose, row transform,
 * transpose; identical for powers of two). */
void orc_fwht_cols(float* a, int64_t rows, int64_t cols, int64_t block);

/* quantize.hpp:138-180 round_code for INT8 / E4M3 / E3M2. */
double orc_round_code(double x, int fmt);

/* quantize.hpp:202-239 per-tensor scale: float(absmax/fmax), 1.0 if zero.
 * Returns 0 and sets *nonfinite when a NaN/Inf is present. */
float orc_tensor_scale(const float* a, int64_t n, int fmt, int* nonfinite);

/* quantize.hpp:244-280: codes[i] = round_code(double(a[i]) / double(scale)).
 * gran: 0 tensor (scales[0]), 1 row (scales[r]), 2 column (scales[c]).
 * When supplied==0 the scales are computed (quantize.hpp:268) into scales. */
void orc_quantize(const float* a, int64_t rows, int64_t cols, int fmt, int gran,
                  int supplied, float* scales, float* codes);

/* codes (exact grid values) -> device byte encodings */
void orc_codes_to_int8(const float* codes, int64_t n, int8_t* out);
void orc_codes_to_e4m3(const float* codes, int64_t n, uint8_t* out);
float orc_e4m3_to_float(uint8_t b);

/* quantize.hpp:339-375 integer path, with the raw accumulators exposed.
 * A is M x K: a_kmajor ? A[m*K+k] : A[k*M+m]
 * B is N x K: b_kmajor ? B[n*K+k] : B[k*N+n]
 * acc (optional) receives the int64 sums as int32 (|acc| < 2^31 here);
 * out (optional) receives float(double(acc) * (double(sa)*double(sb))). */
void orc_qmatmul_i8(const int8_t* A, const int8_t* B, int64_t M, int64_t N, int64_t K,
                    int a_kmajor, int b_kmajor, float sa, float sb, int32_t* acc, float* out);

/* quantize.hpp:377-379 non-integer path: dequantize (code*scale in double,
 * rounded to float, :282-294) then a double-accumulated matmul
 * (tensor.hpp:126-181).  Codes given as floats; per-tensor scales. */
void orc_qmatmul_deq(const float* A, const float* B, int64_t M, int64_t N, int64_t K,
                     int a_kmajor, int b_kmajor, float sa, float sb, float* out);

/* ---- HaloLinearLayer (halo_linear.hpp:227-462), presets halo0/1/2 ---- */
typedef struct {
    int level;        /* 0, 1, 2  (halo_linear.hpp:81-106) */
    int fmt;          /* ORC_INT8 / ORC_FP8_E4M3 for X, W and E alike */
    int64_t block;    /* Hadamard block; 0 => full dimension (reference) */
} orc_scheme;

/* forward (halo_linear.hpp:267-303): Y = q(XH) q(WH)^T.
 * xq/wq (codes, float) and scales are the saved context. */
void orc_linear_forward(const orc_scheme* s, int64_t b, int64_t m, int64_t n,
                        const float* X, const float* W, float* Y,
                        float* xq, float* sx, float* wq, float* sw);

/* backward (halo_linear.hpp:305-439) from the saved context.
 * ehq (b_pad x n, may be NULL) / eq (b x n) receive the two E_Y
 * quantizations with their scales; EX b x m, GW n x m. */
void orc_linear_backward(const orc_scheme* s, int64_t b, int64_t m, int64_t n,
                         const float* xq, float sx, const float* wq, float sw,
                         const float* EY, float* EX, float* GW,
                         float* ehq, float* seh, float* eq, float* se);

/* padded token count used by the left transform (halo_linear.hpp:393-397) */
int64_t orc_padded_batch(const orc_scheme* s, int64_t b);

/* Bounded CPU baseline: one HALO-2 fwd+bwd through the restatement,
 * single thread.  Returns wall seconds. */
double orc_time_linear(const orc_scheme* s, int64_t b, int64_t m, int64_t n, uint64_t seed);

/* reference Rng (tensor.hpp:398-445): mt19937_64 + hand-rolled Box-Muller */
void orc_randn(float* out, int64_t n, uint64_t seed, double stddev);

#ifdef __cplusplus
}
#endif
#endif
