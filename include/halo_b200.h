/*
 * halo_b200.h — C ABI of libhalo_b200.so, the B200-native (sm_100a) HALO
 * quantized linear-layer training path.
 *
 * The reference (/root/reference/proj/include/halo, header-only C++20) has no
 * FFI: its operator surface is the HaloLinearLayerT class plus free functions.
 * Each entry point below replaces one of those interfaces (file:line given
 * relative to /root/reference/proj/include/halo/).  The C++ class
 * halo_b200::HaloLinearLayer in halo_b200.hpp restores the reference's
 * object API on top of this ABI, with the reference's exception types.
 *
 * Conventions
 *  - All tensors are row-major device pointers (cudaMalloc'd or torch
 *    storage); the caller owns them.  Nothing here allocates host copies.
 *  - Every call is stream-ordered and asynchronous; no host synchronisation
 *    happens on the hot path.  Scales live in device memory (float*).
 *  - had_block: Hadamard block B (2^k, or 12*2^k / 20*2^k <= 20480 with the
 *    reference's Paley bases); the transform is I (x) H_B.  0 means "the
 *    full dimension", i.e. the reference's transform verbatim
 *    (hadamard.hpp:62-129).
 *  - Errors are reported through halo_status; halo_last_error() returns a
 *    thread-local message.  Non-finite inputs are detected on the device and
 *    surface as HALO_ERR_NUMERIC from halo_ctx_check().
 */
#ifndef HALO_B200_H
#define HALO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HALO_B200_ABI_VERSION 1

#if defined(__GNUC__)
#define HALO_API __attribute__((visibility("default")))
#else
#define HALO_API
#endif

typedef struct CUstream_st* halo_stream_t; /* == cudaStream_t */

/* std::invalid_argument -> 1, numeric_error -> 2, std::logic_error -> 3
 * (the CLI's exit-code mapping, halo_cli.cpp:730-736, keeps 2/3 distinct). */
typedef enum halo_status {
    HALO_OK = 0,
    HALO_ERR_INVALID_ARGUMENT = 1,
    HALO_ERR_NUMERIC = 2,
    HALO_ERR_LOGIC = 3,
    HALO_ERR_CUDA = 4,
    HALO_ERR_NCCL = 5,
    HALO_ERR_IO = 6 /* io_error, tensor_io.hpp:25-27 */
} halo_status;

/* NumericFormat ids, quantize.hpp:22-29.  MXFP6 = E3M2 codes under a
 * power-of-two scale (compute_scales' MX rule, quantize.hpp:224-232) --
 * per-tensor here; the 1 x 32 block granularity (Granularity::mx) and the
 * BF16 / IDENTITY emulations are not on the device path. */
typedef enum halo_format {
    HALO_FMT_INT8 = 0,
    HALO_FMT_FP8_E4M3 = 1,
    HALO_FMT_FP6_E3M2 = 2,
    HALO_FMT_MXFP6_E3M2 = 3
} halo_format;

typedef enum halo_dtype { HALO_DTYPE_F32 = 0, HALO_DTYPE_BF16 = 1 } halo_dtype;

/* GEMM output kinds */
typedef enum halo_out_kind { HALO_OUT_F32 = 0, HALO_OUT_BF16 = 1, HALO_OUT_S32 = 2 } halo_out_kind;

/* Placement, halo_linear.hpp:29-61 */
typedef struct halo_placement {
    uint8_t left, middle, right, pad_;
} halo_placement;

/* HaloScheme, halo_linear.hpp:63-79, plus the Hadamard block size. */
typedef struct halo_scheme {
    halo_placement F, E, G;
    int32_t format_x, format_w, format_e; /* halo_format */
    int32_t granularity;                  /* HALO_GRAN_TENSOR, HALO_GRAN_ROW or HALO_GRAN_COLUMN (INT8 / FP8; see below) */
    int32_t quantize_f, quantize_e, quantize_g;
    int32_t peft;
    int64_t had_block; /* 0 = full dimension (reference) */
    char name[16];     /* preset id or "" */
} halo_scheme;

/* QuantCallCounters, halo_linear.hpp:161-164 */
typedef struct halo_counters {
    int64_t x, w, e;
} halo_counters;

HALO_API int halo_abi_version(void);
HALO_API const char* halo_last_error(void);

/* hadamard.hpp:69-85 / :87-93 */
HALO_API int halo_is_supported_hadamard_dim(int64_t d);
HALO_API int64_t halo_next_supported_hadamard_dim(int64_t d);

/* halo0/halo1/halo2 presets and "F:..;E:..;G:.." strings,
 * halo_linear.hpp:81-152 (scheme_from_string). */
HALO_API halo_status halo_scheme_from_string(const char* id, int32_t format, int64_t had_block, halo_scheme* out);

/* ------------------------------------------------------------ primitives */

/* quantize(transform_right(A, spec), fmt, Granularity::tensor(), scales)
 * hadamard.hpp:194-197 + quantize.hpp:244-280, fused (K1).
 *   had_block < 0 : no rotation (plain quantize)
 *   supplied_scale: NULL -> absmax scale (written to scale_out);
 *                   else used verbatim (quantize.hpp:259-266; FSDP regather).
 * codes: rows x cols bytes (int8 or OCP e4m3). */
HALO_API halo_status halo_rotate_quantize(const void* a, int32_t a_dtype, int64_t rows, int64_t cols, int64_t had_block,
                                 int32_t format, const float* supplied_scale, uint8_t* codes, float* scale_out,
                                 halo_stream_t stream);

/* max |A H| over the tensor (hqfsdp.hpp:216-225, the per-rank local absmax),
 * written as a float to absmax_out (device). */
/* phase B of halo_rotate_quantize under a given absmax (device float, the
 * value halo_rotate_absmax produces -- e.g. the max over HQ-FSDP ranks,
 * hqfsdp.hpp:172-196): scale = compute_scales(absmax) in-kernel, then the
 * codes.  scale_out may be NULL. */
HALO_API halo_status halo_rotate_quantize_amax(const void* a, int32_t a_dtype, int64_t rows, int64_t cols,
                                               int64_t had_block, int32_t format, const float* amax, uint8_t* codes,
                                               float* scale_out, halo_stream_t stream);
HALO_API halo_status halo_rotate_absmax(const void* a, int32_t a_dtype, int64_t rows, int64_t cols, int64_t had_block,
                               float* absmax_out, halo_stream_t stream);

/* HALO-2 error operand in one pass (K2): with b_pad = padded batch
 * (halo_linear.hpp:393-397; a multiple of had_block, or the next supported
 * dimension when had_block == 0):
 *   codes_rot   (b_pad x n) = quantize(transform_left_h(pad_rows(E, b_pad)))
 *   codes_plain (b x n)     = quantize(E)             (may be NULL)
 * and their scales. */
HALO_API halo_status halo_left_rotate_quantize(const void* e, int32_t e_dtype, int64_t b, int64_t n, int64_t had_block,
                                      int32_t format, uint8_t* codes_rot, float* scale_rot, uint8_t* codes_plain,
                                      float* scale_plain, halo_stream_t stream);
HALO_API int64_t halo_padded_batch(int64_t b, int64_t had_block);

/* transform_right / transform_right_ht on fp32 (identical for powers of
 * two), hadamard.hpp:194-203: out (rows x cols, f32 or bf16). */
HALO_API halo_status halo_transform_right(const float* in, void* out, int32_t out_dtype, int64_t rows, int64_t cols,
                                 int64_t had_block, halo_stream_t stream);

/* transform_left on fp32 rows [0, rows_pad) (hadamard.hpp:208-210) followed
 * by take_rows(rows_out) (tensor.hpp:232-240).  in may alias out. */
HALO_API halo_status halo_transform_left(const float* in, float* out, int64_t rows_pad, int64_t rows_out, int64_t cols,
                                int64_t had_block, halo_stream_t stream);

/* qmatmul, quantize.hpp:339-380 (K3, tcgen05):
 *   C[M x N] = A[M x K] * B^T,  A: a_kmajor ? [M][K] : [K][M]
 *                               B: b_kmajor ? [N][K] : [K][N]
 * INT8: C = float(double(acc_s32) * (double(sa) * double(sb))) — bit-exact;
 * HALO_OUT_S32 returns the raw accumulators.  FP8 E4M3: fp32 accumulate. */
HALO_API halo_status halo_qmatmul(int32_t format, const uint8_t* a, int32_t a_kmajor, const uint8_t* b, int32_t b_kmajor,
                         int64_t M, int64_t N, int64_t K, const float* scale_a, const float* scale_b, void* out,
                         int32_t out_kind, halo_stream_t stream);

/* qmatmul followed by transform_right along N (block had_block, 0 = N), the
 * reference's qmatmul -> transform_right_ht composition of the backward
 * (halo_linear.hpp:410-411, 433-437), with the transform fused into the
 * GEMM epilogue (had_block <= 256).  out_transposed != 0 stores C^T
 * ([n_valid][M], rows of C^T at or beyond n_valid dropped: the E path's
 * take_rows after transform_left, :405-409).  out_kind F32 / BF16. */
HALO_API halo_status halo_qmatmul_rotate(int32_t format, const uint8_t* a, int32_t a_kmajor, const uint8_t* b,
                                int32_t b_kmajor, int64_t M, int64_t N, int64_t K, const float* scale_a,
                                const float* scale_b, void* out, int32_t out_kind, int64_t had_block,
                                int32_t out_transposed, int64_t n_valid, halo_stream_t stream);

/* Granularity (quantize.hpp:65-87): per tensor, or one scale per row
 * (per token for X / E_Y, per output channel for W).  Column, block and MX
 * granularities are not on the device path. */
#define HALO_GRAN_TENSOR 0
#define HALO_GRAN_ROW 1
#define HALO_GRAN_COLUMN 2 /* INT8 / FP8; every product is the dequantized double matmul (deq_gemm) */
#define HALO_GRAN_MX 4     /* 1 x 32 blocks along rows, with HALO_FMT_MXFP6_E3M2 only (quantize.hpp:247-250);
                              power-of-two block scales, every product the dequantized double matmul (deq_gemm) */

/* quantize(transform_right(a, block), fmt, Granularity::row()): one scale per
 * row (compute_scales per group, quantize.hpp:202-239); codes bit-exact.
 * cols must be a multiple of 256; scales_out holds `rows` floats. */
HALO_API halo_status halo_rotate_quantize_rows(const void* a, int32_t a_dtype, int64_t rows, int64_t cols,
                                      int64_t had_block, int32_t format, uint8_t* codes, float* scales_out,
                                      halo_stream_t stream);

/* quantize([transform_right](A), mxfp6_e3m2, Granularity::mx()): power-of-two
 * scales per 1 x 32 block along rows (quantize.hpp:224-232), E3M2 codes in
 * bits 7:2; scales [rows x ceil(cols/32)].  had_block < 0: no rotation.
 * transpose_in != 0: A is the (cols x rows) row-major tensor and its
 * transpose is quantized (the gradient path's quantize(transpose(E_Y)),
 * halo_linear.hpp:427-431); no rotation then. */
HALO_API halo_status halo_rotate_quantize_mx(const void* a, int32_t a_dtype, int64_t rows, int64_t cols,
                                             int64_t had_block, int32_t transpose_in, uint8_t* codes, float* scales,
                                             halo_stream_t stream);

/* qmatmul with row-granularity operands whose scales sit on non-contracted
 * dims: a_per_row != 0 -> scale_a has M entries (rows of C), b_per_row != 0
 * -> scale_b has N entries (columns of C); C = float(double(acc) *
 * (double(sa_i) * double(sb_j))).  The reference dequantizes and multiplies
 * in double for non-tensor scales (quantize.hpp:345-349, 377-379): parity
 * within the tolerance stated in the tests.  out_kind F32 / BF16. */
HALO_API halo_status halo_qmatmul_scaled(int32_t format, const uint8_t* a, int32_t a_kmajor, const uint8_t* b,
                                int32_t b_kmajor, int64_t M, int64_t N, int64_t K, const float* scale_a,
                                int32_t a_per_row, const float* scale_b, int32_t b_per_row, void* out,
                                int32_t out_kind, halo_stream_t stream);

/* Granularity::row / ::column layers (scales on a contracted dim of E / G,
 * or of F for column) are served by the reference's dequantized double
 * products restated bit-exactly on the FP64 pipe (deq_gemm) -- a
 * full-precision matmul, off the tensor-core contract path.  Creating such a
 * layer returns HALO_ERR_INVALID_ARGUMENT unless this process-wide opt-in is
 * on (default off). */
HALO_API halo_status halo_allow_dequantized_products(int32_t on);

/* ----------------------------------------------------------------- layer */

typedef struct halo_linear halo_linear; /* HaloLinearLayerT, halo_linear.hpp:227 */
typedef struct halo_ctx halo_ctx;       /* SavedContextT,    halo_linear.hpp:207 */

/* HaloLinearLayerT(W, scheme), halo_linear.hpp:230-234: W is out x in
 * (n x m), device, caller-owned, read at every forward. */
HALO_API halo_status halo_linear_create(const halo_scheme* scheme, const void* w, int32_t w_dtype, int64_t out_features,
                               int64_t in_features, halo_linear** out);
HALO_API halo_status halo_linear_destroy(halo_linear* layer);
/* point the layer at new weights (e.g. after an optimizer step) */
HALO_API halo_status halo_linear_set_weight(halo_linear* layer, const void* w, int32_t w_dtype);
/* use an already rotated+quantized weight, e.g. the HQ-FSDP gathered
 * (WH)_Q (hqfsdp.hpp:204-237) or a frozen PEFT weight (halo_linear.hpp:248):
 * forward skips the weight quantization.  codes == NULL reverts. */
HALO_API halo_status halo_linear_set_qweight(halo_linear* layer, const uint8_t* codes, const float* scale);
/* HQ-FSDP without the all-gather (replaces quantized_all_gather +
 * backward_regather, hqfsdp.hpp:204-266, for this layer): (WH)_Q is the row
 * concatenation of n_parts equal shards, parts[i] (host array of device
 * pointers: local memory or a peer GPU's, e.g. halo_ipc_open) holding rows
 * [i*n/n_parts, (i+1)*n/n_parts).  The forward and E GEMMs read the shards in
 * place over NVLink; `scale` is the shared per-tensor scale.  Requires
 * n/n_parts % 256 == 0.  parts == NULL reverts. */
HALO_API halo_status halo_linear_set_qweight_sharded(halo_linear* layer, const uint8_t* const* parts, int32_t n_parts,
                                                     const float* scale);

HALO_API halo_status halo_ctx_create(halo_ctx** out);
HALO_API halo_status halo_ctx_destroy(halo_ctx* ctx);

/* forward, halo_linear.hpp:267-303: y (b x n) in y_dtype. */
HALO_API halo_status halo_linear_forward(halo_linear* layer, const void* x, int32_t x_dtype, int64_t b, void* y,
                                int32_t y_dtype, halo_ctx* ctx, halo_stream_t stream);

/* forward() fed the (XH)_Q already held by `src` (a context of another
 * layer with the same in_features and X quantizer: format, placement,
 * Hadamard block, granularity) -- the Llama gate/up pattern: X is quantized
 * once for both.  Same results as halo_linear_forward on the same X; `src`
 * must stay alive (and not be re-forwarded) until `ctx`'s backward. */
HALO_API halo_status halo_linear_forward_shared(halo_linear* layer, const halo_ctx* src, halo_ctx* ctx, void* y,
                                       int32_t y_dtype, halo_stream_t stream);

/* halo_linear_forward_shared for the up projection of a Llama MLP with the
 * SwiGLU product fused into the GEMM epilogue: u (b x n, bf16) = the
 * projection's output, h = silu(g) * u (bf16, exactly halo_swiglu_forward of
 * g and u) with g (b x n, bf16) the gate projection's output, read tile by
 * tile while the tensor cores run (model.hpp:169-171 with the Llama gate).
 * n must be a multiple of 256 and u, g, h 16-byte aligned
 * (HALO_ERR_INVALID_ARGUMENT otherwise: use halo_linear_forward_shared +
 * halo_swiglu_forward). */
HALO_API halo_status halo_linear_forward_shared_swiglu(halo_linear* layer, const halo_ctx* src, halo_ctx* ctx,
                                                       const void* g, void* u, void* h, halo_stream_t stream);

/* halo_linear_forward with the residual add of the block that follows the
 * projection (model.hpp:159-209: y = h + MLP(.), the MLP's last projection)
 * in the GEMM epilogue: y = RN_bf16(res + RN_bf16(x W^T)) (bf16), exactly a
 * bf16 forward output added to res as torch adds two bf16 tensors.  res and
 * y b x n bf16, n a multiple of 256, 16-byte aligned (HALO_ERR_INVALID_ARGUMENT
 * otherwise: use halo_linear_forward + halo_add). */
HALO_API halo_status halo_linear_forward_residual(halo_linear* layer, const void* x, int32_t x_dtype, int64_t b,
                                                  const void* res, void* y, halo_ctx* ctx, halo_stream_t stream);

/* halo_linear_backward with e_x accumulated onto a bf16 addend: e_x =
 * RN_bf16(e_x_add + RN_bf16(E_X)) -- the sum of the input gradients of two
 * projections reading the same X (the Llama gate / up pair), fused into the
 * E path's K4 store where the scheme has one (HALO-2, block 64..256), else a
 * separate add.  Identical to halo_linear_backward + halo_add. */
HALO_API halo_status halo_linear_backward_acc(halo_linear* layer, const halo_ctx* ctx, const void* e_y,
                                              int32_t e_dtype, const void* e_x_add, void* e_x, int32_t ex_dtype,
                                              void* grad_w, int32_t gw_dtype, halo_stream_t stream);

/* backward, halo_linear.hpp:305-439: e_y (b x n) -> e_x (b x m), grad_w
 * (n x m; may be NULL to skip G).  Granularity::row: the row scales sit on
 * the contracted dim of E and G, so both products are the reference's
 * dequantized double matmuls (quantize.hpp:377-379), bit-exact, on the FP64
 * pipe; out_features % 256 == 0, no PEFT / sharded / scattered layers. */
HALO_API halo_status halo_linear_backward(halo_linear* layer, const halo_ctx* ctx, const void* e_y, int32_t e_dtype,
                                 void* e_x, int32_t ex_dtype, void* grad_w, int32_t gw_dtype, halo_stream_t stream);

/* export_inference_weights, halo_linear.hpp:332-338: (WH)_Q codes + scale */
HALO_API halo_status halo_linear_export_inference_weights(halo_linear* layer, uint8_t* codes, float* scale,
                                                 halo_stream_t stream);

HALO_API halo_status halo_linear_counters(const halo_linear* layer, halo_counters* out);
HALO_API halo_status halo_linear_reset_counters(halo_linear* layer);

/* saved context views (device pointers owned by ctx) */
HALO_API halo_status halo_ctx_saved(const halo_ctx* ctx, const uint8_t** xq, const float** sx, const uint8_t** wq,
                           const float** sw, int64_t* batch_rows);
/* backward scratch views of the last backward: E quantizations and scales */
HALO_API halo_status halo_ctx_error_operands(const halo_ctx* ctx, const uint8_t** ehq, const float** seh,
                                    const uint8_t** eq, const float** se, int64_t* b_pad);
/* the backward scratch of `ctx` (error-operand codes and scales, the E / G
 * products' fp32 buffers) lives in `owner` from now on (NULL: its own again):
 * contexts whose backwards run one after another on one stream -- e.g. the
 * layers of a stack without activation checkpointing -- share one set
 * instead of holding one each.  `owner` must outlive `ctx`'s backward calls;
 * halo_ctx_error_operands then reports the shared buffers. */
HALO_API halo_status halo_ctx_share_scratch(halo_ctx* ctx, halo_ctx* owner);
/* synchronises `stream` and reports device-side numeric errors (NaN/Inf in
 * an input: tensor.hpp:86-91, quantize.hpp:292/373) as HALO_ERR_NUMERIC,
 * then clears the flag. */
HALO_API halo_status halo_ctx_check(halo_ctx* ctx, halo_stream_t stream);

/* stream-ordered device-to-device copy (used to snapshot ctx views) */
HALO_API halo_status halo_device_copy(void* dst, const void* src, int64_t bytes, halo_stream_t stream);

/* ------------------------------------------------- Llama MLP block glue */
/* h = silu(g) * u ; bf16, n elements (n % 8 == 0).  model.hpp:77-96 is the
 * reference's silu; the Llama MLP gates it with the up projection. */
HALO_API halo_status halo_swiglu_forward(const void* g, const void* u, void* h, int64_t n, halo_stream_t stream);
HALO_API halo_status halo_swiglu_backward(const void* dh, const void* g, const void* u, void* dg, void* du, int64_t n,
                                          halo_stream_t stream);
/* halo_swiglu_forward over [rows x cols] fused with phase A (the absmax pass)
 * of the down projection's X quantization (halo_linear.hpp:292-294; rotated
 * X with a 256 Hadamard block): the following halo_linear_forward(down, h,
 * ..., dctx) with this exact h buffer and batch reuses the absmax word.
 * Other configurations: identical to halo_swiglu_forward. */
HALO_API halo_status halo_swiglu_forward_absmax(const halo_linear* down, halo_ctx* dctx, const void* g, const void* u,
                                                void* h, int64_t rows, int64_t cols, halo_stream_t stream);
/* halo_swiglu_backward over [b x cols] fused with phase A (the absmax
 * pass) of the error-path quantization of both input projections
 * (halo_linear.hpp:393-399 and :371 for `gate` and `up`, HALO-2 family:
 * E.left).  The following halo_linear_backward(gate, gctx, dg, ...) and
 * halo_linear_backward(up, uctx, du, ...) — called with these exact dg / du
 * buffers and batch — reuse the absmax words instead of re-reading dg / du.
 * Other schemes: identical to halo_swiglu_backward. */
HALO_API halo_status halo_swiglu_backward_absmax(const halo_linear* gate, halo_ctx* gctx, const halo_linear* up,
                                                 halo_ctx* uctx, const void* dh, const void* g, const void* u,
                                                 void* dg, void* du, int64_t b, int64_t cols, halo_stream_t stream);
/* out = a + b elementwise (f32 or bf16), n % 8 == 0 */
HALO_API halo_status halo_add(const void* a, const void* b, void* out, int32_t dtype, int64_t n,
                              halo_stream_t stream);

/* ------------------------------------------- HQ-FSDP over peer memory */
/* Gradient reduce-scatter fused into the backward's G GEMM (replaces
 * reduce_scatter_grads' transfer, hqfsdp.hpp:271-300): recv[i] (host array
 * of `parts` device pointers, recv[rank] local, the others e.g. from
 * halo_ipc_open) is rank i's receive buffer [parts][out_features/parts][in]
 * fp32; every backward then TMA-stores this rank's fp32 partial G rows
 * owned by rank i into slot `rank` of recv[i] (grad_w is not written).
 * out_features/parts % 256 == 0.  recv == NULL reverts. */
HALO_API halo_status halo_linear_set_grad_scatter(halo_linear* layer, void* const* recv, int32_t parts, int32_t rank);
/* Owner side: out = T(sum_w double(recv[w]) / world) over [world][rows][cols]
 * fp32 partials, rank order (hqfsdp.hpp:288-292); T = out_dtype. */
HALO_API halo_status halo_reduce_scatter_shard(const float* recv, int32_t world, int64_t rows, int64_t cols, void* out,
                                               int32_t out_dtype, halo_stream_t stream);
/* Device buffers shareable across processes (CUDA IPC), zero-filled: the
 * local weight shard's codes and the rank's mailbox (3*world u32). */
#define HALO_PEER_MAX 8
#define HALO_IPC_HANDLE_BYTES 64
HALO_API halo_status halo_peer_alloc(int64_t bytes, void** ptr);
HALO_API halo_status halo_peer_free(void* ptr);
HALO_API halo_status halo_ipc_handle(const void* ptr, void* handle /* HALO_IPC_HANDLE_BYTES */);
HALO_API halo_status halo_ipc_open(const void* handle, void** ptr);
HALO_API halo_status halo_ipc_close(void* ptr);
/* Stream-ordered barrier of `world` ranks over their mailboxes (host array
 * of world device pointers, mailboxes[rank] local): posts *amax_in (if not
 * NULL) to every rank, waits until every rank reached `epoch` (> 0, the same
 * increasing sequence on all ranks), then writes the max of the posted
 * values to *amax_out (if not NULL).  Replaces the absmax all-reduce of
 * hqfsdp.hpp:172-196 and orders shard writes before peer reads. */
HALO_API halo_status halo_peer_sync(void* const* mailboxes, int32_t world, int32_t rank, uint32_t epoch,
                                    const float* amax_in, float* amax_out, halo_stream_t stream);

/* ------------------------------------------------ quantized tensor files */
/* write_quantized_tensor / read_quantized_tensor (quantize.hpp:405-474) in
 * the reference's HALT container (tensor_io.hpp:1-135): a file written here
 * is read by the reference and vice versa.  HOST buffers in the device code
 * layouts (INT8 bytes, OCP E4M3 bytes, E3M2 codes in bits 7:2); granularity
 * HALO_GRAN_TENSOR (1 scale), _ROW (rows), _COLUMN (cols).  FP8 / FP6 codes
 * travel as f32 grid values (the reference's QF32 payload); reading a value
 * off the grid, a block / mx granularity or an emulation-only format fails
 * with HALO_ERR_IO. */
HALO_API halo_status halo_quantized_tensor_write(const char* path, int32_t format, int32_t granularity, int64_t rows,
                                                 int64_t cols, const uint8_t* codes, const float* scales,
                                                 int64_t n_scales);
HALO_API halo_status halo_quantized_tensor_info(const char* path, int32_t* format, int32_t* granularity,
                                                int64_t* rows, int64_t* cols, int64_t* n_scales);
HALO_API halo_status halo_quantized_tensor_read(const char* path, uint8_t* codes, float* scales);

/* ------------------------------------------------- transformer block glue */
/* RMSNorm (rmsnorm.hpp:27-100): y = x * r * gain, r = 1/sqrt(S/D + eps),
 * S = sum x^2 in double, D = dim if `mean` (Llama) else 1 -- mean = 0,
 * eps = 0 is the reference's x/||x|| (a zero row then gives non-finite y,
 * which the next HALO quantizer reports as HALO_ERR_NUMERIC; the reference
 * raises numeric_error).  x bf16 [rows x dim], gain fp32 [dim], y bf16 or
 * fp32, rstd (fp32 [rows], may be NULL) saved for the backward. */
HALO_API halo_status halo_rmsnorm_forward(const void* x, const float* gain, void* y, int32_t y_dtype, float* rstd,
                                          int64_t rows, int64_t dim, int32_t mean, double eps, halo_stream_t stream);
/* rmsnorm_backward + rmsnorm_gain_gradient (rmsnorm.hpp:52-100):
 * dx = r g dy - (r^3 x / D) sum(g dy x) (bf16), dgain = sum_rows dy x r (fp32,
 * deterministic order); dy bf16 or fp32. */
HALO_API halo_status halo_rmsnorm_backward(const void* x, const void* dy, int32_t dy_dtype, const float* gain,
                                           const float* rstd, void* dx, float* dgain, int64_t rows, int64_t dim,
                                           int32_t mean, halo_stream_t stream);
/* The pre-norm residual pattern of the Llama block (model.hpp:159-209:
 * h = x + r; y = rmsnorm(h)) in one pass: h = RN_bf16(x + r) (bf16, as a
 * bf16 tensor add rounds) is written to h and normalised into y (bf16);
 * mean = 1 (the Llama form) only. */
HALO_API halo_status halo_add_rmsnorm_forward(const void* x, const void* r, const float* gain, void* h, void* y,
                                              float* rstd, int64_t rows, int64_t dim, double eps,
                                              halo_stream_t stream);
/* Its backward: dx = RN_bf16(RN_bf16(rmsnorm_backward(h, dy)) + dres) --
 * the residual-stream gradient dres (bf16) accumulated the way autograd
 * sums two bf16 gradients -- and dgain as halo_rmsnorm_backward; the result
 * is the gradient of both x and r.  mean = 1 only. */
HALO_API halo_status halo_rmsnorm_backward_res(const void* h, const void* dy, int32_t dy_dtype, const float* gain,
                                               const float* rstd, const void* dres, void* dx, float* dgain,
                                               int64_t rows, int64_t dim, halo_stream_t stream);
/* Rotary embedding over fused qkv rows [rows x heads*head_dim] (bf16): the
 * first rot_heads heads (q and k) rotated by (cos, sin) pairs of
 * cos_sin[(row % seq) * head_dim/2 + i] (fp32 interleaved), the rest (v)
 * copied; backward = the transpose rotation.  in may not alias out. */
HALO_API halo_status halo_rope_qkv(const void* in, void* out, const float* cos_sin, int64_t rows, int32_t seq,
                                   int32_t rot_heads, int32_t heads, int32_t head_dim, int32_t backward,
                                   halo_stream_t stream);

/* ------------------------------------------------- FP6 E3M2 wire format */
/* The packed FP6 payload of the HQ-FSDP gather (hqfsdp.hpp:36-49: four
 * codes in three bytes, 0.375 x BF16): n device codes (E3M2 in bits 7:2 of a
 * byte each, n % 4 == 0) <-> 3n/4 bytes; group g = codes 4g..4g+3 packed as
 * the 24-bit little-endian word c0 | c1 << 6 | c2 << 12 | c3 << 18. */
HALO_API halo_status halo_fp6_pack(const uint8_t* codes, uint8_t* packed, int64_t n, halo_stream_t stream);
HALO_API halo_status halo_fp6_unpack(const uint8_t* packed, uint8_t* codes, int64_t n, halo_stream_t stream);

/* ------------------------------------------------ optimizer (HQ-FSDP) */
/* AdamWT::step for one parameter (trainer.hpp:104-160), e.g. this rank's
 * row shard of a master weight in the HQ-FSDP training loop
 * (hqfsdp.hpp:340-411): m, v (fp32 state, n each) and param (bf16 or fp32)
 * updated in place from grad (bf16 or fp32) in IEEE double as the reference
 * writes it; lr = lr_at(t), bc1 = 1 - beta1^t, bc2 = 1 - beta2^t (:127-131).
 * n % 4 == 0; 16 B aligned pointers. */
HALO_API halo_status halo_adamw_step(void* param, int32_t p_dtype, const void* grad, int32_t g_dtype, float* m,
                                     float* v, int64_t n, double lr, double beta1, double beta2, double eps,
                                     double weight_decay, double bc1, double bc2, halo_stream_t stream);

/* --------------------------------------- HQ-FSDP data plane over NCCL */
/* The weight protocol of hqfsdp.hpp:172-300 between real ranks (one process
 * per GPU), stream-ordered, NCCL resolved at run time (libnccl.so.2).
 * Every rank owns rows [rank*shard_rows, (rank+1)*shard_rows) of a weight
 * padded to world*shard_rows rows (shard, :131-148). */
typedef struct halo_fsdp halo_fsdp;
#define HALO_FSDP_ID_BYTES 128 /* ncclUniqueId */
HALO_API halo_status halo_fsdp_get_unique_id(void* id);
HALO_API halo_status halo_fsdp_create(const void* id, int32_t world, int32_t rank, halo_fsdp** out);
HALO_API halo_status halo_fsdp_destroy(halo_fsdp* f);
HALO_API halo_status halo_fsdp_world(const halo_fsdp* f, int32_t* world, int32_t* rank);
/* quantized_all_gather (:204-237): absmax of the rotated shard, max over
 * ranks, shared scale compute_scales(max) (device, scale_out), codes of the
 * local rows under it, all-gather: gathered = (world*shard_rows x cols)
 * codes, bit-identical to a single-process quantize of the rotated padded
 * weight.  local_absmax_out (device float, may be NULL) keeps this rank's
 * absmax for the backward's stale check. */
HALO_API halo_status halo_fsdp_quantized_all_gather(halo_fsdp* f, const void* shard, int32_t dtype, int64_t shard_rows,
                                                    int64_t cols, int64_t had_block, int32_t format,
                                                    uint8_t* gathered, float* scale_out, float* local_absmax_out,
                                                    halo_stream_t stream);
/* backward_regather (:243-266): the same codes under the saved forward
 * scale, no scale traffic; with saved_local_absmax and stale_flag, a shard
 * whose absmax changed since the forward sets *stale_flag (device u32; the
 * reference throws std::logic_error, :256-259 -- test the flag once). */
HALO_API halo_status halo_fsdp_backward_regather(halo_fsdp* f, const void* shard, int32_t dtype, int64_t shard_rows,
                                                 int64_t cols, int64_t had_block, int32_t format, const float* scale,
                                                 const float* saved_local_absmax, uint32_t* stale_flag,
                                                 uint8_t* gathered, halo_stream_t stream);
/* reduce_scatter_grads (:271-300): shard_out (shard_rows x cols) = this
 * rank's rows of sum_ranks(grad) / world; grad (world*shard_rows x cols)
 * f32 or bf16 (NCCL's reduction order; the reference sums in double in rank
 * order -- tolerance parity). */
HALO_API halo_status halo_fsdp_reduce_scatter(halo_fsdp* f, const void* grad, int32_t dtype, int64_t shard_rows,
                                              int64_t cols, void* shard_out, halo_stream_t stream);
/* mean over ranks in place (replicated parameters' gradients, e.g. norm gains) */
HALO_API halo_status halo_fsdp_all_reduce_mean(halo_fsdp* f, void* buf, int32_t dtype, int64_t n,
                                               halo_stream_t stream);

/* ------------------------------------------------------------- profiling */
/* Kernel classes: 0 K1 row-FWHT+quantize, 1 K2 column-FWHT+dual quantize,
 * 2 K3 tcgen05 GEMM, 3 K4 output un-rotation, 4 elementwise glue.
 * work = algorithmic bytes (classes 0,1,3,4) or integer ops (class 2). */
typedef struct halo_profile {
    int64_t launches[5];
    double ms[5];
    double work[5];
} halo_profile;
/* bracket every kernel launch with CUDA events on its stream (off by default) */
HALO_API halo_status halo_profile_enable(int on);
/* synchronises the device, reduces the recorded launches, clears them */
HALO_API halo_status halo_profile_read(halo_profile* out);

#ifdef __cplusplus
}
#endif
#endif /* HALO_B200_H */
