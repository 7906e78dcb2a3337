// halo_internal.h — internal launch interface between the host layer
// (halo_capi.cpp) and the kernels (fwht_quant.cu, gemm_sm100.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace halo_b200 {

int num_sms();
// stream-ordered scratch (cudaMallocAsync) comes from the device's default
// pool; with the default release threshold (0) every synchronisation hands
// the pages back and the next allocation re-maps them (tens of ms for the
// large-block K2 scratch).  Called before such allocations: keep the pool.
void retain_async_pool();
// MXFP6 (NumericFormat::MxFp6E3M2, id 3) has E3M2 codes under power-of-two
// 1 x 32 block scales (quantize.hpp:224-232, mx_quantize); kernels that only
// see codes (GEMMs, deq_gemm) treat it as FMT_E3M2
constexpr int FMT_MXFP6 = 3;
inline int code_format(int fmt) { return fmt == FMT_MXFP6 ? 2 : fmt; }

float hadamard_norm(int64_t B);

// K1 / K4-right: right transform over the contiguous dim (block B), then
// mode 0 absmax / 1 quantize (fmt) / 2 write transformed values (out_dtype).
void run_rows(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t B, int mode, int fmt,
              unsigned* amax, const float* supplied, uint8_t* codes, void* out, int out_dtype, unsigned* err,
              float* scale_out, cudaStream_t st);

// K2 / K4-left: left transform over rows (block B, rows_pad a multiple of
// B; rows [b, rows_pad) are zero padding), plus the un-rotated E_Y path.
void run_cols(const void* in, int in_dtype, int64_t b, int64_t rows_pad, int64_t cols, int64_t B, int mode, int fmt,
              unsigned* amax_rot, unsigned* amax_plain, const float* sup_rot, const float* sup_plain,
              uint8_t* codes_rot, uint8_t* codes_plain, float* out, int64_t rows_out, unsigned* err,
              float* scale_rot_out, float* scale_plain_out, cudaStream_t st);

// un-rotated absmax / quantize
void run_plain(const void* in, int in_dtype, int64_t n, int mode, int fmt, unsigned* amax, const float* supplied,
               uint8_t* codes, unsigned* err, float* scale_out, cudaStream_t st);

// K3: C[M x N] = A[M x K] * B[N x K]^T with per-tensor scales.
//   A: a_kmajor ? [M][K] row-major : [K][M] row-major
//   B: b_kmajor ? [N][K] row-major : [K][N] row-major
//   out_kind: 0 fp32, 1 bf16, 2 raw int32 accumulators (INT8 only)
// Returns 0 on success, else a cudaError_t / -1 for unsupported shapes.
int run_gemm(int fmt, const uint8_t* A, const uint8_t* B, int64_t M, int64_t N, int64_t K, int a_kmajor,
             int b_kmajor, const float* sa, const float* sb, void* out, int out_kind, cudaStream_t st);
// K3 + fused K4: as run_gemm, then a blockwise FWHT (block 2^xf_lb <= 256,
// reference stage order, final multiply by xf_norm) along N inside the
// epilogue; out_trans stores C^T ([n_valid][M], rows of C^T beyond n_valid
// dropped).  out_kind 0/1 only.
int run_gemm_x(int fmt, const uint8_t* A, const uint8_t* B, int64_t M, int64_t N, int64_t K, int a_kmajor,
               int b_kmajor, const float* sa, const float* sb, void* out, int out_kind, int xf_lb, float xf_norm,
               int out_trans, int64_t n_valid, cudaStream_t st);
// Sharded GEMM operand (HQ-FSDP without an all-gather): the operand is the
// row-concatenation of n equal parts of `len` rows (rows along K when
// along_k, else along M / N), part i behind maps[i] (device array, u8,
// box 128 x 128, 128 B swizzle: encode_shard_maps).  Parts may be peer
// GPUs' memory (CUDA IPC over NVLink).  Installed for the run_gemm* calls of
// the current thread by a ShardScope; the corresponding A / B pointer is
// then ignored.
struct ShardSpec {
    const CUtensorMap* maps;  // device
    CUtensorMap maps_host0;   // host copy of part 0 (kernel parameter placeholder)
    int n;
    int64_t len;
    int along_k;
};
// Scattered fp32 C (the HQ-FSDP gradient reduce-scatter fused into the G
// GEMM): rows [i*len, (i+1)*len) of C are TMA-stored through maps[i] into
// this rank's slot of rank i's receive buffer (encode_scatter_maps).
struct ScatterSpec {
    const CUtensorMap* maps;  // device
    CUtensorMap maps_host0;
    int parts;
    int64_t len;
};
struct ShardScope {
    ShardScope(const ShardSpec* a, const ShardSpec* b, const ScatterSpec* c = nullptr);
    ~ShardScope();
    static bool active();  // sharded / scattered operands installed on this thread
};
// K4 with a fused bf16 addend (fwht3.cu): out = RN(add + RN(rotated in)),
// B in {64, 128, 256}; false = not handled (caller adds separately)
bool rows_xform_add(const float* in, int64_t n, int64_t B, const void* add, void* out, cudaStream_t st);
// SwiGLU epilogue for the next run_gemm_v on this thread (the up projection
// of a Llama MLP): C = u (bf16), h = silu(g) * u; g, h [M][N] bf16.  h null:
// the residual epilogue, C = RN_bf16(g + RN_bf16(acc))
struct GluScope {
    GluScope(const void* g, void* h);
    ~GluScope();
    static bool used();  // the GEMM under this scope took the SwiGLU epilogue
};
// receive buffers recv[i] = [parts][len][cols] fp32 of rank i; maps for slot `slot`
bool encode_scatter_maps(void* const* recv, int parts, int slot, int64_t len, int64_t cols, CUtensorMap* out);
bool encode_shard_maps(const uint8_t* const* parts, int n, int64_t inner, int64_t rows, CUtensorMap* out);

// as run_gemm_x with optional per-row (sa_vec[M]) / per-column (sb_vec[N])
// scales (Granularity::row on the non-contracted dims); no transform then.
int run_gemm_v(int fmt, const uint8_t* A, const uint8_t* B, int64_t M, int64_t N, int64_t K, int a_kmajor,
               int b_kmajor, const float* sa, const float* sa_vec, const float* sb, const float* sb_vec, void* out,
               int out_kind, int xf_lb, float xf_norm, int out_trans, int64_t n_valid, cudaStream_t st);

// production K1/K2/K4 kernels for blocks <= 256 (fwht2.cu); false = not handled
bool rows_v2(int mode, int fmt, int in_dtype, const void* in, int64_t n, int64_t B, unsigned* amax, const float* sup,
             uint8_t* codes, void* out, int out_dtype, unsigned* err, float* sout, cudaStream_t st);
bool cols_v2(int mode, int fmt, int in_dtype, const void* in, int64_t b, int64_t rows_pad, int64_t cols, int64_t B,
             unsigned* ar, unsigned* ap, const float* sr, const float* sp, uint8_t* cr, uint8_t* cp, float* out,
             int64_t rows_out, unsigned* err, float* sro, float* spo, cudaStream_t st);

// 2-D 128B-swizzled TMA descriptor (gemm_sm100.cu); dtype 0 f32, 1 bf16, 2 u8
bool encode_2d_sw128(CUtensorMap* map, int dtype, const void* base, uint64_t inner, uint64_t outer,
                     uint32_t box_outer);

// 2-D tensor map without swizzle, zero OOB fill (gemm_sm100.cu)
bool encode_2d_plain(CUtensorMap* map, int dtype, const void* base, uint64_t inner, uint64_t outer, uint64_t row_bytes,
                     uint32_t box_inner, uint32_t box_outer);

// K1 kernel generation (HALO_K1_VERSION, default 4)
int k1_version();

// third-generation K1 / K4-right (fwht3.cu): B = 2^k <= 256, FADD2 butterflies
bool rows_v3(int mode, int fmt, int in_dtype, const void* in, int64_t n, int64_t B, unsigned* amax, const float* sup,
             uint8_t* codes, void* out, int out_dtype, unsigned* err, float* sout, cudaStream_t st);

// K1 / K4 for large blocks (fwht_big.cu): 512 <= B <= 16384, B = 2^k
// K1 / K4 for 512 <= B <= 8192 (fwht3.cu, radix-8 float4 rounds); false = not applicable
bool rows_lb(int mode, int fmt, int in_dtype, const void* in, int64_t n, int64_t B, unsigned* amax, const float* sup,
             uint8_t* codes, void* out, int out_dtype, unsigned* err, float* sout, cudaStream_t st);
bool rows_big(int mode, int fmt, int in_dtype, const void* in, int64_t n, int64_t B, unsigned* amax, const float* sup,
              uint8_t* codes, void* out, int out_dtype, unsigned* err, float* sout, cudaStream_t st);

// K2 for 512 <= B <= 4096 along the token axis, one kernel per phase
// (fwht_cols_lb.cu); false = shape not covered (the caller falls back)
bool cols_lb(int mode, int fmt, int in_dtype, const void* in, int64_t b, int64_t rows_pad, int64_t cols, int64_t B,
             unsigned* ar, unsigned* ap, const float* sr, const float* sp, uint8_t* cr, uint8_t* cp, unsigned* err,
             float* sro, float* spo, cudaStream_t st, float* xout, int64_t rows_out);
// K2 for large blocks along the token axis (fwht_cols_big.cu): 512 <= B <= 16384
bool cols_big(int mode, int fmt, int in_dtype, const void* in, int64_t b, int64_t rows_pad, int64_t cols, int64_t B,
              unsigned* ar, unsigned* ap, const float* sr, const float* sp, uint8_t* cr, uint8_t* cp, unsigned* err,
              float* sro, float* spo, cudaStream_t st, float* xout = nullptr, int64_t rows_out = 0);

// Hadamard blocks 12·2^k / 20·2^k (fwht_base.cu): the reference's Paley
// bases.  Orientation (H or H^T, transpose_base of hadamard.hpp:136) from
// the enclosing BaseScope; power-of-two blocks ignore it (H = H^T).
struct BaseScope {
    explicit BaseScope(bool transpose_base);
    ~BaseScope();
};
int base_dim_of(int64_t B);  // 12, 20 or 0
bool rows_base(int mode, int fmt, int in_dtype, const void* in, int64_t n, int64_t B, unsigned* amax,
               const float* sup, uint8_t* codes, void* out, int out_dtype, unsigned* err, float* sout,
               cudaStream_t st);
bool cols_base(int mode, int fmt, int in_dtype, const void* in, int64_t b, int64_t rows_pad, int64_t cols, int64_t B,
               unsigned* ar, unsigned* ap, const float* sr, const float* sp, uint8_t* cr, uint8_t* cp, unsigned* err,
               float* sro, float* spo, cudaStream_t st, float* xout, int64_t rows_out);

// third-generation K2 (fwht_cols3.cu): absmax / quantize, B = 2^k <= 256
bool cols_v3(int mode, int fmt, int in_dtype, const void* in, int64_t b, int64_t rows_pad, int64_t cols, int64_t B,
             unsigned* ar, unsigned* ap, const float* sr, const float* sp, uint8_t* cr, uint8_t* cp, unsigned* err,
             float* sro, float* spo, cudaStream_t st);

// Granularity::row quantization (fwht3.cu): rows*cols input, cols % 256 == 0;
// amax_rows / row_scales: `rows` words / floats of device scratch / output
bool rows_v3_per_row(int fmt, int in_dtype, const void* in, int64_t rows, int64_t cols, int64_t B,
                     unsigned* amax_rows, float* row_scales, uint8_t* codes, unsigned* err, cudaStream_t st);

// Granularity::row backward products (deq_gemm.cu): C[i,j] (fp32, ldc) =
// sum_k deq(A(i,k)) * deq(B(k,j)) in double, k ascending (qmatmul's
// dequantized path, quantize.hpp:377-379).  Views by element / scale strides.
// scale index of A(i, k) = (i >> a_sh_i) * as_si + (k >> a_sh_k) * as_sk (B likewise):
// shift 5 walks the 32-wide MX blocks
bool deq_gemm(int fmt, const uint8_t* a, const float* as, int64_t a_si, int64_t a_sk, int64_t as_si, int64_t as_sk,
              const uint8_t* b, const float* bs, int64_t b_sk, int64_t b_sj, int64_t bs_sk, int64_t bs_sj, float* c,
              int64_t M, int64_t N, int64_t K, int64_t ldc, cudaStream_t st, int a_sh_i = 0, int a_sh_k = 0,
              int b_sh_k = 0, int b_sh_j = 0);
// Granularity::mx quantization (MxFp6E3M2): view in[r*rs + c*cs] (rows x cols)
// -> codes [rows x cols] (E3M2 in bits 7:2), scales [rows x ceil(cols/32)]
bool mx_quantize(int in_dtype, const void* in, int64_t rows, int64_t cols, int64_t rs, int64_t cs, uint8_t* codes,
                 float* scales, unsigned* err, cudaStream_t st);
// quantize(A, fmt, Granularity::column()) (deq_gemm.cu): `cols` scales
bool col_quantize(int fmt, int in_dtype, const void* in, int64_t rows, int64_t cols, unsigned* amax, float* scales,
                  uint8_t* codes, unsigned* err, cudaStream_t st);
// fp32 copy of a (b x cols) bf16 / fp32 tensor with zero rows up to b_pad
void pad_rows_f32(const void* in, int in_dtype, int64_t b, int64_t b_pad, int64_t cols, float* out, cudaStream_t st);

// K2 phase A of the MLP gate/up projections fused with the SwiGLU backward
// (fwht_cols3.cu)
bool cols_swiglu_absmax(const void* dh, const void* g, const void* u, void* dg, void* du, int64_t b, int64_t rows_pad,
                        int64_t cols, int64_t B, unsigned* gr, unsigned* gp, unsigned* ur, unsigned* up, unsigned* err,
                        cudaStream_t st);

// halo_last_error() text (halo_capi.cu)
void set_last_error(const char* msg);

// SwiGLU forward fused with K1 phase A of the down projection (fwht3.cu):
// h = swiglu(g, u) in bf16 plus the absmax of h's 256-blockwise rotation
bool swiglu_absmax(const void* g, const void* u, void* h, int64_t n, int64_t cols, unsigned* amax, unsigned* err,
                   cudaStream_t st);

// elementwise glue (glue.cu)
void run_swiglu_fwd(const void* G, const void* U, void* H, int64_t n, cudaStream_t st);
void run_swiglu_bwd(const void* dH, const void* G, const void* U, void* dG, void* dU, int64_t n, cudaStream_t st);
void run_add(const void* a, const void* b, void* out, int dtype, int64_t n, cudaStream_t st);
// out[i] = T(sum_w double(recv[w*n + i]) / world), n % 4 == 0
void run_rank_mean(const float* recv, int world, int64_t n, void* out, int dtype, cudaStream_t st);
// FP6 E3M2 wire format: 4 codes (bits 7:2 of a byte each) <-> 3 bytes; n % 4 == 0
void run_fp6_pack(const uint8_t* codes, uint8_t* packed, int64_t n, cudaStream_t st);
void run_fp6_unpack(const uint8_t* packed, uint8_t* codes, int64_t n, cudaStream_t st);
// Llama block glue (llama_glue.cu)
// res / hout: h = RN_bf16(x + res) is written to hout and normalised (Llama form)
bool run_rmsnorm_fwd(const void* x, const float* gain, void* y, int y_dtype, float* rstd, int64_t rows, int dim,
                     bool mean, double eps, cudaStream_t st, const void* res = nullptr, void* hout = nullptr);
// dres: dx = RN_bf16(RN_bf16(dx_norm) + dres) (Llama form)
bool run_rmsnorm_bwd(const void* x, const void* dy, int dy_dtype, const float* gain, const float* rstd, void* dx,
                     float* dgain, float* scratch, int64_t rows, int dim, bool mean, cudaStream_t st,
                     const void* dres = nullptr);
int64_t rmsnorm_bwd_scratch(int64_t rows, int dim);
bool run_rope(const void* in, void* out, const float* cs, int64_t rows, int seq, int nrot, int nall, int hd,
              bool backward, cudaStream_t st);
// AdamWT::step on one parameter (trainer.hpp:104-160), n % 4 == 0
void run_adamw(void* p, int p_dtype, const void* g, int g_dtype, float* m, float* v, int64_t n, double lr, double b1,
               double b2, double eps, double wd, double bc1, double bc2, cudaStream_t st);
// INT8 split-K: acc (+)= part (int64 sum of s32 slices); out = T(double(acc) * (double(*sa) * double(*sb)))
void run_acc_s64(const int* part, long long* acc, int64_t n, int first, cudaStream_t st);
void run_epi_s64(const long long* acc, const float* sa, const float* sb, void* out, int dtype, int64_t n,
                 cudaStream_t st);

}  // namespace halo_b200
