// halo_capi.cu — host layer: the C ABI of include/halo_b200.h and the HALO
// linear operator (HaloLinearLayerT, halo_linear.hpp:227-462) composed from
// the K1/K2/K3/K4 kernels.  Everything is stream-ordered; scales and absmax
// words live in a per-context device block, so a forward/backward pair never
// synchronises with the host.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <string>
#include <vector>

#include "../../include/halo_b200.h"
#include "common.cuh"
#include "halo_internal.h"

using namespace halo_b200;

namespace {

thread_local std::string g_err;

halo_status fail(halo_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

}  // namespace

// error text for the C ABI entries outside this file (peer.cu)
void halo_b200::set_last_error(const char* msg) { g_err = msg; }

namespace {

halo_status cuda_check(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(HALO_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
    return HALO_OK;
}

bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

// Resolve the Hadamard block for a transformed dimension d.
// had_block == 0: the reference's full-dimension transform (power-of-two
// dimensions only on this path; 2^n*12 / 2^n*20 bases are not built).
halo_status resolve_block(int64_t d, int64_t had_block, int64_t* B, const char* what) {
    if (had_block < 0) return fail(HALO_ERR_INVALID_ARGUMENT, std::string(what) + ": negative Hadamard block");
    const int64_t blk = had_block ? had_block : d;
    // 2^k, or 2^k * 12 / 2^k * 20 (the Paley bases, fwht_base.cu) up to 20480
    if (!is_pow2(blk) && !(base_dim_of(blk) && blk <= 20480))
        return fail(HALO_ERR_INVALID_ARGUMENT,
                    std::string(what) + ": Hadamard block " + std::to_string(blk) +
                        " is not 2^k, 12*2^k or 20*2^k (<= 20480) (hadamard.hpp:69-98)");
    if (d % blk != 0)
        return fail(HALO_ERR_INVALID_ARGUMENT, std::string(what) + ": Hadamard block " + std::to_string(blk) +
                                                   " does not divide dimension " + std::to_string(d));
    *B = blk;
    return HALO_OK;
}

// INT8, FP8 E4M3 and FP6 E3M2 (one code per byte, the E3M2 bits in 7:2:
// the tcgen05 kind::f8f6f4 operand form)
bool valid_format(int32_t f) {
    return f == HALO_FMT_INT8 || f == HALO_FMT_FP8_E4M3 || f == HALO_FMT_FP6_E3M2 || f == HALO_FMT_MXFP6_E3M2;
}
bool valid_gemm_format(int32_t f) { return valid_format(f); }
bool valid_dtype(int32_t d) { return d == HALO_DTYPE_F32 || d == HALO_DTYPE_BF16; }

// device scalar block: absmax words, scales, error flag
enum Slot { SX = 0, SW = 1, SEH = 2, SE = 3, SW2 = 4, SLOTS = 8 };
struct DevScalars {
    unsigned amax[SLOTS];
    float scale[SLOTS];
    unsigned err;
    unsigned pad[7];
};

struct Buffer {
    void* p = nullptr;
    size_t bytes = 0;
    halo_status ensure(size_t want) {
        if (want <= bytes) return HALO_OK;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        if (cudaMalloc(&p, want) != cudaSuccess) return fail(HALO_ERR_CUDA, "cudaMalloc failed");
        bytes = want;
        return HALO_OK;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <class T>
    T* as() const {
        return static_cast<T*>(p);
    }
};

// ---------------------------------------------------------------- profiler
// When enabled, every kernel launch of the layer is bracketed by CUDA events
// on its stream and tagged with its class and algorithmic work (bytes for
// the HBM-bound kernels, int ops for the GEMM).  halo_profile_read()
// synchronises and reduces.  Off by default: zero cost on the hot path.
struct ProfRec {
    int cls;
    double work;
    cudaEvent_t a, b;
};
struct Profiler {
    bool on = false;
    std::vector<ProfRec> recs;
    std::vector<cudaEvent_t> pool;
    std::mutex mu;
    cudaEvent_t ev() {
        if (!pool.empty()) {
            cudaEvent_t e = pool.back();
            pool.pop_back();
            return e;
        }
        cudaEvent_t e;
        cudaEventCreate(&e);
        return e;
    }
};
Profiler g_prof;

struct ProfScope {
    bool active;
    ProfRec r;
    cudaStream_t st;
    ProfScope(int cls, double work, cudaStream_t s) : active(g_prof.on), st(s) {
        if (!active) return;
        std::lock_guard<std::mutex> lk(g_prof.mu);
        r.cls = cls;
        r.work = work;
        r.a = g_prof.ev();
        r.b = g_prof.ev();
        cudaEventRecord(r.a, st);
    }
    ~ProfScope() {
        if (!active) return;
        cudaEventRecord(r.b, st);
        std::lock_guard<std::mutex> lk(g_prof.mu);
        g_prof.recs.push_back(r);
    }
};

enum ProfClass { PC_K1 = 0, PC_K2 = 1, PC_GEMM = 2, PC_K4 = 3, PC_GLUE = 4 };

int dt_bytes(int dt) { return dt == HALO_DTYPE_BF16 ? 2 : 4; }

}  // namespace

struct halo_ctx {
    bool valid = false;
    int64_t b = 0, m = 0, n = 0, b_pad = 0;
    bool xq_rotated = false, wq_rotated = false;
    int32_t fmt = 0;
    Buffer xq, wq, ehq, eq, wq2, scratch, gscratch;
    Buffer dev;  // DevScalars
    // Granularity::row: per-token X scales, per-output-channel W scales and
    // the per-row absmax scratch
    Buffer xs_rows, ws_rows, amax_rows;
    Buffer es_rows, ehs_rows;  // row-granularity backward: per-token E_Y / (H_b E_Y) scales
    Buffer mx_t, mx_ts;        // Granularity::mx backward: quantize(transpose(E_Y)) codes / block scales
    bool row_gran = false;
    int32_t gran = HALO_GRAN_TENSOR;
    const uint8_t* wq_codes = nullptr;  // ctx.wq (own buffer or the layer's qweight)
    const float* wq_scale = nullptr;
    const float* xq_scale = nullptr;
    const uint8_t* xq_borrow = nullptr;  // (XH)_Q shared from another context (halo_linear_forward_shared)
    int64_t had_block = 0;
    // halo_swiglu_backward_absmax: the absmax words of E_Y (SEH, SE) were
    // computed by the fused pass for this exact E_Y buffer and batch
    const void* e_amax_src = nullptr;
    int64_t e_amax_b = 0;
    bool wq_sharded = false;  // forward used the layer's sharded (WH)_Q
    // halo_swiglu_forward_absmax: the absmax word of (X H) (SX) was produced
    // with this X buffer (h) by the fused pass
    const void* x_amax_src = nullptr;
    int64_t x_amax_b = 0;
    // backward scratch (eq, ehq, scratch, gscratch, per-row / MX scale
    // scratch) may live in another context: contexts whose backwards run
    // one after another on one stream share one set (halo_ctx_share_scratch)
    halo_ctx* sowner = nullptr;
    halo_ctx* S() { return sowner ? sowner : this; }
    const uint8_t* xq_codes() const { return xq_borrow ? xq_borrow : xq.as<uint8_t>(); }
    DevScalars* d() const { return dev.as<DevScalars>(); }
    ~halo_ctx() {
        xq.release(); wq.release(); ehq.release(); eq.release(); wq2.release(); scratch.release();
        gscratch.release(); dev.release(); xs_rows.release(); ws_rows.release(); amax_rows.release(); es_rows.release(); ehs_rows.release();
        mx_t.release(); mx_ts.release();
    }
};

struct halo_linear {
    halo_scheme s;
    int64_t m = 0, n = 0;  // in_features, out_features
    const void* w = nullptr;
    int32_t w_dtype = HALO_DTYPE_BF16;
    const uint8_t* qcodes = nullptr;
    const float* qscale = nullptr;
    std::atomic<int64_t> cx{0}, cw{0}, ce{0};
    // PEFT: (WH)_Q frozen at construction (halo_linear.hpp:237-250)
    Buffer frozen, frozen_dev;
    // HQ-FSDP without the all-gather: (WH)_Q as row shards in place (local
    // or peer HBM), read by the GEMMs' TMA through per-shard maps
    bool sharded = false;
    Buffer shard_maps;
    ShardSpec shard_n{}, shard_k{};  // split along N (F GEMM) / along K (E GEMM)
    // HQ-FSDP gradient reduce-scatter fused into the G GEMM: fp32 partial
    // rows stored straight into the owners' receive buffers
    bool scatter = false;
    Buffer scatter_maps;
    ScatterSpec scatter_c{};
    ~halo_linear() {
        frozen.release();
        frozen_dev.release();
        shard_maps.release();
        scatter_maps.release();
    }
};

// The INT8 GEMM accumulates in s32 TMEM: exact while K*127^2 < 2^31, i.e.
// K <= 133,144.  The reference accumulates in int64 (quantize.hpp:358-371),
// so longer contractions -- the G GEMM over more than 131072 tokens -- run
// as K slices of raw s32 accumulators summed in int64, then the reference's
// double epilogue.  The slices need row offsets along K, i.e. MN-major
// operands (the G GEMM's layout); K-major operands that long are rejected.
constexpr int64_t kI8SliceK = 131072;

namespace {
struct SplitScratch {
    Buffer s32, s64, f32;
    ~SplitScratch() {
        s32.release();
        s64.release();
        f32.release();
    }
};
thread_local SplitScratch t_split;
}  // namespace

// returns as run_gemm; out_f32: epilogue into this fp32 buffer instead of out
static int gemm_i8_split(const uint8_t* A, const uint8_t* B, int64_t M, int64_t N, int64_t K, int a_kmajor,
                         int b_kmajor, const float* sa, const float* sb, void* out, int out_kind, cudaStream_t st) {
    if (a_kmajor || b_kmajor || out_kind == 2 || ShardScope::active()) return -1;
    const size_t mn = (size_t)M * (size_t)N;
    if (t_split.s32.ensure(mn * 4) != HALO_OK || t_split.s64.ensure(mn * 8) != HALO_OK) return (int)cudaErrorMemoryAllocation;
    for (int64_t k0 = 0; k0 < K; k0 += kI8SliceK) {
        const int64_t kc = K - k0 < kI8SliceK ? K - k0 : kI8SliceK;
        const int r = run_gemm(HALO_FMT_INT8, A + k0 * M, B + k0 * N, M, N, kc, 0, 0, sa, sb, t_split.s32.p, 2, st);
        if (r != 0) return r;
        run_acc_s64(t_split.s32.as<int>(), t_split.s64.as<long long>(), (int64_t)mn, k0 == 0, st);
    }
    run_epi_s64(t_split.s64.as<long long>(), sa, sb, out, out_kind == 1 ? HALO_DTYPE_BF16 : HALO_DTYPE_F32,
                (int64_t)mn, st);
    return 0;
}

static int prof_gemm(int fmt, const uint8_t* A, const uint8_t* B, int64_t M, int64_t N, int64_t K, int a_kmajor,
                     int b_kmajor, const float* sa, const float* sb, void* out, int out_kind, cudaStream_t st) {
    ProfScope ps(PC_GEMM, 2.0 * (double)M * (double)N * (double)K, st);
    if (fmt == HALO_FMT_INT8 && K > kI8SliceK)
        return gemm_i8_split(A, B, M, N, K, a_kmajor, b_kmajor, sa, sb, out, out_kind, st);
    return run_gemm(fmt, A, B, M, N, K, a_kmajor, b_kmajor, sa, sb, out, out_kind, st);
}

static int prof_gemm_x(int fmt, const uint8_t* A, const uint8_t* B, int64_t M, int64_t N, int64_t K, int a_kmajor,
                       int b_kmajor, const float* sa, const float* sb, void* out, int out_kind, int64_t xf_block,
                       int out_trans, int64_t n_valid, cudaStream_t st) {
    if (fmt == HALO_FMT_INT8 && K > kI8SliceK) {
        // sliced products into fp32, then the standalone right transform
        if (out_trans) return -1;
        if (t_split.f32.ensure((size_t)M * (size_t)N * 4) != HALO_OK) return (int)cudaErrorMemoryAllocation;
        {
            ProfScope ps(PC_GEMM, 2.0 * (double)M * (double)N * (double)K, st);
            const int r = gemm_i8_split(A, B, M, N, K, a_kmajor, b_kmajor, sa, sb, t_split.f32.p, 0, st);
            if (r != 0) return r;
        }
        ProfScope ps(PC_K4, (double)M * N * (4 + (out_kind == 1 ? 2 : 4)), st);
        run_rows(t_split.f32.p, HALO_DTYPE_F32, M, N, xf_block, 2, 0, nullptr, nullptr, nullptr, out,
                 out_kind == 1 ? HALO_DTYPE_BF16 : HALO_DTYPE_F32, nullptr, nullptr, st);
        return 0;
    }
    ProfScope ps(PC_GEMM, 2.0 * (double)M * (double)N * (double)K, st);
    int lb = 0;
    while ((int64_t(1) << lb) < xf_block) ++lb;
    return run_gemm_x(fmt, A, B, M, N, K, a_kmajor, b_kmajor, sa, sb, out, out_kind, lb, hadamard_norm(xf_block),
                      out_trans, n_valid, st);
}

// the GEMM epilogue can apply a block-B transform along its 256-column tile
static bool fusable_block(int64_t B) { return B >= 2 && B <= 256 && (B & (B - 1)) == 0; }

// HALO_FUSE_K4=0 keeps the un-rotation in separate K4 kernels (A/B runs)
static bool fuse_k4() {
    static const bool on = [] {
        const char* e = getenv("HALO_FUSE_K4");
        return !(e && e[0] == '0');
    }();
    return on;
}

// ================================================================= helpers

extern "C" int halo_abi_version(void) { return HALO_B200_ABI_VERSION; }
extern "C" const char* halo_last_error(void) { return g_err.c_str(); }

// hadamard.hpp:69-85
extern "C" int halo_is_supported_hadamard_dim(int64_t d) {
    if (d < 1) return 0;
    int64_t odd = d;
    int twos = 0;
    while (odd % 2 == 0) {
        odd /= 2;
        ++twos;
    }
    if (odd == 1) return 1;
    if ((odd == 3 || odd == 5) && twos >= 2) return 1;
    return 0;
}

// hadamard.hpp:87-93
extern "C" int64_t halo_next_supported_hadamard_dim(int64_t d) {
    if (d < 1) d = 1;
    while (!halo_is_supported_hadamard_dim(d)) ++d;
    return d;
}

// halo_linear.hpp:393-397: rows padded for the left transform; with a block
// the pad goes to the next multiple of the block.
extern "C" int64_t halo_padded_batch(int64_t b, int64_t had_block) {
    if (had_block > 0) return (b + had_block - 1) / had_block * had_block;
    return halo_next_supported_hadamard_dim(b);
}

static halo_status placement_from(const char* s, size_t len, halo_placement* p) {
    *p = halo_placement{0, 0, 0, 0};
    for (size_t i = 0; i < len; ++i) {
        switch (toupper((unsigned char)s[i])) {
        case 'L': p->left = 1; break;
        case 'M': p->middle = 1; break;
        case 'R': p->right = 1; break;
        case 'O': break;
        default: return fail(HALO_ERR_INVALID_ARGUMENT, "placement: unknown letter in '" + std::string(s, len) + "'");
        }
    }
    return HALO_OK;
}

// halo_linear.hpp:81-152
extern "C" halo_status halo_scheme_from_string(const char* id, int32_t format, int64_t had_block, halo_scheme* out) {
    if (!id || !out) return fail(HALO_ERR_INVALID_ARGUMENT, "scheme: null argument");
    if (!valid_format(format)) return fail(HALO_ERR_INVALID_ARGUMENT, "scheme: format must be int8, fp8_e4m3 or fp6_e3m2");
    halo_scheme s;
    std::memset(&s, 0, sizeof(s));
    s.format_x = s.format_w = s.format_e = format;
    s.quantize_f = s.quantize_e = s.quantize_g = 1;
    s.had_block = had_block;
    const std::string sid(id);
    if (sid == "halo0" || sid == "halo1" || sid == "halo2" || sid == "halo-peft") {
        if (sid != "halo0") {
            s.F.middle = 1;  // halo1: F:M, E:R, G:R  (:90-98)
            s.E.right = 1;
            s.G.right = 1;
        }
        if (sid == "halo2" || sid == "halo-peft") s.E.left = 1;  // (:100-106)
        if (sid == "halo-peft") s.peft = 1;
        std::strncpy(s.name, sid.c_str(), sizeof(s.name) - 1);
        *out = s;
        return HALO_OK;
    }
    size_t pos = 0;
    int seen = 0;
    while (pos < sid.size()) {
        size_t semi = sid.find(';', pos);
        const std::string part = sid.substr(pos, semi == std::string::npos ? std::string::npos : semi - pos);
        const size_t colon = part.find(':');
        if (colon != 1 || part.empty())
            return fail(HALO_ERR_INVALID_ARGUMENT, "scheme: expected 'F:..;E:..;G:..', got '" + sid + "'");
        halo_placement p;
        if (placement_from(part.c_str() + 2, part.size() - 2, &p) != HALO_OK) return HALO_ERR_INVALID_ARGUMENT;
        switch (toupper((unsigned char)part[0])) {
        case 'F': s.F = p; break;
        case 'E': s.E = p; break;
        case 'G': s.G = p; break;
        default: return fail(HALO_ERR_INVALID_ARGUMENT, "scheme: unknown matmul tag in '" + part + "'");
        }
        ++seen;
        pos = semi == std::string::npos ? sid.size() : semi + 1;
    }
    if (seen == 0) return fail(HALO_ERR_INVALID_ARGUMENT, "scheme: empty id");
    *out = s;
    return HALO_OK;
}

// ============================================================ primitives

static halo_status rotate_quantize_impl(const void* a, int32_t dt, int64_t rows, int64_t cols, int64_t B,
                                        bool rotate, int32_t fmt, const float* supplied, uint8_t* codes,
                                        unsigned* amax_word, float* scale_out, unsigned* err, cudaStream_t st,
                                        bool have_amax = false) {
    const double n = (double)rows * (double)cols;
    if (!supplied && !have_amax) {
        cudaMemsetAsync(amax_word, 0, sizeof(unsigned), st);
        ProfScope ps(PC_K1, 0.0, st);  // phase A: its bytes are booked on phase B
        if (rotate) run_rows(a, dt, rows, cols, B, 0, fmt, amax_word, nullptr, nullptr, nullptr, 0, err, nullptr, st);
        else run_plain(a, dt, rows * cols, 0, fmt, amax_word, nullptr, nullptr, err, nullptr, st);
    }
    // algorithmic bytes of the whole op: one read of the input + the codes
    ProfScope ps(PC_K1, n * (dt_bytes(dt) + 1), st);
    if (rotate) run_rows(a, dt, rows, cols, B, 1, fmt, amax_word, supplied, codes, nullptr, 0, err, scale_out, st);
    else run_plain(a, dt, rows * cols, 1, fmt, amax_word, supplied, codes, err, scale_out, st);
    return cuda_check("rotate_quantize");
}

namespace {
// device scratch words (absmax, scale, error flag) for the free-function
// entry points: one set per (host thread, stream), so calls on different
// streams never share an absmax word
struct FreeScratch {
    std::unordered_map<cudaStream_t, Buffer> dev, rows;
    ~FreeScratch() {
        for (auto& kv : dev) kv.second.release();
        for (auto& kv : rows) kv.second.release();
    }
};
thread_local FreeScratch t_scratch;
DevScalars* free_scalars(halo_stream_t stream) {
    Buffer& b = t_scratch.dev[(cudaStream_t)stream];
    if (b.ensure(sizeof(DevScalars)) != HALO_OK) return nullptr;
    return b.as<DevScalars>();
}
}  // namespace

extern "C" halo_status halo_rotate_quantize(const void* a, int32_t a_dtype, int64_t rows, int64_t cols,
                                            int64_t had_block, int32_t format, const float* supplied_scale,
                                            uint8_t* codes, float* scale_out, halo_stream_t stream) {
    if (format == HALO_FMT_MXFP6_E3M2)
        return fail(HALO_ERR_INVALID_ARGUMENT, "rotate_quantize: mxfp6_e3m2 requires mx granularity (quantize.hpp:249-250): "
                    "halo_rotate_quantize_mx");
    if (!a || !codes) return fail(HALO_ERR_INVALID_ARGUMENT, "rotate_quantize: null pointer");
    if (!valid_dtype(a_dtype) || !valid_format(format)) return fail(HALO_ERR_INVALID_ARGUMENT, "rotate_quantize: bad dtype/format");
    if (rows < 0 || cols <= 0 || cols % 16) return fail(HALO_ERR_INVALID_ARGUMENT, "rotate_quantize: cols must be a positive multiple of 16");
    if (rows == 0) return HALO_OK;
    int64_t B = 1;
    const bool rotate = had_block >= 0;
    if (rotate && resolve_block(cols, had_block, &B, "rotate_quantize") != HALO_OK) return HALO_ERR_INVALID_ARGUMENT;
    DevScalars* d = free_scalars(stream);
    if (!d) return HALO_ERR_CUDA;
    return rotate_quantize_impl(a, a_dtype, rows, cols, B, rotate, format, supplied_scale, codes, &d->amax[0],
                                scale_out, &d->err, (cudaStream_t)stream);
}

namespace {
__global__ void k_word_to_float(const unsigned* w, float* out) { *out = __uint_as_float(*w); }
}  // namespace

// Phase B only, under a given absmax (e.g. the HQ-FSDP absmax exchanged
// over the ranks): the scale is derived in-kernel exactly as from the
// layer's own phase A (compute_scales, quantize.hpp:134-160).
extern "C" halo_status halo_rotate_quantize_amax(const void* a, int32_t a_dtype, int64_t rows, int64_t cols,
                                                 int64_t had_block, int32_t format, const float* amax,
                                                 uint8_t* codes, float* scale_out, halo_stream_t stream) {
    if (format == HALO_FMT_MXFP6_E3M2)
        return fail(HALO_ERR_INVALID_ARGUMENT, "rotate_quantize_amax: mxfp6_e3m2 requires mx granularity (quantize.hpp:249-250): "
                    "halo_rotate_quantize_mx");
    if (!a || !codes || !amax) return fail(HALO_ERR_INVALID_ARGUMENT, "rotate_quantize_amax: null pointer");
    if (!valid_dtype(a_dtype) || !valid_format(format))
        return fail(HALO_ERR_INVALID_ARGUMENT, "rotate_quantize_amax: bad dtype/format");
    if (rows < 0 || cols <= 0 || cols % 16)
        return fail(HALO_ERR_INVALID_ARGUMENT, "rotate_quantize_amax: cols must be a positive multiple of 16");
    if (rows == 0) return HALO_OK;
    DevScalars* d = free_scalars(stream);
    if (!d) return HALO_ERR_CUDA;
    cudaStream_t st = (cudaStream_t)stream;
    // the absmax word is the float's bit pattern (non-negative)
    unsigned* word = reinterpret_cast<unsigned*>(const_cast<float*>(amax));
    ProfScope ps(PC_K1, (double)rows * cols * (dt_bytes(a_dtype) + 1), st);
    const float* sup = nullptr;
    if (had_block >= 0) {
        int64_t B;
        if (resolve_block(cols, had_block, &B, "rotate_quantize_amax") != HALO_OK) return HALO_ERR_INVALID_ARGUMENT;
        run_rows(a, a_dtype, rows, cols, B, 1, format, word, sup, codes, nullptr, 0, &d->err, scale_out, st);
    } else {
        run_plain(a, a_dtype, rows * cols, 1, format, word, sup, codes, &d->err, scale_out, st);
    }
    return cuda_check("rotate_quantize_amax");
}

extern "C" halo_status halo_rotate_absmax(const void* a, int32_t a_dtype, int64_t rows, int64_t cols,
                                          int64_t had_block, float* absmax_out, halo_stream_t stream) {
    if (!a || !absmax_out) return fail(HALO_ERR_INVALID_ARGUMENT, "rotate_absmax: null pointer");
    if (!valid_dtype(a_dtype) || cols <= 0 || cols % 16) return fail(HALO_ERR_INVALID_ARGUMENT, "rotate_absmax: bad arguments");
    DevScalars* d = free_scalars(stream);
    if (!d) return HALO_ERR_CUDA;
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(&d->amax[0], 0, sizeof(unsigned), st);
    if (rows > 0) {
        if (had_block >= 0) {
            int64_t B;
            if (resolve_block(cols, had_block, &B, "rotate_absmax") != HALO_OK) return HALO_ERR_INVALID_ARGUMENT;
            run_rows(a, a_dtype, rows, cols, B, 0, 0, &d->amax[0], nullptr, nullptr, nullptr, 0, &d->err, nullptr, st);
        } else {
            run_plain(a, a_dtype, rows * cols, 0, 0, &d->amax[0], nullptr, nullptr, &d->err, nullptr, st);
        }
    }
    k_word_to_float<<<1, 1, 0, st>>>(&d->amax[0], absmax_out);
    return cuda_check("rotate_absmax");
}

static halo_status left_quant_impl(const void* e, int32_t dt, int64_t b, int64_t n, int64_t B, int64_t b_pad,
                                   int32_t fmt, uint8_t* codes_rot, uint8_t* codes_plain, unsigned* amax_r,
                                   unsigned* amax_p, float* s_r, float* s_p, unsigned* err, cudaStream_t st,
                                   bool have_amax = false, bool transpose_base = true) {
    // transform_left_h (H E, halo_linear.hpp:399) or, for PEFT, transform_left (:449)
    BaseScope orient(transpose_base);
    if (!have_amax) {
        cudaMemsetAsync(amax_r, 0, sizeof(unsigned), st);
        cudaMemsetAsync(amax_p, 0, sizeof(unsigned), st);
        ProfScope ps(PC_K2, 0.0, st);
        run_cols(e, dt, b, b_pad, n, B, 0, fmt, amax_r, amax_p, nullptr, nullptr, nullptr, nullptr, nullptr, 0, err,
                 nullptr, nullptr, st);
    }
    // one read of E_Y, rotated codes (b_pad rows) and plain codes (b rows)
    ProfScope ps(PC_K2, (double)b * n * dt_bytes(dt) + (double)b_pad * n + (codes_plain ? (double)b * n : 0.0), st);
    run_cols(e, dt, b, b_pad, n, B, 1, fmt, amax_r, amax_p, nullptr, nullptr, codes_rot, codes_plain, nullptr, 0, err,
             s_r, s_p, st);
    return cuda_check("left_rotate_quantize");
}

extern "C" halo_status halo_left_rotate_quantize(const void* e, int32_t e_dtype, int64_t b, int64_t n,
                                                 int64_t had_block, int32_t format, uint8_t* codes_rot,
                                                 float* scale_rot, uint8_t* codes_plain, float* scale_plain,
                                                 halo_stream_t stream) {
    if (format == HALO_FMT_MXFP6_E3M2)
        return fail(HALO_ERR_INVALID_ARGUMENT, "left_rotate_quantize: mxfp6_e3m2 requires mx granularity (quantize.hpp:249-250): "
                    "halo_rotate_quantize_mx");
    if (!e || !codes_rot) return fail(HALO_ERR_INVALID_ARGUMENT, "left_rotate_quantize: null pointer");
    if (!valid_dtype(e_dtype) || !valid_format(format)) return fail(HALO_ERR_INVALID_ARGUMENT, "left_rotate_quantize: bad dtype/format");
    if (b <= 0 || n <= 0 || n % 16) return fail(HALO_ERR_INVALID_ARGUMENT, "left_rotate_quantize: n must be a positive multiple of 16");
    const int64_t b_pad = halo_padded_batch(b, had_block);
    int64_t B;
    if (resolve_block(b_pad, had_block, &B, "left_rotate_quantize") != HALO_OK) return HALO_ERR_INVALID_ARGUMENT;
    DevScalars* d = free_scalars(stream);
    if (!d) return HALO_ERR_CUDA;
    return left_quant_impl(e, e_dtype, b, n, B, b_pad, format, codes_rot, codes_plain, &d->amax[SEH], &d->amax[SE],
                           scale_rot, scale_plain, &d->err, (cudaStream_t)stream);
}

extern "C" halo_status halo_transform_right(const float* in, void* out, int32_t out_dtype, int64_t rows, int64_t cols,
                                            int64_t had_block, halo_stream_t stream) {
    if (!in || !out || !valid_dtype(out_dtype)) return fail(HALO_ERR_INVALID_ARGUMENT, "transform_right: bad arguments");
    if (cols <= 0 || cols % 16) return fail(HALO_ERR_INVALID_ARGUMENT, "transform_right: cols must be a multiple of 16");
    int64_t B;
    if (resolve_block(cols, had_block, &B, "transform_right") != HALO_OK) return HALO_ERR_INVALID_ARGUMENT;
    if (rows == 0) return HALO_OK;
    run_rows(in, HALO_DTYPE_F32, rows, cols, B, 2, 0, nullptr, nullptr, nullptr, out, out_dtype, nullptr, nullptr,
             (cudaStream_t)stream);
    return cuda_check("transform_right");
}

extern "C" halo_status halo_transform_left(const float* in, float* out, int64_t rows_pad, int64_t rows_out,
                                           int64_t cols, int64_t had_block, halo_stream_t stream) {
    if (!in || !out || rows_out > rows_pad) return fail(HALO_ERR_INVALID_ARGUMENT, "transform_left: bad arguments");
    if (cols <= 0 || cols % 8) return fail(HALO_ERR_INVALID_ARGUMENT, "transform_left: cols must be a multiple of 8");
    int64_t B;
    if (resolve_block(rows_pad, had_block, &B, "transform_left") != HALO_OK) return HALO_ERR_INVALID_ARGUMENT;
    run_cols(in, HALO_DTYPE_F32, rows_pad, rows_pad, cols, B, 2, 0, nullptr, nullptr, nullptr, nullptr, nullptr,
             nullptr, out, rows_out, nullptr, nullptr, nullptr, (cudaStream_t)stream);
    return cuda_check("transform_left");
}

extern "C" halo_status halo_qmatmul(int32_t format, const uint8_t* a, int32_t a_kmajor, const uint8_t* b,
                                    int32_t b_kmajor, int64_t M, int64_t N, int64_t K, const float* scale_a,
                                    const float* scale_b, void* out, int32_t out_kind, halo_stream_t stream) {
    if (!a || !b || !out || !scale_a || !scale_b) return fail(HALO_ERR_INVALID_ARGUMENT, "qmatmul: null pointer");
    if (!valid_gemm_format(format)) return fail(HALO_ERR_INVALID_ARGUMENT, "qmatmul: bad format");
    if (out_kind < 0 || out_kind > 2) return fail(HALO_ERR_INVALID_ARGUMENT, "qmatmul: bad out kind");
    if (format == HALO_FMT_INT8 && K > kI8SliceK && (out_kind == HALO_OUT_S32 || a_kmajor || b_kmajor))
        return fail(HALO_ERR_INVALID_ARGUMENT,
                    "qmatmul: INT8 with K > 131072 needs MN-major operands and a float output (s32 accumulators "
                    "would overflow; the product is summed in int64 over K slices)");
    const int r = prof_gemm(format, a, b, M, N, K, a_kmajor, b_kmajor, scale_a, scale_b, out, out_kind,
                           (cudaStream_t)stream);
    if (r == -1) return fail(HALO_ERR_INVALID_ARGUMENT, "qmatmul: unsupported shape (strides must be multiples of 16 B)");
    if (r == -2) return fail(HALO_ERR_CUDA, "qmatmul: cuTensorMapEncodeTiled failed");
    if (r != 0) return fail(HALO_ERR_CUDA, std::string("qmatmul: ") + cudaGetErrorString((cudaError_t)r));
    return HALO_OK;
}

extern "C" halo_status halo_qmatmul_rotate(int32_t format, const uint8_t* a, int32_t a_kmajor, const uint8_t* b,
                                           int32_t b_kmajor, int64_t M, int64_t N, int64_t K, const float* scale_a,
                                           const float* scale_b, void* out, int32_t out_kind, int64_t had_block,
                                           int32_t out_transposed, int64_t n_valid, halo_stream_t stream) {
    if (!a || !b || !out || !scale_a || !scale_b) return fail(HALO_ERR_INVALID_ARGUMENT, "qmatmul_rotate: null pointer");
    if (!valid_format(format)) return fail(HALO_ERR_INVALID_ARGUMENT, "qmatmul_rotate: bad format");
    if (out_kind != 0 && out_kind != 1) return fail(HALO_ERR_INVALID_ARGUMENT, "qmatmul_rotate: out kind must be f32 or bf16");
    int64_t B;
    if (resolve_block(N, had_block, &B, "qmatmul_rotate") != HALO_OK) return HALO_ERR_INVALID_ARGUMENT;
    if (!fusable_block(B))
        return fail(HALO_ERR_INVALID_ARGUMENT, "qmatmul_rotate: the fused transform needs a block of 2..256");
    if (n_valid < 0 || n_valid > N) return fail(HALO_ERR_INVALID_ARGUMENT, "qmatmul_rotate: bad n_valid");
    const int r = prof_gemm_x(format, a, b, M, N, K, a_kmajor, b_kmajor, scale_a, scale_b, out, out_kind, B,
                              out_transposed ? 1 : 0, out_transposed ? n_valid : N, (cudaStream_t)stream);
    if (r == -1) return fail(HALO_ERR_INVALID_ARGUMENT, "qmatmul_rotate: unsupported shape (strides must be multiples of 16 B)");
    if (r == -2) return fail(HALO_ERR_CUDA, "qmatmul_rotate: cuTensorMapEncodeTiled failed");
    if (r != 0) return fail(HALO_ERR_CUDA, std::string("qmatmul_rotate: ") + cudaGetErrorString((cudaError_t)r));
    return HALO_OK;
}

extern "C" halo_status halo_rotate_quantize_mx(const void* a, int32_t a_dtype, int64_t rows, int64_t cols,
                                               int64_t had_block, int32_t transpose_in, uint8_t* codes, float* scales,
                                               halo_stream_t stream) {
    if (!a || !codes || !scales) return fail(HALO_ERR_INVALID_ARGUMENT, "rotate_quantize_mx: null pointer");
    if (!valid_dtype(a_dtype) || rows < 0 || cols <= 0) return fail(HALO_ERR_INVALID_ARGUMENT, "rotate_quantize_mx: bad arguments");
    if (transpose_in && had_block >= 0)
        return fail(HALO_ERR_INVALID_ARGUMENT, "rotate_quantize_mx: a transposed view is not rotated (halo_linear.hpp:427-431)");
    if (rows == 0) return HALO_OK;
    cudaStream_t st = (cudaStream_t)stream;
    DevScalars* d = free_scalars(stream);
    if (!d) return HALO_ERR_CUDA;
    if (transpose_in) {  // quantize(transpose(A)): A is cols x rows row-major
        if (!mx_quantize(a_dtype, a, rows, cols, 1, rows, codes, scales, &d->err, st))
            return fail(HALO_ERR_CUDA, "rotate_quantize_mx: launch failed");
        return cuda_check("rotate_quantize_mx");
    }
    if (had_block < 0) {
        if (!mx_quantize(a_dtype, a, rows, cols, cols, 1, codes, scales, &d->err, st))
            return fail(HALO_ERR_CUDA, "rotate_quantize_mx: launch failed");
        return cuda_check("rotate_quantize_mx");
    }
    int64_t B;
    if (resolve_block(cols, had_block, &B, "rotate_quantize_mx") != HALO_OK) return HALO_ERR_INVALID_ARGUMENT;
    Buffer& tmp = t_scratch.rows[st];
    if (tmp.ensure((size_t)(rows * cols) * 2 * sizeof(float)) != HALO_OK) return HALO_ERR_CUDA;
    float* T0 = tmp.as<float>();
    float* T1 = T0 + rows * cols;
    pad_rows_f32(a, a_dtype, rows, rows, cols, T0, st);
    BaseScope h(false);
    run_rows(T0, HALO_DTYPE_F32, rows, cols, B, 2, 0, nullptr, nullptr, nullptr, T1, HALO_DTYPE_F32, nullptr, nullptr, st);
    if (!mx_quantize(HALO_DTYPE_F32, T1, rows, cols, cols, 1, codes, scales, &d->err, st))
        return fail(HALO_ERR_CUDA, "rotate_quantize_mx: launch failed");
    return cuda_check("rotate_quantize_mx");
}

extern "C" halo_status halo_rotate_quantize_rows(const void* a, int32_t a_dtype, int64_t rows, int64_t cols,
                                                 int64_t had_block, int32_t format, uint8_t* codes, float* scales_out,
                                                 halo_stream_t stream) {
    if (!a || !codes || !scales_out) return fail(HALO_ERR_INVALID_ARGUMENT, "rotate_quantize_rows: null pointer");
    if (!valid_dtype(a_dtype) || !valid_format(format) || format == HALO_FMT_FP6_E3M2 || format == HALO_FMT_MXFP6_E3M2)
        return fail(HALO_ERR_INVALID_ARGUMENT, "rotate_quantize_rows: bad dtype/format (int8 or fp8_e4m3)");
    if (rows < 0 || cols <= 0 || cols % 256)
        return fail(HALO_ERR_INVALID_ARGUMENT, "rotate_quantize_rows: cols must be a positive multiple of 256");
    if (rows == 0) return HALO_OK;
    int64_t B = 1;
    if (had_block >= 0 && resolve_block(cols, had_block, &B, "rotate_quantize_rows") != HALO_OK) return HALO_ERR_INVALID_ARGUMENT;
    if (B > 256) return fail(HALO_ERR_INVALID_ARGUMENT, "rotate_quantize_rows: Hadamard block must be <= 256");
    DevScalars* d = free_scalars(stream);
    Buffer& arows = t_scratch.rows[(cudaStream_t)stream];
    if (!d || arows.ensure((size_t)rows * sizeof(unsigned)) != HALO_OK) return HALO_ERR_CUDA;
    if (!rows_v3_per_row(format, a_dtype, a, rows, cols, B, arows.as<unsigned>(), scales_out, codes, &d->err,
                         (cudaStream_t)stream))
        return fail(HALO_ERR_INVALID_ARGUMENT, "rotate_quantize_rows: operands must be 32 B aligned");
    return cuda_check("rotate_quantize_rows");
}

extern "C" halo_status halo_qmatmul_scaled(int32_t format, const uint8_t* a, int32_t a_kmajor, const uint8_t* b,
                                           int32_t b_kmajor, int64_t M, int64_t N, int64_t K, const float* scale_a,
                                           int32_t a_per_row, const float* scale_b, int32_t b_per_row, void* out,
                                           int32_t out_kind, halo_stream_t stream) {
    if (!a || !b || !out || !scale_a || !scale_b) return fail(HALO_ERR_INVALID_ARGUMENT, "qmatmul_scaled: null pointer");
    if (!valid_format(format)) return fail(HALO_ERR_INVALID_ARGUMENT, "qmatmul_scaled: bad format");
    if (out_kind != 0 && out_kind != 1) return fail(HALO_ERR_INVALID_ARGUMENT, "qmatmul_scaled: out kind must be f32 or bf16");
    ProfScope ps(PC_GEMM, 2.0 * (double)M * (double)N * (double)K, (cudaStream_t)stream);
    const int r = run_gemm_v(format, a, b, M, N, K, a_kmajor, b_kmajor, a_per_row ? nullptr : scale_a,
                             a_per_row ? scale_a : nullptr, b_per_row ? nullptr : scale_b, b_per_row ? scale_b : nullptr,
                             out, out_kind, 0, 1.0f, 0, N, (cudaStream_t)stream);
    if (r == -1) return fail(HALO_ERR_INVALID_ARGUMENT, "qmatmul_scaled: unsupported shape (strides must be multiples of 16 B)");
    if (r == -2) return fail(HALO_ERR_CUDA, "qmatmul_scaled: cuTensorMapEncodeTiled failed");
    if (r != 0) return fail(HALO_ERR_CUDA, std::string("qmatmul_scaled: ") + cudaGetErrorString((cudaError_t)r));
    return HALO_OK;
}

// ================================================================= layer

static halo_status validate_scheme(const halo_scheme& s, int64_t m, int64_t n) {
    if (s.peft && !(s.F.middle && !s.F.left && !s.F.right && s.E.left && s.E.right && !s.E.middle))
        return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: peft fixes placements F:M and E:LR");  // :242-244
    if (s.peft && s.granularity != HALO_GRAN_TENSOR)
        return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: peft on the device path uses tensor granularity");
    if (!s.quantize_f || !s.quantize_e || !s.quantize_g)
        return fail(HALO_ERR_INVALID_ARGUMENT,
                    "halo layer: unquantized matmuls run in working precision in the reference; the device path has no full-precision fallback");
    if (s.granularity != HALO_GRAN_TENSOR && s.granularity != HALO_GRAN_ROW && s.granularity != HALO_GRAN_COLUMN &&
        s.granularity != HALO_GRAN_MX)
        return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: tensor, row, column and mx granularity are on the device path");
    if (s.granularity == HALO_GRAN_ROW && (m % 256 || n % 256 || (s.had_block ? s.had_block : m) > 256 ||
                                           !is_pow2(s.had_block ? s.had_block : m)))
        return fail(HALO_ERR_INVALID_ARGUMENT,
                    "halo layer: row granularity needs in_features % 256 == 0, out_features % 256 == 0 (the "
                    "per-row error quantizer of the backward) and a Hadamard block <= 256");
    if (!valid_format(s.format_x) || s.format_x != s.format_w || s.format_x != s.format_e)
        return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: X/W/E formats must agree and be int8, fp8_e4m3 or fp6_e3m2");
    // quantize.hpp:247-250: mx granularity <=> the mxfp6_e3m2 format
    if ((s.format_x == HALO_FMT_MXFP6_E3M2) != (s.granularity == HALO_GRAN_MX))
        return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: mxfp6_e3m2 requires mx granularity and vice versa (quantize.hpp:247-250)");
    if (s.granularity == HALO_GRAN_MX && (m % 32 || n % 32))
        return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: mx granularity needs in/out features % 32 == 0");
    if (s.format_x == HALO_FMT_FP6_E3M2 && s.granularity != HALO_GRAN_TENSOR)
        return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: fp6_e3m2 on the device path uses tensor granularity");
    if (s.F.left || s.F.right) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: placement_F must be O or M (apply_placement engine is not on the device path)");
    if (s.E.middle) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: placement_E with M is not on the device path");
    if (s.G.left || s.G.middle) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: placement_G must be O or R");
    if ((bool)s.G.right != (bool)s.F.middle)
        return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: G's rotation must match F's (X is not kept in full precision)");
    if (m <= 0 || n <= 0 || m % 16 || n % 16) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: in/out features must be positive multiples of 16");
    // validate_scheme_dims, halo_linear.hpp:343-348
    const bool needs_m = s.F.middle || s.E.right || s.G.right;
    if (needs_m) {
        if (!halo_is_supported_hadamard_dim(s.had_block ? s.had_block : m))
            return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: in_features is not a supported Hadamard dim");
        int64_t B;
        if (resolve_block(m, s.had_block, &B, "halo layer") != HALO_OK) return HALO_ERR_INVALID_ARGUMENT;
    }
    return HALO_OK;
}

// Granularity::row / ::column backwards (and ::column forwards) are the
// reference's dequantized double products (quantize.hpp:377-379), restated
// bit-exactly on the FP64 pipe by deq_gemm -- a full-precision matmul that
// north_star keeps off the contract path.  Opt-in only.
static std::atomic<int> g_allow_deq{0};
extern "C" halo_status halo_allow_dequantized_products(int32_t on) {
    g_allow_deq.store(on ? 1 : 0);
    return HALO_OK;
}

extern "C" halo_status halo_linear_create(const halo_scheme* scheme, const void* w, int32_t w_dtype,
                                          int64_t out_features, int64_t in_features, halo_linear** out) {
    if (!scheme || !out) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: null argument");
    if (!valid_dtype(w_dtype)) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: bad weight dtype");
    if (validate_scheme(*scheme, in_features, out_features) != HALO_OK) return HALO_ERR_INVALID_ARGUMENT;
    if (scheme->granularity != HALO_GRAN_TENSOR && !g_allow_deq.load())
        return fail(HALO_ERR_INVALID_ARGUMENT,
                    "halo layer: row / column granularity puts scales on a contracted dim, where the reference "
                    "multiplies dequantized values in double (quantize.hpp:377-379); that full-precision product "
                    "(deq_gemm, FP64 pipe, ~80x slower than the tensor-core path) is opt-in: "
                    "halo_allow_dequantized_products(1)");
    auto* l = new halo_linear();
    l->s = *scheme;
    l->m = in_features;
    l->n = out_features;
    l->w = w;
    l->w_dtype = w_dtype;
    if (scheme->peft) {
        // frozen_wq_ = quantize(transform_right(w, spec_m)) once (:248-249)
        if (!w) {
            delete l;
            return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: peft needs the weight at construction");
        }
        int64_t B;
        if (resolve_block(in_features, scheme->had_block, &B, "peft") != HALO_OK ||
            l->frozen.ensure((size_t)(out_features * in_features)) != HALO_OK ||
            l->frozen_dev.ensure(sizeof(DevScalars)) != HALO_OK) {
            delete l;
            return HALO_ERR_CUDA;
        }
        cudaMemset(l->frozen_dev.p, 0, sizeof(DevScalars));
        DevScalars* d = l->frozen_dev.as<DevScalars>();
        const halo_status r = rotate_quantize_impl(w, w_dtype, out_features, in_features, B, true, scheme->format_w,
                                                   nullptr, l->frozen.as<uint8_t>(), &d->amax[SW], &d->scale[SW],
                                                   &d->err, (cudaStream_t)0);
        if (r != HALO_OK || cudaStreamSynchronize((cudaStream_t)0) != cudaSuccess) {
            delete l;
            return r != HALO_OK ? r : fail(HALO_ERR_CUDA, "peft: freezing the weight failed");
        }
        l->qcodes = l->frozen.as<uint8_t>();
        l->qscale = &d->scale[SW];
        l->cw = 1;
    }
    *out = l;
    return HALO_OK;
}

extern "C" halo_status halo_linear_destroy(halo_linear* layer) {
    delete layer;
    return HALO_OK;
}

extern "C" halo_status halo_linear_set_weight(halo_linear* l, const void* w, int32_t w_dtype) {
    if (!l || !valid_dtype(w_dtype)) return fail(HALO_ERR_INVALID_ARGUMENT, "set_weight: bad arguments");
    l->w = w;
    l->w_dtype = w_dtype;
    return HALO_OK;
}

extern "C" halo_status halo_linear_set_qweight(halo_linear* l, const uint8_t* codes, const float* scale) {
    if (!l) return fail(HALO_ERR_INVALID_ARGUMENT, "set_qweight: null layer");
    if (l->s.peft) return fail(HALO_ERR_INVALID_ARGUMENT, "set_qweight: a peft layer's weight codes are frozen");
    if (codes && !scale) return fail(HALO_ERR_INVALID_ARGUMENT, "set_qweight: codes without a scale");
    l->qcodes = codes;
    l->qscale = scale;
    l->sharded = false;
    return HALO_OK;
}

extern "C" halo_status halo_linear_set_qweight_sharded(halo_linear* l, const uint8_t* const* parts, int32_t n_parts,
                                                       const float* scale) {
    if (!l) return fail(HALO_ERR_INVALID_ARGUMENT, "set_qweight_sharded: null layer");
    if (l->s.peft) return fail(HALO_ERR_INVALID_ARGUMENT, "set_qweight_sharded: a peft layer's weight codes are frozen");
    if (!parts || n_parts <= 0) {
        l->sharded = false;
        l->qcodes = nullptr;
        l->qscale = nullptr;
        return HALO_OK;
    }
    if (!scale) return fail(HALO_ERR_INVALID_ARGUMENT, "set_qweight_sharded: codes without a scale");
    if (l->s.granularity == HALO_GRAN_ROW)
        return fail(HALO_ERR_INVALID_ARGUMENT, "set_qweight_sharded: row granularity keeps per-channel scales local");
    if (n_parts > 64 || l->n % n_parts)
        return fail(HALO_ERR_INVALID_ARGUMENT, "set_qweight_sharded: out_features must split evenly into the parts");
    const int64_t len = l->n / n_parts;
    // the F GEMM's 256-row N tiles and the E GEMM's 128-deep k-blocks must
    // each fall inside one part; TMA rows are m bytes (a multiple of 16)
    if (len % 256 || l->m % 16)
        return fail(HALO_ERR_INVALID_ARGUMENT,
                    "set_qweight_sharded: rows per part must be a multiple of 256 and in_features of 16");
    for (int i = 0; i < n_parts; ++i)
        if (!parts[i] || (uintptr_t)parts[i] % 16)
            return fail(HALO_ERR_INVALID_ARGUMENT, "set_qweight_sharded: parts must be 16 B aligned device pointers");
    std::vector<CUtensorMap> maps((size_t)n_parts);
    if (!encode_shard_maps(parts, n_parts, l->m, len, maps.data()))
        return fail(HALO_ERR_INVALID_ARGUMENT, "set_qweight_sharded: tensor map encoding failed");
    if (l->shard_maps.ensure(maps.size() * sizeof(CUtensorMap)) != HALO_OK) return HALO_ERR_CUDA;
    if (cudaMemcpy(l->shard_maps.p, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice) !=
        cudaSuccess)
        return fail(HALO_ERR_CUDA, "set_qweight_sharded: map upload failed");
    l->shard_n = ShardSpec{l->shard_maps.as<CUtensorMap>(), maps[0], (int)n_parts, len, 0};
    l->shard_k = ShardSpec{l->shard_maps.as<CUtensorMap>(), maps[0], (int)n_parts, len, 1};
    l->sharded = true;
    l->qcodes = nullptr;
    l->qscale = scale;
    return HALO_OK;
}

extern "C" halo_status halo_linear_set_grad_scatter(halo_linear* l, void* const* recv, int32_t parts, int32_t rank) {
    if (!l) return fail(HALO_ERR_INVALID_ARGUMENT, "set_grad_scatter: null layer");
    if (!recv || parts <= 0) {
        l->scatter = false;
        return HALO_OK;
    }
    if (parts > 64 || rank < 0 || rank >= parts || l->n % parts || (l->n / parts) % 256 || l->m % 4)
        return fail(HALO_ERR_INVALID_ARGUMENT,
                    "set_grad_scatter: out_features must split into parts of a multiple of 256 rows");
    for (int i = 0; i < parts; ++i)
        if (!recv[i] || (uintptr_t)recv[i] % 16)
            return fail(HALO_ERR_INVALID_ARGUMENT, "set_grad_scatter: receive buffers must be 16 B aligned");
    std::vector<CUtensorMap> maps((size_t)parts);
    const int64_t len = l->n / parts;
    if (!encode_scatter_maps(recv, parts, rank, len, l->m, maps.data()))
        return fail(HALO_ERR_INVALID_ARGUMENT, "set_grad_scatter: tensor map encoding failed");
    if (l->scatter_maps.ensure(maps.size() * sizeof(CUtensorMap)) != HALO_OK) return HALO_ERR_CUDA;
    if (cudaMemcpy(l->scatter_maps.p, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice) !=
        cudaSuccess)
        return fail(HALO_ERR_CUDA, "set_grad_scatter: map upload failed");
    l->scatter_c = ScatterSpec{l->scatter_maps.as<CUtensorMap>(), maps[0], (int)parts, len};
    l->scatter = true;
    return HALO_OK;
}

extern "C" halo_status halo_reduce_scatter_shard(const float* recv, int32_t world, int64_t rows, int64_t cols,
                                                 void* out, int32_t out_dtype, halo_stream_t stream) {
    if (!recv || !out || world < 1 || rows <= 0 || cols <= 0 || !valid_dtype(out_dtype) || (rows * cols) % 4)
        return fail(HALO_ERR_INVALID_ARGUMENT, "reduce_scatter_shard: bad argument");
    ProfScope ps(PC_GLUE, (double)rows * cols * (4.0 * world + dt_bytes(out_dtype)), (cudaStream_t)stream);
    run_rank_mean(recv, world, rows * cols, out, out_dtype, (cudaStream_t)stream);
    return cuda_check("reduce_scatter_shard");
}

extern "C" halo_status halo_ctx_create(halo_ctx** out) {
    if (!out) return fail(HALO_ERR_INVALID_ARGUMENT, "ctx: null");
    auto* c = new halo_ctx();
    if (c->dev.ensure(sizeof(DevScalars)) != HALO_OK) {
        delete c;
        return HALO_ERR_CUDA;
    }
    cudaMemset(c->dev.p, 0, sizeof(DevScalars));
    *out = c;
    return HALO_OK;
}

extern "C" halo_status halo_ctx_destroy(halo_ctx* ctx) {
    delete ctx;
    return HALO_OK;
}

// weight operand rotated as requested (weight_operand, halo_linear.hpp:352-358)
static halo_status quantize_weight(halo_linear* l, halo_ctx* c, bool rotated, Buffer& dst, int slot,
                                   const uint8_t** codes, const float** scale, cudaStream_t st) {
    if (!l->w) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: no weight set");
    if (dst.ensure((size_t)(l->n * l->m)) != HALO_OK) return HALO_ERR_CUDA;
    int64_t B = 1;
    if (rotated && resolve_block(l->m, l->s.had_block, &B, "weight") != HALO_OK) return HALO_ERR_INVALID_ARGUMENT;
    DevScalars* d = c->d();
    const halo_status r = rotate_quantize_impl(l->w, l->w_dtype, l->n, l->m, B, rotated, l->s.format_w, nullptr,
                                               dst.as<uint8_t>(), &d->amax[slot], &d->scale[slot], &d->err, st);
    if (r != HALO_OK) return r;
    ++l->cw;
    *codes = dst.as<uint8_t>();
    *scale = &d->scale[slot];
    return HALO_OK;
}

static void finish_right(const float* P, void* out, int32_t dtype, int64_t rows, int64_t cols, int64_t B, bool rotate,
                         cudaStream_t st, const void* add = nullptr, bool* add_used = nullptr);

extern "C" halo_status halo_linear_forward(halo_linear* l, const void* x, int32_t x_dtype, int64_t b, void* y,
                                           int32_t y_dtype, halo_ctx* c, halo_stream_t stream) {
    if (!l || !x || !y || !c) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: null argument");
    if (!valid_dtype(x_dtype) || !valid_dtype(y_dtype)) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: bad dtype");
    if (b <= 0) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: empty batch");
    cudaStream_t st = (cudaStream_t)stream;
    const halo_scheme& s = l->s;
    const bool rot = s.F.middle;
    // ctx = SavedContextT{}  (:270-273)
    c->valid = false;
    c->e_amax_src = nullptr;
    c->b = b;
    c->m = l->m;
    c->n = l->n;
    c->fmt = s.format_x;
    c->xq_rotated = c->wq_rotated = rot;
    if (c->xq.ensure((size_t)(b * l->m)) != HALO_OK) return HALO_ERR_CUDA;
    DevScalars* d = c->d();
    int64_t B = 1;
    if (rot && resolve_block(l->m, s.had_block, &B, "forward") != HALO_OK) return HALO_ERR_INVALID_ARGUMENT;
    c->row_gran = s.granularity == HALO_GRAN_ROW;
    c->gran = s.granularity;
    c->xq_borrow = nullptr;
    c->had_block = s.had_block;
    if (s.granularity == HALO_GRAN_MX) {
        // NumericFormat::MxFp6E3M2 under Granularity::mx (quantize.hpp:224-232,
        // 247-250): 1 x 32 power-of-two block scales along in_features, on
        // F's contracted dim -- Y is qmatmul's dequantized double product
        // (:377-379), restated bit-exactly by deq_gemm
        if (l->qcodes || l->sharded)
            return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: mx granularity with installed qweight codes");
        c->wq_sharded = false;
        const int64_t m = l->m, n = l->n, nb = m / 32, rmax = b > n ? b : n;
        const int64_t tmp = (rmax * m > b * n ? rmax * m : b * n) * (int64_t)sizeof(float);
        if (c->xs_rows.ensure((size_t)(b * nb) * sizeof(float)) != HALO_OK ||
            c->ws_rows.ensure((size_t)(n * nb) * sizeof(float)) != HALO_OK || c->wq.ensure((size_t)(n * m)) != HALO_OK ||
            c->S()->gscratch.ensure((size_t)tmp) != HALO_OK || c->S()->scratch.ensure((size_t)(rmax * m) * sizeof(float)) != HALO_OK)
            return HALO_ERR_CUDA;
        // quantize([A H], mxfp6, mx) (:292-297)
        auto quant_side = [&](const void* src, int32_t dt, int64_t rows, uint8_t* codes, float* scales) -> bool {
            if (rot) {
                float* T0 = c->S()->gscratch.as<float>();
                float* T1 = c->S()->scratch.as<float>();
                pad_rows_f32(src, dt, rows, rows, m, T0, st);
                BaseScope h(false);  // transform_right (H)
                run_rows(T0, HALO_DTYPE_F32, rows, m, B, 2, 0, nullptr, nullptr, nullptr, T1, HALO_DTYPE_F32, nullptr,
                         nullptr, st);
                return mx_quantize(HALO_DTYPE_F32, T1, rows, m, m, 1, codes, scales, &d->err, st);
            }
            return mx_quantize(dt, src, rows, m, m, 1, codes, scales, &d->err, st);
        };
        {
            ProfScope ps(PC_K1, (double)b * m * (dt_bytes(x_dtype) + 1), st);
            if (!quant_side(x, x_dtype, b, c->xq.as<uint8_t>(), c->xs_rows.as<float>()))
                return fail(HALO_ERR_CUDA, "forward: mx quantization failed");
        }
        ++l->cx;
        {
            ProfScope ps(PC_K1, (double)n * m * (dt_bytes(l->w_dtype) + 1), st);
            if (!quant_side(l->w, l->w_dtype, n, c->wq.as<uint8_t>(), c->ws_rows.as<float>()))
                return fail(HALO_ERR_CUDA, "forward: mx quantization failed");
        }
        ++l->cw;
        c->wq_codes = c->wq.as<uint8_t>();
        c->wq_scale = c->ws_rows.as<float>();
        c->xq_scale = c->xs_rows.as<float>();
        float* P = c->S()->gscratch.as<float>();
        {
            // A = xq (i = token, k = in): scale [i][k >> 5]; B = wq^T (k = in,
            // j = out): scale [j][k >> 5]
            ProfScope ps(PC_GEMM, 2.0 * (double)b * n * m, st);
            if (!deq_gemm(s.format_x, c->xq.as<uint8_t>(), c->xs_rows.as<float>(), m, 1, nb, 1, c->wq_codes,
                          c->wq_scale, 1, m, 1, nb, P, b, n, m, n, st, 0, 5, 5, 0))
                return fail(HALO_ERR_CUDA, "forward: mx product launch failed");
        }
        finish_right(P, y, y_dtype, b, n, 1, false, st);
        c->valid = true;
        return cuda_check("forward");
    }
    if (s.granularity == HALO_GRAN_COLUMN) {
        // Granularity::column: X's and W's scales both sit on F's contracted
        // dim, so Y is qmatmul's dequantized double product
        // (quantize.hpp:377-379), restated bit-exactly by deq_gemm
        if (l->qcodes || l->sharded)
            return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: column granularity with installed qweight codes");
        c->wq_sharded = false;
        const int64_t m = l->m, n = l->n, rmax = b > n ? b : n;
        const int64_t tmp = (rmax * m > b * n ? rmax * m : b * n) * (int64_t)sizeof(float);
        if (c->xs_rows.ensure((size_t)m * sizeof(float)) != HALO_OK || c->ws_rows.ensure((size_t)m * sizeof(float)) != HALO_OK ||
            c->amax_rows.ensure((size_t)m * sizeof(unsigned)) != HALO_OK || c->wq.ensure((size_t)(n * m)) != HALO_OK ||
            c->S()->gscratch.ensure((size_t)tmp) != HALO_OK || c->S()->scratch.ensure((size_t)(rmax * m) * sizeof(float)) != HALO_OK)
            return HALO_ERR_CUDA;
        // quantize([A H], fmt, column) (:292-297)
        auto quant_side = [&](const void* src, int32_t dt, int64_t rows, uint8_t* codes, float* scales) -> bool {
            const void* q = src;
            int32_t qdt = dt;
            if (rot) {
                float* T0 = c->S()->gscratch.as<float>();
                float* T1 = c->S()->scratch.as<float>();
                pad_rows_f32(src, dt, rows, rows, m, T0, st);
                BaseScope h(false);  // transform_right (H)
                run_rows(T0, HALO_DTYPE_F32, rows, m, B, 2, 0, nullptr, nullptr, nullptr, T1, HALO_DTYPE_F32, nullptr,
                         nullptr, st);
                q = T1;
                qdt = HALO_DTYPE_F32;
            }
            return col_quantize(s.format_x, qdt, q, rows, m, c->amax_rows.as<unsigned>(), scales, codes, &d->err, st);
        };
        {
            ProfScope ps(PC_K1, (double)b * l->m * (dt_bytes(x_dtype) + 1), st);
            if (!quant_side(x, x_dtype, b, c->xq.as<uint8_t>(), c->xs_rows.as<float>()))
                return fail(HALO_ERR_INVALID_ARGUMENT, "forward: column-granularity quantization failed");
        }
        ++l->cx;
        {
            ProfScope ps(PC_K1, (double)n * m * (dt_bytes(l->w_dtype) + 1), st);
            if (!quant_side(l->w, l->w_dtype, n, c->wq.as<uint8_t>(), c->ws_rows.as<float>()))
                return fail(HALO_ERR_INVALID_ARGUMENT, "forward: column-granularity quantization failed");
        }
        ++l->cw;
        c->wq_codes = c->wq.as<uint8_t>();
        c->wq_scale = c->ws_rows.as<float>();
        c->xq_scale = c->xs_rows.as<float>();
        float* P = c->S()->gscratch.as<float>();
        {
            ProfScope ps(PC_GEMM, 2.0 * (double)b * n * m, st);
            if (!deq_gemm(s.format_x, c->xq.as<uint8_t>(), c->xs_rows.as<float>(), m, 1, 0, 1, c->wq_codes,
                          c->wq_scale, 1, m, 1, 0, P, b, n, m, n, st))
                return fail(HALO_ERR_CUDA, "forward: column-granularity product launch failed");
        }
        finish_right(P, y, y_dtype, b, n, 1, false, st);
        c->valid = true;
        return cuda_check("forward");
    }
    if (c->row_gran) {
        // Granularity::row (quantize.hpp:73-132): X per token, W per output
        // channel -- both on non-contracted dims of F, so the integer GEMM
        // stays exact and the epilogue applies sx[i] * sw[j]
        if (l->qcodes || l->sharded)
            return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: row granularity with installed qweight codes");
        c->wq_sharded = false;
        const int64_t mx = b > l->n ? b : l->n;
        if (c->xs_rows.ensure((size_t)b * sizeof(float)) != HALO_OK || c->wq.ensure((size_t)(l->n * l->m)) != HALO_OK ||
            c->ws_rows.ensure((size_t)l->n * sizeof(float)) != HALO_OK ||
            c->amax_rows.ensure((size_t)mx * sizeof(unsigned)) != HALO_OK)
            return HALO_ERR_CUDA;
        {
            ProfScope ps(PC_K1, (double)b * l->m * (dt_bytes(x_dtype) + 1), st);
            if (!rows_v3_per_row(s.format_x, x_dtype, x, b, l->m, B, c->amax_rows.as<unsigned>(), c->xs_rows.as<float>(),
                                 c->xq.as<uint8_t>(), &d->err, st))
                return fail(HALO_ERR_INVALID_ARGUMENT, "forward: row-granularity operands must be 32 B aligned");
        }
        ++l->cx;
        {
            ProfScope ps(PC_K1, (double)l->n * l->m * (dt_bytes(l->w_dtype) + 1), st);
            if (!rows_v3_per_row(s.format_w, l->w_dtype, l->w, l->n, l->m, B, c->amax_rows.as<unsigned>(),
                                 c->ws_rows.as<float>(), c->wq.as<uint8_t>(), &d->err, st))
                return fail(HALO_ERR_INVALID_ARGUMENT, "forward: row-granularity operands must be 32 B aligned");
        }
        ++l->cw;
        c->wq_codes = c->wq.as<uint8_t>();
        c->wq_scale = c->ws_rows.as<float>();
        c->xq_scale = c->xs_rows.as<float>();
        ProfScope ps(PC_GEMM, 2.0 * (double)b * l->n * l->m, st);
        const int gr = run_gemm_v(s.format_x, c->xq.as<uint8_t>(), c->wq_codes, b, l->n, l->m, 1, 1, nullptr,
                                  c->xs_rows.as<float>(), nullptr, c->ws_rows.as<float>(), y,
                                  y_dtype == HALO_DTYPE_F32 ? 0 : 1, 0, 1.0f, 0, l->n, st);
        if (gr != 0) return fail(gr == -1 ? HALO_ERR_INVALID_ARGUMENT : HALO_ERR_CUDA, "forward: GEMM launch failed");
        c->valid = true;
        return cuda_check("forward");
    }
    c->xq_scale = &d->scale[SX];
    // ctx.xq = quantize(XH)  (:292-294)
    // phase A already done by halo_swiglu_forward_absmax for this exact X
    const bool have_amax = c->x_amax_src == x && c->x_amax_b == b && x_dtype == HALO_DTYPE_BF16 && rot && B == 256;
    c->x_amax_src = nullptr;
    halo_status r = rotate_quantize_impl(x, x_dtype, b, l->m, B, rot, s.format_x, nullptr, c->xq.as<uint8_t>(),
                                         &d->amax[SX], &d->scale[SX], &d->err, st, have_amax);
    if (r != HALO_OK) return r;
    ++l->cx;
    // ctx.wq = quantize(WH)  (:295-297), or the gathered / frozen / sharded codes
    c->wq_sharded = l->sharded;
    if (l->sharded) {
        c->wq_codes = nullptr;  // read in place by the GEMM (ShardScope)
        c->wq_scale = l->qscale;
    } else if (l->qcodes) {
        c->wq_codes = l->qcodes;
        c->wq_scale = l->qscale;
    } else {
        r = quantize_weight(l, c, rot, c->wq, SW, &c->wq_codes, &c->wq_scale, st);
        if (r != HALO_OK) return r;
    }
    // Y = qmatmul(xq, wq, transpose_b=true)  (:299)
    ShardScope shards(nullptr, l->sharded ? &l->shard_n : nullptr);
    const int gr = prof_gemm(s.format_x, c->xq.as<uint8_t>(), c->wq_codes, b, l->n, l->m, 1, 1, &d->scale[SX],
                            c->wq_scale, y, y_dtype == HALO_DTYPE_F32 ? 0 : 1, st);
    if (gr != 0) return fail(gr == -1 ? HALO_ERR_INVALID_ARGUMENT : HALO_ERR_CUDA, "forward: GEMM launch failed");
    c->valid = true;
    return cuda_check("forward");
}

// Forward that reuses another context's (XH)_Q: two layers fed the same X
// under the same quantizer (Llama gate/up projections) quantize it once.
// The reference quantizes per layer (halo_linear.hpp:292-294); the codes are
// identical, so results are unchanged and the input counter is not bumped.
extern "C" halo_status halo_linear_forward_shared(halo_linear* l, const halo_ctx* src, halo_ctx* c, void* y,
                                                  int32_t y_dtype, halo_stream_t stream) {
    if (!l || !src || !c || !y) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: null argument");
    if (src == c) return fail(HALO_ERR_INVALID_ARGUMENT, "forward_shared: source and target context are the same");
    if (!src->valid) return fail(HALO_ERR_INVALID_ARGUMENT, "forward_shared: source context has no forward");
    if (!valid_dtype(y_dtype)) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: bad dtype");
    const halo_scheme& s = l->s;
    if (s.granularity == HALO_GRAN_COLUMN || src->gran == HALO_GRAN_COLUMN)
        return fail(HALO_ERR_INVALID_ARGUMENT, "forward_shared: column granularity is not shared");
    if (src->m != l->m || src->fmt != s.format_x || src->xq_rotated != (bool)s.F.middle ||
        src->row_gran != (s.granularity == HALO_GRAN_ROW) || src->had_block != s.had_block)
        return fail(HALO_ERR_INVALID_ARGUMENT, "forward_shared: the source context's X quantizer differs from this layer's");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t b = src->b;
    c->valid = false;
    c->e_amax_src = nullptr;
    c->b = b;
    c->m = l->m;
    c->n = l->n;
    c->fmt = s.format_x;
    c->xq_rotated = c->wq_rotated = s.F.middle;
    c->row_gran = src->row_gran;
    c->gran = src->gran;
    c->had_block = s.had_block;
    c->xq_borrow = src->xq_codes();
    c->xq_scale = src->xq_scale;
    DevScalars* d = c->d();
    if (c->row_gran) {
        if (l->qcodes || l->sharded)
            return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: row granularity with installed qweight codes");
        c->wq_sharded = false;
        int64_t B = 1;
        if (s.F.middle && resolve_block(l->m, s.had_block, &B, "forward") != HALO_OK) return HALO_ERR_INVALID_ARGUMENT;
        if (c->wq.ensure((size_t)(l->n * l->m)) != HALO_OK || c->ws_rows.ensure((size_t)l->n * sizeof(float)) != HALO_OK ||
            c->amax_rows.ensure((size_t)l->n * sizeof(unsigned)) != HALO_OK)
            return HALO_ERR_CUDA;
        {
            ProfScope ps(PC_K1, (double)l->n * l->m * (dt_bytes(l->w_dtype) + 1), st);
            if (!rows_v3_per_row(s.format_w, l->w_dtype, l->w, l->n, l->m, B, c->amax_rows.as<unsigned>(),
                                 c->ws_rows.as<float>(), c->wq.as<uint8_t>(), &d->err, st))
                return fail(HALO_ERR_INVALID_ARGUMENT, "forward: row-granularity operands must be 32 B aligned");
        }
        ++l->cw;
        c->wq_codes = c->wq.as<uint8_t>();
        c->wq_scale = c->ws_rows.as<float>();
        ProfScope ps(PC_GEMM, 2.0 * (double)b * l->n * l->m, st);
        const int gr = run_gemm_v(s.format_x, c->xq_codes(), c->wq_codes, b, l->n, l->m, 1, 1, nullptr, c->xq_scale,
                                  nullptr, c->wq_scale, y, y_dtype == HALO_DTYPE_F32 ? 0 : 1, 0, 1.0f, 0, l->n, st);
        if (gr != 0) return fail(gr == -1 ? HALO_ERR_INVALID_ARGUMENT : HALO_ERR_CUDA, "forward: GEMM launch failed");
        c->valid = true;
        return cuda_check("forward_shared");
    }
    c->wq_sharded = l->sharded;
    if (l->sharded) {
        c->wq_codes = nullptr;
        c->wq_scale = l->qscale;
    } else if (l->qcodes) {
        c->wq_codes = l->qcodes;
        c->wq_scale = l->qscale;
    } else {
        const halo_status r = quantize_weight(l, c, s.F.middle, c->wq, SW, &c->wq_codes, &c->wq_scale, st);
        if (r != HALO_OK) return r;
    }
    ShardScope shards(nullptr, l->sharded ? &l->shard_n : nullptr);
    const int gr = prof_gemm(s.format_x, c->xq_codes(), c->wq_codes, b, l->n, l->m, 1, 1, c->xq_scale, c->wq_scale, y,
                             y_dtype == HALO_DTYPE_F32 ? 0 : 1, st);
    if (gr != 0) return fail(gr == -1 ? HALO_ERR_INVALID_ARGUMENT : HALO_ERR_CUDA, "forward: GEMM launch failed");
    c->valid = true;
    return cuda_check("forward_shared");
}

extern "C" halo_status halo_linear_forward_shared_swiglu(halo_linear* l, const halo_ctx* src, halo_ctx* c,
                                                         const void* g, void* u, void* h, halo_stream_t stream) {
    if (!g || !h || !u) return fail(HALO_ERR_INVALID_ARGUMENT, "forward_shared_swiglu: null argument");
    if (l && (l->n % 256 || (uintptr_t)g % 16 || (uintptr_t)u % 16 || (uintptr_t)h % 16))
        return fail(HALO_ERR_INVALID_ARGUMENT, "forward_shared_swiglu: out_features % 256 and 16 B alignment required");
    GluScope glu(g, h);
    const halo_status r = halo_linear_forward_shared(l, src, c, u, HALO_DTYPE_BF16, stream);
    if (r != HALO_OK) return r;
    if (!GluScope::used()) {
        c->valid = false;
        return fail(HALO_ERR_INVALID_ARGUMENT, "forward_shared_swiglu: the GEMM did not run the SwiGLU epilogue");
    }
    return HALO_OK;
}

extern "C" halo_status halo_linear_forward_residual(halo_linear* l, const void* x, int32_t x_dtype, int64_t b,
                                                    const void* res, void* y, halo_ctx* c, halo_stream_t stream) {
    if (!res || !y) return fail(HALO_ERR_INVALID_ARGUMENT, "forward_residual: null argument");
    if (l && (l->n % 256 || (uintptr_t)res % 16 || (uintptr_t)y % 16))
        return fail(HALO_ERR_INVALID_ARGUMENT, "forward_residual: out_features % 256 and 16 B alignment required");
    GluScope glu(res, nullptr);
    const halo_status r = halo_linear_forward(l, x, x_dtype, b, y, HALO_DTYPE_BF16, c, stream);
    if (r != HALO_OK) return r;
    if (!GluScope::used()) {
        c->valid = false;
        return fail(HALO_ERR_INVALID_ARGUMENT, "forward_residual: the GEMM did not run the residual epilogue");
    }
    return HALO_OK;
}

// halo_linear_backward_acc: a bf16 addend for the E path of this thread's
// next halo_linear_backward (e_x = add + E_X), fused when the K4 kernel can
namespace {
thread_local const void* t_ex_add = nullptr;
thread_local bool t_ex_add_used = false;
}  // namespace

// out = P (fp32, rows x cols) optionally right-rotated, converted to dtype
// (add: a bf16 addend fused into the store when the K4 kernel can, *add_used
// then set -- the E path of halo_linear_backward_acc)
static void finish_right(const float* P, void* out, int32_t dtype, int64_t rows, int64_t cols, int64_t B, bool rotate,
                         cudaStream_t st, const void* add, bool* add_used) {
    if (add && rotate && dtype == HALO_DTYPE_BF16) {
        ProfScope ps(PC_K4, (double)rows * cols * (4 + 2 + 2), st);
        if (rows_xform_add(P, rows * cols, B, add, out, st)) {
            *add_used = true;
            return;
        }
    }
    // B == 1 is the identity transform with norm 1: an exact copy/convert
    ProfScope ps(PC_K4, (double)rows * cols * (4 + dt_bytes(dtype)), st);
    BaseScope ht(true);  // transform_right_ht (H^T; = H for power-of-two blocks)
    run_rows(P, HALO_DTYPE_F32, rows, cols, rotate ? B : 1, 2, 0, nullptr, nullptr, nullptr, out, dtype, nullptr,
             nullptr, st);
}

// Granularity::row / ::column backward (halo_linear.hpp:381-439 with
// per-row or per-column scales).  Some scale vector of (WH)_Q / (E_Y)_Q /
// (H_b E_Y)_Q sits on the contracted dim of the E and G products, so both run
// through qmatmul's dequantized double path (quantize.hpp:377-379), restated
// bit-exactly by deq_gemm; the quantizations are the per-row K1
// (rows_v3_per_row) or col_quantize, the transforms the same K4 kernels as
// the tensor path.
static halo_status backward_grouped(halo_linear* l, halo_ctx* c, const void* e_y, int32_t e_dtype, void* e_x,
                                 int32_t ex_dtype, void* grad_w, int32_t gw_dtype, cudaStream_t st) {
    const halo_scheme& s = l->s;
    const int64_t b = c->b, m = l->m, n = l->n;
    const int fmt = s.format_e;
    if (c->m != m || c->n != n) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: upstream error shape mismatch");
    if (!valid_dtype(e_dtype) || !valid_dtype(ex_dtype) || (grad_w && !valid_dtype(gw_dtype)))
        return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: bad dtype");
    if (s.peft || l->scatter || c->wq_sharded)
        return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: row-granularity backward: no PEFT / sharded / scattered path");
    // the saved operands are reused as in error_path / gradient_path (:390,
    // :432): their rotation must be the one E and G ask for
    if ((bool)s.E.right != c->wq_rotated || (bool)s.G.right != c->xq_rotated)
        return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: row-granularity backward needs the saved operand rotations");
    if (fmt != HALO_FMT_INT8 && fmt != HALO_FMT_FP8_E4M3)
        return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: row / column granularity supports INT8 / FP8 E4M3");
    // Granularity::column (c->gran): every scale vector indexes columns, and
    // E_Y^T's column scales become row scales (transpose_quantized :317-320)
    const bool col = c->gran == HALO_GRAN_COLUMN;
    if (!col && n % 256)
        return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: row-granularity backward needs out_features % 256 == 0");
    auto gquant = [&](int32_t dt, const void* in, int64_t rows, float* scales, uint8_t* codes) -> bool {
        unsigned* err = &c->d()->err;
        return col ? col_quantize(fmt, dt, in, rows, n, c->amax_rows.as<unsigned>(), scales, codes, err, st)
                   : rows_v3_per_row(fmt, dt, in, rows, n, 1, c->amax_rows.as<unsigned>(), scales, codes, err, st);
    };
    // scale strides (index pair of each product operand): per-row scales
    // follow the operand's row, per-column its column
    const int64_t e_si = col ? 0 : 1, e_sk = col ? 1 : 0;     // E / (H_b E) codes as A (i = token, k = out)
    const int64_t w_sk = col ? 0 : 1, w_sj = col ? 1 : 0;     // (WH)_Q as B (k = out, j = in)
    const int64_t g_si = col ? 1 : 0, g_sk = col ? 0 : 1;     // E^T as A (i = out, k = token)
    const int64_t x_sk = col ? 0 : 1, x_sj = col ? 1 : 0;     // (XH)_Q as B (k = token, j = in)
    if (!grad_w && !e_x) return HALO_OK;
    int64_t Bm = 1;
    if ((s.E.right || s.G.right) && resolve_block(m, s.had_block, &Bm, "backward") != HALO_OK)
        return HALO_ERR_INVALID_ARGUMENT;
    DevScalars* d = c->d();
    const bool left = s.E.left;
    const int64_t b_pad = left ? halo_padded_batch(b, s.had_block) : b;
    int64_t Bb = 1;
    if (left && resolve_block(b_pad, s.had_block, &Bb, "backward (token dim)") != HALO_OK)
        return HALO_ERR_INVALID_ARGUMENT;
    c->b_pad = b_pad;
    const int64_t mx = b_pad > n ? b_pad : n;
    if (c->S()->eq.ensure((size_t)(b * n)) != HALO_OK || c->S()->es_rows.ensure((size_t)mx * sizeof(float)) != HALO_OK ||
        c->amax_rows.ensure((size_t)mx * sizeof(unsigned)) != HALO_OK ||
        c->S()->scratch.ensure((size_t)(b_pad * m) * sizeof(float)) != HALO_OK)
        return HALO_ERR_CUDA;
    // (E_Y)_Q per token (:371); feeds E (no left rotation) and G
    const bool plain = grad_w || !left;
    if (plain) {
        ProfScope ps(PC_K2, (double)b * n * (dt_bytes(e_dtype) + 1), st);
        if (!gquant(e_dtype, e_y, b, c->S()->es_rows.as<float>(), c->S()->eq.as<uint8_t>()))
            return fail(HALO_ERR_INVALID_ARGUMENT, "backward: row-granularity operands must be 32 B aligned");
        ++l->ce;
    }
    float* P = c->S()->scratch.as<float>();
    // ---- error path (:381-413)
    if (left) {
        // (H_b pad(E_Y))_Q per padded token (:393-399)
        if (c->S()->ehq.ensure((size_t)(b_pad * n)) != HALO_OK || c->S()->ehs_rows.ensure((size_t)mx * sizeof(float)) != HALO_OK ||
            c->S()->gscratch.ensure((size_t)(b_pad * n) * sizeof(float)) != HALO_OK)
            return HALO_ERR_CUDA;
        float* T = c->S()->gscratch.as<float>();
        {
            ProfScope ps(PC_K2, (double)b * n * dt_bytes(e_dtype) + (double)b_pad * n * 9, st);
            pad_rows_f32(e_y, e_dtype, b, b_pad, n, T, st);
            BaseScope orient(true);  // transform_left_h (:398)
            run_cols(T, HALO_DTYPE_F32, b_pad, b_pad, n, Bb, 2, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                     T, b_pad, nullptr, nullptr, nullptr, st);
            if (!gquant(HALO_DTYPE_F32, T, b_pad, c->S()->ehs_rows.as<float>(), c->S()->ehq.as<uint8_t>()))
                return fail(HALO_ERR_INVALID_ARGUMENT, "backward: row-granularity operands must be 32 B aligned");
        }
        ++l->ce;
        if (e_x) {
            {
                ProfScope ps(PC_GEMM, 2.0 * (double)b_pad * m * n, st);
                if (!deq_gemm(fmt, c->S()->ehq.as<uint8_t>(), c->S()->ehs_rows.as<float>(), n, 1, e_si, e_sk, c->wq_codes,
                              c->wq_scale, m, 1, w_sk, w_sj, P, b_pad, m, n, m, st))
                    return fail(HALO_ERR_CUDA, "backward: E product launch failed");
            }
            // transform_left, take_rows(b) (:405-409), in place
            ProfScope ps(PC_K4, (double)b_pad * m * 4 + (double)b * m * 4, st);
            BaseScope orient(false);
            run_cols(P, HALO_DTYPE_F32, b_pad, b_pad, m, Bb, 2, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                     P, b, nullptr, nullptr, nullptr, st);
        }
    } else if (e_x) {
        ProfScope ps(PC_GEMM, 2.0 * (double)b * m * n, st);
        if (!deq_gemm(fmt, c->S()->eq.as<uint8_t>(), c->S()->es_rows.as<float>(), n, 1, e_si, e_sk, c->wq_codes, c->wq_scale, m,
                      1, w_sk, w_sj, P, b, m, n, m, st))
            return fail(HALO_ERR_CUDA, "backward: E product launch failed");
    }
    // transform_right_ht (:410-411) or the exact copy / convert
    if (e_x) finish_right(P, e_x, ex_dtype, b, m, Bm, s.E.right, st);
    // ---- gradient path (:418-439): G = transpose_quantized(eq) (XH)_Q [H^T];
    // E_Y^T's scales become per-column (:312-316)
    if (grad_w) {
        if (c->S()->gscratch.ensure((size_t)(n * m) * sizeof(float)) != HALO_OK) return HALO_ERR_CUDA;
        float* G = c->S()->gscratch.as<float>();
        {
            ProfScope ps(PC_GEMM, 2.0 * (double)n * m * b, st);
            if (!deq_gemm(fmt, c->S()->eq.as<uint8_t>(), c->S()->es_rows.as<float>(), 1, n, g_si, g_sk, c->xq_codes(), c->xq_scale,
                          m, 1, x_sk, x_sj, G, n, m, b, m, st))
                return fail(HALO_ERR_CUDA, "backward: G product launch failed");
        }
        finish_right(G, grad_w, gw_dtype, n, m, Bm, s.G.right, st);
    }
    return cuda_check("backward");
}

// Granularity::mx backward (halo_linear.hpp:381-439 with MxFp6E3M2): the
// error path quantizes (H_b pad(E_Y)) or E_Y with 1 x 32 blocks along out
// features, the gradient path quantizes transpose(E_Y) itself -- MX blocks do
// not survive a transpose (:427-431) -- with blocks along tokens; both
// products are dequantized double matmuls (deq_gemm, bit-exact).
static halo_status backward_mx(halo_linear* l, halo_ctx* c, const void* e_y, int32_t e_dtype, void* e_x,
                               int32_t ex_dtype, void* grad_w, int32_t gw_dtype, cudaStream_t st) {
    const halo_scheme& s = l->s;
    const int64_t b = c->b, m = l->m, n = l->n;
    const int fmt = s.format_e;
    if (c->m != m || c->n != n) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: upstream error shape mismatch");
    if (!valid_dtype(e_dtype) || !valid_dtype(ex_dtype) || (grad_w && !valid_dtype(gw_dtype)))
        return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: bad dtype");
    if (s.peft || l->scatter || c->wq_sharded)
        return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: mx backward: no PEFT / sharded / scattered path");
    if ((bool)s.E.right != c->wq_rotated || (bool)s.G.right != c->xq_rotated)
        return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: mx backward needs the saved operand rotations");
    int64_t Bm = 1;
    if ((s.E.right || s.G.right) && resolve_block(m, s.had_block, &Bm, "backward") != HALO_OK)
        return HALO_ERR_INVALID_ARGUMENT;
    DevScalars* d = c->d();
    const bool left = s.E.left;
    const int64_t b_pad = left ? halo_padded_batch(b, s.had_block) : b;
    int64_t Bb = 1;
    if (left && resolve_block(b_pad, s.had_block, &Bb, "backward (token dim)") != HALO_OK)
        return HALO_ERR_INVALID_ARGUMENT;
    c->b_pad = b_pad;
    const int64_t nbn = n / 32, nbm = m / 32, nbb = (b + 31) / 32;
    if (c->S()->eq.ensure((size_t)(b_pad * n)) != HALO_OK || c->S()->es_rows.ensure((size_t)(b_pad * nbn) * sizeof(float)) != HALO_OK ||
        c->S()->scratch.ensure((size_t)(b_pad * m) * sizeof(float)) != HALO_OK)
        return HALO_ERR_CUDA;
    float* P = c->S()->scratch.as<float>();
    // ---- error path (:381-413): A = E codes (i = token, k = out, scale
    // [i][k >> 5]); B = wq (k = out, j = in, scale [k][j >> 5])
    if (e_x) {
        const uint8_t* ecodes;
        const float* escales;
        int64_t rows = b;
        if (left) {
            if (c->S()->ehq.ensure((size_t)(b_pad * n)) != HALO_OK || c->S()->ehs_rows.ensure((size_t)(b_pad * nbn) * sizeof(float)) != HALO_OK ||
                c->S()->gscratch.ensure((size_t)(b_pad * n) * sizeof(float)) != HALO_OK)
                return HALO_ERR_CUDA;
            float* T = c->S()->gscratch.as<float>();
            ProfScope ps(PC_K2, (double)b * n * dt_bytes(e_dtype) + (double)b_pad * n * 9, st);
            pad_rows_f32(e_y, e_dtype, b, b_pad, n, T, st);
            BaseScope orient(true);  // transform_left_h (:398)
            run_cols(T, HALO_DTYPE_F32, b_pad, b_pad, n, Bb, 2, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                     T, b_pad, nullptr, nullptr, nullptr, st);
            if (!mx_quantize(HALO_DTYPE_F32, T, b_pad, n, n, 1, c->S()->ehq.as<uint8_t>(), c->S()->ehs_rows.as<float>(), &d->err, st))
                return fail(HALO_ERR_CUDA, "backward: mx quantization failed");
            ecodes = c->S()->ehq.as<uint8_t>();
            escales = c->S()->ehs_rows.as<float>();
            rows = b_pad;
        } else {
            ProfScope ps(PC_K2, (double)b * n * (dt_bytes(e_dtype) + 1), st);
            if (!mx_quantize(e_dtype, e_y, b, n, n, 1, c->S()->eq.as<uint8_t>(), c->S()->es_rows.as<float>(), &d->err, st))
                return fail(HALO_ERR_CUDA, "backward: mx quantization failed");
            ecodes = c->S()->eq.as<uint8_t>();
            escales = c->S()->es_rows.as<float>();
        }
        ++l->ce;
        {
            ProfScope ps(PC_GEMM, 2.0 * (double)rows * m * n, st);
            if (!deq_gemm(fmt, ecodes, escales, n, 1, nbn, 1, c->wq_codes, c->wq_scale, m, 1, nbm, 1, P, rows, m, n, m,
                          st, 0, 5, 0, 5))
                return fail(HALO_ERR_CUDA, "backward: E product launch failed");
        }
        if (left) {  // transform_left, take_rows(b) (:405-409), in place
            ProfScope ps(PC_K4, (double)b_pad * m * 4 + (double)b * m * 4, st);
            BaseScope orient(false);
            run_cols(P, HALO_DTYPE_F32, b_pad, b_pad, m, Bb, 2, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                     P, b, nullptr, nullptr, nullptr, st);
        }
        finish_right(P, e_x, ex_dtype, b, m, Bm, s.E.right, st);
    }
    // ---- gradient path (:418-439): quantize(transpose(E_Y)) [n x b] with
    // blocks along tokens (A: i = out, k = token, scale [i][k >> 5]); B =
    // (XH)_Q (k = token, j = in, scale [k][j >> 5])
    if (grad_w) {
        if (c->S()->gscratch.ensure((size_t)(n * m) * sizeof(float)) != HALO_OK || c->S()->mx_t.ensure((size_t)(n * b)) != HALO_OK ||
            c->S()->mx_ts.ensure((size_t)(n * nbb) * sizeof(float)) != HALO_OK)
            return HALO_ERR_CUDA;
        uint8_t* et = c->S()->mx_t.as<uint8_t>();
        float* ets = c->S()->mx_ts.as<float>();
        {
            ProfScope ps(PC_K2, (double)b * n * (dt_bytes(e_dtype) + 1), st);
            if (!mx_quantize(e_dtype, e_y, n, b, 1, n, et, ets, &d->err, st))
                return fail(HALO_ERR_CUDA, "backward: mx quantization failed");
        }
        ++l->ce;
        float* G = c->S()->gscratch.as<float>();
        {
            ProfScope ps(PC_GEMM, 2.0 * (double)n * m * b, st);
            if (!deq_gemm(fmt, et, ets, b, 1, nbb, 1, c->xq_codes(), c->xq_scale, m, 1, nbm, 1, G, n, m, b, m, st, 0, 5,
                          0, 5))
                return fail(HALO_ERR_CUDA, "backward: G product launch failed");
        }
        finish_right(G, grad_w, gw_dtype, n, m, Bm, s.G.right, st);
    }
    return cuda_check("backward");
}

extern "C" halo_status halo_linear_backward(halo_linear* l, const halo_ctx* cc, const void* e_y, int32_t e_dtype,
                                            void* e_x, int32_t ex_dtype, void* grad_w, int32_t gw_dtype,
                                            halo_stream_t stream) {
    if (!l || !cc || !e_y || !e_x) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: null argument");
    halo_ctx* c = const_cast<halo_ctx*>(cc);  // scratch buffers only; saved codes are read-only
    // halo_linear_backward_acc's addend: only the tensor path's E K4 takes it
    const void* ex_add = t_ex_add;
    t_ex_add = nullptr;
    if (!c->valid) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: backward without forward context");
    if (c->gran == HALO_GRAN_MX) return backward_mx(l, c, e_y, e_dtype, e_x, ex_dtype, grad_w, gw_dtype, (cudaStream_t)stream);
    if (c->row_gran || c->gran == HALO_GRAN_COLUMN) return backward_grouped(l, c, e_y, e_dtype, e_x, ex_dtype, grad_w, gw_dtype, (cudaStream_t)stream);
    if (c->m != l->m || c->n != l->n) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: upstream error shape mismatch");
    if (!valid_dtype(e_dtype) || !valid_dtype(ex_dtype) || (grad_w && !valid_dtype(gw_dtype)))
        return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: bad dtype");
    cudaStream_t st = (cudaStream_t)stream;
    const halo_scheme& s = l->s;
    const int64_t b = c->b, m = l->m, n = l->n;
    const int fmt = s.format_e;
    DevScalars* d = c->d();
    int64_t Bm = 1;
    if ((s.E.right || s.G.right) && resolve_block(m, s.had_block, &Bm, "backward") != HALO_OK)
        return HALO_ERR_INVALID_ARGUMENT;
    if (c->S()->eq.ensure((size_t)(b * n)) != HALO_OK) return HALO_ERR_CUDA;

    // weight operand for E with E's right rotation (:390)
    const uint8_t* wq = c->wq_codes;
    const float* sw = c->wq_scale;
    // sharded (WH)_Q: the E GEMM reads the parts in place, split along its
    // contracted dim (out_features) -- the backward "regather" of
    // hqfsdp.hpp:200-226 without moving a byte
    const ShardSpec* wsh = nullptr;
    if (c->wq_sharded) {
        if (!l->sharded) return fail(HALO_ERR_LOGIC, "halo layer: sharded weight codes were uninstalled before backward");
        wsh = &l->shard_k;
    }
    if ((bool)s.E.right != c->wq_rotated) {
        if (wsh) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: sharded codes cannot be re-quantized for E");
        const halo_status r = quantize_weight(l, c, s.E.right, c->wq2, SW2, &wq, &sw, st);
        if (r != HALO_OK) return r;
    }

    // ---- error path (:381-413)
    if (s.E.left) {
        const int64_t b_pad = halo_padded_batch(b, s.had_block);
        int64_t Bb;
        if (resolve_block(b_pad, s.had_block, &Bb, "backward (token dim)") != HALO_OK) return HALO_ERR_INVALID_ARGUMENT;
        c->b_pad = b_pad;
        if (c->S()->ehq.ensure((size_t)(b_pad * n)) != HALO_OK) return HALO_ERR_CUDA;
        if (c->S()->scratch.ensure((size_t)(b_pad * m) * sizeof(float)) != HALO_OK) return HALO_ERR_CUDA;
        // (H_b E_Y)_Q and (E_Y)_Q in one pass (:399 and :371); the plain
        // codes only feed G, so PEFT / no-grad_w backwards skip them (:446-448)
        const bool plain = (grad_w || l->scatter) && !s.peft;
        // absmax words already produced by halo_swiglu_backward_absmax for
        // this E_Y: skip K2's phase A
        const bool have_amax = c->e_amax_src == e_y && c->e_amax_b == b && e_dtype == HALO_DTYPE_BF16;
        c->e_amax_src = nullptr;
        halo_status r = left_quant_impl(e_y, e_dtype, b, n, Bb, b_pad, fmt, c->S()->ehq.as<uint8_t>(),
                                        plain ? c->S()->eq.as<uint8_t>() : nullptr, &d->amax[SEH], &d->amax[SE],
                                        &d->scale[SEH], &d->scale[SE], &d->err, st, have_amax, !s.peft);
        if (r != HALO_OK) return r;
        l->ce += plain ? 2 : 1;
        float* P = c->S()->scratch.as<float>();
        if (fuse_k4() && fusable_block(Bb)) {
            // prod^T = wq^T ehq^T (:401, transposed: M = in-features,
            // N = padded tokens); the epilogue applies transform_left over
            // the token axis (:405-408) and stores take_rows(b) of prod
            // (:409) row-major.  ss = sw * s_ehq: same exact double product.
            ShardScope shards(wsh, nullptr);  // A = (WH)_Q, MN-major, K = out_features
            int gr = prof_gemm_x(fmt, wq, c->S()->ehq.as<uint8_t>(), m, b_pad, n, 0, 1, sw, &d->scale[SEH], P, 0, Bb, 1, b,
                                 st);
            if (gr != 0) return fail(HALO_ERR_CUDA, "backward: E GEMM launch failed");
        } else {
            // prod = qmatmul(eq, wq)  (:401): B operand (n x m) is MN-major
            ShardScope shards(nullptr, wsh);
            int gr = prof_gemm(fmt, c->S()->ehq.as<uint8_t>(), wq, b_pad, m, n, 1, 0, &d->scale[SEH], sw, P, 0, st);
            if (gr != 0) return fail(HALO_ERR_CUDA, "backward: E GEMM launch failed");
            // prod = transform_left(prod); take_rows(b)  (:405-409), in place
            ProfScope ps(PC_K4, (double)b_pad * m * 4 + (double)b * m * 4, st);
            BaseScope orient(s.peft);  // transform_left (:406), PEFT transform_left_h (:451)
            run_cols(P, HALO_DTYPE_F32, b_pad, b_pad, m, Bb, 2, 0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                     P, b, nullptr, nullptr, nullptr, st);
        }
        // prod = transform_right_ht(prod)  (:410-411)
        finish_right(P, e_x, ex_dtype, b, m, Bm, s.E.right, st, ex_add, &t_ex_add_used);
    } else {
        c->b_pad = b;
        const halo_status r = rotate_quantize_impl(e_y, e_dtype, b, n, 1, false, fmt, nullptr, c->S()->eq.as<uint8_t>(),
                                                   &d->amax[SE], &d->scale[SE], &d->err, st);
        if (r != HALO_OK) return r;
        l->ce += 1;
        ShardScope shards(nullptr, wsh);  // B = (W[H])_Q, MN-major, K = out_features
        if (s.E.right && fuse_k4() && fusable_block(Bm)) {
            // E_X = (E_Y)_Q (WH)_Q H^T (:410-411) with the right transform in
            // the GEMM epilogue
            int gr = prof_gemm_x(fmt, c->S()->eq.as<uint8_t>(), wq, b, m, n, 1, 0, &d->scale[SE], sw, e_x,
                                 ex_dtype == HALO_DTYPE_F32 ? 0 : 1, Bm, 0, m, st);
            if (gr != 0) return fail(HALO_ERR_CUDA, "backward: E GEMM launch failed");
        } else if (s.E.right) {
            if (c->S()->scratch.ensure((size_t)(b * m) * sizeof(float)) != HALO_OK) return HALO_ERR_CUDA;
            float* P = c->S()->scratch.as<float>();
            int gr = prof_gemm(fmt, c->S()->eq.as<uint8_t>(), wq, b, m, n, 1, 0, &d->scale[SE], sw, P, 0, st);
            if (gr != 0) return fail(HALO_ERR_CUDA, "backward: E GEMM launch failed");
            finish_right(P, e_x, ex_dtype, b, m, Bm, true, st, ex_add, &t_ex_add_used);
        } else {
            int gr = prof_gemm(fmt, c->S()->eq.as<uint8_t>(), wq, b, m, n, 1, 0, &d->scale[SE], sw, e_x,
                              ex_dtype == HALO_DTYPE_F32 ? 0 : 1, st);
            if (gr != 0) return fail(HALO_ERR_CUDA, "backward: E GEMM launch failed");
        }
    }

    // ---- gradient path (:418-439): G = (E_Y^T)_Q (XH)_Q [H^T]; a PEFT layer
    // has no weight gradient (its U/V gradients are working-precision
    // matmuls of the caller, :312-318)
    if ((grad_w || l->scatter) && !s.peft) {
        const uint8_t* xq = c->xq_codes();
        const float* sxp = c->xq_scale;
        if (l->scatter) {
            // fp32 partial G of this rank's tokens, rows scattered to their
            // owners (the reduce-scatter of hqfsdp.hpp:271-300 fused into the
            // GEMM); halo_reduce_scatter_shard finishes the mean
            if (s.G.right && !(fuse_k4() && fusable_block(Bm)))
                return fail(HALO_ERR_INVALID_ARGUMENT, "backward: scattered G needs the fused right transform");
            ShardScope scat(nullptr, nullptr, &l->scatter_c);
            const int gr = s.G.right ? prof_gemm_x(fmt, c->S()->eq.as<uint8_t>(), xq, n, m, b, 0, 0, &d->scale[SE], sxp,
                                                   nullptr, 0, Bm, 0, m, st)
                                     : prof_gemm(fmt, c->S()->eq.as<uint8_t>(), xq, n, m, b, 0, 0, &d->scale[SE], sxp,
                                                 nullptr, 0, st);
            if (gr != 0) return fail(HALO_ERR_CUDA, "backward: scattered G GEMM launch failed");
            return cuda_check("backward");
        }
        if (s.G.right && fuse_k4() && fusable_block(Bm)) {
            // grad_w = (E_Y^T)_Q (XH)_Q H^T (:433-437), the right transform in
            // the GEMM epilogue
            int gr = prof_gemm_x(fmt, c->S()->eq.as<uint8_t>(), xq, n, m, b, 0, 0, &d->scale[SE], sxp, grad_w,
                                 gw_dtype == HALO_DTYPE_F32 ? 0 : 1, Bm, 0, m, st);
            if (gr != 0) return fail(HALO_ERR_CUDA, "backward: G GEMM launch failed");
        } else if (s.G.right) {
            if (c->S()->gscratch.ensure((size_t)(n * m) * sizeof(float)) != HALO_OK) return HALO_ERR_CUDA;
            float* G = c->S()->gscratch.as<float>();
            int gr = prof_gemm(fmt, c->S()->eq.as<uint8_t>(), xq, n, m, b, 0, 0, &d->scale[SE], sxp, G, 0, st);
            if (gr != 0) return fail(HALO_ERR_CUDA, "backward: G GEMM launch failed");
            finish_right(G, grad_w, gw_dtype, n, m, Bm, true, st);
        } else {
            int gr = prof_gemm(fmt, c->S()->eq.as<uint8_t>(), xq, n, m, b, 0, 0, &d->scale[SE], sxp, grad_w,
                              gw_dtype == HALO_DTYPE_F32 ? 0 : 1, st);
            if (gr != 0) return fail(HALO_ERR_CUDA, "backward: G GEMM launch failed");
        }
    }
    return cuda_check("backward");
}

extern "C" halo_status halo_linear_backward_acc(halo_linear* l, const halo_ctx* cc, const void* e_y, int32_t e_dtype,
                                                const void* e_x_add, void* e_x, int32_t ex_dtype, void* grad_w,
                                                int32_t gw_dtype, halo_stream_t stream) {
    if (!e_x_add) return fail(HALO_ERR_INVALID_ARGUMENT, "backward_acc: null addend");
    if (ex_dtype != HALO_DTYPE_BF16) return fail(HALO_ERR_INVALID_ARGUMENT, "backward_acc: e_x must be bf16");
    if (!l || !cc) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: null argument");
    t_ex_add = e_x_add;  // taken (and cleared) by halo_linear_backward on entry
    t_ex_add_used = false;
    const halo_status r = halo_linear_backward(l, cc, e_y, e_dtype, e_x, ex_dtype, grad_w, gw_dtype, stream);
    const bool fused = t_ex_add_used;
    t_ex_add = nullptr;
    t_ex_add_used = false;
    if (r != HALO_OK || fused) return r;
    // the E path had no fusable K4 (other schemes / blocks): a separate add
    run_add(e_x_add, e_x, e_x, DT_BF16, cc->b * l->m, (cudaStream_t)stream);
    return cuda_check("backward_acc");
}

extern "C" halo_status halo_linear_export_inference_weights(halo_linear* l, uint8_t* codes, float* scale,
                                                            halo_stream_t stream) {
    if (!l || !codes || !scale) return fail(HALO_ERR_INVALID_ARGUMENT, "export: null argument");
    if (!l->s.F.middle) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: export requires a rotated-forward scheme");
    if (!l->w) return fail(HALO_ERR_INVALID_ARGUMENT, "halo layer: no weight set");
    int64_t B;
    if (resolve_block(l->m, l->s.had_block, &B, "export") != HALO_OK) return HALO_ERR_INVALID_ARGUMENT;
    if (l->s.peft) {  // export_inference_weights returns frozen_wq_ (:333-334)
        cudaStream_t st = (cudaStream_t)stream;
        cudaMemcpyAsync(codes, l->qcodes, (size_t)(l->n * l->m), cudaMemcpyDeviceToDevice, st);
        cudaMemcpyAsync(scale, l->qscale, sizeof(float), cudaMemcpyDeviceToDevice, st);
        return cuda_check("export");
    }
    if (l->s.granularity == HALO_GRAN_COLUMN)
        return fail(HALO_ERR_INVALID_ARGUMENT, "export: column granularity is not exported");
    if (l->s.granularity == HALO_GRAN_ROW)  // `scale` receives out_features floats
        return halo_rotate_quantize_rows(l->w, l->w_dtype, l->n, l->m, l->s.had_block, l->s.format_w, codes, scale,
                                         stream);
    DevScalars* d = free_scalars(stream);
    if (!d) return HALO_ERR_CUDA;
    return rotate_quantize_impl(l->w, l->w_dtype, l->n, l->m, B, true, l->s.format_w, nullptr, codes, &d->amax[SW],
                                scale, &d->err, (cudaStream_t)stream);
}

extern "C" halo_status halo_linear_counters(const halo_linear* l, halo_counters* out) {
    if (!l || !out) return fail(HALO_ERR_INVALID_ARGUMENT, "counters: null");
    out->x = l->cx.load();
    out->w = l->cw.load();
    out->e = l->ce.load();
    return HALO_OK;
}

extern "C" halo_status halo_linear_reset_counters(halo_linear* l) {
    if (!l) return fail(HALO_ERR_INVALID_ARGUMENT, "counters: null");
    l->cx = 0;
    l->cw = 0;
    l->ce = 0;
    return HALO_OK;
}

extern "C" halo_status halo_ctx_saved(const halo_ctx* c, const uint8_t** xq, const float** sx, const uint8_t** wq,
                                      const float** sw, int64_t* batch_rows) {
    if (!c || !c->valid) return fail(HALO_ERR_INVALID_ARGUMENT, "ctx: no forward context");
    if (xq) *xq = c->xq_codes();
    if (sx) *sx = c->xq_scale ? c->xq_scale : &c->d()->scale[SX];
    if (wq) *wq = c->wq_codes;
    if (sw) *sw = c->wq_scale;
    if (batch_rows) *batch_rows = c->b;
    return HALO_OK;
}

extern "C" halo_status halo_ctx_error_operands(const halo_ctx* c, const uint8_t** ehq, const float** seh,
                                               const uint8_t** eq, const float** se, int64_t* b_pad) {
    if (!c || !c->valid) return fail(HALO_ERR_INVALID_ARGUMENT, "ctx: no forward context");
    // row / column granularity: the scale vectors of the last backward
    // (per token for ROW: b_pad / b floats; per column for COLUMN: out_features)
    const bool grouped = c->gran != HALO_GRAN_TENSOR;
    const halo_ctx* sc = c->sowner ? c->sowner : c;
    if (ehq) *ehq = sc->ehq.as<uint8_t>();
    if (seh) *seh = grouped ? sc->ehs_rows.as<float>() : &c->d()->scale[SEH];
    if (eq) *eq = sc->eq.as<uint8_t>();
    if (se) *se = grouped ? sc->es_rows.as<float>() : &c->d()->scale[SE];
    if (b_pad) *b_pad = c->b_pad;
    return HALO_OK;
}

extern "C" halo_status halo_ctx_share_scratch(halo_ctx* ctx, halo_ctx* owner) {
    if (!ctx) return fail(HALO_ERR_INVALID_ARGUMENT, "ctx: null");
    if (owner == ctx) owner = nullptr;
    if (owner && owner->sowner) owner = owner->sowner;
    ctx->sowner = owner;
    return HALO_OK;
}

extern "C" halo_status halo_ctx_check(halo_ctx* c, halo_stream_t stream) {
    if (!c) return fail(HALO_ERR_INVALID_ARGUMENT, "ctx: null");
    if (cudaStreamSynchronize((cudaStream_t)stream) != cudaSuccess)
        return fail(HALO_ERR_CUDA, std::string("ctx check: ") + cudaGetErrorString(cudaGetLastError()));
    unsigned err = 0;
    cudaMemcpy(&err, &c->d()->err, sizeof(unsigned), cudaMemcpyDeviceToHost);
    if (err) {
        cudaMemset(&c->d()->err, 0, sizeof(unsigned));
        return fail(HALO_ERR_NUMERIC, "tensor: non-finite value in a quantized operand");
    }
    return HALO_OK;
}

extern "C" halo_status halo_device_copy(void* dst, const void* src, int64_t bytes, halo_stream_t stream) {
    if (bytes < 0 || (bytes && (!dst || !src))) return fail(HALO_ERR_INVALID_ARGUMENT, "device_copy: bad arguments");
    if (bytes == 0) return HALO_OK;
    if (cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream) != cudaSuccess)
        return fail(HALO_ERR_CUDA, "device_copy failed");
    return HALO_OK;
}

// ============================================================ glue + profile

extern "C" halo_status halo_swiglu_forward(const void* g, const void* u, void* h, int64_t n, halo_stream_t stream) {
    if (!g || !u || !h || n < 0 || n % 8) return fail(HALO_ERR_INVALID_ARGUMENT, "swiglu_forward: bad arguments");
    if (n == 0) return HALO_OK;
    cudaStream_t st = (cudaStream_t)stream;
    ProfScope ps(PC_GLUE, (double)n * 6, st);
    run_swiglu_fwd(g, u, h, n, st);
    return cuda_check("swiglu_forward");
}

extern "C" halo_status halo_swiglu_backward(const void* dh, const void* g, const void* u, void* dg, void* du, int64_t n,
                                            halo_stream_t stream) {
    if (!dh || !g || !u || !dg || !du || n < 0 || n % 8)
        return fail(HALO_ERR_INVALID_ARGUMENT, "swiglu_backward: bad arguments");
    if (n == 0) return HALO_OK;
    cudaStream_t st = (cudaStream_t)stream;
    ProfScope ps(PC_GLUE, (double)n * 10, st);
    run_swiglu_bwd(dh, g, u, dg, du, n, st);
    return cuda_check("swiglu_backward");
}

// SwiGLU forward fused with phase A of the down projection's X quantization
// (rotated X, Hadamard block 256, bf16): h is written as by
// halo_swiglu_forward and the absmax word of (h H) lands in `dctx`, so the
// following halo_linear_forward(down, h, ..., dctx) skips its absmax pass.
// Other configurations: identical to halo_swiglu_forward.
extern "C" halo_status halo_swiglu_forward_absmax(const halo_linear* down, halo_ctx* dctx, const void* g,
                                                  const void* u, void* h, int64_t rows, int64_t cols,
                                                  halo_stream_t stream) {
    if (!down || !dctx || !g || !u || !h || rows <= 0 || cols <= 0)
        return fail(HALO_ERR_INVALID_ARGUMENT, "swiglu_forward_absmax: bad argument");
    cudaStream_t st = (cudaStream_t)stream;
    dctx->x_amax_src = nullptr;
    int64_t B = 0;
    const bool fuse = down->s.F.middle && down->s.granularity == HALO_GRAN_TENSOR && down->m == cols &&
                      resolve_block(cols, down->s.had_block, &B, "swiglu forward") == HALO_OK && B == 256 &&
                      (rows * cols) % 1024 == 0;
    if (fuse) {
        if (dctx->dev.ensure(sizeof(DevScalars)) != HALO_OK) return HALO_ERR_CUDA;
        DevScalars* d = dctx->d();
        cudaMemsetAsync(&d->amax[SX], 0, sizeof(unsigned), st);
        bool ok;
        {
            ProfScope ps(PC_GLUE, (double)rows * cols * 6.0, st);
            ok = swiglu_absmax(g, u, h, rows * cols, cols, &d->amax[SX], &d->err, st);
        }
        if (ok) {
            dctx->x_amax_src = h;
            dctx->x_amax_b = rows;
            return cuda_check("swiglu_forward_absmax");
        }
    }
    {
        ProfScope ps(PC_GLUE, (double)rows * cols * 6.0, st);
        run_swiglu_fwd(g, u, h, rows * cols, st);
    }
    return cuda_check("swiglu_forward");
}

// SwiGLU backward fused with K2's phase A of both input projections (HALO-2
// family: E.left).  dG, dU are written as by halo_swiglu_backward and the
// absmax words of (H_b dG), dG, (H_b dU), dU land in the two contexts, so
// the following halo_linear_backward(gate, gctx, dG, ...) and
// halo_linear_backward(up, uctx, dU, ...) skip their absmax passes.  For
// schemes without the left rotation this is halo_swiglu_backward.
extern "C" halo_status halo_swiglu_backward_absmax(const halo_linear* gate, halo_ctx* gctx, const halo_linear* up,
                                                   halo_ctx* uctx, const void* dh, const void* g, const void* u,
                                                   void* dg, void* du, int64_t b, int64_t cols, halo_stream_t stream) {
    if (!gate || !gctx || !up || !uctx || !dh || !g || !u || !dg || !du || b <= 0 || cols <= 0)
        return fail(HALO_ERR_INVALID_ARGUMENT, "swiglu_backward_absmax: bad argument");
    cudaStream_t st = (cudaStream_t)stream;
    gctx->e_amax_src = nullptr;
    uctx->e_amax_src = nullptr;
    const bool fuse = gate->s.E.left && up->s.E.left && gate->s.had_block == up->s.had_block && gate->n == cols &&
                      up->n == cols && gctx->valid && uctx->valid && gctx->b == b && uctx->b == b && cols % 4 == 0;
    if (fuse) {
        const int64_t b_pad = halo_padded_batch(b, gate->s.had_block);
        int64_t Bb;
        if (resolve_block(b_pad, gate->s.had_block, &Bb, "swiglu backward (token dim)") != HALO_OK)
            return HALO_ERR_INVALID_ARGUMENT;
        DevScalars* dgs = gctx->d();
        DevScalars* dus = uctx->d();
        cudaMemsetAsync(&dgs->amax[SEH], 0, 2 * sizeof(unsigned), st);  // SEH, SE adjacent
        cudaMemsetAsync(&dus->amax[SEH], 0, 2 * sizeof(unsigned), st);
        bool ok;
        {
            ProfScope ps(PC_GLUE, (double)b * cols * 10.0, st);
            ok = cols_swiglu_absmax(dh, g, u, dg, du, b, b_pad, cols, Bb, &dgs->amax[SEH], &dgs->amax[SE],
                                    &dus->amax[SEH], &dus->amax[SE], &dgs->err, st);
        }
        if (ok) {
            gctx->e_amax_src = dg;
            gctx->e_amax_b = b;
            uctx->e_amax_src = du;
            uctx->e_amax_b = b;
            return cuda_check("swiglu_backward_absmax");
        }
    }
    {
        ProfScope ps(PC_GLUE, (double)b * cols * 10.0, st);
        run_swiglu_bwd(dh, g, u, dg, du, b * cols, st);
    }
    return cuda_check("swiglu_backward");
}

extern "C" halo_status halo_add(const void* a, const void* b, void* out, int32_t dtype, int64_t n,
                                halo_stream_t stream) {
    if (!a || !b || !out || !valid_dtype(dtype) || n < 0 || n % 8)
        return fail(HALO_ERR_INVALID_ARGUMENT, "add: bad arguments");
    if (n == 0) return HALO_OK;
    cudaStream_t st = (cudaStream_t)stream;
    ProfScope ps(PC_GLUE, (double)n * 3 * dt_bytes(dtype), st);
    run_add(a, b, out, dtype, n, st);
    return cuda_check("add");
}

extern "C" halo_status halo_rmsnorm_forward(const void* x, const float* gain, void* y, int32_t y_dtype, float* rstd,
                                            int64_t rows, int64_t dim, int32_t mean, double eps, halo_stream_t stream) {
    if (!x || !gain || !y || !valid_dtype(y_dtype)) return fail(HALO_ERR_INVALID_ARGUMENT, "rmsnorm: bad arguments");
    if (rows < 0 || dim <= 0 || dim % 8 || !(eps >= 0.0)) return fail(HALO_ERR_INVALID_ARGUMENT, "rmsnorm: dim must be a positive multiple of 8, eps >= 0");
    if (rows == 0) return HALO_OK;
    ProfScope ps(PC_GLUE, (double)rows * dim * (2 + dt_bytes(y_dtype)), (cudaStream_t)stream);
    run_rmsnorm_fwd(x, gain, y, y_dtype, rstd, rows, (int)dim, mean != 0, eps, (cudaStream_t)stream);
    return cuda_check("rmsnorm_forward");
}

namespace {
thread_local std::unordered_map<cudaStream_t, Buffer> t_norm_scratch;
}

extern "C" halo_status halo_rmsnorm_backward(const void* x, const void* dy, int32_t dy_dtype, const float* gain,
                                             const float* rstd, void* dx, float* dgain, int64_t rows, int64_t dim,
                                             int32_t mean, halo_stream_t stream) {
    if (!x || !dy || !gain || !rstd || !dx || !dgain || !valid_dtype(dy_dtype))
        return fail(HALO_ERR_INVALID_ARGUMENT, "rmsnorm_backward: bad arguments");
    if (rows < 0 || dim <= 0 || dim % 8) return fail(HALO_ERR_INVALID_ARGUMENT, "rmsnorm_backward: dim must be a positive multiple of 8");
    cudaStream_t st = (cudaStream_t)stream;
    if (rows == 0) return cudaMemsetAsync(dgain, 0, sizeof(float) * dim, st) == cudaSuccess ? HALO_OK : cuda_check("rmsnorm_backward");
    Buffer& sc = t_norm_scratch[st];
    if (sc.ensure((size_t)rmsnorm_bwd_scratch(rows, (int)dim) * sizeof(float)) != HALO_OK) return HALO_ERR_CUDA;
    ProfScope ps(PC_GLUE, (double)rows * dim * (2 + dt_bytes(dy_dtype) + 2), st);
    run_rmsnorm_bwd(x, dy, dy_dtype, gain, rstd, dx, dgain, sc.as<float>(), rows, (int)dim, mean != 0, st);
    return cuda_check("rmsnorm_backward");
}

extern "C" halo_status halo_add_rmsnorm_forward(const void* x, const void* r, const float* gain, void* h, void* y,
                                                float* rstd, int64_t rows, int64_t dim, double eps,
                                                halo_stream_t stream) {
    if (!x || !r || !gain || !h || !y) return fail(HALO_ERR_INVALID_ARGUMENT, "add_rmsnorm: bad arguments");
    if (rows < 0 || dim <= 0 || dim % 8 || !(eps >= 0.0))
        return fail(HALO_ERR_INVALID_ARGUMENT, "add_rmsnorm: dim must be a positive multiple of 8, eps >= 0");
    if (rows == 0) return HALO_OK;
    ProfScope ps(PC_GLUE, (double)rows * dim * 8, (cudaStream_t)stream);
    if (!run_rmsnorm_fwd(x, gain, y, HALO_DTYPE_BF16, rstd, rows, (int)dim, true, eps, (cudaStream_t)stream, r, h))
        return fail(HALO_ERR_INVALID_ARGUMENT, "add_rmsnorm: unsupported arguments");
    return cuda_check("add_rmsnorm_forward");
}

extern "C" halo_status halo_rmsnorm_backward_res(const void* h, const void* dy, int32_t dy_dtype, const float* gain,
                                                 const float* rstd, const void* dres, void* dx, float* dgain,
                                                 int64_t rows, int64_t dim, halo_stream_t stream) {
    if (!h || !dy || !gain || !rstd || !dres || !dx || !dgain || !valid_dtype(dy_dtype))
        return fail(HALO_ERR_INVALID_ARGUMENT, "rmsnorm_backward_res: bad arguments");
    if (rows < 0 || dim <= 0 || dim % 8) return fail(HALO_ERR_INVALID_ARGUMENT, "rmsnorm_backward_res: dim must be a positive multiple of 8");
    cudaStream_t st = (cudaStream_t)stream;
    if (rows == 0) return cudaMemsetAsync(dgain, 0, sizeof(float) * dim, st) == cudaSuccess ? HALO_OK : cuda_check("rmsnorm_backward_res");
    Buffer& sc = t_norm_scratch[st];
    if (sc.ensure((size_t)rmsnorm_bwd_scratch(rows, (int)dim) * sizeof(float)) != HALO_OK) return HALO_ERR_CUDA;
    ProfScope ps(PC_GLUE, (double)rows * dim * (2 + dt_bytes(dy_dtype) + 4), st);
    run_rmsnorm_bwd(h, dy, dy_dtype, gain, rstd, dx, dgain, sc.as<float>(), rows, (int)dim, true, st, dres);
    return cuda_check("rmsnorm_backward_res");
}

extern "C" halo_status halo_rope_qkv(const void* in, void* out, const float* cos_sin, int64_t rows, int32_t seq,
                                     int32_t rot_heads, int32_t heads, int32_t head_dim, int32_t backward,
                                     halo_stream_t stream) {
    if (!in || !out || !cos_sin) return fail(HALO_ERR_INVALID_ARGUMENT, "rope: null pointer");
    if (rows < 0 || seq <= 0 || head_dim % 16 || rot_heads < 0 || rot_heads > heads)
        return fail(HALO_ERR_INVALID_ARGUMENT, "rope: head_dim % 16, 0 <= rot_heads <= heads, seq > 0");
    ProfScope ps(PC_GLUE, (double)rows * heads * head_dim * 4, (cudaStream_t)stream);
    run_rope(in, out, cos_sin, rows, seq, rot_heads, heads, head_dim, backward != 0, (cudaStream_t)stream);
    return cuda_check("rope_qkv");
}

extern "C" halo_status halo_fp6_pack(const uint8_t* codes, uint8_t* packed, int64_t n, halo_stream_t stream) {
    if (!codes || !packed || n < 0 || n % 4) return fail(HALO_ERR_INVALID_ARGUMENT, "fp6_pack: n must be a multiple of 4");
    run_fp6_pack(codes, packed, n, (cudaStream_t)stream);
    return cuda_check("fp6_pack");
}

extern "C" halo_status halo_fp6_unpack(const uint8_t* packed, uint8_t* codes, int64_t n, halo_stream_t stream) {
    if (!codes || !packed || n < 0 || n % 4) return fail(HALO_ERR_INVALID_ARGUMENT, "fp6_unpack: n must be a multiple of 4");
    run_fp6_unpack(packed, codes, n, (cudaStream_t)stream);
    return cuda_check("fp6_unpack");
}

extern "C" halo_status halo_adamw_step(void* param, int32_t p_dtype, const void* grad, int32_t g_dtype, float* m,
                                       float* v, int64_t n, double lr, double beta1, double beta2, double eps,
                                       double weight_decay, double bc1, double bc2, halo_stream_t stream) {
    if (!param || !grad || !m || !v) return fail(HALO_ERR_INVALID_ARGUMENT, "adamw: null pointer");
    if (!valid_dtype(p_dtype) || !valid_dtype(g_dtype)) return fail(HALO_ERR_INVALID_ARGUMENT, "adamw: bad dtype");
    if (n < 0 || n % 4) return fail(HALO_ERR_INVALID_ARGUMENT, "adamw: n must be a non-negative multiple of 4");
    if (!(bc1 > 0.0) || !(bc2 > 0.0)) return fail(HALO_ERR_INVALID_ARGUMENT, "adamw: bias corrections must be > 0");
    if (n == 0) return HALO_OK;
    ProfScope ps(PC_GLUE, (double)n * (2 * dt_bytes(p_dtype) + dt_bytes(g_dtype) + 16), (cudaStream_t)stream);
    run_adamw(param, p_dtype, grad, g_dtype, m, v, n, lr, beta1, beta2, eps, weight_decay, bc1, bc2,
              (cudaStream_t)stream);
    return cuda_check("adamw");
}

extern "C" halo_status halo_profile_enable(int on) {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.on = on != 0;
    return HALO_OK;
}

extern "C" halo_status halo_profile_read(halo_profile* out) {
    if (!out) return fail(HALO_ERR_INVALID_ARGUMENT, "profile_read: null");
    std::memset(out, 0, sizeof(*out));
    if (cudaDeviceSynchronize() != cudaSuccess) return fail(HALO_ERR_CUDA, "profile_read: device error");
    std::lock_guard<std::mutex> lk(g_prof.mu);
    for (const ProfRec& r : g_prof.recs) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        out->launches[r.cls] += 1;
        out->ms[r.cls] += ms;
        out->work[r.cls] += r.work;
        g_prof.pool.push_back(r.a);
        g_prof.pool.push_back(r.b);
    }
    g_prof.recs.clear();
    return HALO_OK;
}
