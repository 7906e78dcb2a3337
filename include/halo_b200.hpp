// halo_b200.hpp — header-only C++ object API over the C ABI (halo_b200.h),
// restoring the reference's operator surface (halo_linear.hpp:227-462):
//
//   halo_b200::HaloLinearLayer layer(w, n, m, halo_b200::halo2(INT8, 256));
//   halo_b200::SavedContext ctx;
//   layer.forward(x, b, y, ctx, stream);                 // forward(x, ctx)
//   layer.backward(ctx, e_y, e_x, grad_w, stream);       // backward(ctx, e_y)
//   layer.counters();                                    // QuantCallCounters
//
// Tensors are device pointers (row-major, caller-owned).  Status codes are
// rethrown as the reference's exception types: std::invalid_argument,
// numeric_error, std::logic_error, halo_b200::io_error (HALO_ERR_IO) and
// std::runtime_error for CUDA / NCCL failures.
//
// numeric_error: define HALO_B200_REFERENCE_EXCEPTIONS before including this
// header (with the reference's include dir on the path) and it IS
// halo::numeric_error (tensor.hpp:21-23), so a reference caller's divergence
// handler (halo_cli.cpp:730-732) catches it; otherwise a standalone type of
// the same shape.
#pragma once

#include <stdexcept>
#include <string>

#include "halo_b200.h"

#ifdef HALO_B200_REFERENCE_EXCEPTIONS
#include <halo/tensor.hpp>
#endif

namespace halo_b200 {

#ifdef HALO_B200_REFERENCE_EXCEPTIONS
using numeric_error = ::halo::numeric_error;
#else
struct numeric_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
#endif
struct io_error : std::runtime_error {  // tensor_io.hpp:25-27
    using std::runtime_error::runtime_error;
};

inline void check(halo_status s) {
    switch (s) {
    case HALO_OK: return;
    case HALO_ERR_INVALID_ARGUMENT: throw std::invalid_argument(halo_last_error());
    case HALO_ERR_NUMERIC: throw numeric_error(halo_last_error());
    case HALO_ERR_LOGIC: throw std::logic_error(halo_last_error());
    case HALO_ERR_IO: throw io_error(halo_last_error());
    default: throw std::runtime_error(std::string("halo_b200: ") + halo_last_error());
    }
}

// halo_linear.hpp:81-152
inline halo_scheme scheme_from_string(const std::string& id, halo_format f = HALO_FMT_INT8, int64_t had_block = 0) {
    halo_scheme s;
    check(halo_scheme_from_string(id.c_str(), f, had_block, &s));
    return s;
}
inline halo_scheme halo0(halo_format f = HALO_FMT_INT8, int64_t had_block = 0) { return scheme_from_string("halo0", f, had_block); }
inline halo_scheme halo1(halo_format f = HALO_FMT_INT8, int64_t had_block = 0) { return scheme_from_string("halo1", f, had_block); }
inline halo_scheme halo2(halo_format f = HALO_FMT_INT8, int64_t had_block = 0) { return scheme_from_string("halo2", f, had_block); }

inline std::string to_string(const halo_scheme& s) {  // halo_linear.hpp:154-159
    if (s.name[0]) return s.name;
    auto p = [](const halo_placement& q) {
        std::string r;
        if (q.left) r += 'L';
        if (q.middle) r += 'M';
        if (q.right) r += 'R';
        return r.empty() ? std::string("O") : r;
    };
    return "F:" + p(s.F) + ";E:" + p(s.E) + ";G:" + p(s.G);
}

// SavedContextT (halo_linear.hpp:207-216): device-resident (XH)_Q, (WH)_Q
class SavedContext {
public:
    SavedContext() { check(halo_ctx_create(&h_)); }
    ~SavedContext() { halo_ctx_destroy(h_); }
    SavedContext(const SavedContext&) = delete;
    SavedContext& operator=(const SavedContext&) = delete;
    halo_ctx* get() const { return h_; }
    void check_numeric(halo_stream_t st = nullptr) { check(halo_ctx_check(h_, st)); }

private:
    halo_ctx* h_ = nullptr;
};

class HaloLinearLayer {
public:
    // HaloLinearLayerT(W, scheme), halo_linear.hpp:230-234 (W: n x m, device)
    HaloLinearLayer(const void* w, int64_t out_features, int64_t in_features, const halo_scheme& scheme,
                    halo_dtype w_dtype = HALO_DTYPE_BF16)
        : n_(out_features), m_(in_features), scheme_(scheme) {
        check(halo_linear_create(&scheme_, w, w_dtype, out_features, in_features, &h_));
    }
    ~HaloLinearLayer() { halo_linear_destroy(h_); }
    HaloLinearLayer(const HaloLinearLayer&) = delete;
    HaloLinearLayer& operator=(const HaloLinearLayer&) = delete;

    int64_t in_features() const { return m_; }
    int64_t out_features() const { return n_; }
    const halo_scheme& scheme() const { return scheme_; }

    void set_weight(const void* w, halo_dtype dt = HALO_DTYPE_BF16) { check(halo_linear_set_weight(h_, w, dt)); }
    void set_qweight(const uint8_t* codes, const float* scale) { check(halo_linear_set_qweight(h_, codes, scale)); }

    // forward(x, ctx) -> y  (halo_linear.hpp:267-303)
    void forward(const void* x, int64_t batch, void* y, SavedContext& ctx, halo_stream_t st = nullptr,
                 halo_dtype x_dtype = HALO_DTYPE_BF16, halo_dtype y_dtype = HALO_DTYPE_BF16) {
        check(halo_linear_forward(h_, x, x_dtype, batch, y, y_dtype, ctx.get(), st));
    }
    // backward(ctx, e_y) -> {e_x, grad_w}  (halo_linear.hpp:305-439)
    void backward(const SavedContext& ctx, const void* e_y, void* e_x, void* grad_w, halo_stream_t st = nullptr,
                  halo_dtype e_dtype = HALO_DTYPE_BF16, halo_dtype ex_dtype = HALO_DTYPE_BF16,
                  halo_dtype gw_dtype = HALO_DTYPE_F32) {
        check(halo_linear_backward(h_, ctx.get(), e_y, e_dtype, e_x, ex_dtype, grad_w, gw_dtype, st));
    }
    // export_inference_weights (halo_linear.hpp:332-338)
    void export_inference_weights(uint8_t* codes, float* scale, halo_stream_t st = nullptr) {
        check(halo_linear_export_inference_weights(h_, codes, scale, st));
    }
    halo_counters counters() const {
        halo_counters c;
        check(halo_linear_counters(h_, &c));
        return c;
    }
    void reset_counters() { check(halo_linear_reset_counters(h_)); }

    // forward on the (XH)_Q already held by `src` (same X quantizer): the
    // Llama gate/up pattern quantizes X once (halo_linear_forward_shared)
    void forward_shared(const SavedContext& src, void* y, SavedContext& ctx, halo_stream_t st = nullptr,
                        int32_t y_dtype = HALO_DTYPE_BF16) const {
        check(halo_linear_forward_shared(h_, src.get(), ctx.get(), y, y_dtype, st));
    }

private:
    int64_t n_, m_;
    halo_scheme scheme_;
    halo_linear* h_ = nullptr;
};

}  // namespace halo_b200
