// integration_adapter.cpp — INTEGRATION.md §1 compiled: the adapter a
// reference maintainer adds (halo::Tensor in, halo::Tensor out) over
// include/halo_b200.hpp, run against the UNMODIFIED reference layer
// (halo_linear.hpp) on the same inputs.  Built against /root/reference's
// headers by oracle/Makefile (target `adapter`, output oracle/_ref/).
//   integration_adapter host   -> exception mapping only (no GPU)
//   integration_adapter gpu    -> Y / E_X / grad_W equal the reference's
#define HALO_B200_REFERENCE_EXCEPTIONS 1
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <type_traits>

#include "halo/halo_linear.hpp"
#include "halo_b200.hpp"

static_assert(std::is_same_v<halo_b200::numeric_error, halo::numeric_error>,
              "the C++ API throws the reference's numeric_error");

// ---- the adapter
struct B200HaloLinear {
    float *w = nullptr, *x = nullptr, *y = nullptr, *e = nullptr, *ex = nullptr, *gw = nullptr;
    int64_t n, m;
    halo_b200::HaloLinearLayer layer;
    halo_b200::SavedContext ctx;

    B200HaloLinear(const halo::Tensor& W, int64_t had_block)
        : n(W.rows()), m(W.cols()),
          layer((cudaMalloc(&w, W.size() * 4), w), W.rows(), W.cols(), halo_b200::halo2(HALO_FMT_INT8, had_block),
                HALO_DTYPE_F32) {
        cudaMemcpy(w, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
    }
    ~B200HaloLinear() {
        for (float* p : {w, x, y, e, ex, gw}) cudaFree(p);
    }
    halo::Tensor forward(const halo::Tensor& X) {  // halo_linear.hpp:267
        const int64_t b = X.rows();
        cudaMalloc(&x, X.size() * 4);
        cudaMalloc(&y, b * n * 4);
        cudaMemcpy(x, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
        layer.forward(x, b, y, ctx, nullptr, HALO_DTYPE_F32, HALO_DTYPE_F32);
        halo::Tensor Y(b, n);
        cudaMemcpy(Y.data(), y, Y.size() * 4, cudaMemcpyDeviceToHost);
        return Y;
    }
    halo::BackwardResultT<float> backward(const halo::Tensor& EY) {  // halo_linear.hpp:305
        const int64_t b = EY.rows();
        cudaMalloc(&e, EY.size() * 4);
        cudaMalloc(&ex, b * m * 4);
        cudaMalloc(&gw, n * m * 4);
        cudaMemcpy(e, EY.data(), EY.size() * 4, cudaMemcpyHostToDevice);
        layer.backward(ctx, e, ex, gw, nullptr, HALO_DTYPE_F32, HALO_DTYPE_F32, HALO_DTYPE_F32);
        ctx.check_numeric();
        halo::BackwardResultT<float> r;
        r.e_x = halo::Tensor(b, m);
        r.grad_w = halo::Tensor(n, m);
        cudaMemcpy(r.e_x.data(), ex, r.e_x.size() * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(r.grad_w.data(), gw, r.grad_w.size() * 4, cudaMemcpyDeviceToHost);
        return r;
    }
};

static int differ(const halo::Tensor& a, const halo::Tensor& b) {
    if (a.rows() != b.rows() || a.cols() != b.cols()) return -1;
    int d = 0;
    for (halo::index_t i = 0; i < a.size(); ++i) d += std::memcmp(&a.data()[i], &b.data()[i], 4) != 0;
    return d;
}

int main(int argc, char** argv) {
    // a reference caller's divergence handler (halo_cli.cpp:730-732) catches
    // the device path's numeric errors
    int fails = 0;
    try {
        halo_b200::check(HALO_ERR_NUMERIC);
    } catch (const halo::numeric_error&) {
    } catch (...) {
        ++fails;
    }
    if (argc > 1 && std::strcmp(argv[1], "gpu") == 0) {
        const halo::index_t b = 64, m = 256, n = 128;  // power-of-two dims: had_block 0 == the reference transform
        halo::Tensor X = halo::randn<float>(b, m, 1), W = halo::randn<float>(n, m, 2, 1.0 / 16), E = halo::randn<float>(b, n, 3, 1e-3);
        for (halo::index_t i = 0; i < b; ++i) X(i, 3) *= 40.0f;
        halo::HaloLinearLayer ref(W, halo::halo2());
        halo::SavedContext rctx;
        const halo::Tensor ry = ref.forward(X, rctx);
        const halo::BackwardResultT<float> rb = ref.backward(rctx, E);
        B200HaloLinear dev(W, 0);
        const halo::Tensor y = dev.forward(X);
        const halo::BackwardResultT<float> bb = dev.backward(E);
        const int dy = differ(y, ry), dex = differ(bb.e_x, rb.e_x), dgw = differ(bb.grad_w, rb.grad_w);
        std::printf("Y %d E_X %d grad_W %d differing elements\n", dy, dex, dgw);
        fails += (dy != 0) + (dex != 0) + (dgw != 0);
    }
    std::printf("%d failures\n", fails);
    return fails ? 1 : 0;
}
