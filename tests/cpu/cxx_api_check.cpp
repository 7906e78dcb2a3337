// C++ object API (include/halo_b200.hpp) over libhalo_b200.so.
//   host mode  : scheme parsing, validation and the reference exception
//                types (no device needed)
//   gpu  mode  : HALO-2 INT8 forward + backward on cudaMalloc'd buffers,
//                inputs read from / outputs written to raw files
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <fstream>
#include <vector>

#include "../../include/halo_b200.hpp"

using namespace halo_b200;

static int host_mode() {
    int fails = 0;
    auto expect = [&](bool ok, const char* what) {
        if (!ok) {
            std::printf("FAIL %s\n", what);
            ++fails;
        }
    };
    expect(to_string(halo2()) == "halo2", "preset name");
    const halo_scheme s = scheme_from_string("F:M;E:LR;G:R", HALO_FMT_FP8_E4M3, 256);
    expect(to_string(s) == "F:M;E:LR;G:R" && s.format_x == HALO_FMT_FP8_E4M3, "placement string");
    bool threw = false;
    try {
        scheme_from_string("halo3");
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    expect(threw, "halo3 rejected with std::invalid_argument");
    threw = false;
    try {  // 112 = 7 * 16 is not 2^k, 12*2^k or 20*2^k (hadamard.hpp:69-98)
        HaloLinearLayer l(nullptr, 16, 112, halo1());
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    expect(threw, "unsupported dim rejected");
    HaloLinearLayer ok(nullptr, 128, 256, halo2(HALO_FMT_INT8, 256));
    expect(ok.in_features() == 256 && ok.out_features() == 128, "shape accessors");
    const halo_counters c = ok.counters();
    expect(c.x == 0 && c.w == 0 && c.e == 0, "fresh counters");
    std::printf("host checks: %d failures\n", fails);
    return fails != 0;
}

template <class T>
static std::vector<T> read_file(const char* path, size_t n) {
    std::vector<T> v(n);
    std::ifstream f(path, std::ios::binary);
    f.read(reinterpret_cast<char*>(v.data()), n * sizeof(T));
    return v;
}

static int gpu_mode(const char* dir, int64_t b, int64_t m, int64_t n, int64_t block) {
    const std::string d(dir);
    auto X = read_file<float>((d + "/X.f32").c_str(), b * m);
    auto W = read_file<float>((d + "/W.f32").c_str(), n * m);
    auto E = read_file<float>((d + "/E.f32").c_str(), b * n);
    float *dX, *dW, *dE, *dY, *dEX, *dGW;
    cudaMalloc(&dX, X.size() * 4);
    cudaMalloc(&dW, W.size() * 4);
    cudaMalloc(&dE, E.size() * 4);
    cudaMalloc(&dY, b * n * 4);
    cudaMalloc(&dEX, b * m * 4);
    cudaMalloc(&dGW, n * m * 4);
    cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dE, E.data(), E.size() * 4, cudaMemcpyHostToDevice);
    HaloLinearLayer layer(dW, n, m, halo2(HALO_FMT_INT8, block), HALO_DTYPE_F32);
    SavedContext ctx;
    layer.forward(dX, b, dY, ctx, nullptr, HALO_DTYPE_F32, HALO_DTYPE_F32);
    layer.backward(ctx, dE, dEX, dGW, nullptr, HALO_DTYPE_F32, HALO_DTYPE_F32, HALO_DTYPE_F32);
    ctx.check_numeric();
    std::vector<float> Y(b * n), EX(b * m), GW(n * m);
    cudaMemcpy(Y.data(), dY, Y.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(EX.data(), dEX, EX.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(GW.data(), dGW, GW.size() * 4, cudaMemcpyDeviceToHost);
    std::ofstream((d + "/Y.out").c_str(), std::ios::binary).write(reinterpret_cast<char*>(Y.data()), Y.size() * 4);
    std::ofstream((d + "/EX.out").c_str(), std::ios::binary).write(reinterpret_cast<char*>(EX.data()), EX.size() * 4);
    std::ofstream((d + "/GW.out").c_str(), std::ios::binary).write(reinterpret_cast<char*>(GW.data()), GW.size() * 4);
    const halo_counters c = layer.counters();
    std::printf("counters %lld %lld %lld\n", (long long)c.x, (long long)c.w, (long long)c.e);
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 1 && std::strcmp(argv[1], "gpu") == 0)
        return gpu_mode(argv[2], atoll(argv[3]), atoll(argv[4]), atoll(argv[5]), atoll(argv[6]));
    return host_mode();
}
