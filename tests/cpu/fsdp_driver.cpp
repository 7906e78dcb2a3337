// fsdp_driver.cpp — a C++ trainer step over the C ABI with the HQ-FSDP NCCL
// data plane, no Python:
//   quantized_all_gather -> forward -> backward_regather (stale check) ->
//   backward -> reduce_scatter_grads,   one HALO-2 INT8 layer.
// Usage: fsdp_driver <dir> <b> <m> <n> <block> <world> <rank>
//   reads X.f32 W.f32 E.f32 (rank 0 writes the NCCL id to <dir>/id, other
//   ranks wait for it); writes Y.out EX.out GW<rank>.out (this rank's dW
//   rows) and prints "stale-before <f> stale-after <f>".
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#include "../../include/halo_b200.h"

#define CK(x)                                                                         \
    do {                                                                              \
        halo_status s_ = (x);                                                         \
        if (s_ != HALO_OK) {                                                          \
            std::printf("FAIL %s: %d %s\n", #x, (int)s_, halo_last_error());           \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

static std::vector<float> rd(const std::string& p, size_t n) {
    std::vector<float> v(n);
    std::ifstream f(p, std::ios::binary);
    f.read(reinterpret_cast<char*>(v.data()), n * 4);
    return v;
}
static void wr(const std::string& p, const float* d, size_t n) {
    std::vector<float> h(n);
    cudaMemcpy(h.data(), d, n * 4, cudaMemcpyDeviceToHost);
    std::ofstream f(p, std::ios::binary);
    f.write(reinterpret_cast<const char*>(h.data()), n * 4);
}
static __nv_bfloat16* up_bf16(const std::vector<float>& v) {
    std::vector<__nv_bfloat16> h(v.size());
    for (size_t i = 0; i < v.size(); ++i) h[i] = __float2bfloat16(v[i]);  // inputs are bf16-exact
    __nv_bfloat16* d;
    cudaMalloc(&d, h.size() * 2);
    cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    return d;
}

int main(int argc, char** argv) {
    if (argc < 8) return 2;
    const std::string dir = argv[1];
    const int64_t b = std::atoll(argv[2]), m = std::atoll(argv[3]), n = std::atoll(argv[4]), blk = std::atoll(argv[5]);
    const int world = std::atoi(argv[6]), rank = std::atoi(argv[7]);
    const int64_t rows = n / world;  // n divisible by world here (no padding)
    char id[HALO_FSDP_ID_BYTES];
    if (rank == 0) {
        CK(halo_fsdp_get_unique_id(id));
        std::ofstream(dir + "/id.tmp", std::ios::binary).write(id, sizeof(id));
        std::rename((dir + "/id.tmp").c_str(), (dir + "/id").c_str());
    } else {
        for (;;) {
            std::ifstream f(dir + "/id", std::ios::binary);
            if (f && f.read(id, sizeof(id))) break;
            std::this_thread::sleep_for(std::chrono::milliseconds(20));
        }
    }
    halo_fsdp* fs = nullptr;
    CK(halo_fsdp_create(id, world, rank, &fs));
    cudaStream_t st;
    cudaStreamCreate(&st);
    const auto X = rd(dir + "/X.f32", b * m), W = rd(dir + "/W.f32", n * m), E = rd(dir + "/E.f32", b * n);
    std::vector<float> Wl(W.begin() + rank * rows * m, W.begin() + (rank + 1) * rows * m);
    __nv_bfloat16 *dx = up_bf16(X), *dw = up_bf16(Wl), *de = up_bf16(E);
    uint8_t* gathered;
    float *scale, *amax, *y, *ex, *gw, *gshard;
    uint32_t* stale;
    cudaMalloc(&gathered, n * m);
    cudaMalloc(&scale, 4);
    cudaMalloc(&amax, 4);
    cudaMalloc(&stale, 4);
    cudaMemset(stale, 0, 4);
    cudaMalloc(&y, b * n * 4);
    cudaMalloc(&ex, b * m * 4);
    cudaMalloc(&gw, n * m * 4);
    cudaMalloc(&gshard, rows * m * 4);
    halo_scheme sch;
    CK(halo_scheme_from_string("halo2", HALO_FMT_INT8, blk, &sch));
    halo_linear* layer = nullptr;
    halo_ctx* ctx = nullptr;
    CK(halo_linear_create(&sch, dw /* placeholder: codes are installed */, HALO_DTYPE_BF16, n, m, &layer));
    CK(halo_ctx_create(&ctx));
    // forward: gather (WH)_Q under the shared scale, install, run
    CK(halo_fsdp_quantized_all_gather(fs, dw, HALO_DTYPE_BF16, rows, m, blk, HALO_FMT_INT8, gathered, scale, amax, st));
    CK(halo_linear_set_qweight(layer, gathered, scale));
    CK(halo_linear_forward(layer, dx, HALO_DTYPE_BF16, b, y, HALO_DTYPE_F32, ctx, st));
    if (std::getenv("HALO_DRIVER_DUMP")) {
        const uint8_t *xq, *wq;
        const float *sx, *sw;
        int64_t br;
        CK(halo_ctx_saved(ctx, &xq, &sx, &wq, &sw, &br));
        cudaStreamSynchronize(st);
        std::vector<uint8_t> h(b * m);
        cudaMemcpy(h.data(), xq, b * m, cudaMemcpyDeviceToHost);
        std::ofstream(dir + "/xq.out", std::ios::binary).write(reinterpret_cast<const char*>(h.data()), b * m);
        float sxh = 0, swh = 0;
        cudaMemcpy(&sxh, sx, 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(&swh, sw, 4, cudaMemcpyDeviceToHost);
        std::printf("sx %.9g sw %.9g\n", sxh, swh);
    }
    // backward: regather under the saved scale (the codes the backward reads)
    CK(halo_fsdp_backward_regather(fs, dw, HALO_DTYPE_BF16, rows, m, blk, HALO_FMT_INT8, scale, amax, stale, gathered, st));
    CK(halo_linear_backward(layer, ctx, de, HALO_DTYPE_BF16, ex, HALO_DTYPE_F32, gw, HALO_DTYPE_F32, st));
    CK(halo_fsdp_reduce_scatter(fs, gw, HALO_DTYPE_F32, rows, m, gshard, st));
    CK(halo_ctx_check(ctx, st));
    uint32_t s_before = 0, s_after = 0;
    cudaMemcpy(&s_before, stale, 4, cudaMemcpyDeviceToHost);
    // a master changed after the forward gather trips the stale flag
    const __nv_bfloat16 one = __float2bfloat16(3.0f);
    cudaMemcpy(dw, &one, 2, cudaMemcpyHostToDevice);
    CK(halo_fsdp_backward_regather(fs, dw, HALO_DTYPE_BF16, rows, m, blk, HALO_FMT_INT8, scale, amax, stale, gathered, st));
    cudaStreamSynchronize(st);
    cudaMemcpy(&s_after, stale, 4, cudaMemcpyDeviceToHost);
    if (rank == 0) {
        wr(dir + "/Y.out", y, b * n);
        wr(dir + "/EX.out", ex, b * m);
    }
    wr(dir + "/GW" + std::to_string(rank) + ".out", gshard, rows * m);
    std::printf("stale-before %u stale-after %u\n", s_before, s_after);
    halo_linear_destroy(layer);
    halo_ctx_destroy(ctx);
    halo_fsdp_destroy(fs);
    return 0;
}
