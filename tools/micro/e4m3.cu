// Check the hardware e4m3x2 conversion: byte order, rounding, and how often
// the bracketed conversions disagree.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cstring>
#include <cmath>
__global__ void k(const float* x, uint32_t* w, int n, float lo, float hi, unsigned* cnt) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i * 4 + 3 >= n) return;
    float a0 = x[4*i], a1 = x[4*i+1], c0 = x[4*i+2], c1 = x[4*i+3];
    uint32_t wl, wh, wm;
    asm("{\n\t.reg .b16 l, h;\n\tcvt.rn.satfinite.e4m3x2.f32 l, %2, %1;\n\tcvt.rn.satfinite.e4m3x2.f32 h, %4, %3;\n\tmov.b32 %0, {l, h};\n\t}" : "=r"(wm) : "f"(a0), "f"(a1), "f"(c0), "f"(c1));
    asm("{\n\t.reg .b16 l, h;\n\tcvt.rn.satfinite.e4m3x2.f32 l, %2, %1;\n\tcvt.rn.satfinite.e4m3x2.f32 h, %4, %3;\n\tmov.b32 %0, {l, h};\n\t}" : "=r"(wl) : "f"(a0*lo), "f"(a1*lo), "f"(c0*lo), "f"(c1*lo));
    asm("{\n\t.reg .b16 l, h;\n\tcvt.rn.satfinite.e4m3x2.f32 l, %2, %1;\n\tcvt.rn.satfinite.e4m3x2.f32 h, %4, %3;\n\tmov.b32 %0, {l, h};\n\t}" : "=r"(wh) : "f"(a0*hi), "f"(a1*hi), "f"(c0*hi), "f"(c1*hi));
    w[i] = wm;
    if (wl != wh) atomicAdd(cnt, 1u);
}
int main() {
    const int n = 1 << 20;
    float* hx = new float[n];
    unsigned s = 12345;
    // bf16-rounded gaussian-ish values scaled like E_Y codes: y = x * inv, inv = 448 / absmax
    float amax = 0;
    for (int i = 0; i < n; ++i) {
        float u = 0; for (int j = 0; j < 4; ++j) { s = s * 1664525u + 1013904223u; u += (s >> 8) * (1.0f / 16777216.0f) - 0.5f; }
        float x = u * 1e-3f; unsigned b; memcpy(&b, &x, 4); b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000u; memcpy(&x, &b, 4);
        hx[i] = x; amax = fabsf(x) > amax ? fabsf(x) : amax;
    }
    const float sc = (float)((double)amax / 448.0), inv = 1.0f / sc;
    for (int i = 8; i < n; ++i) hx[i] *= inv;
    hx[0] = 1.0f; hx[1] = 2.0f; hx[2] = 3.0f; hx[3] = -1.0f;   // bytes: 0x38 0x40 0x44 0xB8
    hx[4] = 1.0625f; hx[5] = 1.1875f; hx[6] = -0.0001f; hx[7] = 500.f;  // tie->1.0 (0x38), tie->1.25 (0x3A), -0 (0x80), 448 (0x7E)
    float* dx; uint32_t* dw; unsigned* dc;
    cudaMalloc(&dx, n * 4); cudaMalloc(&dw, n); cudaMalloc(&dc, 4);
    cudaMemcpy(dx, hx, n * 4, cudaMemcpyHostToDevice); cudaMemset(dc, 0, 4);
    k<<<(n / 4 + 255) / 256, 256>>>(dx, dw, n, 1.0f - 4.76837158203125e-07f, 1.0f + 4.76837158203125e-07f, dc);
    uint32_t hw[2]; unsigned c;
    cudaMemcpy(hw, dw, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&c, dc, 4, cudaMemcpyDeviceToHost);
    printf("word0 %08x (want b8443840)  word1 %08x (want 7e803a38)\n", hw[0], hw[1]);
    printf("bracket disagreements: %u of %d words (%s)\n", c, n / 4, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
