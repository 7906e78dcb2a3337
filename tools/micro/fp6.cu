// probe: cvt.rn.satfinite.e3m2x2.f32 output layout on sm_100a
#include <cstdio>
#include <cstdint>
__global__ void k(const float* x, uint16_t* out, int n) {
    int i = threadIdx.x;
    if (i < n) {
        uint16_t r;
        asm("cvt.rn.satfinite.e3m2x2.f32 %0, %1, %2;" : "=h"(r) : "f"(x[2 * i]), "f"(x[2 * i + 1]));
        out[i] = r;
    }
}
int main() {
    const int n = 8;
    float hx[2 * n] = {1.0f, 0.0f, 28.0f, -28.0f, 30.0f, 0.0625f, 0.25f, 1.75f, 0.03125f, 0.09375f, -1.0f, 3.0f, 100.f, -0.0f, 0.125f, 0.1875f};
    float* dx; uint16_t* dout; uint16_t hout[n];
    cudaMalloc(&dx, sizeof(hx)); cudaMalloc(&dout, sizeof(hout));
    cudaMemcpy(dx, hx, sizeof(hx), cudaMemcpyHostToDevice);
    k<<<1, 32>>>(dx, dout, n);
    cudaMemcpy(hout, dout, sizeof(hout), cudaMemcpyDeviceToHost);
    for (int i = 0; i < n; ++i) printf("(%g, %g) -> 0x%04x\n", hx[2 * i], hx[2 * i + 1], hout[i]);
    return 0;
}
