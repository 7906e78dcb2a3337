// Throughput of conversion / fp64 instructions on this GPU: 8 independent
// chains per thread, 1024 threads per SM; prints instructions/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
template <int OP>
__global__ void k(const int* in, float* out, long long* cyc, int iters) {
    int a[8]; float f[8]; double d[8];
    for (int i = 0; i < 8; ++i) { a[i] = in[threadIdx.x + i] + i; f[i] = (float)a[i] * 1.0001f; d[i] = f[i]; }
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) { f[i] = __int2float_rn(a[i]); a[i] = __float_as_int(f[i]) ^ it; }          // I2FP + LOP
            if (OP == 1) { a[i] = __float2int_rz(f[i]); f[i] = __int_as_float(a[i] ^ 0x3f800000); }  // F2I + LOP
            if (OP == 2) d[i] = d[i] * 1.0000001;                                                       // DMUL
            if (OP == 3) { d[i] = (double)a[i]; a[i] = (int)(__double2hiint(d[i]) ^ it); }             // I2F.F64 + ...
            if (OP == 4) { f[i] = (float)d[i]; d[i] = __hiloint2double(__float_as_int(f[i]) ^ it, it); } // F2F.F32.F64
            if (OP == 5) f[i] = f[i] * 1.0001f + 0.5f;                                                 // FFMA
            if (OP == 6) { __nv_bfloat162 h = __floats2bfloat162_rn(f[i], f[(i + 1) & 7]);             // F2FP.BF16
                           f[i] = __int_as_float(*reinterpret_cast<int*>(&h) ^ it); }
            if (OP == 7) { a[i] = a[i] * 7 + it; }                                                      // IMAD
        }
    }
    long long t1 = clock64();
    float s = 0; for (int i = 0; i < 8; ++i) s += f[i] + (float)a[i] + (float)d[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    int* in; float* out; long long* cyc;
    cudaMalloc(&in, 4096 * 4); cudaMemset(in, 1, 4096 * 4);
    cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 8);
    const char* names[] = {"I2FP.F32.S32 (+LOP)", "F2I.TRUNC (+LOP)", "DMUL", "I2F.F64 (+MOV,LOP)", "F2F.F32.F64 (+...)",
                           "FFMA", "F2FP.BF16 pack (+LOP)", "IMAD"};
    for (int op = 0; op < 8; ++op) {
        const int iters = 1000, threads = 1024;
        void (*kern)(const int*, float*, long long*, int) = op == 0 ? k<0> : op == 1 ? k<1> : op == 2 ? k<2> : op == 3 ? k<3> : op == 4 ? k<4> : op == 5 ? k<5> : op == 6 ? k<6> : k<7>;
        kern<<<148, threads>>>(in, out, cyc, iters);
        cudaDeviceSynchronize();
        kern<<<148, threads>>>(in, out, cyc, iters);
        cudaDeviceSynchronize();
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        const double ops = (double)threads * iters * 8;
        printf("%-24s %8.2f per clk per SM  (%s)\n", names[op], ops / c, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
