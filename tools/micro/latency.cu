// Micro-benchmark: dependent-chain latencies (cycles) of the instructions the tiled kernel is made of.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(long long *out, double a, double b, int n)
{
    __shared__ double sm[64];
    sm[threadIdx.x & 63] = 1.0 + threadIdx.x;
    __syncwarp();
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) x = fma(x, a, b);
    }
    long long t1 = clock64();
    double y = x;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) y = __shfl_sync(0xffffffffu, y, (u + 1) & 15, 16);
    }
    long long t2 = clock64();
    double z = y;
    int idx = threadIdx.x & 31;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) { z = sm[idx]; idx = ((int)z + u) & 31; }
    }
    long long t3 = clock64();
    double w = z;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) { w = fma(w, a, b); w = __shfl_sync(0xffffffffu, w, 3, 16); }
    }
    long long t4 = clock64();
    double m = w;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) m = m * a;
    }
    long long t5 = clock64();
    float f = (float)m;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) f = fmaf(f, 1.0001f, 0.5f);
    }
    long long t6 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; out[4] = t5 - t4; out[5] = t6 - t5;
    }
    if (x + y + z + w + m + f == 1.2345) out[7] = 1;
}
int main()
{
    long long *d, h[8];
    cudaMalloc(&d, 64);
    const int n = 256;
    for (int rep = 0; rep < 2; ++rep) {
        lat<<<1, 32>>>(d, 0.999, 1e-3, n);
        cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
    }
    double k = n * 16.0;
    printf("dependent DFMA          %.1f cycles\n", h[0] / k);
    printf("dependent SHFL (double) %.1f cycles (2 x 32-bit shuffles)\n", h[1] / k);
    printf("dependent LDS.64 + cvt  %.1f cycles (includes F2I + IADD + LOP)\n", h[2] / k);
    printf("DFMA -> SHFL(double)    %.1f cycles per pair\n", h[3] / k);
    printf("dependent DMUL          %.1f cycles\n", h[4] / k);
    printf("dependent FFMA          %.1f cycles\n", h[5] / k);
    return 0;
}
