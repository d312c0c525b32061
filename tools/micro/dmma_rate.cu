// Micro-benchmark: FP64 tensor-core MMA (mma.sync m8n8k4 f64) issue rate on B200, against the DFMA pipe.
// Informational: the north star excludes tensor cores from this path; the number tells what a tile-fragment
// factorization (rank-k updates inside the MMA datapath, no shared-memory broadcast) could draw on.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, int iters)
{
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) { c[i][0] = threadIdx.x; c[i][1] = i; }
    double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
    if (s == 1.2345) out[0] = s;
}
int main()
{
    double *out; cudaMalloc(&out, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int threads : {128, 256, 512}) {
        const int iters = 8192, blocks = 148 * 2;
        k<<<blocks, threads>>>(out, 16);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        k<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double mmas = (double)iters * 8 * (threads / 32) * blocks;
        const double flops = mmas * 2.0 * 8 * 8 * 4;
        printf("threads/block %3d: %.2f TFLOP/s FP64 via mma.m8n8k4 (%.2f SM-cycles per warp-MMA)\n", threads, flops / (ms * 1e-3) / 1e12,
               ms * 1e-3 * 1.965e9 * 148 / mmas);
    }
    return 0;
}
