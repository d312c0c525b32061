// Micro-benchmark: DFMA throughput as a function of how many REGISTER operands it reads
// (the peak microbenchmark used fma(a, const, const); the factorization issues fma(-L, v, K) with three
// 64-bit register operands).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double *out, const double *in, int iters)
{
    double a[8], b[8], c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = in[threadIdx.x + i]; b[i] = in[threadIdx.x + 8 + i]; c[i] = in[threadIdx.x + 16 + i]; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (MODE == 0) a[i] = fma(a[i], 1.0000001, 1e-9);          // 1 register operand
                if (MODE == 1) a[i] = fma(a[i], b[i], 1e-9);               // 2 register operands
                if (MODE == 2) a[i] = fma(b[i], c[i], a[i]);               // 3 distinct register operands
                if (MODE == 3) a[i] = fma(b[0], c[i], a[i]);               // 3, one shared multiplier (like -L * v + K)
                if (MODE == 4) a[i] = fma(b[i & 1], c[i >> 1], a[i]);      // 2 multipliers x 4 values (S = 2 rows)
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 1.2345) out[0] = s;
}
template <int MODE>
void run(const char *name, int threads)
{
    double *out, *in; cudaMalloc(&out, 8); cudaMalloc(&in, 8 * 2048); cudaMemset(in, 0, 8 * 2048);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096, blocks = 148;
    k<MODE><<<blocks, threads>>>(out, in, 16);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(out, in, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double cycles = ms * 1e-3 * 1.965e9;
    printf("%-52s warps/SM %2d: %.3f SM-cycles per warp-DFMA (%.1f FMA lanes/clk/SM)\n", name, threads / 32,
           cycles / (iters * 32.0 * (threads / 32)), 32.0 / (cycles / (iters * 32.0 * (threads / 32))));
    cudaFree(out); cudaFree(in);
}
int main()
{
    for (int th : {128, 384}) {
        run<0>("fma(a, const, const)", th);
        run<1>("fma(a, b, const)", th);
        run<2>("fma(b, c, a) all distinct", th);
        run<3>("fma(b0, c_i, a_i) shared multiplier", th);
        run<4>("fma(b_{i&1}, c_{i>>1}, a_i) 2 multipliers x 4 values", th);
    }
    return 0;
}
