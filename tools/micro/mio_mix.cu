// Micro-benchmark: do SHFL and LDS share one data pipe?  And how fast can ONE warp per SM sub-partition issue
// independent DFMAs (issue cadence), alone and with 2 / 3 warps?
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double *out, int iters)
{
    __shared__ __align__(16) double sm[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double a0 = lane, a1 = 1, a2 = 2, a3 = 3, a4 = 4, a5 = 5, a6 = 6, a7 = 7;
    int s0 = lane;
    const double *p = sm + lane;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            if (MODE == 0 || MODE == 2) { // LDS.64 32 distinct (2 wavefronts)
                double x; unsigned addr = (unsigned)__cvta_generic_to_shared(p + ((u * 34 + it) & 1023));
                asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(addr)); a0 += x;
            }
            if (MODE == 1 || MODE == 2) { // 2 x SHFL.32
                s0 += __shfl_sync(0xffffffffu, s0, (lane + u) & 31);
                s0 += __shfl_sync(0xffffffffu, s0, (lane + u + 1) & 31);
            }
            if (MODE == 3) { // 8 independent DFMA chains
                a0 = fma(a0, 1.0000001, 1e-9); a1 = fma(a1, 1.0000001, 1e-9); a2 = fma(a2, 1.0000001, 1e-9); a3 = fma(a3, 1.0000001, 1e-9);
                a4 = fma(a4, 1.0000001, 1e-9); a5 = fma(a5, 1.0000001, 1e-9); a6 = fma(a6, 1.0000001, 1e-9); a7 = fma(a7, 1.0000001, 1e-9);
            }
        }
    }
    if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 + s0 == 1.2345) out[0] = a0;
}
template <int MODE>
void run(const char *name, int threads, double per_iter_ops)
{
    double *out; cudaMalloc(&out, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 2048, blocks = 148;
    k<MODE><<<blocks, threads>>>(out, 16);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double cycles = ms * 1e-3 * 1.965e9;
    double warps = threads / 32.0;
    printf("%-52s warps/SM %2.0f: %.2f cycles per (warp x unrolled step), %.2f SM-cycles per op\n", name, warps, cycles / (iters * 16.0),
           cycles / (iters * 16.0 * warps * per_iter_ops));
    cudaFree(out);
}
int main()
{
    for (int th : {128, 256, 512}) {
        run<0>("LDS.64 distinct", th, 1);
        run<1>("2 x SHFL.32", th, 2);
        run<2>("LDS.64 distinct + 2 x SHFL.32", th, 3);
    }
    for (int th : {128, 256, 384, 512}) run<3>("8 independent DFMA per step", th, 8);
    return 0;
}
