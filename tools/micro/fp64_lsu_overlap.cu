// Micro-benchmark: do FP64 (DFMA) and shared-memory / shuffle instructions overlap on B200, or do they
// contend for one dispatch path?  Per unrolled step: 8 independent DFMA (mode bit 0), 4 LDS.64 with 32
// distinct addresses (bit 1), 4 independent SHFL.32 (bit 2), 8 independent FFMA (bit 3).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double *out, int iters)
{
    __shared__ __align__(16) double sm[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double a0 = lane, a1 = 1, a2 = 2, a3 = 3, a4 = 4, a5 = 5, a6 = 6, a7 = 7, l0 = 0, l1 = 0, l2 = 0, l3 = 0;
    float f0 = lane, f1 = 1, f2 = 2, f3 = 3, f4 = 4, f5 = 5, f6 = 6, f7 = 7;
    int s0 = lane, s1 = lane + 1, s2 = lane + 2, s3 = lane + 3;
    const double *p = sm + lane;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (MODE & 2) {
                double x0, x1, x2, x3; unsigned addr = (unsigned)__cvta_generic_to_shared(p + ((u * 34 + it) & 1023));
                asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x0) : "r"(addr));
                asm volatile("ld.shared.f64 %0, [%1+256];" : "=d"(x1) : "r"(addr));
                asm volatile("ld.shared.f64 %0, [%1+512];" : "=d"(x2) : "r"(addr));
                asm volatile("ld.shared.f64 %0, [%1+768];" : "=d"(x3) : "r"(addr));
                l0 += x0; l1 += x1; l2 += x2; l3 += x3;   // (4 DADD: counted with the loads)
            }
            if (MODE & 4) {
                s0 = __shfl_sync(0xffffffffu, s0, (lane + 1) & 31); s1 = __shfl_sync(0xffffffffu, s1, (lane + 2) & 31);
                s2 = __shfl_sync(0xffffffffu, s2, (lane + 3) & 31); s3 = __shfl_sync(0xffffffffu, s3, (lane + 4) & 31);
            }
            if (MODE & 1) {
                a0 = fma(a0, 1.0000001, 1e-9); a1 = fma(a1, 1.0000001, 1e-9); a2 = fma(a2, 1.0000001, 1e-9); a3 = fma(a3, 1.0000001, 1e-9);
                a4 = fma(a4, 1.0000001, 1e-9); a5 = fma(a5, 1.0000001, 1e-9); a6 = fma(a6, 1.0000001, 1e-9); a7 = fma(a7, 1.0000001, 1e-9);
            }
            if (MODE & 8) {
                f0 = fmaf(f0, 1.0001f, 1e-3f); f1 = fmaf(f1, 1.0001f, 1e-3f); f2 = fmaf(f2, 1.0001f, 1e-3f); f3 = fmaf(f3, 1.0001f, 1e-3f);
                f4 = fmaf(f4, 1.0001f, 1e-3f); f5 = fmaf(f5, 1.0001f, 1e-3f); f6 = fmaf(f6, 1.0001f, 1e-3f); f7 = fmaf(f7, 1.0001f, 1e-3f);
            }
        }
    }
    if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 + l0 + l1 + l2 + l3 + s0 + s1 + s2 + s3 + f0 + f1 + f2 + f3 + f4 + f5 + f6 + f7 == 1.2345) out[0] = a0;
}
template <int MODE>
void run(const char *name)
{
    double *out; cudaMalloc(&out, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 2048, blocks = 148, threads = 384; // 12 warps per SM, like the kernel
    k<MODE><<<blocks, threads>>>(out, 16);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double cycles = ms * 1e-3 * 1.965e9;
    printf("%-44s %.1f SM-cycles per (12 warps x 1 unrolled step)\n", name, cycles / (iters * 8.0));
    cudaFree(out);
}
int main()
{
    run<1>("8 DFMA");
    run<2>("4 LDS.64 distinct (+4 DADD)");
    run<3>("8 DFMA + 4 LDS.64 (+4 DADD)");
    run<4>("4 SHFL.32");
    run<5>("8 DFMA + 4 SHFL.32");
    run<6>("4 LDS.64 (+4 DADD) + 4 SHFL.32");
    run<7>("8 DFMA + 4 LDS.64 (+4 DADD) + 4 SHFL.32");
    run<8>("8 FFMA");
    run<9>("8 DFMA + 8 FFMA");
    run<10>("8 FFMA + 4 LDS.64 (+4 DADD)");
    return 0;
}
