// Micro-benchmark: do three-register-operand DFMAs and LDS.128 write-backs contend (register-file bandwidth)?
// Per unrolled step and warp: 8 DFMA fma(b_i, c_i, a_i) with all operands in registers (bit 0) and/or
// 2 broadcast LDS.128 whose results feed the next step's multipliers (bit 1).  12 warps per SM.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double *out, const double *in, int iters)
{
    __shared__ __align__(16) double sm[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) sm[i] = 1.0 + 1e-9 * i;
    __syncthreads();
    double a[8], b[8], c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = in[threadIdx.x + i]; b[i] = in[threadIdx.x + 8 + i]; c[i] = in[threadIdx.x + 16 + i]; }
    double2 v0 = make_double2(1.0, 1.0), v1 = v0;
    double s0 = 0, s1 = 0;
    const int g = (threadIdx.x & 31) >> 4;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (MODE & 2) {
                const double *p = sm + g * 18 + ((u * 34 + it * 2) & 1023);
                v0 = *reinterpret_cast<const double2 *>(p);
                v1 = *reinterpret_cast<const double2 *>(p + 512);
                if (!(MODE & 1)) { s0 += v0.x + v0.y; s1 += v1.x + v1.y; }
            }
            if (MODE & 1) {
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    a[i] = fma(b[i], (MODE & 2) ? ((i & 2) ? ((i & 1) ? v1.y : v1.x) : ((i & 1) ? v0.y : v0.x)) : c[i], a[i]);
            }
        }
    }
    double s = s0 + s1;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 1.2345) out[0] = s;
}
template <int MODE>
void run(const char *name)
{
    double *out, *in; cudaMalloc(&out, 8); cudaMalloc(&in, 8 * 2048); cudaMemset(in, 0, 8 * 2048);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 4096, blocks = 148, threads = 384;
    k<MODE><<<blocks, threads>>>(out, in, 16);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    k<MODE><<<blocks, threads>>>(out, in, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double cycles = ms * 1e-3 * 1.965e9;
    printf("%-60s %.1f SM-cycles per (12 warps x 1 unrolled step)\n", name, cycles / (iters * 8.0));
    cudaFree(out); cudaFree(in);
}
int main()
{
    run<1>("8 DFMA fma(b_i, c_i, a_i), three register operands");
    run<2>("2 broadcast LDS.128 (+4 DADD)");
    run<3>("8 DFMA fma(b_i, v_loaded, a_i) + 2 broadcast LDS.128");
    return 0;
}
