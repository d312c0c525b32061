// Micro-benchmark for the FP64 tensor-core arm of the layout study (round-1 verdict, arm ii): a blocked Cholesky
// factorization of 32 x 32 SPD matrices on 8 x 8 register tiles, ONE matrix per warp, trailing updates by
// mma.sync.m8n8k4.f64 (SASS DMMA).  It measures ONLY the factorization (no pair terms, no triangular solves, no
// contraction) so that the number can be put next to the factorization phase of the production kernel
// (profiles/r2_experiments.md: 8 635 cycles per two observations at 12 warps per SM = 1.37 ms of the 4.33 ms at n = 2^20).
//
// Layout: tile (I, J), I >= J, of the lower triangle lives in the C-fragment layout of the MMA: lane = 4 g + t holds
// X[8I + g][8J + 2t] and X[8I + g][8J + 2t + 1] (10 tiles = 20 doubles per lane).  That fragment is directly the A
// operand of L_IJ (k <-> column 2t + s, one MMA per register slot s) AND the B operand of L_KJ^T, so the trailing update
// C_IK -= L_IJ L_KJ^T is two DMMAs with no data movement.  What is NOT free is the scalar part: the 8 x 8 diagonal tile is
// factored column by column with shuffles (pivot, the lane's row entry, the two column entries), and the panel tiles
// below it are solved by the same column sweep (one more shuffle per tile and column).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dmma_chol dmma_chol.cu && ./dmma_chol
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>
#include <vector>

#define FULL 0xffffffffu

__host__ __device__ inline double entry(int a, int c, unsigned id)
{
    if (a < c) {
        const int t = a;
        a = c;
        c = t;
    }
    unsigned h = (unsigned)(a * 73856093u) ^ (unsigned)(c * 19349663u) ^ (id * 83492791u);
    h ^= h >> 13;
    h *= 0x5bd1e995u;
    h ^= h >> 15;
    const double u = (double)(h & 0xffffu) * (1.0 / 65536.0);
    return (a == c) ? 4.0 + u : 0.1 * (u - 0.5);
}

__device__ __forceinline__ double rsqrt_pos(double a)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
    const double e = fma(a, -(y * y), 1.0);
    return fma(fma(e, 0.375, 0.5), y * e, y);
}

__device__ __forceinline__ void dmma_sub(double &c0, double &c1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(-a), "d"(b));
}

// tile index of (I, J), I >= J, in the packed list of 10 lower tiles
__host__ __device__ constexpr int tix(int I, int J) { return I * (I + 1) / 2 + J; }

template <bool FACTOR>
__global__ void __launch_bounds__(128) dmma_chol_kernel(unsigned nmat, double *sums)
{
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    double acc = 0.0;
    for (unsigned id = warp; id < nmat; id += nwarps) {
        double X[10][2];
#pragma unroll
        for (int I = 0; I < 4; ++I)
#pragma unroll
            for (int J = 0; J <= I; ++J) {
                X[tix(I, J)][0] = entry(8 * I + g, 8 * J + 2 * t, id);
                X[tix(I, J)][1] = entry(8 * I + g, 8 * J + 2 * t + 1, id);
            }
        double pivsum = 0.0;
        if (!FACTOR) { // generation only: the cost to subtract
#pragma unroll
            for (int k = 0; k < 10; ++k)
                pivsum += X[k][0] + X[k][1];
        }
#pragma unroll
        for (int J = 0; J < (FACTOR ? 4 : 0); ++J) {
            // ---- diagonal tile (J, J) and the panel tiles below it: one column at a time ----
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int jj = j >> 1, js = j & 1;
                double &d0 = X[tix(J, J)][0], &d1 = X[tix(J, J)][1];
                const double src = js ? d1 : d0;
                const double piv = __shfl_sync(FULL, src, 4 * j + jj);
                const double mycol = __shfl_sync(FULL, src, (lane & ~3) | jj);
                const double c0 = __shfl_sync(FULL, src, 4 * (2 * t) + jj);
                const double c1 = __shfl_sync(FULL, src, 4 * (2 * t + 1) + jj);
                const double r = rsqrt_pos(piv);
                pivsum += piv;
                const double lgj = mycol * r, lc0 = c0 * r, lc1 = c1 * r;
                d0 = (2 * t == j) ? lgj : ((2 * t > j) ? fma(-lgj, lc0, d0) : d0);
                d1 = (2 * t + 1 == j) ? lgj : ((2 * t + 1 > j) ? fma(-lgj, lc1, d1) : d1);
#pragma unroll
                for (int I = J + 1; I < 4; ++I) {
                    double &p0 = X[tix(I, J)][0], &p1 = X[tix(I, J)][1];
                    const double myp = __shfl_sync(FULL, js ? p1 : p0, (lane & ~3) | jj);
                    const double lij = myp * r;
                    p0 = (2 * t == j) ? lij : ((2 * t > j) ? fma(-lij, lc0, p0) : p0);
                    p1 = (2 * t + 1 == j) ? lij : ((2 * t + 1 > j) ? fma(-lij, lc1, p1) : p1);
                }
            }
            // ---- trailing update: C_IK -= L_IJ L_KJ^T, I >= K > J (two DMMAs per tile, operands in place) ----
#pragma unroll
            for (int I = J + 1; I < 4; ++I)
#pragma unroll
                for (int K = J + 1; K <= I; ++K) {
                    dmma_sub(X[tix(I, K)][0], X[tix(I, K)][1], X[tix(I, J)][0], X[tix(K, J)][0]);
                    dmma_sub(X[tix(I, K)][0], X[tix(I, K)][1], X[tix(I, J)][1], X[tix(K, J)][1]);
                }
        }
        acc += pivsum;
        if (FACTOR && id < 8 && lane == 0)
            sums[id] = pivsum;
    }
    if (acc == 1.2345)
        sums[8] = acc;
}

static double host_pivsum(unsigned id)
{
    double A[32][32];
    for (int a = 0; a < 32; ++a)
        for (int c = 0; c < 32; ++c)
            A[a][c] = entry(a, c, id);
    double s = 0.0;
    for (int j = 0; j < 32; ++j) { // right-looking, same pivot definition as the device (pivot before the square root)
        s += A[j][j];
        const double r = 1.0 / std::sqrt(A[j][j]);
        for (int a = j; a < 32; ++a)
            A[a][j] *= r;
        for (int a = j + 1; a < 32; ++a)
            for (int c = j + 1; c <= a; ++c)
                A[a][c] -= A[a][j] * A[c][j];
    }
    return s;
}

int main()
{
    double *sums;
    cudaMalloc(&sums, 16 * sizeof(double));
    cudaMemset(sums, 0, 16 * sizeof(double));
    const unsigned nmat = 1u << 20;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int wpb : {1, 2, 4}) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dmma_chol_kernel<true>, 32 * wpb, 0);
        const int blocks = sms * per_sm;
        dmma_chol_kernel<true><<<blocks, 32 * wpb>>>(4096, sums);
        cudaDeviceSynchronize();
        float best = 1e30f, gen = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            float ms;
            cudaEventRecord(e0);
            dmma_chol_kernel<true><<<blocks, 32 * wpb>>>(nmat, sums);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
            cudaEventRecord(e0);
            dmma_chol_kernel<false><<<blocks, 32 * wpb>>>(nmat, sums);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            gen = ms < gen ? ms : gen;
        }
        cudaFuncAttributes fa;
        cudaFuncGetAttributes(&fa, dmma_chol_kernel<true>);
        printf("warps/block %d, blocks/SM %d (%d warps/SM, %d registers): %.3f ms for 2^20 factorizations of 32x32 "
               "(generating the matrices alone: %.3f ms => factorization %.3f ms)\n",
               wpb, per_sm, per_sm * wpb, fa.numRegs, best, gen, best - gen);
    }
    std::vector<double> h(8);
    cudaMemcpy(h.data(), sums, 8 * sizeof(double), cudaMemcpyDeviceToHost);
    double worst = 0.0;
    for (unsigned id = 0; id < 8; ++id)
        worst = fmax(worst, fabs(h[id] - host_pivsum(id)) / fabs(host_pivsum(id)));
    printf("check: sum of the 32 pivots of matrices 0..7 against a host Cholesky: max relative difference %.2e\n", worst);
    printf("production kernel, factorization phase only (clock64 accounting): 8 635 cycles per 2 observations at 12 warps/SM "
           "= 1.37 ms for 2^20\n");
    return worst < 1e-12 ? 0 : 1;
}
