// Micro-benchmark: LSU cost (cycles per warp-instruction per SM) of shared-memory loads as a function of
// how many distinct addresses a warp touches and how they fall on the banks, plus SHFL and STS throughput.
// Per-lane offsets (in doubles) come from a table, so one kernel serves every pattern.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lds_groups lds_groups.cu && ./lds_groups
#include <cstdio>
#include <cstring>
#include <cuda_runtime.h>

struct Pat { int off[32]; };

template <int W> // 64 or 128 bit loads; 1 = SHFL.32; 2 = STS.64; 3 = STS.128
__global__ void k(double *out, int iters, Pat pat)
{
    __shared__ __align__(16) double sm[6000];
    for (int i = threadIdx.x; i < 6000; i += blockDim.x)
        sm[i] = i;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const double *p = sm + pat.off[lane];
    double a0 = lane, a1 = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int rot = ((u * 34 + it * 2) & 1023);
            unsigned addr = (unsigned)__cvta_generic_to_shared(p + rot);
            if (W == 128) {
                double x, y;
                asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(addr));
                a0 += x; a1 += y;
            } else if (W == 64) {
                double x;
                asm volatile("ld.shared.f64 %0, [%1];" : "=d"(x) : "r"(addr));
                a0 += x;
            } else if (W == 1) {
                int v = __shfl_sync(0xffffffffu, __double2loint(a0), (pat.off[lane] + u) & 31);
                a1 += v;
            } else if (W == 2) {
                asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(a0));
            } else if (W == 3) {
                asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(addr), "d"(a0), "d"(a1));
            }
        }
    }
    if (a0 + a1 == 1.2345) out[0] = a0 + sm[lane];
}

template <int W>
void run(const char *name, const Pat &pat)
{
    double *out; cudaMalloc(&out, 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 2048, blocks = 148 * 4, threads = 256;
    k<W><<<blocks, threads>>>(out, 16, pat);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    k<W><<<blocks, threads>>>(out, iters, pat);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double per_sm = 4.0 * 8 * iters * 16;
    double cycles = ms * 1e-3 * 1.965e9;
    printf("%-4d %-58s %.2f cycles per warp-instr per SM\n", W, name, cycles / per_sm);
    cudaFree(out);
}

static Pat groups(int lanes_per_group, int stride)
{
    Pat p;
    for (int l = 0; l < 32; ++l) p.off[l] = (l / lanes_per_group) * stride;
    return p;
}

int main()
{
    char nm[128];
    const int gl[] = {32, 16, 8, 4, 2, 1};
    const int strides64[] = {1, 2, 16, 17, 18, 34};
    for (int gi = 0; gi < 6; ++gi)
        for (int si = 0; si < 6; ++si) {
            if (gl[gi] == 32 && si > 0) continue;
            snprintf(nm, sizeof nm, "LDS.64  groups of %2d lanes, group stride %3d doubles", gl[gi], strides64[si]);
            run<64>(nm, groups(gl[gi], strides64[si]));
        }
    const int strides128[] = {2, 4, 16, 18, 34, 66};
    for (int gi = 0; gi < 6; ++gi)
        for (int si = 0; si < 6; ++si) {
            if (gl[gi] == 32 && si > 0) continue;
            snprintf(nm, sizeof nm, "LDS.128 groups of %2d lanes, group stride %3d doubles", gl[gi], strides128[si]);
            run<128>(nm, groups(gl[gi], strides128[si]));
        }
    // "one of two addresses inside each 16-lane group" (row-owner pair scheme): lanes below a threshold read A, others B
    for (int thr = 0; thr <= 16; thr += 4) {
        Pat p;
        for (int l = 0; l < 32; ++l) p.off[l] = (l / 16) * 1170 + ((l % 16) < thr ? 0 : 38);
        snprintf(nm, sizeof nm, "LDS.128 2 groups, lanes < %2d read A else B", thr);
        run<128>(nm, p);
    }
    {
        Pat p;
        for (int l = 0; l < 32; ++l) p.off[l] = (l / 16) * 1170 + 2 * (l % 16);
        run<128>("LDS.128 2 groups, each lane its own 16B (contiguous)", p);
        for (int l = 0; l < 32; ++l) p.off[l] = (l / 16) * 1170 + 2 * ((l * 7) % 16) + 32 * (l % 3);
        run<128>("LDS.128 scattered 16B chunks", p);
        for (int l = 0; l < 32; ++l) p.off[l] = (l / 16) * 1170 + ((l * 5) % 16);
        run<64>("LDS.64 2 groups, per-lane distinct contiguous permuted", p);
    }
    run<1>("SHFL.32 (per 32-bit shuffle)", groups(1, 1));
    run<2>("STS.64 32 distinct contiguous", groups(1, 1));
    run<2>("STS.64 groups of 16, stride 18", groups(16, 18));
    run<3>("STS.128 32 distinct contiguous", groups(1, 2));
    return 0;
}
