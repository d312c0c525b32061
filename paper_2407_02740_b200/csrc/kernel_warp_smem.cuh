// kernel_warp_smem.cuh -- layout WARP_SMEM: one warp per observation, every local
// matrix in shared memory.  Fully general in (m, p, q, d); it is the shape-agnostic
// path and the "warp per observation" arm of the layout study.  The fast path
// for the standard shapes is kernel_tiled.cuh.
//
// Per-observation algorithm (restates _obs_kernel, /root/reference/pkg/src/vecchiagp/
// engine/_kernels.pyx:347-381, with the algebraic shortcuts of SURVEY.md section 7):
//   gather (reversed row, observation last)         _kernels.pyx:188-205
//   K and the qd range-derivative matrices, one exp per pair   :208-232
//   in-place lower Cholesky, first non-positive pivot reported :235-251
//   z = B^-1 y, W = B^-1 X                          :254-263, 374-376
//   u = B^-T e_last                                 :266-275
//   w = B^-1 u; c_0 = (e_last - jitter w)/sigma^2; c_nugget = sigma^2 w   (exact forms of
//       B^-1 D_0 u and B^-1 D_nugget u, D_0 = (K - jitter I)/sigma^2, D_nugget = sigma^2 I)
//   c_j = B^-1 D_j u for the range-like parameters  :278-291
//   contraction into the L accumulators             :294-344
#pragma once
#include "common.cuh"

#define WS_WARPS_MAX 4

// doubles of shared scratch per warp
__host__ __device__ inline int warp_smem_doubles(int mp1, int d, int p, int q)
{
    const int ld = mp1 | 1;
    const int qd = q - 2;
    AccLayout A(p, q);
    // pts, ys(+z), xs(+W), K, D[qd], u, c[q], dots (q + p*q + q*q), acc[L]
    int n = mp1 * d + mp1 + mp1 * p + mp1 * ld * (1 + qd) + mp1 + q * mp1 + (q + p * q + q * q) + A.L;
    return (n + 1) & ~1;
}

// solve B x = rhs in place for nrhs vectors (stride apart), lane-parallel column sweep
__device__ __forceinline__ void ws_forward(const double *B, int ld, int k, double *rhs, int stride, int nrhs,
                                           int lane)
{
    for (int r = 0; r < nrhs; ++r) {
        double *x = rhs + r * stride;
        for (int j = 0; j < k; ++j) {
            const double xj = x[j] / B[j * ld + j];
            __syncwarp();
            if (lane == 0)
                x[j] = xj;
            for (int a = j + 1 + lane; a < k; a += 32)
                x[a] = fma(-B[a * ld + j], xj, x[a]);
            __syncwarp();
        }
    }
}

template <int FAM>
__global__ void __launch_bounds__(WS_WARPS_MAX * 32) vecchia_warp_smem_kernel(const EvalParams P)
{
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    const int mp1 = P.mp1, ld = mp1 | 1, d = P.d, p = P.p, q = P.q, qd = P.qd;
    const AccLayout A(p, q);

    double *pts = smem + (size_t)warp * P.ws_doubles;
    double *ys = pts + mp1 * d;
    double *xs = ys + mp1;              // column-major: xs[b*mp1 + a]
    double *Km = xs + mp1 * p;
    double *Dm = Km + mp1 * ld;         // qd full symmetric matrices
    double *u = Dm + (size_t)qd * mp1 * ld;
    double *cv = u + mp1;               // q vectors of length mp1
    double *zc = cv + q * mp1;          // dots: zc[q], wc[p*q], cc[q*q]
    double *wc = zc + q;
    double *cc = wc + p * q;
    double *acc = cc + q * q;           // L running totals of this warp
    const int acc_off = (int)(acc - pts);

    for (int o = lane; o < A.L; o += 32)
        acc[o] = 0.0;

    const int64_t gw = (int64_t)blockIdx.x * nwarps + warp;
    const int64_t nw = (int64_t)gridDim.x * nwarps;

    for (int64_t i = P.i0 + gw; i < P.i1; i += nw) {
        const int64_t *row = P.nn + (i - P.nn_row0) * mp1;
        // ---- live count and gather (local frame = reversed row) ----
        int cnt = 0;
        for (int c = lane; c < mp1; c += 32)
            cnt += (row[c] >= 0);
        for (int off = 16; off > 0; off >>= 1)
            cnt += __shfl_xor_sync(0xffffffffu, cnt, off);
        const int k = cnt, e = k - 1;
        __syncwarp();
        for (int a = lane; a < k; a += 32) {
            const double *r = P.rec + row[k - 1 - a] * P.rs;
            for (int l = 0; l < d; ++l)
                pts[a * d + l] = r[l];
            ys[a] = r[d];
            for (int b = 0; b < p; ++b)
                xs[b * mp1 + a] = r[d + 1 + b];
        }
        __syncwarp();
        // ---- covariance and range-derivative fill, one transcendental per pair ----
        const int T = k * (k + 1) / 2;
        for (int t = lane; t < T; t += 32) {
            int a = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
            while (a * (a + 1) / 2 > t)
                --a;
            while ((a + 1) * (a + 2) / 2 <= t)
                ++a;
            const int c = t - a * (a + 1) / 2;
            if (a == c) {
                Km[a * ld + a] = P.diag;
                for (int j = 0; j < qd; ++j)
                    Dm[((size_t)j * mp1 + a) * ld + a] = 0.0;
            } else {
                double dl[VB_MAXD], Dv[VB_MAXD], Kv;
                for (int l = 0; l < d; ++l)
                    dl[l] = pts[a * d + l] - pts[c * d + l];
                pair_terms<FAM>(P, dl, Kv, Dv);
                Km[a * ld + c] = Kv;
                for (int j = 0; j < qd; ++j) {
                    Dm[((size_t)j * mp1 + a) * ld + c] = Dv[j];
                    Dm[((size_t)j * mp1 + c) * ld + a] = Dv[j];
                }
            }
        }
        __syncwarp();
        // ---- in-place Cholesky (right-looking, lane per row) ----
        int failed = 0;
        for (int j = 0; j < k; ++j) {
            const double piv = Km[j * ld + j];
            if (piv <= P.piv_floor) {
                failed = j + 1;
                break;
            }
            const double dj = sqrt(piv);
            __syncwarp();
            if (lane == 0)
                Km[j * ld + j] = dj;
            for (int a = j + 1 + lane; a < k; a += 32)
                Km[a * ld + j] = Km[a * ld + j] / dj;
            __syncwarp();
            for (int a = j + 1 + lane; a < k; a += 32) {
                const double laj = Km[a * ld + j];
                for (int c = j + 1; c <= a; ++c)
                    Km[a * ld + c] = fma(-laj, Km[c * ld + j], Km[a * ld + c]);
            }
            __syncwarp();
        }
        if (failed) {
            if (lane == 0) {
                report_failure(P, i, failed);
                if (P.fail_rows)
                    P.fail_rows[i - P.i0] = failed;
            }
            continue;
        }
        // ---- z, W ----
        ws_forward(Km, ld, k, ys, mp1, 1 + p, lane);
        // ---- u = B^-T e_last ----
        for (int a = lane; a < k; a += 32)
            u[a] = (a == e) ? 1.0 : 0.0;
        __syncwarp();
        for (int j = k - 1; j >= 0; --j) {
            const double uj = u[j] / Km[j * ld + j];
            __syncwarp();
            if (lane == 0)
                u[j] = uj;
            for (int a = lane; a < j; a += 32)
                u[a] = fma(-Km[j * ld + a], uj, u[a]);
            __syncwarp();
        }
        // ---- t_j = D_j u (range-like), and u itself as the last right-hand side ----
        for (int a = lane; a < k; a += 32) {
            for (int j = 0; j < qd; ++j) {
                const double *Dr = Dm + ((size_t)j * mp1 + a) * ld;
                double s = 0.0;
                for (int c = 0; c < k; ++c)
                    s = fma(Dr[c], u[c], s);
                cv[(1 + j) * mp1 + a] = s;
            }
            cv[(q - 1) * mp1 + a] = u[a];
        }
        __syncwarp();
        ws_forward(Km, ld, k, cv + mp1, mp1, q - 1, lane);
        for (int a = lane; a < k; a += 32) {
            const double w = cv[(q - 1) * mp1 + a];
            cv[a] = (((a == e) ? 1.0 : 0.0) - P.jitter * w) * P.inv_sig2;
            cv[(q - 1) * mp1 + a] = P.sig2 * w;
        }
        __syncwarp();
        // ---- dot products over the local index ----
        const double *z = ys, *W = xs;
        for (int j = 0; j < q; ++j) {
            const double *cj = cv + j * mp1;
            double s = 0.0;
            for (int a = lane; a < k; a += 32)
                s = fma(z[a], cj[a], s);
            s = warp_sum(s);
            if (lane == 0)
                zc[j] = s;
            for (int b = 0; b < p; ++b) {
                double sw = 0.0;
                for (int a = lane; a < k; a += 32)
                    sw = fma(W[b * mp1 + a], cj[a], sw);
                sw = warp_sum(sw);
                if (lane == 0)
                    wc[b * q + j] = sw;
            }
            for (int l = 0; l <= j; ++l) {
                const double *cl = cv + l * mp1;
                double sc = 0.0;
                for (int a = lane; a < k; a += 32)
                    sc = fma(cj[a], cl[a], sc);
                sc = warp_sum(sc);
                if (lane == 0) {
                    cc[j * q + l] = sc;
                    cc[l * q + j] = sc;
                }
            }
        }
        __syncwarp();
        // ---- emit ----
        {
            const double logdet = 2.0 * log(Km[e * ld + e]);
            const double ze = z[e];
            double we[VB_MAXP], ce[VB_MAXQ];
            for (int b = 0; b < p; ++b)
                we[b] = W[b * mp1 + e];
            for (int j = 0; j < q; ++j)
                ce[j] = cv[j * mp1 + e];
            for (int o = lane; o < A.L; o += 32) {
                const double v = emit_value(o, p, q, A, logdet, ze, we, ce, zc, wc, cc);
                if (P.rows)
                    P.rows[(size_t)(i - P.i0) * A.L + o] = v;
                acc[o] += v;
            }
        }
        __syncwarp();
    }
    // ---- block partial: fixed warp order ----
    __syncthreads();
    for (int o = threadIdx.x; o < A.L; o += blockDim.x) {
        double s = 0.0;
        for (int w = 0; w < nwarps; ++w) {
            s += smem[(size_t)w * P.ws_doubles + acc_off + o];
        }
        P.partials[(size_t)blockIdx.x * A.L + o] = s;
    }
    vb_finish(P, 1);
}
