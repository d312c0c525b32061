// kernel_thread.cuh -- layout THREAD: one THREAD per observation, the paper's layout (arXiv 2407.02740,
// "thread-per-observation": every thread runs the whole per-observation algorithm serially on private
// matrices).  It is the third arm of the layout study BASELINE.json asks for, not a production path:
// VB200_LAYOUT_AUTO never selects it.
//
// Two storage variants of the packed lower triangle of the local covariance matrix K (the matrix the
// factorization works on):
//   SMEM_TRI = false   thread-local array (what GpGpU does): dynamic indexing puts it in LOCAL memory, i.e.
//                      L1 / L2 traffic -- 32 lanes x 4 KB strided by the array size;
//   SMEM_TRI = true    the triangle of every thread staged in SHARED memory, element-interleaved across the
//                      32 lanes (conflict-free), "as the paper's new method argues": 132 KB per warp, so one
//                      warp per SM.
// Everything else (points, right-hand sides, the range-derivative triangles) is thread-local in both variants.
//
// Per-observation algorithm = the reference's _obs_kernel (/root/reference/pkg/src/vecchiagp/engine/
// _kernels.pyx:347-381): gather :195-205, covariance + derivative fill :208-232 (one exp per pair), row-oriented
// Cholesky :235-251, forward solves :254-263, u = B^-T e_last :266-275, derivative solves :278-291 (with the
// exact variance / nugget shortcuts of kernel_warp_smem.cuh), contraction :294-344.
#pragma once
#include "common.cuh"

#define TH_MAXK 32                       // local rows (m + 1 <= 32)
#define TH_TRI (TH_MAXK * (TH_MAXK + 1) / 2)
#define TH_MAXD 3
#define TH_MAXP 4
#define TH_MAXQD 2                       // range-like parameters (iso 1, space-time 2, general Matern 2)
#define TH_MAXQ (TH_MAXQD + 2)
#define TH_MAXL ((1 + TH_MAXQ) * (2 + TH_MAXP + TH_MAXP * TH_MAXP) + TH_MAXQ * TH_MAXQ)

__host__ __device__ inline bool thread_layout_supported(int mp1, int d, int p, int q)
{
    return mp1 <= TH_MAXK && d <= TH_MAXD && p <= TH_MAXP && q - 2 <= TH_MAXQD;
}

template <bool SMEM_TRI>
struct ThreadTri {
    double *base;
    __device__ __forceinline__ double &operator()(int a, int c) const
    {
        const int t = a * (a + 1) / 2 + c;
        return SMEM_TRI ? base[t * 32] : base[t]; // shared: element t of lane l at [t*32 + l]
    }
};

template <int FAM, bool SMEM_TRI>
__global__ void __launch_bounds__(SMEM_TRI ? 32 : 128) vecchia_thread_kernel(const EvalParams P)
{
    extern __shared__ double smem[];
    const int mp1 = P.mp1, d = P.d, p = P.p, q = P.q, qd = P.qd;
    const AccLayout A(p, q);
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;

    double Kloc[SMEM_TRI ? 1 : TH_TRI];
    ThreadTri<SMEM_TRI> K{SMEM_TRI ? (smem + (threadIdx.x & 31)) : Kloc};
    double Dm[TH_MAXQD][TH_TRI];           // packed strict-lower range-derivative matrices (diagonal = 0)
    double pts[TH_MAXK][TH_MAXD], ys[TH_MAXK], xs[TH_MAXP][TH_MAXK];
    double u[TH_MAXK], cv[TH_MAXQ][TH_MAXK];
    double acc[TH_MAXL];
    for (int o = 0; o < A.L; ++o)
        acc[o] = 0.0;

    for (int64_t i = P.i0 + tid; i < P.i1; i += nthreads) {
        const int64_t *row = P.nn + (i - P.nn_row0) * mp1;
        int k = 0;
        while (k < mp1 && row[k] >= 0)
            ++k;
        const int e = k - 1;
        for (int a = 0; a < k; ++a) { // local frame = reversed row, observation last
            const double *r = P.rec + row[k - 1 - a] * P.rs;
            for (int l = 0; l < d; ++l)
                pts[a][l] = r[l];
            ys[a] = r[d];
            for (int b = 0; b < p; ++b)
                xs[b][a] = r[d + 1 + b];
        }
        for (int a = 0; a < k; ++a) {
            for (int c = 0; c < a; ++c) {
                double dl[VB_MAXD], Dv[VB_MAXD], Kv;
                for (int l = 0; l < d; ++l)
                    dl[l] = pts[a][l] - pts[c][l];
                pair_terms<FAM>(P, dl, Kv, Dv);
                K(a, c) = Kv;
                for (int j = 0; j < qd; ++j)
                    Dm[j][a * (a + 1) / 2 + c] = Dv[j];
            }
            K(a, a) = P.diag;
            for (int j = 0; j < qd; ++j)
                Dm[j][a * (a + 1) / 2 + a] = 0.0;
        }
        // row-oriented Cholesky (Cholesky-Banachiewicz), in place
        int failed = 0;
        for (int a = 0; a < k && !failed; ++a) {
            for (int c = 0; c <= a; ++c) {
                double s = K(a, c);
                for (int b = 0; b < c; ++b)
                    s = fma(-K(a, b), K(c, b), s);
                if (c == a) {
                    if (s <= P.piv_floor) {
                        failed = a + 1;
                        break;
                    }
                    K(a, a) = sqrt(s);
                } else {
                    K(a, c) = s / K(c, c);
                }
            }
        }
        if (failed) {
            report_failure(P, i, failed);
            if (P.fail_rows)
                P.fail_rows[i - P.i0] = failed;
            continue;
        }
        auto forward = [&](double *x) { // x <- B^-1 x
            for (int a = 0; a < k; ++a) {
                double s = x[a];
                for (int b = 0; b < a; ++b)
                    s = fma(-K(a, b), x[b], s);
                x[a] = s / K(a, a);
            }
        };
        forward(ys);
        for (int b = 0; b < p; ++b)
            forward(xs[b]);
        for (int a = 0; a < k; ++a)
            u[a] = 0.0;
        u[e] = 1.0;
        for (int a = k - 1; a >= 0; --a) { // u = B^-T e_last
            double s = u[a];
            for (int b = a + 1; b < k; ++b)
                s = fma(-K(b, a), u[b], s);
            u[a] = s / K(a, a);
        }
        for (int j = 0; j < qd; ++j) { // t_j = D_j u from the strict lower triangle (symmetric mat-vec)
            double *t = cv[1 + j];
            for (int a = 0; a < k; ++a)
                t[a] = 0.0;
            for (int a = 0; a < k; ++a)
                for (int c = 0; c < a; ++c) {
                    const double v = Dm[j][a * (a + 1) / 2 + c];
                    t[a] = fma(v, u[c], t[a]);
                    t[c] = fma(v, u[a], t[c]);
                }
            forward(t);
        }
        double *w = cv[q - 1];
        for (int a = 0; a < k; ++a)
            w[a] = u[a];
        forward(w);
        for (int a = 0; a < k; ++a) {
            cv[0][a] = (((a == e) ? 1.0 : 0.0) - P.jitter * w[a]) * P.inv_sig2;
            w[a] = P.sig2 * w[a];
        }
        double zc[TH_MAXQ], wc[TH_MAXP * TH_MAXQ], cc[TH_MAXQ * TH_MAXQ], we[TH_MAXP], ce[TH_MAXQ];
        for (int j = 0; j < q; ++j) {
            double s = 0.0;
            for (int a = 0; a < k; ++a)
                s = fma(ys[a], cv[j][a], s);
            zc[j] = s;
            for (int b = 0; b < p; ++b) {
                double sw = 0.0;
                for (int a = 0; a < k; ++a)
                    sw = fma(xs[b][a], cv[j][a], sw);
                wc[b * q + j] = sw;
            }
            for (int l = 0; l <= j; ++l) {
                double sc = 0.0;
                for (int a = 0; a < k; ++a)
                    sc = fma(cv[j][a], cv[l][a], sc);
                cc[j * q + l] = sc;
                cc[l * q + j] = sc;
            }
            ce[j] = cv[j][e];
        }
        for (int b = 0; b < p; ++b)
            we[b] = xs[b][e];
        const double logdet = 2.0 * log(K(e, e));
        for (int o = 0; o < A.L; ++o) {
            const double v = emit_value(o, p, q, A, logdet, ys[e], we, ce, zc, wc, cc);
            if (P.rows)
                P.rows[(size_t)(i - P.i0) * A.L + o] = v;
            acc[o] += v;
        }
    }
    // one partial row per THREAD (the fixed-order reduction kernel adds them)
    for (int o = 0; o < A.L; ++o)
        P.partials[(size_t)tid * A.L + o] = acc[o];
    vb_finish(P, (int)blockDim.x);
}
