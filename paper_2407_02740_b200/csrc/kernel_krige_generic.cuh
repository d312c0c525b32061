// kernel_krige_generic.cuh -- shape-agnostic nearest-neighbour kriging / conditional simulation.
//
// The tiled kriging kernel (kernel_krige.cuh) is instantiated for d in {2, 3} and m_pred <= 62; the reference's
// predict.krige (/root/reference/pkg/src/vecchiagp/predict.py:35-90) and simulate_nn_gp (file:line in include/vecchia_b200.h) accept
// any d and any m_pred <= n.  This kernel serves every other shape: ONE WARP per prediction point, the packed lower
// triangle of the local matrix, the points and the right-hand side in shared memory, run-time d and m_pred (up to
// the shared-memory capacity: m_pred + 1 <= ~230 on B200), lane-per-row square-root-free elimination.  Same local
// frame and outputs as the tiled kernel: the prediction point is the LAST row (diagonal = prior variance,
// off-diagonals = nugget-free cross covariance), its last pivot is the kriging variance and the forward
// substitution of (residuals..., 0) leaves minus the conditional mean of the residual in the last entry.
#pragma once
#include "kernel_krige.cuh"

__host__ __device__ inline int krige_generic_doubles(int k, int d)
{
    return k * (k + 1) / 2 + k * d + k + 2; // packed triangle, points, right-hand side
}

template <int FAM>
__global__ void __launch_bounds__(128) vecchia_krige_generic_kernel(const EvalParams E, const KrigeParams Q)
{
    extern __shared__ double smem[];
    const int lane = threadIdx.x % 32, warp = threadIdx.x / 32, nwarps = blockDim.x / 32;
    const bool sim = Q.sim_order != nullptr;
    const int d = E.d, k = Q.m_pred + 1, e = k - 1;
    double *Km = smem + (size_t)warp * krige_generic_doubles(k, d); // element (a, c), a >= c, at a(a+1)/2 + c
    double *pts = Km + k * (k + 1) / 2;
    double *rhs = pts + k * d;
    auto tri = [](int a, int c) { return a * (a + 1) / 2 + c; };

    for (int64_t t = (int64_t)blockIdx.x * nwarps + warp; t < Q.npred; t += (int64_t)gridDim.x * nwarps) {
        const int64_t isim = sim ? Q.sim_order[t] : 0;
        const int64_t *nrow = sim ? (E.nn + (isim - E.nn_row0) * E.mp1 + 1) : (Q.nn_star + t * Q.m_pred);
        // ---- gather: rows 0..m_pred-1 = neighbours (a missing neighbour, index < 0, is an identity row), row e =
        //      the point itself ----
        for (int a = lane; a < k; a += 32) {
            double dg = 1.0, res = 0.0;
            bool live = false;
            if (a == e) {
                live = true;
                dg = Q.prior;
                for (int l = 0; l < d; ++l)
                    pts[a * d + l] = sim ? E.rec[isim * E.rs + l] : Q.locs_star[t * d + l];
            } else {
                const int64_t idx = nrow[a];
                if (idx >= 0) {
                    live = true;
                    dg = E.diag;
                    const double *r = E.rec + idx * E.rs;
                    for (int l = 0; l < d; ++l)
                        pts[a * d + l] = r[l];
                    res = r[d];
                    for (int b = 0; b < E.p; ++b)
                        res = fma(-r[d + 1 + b], Q.beta[b], res);
                }
            }
            if (!live)
                for (int l = 0; l < d; ++l)
                    pts[a * d + l] = __longlong_as_double(0x7ff8000000000000ll); // marks an identity row
            rhs[a] = res;
            Km[tri(a, a)] = dg;
        }
        __syncwarp();
        // ---- pair terms (covariance only), pairs dealt round-robin to the lanes ----
        const int npairs = k * (k - 1) / 2;
        for (int idx = lane; idx < npairs; idx += 32) {
            // idx -> (a, c), a > c: a = floor((1 + sqrt(1 + 8 idx)) / 2)
            int a = (int)((1.0 + sqrt(1.0 + 8.0 * (double)idx)) * 0.5);
            while (a * (a - 1) / 2 > idx)
                --a;
            while ((a + 1) * a / 2 <= idx)
                ++a;
            const int c = idx - a * (a - 1) / 2;
            double dl[VB_MAXD], Dv[VB_MAXQ];
            bool real = true;
            for (int l = 0; l < d; ++l) {
                dl[l] = pts[a * d + l] - pts[c * d + l];
                real = real && (dl[l] == dl[l]);
            }
            double Kv = 0.0;
            if (real) {
                pair_terms<FAM>(E, dl, Kv, Dv);
                if (FAM == FAM_MATERN && !(Kv == Kv))
                    Kv = 0.0;
            }
            Km[tri(a, c)] = Kv;
        }
        __syncwarp();
        // ---- K = Lt D Lt^T, right-looking, lane per row; the forward substitution of the right-hand side rides
        //      along.  Column j stays unscaled until every lane has used it. ----
        bool bad = false;
        for (int j = 0; j < k; ++j) {
            const double dj = Km[tri(j, j)];
            if (!(dj > E.piv_floor)) {
                bad = true;
                break;
            }
            const double rj = 1.0 / dj, zj = rhs[j];
            __syncwarp();
            for (int a = j + 1 + lane; a < k; a += 32) {
                const double la = Km[tri(a, j)] * rj;
                for (int c = j + 1; c <= a; ++c)
                    Km[tri(a, c)] = fma(-la, Km[tri(c, j)], Km[tri(a, c)]);
                rhs[a] = fma(-la, zj, rhs[a]);
            }
            __syncwarp();
        }
        if (lane == 0) {
            const double var = bad ? __longlong_as_double(0x7ff8000000000000ll) : Km[tri(e, e)];
            if (sim) {
                const double *r = E.rec + isim * E.rs;
                double yv = -rhs[e];
                for (int b = 0; b < E.p; ++b)
                    yv = fma(r[d + 1 + b], Q.beta[b], yv);
                yv = fma(sqrt(fmax(var, 0.0)), Q.xi[isim], yv);
                Q.rec_w[isim * E.rs + d] = yv;
                Q.sim_y[isim] = yv;
            } else {
                Q.var[t] = var;
                Q.mean_resid[t] = -rhs[e];
            }
            if (bad)
                report_failure(E, sim ? isim : t, 1);
        }
        __syncwarp();
    }
}

typedef void (*krige_generic_kernel_t)(const EvalParams, const KrigeParams);

static inline krige_generic_kernel_t krige_generic_for(int family)
{
    switch (family) {
    case FAM_EXP_ISO: return vecchia_krige_generic_kernel<FAM_EXP_ISO>;
    case FAM_EXP_ANISO: return vecchia_krige_generic_kernel<FAM_EXP_ANISO>;
    case FAM_EXP_SPACETIME: return vecchia_krige_generic_kernel<FAM_EXP_SPACETIME>;
    case FAM_MATERN15: return vecchia_krige_generic_kernel<FAM_MATERN15>;
    case FAM_MATERN: return vecchia_krige_generic_kernel<FAM_MATERN>;
    default: return vecchia_krige_generic_kernel<FAM_MATERN25>;
    }
}
