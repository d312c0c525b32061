// kernel_krige.cuh -- nearest-neighbour kriging on the tiled machinery.
//
// Restates the per-point body of the reference's predict.krige (/root/reference/pkg/src/vecchiagp/
// predict.py:77-89): joint covariance K of the m_pred nearest training rows (nugget on the diagonal),
// nugget-free cross covariance k*, Cholesky, two forward solves, mean = x* beta + half_k . half_r,
// var = prior - half_k . half_k.  Here the prediction point is appended as the LAST row of the local
// matrix (diagonal = prior variance, off-diagonals = k*), exactly the local frame of the likelihood
// kernel: after the LDL^T sweep the last pivot d_e IS prior - k*' K^-1 k* (the Schur complement), and
// the fused forward substitution of (residuals..., 0) leaves -(k*' K^-1 r) in the last entry.  So the
// kriging kernel is the likelihood kernel's gather + pair loop + factorization with one right-hand
// side and nothing else.  Same lane-group / register layout as kernel_tiled.cuh (G lanes per point,
// S rows per lane, local row 0 always padding: serves m_pred + 1 <= CAP - 1).
#pragma once
#include "tiled_common.cuh"

struct KrigeParams {
    const double *locs_star;  // (npred, d) working coordinates of the prediction points
    const int64_t *nn_star;   // (npred, m_pred) training indices, any order
    int64_t npred;
    int m_pred;
    double prior;             // sigma^2 (latent) or sigma^2 (1 + nugget)
    double beta[VB_MAXP];     // mean parameters: residual = y - X beta is formed in the gather
    double *mean_resid;       // out (npred): conditional mean of the residual at the point
    double *var;              // out (npred): conditional variance (not clamped)
    // conditional SIMULATION (the reference's simulate_nn_gp; file:line in include/vecchia_b200.h): when sim_order is set,
    // point t is training observation i = sim_order[t]; its neighbours are columns 1.. of row i of the
    // training table, its location the one of record i, and instead of (mean_resid, var) the kernel writes
    // y_i = x_i' beta + E[r_i | neighbours] + sqrt(max(var_i, 0)) xi_i into record i and into sim_y[i].
    const int64_t *sim_order;
    const double *xi;
    double *sim_y;
    double *rec_w;            // the (writable) point records of the problem
};

template <int G, int S, int D>
struct KrigeSmem {
    using Geo = TileGeom<G, S>;
    static constexpr int DP = (D + 1) & ~1;
    static constexpr int PTS = Geo::CAP * DP;
    static constexpr int PER_OBS = PTS + Geo::KL;
    static constexpr int TOTAL = VB_EXPTAB + Geo::OPW * PER_OBS;
};

template <int G, int S, int FAM, int D>
__global__ void __launch_bounds__(32, tiled_min_blocks(G, S)) vecchia_krige_kernel(const EvalParams E, const KrigeParams Q)
{
    using Geo = TileGeom<G, S>;
    using FT = FamTraits<FAM, D>;
    constexpr int CAP = Geo::CAP, OPW = Geo::OPW, QD = FT::QD;
    using SM = KrigeSmem<G, S, D>;
    using TS = TileSmem<G, S, D, QD>; // pair-table geometry (TOFF, TPAD, NI) is shared with the likelihood kernel
    constexpr int DP = SM::DP;

    extern __shared__ double smem[];
    double *etab = smem;
    const int lane = threadIdx.x;
    const int g = lane / G, lg = lane % G;
    double *obs = smem + VB_EXPTAB + g * SM::PER_OBS;
    double *pts = obs;
    double *KLs = obs + SM::PTS;

    for (int t = lane; t < VB_EXPTAB; t += 32)
        etab[t] = exp2((double)t * (1.0 / VB_EXPTAB));
    int rowi[S], colb_r[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        rowi[s] = s * G + ((s & 1) ? (G - 1 - lg) : lg);
        colb_r[s] = Geo::colbase(rowi[s]);
    }
    __syncwarp();

    const int64_t nbatch = (Q.npred + OPW - 1) / OPW;
    for (int64_t batch = blockIdx.x; batch < nbatch; batch += gridDim.x) {
        const int64_t t = batch * OPW + g;
        const bool active = t < Q.npred;
        const bool sim = Q.sim_order != nullptr;
        const int64_t isim = (sim && active) ? Q.sim_order[t] : 0;
        const int64_t *nrow = sim ? (E.nn + (isim - E.nn_row0) * E.mp1 + 1) : (Q.nn_star + (active ? t : 0) * Q.m_pred);

        // ---- gather: local row CAP-1 = the prediction point, rows CAP-1-m_pred .. CAP-2 = neighbours ----
        double rhs[S];
        int nlive = 0;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int a = rowi[s], col = CAP - 2 - a; // neighbour column of this local row (-1: the point itself)
            double cx[DP];
#pragma unroll
            for (int l = 0; l < DP; ++l)
                cx[l] = 0.0;
            rhs[s] = 0.0;
            bool live = false;
            double dg = 1.0;
            if (active && col == -1) {
                live = true;
                dg = Q.prior;
#pragma unroll
                for (int l = 0; l < D; ++l)
                    cx[l] = (sim ? E.rec[isim * E.rs + l] : Q.locs_star[t * D + l]) * E.inv_rho[l];
            } else if (active && col >= 0 && col < Q.m_pred) {
                const int64_t idx = nrow[col];
                if (idx >= 0) {
                    live = true;
                    dg = E.diag;
                    const double *r = E.rec + idx * E.rs;
#pragma unroll
                    for (int l = 0; l < D; ++l)
                        cx[l] = r[l] * E.inv_rho[l];
                    double res = r[D];
                    for (int b = 0; b < E.p; ++b)
                        res = fma(-r[D + 1 + b], Q.beta[b], res);
                    rhs[s] = res;
                }
            }
#pragma unroll
            for (int l = 0; l < DP; l += 2)
                *reinterpret_cast<double2 *>(pts + a * DP + l) = make_double2(cx[l], cx[l + 1]);
            KLs[colb_r[s] + a] = dg;
            const unsigned bal = __ballot_sync(FULLMASK, live);
            nlive += __popc((G == 32) ? bal : ((bal >> (g * G)) & ((1u << (G & 31)) - 1u)));
        }
        __syncwarp();

        // ---- pair terms (covariance only) ----
        const int nlp = nlive * (nlive - 1) / 2;
        {
            constexpr int NI = TS::NI;
            for (int t0 = lg; t0 < nlp; t0 += NI * G) {
                unsigned ent[NI];
                double Kv[NI];
#pragma unroll
                for (int h = 0; h < NI; ++h) {
                    ent[h] = E.pair_tab[t0 + h * G];
                    const double *pa = pts + (ent[h] >> 24) * DP;
                    const double *pc = pts + ((ent[h] >> 16) & 255) * DP;
                    double dl[D], Dv[QD];
#pragma unroll
                    for (int l = 0; l < DP; l += 2) {
                        const double2 va = *reinterpret_cast<const double2 *>(pa + l);
                        const double2 vc = *reinterpret_cast<const double2 *>(pc + l);
                        dl[l] = va.x - vc.x;
                        if (l + 1 < D)
                            dl[l + 1 < D ? l + 1 : l] = va.y - vc.y;
                    }
                    pair_terms_s<FAM, D, false>(E, etab, dl, Kv[h], Dv);
                }
#pragma unroll
                for (int h = 0; h < NI; ++h)
                    KLs[ent[h] & 0xffff] = Kv[h];
            }
            __syncwarp();
            for (int t1 = nlp + lg; t1 < TS::TOFF; t1 += G)
                KLs[E.pair_tab[t1] & 0xffff] = 0.0;
        }
        __syncwarp();

        double Kr[S][CAP];
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int c = 0; c < (s + 1) * G; ++c)
                Kr[s][c] = KLs[Geo::colbase(c) + rowi[s]];
        __syncwarp();

        // ---- LDL^T sweep with the residual vector riding along (see kernel_tiled.cuh) ----
        bool bad = false;
#pragma unroll
        for (int j = 1; j < CAP - 1; ++j) {
            const int sj = j / G;
            const int oj = (sj & 1) ? (G - 1 - j % G) : (j % G);
            const double *col = KLs + Geo::colbase(j);
#pragma unroll
            for (int s = 0; s < S; ++s)
                if ((s + 1) * G - 1 >= j && rowi[s] >= j)
                    KLs[Geo::colbase(j) + rowi[s]] = Kr[s][j];
            const double xr = __shfl_sync(FULLMASK, rhs[sj], oj, G);
            __syncwarp();
            const int cs = ((Geo::colbase(j) + j) & 1) ? j + 1 : j;
            double dj;
            if (cs != j)
                dj = col[j];
            double2 v0;
            if (cs == j) {
                v0 = *reinterpret_cast<const double2 *>(col + j);
                dj = v0.x;
            }
            bad = bad || (dj <= E.piv_floor);
            const double rj = rcp_pos(dj);
            double Lo[S];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if ((s + 1) * G - 1 > j) {
                    const double Ls = Kr[s][j] * rj;
                    Lo[s] = (rowi[s] > j) ? Ls : 0.0;
                    rhs[s] = fma(-Lo[s], xr, rhs[s]);
                } else {
                    Lo[s] = 0.0;
                }
            }
            if (cs == j) {
#pragma unroll
                for (int s = 0; s < S; ++s)
                    if ((s + 1) * G - 1 >= j + 1)
                        Kr[s][j + 1] = fma(-Lo[s], v0.y, Kr[s][j + 1]);
            }
#pragma unroll
            for (int c0 = (cs == j) ? j + 2 : j + 1; c0 < CAP; c0 += 2) {
                const double2 v = *reinterpret_cast<const double2 *>(col + c0);
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    if ((s + 1) * G - 1 >= c0)
                        Kr[s][c0] = fma(-Lo[s], v.x, Kr[s][c0]);
                    if (c0 + 1 < CAP && (s + 1) * G - 1 >= c0 + 1)
                        Kr[s][c0 + 1] = fma(-Lo[s], v.y, Kr[s][c0 + 1]);
                }
            }
        }
        constexpr int se = S - 1;
        constexpr int oe = Geo::lane_of(CAP - 1);
        if (active && lg == oe) {
            // Schur complement of the prediction point and minus the conditional mean of its residual
            const double var = bad ? __longlong_as_double(0x7ff8000000000000ll) : Kr[se][CAP - 1];
            if (sim) {
                const double *r = E.rec + isim * E.rs;
                double yv = -rhs[se];
                for (int b = 0; b < E.p; ++b)
                    yv = fma(r[D + 1 + b], Q.beta[b], yv);
                yv = fma(sqrt(fmax(var, 0.0)), Q.xi[isim], yv); // NaN variance (failed factorization) propagates
                Q.rec_w[isim * E.rs + D] = yv;
                Q.sim_y[isim] = yv;
            } else {
                Q.var[t] = var;
                Q.mean_resid[t] = -rhs[se];
            }
        }
        if (active && bad && lg == 0)
            report_failure(E, sim ? isim : t, 1);
        __syncwarp();
    }
}

struct KrigeInstance {
    int g, s, cap, family, d;
    void (*kernel)(const EvalParams, const KrigeParams);
    int smem_doubles;
    const char *name;
};

#define KRIGE_INST(G_, S_, FAM_, D_)                                                                             \
    {                                                                                                            \
        G_, S_, (G_) * (S_), FAM_, D_, vecchia_krige_kernel<G_, S_, FAM_, D_>, KrigeSmem<G_, S_, D_>::TOTAL,     \
            "vecchia_krige_kernel<G=" #G_ ",S=" #S_ "," #FAM_ ",D=" #D_ ">"                                      \
    }
