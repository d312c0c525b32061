// kernel_tiled_pt.cuh -- layout TILED_REG, PAIR-TABLE variant (the first generation of the tiled kernel).
//
// Same lane-group / register layout and the same factorization, back-substitution and sweeps as
// kernel_tiled.cuh, but the pair terms are computed PAIR-parallel from a device pair table (perfectly
// balanced, two pairs in flight per lane), staged in the packed triangle in shared memory and read back
// row-wise into registers.  The pair loop is a rolled loop, so the kernel is much smaller than the
// row-owner kernel, whose fully unrolled pair phase grows with CAP: on the two widest tiers
// (CAP = 48 and 64, m = 40 / 60: 255 registers, shared-memory-capacity-bound occupancy) this variant is
// 15-20 % faster (measured, profiles/r1_experiments.md); the narrower tiers use kernel_tiled.cuh.
//
// Reference map: /root/reference/pkg/src/vecchiagp/engine/_kernels.pyx:347-381 (_obs_kernel); see common.cuh.
#pragma once
#include "tiled_common.cuh"

template <int G, int S, int FAM, int D, int P>
__global__ void __launch_bounds__(32, tiled_min_blocks(G, S)) vecchia_tiled_pt_kernel(const EvalParams E)
{
    using Geo = TileGeom<G, S>;
    using FT = FamTraits<FAM, D>;
    constexpr int CAP = Geo::CAP, OPW = Geo::OPW, QD = FT::QD, Q = FT::Q;
    using SM = TileSmem<G, S, D, QD>;
    constexpr int DP = SM::DP, DSZ = SM::DSZ;
    constexpr int L = (1 + Q) * (2 + P + P * P) + Q * Q;
    constexpr int NACC = (L + G - 1) / G;
    const AccLayout A(P, Q);
    static_assert(CAP % 2 == 0 && CAP <= 128, "tier geometry");

    extern __shared__ double smem[];
    double *etab = smem;                             // 2^(j/64), j < 64
    const int lane = threadIdx.x;
    const int g = lane / G, lg = lane % G;
    double *obs = smem + VB_EXPTAB + g * SM::PER_OBS;
    double *pts = obs;                               // CAP x DP scaled coordinates of the local frame
    double *KLs = obs + SM::PTS;                     // packed K staging, then the column store of L
    double *Dms = KLs + Geo::KL;                     // QD packed strict-lower derivative matrices (+ zero slot)

    for (int t = lane; t < VB_EXPTAB; t += 32)
        etab[t] = exp2((double)t * (1.0 / VB_EXPTAB));
    // diagonal and column 0 of every D_j are zero and never written by the pair loop
#pragma unroll
    for (int j = 0; j < QD; ++j)
        for (int a = lg; a < CAP; a += G) {
            Dms[j * DSZ + a] = 0.0;
            Dms[j * DSZ + Geo::colbase(a) + a] = 0.0;
        }
    int rowi[S], colb_r[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        rowi[s] = s * G + ((s & 1) ? (G - 1 - lg) : lg);
        colb_r[s] = Geo::colbase(rowi[s]);
    }
    double acc[NACC];
#pragma unroll
    for (int t = 0; t < NACC; ++t)
        acc[t] = 0.0;
    __syncwarp();

    const int64_t nbatch = (E.i1 - E.i0 + OPW - 1) / OPW;
    for (int64_t batch = blockIdx.x; batch < nbatch; batch += gridDim.x) {
        const int64_t i = E.i0 + batch * OPW + g;
        const bool active = i < E.i1;
        const int64_t *nrow = E.nn + (active ? (i - E.nn_row0) : 0) * E.mp1;

        // ---- gather: local index a <-> neighbor column CAP-1-a (observation last).  Coordinates are
        //      stored divided by the range of their axis.  Padding rows: diagonal 1, data 0. ----
        double rhs[1 + P][S];
        int nlive = 0;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int a = rowi[s], col = CAP - 1 - a;
            int64_t idx = -1;
            if (active && col < E.mp1)
                idx = nrow[col];
            const bool live = idx >= 0;
            double cx[DP];
#pragma unroll
            for (int l = 0; l < DP; ++l)
                cx[l] = 0.0;
            rhs[0][s] = 0.0;
#pragma unroll
            for (int b = 0; b < P; ++b)
                rhs[1 + b][s] = 0.0;
            if (live) {
                const double *r = E.rec + idx * E.rs;
#pragma unroll
                for (int l = 0; l < D; ++l)
                    cx[l] = r[l] * E.inv_rho[l];
                rhs[0][s] = r[D];
#pragma unroll
                for (int b = 0; b < P; ++b)
                    rhs[1 + b][s] = r[D + 1 + b];
            }
#pragma unroll
            for (int l = 0; l < DP; l += 2)
                *reinterpret_cast<double2 *>(pts + a * DP + l) = make_double2(cx[l], cx[l + 1]);
            KLs[colb_r[s] + a] = live ? E.diag : 1.0;
            const unsigned bal = __ballot_sync(FULLMASK, live);
            nlive += __popc((G == 32) ? bal : ((bal >> (g * G)) & ((1u << (G & 31)) - 1u)));
        }
        const int pad = CAP - nlive; // identity rows at the front of the local frame
        __syncwarp();

        // ---- pair terms.  The table lists the off-diagonal pairs (a > c) by DESCENDING c, so the
        //      k(k-1)/2 pairs of the live points come first; they are dealt round-robin to the lanes
        //      of the group, two independent pairs per iteration (ILP), and staged in the packed
        //      triangles.  Pairs that touch a padding row are just zero-filled. ----
        const int nlp = nlive * (nlive - 1) / 2;
        {
            constexpr int NI = SM::NI; // independent pairs in flight per lane (ILP; registers are free here)
            unsigned nxt[NI];
#pragma unroll
            for (int h = 0; h < NI; ++h)
                nxt[h] = E.pair_tab[lg + h * G];
            for (int t0 = lg; t0 < nlp; t0 += NI * G) {
                unsigned ent[NI];
#pragma unroll
                for (int h = 0; h < NI; ++h)
                    ent[h] = nxt[h];
                if (t0 + NI * G < SM::TPAD) { // prefetch the next entries (L1-resident table)
#pragma unroll
                    for (int h = 0; h < NI; ++h)
                        nxt[h] = E.pair_tab[t0 + (NI + h) * G];
                }
                double Kv[NI], Dv[NI][QD];
#pragma unroll
                for (int h = 0; h < NI; ++h) {
                    const double *pa = pts + (ent[h] >> 24) * DP;
                    const double *pc = pts + ((ent[h] >> 16) & 255) * DP;
                    double dl[D];
#pragma unroll
                    for (int l = 0; l < DP; l += 2) {
                        const double2 va = *reinterpret_cast<const double2 *>(pa + l);
                        const double2 vc = *reinterpret_cast<const double2 *>(pc + l);
                        dl[l] = va.x - vc.x;
                        if (l + 1 < D)
                            dl[l + 1 < D ? l + 1 : l] = va.y - vc.y;
                    }
                    pair_terms_s<FAM, D>(E, etab, dl, Kv[h], Dv[h]);
                }
                // entries past nlp in the last iteration belong to padding pairs: they are written
                // here and overwritten with zeros below (after the warp sync)
#pragma unroll
                for (int h = 0; h < NI; ++h) {
                    const int kidx = ent[h] & 0xffff;
                    KLs[kidx] = Kv[h];
#pragma unroll
                    for (int j = 0; j < QD; ++j)
                        Dms[j * DSZ + kidx] = Dv[h][j];
                }
            }
            __syncwarp();
            for (int t = nlp + lg; t < SM::TOFF; t += G) {
                const unsigned e0 = E.pair_tab[t];
                const int kidx = e0 & 0xffff;
                KLs[kidx] = 0.0;
#pragma unroll
                for (int j = 0; j < QD; ++j)
                    Dms[j * DSZ + kidx] = 0.0;
            }
        }
        __syncwarp();

        // ---- own rows into registers ----
        double Kr[S][CAP];
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int c = 0; c < (s + 1) * G; ++c)
                Kr[s][c] = KLs[Geo::colbase(c) + rowi[s]];
        __syncwarp();

        // ---- square-root-free factorization K = Lt D Lt^T (Lt unit lower, D = diag(d)), right-looking,
        //      with the forward substitutions of y and X fused in.  The Cholesky factor of the reference
        //      is B = Lt D^(1/2); working with Lt and d keeps sqrt AND the diagonal scalings out of every
        //      dependent chain: at step j the UNSCALED column j (d_j on top) goes to the column store
        //      as soon as the previous update is done, and 1/d_j is formed by all lanes from the
        //      broadcast read, in parallel with the rest of the column loads. ----
        double invd[S]; // 1/d_a of the own rows
#pragma unroll
        for (int s = 0; s < S; ++s)
            invd[s] = 1.0;
        int failpiv = 0;
#pragma unroll
        for (int j = 1; j < CAP - 1; ++j) { // local row 0 is always padding: step 0 is the identity
            const int sj = j / G;
            const int oj = (sj & 1) ? (G - 1 - j % G) : (j % G);
            const double *col = KLs + Geo::colbase(j);
#pragma unroll
            for (int s = 0; s < S; ++s)
                if ((s + 1) * G - 1 >= j && rowi[s] >= j)
                    KLs[Geo::colbase(j) + rowi[s]] = Kr[s][j];
            double xr[1 + P];
#pragma unroll
            for (int r = 0; r < 1 + P; ++r)
                xr[r] = __shfl_sync(FULLMASK, rhs[r][sj], oj, G); // (Lt^-1 rhs)_j is final at step j
            __syncwarp();
            // pairs (c0, c0+1) are read as one 128-bit broadcast load; the parity of the first pair is
            // static (colbase(j) + c0 must be even)
            const int cs = ((Geo::colbase(j) + j) & 1) ? j + 1 : j;
            double dj;
            if (cs != j)
                dj = col[j];
            double2 v0;
            if (cs == j) {
                v0 = *reinterpret_cast<const double2 *>(col + j);
                dj = v0.x;
            }
            failpiv = (failpiv == 0 && dj <= E.piv_floor) ? (j + 1) : failpiv;
            const double rj = rcp_pos(dj);
            // Lo[s] = Lt[row][j] for rows below the pivot row, exactly 0 for finished rows, so the
            // updates need no per-row predicates (a finished row just adds -0 * x)
            double Lo[S];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if ((s + 1) * G - 1 > j) {
                    const double Ls = Kr[s][j] * rj;
                    Lo[s] = (rowi[s] > j) ? Ls : 0.0;
                    Kr[s][j] = Ls;
                } else {
                    Lo[s] = 0.0;
                }
                if ((s + 1) * G - 1 >= j)
                    invd[s] = (rowi[s] == j) ? rj : invd[s];
            }
#pragma unroll
            for (int r = 0; r < 1 + P; ++r)
#pragma unroll
                for (int s = 0; s < S; ++s)
                    if ((s + 1) * G - 1 > j)
                        rhs[r][s] = fma(-Lo[s], xr[r], rhs[r][s]);
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
        // last pivot d_e (row CAP-1 = the observation itself): nothing left to update
        constexpr int se = S - 1;
        constexpr int oe = Geo::lane_of(CAP - 1);
        const double d_e = __shfl_sync(FULLMASK, Kr[se][CAP - 1], oe, G);
        failpiv = (failpiv == 0 && d_e <= E.piv_floor) ? CAP : failpiv;
        const double rho_e = rcp_pos(d_e);
        invd[se] = (rowi[se] == CAP - 1) ? rho_e : invd[se];

        // ---- ut = Lt^-T e_last (u = ut / sqrt(d_e)): the lane owning index j accumulates
        //      sb_j = sum_{l>j} K(l,j) ut_l from the unscaled column store, ut_j = e_j - sb_j / d_j.  As
        //      soon as ut_l is known (and broadcast) it is also applied to the packed derivative
        //      matrices, tt_r += D_r[., l] ut_l, so D_r u needs no separate mat-vec pass.  Element
        //      (a, l) of the symmetric D_r lives at colbase(a) + l (a < l) or colbase(l) + a (a >= l;
        //      the diagonal holds zeros). ----
        double sb[S], eb[S], rr[QD + 1][S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            sb[s] = 0.0;
            eb[s] = (rowi[s] == CAP - 1) ? 1.0 : 0.0;
#pragma unroll
            for (int r = 0; r < QD; ++r)
                rr[r][s] = 0.0;
        }
#pragma unroll
        for (int l = CAP - 1; l >= 1; --l) {
            const int sl = l / G;
            const int ol = (sl & 1) ? (G - 1 - l % G) : (l % G);
            const double ul = __shfl_sync(FULLMASK, fma(-sb[sl], invd[sl], eb[sl]), ol, G);
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const bool above = rowi[s] < l;
                if (s * G < l) { // slot has rows < l
                    const double Klj = above ? KLs[colb_r[s] + l] : 0.0;
                    sb[s] = fma(Klj, ul, sb[s]);
                }
                const int addr = above ? (colb_r[s] + l) : (Geo::colbase(l) + rowi[s]);
#pragma unroll
                for (int r = 0; r < QD; ++r)
                    rr[r][s] = fma(Dms[r * DSZ + addr], ul, rr[r][s]);
            }
        }
#pragma unroll
        for (int s = 0; s < S; ++s) // padding rows: ut = 0 whatever was read
            rr[QD][s] = (rowi[s] < pad) ? 0.0 : fma(-sb[s], invd[s], eb[s]);

        // ---- [tt_1..tt_QD, ut] through Lt^-1 (unit-diagonal forward sweeps on the register-resident rows) ----
#pragma unroll
        for (int j = 1; j < CAP - 1; ++j) {
            const int sj = j / G;
            const int oj = (sj & 1) ? (G - 1 - j % G) : (j % G);
            double Lm[S];
#pragma unroll
            for (int s = 0; s < S; ++s)
                Lm[s] = ((s + 1) * G - 1 > j && rowi[s] > j) ? Kr[s][j] : 0.0;
#pragma unroll
            for (int r = 0; r < QD + 1; ++r) {
                const double x = __shfl_sync(FULLMASK, rr[r][sj], oj, G);
#pragma unroll
                for (int s = 0; s < S; ++s)
                    if ((s + 1) * G - 1 > j)
                        rr[r][s] = fma(-Lm[s], x, rr[r][s]);
            }
        }
        // Now, with <a,b> = sum_a a_a b_a / d_a and s = 1/sqrt(d_e):
        //   z = D^-1/2 yt, W = D^-1/2 Xt            (yt = rhs[0], Xt = rhs[1+b])
        //   c_r = s D^-1/2 ct_r, w = B^-1 u = s D^-1/2 wt   (ct_r = rr[r], wt = rr[QD])
        // so every dot product below is a weighted dot of the tilde vectors times s or s^2.
        auto gsum = [](double v) {
#pragma unroll
            for (int off = G / 2; off > 0; off >>= 1)
                v += __shfl_xor_sync(FULLMASK, v, off, G);
            return v;
        };
        auto dot = [&](const double (&x)[S], const double (&y)[S]) {
            double s0 = 0.0;
#pragma unroll
            for (int s = 0; s < S; ++s)
                s0 = fma(x[s], y[s], s0);
            return gsum(s0);
        };
        const double sq = rsqrt_pos(d_e); // s = 1/sqrt(d_e)
        const double ze = __shfl_sync(FULLMASK, rhs[0][se], oe, G) * sq;
        const double w_e = __shfl_sync(FULLMASK, rr[QD][se], oe, G) * rho_e;
        double we[P], ce[Q], zc[Q], wc[P * Q], cc[Q * Q];
#pragma unroll
        for (int b = 0; b < P; ++b)
            we[b] = __shfl_sync(FULLMASK, rhs[1 + b][se], oe, G) * sq;
        double rrw[QD + 1][S]; // ct_r / d, wt / d
#pragma unroll
        for (int r = 0; r < QD + 1; ++r)
#pragma unroll
            for (int s = 0; s < S; ++s)
                rrw[r][s] = rr[r][s] * invd[s];
        const double jit = E.jitter, is2 = E.inv_sig2, s2 = E.sig2;
        {
            const double zw = dot(rhs[0], rrw[QD]) * sq;
            const double ww = dot(rr[QD], rrw[QD]) * rho_e;
            ce[0] = (1.0 - jit * w_e) * is2;
            ce[Q - 1] = s2 * w_e;
            zc[0] = (ze - jit * zw) * is2;
            zc[Q - 1] = s2 * zw;
            cc[0] = (1.0 - 2.0 * jit * w_e + jit * jit * ww) * is2 * is2;
            cc[Q - 1] = cc[(Q - 1) * Q] = w_e - jit * ww;
            cc[(Q - 1) * Q + Q - 1] = s2 * s2 * ww;
#pragma unroll
            for (int b = 0; b < P; ++b) {
                const double Ww = dot(rhs[1 + b], rrw[QD]) * sq;
                wc[b * Q] = (we[b] - jit * Ww) * is2;
                wc[b * Q + Q - 1] = s2 * Ww;
            }
#pragma unroll
            for (int r = 0; r < QD; ++r) {
                const double cde = __shfl_sync(FULLMASK, rr[r][se], oe, G) * rho_e;
                const double wcd = dot(rr[QD], rrw[r]) * rho_e;
                ce[1 + r] = cde;
                zc[1 + r] = dot(rhs[0], rrw[r]) * sq;
                cc[1 + r] = cc[(1 + r) * Q] = (cde - jit * wcd) * is2;
                cc[(1 + r) * Q + Q - 1] = cc[(Q - 1) * Q + 1 + r] = s2 * wcd;
#pragma unroll
                for (int b = 0; b < P; ++b)
                    wc[b * Q + 1 + r] = dot(rhs[1 + b], rrw[r]) * sq;
#pragma unroll
                for (int r2 = 0; r2 <= r; ++r2) {
                    const double v = dot(rr[r], rrw[r2]) * rho_e;
                    cc[(1 + r) * Q + 1 + r2] = v;
                    cc[(1 + r2) * Q + 1 + r] = v;
                }
            }
        }
        const double logdet = log(d_e);
        const bool emit = active && failpiv == 0;
        // every lane evaluates every term (they are a handful of flops each) and keeps the ones it
        // owns (o mod G == lane); selects instead of L divergent branches
#pragma unroll
        for (int o = 0; o < L; ++o) {
            const double v = emit_value(o, P, Q, A, logdet, ze, we, ce, zc, wc, cc);
            acc[o / G] += (emit && lg == (o % G)) ? v : 0.0;
        }
        if (E.rows != nullptr && emit) {
#pragma unroll
            for (int o = 0; o < L; ++o)
                if (lg == (o % G))
                    E.rows[(size_t)(i - E.i0) * L + o] = emit_value(o, P, Q, A, logdet, ze, we, ce, zc, wc, cc);
        }
        if (active && failpiv != 0 && lg == 0) {
            report_failure(E, i, failpiv - pad);
            if (E.fail_rows)
                E.fail_rows[i - E.i0] = failpiv - pad;
        }
        __syncwarp();
    }

    // ---- block partial: add the groups of this warp in fixed order, one row of `partials` per block ----
#pragma unroll
    for (int t = 0; t < NACC; ++t) {
        double v = acc[t];
#pragma unroll
        for (int off = G; off < 32; off <<= 1)
            v += __shfl_xor_sync(FULLMASK, v, off);
        const int o = t * G + lg;
        if (g == 0 && o < L)
            E.partials[(size_t)blockIdx.x * L + o] = v;
    }
    vb_finish(E, 1);
}

