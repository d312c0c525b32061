// kernel_tiled.cuh -- layout TILED_REG: the fast path of the likelihood evaluation.
//
// G lanes of a warp cooperate on one observation (32/G observations per warp).  Every lane owns S
// rows of the local (CAP x CAP, CAP = G*S) covariance matrix, folded boustrophedon-wise (slot s even:
// row s*G + lane, slot s odd: row s*G + G-1-lane) so that the triangular work is balanced, and keeps
// those rows IN REGISTERS from the moment their entries are computed until the last sweep.
//
// The kernel is bound by the shared-memory / shuffle data pipe (LSU), not by FP64 issue (measured:
// tools/micro/lds_groups.cu -- a broadcast LDS.128 costs 2.2 LSU cycles per warp whatever the number
// of lane groups, a 32-bit SHFL 1.1, 32 distinct doubles 2), so the design minimises LSU traffic per
// observation:
//   * ROW-OWNER pair terms: the lane that owns rows a0 (slot 2h) and a1 (slot 2h+1) evaluates all
//     pairs (a1, c), c < a1, then (a0, c), c < a0 -- a0 + a1 is the same for every lane, so the pair
//     work is balanced with NO pair table and NO staging of K: the covariance goes straight into the
//     register that the factorization will use (static register index: the loop is fully unrolled),
//     the point of row a is already in registers and the point of column c is one (mostly broadcast)
//     128-bit load.  Only the range-derivative values go to shared memory (packed triangle D_r).
//   * at factorization step j the unscaled column j is written once and read back as broadcast
//     128-bit loads; the columns stay in shared memory and serve the transposed back-substitution
//     for u = B^-T e_last, into which the symmetric mat-vec D_r u is fused.
// The forward substitutions of y and X ride along inside the factorization sweep.
//
// Exact-size instances (template parameter NP, pair-table variant): an instance may declare its first NP local rows
// padding rows of EVERY observation it serves (m+1 <= CAP-NP); the shared-memory triangles are then packed for
// CAP-NP+1 rows and the column loops start at NP -- fewer bytes per observation, more resident warps (TileGeom).
// How many resident blocks an instance is compiled for: tiled_launch_blocks below (measured rules).
//
// Rows with fewer than CAP live points (local row 0 always; the ragged head rows i < m; m+1 < CAP-1)
// are padding rows at the FRONT of the local frame: unit diagonal, zero data, and coordinates 1e30
// scaled units away from everything (distinct per row), so every pair term that touches them
// underflows to (at most) 1e-200 without any mask in the pair loop; chol([[I,0],[0,K]]) =
// [[I,0],[0,B]] leaves every accumulator term of the real block unchanged.
//
// Same per-observation mathematics as kernel_warp_smem.cuh / the reference's _obs_kernel
// (/root/reference/pkg/src/vecchiagp/engine/_kernels.pyx:347-381); see common.cuh for the map.
#pragma once
#include "tiled_common.cuh"
#include <type_traits>

// Experiment knobs (ablations, clock accounting, alternative schedules) are honoured only in builds made with
// -DVB200_EXPERIMENTS (tools/build_variant.py); the product build always uses the defaults below.
#if !defined(VB200_EXPERIMENTS) && (defined(TILED_ABLATE) || defined(TILED_STAGGER_NS) || defined(TILED_CLOCKS) || \
                                    defined(TILED_HEAD_SHFL) || defined(TILED_WPB) || defined(TILED_MINB) || \
                                    defined(TILED_NO_SMEM_BLOCKS) || defined(TILED_DYNAMIC) || defined(TILED_RHS_LATE))
#error "TILED_* experiment knobs need -DVB200_EXPERIMENTS"
#endif
#ifndef TILED_WPB
#define TILED_WPB 1 // warps per block; > 1: the warps of a block pass the phases of a batch together (barriers)
#endif
#ifndef TILED_ABLATE
#define TILED_ABLATE 0 // timing experiments only: bit 0 skips the pair phase, 1 factorization, 2 back-substitution, 3 sweeps,
                       // 5 replaces exp by a product, 6 adds 320 independent DFMAs per batch
#endif
#ifndef TILED_PD
#define TILED_PD 2 // broadcast loads in flight ahead of their FMAs in the factorization (2..5 measured within 2 %)
#endif
#ifndef TILED_STAGGER_NS
#define TILED_STAGGER_NS 0 // experiment: start offset between the resident blocks of an SM (measured: no effect)
#endif
#ifndef TILED_PREFETCH
#define TILED_PREFETCH 0 // 1: software-pipelined gather (next batch's indices / records requested one batch ahead);
                         // measured slower at 12 warps per SM (registers), faster stand-alone: profiles/r2_experiments.md
#endif
#ifndef TILED_FUSE_DU
#define TILED_FUSE_DU 1 // the mat-vec D_r u rides in the stalls of the back-substitution chain (0: separate pass; 4 % slower)
#endif
#ifndef TILED_DD
#define TILED_DD 2 // steps (of two columns) of D_r loads in flight ahead of the mat-vec FMAs
#endif
#ifndef TILED_BD
#define TILED_BD 4 // column-store loads in flight ahead of the back-substitution chain
#endif
#ifndef TILED_RHS_LATE
#define TILED_RHS_LATE 0 // 1: the forward substitutions of y and X run in the sweep loop after the back-substitution
                         // (next to [D_r u, u]) instead of inside the factorization sweep
#endif
#ifndef TILED_RNI
#define TILED_RNI 4 // independent pair evaluations in flight per lane (row-owner pair phase)
#endif
// experiment (-DTILED_CLOCKS): per-phase clock64 accounting, summed over warps into E.dbg_clocks[0..15]
// (and per factorization step into [16..16+CAP)); read back with vb200_debug_clocks.
#ifdef TILED_CLOCKS
#define PHASE_MARK(k)                                                                                    \
    do {                                                                                                 \
        const long long _t = clock64();                                                                  \
        phc[k] += _t - pht;                                                                              \
        pht = _t;                                                                                        \
    } while (0)
#else
#define PHASE_MARK(k) do { } while (0)
#endif

// exp table premultiplied by sigma^2 (every family's covariance is sigma^2 * exp(-.) * polynomial)
// and range-derivative values WITHOUT their constant factor (1/range, 1/(3 range), 1/range_axis):
// the factor is applied once per row to D_r u after the back-substitution (dscale below).
template <int FAM, int D>
__device__ __forceinline__ void pair_terms_r(const EvalParams &E, const double *etab, const double (&dl)[D],
                                             double &Kv, double (&Dv)[FamTraits<FAM, D>::QD])
{
    if constexpr (FAM == FAM_MATERN) {
        double x2 = 1e-300;
#pragma unroll
        for (int l = 0; l < D; ++l)
            x2 = fma(dl[l], dl[l], x2);
        // inlined: the general Matern only runs the ROLLED pair-table pair phase, and an out-of-line callee would take
        // the kernel parameters by address, i.e. from a local-memory copy instead of the constant bank (measured 2x)
        matern_terms(E, x2 * rsqrt_pos(x2), E.inv_rho[0], Kv, Dv[0], Dv[1]);
    } else if constexpr (FAM == FAM_EXP_ISO || FAM == FAM_MATERN15 || FAM == FAM_MATERN25) {
        double x2 = 1e-300;
#pragma unroll
        for (int l = 0; l < D; ++l)
            x2 = fma(dl[l], dl[l], x2);
        // x = sqrt(x2) = g (1 + e/2 + 3 e^2/8), g = x2 y, e = 1 - x2 y^2, y = MUFU.RSQ64H seed
        // e from g (one FMA instead of a product and an FMA; same chain depth)
        const double y = rsqrt_seed(x2);
        const double g = x2 * y;
        const double e = fma(-g, y, 1.0);
        const double x = fma(fma(e, 0.375, 0.5), g * e, g);
#if (TILED_ABLATE & 32)
        const double se = 1e-3 * x2; // timing experiment: no exp (11 FP64 + 6 integer instructions + 1 table load less)
#else
        const double se = exp_neg(x, etab); // sigma^2 exp(-x)
#endif
        if constexpr (FAM == FAM_EXP_ISO) {
            Kv = se;
            Dv[0] = se * x;                 // * 1/range
        } else if constexpr (FAM == FAM_MATERN15) {
            Kv = fma(se, x, se);
            Dv[0] = se * x2;                // * 1/range
        } else {
            const double x1 = 1.0 + x;
            Kv = se * fma(x2, 1.0 / 3.0, x1);
            Dv[0] = (se * x2) * x1;         // * 1/(3 range)
        }
    } else {
        double sc[D];
        double s2 = 1e-300, sp2 = 0.0;
#pragma unroll
        for (int l = 0; l < D; ++l) {
            sc[l] = dl[l] * dl[l];
            s2 += sc[l];
            if (l < D - 1)
                sp2 += sc[l];
        }
        const double rs = rsqrt_pos(s2);
        Kv = exp_neg(s2 * rs, etab);
        const double g = Kv * rs;
        if constexpr (FAM == FAM_EXP_ANISO) {
#pragma unroll
            for (int l = 0; l < D; ++l)
                Dv[l] = g * sc[l];          // * 1/range_l
        } else {
            Dv[0] = g * sp2;                // * 1/range_space
            Dv[1] = g * sc[D - 1];          // * 1/range_time
        }
    }
}

// the constant factor of range-derivative matrix r that pair_terms_r leaves out
template <int FAM, int D>
__device__ __forceinline__ double deriv_scale(const EvalParams &E, int r)
{
    if constexpr (FAM == FAM_MATERN)
        return 1.0;
    else if constexpr (FAM == FAM_MATERN25)
        return E.inv_rho[0] * (1.0 / 3.0);
    else if constexpr (FAM == FAM_EXP_ISO || FAM == FAM_MATERN15)
        return E.inv_rho[0];
    else if constexpr (FAM == FAM_EXP_ANISO)
        return E.inv_rho[r];
    else
        return r == 0 ? E.inv_rho[0] : E.inv_rho[D - 1];
}

// compile-time loop: f(std::integral_constant<int, K>) for K0 <= K < K1 (register indices must be static)
template <int K0, int K1, class F>
__device__ __forceinline__ void static_for(F &&f)
{
    if constexpr (K0 < K1) {
        f(std::integral_constant<int, K0>{});
        static_for<K0 + 1, K1>(f);
    }
}

// Static schedule of the row-owner pair phase: flat step k -> slot pair h (h == NH: the unpaired last
// slot of an odd S) and step t within it.
template <int G, int S>
struct PairSched {
    enum : int { ALL1 = 0, ALL0 = 1, MIXED = 2, ODD_MIXED = 3 };
    static constexpr int NH = S / 2;
    __host__ __device__ static constexpr int T(int h) { return (4 * h + 2) * G - 1; }
    // h = 0: lane 0 owns the padding row 0 in slot 0, so its row a1 = 2G-1 needs one more step
    __host__ __device__ static constexpr int steps(int h) { return h < NH ? T(h) - 2 + (h == 0 ? 1 : 0) : S * G - 2; }
    __host__ __device__ static constexpr int total()
    {
        int n = 0;
        for (int h = 0; h < NH + (S % 2); ++h)
            n += steps(h);
        return n;
    }
    static constexpr int NIT = total();
    __host__ __device__ static constexpr int h_of(int k)
    {
        int h = 0;
        while (k >= steps(h)) {
            k -= steps(h);
            ++h;
        }
        return h;
    }
    __host__ __device__ static constexpr int t_of(int k)
    {
        int h = 0;
        while (k >= steps(h)) {
            k -= steps(h);
            ++h;
        }
        return k + 1;
    }
    __host__ __device__ static constexpr int kind(int k)
    {
        const int h = h_of(k), t = t_of(k);
        if (h == NH)
            return t < (S - 1) * G ? ALL1 : ODD_MIXED;
        return t < (2 * h + 1) * G ? ALL1 : (t > (2 * h + 2) * G - 2 ? ALL0 : MIXED);
    }
};

// Element (a, l) of a packed symmetric matrix (lower triangle, columns back to back: (r, c), r >= c, at
// colbase(c) + r) for a row a of slot s and a compile-time l.  Rows of slot s lie in [sG, (s+1)G): l beyond
// the slot is always the column part (static offset from the lane's column base), l before it always the
// row part (static offset from the row index); only inside the diagonal block does the side depend on the
// lane.  `oz` is an opaque zero (see the kernel): it keeps the lane-dependent selects inside the batch loop.
template <int G, int S, int NP, int s, int l>
__device__ __forceinline__ double sym_packed_load(const double *M, const int colb_a, const int a, const int oz)
{
    using Geo = TileGeom<G, S, NP>;
    if constexpr (l >= (s + 1) * G)
        return M[colb_a + l];
    else if constexpr (l < s * G)
        return M[Geo::colbase(l) + a];
    else {
        const int ao = a + oz;
        return M[(ao < l) ? (colb_a + l) : (Geo::colbase(l) + ao)];
    }
}

// rows a = rowi[s] of columns l0 = 2h, l0 + 1 of QD packed symmetric matrices, and the pair (u_l0, u_l0+1)
template <int G, int S, int NP, int QD, int H, int s = 0>
__device__ __forceinline__ void sym_fetch_pair(const double *Dms, const int DSZ, const double *us, const int (&colb_r)[S],
                                               const int (&rowi)[S], const int oz, double (&dv)[2][QD][S], double2 &uv)
{
    constexpr int l0 = 2 * H, l1 = l0 + 1;
    if constexpr (s == 0)
        uv = *reinterpret_cast<const double2 *>(us + l0);
    if constexpr (s < S) {
#pragma unroll
        for (int r = 0; r < QD; ++r) {
            dv[0][r][s] = 0.0;
            if constexpr (l0 >= 1)
                dv[0][r][s] = sym_packed_load<G, S, NP, s, l0>(Dms + r * DSZ, colb_r[s], rowi[s], oz);
            dv[1][r][s] = sym_packed_load<G, S, NP, s, l1>(Dms + r * DSZ, colb_r[s], rowi[s], oz);
        }
        sym_fetch_pair<G, S, NP, QD, H, s + 1>(Dms, DSZ, us, colb_r, rowi, oz, dv, uv);
    }
}

// rows a = rowi[s] of column l of QD packed symmetric matrices
template <int G, int S, int NP, int QD, int l, int s = 0>
__device__ __forceinline__ void sym_fetch_col(const double *Dms, const int DSZ, const int (&colb_r)[S], const int (&rowi)[S],
                                              const int oz, double (&dv)[QD][S])
{
    if constexpr (s < S) {
#pragma unroll
        for (int r = 0; r < QD; ++r)
            dv[r][s] = sym_packed_load<G, S, NP, s, l>(Dms + r * DSZ, colb_r[s], rowi[s], oz);
        sym_fetch_col<G, S, NP, QD, l, s + 1>(Dms, DSZ, colb_r, rowi, oz, dv);
    }
}

template <int G, int S, int D, int QD, int NP = 1>
struct LikSmem {
    using Geo = TileGeom<G, S, NP>;
    static constexpr int DP = (D + 1) & ~1;                 // padded coordinate stride (16-byte rows)
    static constexpr int PTS = Geo::CAP * DP;               // scaled coordinates of the local frame
    // The column store of the factorization and every D_r share ONE packing: element (a, c), a >= c,
    // at colbase(c) + a (columns back to back).
    static constexpr int DSZ = (Geo::TRI + 1) & ~1;
    static constexpr int RAW = PTS + Geo::KL + QD * DSZ;
    // Per-observation stride = 16/OPW (mod 16) doubles: the 16-byte broadcast chunks of the OPW lane
    // groups fall on different banks AND the G-contiguous stores of the groups tile the 16 8-byte
    // banks exactly twice (measured conflict-free: tools/micro/lds_groups.cu).
    static constexpr int WANT = (Geo::OPW >= 2) ? 16 / Geo::OPW : 0;
    static constexpr int PER_OBS = RAW + ((WANT - RAW % 16) + 16) % 16;
    static constexpr int TOTAL = VB_EXPTAB + TILED_WPB * Geo::OPW * PER_OBS;
};

// phase boundary: with several warps per block they walk the (straight-line, > 64 KB) instruction stream
// together, so one instruction-cache fill serves all of them
__device__ __forceinline__ void phase_sync()
{
    if (TILED_WPB > 1)
        __syncthreads();
    else
        __syncwarp();
}

// PT = false: row-owner pair phase (fully unrolled, K straight into registers) -- the narrow tiers.
// PT = true : pair-TABLE pair phase -- a rolled loop over a device pair table (pairs dealt round-robin to the
//             lanes, two in flight per lane), K staged in the packed triangle in shared memory and read back
//             row-wise into registers.  Small code where the unrolled row-owner phase would be 60-80 steps long
//             (CAP = 48 / 64) and cheap around an out-of-line call (general-order Matern: the Bessel routine).
//             Pairs that touch a padding row are not evaluated at all (the table lists live pairs first).
// Everything after the pair phase is shared.
// Resident blocks per SM the kernel is compiled for (__launch_bounds__): the register tier of the geometry, unless the
// instance's shared memory admits fewer blocks anyway -- then it is compiled for the next multiple of four at or below
// what fits (four schedulers per SM: 11 resident warps run no faster than 8, and 8 may use 255 registers instead of
// being held to the 168 of 12 blocks).  Measured at n = 2^20: space-time d = 3 5.75 -> 5.47 ms, anisotropic d = 2
// 5.48 -> 5.05 ms (two derivative matrices: 8 blocks fit), Matern-3/2 d = 3 p = 4 7.24 -> 6.25 ms (11 blocks fit;
// compiled for 11 it got slower, 7.46 ms).
// The design columns cost registers too (1 + P right-hand sides per row, (1+Q)(2+P+P^2)+Q^2 accumulator terms spread
// over the G lanes): measured at n = 2^20, Matern-3/2, d = 2 -- (16,2) tier, 12 -> 8 blocks: P = 1 4.28 -> 4.35 ms
// (kept at 12), P = 2 5.00 -> 4.75, P = 3 5.19 -> 5.08, P = 4 6.39 -> 5.75; (4,3) tier, 16 / 12 / 8 blocks: P = 1
// 0.515 / 0.581 / 0.644, P = 2 0.651 / 0.626 / 0.728, P = 3 0.818 / 0.792 / 0.831, P = 4 1.216 / 1.134 / 0.948;
// (8,3) tier: 12 blocks at every P (P = 4: 2.98 vs 2.99, P = 2: 2.35 vs 2.64).
template <int G, int S, int D, int QD, int NP, int P>
__host__ __device__ constexpr int tiled_launch_blocks()
{
    constexpr int base = tiled_min_blocks(G, S, NP);
#if !defined(TILED_NO_SMEM_BLOCKS) && !defined(TILED_MINB) && TILED_WPB == 1
    constexpr int by_reg = (base == 16) ? (P >= 4 ? 8 : (P >= 2 ? 12 : 16))
                                        : ((base == 12 && G == 16 && P >= 2) ? 8 : base);
    constexpr long long bytes = (long long)LikSmem<G, S, D, QD, NP>::TOTAL * 8 + 1024; // + the per-block reservation
    constexpr int by_smem = (int)(233472 / bytes) < 1 ? 1 : (int)(233472 / bytes);
    return by_smem >= by_reg ? by_reg : (by_smem >= 8 ? (by_smem / 4) * 4 : by_smem);
#else
    return base;
#endif
}

// NP > 1 (pair-table variant only): the first NP local rows are padding rows of every observation the instance
// serves (m+1 <= CAP-NP); see TileGeom.
template <int G, int S, int FAM, int D, int P, bool PT = false, int NP = 1>
__global__ void __launch_bounds__(32 * TILED_WPB, (tiled_launch_blocks<G, S, D, FamTraits<FAM, D>::QD, NP, P>() + TILED_WPB - 1) / TILED_WPB) vecchia_tiled_kernel(const EvalParams E)
{
    static_assert(!PT || TILED_WPB == 1, "the pair-table variant runs one warp per block");
    static_assert(NP == 1 || PT, "static padding rows are implemented for the pair-table variant");
    using Geo = TileGeom<G, S, NP>;
    using FT = FamTraits<FAM, D>;
    constexpr int CAP = Geo::CAP, OPW = Geo::OPW, QD = FT::QD, Q = FT::Q, Z = Geo::Z;
    using SM = LikSmem<G, S, D, QD, NP>;
    constexpr int DP = SM::DP, DSZ = SM::DSZ;
    constexpr int L = (1 + Q) * (2 + P + P * P) + Q * Q;
    constexpr int NACC = (L + G - 1) / G;
    const AccLayout A(P, Q);
    static_assert(CAP % 2 == 0 && CAP <= 128, "tier geometry");

    extern __shared__ double smem[];
    double *etab = smem;                             // sigma^2 2^(j/32), j < 32
    const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
    const int g = lane / G, lg = lane % G;
    double *obs = smem + VB_EXPTAB + (warp * OPW + g) * SM::PER_OBS;
    double *pts = obs;                               // CAP x DP scaled coordinates of the local frame
    double *KLs = obs + SM::PTS;                     // the column store of the factorization
    double *Dms = KLs + Geo::KL;                     // QD packed range-derivative matrices

    for (int t = threadIdx.x; t < VB_EXPTAB; t += 32 * TILED_WPB)
        etab[t] = E.sig2 * exp2((double)t * (1.0 / VB_EXPTAB));
    // never written again: diagonal and column 0 of every D_r (zero), column 0 of the column store
    for (int a = Z + lg; a < CAP; a += G) {
#pragma unroll
        for (int j = 0; j < QD; ++j) {
            Dms[j * DSZ + Geo::colbase(Z) + a] = 0.0;
            Dms[j * DSZ + Geo::colbase(a) + a] = 0.0;
        }
        KLs[Geo::colbase(Z) + a] = 0.0;
    }
    // rowm: the row a lane ADDRESSES in the packed triangles -- its own, or (static padding rows below Z, which are
    // not part of the packing) the padding row Z, whose entries are the zeros a padding row must read
    int rowi[S], rowm[S], colb_r[S];
#pragma unroll
    for (int s = 0; s < S; ++s) {
        rowi[s] = s * G + ((s & 1) ? (G - 1 - lg) : lg);
        rowm[s] = (Z > 0) ? max(rowi[s], Z) : rowi[s];
        colb_r[s] = Geo::colbase(rowm[s]);
    }
    double dscale[QD];
#pragma unroll
    for (int r = 0; r < QD; ++r)
        dscale[r] = deriv_scale<FAM, D>(E, r);
    double acc[NACC];
#pragma unroll
    for (int t = 0; t < NACC; ++t)
        acc[t] = 0.0;
    phase_sync();

    // experiment (profiles/r1_experiments.md): an initial offset between the resident blocks of an SM, to rule out
    // phase-locking of the warps (all in the FP64-heavy pair phase, then all in the factorization).  No effect.
    if (TILED_STAGGER_NS > 0) {
        const unsigned slot = blockIdx.x / E.sm_count; // k-th block of its SM (round-robin placement)
        for (unsigned w = 0; w < slot; ++w)
            __nanosleep(TILED_STAGGER_NS);
    }
    const int64_t nbatch = (E.i1 - E.i0 + OPW - 1) / OPW;
    const int64_t stride = (int64_t)gridDim.x * TILED_WPB;
#ifdef TILED_CLOCKS
    long long phc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, pht = clock64();
#if TILED_CLOCKS > 1
    long long stc[CAP];
#pragma unroll
    for (int t = 0; t < CAP; ++t)
        stc[t] = 0;
#endif
#endif
    // Software-pipelined gather: the neighbor indices of the NEXT batch are requested when the current
    // batch enters its back-substitution, its point records when it enters the contraction (the rows of K
    // are dead by then), so a batch starts with its inputs already in registers instead of waiting for an
    // HBM read (indices) followed by a dependent L2 read (records): 2 900 cycles per batch before.
    constexpr int RV = D + 1 + P; // values of a point record
    int64_t nidx[S];
    double nrec[S][RV];
    auto load_idx = [&](const int64_t batch, int64_t (&idx)[S]) {
        const int64_t i = E.i0 + batch * OPW + g;
        const bool act = batch < nbatch && i < E.i1;
        const int64_t *nrow = E.nn + (act ? (i - E.nn_row0) : 0) * E.mp1;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int col = CAP - 1 - rowi[s];
            idx[s] = -1;
            if (act && col < E.mp1)
                idx[s] = nrow[col];
        }
    };
    auto load_rec = [&](const int64_t (&idx)[S], double (&rv)[S][RV]) {
#pragma unroll
        for (int s = 0; s < S; ++s) {
#pragma unroll
            for (int t = 0; t < RV; ++t)
                rv[s][t] = 0.0;
            if (idx[s] >= 0) {
                const double *r = E.rec + idx[s] * E.rs;
#pragma unroll
                for (int t = 0; t < RV; ++t)
                    rv[s][t] = r[t];
            }
        }
    };
#if TILED_PREFETCH == 1
    load_idx((int64_t)blockIdx.x * TILED_WPB + warp, nidx);
    load_rec(nidx, nrec);
#elif TILED_PREFETCH == 2
    load_idx((int64_t)blockIdx.x * TILED_WPB + warp, nidx);
#elif TILED_PREFETCH == 3
    load_idx((int64_t)blockIdx.x * TILED_WPB + warp, nidx);
    load_rec(nidx, nrec);
#endif
    // every warp of a block runs the same number of rounds (barriers inside); surplus rounds are inactive
#ifdef TILED_DYNAMIC
    // experiment: batches handed out by a global counter instead of the static stride (NOT run-to-run reproducible:
    // the batches a block sums change from launch to launch) -- measures what schedule imbalance costs
    for (;;) {
        unsigned int nb_ = 0;
        if (lane == 0)
            nb_ = atomicAdd(E.tickets + VB_FINISH_MAXGROUPS, 1u);
        nb_ = __shfl_sync(FULLMASK, nb_, 0);
        if ((int64_t)nb_ >= nbatch)
            break;
        const int64_t batch = (int64_t)nb_;
#else
    for (int64_t batch0 = (int64_t)blockIdx.x * TILED_WPB; batch0 < nbatch; batch0 += stride) {
        const int64_t batch = batch0 + warp;
#endif
        const int64_t i = E.i0 + batch * OPW + g;
        const bool active = i < E.i1;
#if !TILED_PREFETCH || TILED_PREFETCH >= 4
        load_idx(batch, nidx);
        load_rec(nidx, nrec);
#if TILED_PREFETCH >= 4 || TILED_PREFETCH == 0
        // register-free: the index row of this warp's NEXT batch is requested into L2 (4) / L1 (6) now.  Product
        // build (TILED_PREFETCH == 0): behind the run-time flag E.prefetch, which the host sets when the point
        // records do not fit L2 (then the gather is an HBM round trip per neighbor instead of an L2 hit: measured at
        // n = 2^22, d = 3, p = 4: 27.2 -> 24.8 ms; at n = 2^20, where the records are L2-resident, it costs 1-2 %)
        // (not compiled into the d = 2, p = 1 instances: their 32-byte records fit L2 up to n = 2^21, and the extra
        // block costs the headline kernel 2 % through register allocation alone)
        if (TILED_PREFETCH >= 4 || (RV > 4 && E.prefetch)) {
            const int64_t inx = i + stride * OPW;
            if (inx < E.i1) {
                const int64_t *nrow = E.nn + (inx - E.nn_row0) * E.mp1;
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    const int col = CAP - 1 - rowi[s];
                    if (col < E.mp1) {
#if TILED_PREFETCH == 6
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(nrow + col));
#else
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(nrow + col));
#endif
                    }
                }
            }
        }
#endif
#elif TILED_PREFETCH == 2
        load_rec(nidx, nrec); // indices arrived one batch ago, the records were prefetched into L1 / L2
#endif
        // opaque zero, data-dependent in every iteration (indices are >= -1): blocks loop-invariant hoisting
        // where it costs registers
        const int oz = (int)((unsigned long long)(nidx[0] + 1) >> 63);

        // ---- gather: local index a <-> neighbor column CAP-1-a (observation last).  Coordinates are
        //      kept divided by the range of their axis.  Padding rows: diagonal 1, data 0, far away. ----
        double rhs[1 + P][S], pa[S][D], Kr[S][CAP];
        int nlive = 0;
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int a = rowi[s], col = CAP - 1 - a;
            (void)col;
            const bool live = nidx[s] >= 0;
            double cx[DP];
#pragma unroll
            for (int l = 0; l < DP; ++l)
                cx[l] = 0.0;
            if constexpr (!PT)
                cx[0] = 1e30 * (double)(a + 1); // far away: every pair term with a padding row underflows
            rhs[0][s] = 0.0;
#pragma unroll
            for (int b = 0; b < P; ++b)
                rhs[1 + b][s] = 0.0;
            if (live) {
#pragma unroll
                for (int l = 0; l < D; ++l)
                    cx[l] = nrec[s][l] * E.inv_rho[l];
                rhs[0][s] = nrec[s][D];
#pragma unroll
                for (int b = 0; b < P; ++b)
                    rhs[1 + b][s] = nrec[s][D + 1 + b];
            }
#pragma unroll
            for (int l = 0; l < D; ++l)
                pa[s][l] = cx[l];
#pragma unroll
            for (int l = 0; l < DP; l += 2)
                *reinterpret_cast<double2 *>(pts + a * DP + l) = make_double2(cx[l], cx[l + 1]);
            // diagonal block of the slot: the diagonal entry, zeros above it (never used, must be finite)
            const double dg = live ? E.diag : 1.0;
            if constexpr (PT) {
                if (Z == 0 || a >= Z)
                    KLs[colb_r[s] + a] = dg;
            } else {
#pragma unroll
                for (int c = s * G; c < (s + 1) * G; ++c)
                    Kr[s][c] = (c == a) ? dg : 0.0;
                if (s > 0)
                    Kr[s][0] = 0.0; // column 0 belongs to the padding row 0
            }
            const unsigned bal = __ballot_sync(FULLMASK, live);
            nlive += __popc((G == 32) ? bal : ((bal >> (g * G)) & ((1u << (G & 31)) - 1u)));
        }
        const int pad = CAP - nlive; // identity rows at the front of the local frame
        // wide tiers: factorization steps whose column belongs to a padding row of EVERY observation of the warp
        // are identity steps (multipliers ~1e-200) and skip their rank-1 update (a warp-uniform branch, only
        // compiled into the first NSKIP steps; the m = 30 tier has none)
        constexpr int NSKIP = (CAP >= 48) ? 16 : 0;
        int pad_w = pad;
        if constexpr (NSKIP > 0) {
#pragma unroll
            for (int off = G; off < 32; off <<= 1)
                pad_w = min(pad_w, __shfl_xor_sync(FULLMASK, pad_w, off));
        }
        phase_sync();
        PHASE_MARK(0);

        // ---- pair terms, row-owner.  Slot pair (s0, s1) = (2h, 2h+1): rows a0 = 2hG + lg and
        //      a1 = (2h+2)G - 1 - lg, a0 + a1 = T for every lane.  Step t: pair (a1, t) while t < a1,
        //      afterwards pair (a0, T-1-t).  Column 0 (t = 0, t = T-1) is the padding row: skipped.
        //      The steps are processed NI at a time -- all loads, then NI independent evaluation
        //      chains (the compiler interleaves them; one chain alone is ~25 dependent FP64
        //      instructions), then all stores -- because a store to D_r between two loads of the
        //      point table would serialise the chains (the compiler cannot prove they do not alias). ----
        if constexpr (PT) {
            // ---- pair-table pair phase.  The table lists the off-diagonal pairs (a > c) by DESCENDING c, so the
            //      k(k-1)/2 pairs among the live points come first; the rest is zero-filled. ----
            using TS = TileSmem<G, S, D, QD, NP>;
            // pairs in flight per lane: two for the closed forms; ONE for the general Matern, whose Bessel evaluations
            // are long enough to spill when two are interleaved (measured 38 ms against 50 ms per evaluation with the
            // three-order central difference; with the analytic smoothness derivative 20.1 against 27.0 ms, and with
            // the NI series sharing one term loop 18.5 / 22.1 / 33.5 / 31.7 ms for NI = 1 / 2 / 3 / 4)
#ifndef TILED_MATERN_NI
#define TILED_MATERN_NI 1
#endif
            constexpr int NI = (FAM == FAM_MATERN) ? TILED_MATERN_NI : TS::NI;
            const int nlp = nlive * (nlive - 1) / 2;
            unsigned nxt[NI];
#pragma unroll
            for (int h = 0; h < NI; ++h)
                nxt[h] = E.pair_tab[lg + h * G];
            for (int t0 = lg; t0 < nlp; t0 += NI * G) {
                unsigned ent[NI];
#pragma unroll
                for (int h = 0; h < NI; ++h)
                    ent[h] = nxt[h];
                if (t0 + NI * G < TS::TPAD) { // prefetch the next entries (L1-resident table)
#pragma unroll
                    for (int h = 0; h < NI; ++h)
                        nxt[h] = E.pair_tab[t0 + (NI + h) * G];
                }
                double Kv[NI], Dv[NI][QD];
#pragma unroll
                for (int h = 0; h < NI; ++h) {
                    const double *pra = pts + (ent[h] >> 24) * DP;
                    const double *prc = pts + ((ent[h] >> 16) & 255) * DP;
                    double dl[D];
#pragma unroll
                    for (int l = 0; l < DP; l += 2) {
                        const double2 va = *reinterpret_cast<const double2 *>(pra + l);
                        const double2 vc = *reinterpret_cast<const double2 *>(prc + l);
                        dl[l] = va.x - vc.x;
                        if (l + 1 < D)
                            dl[l + 1 < D ? l + 1 : l] = va.y - vc.y;
                    }
                    pair_terms_r<FAM, D>(E, etab, dl, Kv[h], Dv[h]);
                }
                // entries past nlp in the last iteration belong to padding pairs: written here, overwritten with
                // zeros below (after the warp sync)
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
            for (int t = nlp + lg; t < TS::TOFF; t += G) {
                const int kidx = E.pair_tab[t] & 0xffff;
                KLs[kidx] = 0.0;
#pragma unroll
                for (int j = 0; j < QD; ++j)
                    Dms[j * DSZ + kidx] = 0.0;
            }
            __syncwarp();
            // own rows into registers (entries above the diagonal: finite, never used)
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int c = Z; c < (s + 1) * G; ++c)
                    Kr[s][c] = KLs[Geo::colbase(c) + rowm[s]];
        } else {
            using PS = PairSched<G, S>;
            constexpr int NI = TILED_RNI;
            if (!(TILED_ABLATE & 1))
            static_for<0, (PS::NIT + NI - 1) / NI>([&](auto chunk_c) {
                constexpr int k0 = decltype(chunk_c)::value * NI;
                double dl[NI][D];
                bool prv[NI];
                static_for<0, NI>([&](auto u_c) {
                    constexpr int u = decltype(u_c)::value, k = k0 + u;
                    if constexpr (k < PS::NIT) {
                        constexpr int h = PS::h_of(k), t = PS::t_of(k), kind = PS::kind(k);
                        constexpr int s1 = (h < PS::NH) ? 2 * h + 1 : S - 1, s0 = (h < PS::NH) ? 2 * h : S - 1;
                        constexpr int c1 = t, c0 = (h < PS::NH) ? PS::T(h) - 1 - t : t;
                        bool pr = true;
                        if constexpr (kind == PS::MIXED)
                            pr = lg < (2 * h + 2) * G - 1 - t; // t < a1
                        if constexpr (kind == PS::ODD_MIXED)
                            pr = t < rowi[S - 1];
                        prv[u] = pr;
                        const double *pc = pts + ((kind == PS::ALL0) ? c0 : (kind == PS::MIXED ? (pr ? c1 : c0) : c1)) * DP;
                        auto own = [&](int l) { // coordinate l of the row point of this step
                            return (kind == PS::ALL0) ? pa[s0][l] : (kind == PS::MIXED ? (pr ? pa[s1][l] : pa[s0][l]) : pa[s1][l]);
                        };
#pragma unroll
                        for (int l = 0; l < DP; l += 2) {
                            const double2 vc = *reinterpret_cast<const double2 *>(pc + l);
                            dl[u][l] = own(l) - vc.x;
                            if (l + 1 < D)
                                dl[u][l + 1 < D ? l + 1 : l] = own(l + 1 < D ? l + 1 : l) - vc.y;
                        }
                    }
                });
                double Kv[NI], Dv[NI][QD];
                static_for<0, NI>([&](auto u_c) {
                    constexpr int u = decltype(u_c)::value;
                    if constexpr (k0 + u < PS::NIT)
                        pair_terms_r<FAM, D>(E, etab, dl[u], Kv[u], Dv[u]);
                });
                static_for<0, NI>([&](auto u_c) {
                    constexpr int u = decltype(u_c)::value, k = k0 + u;
                    if constexpr (k < PS::NIT) {
                        constexpr int h = PS::h_of(k), t = PS::t_of(k), kind = PS::kind(k);
                        constexpr int s1 = (h < PS::NH) ? 2 * h + 1 : S - 1, s0 = (h < PS::NH) ? 2 * h : S - 1;
                        constexpr int c1 = t, c0 = (h < PS::NH) ? PS::T(h) - 1 - t : t;
                        const bool pr = prv[u];
                        if constexpr (kind == PS::ALL1) {
                            Kr[s1][c1] = Kv[u];
#pragma unroll
                            for (int r = 0; r < QD; ++r)
                                Dms[r * DSZ + Geo::colbase(c1) + rowi[s1]] = Dv[u][r];
                        } else if constexpr (kind == PS::ALL0) {
                            Kr[s0][c0] = Kv[u];
#pragma unroll
                            for (int r = 0; r < QD; ++r)
                                Dms[r * DSZ + Geo::colbase(c0) + rowi[s0]] = Dv[u][r];
                        } else if constexpr (kind == PS::MIXED) {
                            Kr[s1][c1] = pr ? Kv[u] : Kr[s1][c1];
                            if constexpr (c0 > 0) {
                                Kr[s0][c0] = pr ? Kr[s0][c0] : Kv[u];
                                const int dst = pr ? (Geo::colbase(c1) + rowi[s1]) : (Geo::colbase(c0) + rowi[s0]);
#pragma unroll
                                for (int r = 0; r < QD; ++r)
                                    Dms[r * DSZ + dst] = Dv[u][r];
                            } else if (pr) { // column 0 is the padding row: only the (a1, t) pairs are real
#pragma unroll
                                for (int r = 0; r < QD; ++r)
                                    Dms[r * DSZ + Geo::colbase(c1) + rowi[s1]] = Dv[u][r];
                            }
                        } else { // unpaired last slot, steps where some lanes have run out of pairs
                            Kr[s1][c1] = pr ? Kv[u] : Kr[s1][c1];
                            if (pr) {
#pragma unroll
                                for (int r = 0; r < QD; ++r)
                                    Dms[r * DSZ + Geo::colbase(c1) + rowi[s1]] = Dv[u][r];
                            }
                        }
                    }
                });
            });
        }
        phase_sync();
        PHASE_MARK(1);

        // ---- square-root-free factorization K = Lt D Lt^T (Lt unit lower, D = diag(d)), right-looking,
        //      with the forward substitutions of y and X fused in.  The Cholesky factor of the reference
        //      is B = Lt D^(1/2); working with Lt and d keeps sqrt AND the diagonal scalings out of every
        //      dependent chain.  The chain of a step is   update of column j+1 -> store column j+1 ->
        //      broadcast read of its head (d_{j+1}, Kt(j+2, j+1)) -> 1/d_{j+1} -> multipliers;
        //      with LOOK-AHEAD: step j first updates column j+1 only, publishes it and starts the
        //      reciprocal of the next pivot, and only then applies column j to the rest of the trailing
        //      matrix, so the bulk of the rank-1 update fills the latency of the chain. ----
        // head of column j: pivot d_j and the next one or two entries.  Pairs (c0, c0+1) of a column are
        // read as one 128-bit broadcast load; cs(j) = first index of column j that starts an aligned pair.
        double Lo[S], xr[1 + P], hd, h1, h2 = 0.0;
        auto publish = [&](const int j) { // store column j, fetch (Lt^-1 rhs)_j (final once step j-1 is applied)
            const int sj = j / G, oj = (sj & 1) ? (G - 1 - j % G) : (j % G);
#pragma unroll
            for (int s = 0; s < S; ++s)
                if ((s + 1) * G - 1 >= j && rowi[s] >= j)
                    KLs[Geo::colbase(j) + rowi[s]] = Kr[s][j];
#pragma unroll
            for (int r = 0; r < 1 + P; ++r)
                if (!TILED_RHS_LATE)
                    xr[r] = __shfl_sync(FULLMASK, rhs[r][sj], oj, G);
            __syncwarp();
            const double *col = KLs + Geo::colbase(j);
            const int cs = ((Geo::colbase(j) + j) & 1) ? j + 1 : j;
#ifdef TILED_HEAD_SHFL
            // experiment: the head of column j straight from the owners' registers (shorter pivot chain,
            // 2-3 double shuffles instead of one or two broadcast loads)
            (void)col;
            hd = __shfl_sync(FULLMASK, Kr[sj][j], oj, G);
            {
                const int j1 = j + 1, s1 = j1 / G, o1 = (s1 & 1) ? (G - 1 - j1 % G) : (j1 % G);
                h1 = __shfl_sync(FULLMASK, Kr[s1][j], o1, G);
            }
            if (cs != j && j + 2 < CAP) {
                const int j2 = j + 2, s2 = j2 / G, o2 = (s2 & 1) ? (G - 1 - j2 % G) : (j2 % G);
                h2 = __shfl_sync(FULLMASK, Kr[s2][j], o2, G);
            }
#else
            if (cs == j) {
                const double2 v = *reinterpret_cast<const double2 *>(col + j);
                hd = v.x;
                h1 = v.y;
            } else {
                hd = col[j];
                const double2 v = *reinterpret_cast<const double2 *>(col + j + 1);
                h1 = v.x;
                h2 = v.y;
            }
#endif
        };
        auto multipliers = [&](const int j) { // Lo[s] = Lt[row][j] below the pivot row, exactly 0 for finished rows
#if (TILED_ABLATE & 128)
            const double rj = 2.0 - hd; // timing experiment: no reciprocal on the pivot chain (wrong numbers)
#else
            const double rj = rcp_pos3(hd);
#endif
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if ((s + 1) * G - 1 > j) {
                    Lo[s] = (rowi[s] > j) ? Kr[s][j] * rj : 0.0;
                    Kr[s][j] = Lo[s]; // the masked multiplier is what the forward sweeps below need
                } else {
                    Lo[s] = 0.0;
                }
            }
        };
        if (!(TILED_ABLATE & 2)) {
        publish(NP); // local rows 0 .. NP-1 are always padding: their steps are the identity
        multipliers(NP);
        }
        if (!(TILED_ABLATE & 2))
        static_for<NP, CAP - 1>([&](auto jc) {
            constexpr int j = decltype(jc)::value;
            constexpr int cs = ((Geo::colbase(j) + j) & 1) ? j + 1 : j;
            const double *col = KLs + Geo::colbase(j);
            // column j is applied with the multipliers of THIS step; the look-ahead below overwrites
            // Lo / xr / h1 / h2 with those of step j+1, so keep copies (SSA renames, no moves)
            double Lc[S];
#pragma unroll
            for (int s = 0; s < S; ++s)
                Lc[s] = Lo[s];
            const double g2 = h2;
            // the pair loads of the rest of column j run PD loads ahead of the FMAs that consume them
            // (left to itself the compiler issues each load right before its first use and the warp eats
            // the full shared-memory latency once per load: measured, profiles/)
            constexpr int cb0 = (cs == j) ? j + 2 : j + 3;
            constexpr int NPAIR = (CAP - cb0 + 1) / 2;
            constexpr int PD = TILED_PD;
            double2 ring[PD];
            const bool work = (j >= NSKIP) || (j >= pad_w); // compile-time true beyond the first NSKIP steps
            if (work) {
#pragma unroll
                for (int i = 0; i < PD; ++i)
                    if (i < NPAIR)
                        ring[i] = *reinterpret_cast<const double2 *>(col + cb0 + 2 * i);
#pragma unroll
                for (int r = 0; r < 1 + P; ++r)
#pragma unroll
                    for (int s = 0; s < S; ++s)
                        if (!TILED_RHS_LATE && (s + 1) * G - 1 > j)
                            rhs[r][s] = fma(-Lc[s], xr[r], rhs[r][s]);
#pragma unroll
                for (int s = 0; s < S; ++s)
                    if ((s + 1) * G - 1 >= j + 1)
                        Kr[s][j + 1] = fma(-Lc[s], h1, Kr[s][j + 1]);
            }
            if constexpr (j + 1 < CAP - 1)
                publish(j + 1);
            // the rest of the trailing update with column j
            if (work) {
                if constexpr (cs != j && j + 2 < CAP) {
#pragma unroll
                    for (int s = 0; s < S; ++s)
                        if ((s + 1) * G - 1 >= j + 2)
                            Kr[s][j + 2] = fma(-Lc[s], g2, Kr[s][j + 2]);
                }
#pragma unroll
                for (int i = 0; i < NPAIR; ++i) {
                    const int c0 = cb0 + 2 * i;
                    const double2 v = ring[i % PD];
                    if (i + PD < NPAIR)
                        ring[i % PD] = *reinterpret_cast<const double2 *>(col + c0 + 2 * PD);
#pragma unroll
                    for (int s = 0; s < S; ++s) {
                        if ((s + 1) * G - 1 >= c0)
                            Kr[s][c0] = fma(-Lc[s], v.x, Kr[s][c0]);
                        if (c0 + 1 < CAP && (s + 1) * G - 1 >= c0 + 1)
                            Kr[s][c0 + 1] = fma(-Lc[s], v.y, Kr[s][c0 + 1]);
                    }
                }
            }
            if constexpr (j + 1 < CAP - 1)
                multipliers(j + 1);
#if defined(TILED_CLOCKS) && TILED_CLOCKS > 1
            {
                const long long _t = clock64();
                stc[j] += _t - pht;
                phc[2] += _t - pht;
                pht = _t;
            }
#endif
        });
        // last pivot d_e (row CAP-1 = the observation itself): nothing left to update
        constexpr int se = S - 1;
        constexpr int oe = Geo::lane_of(CAP - 1);
        const double d_e = __shfl_sync(FULLMASK, Kr[se][CAP - 1], oe, G);
        const double rho_e = rcp_pos(d_e);
        // 1/d_a of the own rows and the failure test, from the diagonal of the column store (the very
        // values the pivot chain used, so the reciprocals are bit-identical to the chain's): keeps the
        // per-step selects (owner-lane invd, running failure index) out of the factorization sweep.
        __syncwarp();
        double invd[S];
        int failpiv = 0;
        {
            unsigned badm[S];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const int a = rowi[s];
                const double da = (a == CAP - 1) ? d_e : KLs[colb_r[s] + rowm[s]];
                const bool real = a >= NP;                      // static padding rows: identity (the store holds 0)
                invd[s] = !real ? 1.0 : ((a == CAP - 1) ? rho_e : rcp_pos3(da));
                badm[s] = __ballot_sync(FULLMASK, real && da <= E.piv_floor);
                if (G < 32)
                    badm[s] = (badm[s] >> (g * G)) & ((1u << (G & 31)) - 1u);
            }
            // lowest failing local row + 1 (slot s even: lane = row - sG, odd: lane = G-1 - (row - sG))
#pragma unroll
            for (int s = S - 1; s >= 0; --s)
                if (badm[s] != 0u)
                    failpiv = s * G + ((s & 1) ? (G - 1 - (31 - __clz(badm[s]))) : (__ffs(badm[s]) - 1)) + 1;
        }

        // ---- ut = Lt^-T e_last (u = ut / sqrt(d_e)): the lane owning index j accumulates
        //      sb_j = sum_{l>j} K(l,j) ut_l from the unscaled column store, ut_j = e_j - sb_j / d_j.  As
        //      soon as ut_l is known (and broadcast) it is also applied to the packed derivative
        //      matrices, tt_r += D_r[., l] ut_l, so D_r u needs no separate mat-vec pass.  Element
        //      (a, l) of the symmetric D_r lives at colbase(a) + l (a < l) or colbase(l) + a (a >= l;
        //      the diagonal holds zeros). ----
        phase_sync();
        PHASE_MARK(2);
#if TILED_PREFETCH == 1 || TILED_PREFETCH == 2
        load_idx(batch + stride, nidx); // next batch of this warp (see the gather pipeline above)
#endif
        double sb[S], eb[S], rr[QD + 1][S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            sb[s] = 0.0;
            eb[s] = (rowi[s] == CAP - 1) ? 1.0 : 0.0;
        }
        // The dependent chain of a step is one FMA + one shuffle; the column-store loads do not depend on
        // ut and run TILED_BD steps ahead (few live registers here: the mat-vec D_r u is a separate pass
        // below -- fused into this loop its loads were serialised behind the chain for lack of registers,
        // 115 cycles per step measured, profiles/r2_experiments.md).  NO masks: a lane whose row a is not
        // above l (a >= l) reads a finite, unrelated element of the store (colbase(a) + l stays inside it)
        // and pollutes sb only at and after its own step l = a, when sb has already been consumed; every lane
        // receives every ut_l, lane 0 of the group writes it to shared memory and every lane
        // reads its own entries back afterwards.
        double *us = pts; // CAP doubles: ut (the coordinate table is dead by now)
        {
            constexpr int BD = TILED_BD;
            double Kq[BD][S];
#if TILED_FUSE_DU
            // the mat-vec D_r ut rides in the stalls of the chain (its loads BD steps ahead as well)
            double Dq[BD][QD][S];
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int r = 0; r < QD; ++r)
                    rr[r][s] = 0.0;
#endif
            auto fetchK = [&](const int l, double (&Kl)[S]) {
#pragma unroll
                for (int s = 0; s < S; ++s)
                    if (s * G < l) // slot has rows < l
                        Kl[s] = KLs[colb_r[s] + l];
            };
            if (lg < NP)
                us[lg] = 0.0;
            if (!(TILED_ABLATE & 4)) {
                static_for<0, BD>([&](auto ic) {
                    constexpr int l = CAP - 1 - decltype(ic)::value;
                    if constexpr (l >= NP) {
                        fetchK(l, Kq[decltype(ic)::value % BD]);
#if TILED_FUSE_DU
                        sym_fetch_col<G, S, NP, QD, l>(Dms, DSZ, colb_r, rowm, oz, Dq[decltype(ic)::value % BD]);
#endif
                    }
                });
                static_for<0, CAP - NP>([&](auto ic) {
                    constexpr int it = decltype(ic)::value, l = CAP - 1 - it;
                    constexpr int sl = l / G, ol = (sl & 1) ? (G - 1 - l % G) : (l % G);
                    const double ul = __shfl_sync(FULLMASK, fma(-sb[sl], invd[sl], eb[sl]), ol, G);
                    if (lg == 0) // every lane of the group holds the same ul; one of them stores it
                        us[l] = ul;
#pragma unroll
                    for (int s = 0; s < S; ++s)
                        if (s * G < l)
                            sb[s] = fma(Kq[it % BD][s], ul, sb[s]);
#if TILED_FUSE_DU
#pragma unroll
                    for (int s = 0; s < S; ++s)
#pragma unroll
                        for (int r = 0; r < QD; ++r)
                            rr[r][s] = fma(Dq[it % BD][r][s], ul, rr[r][s]);
#endif
                    if constexpr (l - BD >= NP) {
                        fetchK(l - BD, Kq[it % BD]);
#if TILED_FUSE_DU
                        sym_fetch_col<G, S, NP, QD, l - BD>(Dms, DSZ, colb_r, rowm, oz, Dq[it % BD]);
#endif
                    }
                });
            }
            __syncwarp();
        }
#pragma unroll
        for (int s = 0; s < S; ++s) // padding rows: ut = 0 whatever was read
            rr[QD][s] = (rowi[s] < pad) ? 0.0 : us[rowi[s]];
        // ---- tt_r = D_r ut: ut goes through shared memory (the coordinate table is dead by now), every lane
        //      reads it back as broadcast pairs and walks its own rows of the packed symmetric D_r:
        //      element (a, l) at colbase(a) + l (a < l) or colbase(l) + a (a >= l; diagonal and column 0 hold
        //      zeros).  No dependent chain: two accumulators per row and matrix. ----
#if TILED_FUSE_DU
#pragma unroll
        for (int s = 0; s < S; ++s)
#pragma unroll
            for (int r = 0; r < QD; ++r)
                rr[r][s] *= dscale[r];
#else
        {
            double t0[QD][S], t1[QD][S];
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int r = 0; r < QD; ++r)
                    t0[r][s] = t1[r][s] = 0.0;
            // software pipeline: the loads of step h + DD are issued before the FMAs of step h (left to itself
            // the compiler, short of registers here, issues each load right before its use: 30 cycles each)
            constexpr int DD = TILED_DD, NH = CAP / 2;
            double dq[DD][2][QD][S];
            double2 uq[DD];
            static_for<0, DD>([&](auto hc) {
                constexpr int h = decltype(hc)::value;
                if constexpr (h < NH)
                    sym_fetch_pair<G, S, NP, QD, h>(Dms, DSZ, us, colb_r, rowm, oz, dq[h % DD], uq[h % DD]);
            });
            static_for<0, NH>([&](auto hc) {
                constexpr int h = decltype(hc)::value;
                double dv[2][QD][S];
#pragma unroll
                for (int s = 0; s < S; ++s)
#pragma unroll
                    for (int r = 0; r < QD; ++r) {
                        dv[0][r][s] = dq[h % DD][0][r][s];
                        dv[1][r][s] = dq[h % DD][1][r][s];
                    }
                const double2 uv = uq[h % DD];
                if constexpr (h + DD < NH)
                    sym_fetch_pair<G, S, NP, QD, h + DD>(Dms, DSZ, us, colb_r, rowm, oz, dq[h % DD], uq[h % DD]);
#pragma unroll
                for (int s = 0; s < S; ++s)
#pragma unroll
                    for (int r = 0; r < QD; ++r) {
                        t0[r][s] = fma(dv[0][r][s], uv.x, t0[r][s]);
                        t1[r][s] = fma(dv[1][r][s], uv.y, t1[r][s]);
                    }
            });
#pragma unroll
            for (int s = 0; s < S; ++s)
#pragma unroll
                for (int r = 0; r < QD; ++r)
                    rr[r][s] = (t0[r][s] + t1[r][s]) * dscale[r];
        }
#endif

        phase_sync();
        PHASE_MARK(3);
        // ---- [tt_1..tt_QD, ut] through Lt^-1 (unit-diagonal forward sweeps on the register-resident rows) ----
#pragma unroll
        for (int j = NP; j < ((TILED_ABLATE & 8) ? NP : CAP - 1); ++j) {
            const int sj = j / G;
            const int oj = (sj & 1) ? (G - 1 - j % G) : (j % G);
            double Lm[S]; // multipliers of column j, stored masked (exactly 0 for rows <= j) by the factorization
#pragma unroll
            for (int s = 0; s < S; ++s)
                Lm[s] = ((s + 1) * G - 1 > j) ? Kr[s][j] : 0.0;
#pragma unroll
            for (int r = 0; r < QD + 1; ++r) {
                const double x = __shfl_sync(FULLMASK, rr[r][sj], oj, G);
#pragma unroll
                for (int s = 0; s < S; ++s)
                    if ((s + 1) * G - 1 > j)
                        rr[r][s] = fma(-Lm[s], x, rr[r][s]);
            }
#if TILED_RHS_LATE
#pragma unroll
            for (int r = 0; r < 1 + P; ++r) {
                const double x = __shfl_sync(FULLMASK, rhs[r][sj], oj, G);
#pragma unroll
                for (int s = 0; s < S; ++s)
                    if ((s + 1) * G - 1 > j)
                        rhs[r][s] = fma(-Lm[s], x, rhs[r][s]);
            }
#endif
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
        phase_sync();
        PHASE_MARK(4);
#if TILED_PREFETCH == 1
        load_rec(nidx, nrec);
#elif TILED_PREFETCH == 3
        // the whole gather of the NEXT batch inside the contraction of this one (the rows of K are dead here, so
        // the 20 registers are free): indices now, records at the end of the loop body
        load_idx(batch + stride, nidx);
#elif TILED_PREFETCH == 2
#pragma unroll
        for (int s = 0; s < S; ++s)
            if (nidx[s] >= 0)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(E.rec + nidx[s] * E.rs));
#elif TILED_PREFETCH == 5 || TILED_PREFETCH == 0
        // the next batch's indices come from L2 by now (requested at the top of this batch); its records are
        // requested into L1 and the indices dropped again (nothing is held across the batch boundary).  Product
        // build: instances with design columns only (their records span two sectors), behind E.prefetch
        if (TILED_PREFETCH == 5 || (P > 1 && E.prefetch)) {
            int64_t pidx[S];
            load_idx(batch + stride, pidx);
#pragma unroll
            for (int s = 0; s < S; ++s)
                if (pidx[s] >= 0)
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(E.rec + pidx[s] * E.rs));
        }
#endif
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
#if (TILED_ABLATE & 64)
        { // timing experiment: +320 independent one-register-operand DFMAs per batch
            double dz[8];
#pragma unroll
            for (int t = 0; t < 8; ++t)
                dz[t] = ze + t;
#pragma unroll
            for (int it = 0; it < 40; ++it)
#pragma unroll
                for (int t = 0; t < 8; ++t)
                    dz[t] = fma(dz[t], 1.0000001, 1e-9);
            double dsum = 0.0;
#pragma unroll
            for (int t = 0; t < 8; ++t)
                dsum += dz[t];
            if (dsum == 1.2345)
                acc[0] += dsum;
        }
#endif
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
#if TILED_PREFETCH == 3
        load_rec(nidx, nrec);
#endif
        phase_sync();
        PHASE_MARK(5);
    }
#ifdef TILED_CLOCKS
    if (E.dbg_clocks != nullptr && lane == 0) {
#pragma unroll
        for (int t = 0; t < 8; ++t)
            atomicAdd(E.dbg_clocks + t, (unsigned long long)phc[t]);
#if TILED_CLOCKS > 1
#pragma unroll
        for (int t = 0; t < CAP; ++t)
            atomicAdd(E.dbg_clocks + 16 + t, (unsigned long long)stc[t]);
#endif
    }
#endif

    // ---- block partial: add the groups of this warp in fixed order, one row of `partials` per block ----
#pragma unroll
    for (int t = 0; t < NACC; ++t) {
        double v = acc[t];
#pragma unroll
        for (int off = G; off < 32; off <<= 1)
            v += __shfl_xor_sync(FULLMASK, v, off);
        const int o = t * G + lg;
        if (g == 0 && o < L)
            E.partials[((size_t)blockIdx.x * TILED_WPB + warp) * L + o] = v;
    }
    vb_finish(E, TILED_WPB);
}

// ---------------------------------------------------------------------------
// host side: instance table and launch
// ---------------------------------------------------------------------------
struct TiledInstance {
    int g, s, cap, family, d, p, wpb;
    int npad; // leading local rows that are padding for every observation served: m+1 <= cap - npad
    int pair_table; // 1: the pair-table pair phase (PT = true) -- needs EvalParams::pair_tab
    void (*kernel)(const EvalParams);
    int smem_doubles;
    const char *name;
};

#define TILED_INST(G_, S_, FAM_, D_, P_)                                                                        \
    {                                                                                                           \
        G_, S_, (G_) * (S_), FAM_, D_, P_, TILED_WPB, 1, 0, vecchia_tiled_kernel<G_, S_, FAM_, D_, P_>,                               \
            LikSmem<G_, S_, D_, FamTraits<FAM_, D_>::QD>::TOTAL,                                                 \
            "vecchia_tiled_kernel<G=" #G_ ",S=" #S_ "," #FAM_ ",D=" #D_ ",P=" #P_ ">"                            \
    }

#define TILED_INST_PT(G_, S_, FAM_, D_, P_)                                                                     \
    {                                                                                                           \
        G_, S_, (G_) * (S_), FAM_, D_, P_, 1, 1, 1, vecchia_tiled_kernel<G_, S_, FAM_, D_, P_, true>,           \
            LikSmem<G_, S_, D_, FamTraits<FAM_, D_>::QD>::TOTAL,                                                \
            "vecchia_tiled_kernel<G=" #G_ ",S=" #S_ "," #FAM_ ",D=" #D_ ",P=" #P_ ",pair-table>"               \
    }

// pair-table variant with NP_ static padding rows: serves m+1 <= G_*S_ - NP_ with the shared memory of a
// (G_*S_ - NP_ + 1)-row tier
#define TILED_INST_PTN(G_, S_, FAM_, D_, P_, NP_)                                                               \
    {                                                                                                           \
        G_, S_, (G_) * (S_), FAM_, D_, P_, 1, NP_, 1, vecchia_tiled_kernel<G_, S_, FAM_, D_, P_, true, NP_>,    \
            LikSmem<G_, S_, D_, FamTraits<FAM_, D_>::QD, NP_>::TOTAL,                                           \
            "vecchia_tiled_kernel<G=" #G_ ",S=" #S_ "," #FAM_ ",D=" #D_ ",P=" #P_ ",pair-table,NP=" #NP_ ">"    \
    }
