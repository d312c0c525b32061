// tiled_common.cuh -- definitions shared by the TILED_REG kernels (likelihood: kernel_tiled.cuh,
// kernel_tiled_pt.cuh; kriging: kernel_krige.cuh): family traits, the pair-parallel pair terms, the
// lane-group geometry (G lanes x S rows per lane, boustrophedon folding), the packed column store.
#pragma once
#include "common.cuh"

#define FULLMASK 0xffffffffu
#ifndef TILED_NI
#define TILED_NI 2 // independent pairs in flight per lane in the pair loop (3 and 4 measured no faster)
#endif

template <int FAM, int D>
struct FamTraits {
    static constexpr int QD = (FAM == FAM_EXP_ANISO) ? D : ((FAM == FAM_EXP_SPACETIME || FAM == FAM_MATERN) ? 2 : 1);
    static constexpr int Q = QD + 2;
};

// Pair terms with a compile-time coordinate count.  dl[] are coordinate differences ALREADY
// divided by the range of their axis (the gather scales the coordinates once per point), so the
// squared norm is x^2 = (r/rho)^2 directly.  Squared norms start from 1e-300 instead of 0:
// coincident points then give x ~ 1e-150, i.e. exactly the reference's values (exp(-0) = 1, zero
// range derivative) without a special case.
template <int FAM, int D, bool DERIV = true>
__device__ __forceinline__ void pair_terms_s(const EvalParams &E, const double *etab, const double (&dl)[D],
                                             double &Kv, double (&Dv)[FamTraits<FAM, D>::QD])
{
    if constexpr (FAM == FAM_MATERN) {
        double x2 = 1e-300;
#pragma unroll
        for (int l = 0; l < D; ++l)
            x2 = fma(dl[l], dl[l], x2);
        if constexpr (DERIV) {
            matern_terms(E, x2 * rsqrt_pos(x2), E.inv_rho[0], Kv, Dv[0], Dv[1]);
        } else { // covariance only (kriging): one Bessel evaluation instead of three
            const double x = x2 * rsqrt_pos(x2);
            double k, km1;
            Kv = E.sig2;
            const int nterms = matern_series_terms(x);
            if (x >= 1e-60) {
                const double lx = log(x);
                const double dd = 0.6931471805599453 - lx;
                bessel_k_pair(x, dd, rcp_pos(x), E.mat[0], exp(E.mat[0].mu * dd), nterms, k, km1);
                Kv = E.sig2 * E.mat[0].nc2 * k; // k = (x/2)^nu K_nu(x)
            }
            Dv[0] = Dv[1] = 0.0;
        }
    } else if constexpr (FAM == FAM_EXP_ISO || FAM == FAM_MATERN15 || FAM == FAM_MATERN25) {
        double x2 = 1e-300;
#pragma unroll
        for (int l = 0; l < D; ++l)
            x2 = fma(dl[l], dl[l], x2);
        const double x = x2 * rsqrt_pos(x2);
        const double se = E.sig2 * exp_neg(x, etab);
        const double xi = x * E.inv_rho[0];
        if constexpr (FAM == FAM_EXP_ISO) {
            Kv = se;
            Dv[0] = se * xi;
        } else if constexpr (FAM == FAM_MATERN15) {
            Kv = fma(se, x, se);
            Dv[0] = (se * x) * xi;
        } else {
            const double x1 = 1.0 + x;
            Kv = se * fma(x * x, 1.0 / 3.0, x1);
            Dv[0] = (se * x) * (xi * x1) * (1.0 / 3.0);
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
        Kv = E.sig2 * exp_neg(s2 * rs, etab);
        const double g = Kv * rs;
        if constexpr (FAM == FAM_EXP_ANISO) {
#pragma unroll
            for (int l = 0; l < D; ++l)
                Dv[l] = g * sc[l] * E.inv_rho[l];
        } else {
            Dv[0] = g * sp2 * E.inv_rho[0];
            Dv[1] = g * sc[D - 1] * E.inv_rho[D - 1];
        }
    }
}

// NP = number of leading local rows that are padding rows for EVERY observation the tier serves (m+1 <= CAP-NP).
// Rows 0 .. NP-2 never touch shared memory; row Z = NP-1 is the one padding row the packing keeps (its column and
// diagonal entries hold zeros), so a tier with NP > 1 packs a (CAP-Z) x (CAP-Z) triangle: less shared memory per
// observation, i.e. more resident warps, and the factorization / sweeps start at column NP.
template <int G, int S, int NP = 1>
struct TileGeom {
    static constexpr int CAP = G * S;
    static constexpr int Z = NP - 1;                   // first local row present in the packed triangles
    static constexpr int CAPE = CAP - Z;               // rows of the packed triangles
    static constexpr int OPW = 32 / G;                 // observations per warp
    static constexpr int TRI = CAPE * (CAPE + 1) / 2;  // packed lower triangle incl. diagonal
    // column store: element (c, j), c >= j >= Z, of the (unscaled) factor lives at colbase(j) + c, columns
    // packed back to back.  colbase(j) = -j(j+1)/2 (mod 16) when CAP = 32, NP = 1, so the 16 lanes of a group
    // reading "their" columns at a common row hit 16 different 8-byte banks.
    __host__ __device__ static constexpr int colbase(int j) { return (j - Z) * (CAPE - 1) - (j - Z) * (j - Z - 1) / 2 - Z; }
    static constexpr int KL = (TRI + 3) & ~1; // one element past the last column may be read by a pair load
    __host__ __device__ static constexpr int slot_of(int r) { return r / G; }
    __host__ __device__ static constexpr int lane_of(int r) { return ((r / G) & 1) ? (G - 1 - r % G) : (r % G); }
};

template <int G, int S, int D, int QD, int NP = 1>
struct TileSmem {
    using Geo = TileGeom<G, S, NP>;
    static constexpr int DP = (D + 1) & ~1;                 // padded coordinate stride (16-byte rows)
    static constexpr int PTS = Geo::CAP * DP;               // scaled coordinates of the local frame
    // K staging, the column store of the factorization and every D_j share ONE packing: element
    // (a, c), a >= c, at colbase(c) + a (columns back to back).  The pair table walks the columns
    // from the last one down, rows ascending, so the staging stores of a lane group are contiguous;
    // the row loads (static c, lane-varying a) are contiguous as well.
    static constexpr int DSZ = (Geo::TRI + 1) & ~1;
    static constexpr int PER_OBS = PTS + Geo::KL + QD * DSZ;
    static constexpr int TOTAL = VB_EXPTAB + Geo::OPW * PER_OBS;
    // Local rows 0 .. NP-1 are ALWAYS padding rows (tiers serve m+1 <= CAP-NP), so nothing is computed for them.
    // off-diagonal pair table (device memory, shared by all blocks): TOFF entries padded to a
    // multiple of NI*G with copies of the last pair; entry = a << 24 | c << 16 | (colbase(c) + a)
    static constexpr int TOFF = (Geo::CAP - NP) * (Geo::CAP - NP - 1) / 2; // pairs among local rows NP..CAP-1
    static constexpr int NI = TILED_NI;                     // pairs in flight per lane in the pair loop
    static constexpr int TPAD = (TOFF + NI * G - 1) / (NI * G) * (NI * G);
};

// blocks per SM (one warp per block) the register budget of a tier is tuned for: the rows a lane
// keeps in registers take G*S(S+1) 32-bit registers; 168 registers = 3 warps per SM sub-partition
__host__ __device__ constexpr int tiled_min_blocks(int G, int S, int NP = 1)
{
#ifdef TILED_MINB
    return TILED_MINB; // development knob
#else
    // 32-bit registers of the row entries a lane keeps: slot s holds columns NP-1 .. (s+1)G-1 of its row
    int regs = 0;
    for (int s = 0; s < S; ++s)
        regs += 2 * (((s + 1) * G - (NP - 1)) > 0 ? ((s + 1) * G - (NP - 1)) : 0);
    return (regs <= 56) ? 16 : ((regs <= 96) ? 12 : 8);
#endif
}
