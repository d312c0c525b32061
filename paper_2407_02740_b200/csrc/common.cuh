// common.cuh -- shared device-side definitions of the B200 Vecchia core.
//
// Reference map (paths relative to /root/reference/pkg/src/vecchiagp):
//   PairTerms / pair_terms   <- engine/_kernels.pyx:34-99 (_cov_entry, _dcov_entry), evaluated ONCE per
//                               pair instead of once per (parameter, pair) as the reference does
//   accumulator layout       <- engine/__init__.py:141-152 (_alloc_slots order)
//   emit_value               <- engine/_kernels.pyx:294-344 (_contract)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define VB_MAXD 20            // coordinates per point
#define VB_MAXQ (VB_MAXD + 2) // covariance parameters
#define VB_MAXP 16            // design columns

enum : int { FAM_EXP_ISO = 0, FAM_EXP_ANISO = 1, FAM_EXP_SPACETIME = 2, FAM_MATERN15 = 3, FAM_MATERN25 = 4,
             FAM_MATERN = 5 };

#define VB_MATERN_TERMS 12 // series terms (x <= 2: (x/2)^(2i)/(i!)^2 < 1e-17 at i = 12)
#define VB_MATERN_CF 48    // tabulated continued-fraction iterations (beyond: plain divisions)

// Order-dependent constants of Temme's method for K_nu (they depend on the smoothness only, so the
// host computes them once per evaluation): nu = mu + nup with |mu| <= 1/2.
struct MaternOrder {
    double nu, mu;
    double gam1, gam2;   // Temme's Gamma_1(mu), Gamma_2(mu)
    double gampl, gammi; // 1/Gamma(1+mu), 1/Gamma(1-mu)
    double gp, gm;       // Gamma(1+mu), Gamma(1-mu) (the series starts from E Gamma(1+mu) / 2 and Gamma(1-mu) / (2 E))
    double fact;         // pi mu / sin(pi mu)
    double normcon;      // 2^(1-nu) / Gamma(nu)
    double nc2;          // 2 / Gamma(nu): correlation = nc2 (x/2)^nu K_nu(x)
    int nup, pad_;
    double inv_mu;       // 1/mu (0 when mu == 0; only used for |mu d| >= 1e-2)
    // reciprocals that depend on (iteration, mu) only -- the divisions of Temme's series and of
    // Steed's continued fraction become multiplications by kernel-parameter (constant-bank) values
    double r1[VB_MATERN_TERMS]; // 1 / (i^2 - mu^2), i = 1..
    double rp[VB_MATERN_TERMS]; // 1 / (i - mu)
    double rq[VB_MATERN_TERMS]; // 1 / (i + mu)
    double ra[VB_MATERN_CF];    // 1 / a_i of CF2, a_i = mu^2 - 1/4 - i(i-1), i = 2..
    // order derivatives of the constants above (central order only): the smoothness derivative of the series branch
    // is the ANALYTIC mu-derivative of Temme's series, carried along term by term (bessel_series_dnu)
    double dgam1, dgam2, dfact; // d/dmu of Gamma_1, Gamma_2, pi mu / sin(pi mu)
    double psi_p, psi_m;        // digamma(1 + mu), digamma(1 - mu): d log Gamma(1 +- mu) / d(+-mu)
    double dlognc2;             // d log(2 / Gamma(nu)) / dnu = -digamma(nu)
    double tm[VB_MATERN_TERMS]; // 2 mu / (i^2 - mu^2) = d log r1[i] / dmu
};
#define VB_MATERN_H 1e-5 // central-difference step of the smoothness derivative

// Everything one evaluation needs, passed by value as the kernel argument.
struct EvalParams {
    const double *rec;      // packed point records, rs doubles each: locs[d], y, X[p], (pad)
    const int64_t *nn;      // neighbor rows of this shard, (nn_rows, mp1), -1 padded
    int64_t nn_row0;        // global index of the first row held in nn
    int64_t i0, i1;         // observation range of this evaluation
    int p, d, q, mp1, rs, family;
    int qd;                 // number of range-like ("dense") parameters = q - 2
    int L;                  // accumulator length
    double sig2, tau2, jitter, diag; // diag = sig2*(1+tau2) + jitter
    double inv_sig2;
    double piv_floor;       // a pivot <= piv_floor fails the factorization (see vecchia_b200.cu fill_params)
    double inv_rho[VB_MAXD]; // per-axis inverse ranges (iso: all equal; space-time: space,..,space,time)
    double *partials;        // [gridDim.x][L] block partial sums
    unsigned long long *fail_word; // min over failures of (index << 16 | pivot+1)
    unsigned int *fail_count;
    double *rows;            // optional (i1-i0, L) per-observation output (diagnostics); nullptr normally
    int *fail_rows;          // optional (i1-i0) pivot+1 per observation
    int ws_doubles;          // per-warp scratch doubles (warp_smem layout)
    const unsigned int *pair_tab; // tiled layout: off-diagonal pair table of the tier (device memory)
    int sm_count;            // SMs of the device (tiled layout: start stagger of the resident blocks)
    int prefetch;            // tiled layout: 1 = the point records exceed L2, request the next batch's inputs ahead
    unsigned long long *dbg_clocks; // experiments only (-DTILED_CLOCKS): per-phase cycle sums; nullptr otherwise
    // in-kernel finish (vb_finish below): the evaluation is ONE launch
    double *out;             // result vector, L+2 doubles (totals, failure count, -(first failing index)-1)
    double *group_sums;      // [ceil(gridDim.x / VB_FINISH_GROUP)][L]
    unsigned int *tickets;   // [0]: groups done, [1 + g]: blocks of group g done; all zero between evaluations
    unsigned long long *fail_latch; // copy of *fail_word of the finished evaluation (what the host reads)
    MaternOrder mat[3];      // FAM_MATERN only: orders nu, nu + h, nu - h
};

// ---------------------------------------------------------------------------
// FP64 math helpers for the pair terms and the pivots.  Arguments are known to be
// positive and normal here, so the special-case slow paths of the CUDA math library
// (a divergent CALL whenever one lane sees 0 / denormal / inf) are not needed.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double rsqrt_seed(double a)
{
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a)); // MUFU.RSQ64H, ~2^-22 relative
    return y;
}

// 1/sqrt(a): seed + one third-order correction (relative error ~1e-16)
__device__ __forceinline__ double rsqrt_pos(double a)
{
    const double y = rsqrt_seed(a);
    const double e = fma(a, -(y * y), 1.0);
    const double t = fma(e, 0.375, 0.5);
    return fma(t, y * e, y);
}

// 1/a for positive normal a: MUFU.RCP64H seed + two Newton steps
__device__ __forceinline__ double rcp_pos(double a)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
    r = fma(fma(-a, r, 1.0), r, r);
    return fma(fma(-a, r, 1.0), r, r);
}

// 1/a for positive normal a: MUFU.RCP64H seed (~2^-22 relative) + ONE third-order step
// r (1 + e + e^2), e = 1 - a r: three dependent DFMA instead of four (it sits on the pivot chain)
__device__ __forceinline__ double rcp_pos3(double a)
{
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
    const double e = fma(-a, r, 1.0);
    return fma(r, fma(e, e, e), r);
}

// sqrt(a): a * rsqrt(a) with one Newton correction of the product (correctly rounded in practice)
__device__ __forceinline__ double sqrt_pos(double a)
{
    const double y = rsqrt_pos(a);
    const double g = a * y;
    const double d = fma(-g, g, a);
    return fma(d, 0.5 * y, g);
}

#ifndef VB_EXPTAB
#define VB_EXPTAB 32 // entries of 2^(j/VB_EXPTAB) in shared memory (32 or 64)
#endif

// exp(-x) for x >= 0: -x = k ln2/N + r, |r| <= ln2/2N (N = VB_EXPTAB); 2^(k/N) from an N-entry table and the
// exponent field, e^r from a polynomial.  N = 32, degree 5: truncation r^6/720 <= 2.2e-15 relative (round 2: was
// degree 6, 3.4e-18 -- the log-likelihood tolerance of 1e-9 needs ~1e-12 of a covariance entry).  N = 64, degree 4
// (3.8e-14, one FMA less) is kept as an option: its 256 bytes more per block cost the m = 30 tier its 12th block per
// SM (12 x (18.6 KB + 1 KB reserved) > 228 KB).  x is clamped at ~700 (result ~1e-304, never denormal).
__device__ __forceinline__ double exp_neg(double x, const double *tab)
{
    // clamp with one integer min on the high word (x >= 0, so the IEEE order is the integer
    // order; the low word of a clamped value is irrelevant)
    x = __hiloint2double(min(__double2hiint(x), 0x4085e000), __double2loint(x));
#if VB_EXPTAB == 64
    const double kf = fma(x, -92.33248261689366, 6755399441055744.0); // -64/ln2, 1.5*2^52
    const int ki = __double2loint(kf);
    const double kd = kf - 6755399441055744.0;
    double r = fma(kd, -0.010830424667801708, -x);   // ln2/64 split hi (low 24 bits clear) ...
    r = fma(kd, -2.8447437476627285e-11, r);         // ... + lo
    double q = fma(r, 1.0 / 24.0, 1.0 / 6.0);
    q = fma(q, r, 0.5);
    q = fma(q, r, 1.0);
    const double T = tab[ki & 63];
    const double v = fma(T, q * r, T);
    return __hiloint2double(__double2hiint(v) + ((ki >> 6) << 20), __double2loint(v));
#else
    const double kf = fma(x, -46.16624130844683, 6755399441055744.0); // -32/ln2, 1.5*2^52
    const int ki = __double2loint(kf);
    const double kd = kf - 6755399441055744.0;
    double r = fma(kd, -0.021660849335603416, -x);   // ln2/32 split hi (low 24 bits clear) ...
    r = fma(kd, -5.689487495325457e-11, r);          // ... + lo (a single-FMA reduction was measured: no faster)
#ifdef VB_EXP_DEG6
    double q = fma(r, 1.0 / 720.0, 1.0 / 120.0);
    q = fma(q, r, 1.0 / 24.0);
#else
    double q = fma(r, 1.0 / 120.0, 1.0 / 24.0);
#endif
    q = fma(q, r, 1.0 / 6.0);
    q = fma(q, r, 0.5);
    q = fma(q, r, 1.0);
    const double T = tab[ki & 31];
    const double v = fma(T, q * r, T);
    return __hiloint2double(__double2hiint(v) + ((ki >> 5) << 20), __double2loint(v));
#endif
}

// K_nu(x) and K_{nu-1}(x), x > 0, by Temme's method (N. M. Temme, J. Comput. Phys. 19 (1975) 324):
// the series in x for x <= 2, Steed's continued fraction CF2 for x > 2, both for the fractional
// order mu, then the upward recurrence K_{a+1} = K_{a-1} + (2a/x) K_a.  CUDA has no Bessel K of
// real order (the reason the paper's package has no general Matern).
// `d` = -log(x/2) and `inv_x` = 1/x are shared by the three orders evaluated per pair.
// inlined into its three call sites per pair (orders nu, nu + h, nu - h): the compiler interleaves the three
// recurrences (62 vs 67 ms per evaluation at config 2); the caller matern_terms_call stays out of line
#ifdef VB_BESSEL_NOINLINE
#define VB_BESSEL_ATTR __noinline__
#else
#define VB_BESSEL_ATTR __forceinline__
#endif
// `E` = exp(mu d) is supplied by the caller (the three orders of a pair differ by 1e-5, so two of the three
// exponentials are a short Taylor factor); `nterms` <= VB_MATERN_TERMS is the warp-uniform series length for this x.
// Outputs are SCALED so that nothing overflows for large orders at small x (K_nu(x) ~ Gamma(nu)/2 (2/x)^nu does):
//   tnu = (x/2)^nu K_nu(x)          (-> Gamma(nu)/2 as x -> 0: bounded by ~1e80 for nu <= 60)
//   bq  = (x/2)^(nu+1) K_(nu-1)(x)
// with the upward recurrence run on T_a = (x/2)^a K_a:  T_(a+1) = a T_a + (x/2)^2 T_(a-1).  The Matern correlation is
// then 2 tnu / Gamma(nu) and its range derivative 4 bq / Gamma(nu) / range -- no x^nu factor is ever formed.
static __device__ VB_BESSEL_ATTR void bessel_k_pair(double x, double d, double inv_x, const MaternOrder &M, const double E,
                                                  const int nterms, double &tnu, double &bq)
{
    const double mu = M.mu;
    double kmu, kmu1;
    const double xh = 0.5 * x, d2 = xh * xh;
    const double Ei = rcp_pos(E); // (x/2)^mu
    if (x <= 2.0) {
        const double e = mu * d;
        const double e2 = e * e;
        // sinh(e)/e: series for small e, (E - 1/E) / (2e) otherwise
        const double shoe = (fabs(e) < 1e-2) ? fma(e2, fma(e2, 1.0 / 120.0, 1.0 / 6.0), 1.0)
                                             : 0.5 * (E - Ei) * M.inv_mu * rcp_pos(d);
        double ff = M.fact * fma(M.gam1, 0.5 * (E + Ei), M.gam2 * shoe * d);
        double sum = ff;
        double p = 0.5 * E * M.gp, q = 0.5 * Ei * M.gm, c = 1.0, sum1 = p;
#pragma unroll
        for (int i = 1; i <= VB_MATERN_TERMS; ++i) { // unrolled (static constant-bank indices), left early (uniform)
            if (i > nterms)
                break;
            ff = fma((double)i, ff, p + q) * M.r1[i - 1];
            c *= d2 * (1.0 / i);
            p *= M.rp[i - 1];
            q *= M.rq[i - 1];
            sum = fma(c, ff, sum);
            sum1 = fma(c, fma(-(double)i, ff, p), sum1);
        }
        kmu = sum;
        kmu1 = sum1 * (2.0 * inv_x);
    } else {
        double b = 2.0 * (1.0 + x), dd = rcp_pos(b), h = dd, delh = dd, q1 = 0.0, q2 = 1.0;
        const double a1 = 0.25 - mu * mu;
        double q = a1, c = a1, a = -a1, s = fma(q, delh, 1.0);
        for (int i = 2; i < 400; ++i) {
            a -= 2 * (i - 1);
            const bool tab = (i - 2) < VB_MATERN_CF;
            const double inv_a = tab ? M.ra[tab ? i - 2 : 0] : 1.0 / a;
            c = -a * c / i;
            const double qnew = (q1 - b * q2) * inv_a;
            q1 = q2;
            q2 = qnew;
            q = fma(c, qnew, q);
            b += 2.0;
            dd = rcp_pos(fma(a, dd, b));
            delh = fma(b, dd, -1.0) * delh;
            h += delh;
            const double dels = q * delh;
            s += dels;
            if (fabs(dels) < fabs(s) * 1e-17)
                break;
        }
        kmu = sqrt(1.5707963267948966 * inv_x) * exp(-x) / s;
        kmu1 = kmu * (mu + x + 0.5 - a1 * h) * inv_x;
    }
    const double s1 = Ei * xh; // (x/2)^(mu+1)
    if (M.nup == 0) {
        tnu = Ei * kmu;
        bq = s1 * fma(-2.0 * mu * inv_x, kmu, kmu1); // (x/2)^(mu+1) K_(mu-1)
    } else {
        double prev = Ei * kmu, cur = s1 * kmu1;     // T_mu, T_(mu+1)
        for (int i = 1; i < M.nup; ++i) {
            const double next = fma(mu + i, cur, d2 * prev);
            prev = cur;
            cur = next;
        }
        tnu = cur;
        bq = d2 * prev;
    }
}

// Series branch (x <= 2) of the central order WITH its analytic order derivative: every quantity of Temme's series is
// differentiated with respect to mu alongside its value (11 more FP64 instructions per term, against 22 for the two
// shifted orders of a central difference, and no difference quotient: the result carries no 1e-16 / 2h rounding
// noise).  d/dnu = d/dmu at fixed nup.  Outputs as bessel_k_pair plus dtnu = d tnu / d nu.
static __device__ __forceinline__ void bessel_series_dnu(double x, double d, double inv_x, const MaternOrder &M, const double E,
                                                         const int nterms, double &tnu, double &bq, double &dtnu)
{
    const double mu = M.mu;
    const double xh = 0.5 * x, d2 = xh * xh;
    const double Ei = rcp_pos(E);        // (x/2)^mu = exp(-mu d)
    const double e = mu * d, e2 = e * e;
    const double ch = 0.5 * (E + Ei);    // cosh(e)
    const double sh = 0.5 * (E - Ei);    // sinh(e)
    // S = sinh(mu d) / mu and dS/dmu = (d cosh(e) - S) / mu; short series in e where the quotients cancel
    double S, dS;
    if (fabs(e) < 1e-2) {
        S = d * fma(e2, fma(e2, 1.0 / 120.0, 1.0 / 6.0), 1.0);
        dS = d * d * e * fma(e2, fma(e2, 1.0 / 840.0, 1.0 / 30.0), 1.0 / 3.0);
    } else {
        S = sh * M.inv_mu;
        dS = fma(d, ch, -S) * M.inv_mu;
    }
    const double g0 = fma(M.gam1, ch, M.gam2 * S);
    double ff = M.fact * g0;
    double dff = fma(M.dfact, g0, M.fact * (fma(M.dgam1, ch, M.gam1 * d * sh) + fma(M.dgam2, S, M.gam2 * dS)));
    double p = 0.5 * E * M.gp, q = 0.5 * Ei * M.gm;
    double dp = p * (d + M.psi_p), dq = -q * (d + M.psi_m);
    double sum = ff, dsum = dff, sum1 = p, dsum1 = dp, c = 1.0;
#pragma unroll
    for (int i = 1; i <= VB_MATERN_TERMS; ++i) {
        if (i > nterms)
            break;
        ff = fma((double)i, ff, p + q) * M.r1[i - 1];
        dff = fma(fma((double)i, dff, dp + dq), M.r1[i - 1], ff * M.tm[i - 1]);
        c *= d2 * (1.0 / i);
        p *= M.rp[i - 1];
        dp = fma(dp, M.rp[i - 1], p * M.rp[i - 1]);
        q *= M.rq[i - 1];
        dq = fma(dq, M.rq[i - 1], -(q * M.rq[i - 1]));
        sum = fma(c, ff, sum);
        dsum = fma(c, dff, dsum);
        sum1 = fma(c, fma(-(double)i, ff, p), sum1);
        dsum1 = fma(c, fma(-(double)i, dff, dp), dsum1);
    }
    const double kmu = sum, dkmu = dsum, tx = 2.0 * inv_x;
    const double kmu1 = sum1 * tx, dkmu1 = dsum1 * tx;
    const double s1 = Ei * xh; // (x/2)^(mu+1)
    // T_mu = Ei kmu, T_(mu+1) = s1 kmu1; d Ei / d mu = -d Ei
    if (M.nup == 0) {
        tnu = Ei * kmu;
        dtnu = Ei * fma(-d, kmu, dkmu);
        bq = s1 * fma(-2.0 * mu * inv_x, kmu, kmu1);
    } else {
        double prev = Ei * kmu, cur = s1 * kmu1;
        double dprev = Ei * fma(-d, kmu, dkmu), dcur = s1 * fma(-d, kmu1, dkmu1);
        for (int i = 1; i < M.nup; ++i) {
            const double next = fma(mu + i, cur, d2 * prev);
            const double dnext = fma(mu + i, dcur, fma(d2, dprev, cur));
            prev = cur;
            dprev = dcur;
            cur = next;
            dcur = dnext;
        }
        tnu = cur;
        dtnu = dcur;
        bq = d2 * prev;
    }
}

// Series length for this x (terms ~ (x/2)^(2i) / (i!)^2 against 1e-17), uniform over the lanes that are active
// here (the callers' pair loops end raggedly, so the vote runs on the active mask).
__device__ __forceinline__ int matern_series_terms(const double x)
{
    const unsigned am = __activemask();
    const bool valid = x <= 2.0;
#ifdef VB_MATERN_FULL_SERIES
    return __any_sync(am, valid && x > 1.0) ? VB_MATERN_TERMS
           : (__any_sync(am, valid && x > 0.4) ? 10 : (__any_sync(am, valid && x > 0.1) ? 7 : 5));
#else
    // first neglected term, (x/2)^(2i) / (i!)^2 at i = nterms + 1, below 1e-14 of the leading one (the covariance
    // needs ~1e-12): 10 / 7 / 5 / 4 terms (6e-16, 9e-15, 8e-15, 7e-18 at the upper end of each bracket); round 2a
    // ran 12 / 10 / 7 / 5 (1e-19 ... 1e-24)
    return __any_sync(am, valid && x > 1.0) ? 10
           : (__any_sync(am, valid && x > 0.4) ? 7 : (__any_sync(am, valid && x > 0.1) ? 5 : 4));
#endif
}

// General Matern pair terms at scaled distance x = r/range: correlation 2^(1-nu)/Gamma(nu) x^nu K_nu(x),
// its range derivative sigma^2 nc x^(nu+1) K_{nu-1}(x) / range, and the smoothness derivative: analytic (the order
// derivative of Temme's series, bessel_series_dnu) for x <= 2, a central difference of step VB_MATERN_H for x > 2
// (the continued-fraction branch; GpGp differentiates the smoothness numerically everywhere, and so do this
// repository's CPU restatements used by the tests -- the two agree to the O(h^2) ~ 1e-10 truncation of the difference quotient).
__device__ __forceinline__ void matern_terms(const EvalParams &P, double x, double inv_rho, double &Kv, double &Drange,
                                             double &Dnu)
{
    const int nterms = matern_series_terms(x); // before any lane leaves
    if (x < 1e-60) { // coincident points: the x -> 0 limits
        Kv = P.sig2;
        Drange = 0.0;
        Dnu = 0.0;
        return;
    }
    if (x > 705.0) { // x^nu K_nu(x) ~ e^-x underflows (also the far-away padding points of kernel_tiled.cuh,
        Kv = 0.0;    // for which the continued fraction below would overflow and never converge)
        Drange = 0.0;
        Dnu = 0.0;
        return;
    }
    const double lx = log(x);
    const double d = 0.6931471805599453 - lx, inv_x = rcp_pos(x); // -log(x/2), 1/x: shared by the three orders
    // exp(mu_t d) and x^nu_t for the three orders: the shifted orders differ from the central one by +-1e-5 in nu (and in
    // mu, unless the shift crosses a half-integer), so exp(delta d) is a degree-5 Taylor factor (|delta d| < 2e-3)
    auto small_exp = [](double z) {
        return fma(z, fma(z, fma(z, fma(z, fma(z, 1.0 / 120.0, 1.0 / 24.0), 1.0 / 6.0), 0.5), 1.0), 1.0);
    };
    const double E0 = exp(P.mat[0].mu * d);
#ifndef VB_MATERN_CENTRAL_DIFF
    if (x <= 2.0) { // one evaluation: value, range derivative and the analytic smoothness derivative
        double t0, b0, dt0;
        bessel_series_dnu(x, d, inv_x, P.mat[0], E0, nterms, t0, b0, dt0);
        const double sn = P.sig2 * P.mat[0].nc2;
        Kv = sn * t0;
        Drange = 2.0 * sn * b0 * inv_rho;
        Dnu = sn * fma(P.mat[0].dlognc2, t0, dt0);
        return;
    }
#endif
    const double dm1 = P.mat[1].mu - P.mat[0].mu, dm2 = P.mat[2].mu - P.mat[0].mu; // uniform
    const double E1 = (fabs(dm1) < 1e-3) ? E0 * small_exp(dm1 * d) : exp(P.mat[1].mu * d);
    const double E2 = (fabs(dm2) < 1e-3) ? E0 * small_exp(dm2 * d) : exp(P.mat[2].mu * d);
    double t0, b0, tp, tm, unused;
    bessel_k_pair(x, d, inv_x, P.mat[0], E0, nterms, t0, b0);
    bessel_k_pair(x, d, inv_x, P.mat[1], E1, nterms, tp, unused);
    bessel_k_pair(x, d, inv_x, P.mat[2], E2, nterms, tm, unused);
    // correlation 2^(1-nu)/Gamma(nu) x^nu K_nu = nc2 (x/2)^nu K_nu with nc2 = 2/Gamma(nu)
    Kv = P.sig2 * P.mat[0].nc2 * t0;
    Drange = P.sig2 * (2.0 * P.mat[0].nc2) * b0 * inv_rho; // sigma^2 nc x^(nu+1) K_(nu-1) / range
    Dnu = P.sig2 * fma(P.mat[1].nc2, tp, -(P.mat[2].nc2 * tm)) * (0.5 / VB_MATERN_H);
}

// Out-of-line entry for the fully unrolled row-owner pair phase of kernel_tiled.cuh (keeps ~60 copies of
// the series / continued-fraction code out of the instruction stream).
static __device__ __noinline__ void matern_terms_call(const EvalParams &P, double x, double &Kv, double &Drange,
                                                      double &Dnu)
{
    matern_terms(P, x, P.inv_rho[0], Kv, Drange, Dnu);
}

// Covariance and range-derivative values of one off-diagonal pair.
//   dl[l] = pa[l] - pc[l] is supplied by the caller (coordinates in the working frame).
// Families follow include/vecchia_b200.h.  Dv has qd entries.
template <int FAM>
__device__ __forceinline__ void pair_terms(const EvalParams &P, const double *dl, double &Kv, double *Dv)
{
    if (FAM == FAM_MATERN) {
        double d2 = 0.0;
        for (int l = 0; l < P.d; ++l)
            d2 = fma(dl[l], dl[l], d2);
        matern_terms(P, sqrt(d2) * P.inv_rho[0], P.inv_rho[0], Kv, Dv[0], Dv[1]);
    } else if (FAM == FAM_EXP_ISO || FAM == FAM_MATERN15 || FAM == FAM_MATERN25) {
        double d2 = 0.0;
        for (int l = 0; l < P.d; ++l)
            d2 = fma(dl[l], dl[l], d2);
        const double ir = P.inv_rho[0];
        const double x = sqrt(d2) * ir;
        const double e = exp(-x);
        if (FAM == FAM_EXP_ISO) {
            Kv = P.sig2 * e;             // sigma^2 exp(-r/rho)            (_kernels.pyx:44-46)
            Dv[0] = Kv * x * ir;         // sigma^2 exp(-r/rho) r / rho^2  (_kernels.pyx:70-76)
        } else if (FAM == FAM_MATERN15) {
            const double se = P.sig2 * e;
            Kv = se * (1.0 + x);
            Dv[0] = se * x * x * ir;
        } else {
            const double se = P.sig2 * e;
            Kv = se * (1.0 + x + x * x * (1.0 / 3.0));
            Dv[0] = se * x * x * (1.0 + x) * ir * (1.0 / 3.0);
        }
    } else {
        // anisotropic / space-time: s = || delta / rho ||              (_kernels.pyx:47-50, 78-99)
        double s2 = 0.0, sp2 = 0.0;
        double sc[VB_MAXD];
        for (int l = 0; l < P.d; ++l) {
            sc[l] = dl[l] * P.inv_rho[l];
            sc[l] *= sc[l];
            s2 += sc[l];
            if (l < P.d - 1)
                sp2 += sc[l];
        }
        const double s = sqrt(s2);
        Kv = P.sig2 * exp(-s);
        const double g = (s == 0.0) ? 0.0 : Kv / s;
        if (FAM == FAM_EXP_ANISO) {
            for (int l = 0; l < P.d; ++l)
                Dv[l] = g * sc[l] * P.inv_rho[l];
        } else {
            Dv[0] = g * sp2 * P.inv_rho[0];
            Dv[1] = g * sc[P.d - 1] * P.inv_rho[P.d - 1];
        }
    }
}

// Accumulator offsets for given (p, q).
struct AccLayout {
    int xsx, ysx, dlogdet, dysy, dysx, dxsx, ainfo, L;
    __host__ __device__ AccLayout(int p, int q)
    {
        xsx = 2;
        ysx = xsx + p * p;
        dlogdet = ysx + p;
        dysy = dlogdet + q;
        dysx = dysy + q;
        dxsx = dysx + p * q;
        ainfo = dxsx + p * p * q;
        L = ainfo + q * q;
    }
};

// Value of accumulator entry o for one observation, from the per-observation
// scalars (restates _contract, _kernels.pyx:294-344):
//   logdet, ze = z_e, we[b] = W_eb, ce[j] = c_je, zc[j] = z.c_j,
//   wc[b*q+j] = (W^T c_j)_b, cc[j*q+l] = c_j.c_l
__device__ __forceinline__ double emit_value(int o, int p, int q, const AccLayout &A, double logdet, double ze,
                                             const double *we, const double *ce, const double *zc,
                                             const double *wc, const double *cc)
{
    if (o == 0)
        return logdet;
    if (o == 1)
        return ze * ze;
    if (o < A.ysx) {
        const int t = o - A.xsx, a = t / p, b = t - a * p;
        return we[a] * we[b];
    }
    if (o < A.dlogdet)
        return ze * we[o - A.ysx];
    if (o < A.dysy)
        return ce[o - A.dlogdet];
    if (o < A.dysx) {
        const int j = o - A.dysy;
        return ce[j] * ze * ze - 2.0 * ze * zc[j];
    }
    if (o < A.dxsx) {
        const int t = o - A.dysx, b = t / q, j = t - b * q;
        return ce[j] * ze * we[b] - ze * wc[b * q + j] - zc[j] * we[b];
    }
    if (o < A.ainfo) {
        const int t = o - A.dxsx, ab = t / q, j = t - ab * q, a = ab / p, b = ab - a * p;
        return ce[j] * we[a] * we[b] - wc[a * q + j] * we[b] - we[a] * wc[b * q + j];
    }
    const int t = o - A.ainfo, j = t / q, l = t - j * q;
    return cc[j * q + l] - 0.5 * ce[j] * ce[l];
}

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// ---------------------------------------------------------------------------
// In-kernel finish: the last block to arrive adds the partial rows in a FIXED order, so the totals do not
// depend on scheduling (run-to-run bit-reproducible) and one evaluation is one launch (the reference
// sums n-leading slot arrays on the host: engine/__init__.py:155-170).
//   level 1: blocks are grouped VB_FINISH_GROUP at a time; the last block of a group to take its ticket adds the
//            group's rows (index order, four interleaved accumulators) into group_sums[g];
//   level 2: the last group to finish adds the group sums (index order) into out[0..L), publishes the
//            failure word of this evaluation and resets tickets / failure word for the next one.
// Every block calls this with ALL its threads after writing its `rpb` rows
// partials[(blockIdx.x * rpb + k) * L + o].
// ---------------------------------------------------------------------------
#define VB_FINISH_GROUP 32
#define VB_FINISH_MAXGROUPS 4096

__device__ __forceinline__ double vb_fixed_sum(const double *base, const int rows, const size_t stride)
{
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
    int r = 0;
    for (; r + 4 <= rows; r += 4) {
        s0 += __ldcg(base + (size_t)r * stride);
        s1 += __ldcg(base + (size_t)(r + 1) * stride);
        s2 += __ldcg(base + (size_t)(r + 2) * stride);
        s3 += __ldcg(base + (size_t)(r + 3) * stride);
    }
    for (; r < rows; ++r)
        s0 += __ldcg(base + (size_t)r * stride);
    return (s0 + s1) + (s2 + s3);
}

struct FinishArgs { // the few fields of EvalParams vb_finish needs (by value: the callee is out of line)
    const double *partials;
    double *group_sums, *out;
    unsigned int *tickets, *fail_count;
    unsigned long long *fail_word, *fail_latch;
    int L;
};

static __device__ __noinline__ void vb_finish_impl(const FinishArgs E, const int rpb)
{
    __shared__ unsigned int s_ticket;
    const unsigned nb = gridDim.x, ng = (nb + VB_FINISH_GROUP - 1) / VB_FINISH_GROUP, grp = blockIdx.x / VB_FINISH_GROUP;
    const unsigned gsize = min((unsigned)VB_FINISH_GROUP, nb - grp * VB_FINISH_GROUP);
    const int L = E.L;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0)
        s_ticket = atomicAdd(E.tickets + 1 + grp, 1u);
    __syncthreads();
    if (s_ticket != gsize - 1)
        return;
    __threadfence();
    for (int o = threadIdx.x; o < L; o += blockDim.x)
        E.group_sums[(size_t)grp * L + o] =
            vb_fixed_sum(E.partials + (size_t)grp * VB_FINISH_GROUP * rpb * L + o, (int)gsize * rpb, (size_t)L);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0)
        s_ticket = atomicAdd(E.tickets, 1u);
    __syncthreads();
    if (s_ticket != ng - 1)
        return;
    __threadfence();
    for (int o = threadIdx.x; o < L; o += blockDim.x)
        E.out[o] = vb_fixed_sum(E.group_sums + o, (int)ng, (size_t)L);
    for (unsigned t = threadIdx.x; t < ng + 1; t += blockDim.x)
        E.tickets[t] = 0u;
#ifdef TILED_DYNAMIC
    if (threadIdx.x == 0)
        E.tickets[VB_FINISH_MAXGROUPS] = 0u; // the batch counter of the dynamic-schedule experiment
#endif
    if (threadIdx.x == 0) {
        const unsigned int cnt = *E.fail_count;
        const unsigned long long w = *E.fail_word;
        E.out[L] = (double)cnt;
        E.out[L + 1] = cnt ? -(double)(w >> 16) - 1.0 : -INFINITY;
        *E.fail_latch = w;
        *E.fail_word = ~0ull;
        *E.fail_count = 0u;
    }
}

__device__ __forceinline__ void vb_finish(const EvalParams &E, const int rpb)
{
    FinishArgs F;
    F.partials = E.partials;
    F.group_sums = E.group_sums;
    F.out = E.out;
    F.tickets = E.tickets;
    F.fail_count = E.fail_count;
    F.fail_word = E.fail_word;
    F.fail_latch = E.fail_latch;
    F.L = E.L;
    vb_finish_impl(F, rpb);
}

__device__ __forceinline__ void report_failure(const EvalParams &P, int64_t i, int pivot_plus1)
{
    atomicMin(P.fail_word, ((unsigned long long)i << 16) | (unsigned long long)(pivot_plus1 & 0xffff));
    atomicAdd(P.fail_count, 1u);
}
