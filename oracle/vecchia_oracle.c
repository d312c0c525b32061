/*
 * vecchia_oracle.c -- CPU ORACLE (test infrastructure, NOT product code).
 *
 * A plain-C restatement of the reference package's per-observation Vecchia
 * kernel, its observation loop and its two reductions.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load this library; the product path (paper_2407_02740_b200) never does.
 *
 * Parity status
 *   exponential_isotropic / exponential_anisotropic (and exponential_sphere,
 *   which is the isotropic kernel on embedded coordinates): PINNED.  The
 *   floating-point operation order below follows the reference statement by
 *   statement and the file is compiled with -ffp-contract=off like the
 *   reference (pkg/setup.py:25), so per-observation values and the
 *   deterministic pairwise-tree totals are bit-identical to the reference's
 *   compiled core; tests/test_oracle_golden.py checks that against fixtures
 *   generated from the reference itself (tests/golden/make_golden.py).
 *   exponential_spacetime: derived (chain rule of the anisotropic family,
 *   SURVEY.md 8c) and checked against the reference's anisotropic output.
 *   matern15_isotropic / matern25_isotropic: PARITY UNPINNED -- the reference
 *   has no Matern family (pkg/src/vecchiagp/covariance.py:187-198); these
 *   follow the published closed forms and are checked only by structural
 *   oracles (finite differences, dense exactness at m = n-1).
 *
 * Reference map (paths relative to /root/reference/pkg/src/vecchiagp):
 *   pair_cov        <- engine/_kernels.pyx:34-50    (_cov_entry)
 *   pair_dcov       <- engine/_kernels.pyx:53-99    (_dcov_entry)
 *   live_count      <- engine/_kernels.pyx:188-192  (_count_row)
 *   gather_local    <- engine/_kernels.pyx:195-205  (_gather_row)
 *   factor_lower    <- engine/_kernels.pyx:235-251  (_chol)
 *   solve_forward   <- engine/_kernels.pyx:254-263  (_fsolve)
 *   solve_back_unit <- engine/_kernels.pyx:266-275  (_bsolve_elast)
 *   deriv_vector    <- engine/_kernels.pyx:278-291  (_deriv_solve)
 *   emit_terms      <- engine/_kernels.pyx:294-344  (_contract)
 *   one_observation <- engine/_kernels.pyx:347-381  (_obs_kernel)
 *   vo_run          <- engine/__init__.py:196-248   (run: head pass, tail pass,
 *                      failure report, reduction) + _kernels.pyx:412-429
 *   tree_reduce     <- engine/__init__.py:124-138   (_tree_sum)
 *   vo_neighbor_scan<- engine/_kernels.pyx:609-651  (_scan_row / neighbor_scan)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum {
    FAM_EXP_ISO = 0,
    FAM_EXP_ANISO = 1,
    FAM_EXP_SPACETIME = 2,
    FAM_MATERN15 = 3,
    FAM_MATERN25 = 4,
    FAM_MATERN = 5 /* general order: theta = variance, range, smoothness, nugget */
};

#define MATERN_H 1e-5 /* central-difference step of the smoothness derivative */

typedef struct {
    const double *y, *X, *locs;
    const int64_t *nn;
    const double *theta;
    int64_t n;
    int p, d, q, mp1, family;
    double jitter;
} problem_t;

/* Accumulator layout of one observation (and of the reduced totals), in the
 * C order of the reference's slot arrays (engine/__init__.py:141-152):
 * logdet, ysy, xsx[p][p], ysx[p], dlogdet[q], dysy[q], dysx[p][q],
 * dxsx[p][p][q], ainfo[q][q]. */
static int acc_len(int p, int q) { return (1 + q) * (2 + p + p * p) + q * q; }

/* ---- covariance entries ------------------------------------------------ */

static double sq_dist(const double *a, const double *b, int d)
{
    double s = 0.0;
    for (int l = 0; l < d; ++l) {
        double diff = a[l] - b[l];
        s += diff * diff;
    }
    return s;
}

static double sq_dist_scaled(const double *a, const double *b, int d, const double *rho)
{
    double s = 0.0;
    for (int l = 0; l < d; ++l) {
        double diff = (a[l] - b[l]) / rho[l];
        s += diff * diff;
    }
    return s;
}

/* space-time: axes 0..d-2 share theta[1], the last axis uses theta[2] */
static double sq_dist_spacetime(const double *a, const double *b, int d, const double *theta)
{
    double s = 0.0;
    for (int l = 0; l < d; ++l) {
        double diff = (a[l] - b[l]) / (l < d - 1 ? theta[1] : theta[2]);
        s += diff * diff;
    }
    return s;
}

/* ---- general-order Matern (PARITY UNPINNED: not in the reference) ------------
 * Modified Bessel function K_nu(x), real nu >= 0, x > 0, by Temme's method
 * (J. Comput. Phys. 19, 1975): power series for x <= 2, Steed's continued
 * fraction for x > 2, then upward recurrence in the order.  Written for the
 * oracle independently of the device code; tests/test_oracle_golden.py checks
 * it against scipy.special.kv. */
static void temme_gammas(double mu, double *g1, double *g2, double *gpl, double *gmi)
{
    long double m = (long double)mu;
    long double gp = 1.0L / tgammal(1.0L + m), gm = 1.0L / tgammal(1.0L - m);
    *gpl = (double)gp;
    *gmi = (double)gm;
    *g2 = (double)((gm + gp) / 2.0L);
    if (fabsl(m) < 1e-4L)
        *g1 = (double)(-(0.5772156649015328606L - 0.0420026350340952L * m * m));
    else
        *g1 = (double)((gm - gp) / (2.0L * m));
}

static double bessel_k(double nu, double x, double *k_lower /* K_{nu-1} */)
{
    const int n = (int)floor(nu + 0.5);
    const double mu = nu - n;
    double kmu, kmu1;
    if (x <= 2.0) {
        double g1, g2, gpl, gmi;
        temme_gammas(mu, &g1, &g2, &gpl, &gmi);
        const double pimu = 3.14159265358979323846 * mu;
        const double fact = fabs(pimu) < 1e-9 ? 1.0 : pimu / sin(pimu);
        const double half = x / 2.0;
        const double dl = -log(half);
        double e = mu * dl;
        const double sh = fabs(e) < 1e-10 ? 1.0 : sinh(e) / e;
        double f = fact * (g1 * cosh(e) + g2 * sh * dl);
        double s0 = f;
        e = exp(e);
        double pp = e / (2.0 * gpl), qq = 1.0 / (2.0 * e * gmi), cc = 1.0, s1 = pp;
        for (int i = 1; i < 400; ++i) {
            f = (i * f + pp + qq) / (i * i - mu * mu);
            cc *= half * half / i;
            pp /= (i - mu);
            qq /= (i + mu);
            double term = cc * f;
            s0 += term;
            s1 += cc * (pp - i * f);
            if (fabs(term) < fabs(s0) * 1e-17)
                break;
        }
        kmu = s0;
        kmu1 = s1 * 2.0 / x;
    } else {
        double b = 2.0 * (1.0 + x), d = 1.0 / b, h = d, dh = d, q1 = 0.0, q2 = 1.0;
        const double a1 = 0.25 - mu * mu;
        double q = a1, c = a1, a = -a1, s = 1.0 + q * dh;
        for (int i = 2; i < 400; ++i) {
            a -= 2.0 * (i - 1);
            c = -a * c / i;
            double qn = (q1 - b * q2) / a;
            q1 = q2;
            q2 = qn;
            q += c * qn;
            b += 2.0;
            d = 1.0 / (b + a * d);
            dh = (b * d - 1.0) * dh;
            h += dh;
            double ds = q * dh;
            s += ds;
            if (fabs(ds) < fabs(s) * 1e-17)
                break;
        }
        kmu = sqrt(3.14159265358979323846 / (2.0 * x)) * exp(-x) / s;
        kmu1 = kmu * (mu + x + 0.5 - a1 * h) / x;
    }
    if (n == 0) {
        if (k_lower)
            *k_lower = kmu1 - (2.0 * mu / x) * kmu;
        return kmu;
    }
    double lo = kmu, hi = kmu1;
    for (int i = 1; i < n; ++i) {
        double up = lo + (2.0 * (mu + i) / x) * hi;
        lo = hi;
        hi = up;
    }
    if (k_lower)
        *k_lower = lo;
    return hi;
}

static double matern_corr(double nu, double x)
{
    if (x < 1e-60)
        return 1.0;
    return exp((1.0 - nu) * 0.69314718055994530942 - lgamma(nu) + nu * log(x)) * bessel_k(nu, x, NULL);
}

/* exported for the tests */
double vo_bessel_k(double nu, double x) { return bessel_k(nu, x, NULL); }

static double pair_cov(const problem_t *P, const double *a, const double *b, int same)
{
    const double *th = P->theta;
    if (same)
        return th[0] * (1.0 + th[P->q - 1]) + P->jitter;
    switch (P->family) {
    case FAM_EXP_ISO:
        return th[0] * exp(-sqrt(sq_dist(a, b, P->d)) / th[1]);
    case FAM_EXP_ANISO:
        return th[0] * exp(-sqrt(sq_dist_scaled(a, b, P->d, th + 1)));
    case FAM_EXP_SPACETIME:
        return th[0] * exp(-sqrt(sq_dist_spacetime(a, b, P->d, th)));
    case FAM_MATERN15: {
        double x = sqrt(sq_dist(a, b, P->d)) / th[1];
        return th[0] * (1.0 + x) * exp(-x);
    }
    case FAM_MATERN:
        return th[0] * matern_corr(th[2], sqrt(sq_dist(a, b, P->d)) / th[1]);
    default: { /* FAM_MATERN25 */
        double x = sqrt(sq_dist(a, b, P->d)) / th[1];
        return th[0] * (1.0 + x + x * x / 3.0) * exp(-x);
    }
    }
}

static double pair_dcov(const problem_t *P, int j, const double *a, const double *b, int same)
{
    const double *th = P->theta;
    const int q = P->q, d = P->d;
    /* variance and nugget derivatives are common to every family */
    if (j == q - 1)
        return same ? th[0] : 0.0;
    if (j == 0) {
        if (same)
            return 1.0 + th[q - 1];
        switch (P->family) {
        case FAM_EXP_ISO:
            return exp(-sqrt(sq_dist(a, b, d)) / th[1]);
        case FAM_EXP_ANISO:
            return exp(-sqrt(sq_dist_scaled(a, b, d, th + 1)));
        case FAM_EXP_SPACETIME:
            return exp(-sqrt(sq_dist_spacetime(a, b, d, th)));
        case FAM_MATERN15: {
            double x = sqrt(sq_dist(a, b, d)) / th[1];
            return (1.0 + x) * exp(-x);
        }
        case FAM_MATERN:
            return matern_corr(th[2], sqrt(sq_dist(a, b, d)) / th[1]);
        default: {
            double x = sqrt(sq_dist(a, b, d)) / th[1];
            return (1.0 + x + x * x / 3.0) * exp(-x);
        }
        }
    }
    /* range-like parameters: zero on the diagonal */
    if (same)
        return 0.0;
    switch (P->family) {
    case FAM_EXP_ISO: {
        double r = sqrt(sq_dist(a, b, d));
        return th[0] * exp(-r / th[1]) * r / (th[1] * th[1]);
    }
    case FAM_EXP_ANISO: {
        double s = sqrt(sq_dist_scaled(a, b, d, th + 1));
        if (s == 0.0)
            return 0.0;
        int ax = j - 1;
        double diff = a[ax] - b[ax];
        return th[0] * exp(-s) * diff * diff / (th[1 + ax] * th[1 + ax] * th[1 + ax] * s);
    }
    case FAM_EXP_SPACETIME: {
        double s = sqrt(sq_dist_spacetime(a, b, d, th));
        if (s == 0.0)
            return 0.0;
        double num = 0.0;
        if (j == 1) {
            for (int l = 0; l < d - 1; ++l) {
                double diff = a[l] - b[l];
                num += diff * diff;
            }
        } else {
            double diff = a[d - 1] - b[d - 1];
            num = diff * diff;
        }
        double rho = th[j];
        return th[0] * exp(-s) * num / (rho * rho * rho * s);
    }
    case FAM_MATERN15: {
        double x = sqrt(sq_dist(a, b, d)) / th[1];
        return th[0] * x * x * exp(-x) / th[1];
    }
    case FAM_MATERN: {
        double x = sqrt(sq_dist(a, b, d)) / th[1], nu = th[2];
        if (x < 1e-60)
            return 0.0;
        if (j == 1) { /* d/d range = variance * nc * x^(nu+1) K_{nu-1}(x) / range */
            double klow;
            bessel_k(nu, x, &klow);
            return th[0] * exp((1.0 - nu) * 0.69314718055994530942 - lgamma(nu) + (nu + 1.0) * log(x)) * klow / th[1];
        }
        /* j == 2: smoothness, central difference */
        return th[0] * (matern_corr(nu + MATERN_H, x) - matern_corr(nu - MATERN_H, x)) / (2.0 * MATERN_H);
    }
    default: {
        double x = sqrt(sq_dist(a, b, d)) / th[1];
        return th[0] * x * x * (1.0 + x) * exp(-x) / (3.0 * th[1]);
    }
    }
}

/* ---- dense pieces on one local problem ---------------------------------- */

static int live_count(const int64_t *row, int mp1)
{
    int k = 0;
    while (k < mp1 && row[k] >= 0)
        ++k;
    return k;
}

/* scratch for one worker: every matrix is k-by-k with row stride cap */
typedef struct {
    int cap;
    double *pts, *xs, *ys, *K, *D, *z, *W, *u, *c, *t, *wc;
} scratch_t;

static size_t scratch_doubles(int cap, int d, int p, int q)
{
    size_t c = (size_t)cap;
    return c * d + c * p + c + c * c * (1 + (size_t)q) + c + c * p + c + (size_t)q * c + c + p;
}

static void scratch_bind(scratch_t *S, double *base, int cap, int d, int p, int q)
{
    size_t c = (size_t)cap;
    S->cap = cap;
    S->pts = base;
    S->xs = S->pts + c * d;
    S->ys = S->xs + c * p;
    S->K = S->ys + c;
    S->D = S->K + c * c;
    S->z = S->D + (size_t)q * c * c;
    S->W = S->z + c;
    S->u = S->W + c * p;
    S->c = S->u + c;
    S->t = S->c + (size_t)q * c;
    S->wc = S->t + c;
}

/* local frame = reversed row: the conditioned observation is last */
static void gather_local(const problem_t *P, const int64_t *row, int k, scratch_t *S)
{
    for (int a = 0; a < k; ++a) {
        int64_t g = row[k - 1 - a];
        for (int b = 0; b < P->d; ++b)
            S->pts[a * P->d + b] = P->locs[g * P->d + b];
        for (int b = 0; b < P->p; ++b)
            S->xs[a * P->p + b] = P->X[g * P->p + b];
        S->ys[a] = P->y[g];
    }
}

static int factor_lower(double *K, int k, int ld)
{
    for (int a = 0; a < k; ++a) {
        for (int b = 0; b < a; ++b) {
            double s = K[a * ld + b];
            for (int l = 0; l < b; ++l)
                s -= K[a * ld + l] * K[b * ld + l];
            K[a * ld + b] = s / K[b * ld + b];
        }
        double s = K[a * ld + a];
        for (int l = 0; l < a; ++l)
            s -= K[a * ld + l] * K[a * ld + l];
        if (s <= 0.0)
            return a + 1;
        K[a * ld + a] = sqrt(s);
    }
    return 0;
}

static void solve_forward(const double *B, int k, int ld, const double *rhs, int rinc,
                          double *out, int oinc)
{
    for (int a = 0; a < k; ++a) {
        double s = rhs[a * rinc];
        for (int l = 0; l < a; ++l)
            s -= B[a * ld + l] * out[l * oinc];
        out[a * oinc] = s / B[a * ld + a];
    }
}

static void solve_back_unit(const double *B, int k, int ld, double *u)
{
    for (int a = k - 1; a >= 0; --a) {
        double s = (a == k - 1) ? 1.0 : 0.0;
        for (int l = a + 1; l < k; ++l)
            s -= B[l * ld + a] * u[l];
        u[a] = s / B[a * ld + a];
    }
}

static void deriv_vector(const double *B, int k, int ld, const double *Dj, const double *u,
                         double *t, double *cj)
{
    for (int a = 0; a < k; ++a)
        t[a] = Dj[a * ld + a] * u[a];
    for (int a = 0; a < k; ++a)
        for (int b = 0; b < a; ++b) {
            double v = Dj[a * ld + b];
            t[a] += v * u[b];
            t[b] += v * u[a];
        }
    solve_forward(B, k, ld, t, 1, cj, 1);
}

static void emit_terms(const problem_t *P, const scratch_t *S, int k, double *out)
{
    const int p = P->p, q = P->q, ld = S->cap, e = k - 1;
    const double *z = S->z, *W = S->W;
    double *o_logdet = out, *o_ysy = out + 1, *o_xsx = out + 2, *o_ysx = o_xsx + p * p,
           *o_dlogdet = o_ysx + p, *o_dysy = o_dlogdet + q, *o_dysx = o_dysy + q,
           *o_dxsx = o_dysx + p * q, *o_ainfo = o_dxsx + p * p * q;
    const double ze = z[e];
    *o_logdet = 2.0 * log(S->K[e * ld + e]);
    *o_ysy = ze * ze;
    for (int b = 0; b < p; ++b)
        o_ysx[b] = ze * W[e * p + b];
    for (int a = 0; a < p; ++a)
        for (int b = 0; b < p; ++b)
            o_xsx[a * p + b] = W[e * p + a] * W[e * p + b];
    for (int j = 0; j < q; ++j) {
        const double *cj = S->c + (size_t)j * ld;
        double cje = cj[e], zc = 0.0;
        for (int a = 0; a < k; ++a)
            zc += z[a] * cj[a];
        for (int b = 0; b < p; ++b) {
            double s = 0.0;
            for (int a = 0; a < k; ++a)
                s += W[a * p + b] * cj[a];
            S->wc[b] = s;
        }
        o_dlogdet[j] = cje;
        o_dysy[j] = cje * ze * ze - 2.0 * ze * zc;
        for (int b = 0; b < p; ++b)
            o_dysx[b * q + j] = (cje * ze * W[e * p + b] - ze * S->wc[b] - zc * W[e * p + b]);
        for (int a = 0; a < p; ++a)
            for (int b = 0; b < p; ++b)
                o_dxsx[(a * p + b) * q + j] = (cje * W[e * p + a] * W[e * p + b]
                                               - S->wc[a] * W[e * p + b]
                                               - W[e * p + a] * S->wc[b]);
    }
    for (int j = 0; j < q; ++j) {
        const double *cj = S->c + (size_t)j * ld;
        for (int l = 0; l <= j; ++l) {
            const double *cl = S->c + (size_t)l * ld;
            double s = 0.0;
            for (int a = 0; a < k; ++a)
                s += cj[a] * cl[a];
            s -= 0.5 * cj[e] * cl[e];
            o_ainfo[j * q + l] = s;
            o_ainfo[l * q + j] = s;
        }
    }
}

/* returns 0, or pivot+1 of the failed factorization */
static int one_observation(const problem_t *P, int64_t i, scratch_t *S, double *out)
{
    const int64_t *row = P->nn + i * P->mp1;
    const int k = live_count(row, P->mp1);
    const int d = P->d, p = P->p, q = P->q, ld = S->cap;
    gather_local(P, row, k, S);
    for (int a = 0; a < k; ++a) {
        for (int b = 0; b < a; ++b)
            S->K[a * ld + b] = pair_cov(P, S->pts + a * d, S->pts + b * d, 0);
        S->K[a * ld + a] = pair_cov(P, S->pts + a * d, S->pts + a * d, 1);
    }
    for (int j = 0; j < q; ++j) {
        double *Dj = S->D + (size_t)j * ld * ld;
        for (int a = 0; a < k; ++a) {
            for (int b = 0; b < a; ++b)
                Dj[a * ld + b] = pair_dcov(P, j, S->pts + a * d, S->pts + b * d, 0);
            Dj[a * ld + a] = pair_dcov(P, j, S->pts + a * d, S->pts + a * d, 1);
        }
    }
    int piv = factor_lower(S->K, k, ld);
    if (piv)
        return piv;
    solve_forward(S->K, k, ld, S->ys, 1, S->z, 1);
    for (int b = 0; b < p; ++b)
        solve_forward(S->K, k, ld, S->xs + b, p, S->W + b, p);
    solve_back_unit(S->K, k, ld, S->u);
    for (int j = 0; j < q; ++j)
        deriv_vector(S->K, k, ld, S->D + (size_t)j * ld * ld, S->u, S->t, S->c + (size_t)j * ld);
    emit_terms(P, S, k, out);
    return 0;
}

/* ---- reductions --------------------------------------------------------- */

/* index-ordered pairwise tree over the leading axis, in place on a copy:
 * level by level x[0::2] + x[1::2], an odd tail is carried (not added). */
static void tree_reduce(double *slots, int64_t n, int L, double *out)
{
    int64_t len = n;
    while (len > 1) {
        int64_t half = len / 2;
        for (int64_t t = 0; t < half; ++t)
            for (int c = 0; c < L; ++c)
                slots[t * L + c] = slots[(2 * t) * L + c] + slots[(2 * t + 1) * L + c];
        if (len % 2) {
            memmove(slots + half * L, slots + (2 * half) * L, sizeof(double) * L);
            len = half + 1;
        } else {
            len = half;
        }
    }
    memcpy(out, slots, sizeof(double) * L);
}

/* numpy's add.reduce over axis 0 of a C-contiguous (n, L) array adds rows in
 * index order (the pairwise blocking only applies along a contiguous reduced
 * axis), so a plain running sum per column reproduces np.sum(axis=0). */
static void running_reduce(const double *slots, int64_t n, int L, double *out)
{
    for (int c = 0; c < L; ++c)
        out[c] = 0.0;
    for (int64_t t = 0; t < n; ++t)
        for (int c = 0; c < L; ++c)
            out[c] += slots[t * L + c];
}

/* ---- public entry points ------------------------------------------------ */

int vo_acc_len(int p, int q) { return acc_len(p, q); }

int vo_max_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/*
 * Per-observation terms for i in [i0, i1) written to slots[(i - i0) * L ...];
 * fail[i - i0] = pivot + 1 on a failed factorization.  Returns the lowest
 * failing observation index or -1.  Rows with fewer than m+1 live entries are
 * processed with their true k (engine/__init__.py:236-239).
 */
int64_t vo_observations(const double *y, const double *X, const double *locs, const int64_t *nn,
                        int64_t n, int p, int d, int mp1, const double *theta, int q, int family,
                        double jitter, int64_t i0, int64_t i1, int workers, double *slots,
                        int32_t *fail)
{
    problem_t P = {y, X, locs, nn, theta, n, p, d, q, mp1, family, jitter};
    const int L = acc_len(p, q);
    const int cap = mp1;
    if (i1 <= i0)
        return -1;
    if (workers < 1)
        workers = 1;
    const size_t ws = scratch_doubles(cap, d, p, q);
    double *pool = (double *)calloc(ws * (size_t)workers, sizeof(double));
    if (!pool)
        return -2;
#pragma omp parallel num_threads(workers)
    {
#ifdef _OPENMP
        int tid = omp_get_thread_num();
#else
        int tid = 0;
#endif
        scratch_t S;
        scratch_bind(&S, pool + ws * (size_t)tid, cap, d, p, q);
#pragma omp for schedule(static)
        for (int64_t i = i0; i < i1; ++i) {
            int piv = one_observation(&P, i, &S, slots + (size_t)(i - i0) * L);
            fail[i - i0] = piv;
        }
    }
    free(pool);
    for (int64_t i = i0; i < i1; ++i)
        if (fail[i - i0])
            return i;
    return -1;
}

/*
 * One whole evaluation over [i0, i1): totals of the L accumulators.
 * deterministic != 0 -> pairwise tree (the reference default), else running
 * sum.  On failure *first_fail / *pivot are set and totals are not written.
 */
int vo_run(const double *y, const double *X, const double *locs, const int64_t *nn, int64_t n,
           int p, int d, int mp1, const double *theta, int q, int family, double jitter,
           int64_t i0, int64_t i1, int workers, int deterministic, double *totals,
           int64_t *first_fail, int32_t *pivot)
{
    const int L = acc_len(p, q);
    const int64_t cnt = i1 - i0;
    *first_fail = -1;
    *pivot = -1;
    if (cnt <= 0) {
        for (int c = 0; c < L; ++c)
            totals[c] = 0.0;
        return 0;
    }
    double *slots = (double *)calloc((size_t)cnt * L, sizeof(double));
    int32_t *fail = (int32_t *)calloc((size_t)cnt, sizeof(int32_t));
    if (!slots || !fail) {
        free(slots);
        free(fail);
        return -2;
    }
    int64_t first = vo_observations(y, X, locs, nn, n, p, d, mp1, theta, q, family, jitter, i0, i1,
                                    workers, slots, fail);
    if (first >= 0) {
        *first_fail = first;
        *pivot = fail[first - i0] - 1;
    } else if (deterministic) {
        tree_reduce(slots, cnt, L, totals);
    } else {
        running_reduce(slots, cnt, L, totals);
    }
    free(slots);
    free(fail);
    return 0;
}

/*
 * Nearest-neighbour kriging, restating predict.py:35-90 (krige): for every
 * prediction point, the m_pred training rows with the smallest (d2, index) in
 * working coordinates (predict.py:27-32), their joint covariance with the
 * nugget on the diagonal, the nugget-free cross covariance, a lower Cholesky
 * factor and two forward solves.  mean_resid = half_k . half_r is the
 * conditional mean of the residual y - X beta (the caller adds X* beta);
 * var = prior - half_k . half_k BEFORE the clamp at 0 and the square root.
 * nbrs (nstar, m_pred) receives the chosen training indices.  Returns 0, or
 * 1 + the index of the first point whose factorization failed.
 */
int64_t vo_krige(const double *y, const double *X, const double *locs, int64_t n, int p, int d,
                 const double *theta, int q, int family, const double *beta, const double *locs_star,
                 int64_t nstar, int m_pred, int latent, int workers, double *mean_resid, double *var,
                 int64_t *nbrs)
{
    problem_t P = {y, X, locs, NULL, theta, n, p, d, q, m_pred, family, 0.0};
    const int k = m_pred;
    int64_t failed = 0;
    if (workers < 1)
        workers = 1;
    const double prior = latent ? theta[0] : theta[0] * (1.0 + theta[q - 1]);
#pragma omp parallel num_threads(workers)
    {
        double *bd = (double *)malloc(sizeof(double) * (size_t)k);
        int64_t *bi = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
        double *K = (double *)malloc(sizeof(double) * (size_t)k * k);
        double *kv = (double *)malloc(sizeof(double) * (size_t)k * 3);
        double *hk = kv + k, *hr = kv + 2 * k;
#pragma omp for schedule(static)
        for (int64_t t = 0; t < nstar; ++t) {
            const double *xs = locs_star + t * d;
            int nb = 0;
            for (int64_t j = 0; j < n; ++j) {
                double d2 = 0.0;
                for (int l = 0; l < d; ++l) {
                    double diff = locs[j * d + l] - xs[l];
                    d2 += diff * diff;
                }
                if (nb == k && d2 >= bd[k - 1])
                    continue;
                if (nb < k)
                    ++nb;
                int pos = nb - 1;
                while (pos > 0 && bd[pos - 1] > d2) {
                    bd[pos] = bd[pos - 1];
                    bi[pos] = bi[pos - 1];
                    --pos;
                }
                bd[pos] = d2;
                bi[pos] = j;
            }
            for (int a = 0; a < k; ++a) {
                if (nbrs)
                    nbrs[t * k + a] = bi[a];
                for (int b = 0; b < a; ++b)
                    K[a * k + b] = pair_cov(&P, locs + bi[a] * d, locs + bi[b] * d, 0);
                K[a * k + a] = pair_cov(&P, locs + bi[a] * d, locs + bi[a] * d, 1);
                kv[a] = pair_cov(&P, locs + bi[a] * d, xs, 0);
            }
            if (factor_lower(K, k, k)) {
#pragma omp critical
                if (!failed || t + 1 < failed)
                    failed = t + 1;
                continue;
            }
            solve_forward(K, k, k, kv, 1, hk, 1);
            for (int a = 0; a < k; ++a) {
                double r = y[bi[a]];
                for (int b = 0; b < p; ++b)
                    r -= X[bi[a] * p + b] * beta[b];
                kv[a] = r;
            }
            solve_forward(K, k, k, kv, 1, hr, 1);
            double m0 = 0.0, v0 = 0.0;
            for (int a = 0; a < k; ++a) {
                m0 += hk[a] * hr[a];
                v0 += hk[a] * hk[a];
            }
            mean_resid[t] = m0;
            var[t] = prior - v0;
        }
        free(bd);
        free(bi);
        free(K);
        free(kv);
    }
    return failed;
}

/* exhaustive ordered nearest-predecessor scan; out is (n, m+1), pre-filled -1 */
void vo_neighbor_scan(const double *locs, int64_t n, int d, int m, int workers, int64_t *out)
{
    if (workers < 1)
        workers = 1;
#pragma omp parallel num_threads(workers)
    {
        double *bd = (double *)malloc(sizeof(double) * (size_t)m);
        int64_t *bi = (int64_t *)malloc(sizeof(int64_t) * (size_t)m);
#pragma omp for schedule(static, 64)
        for (int64_t i = 0; i < n; ++i) {
            int nb = 0;
            out[i * (m + 1)] = i;
            for (int64_t j = 0; j < i; ++j) {
                double d2 = 0.0;
                for (int l = 0; l < d; ++l) {
                    double diff = locs[i * d + l] - locs[j * d + l];
                    d2 += diff * diff;
                }
                if (nb == m && d2 >= bd[m - 1])
                    continue; /* ties keep the earlier index */
                if (nb < m)
                    ++nb;
                int pos = nb - 1;
                while (pos > 0 && bd[pos - 1] > d2) {
                    bd[pos] = bd[pos - 1];
                    bi[pos] = bi[pos - 1];
                    --pos;
                }
                bd[pos] = d2;
                bi[pos] = j;
            }
            for (int j = 0; j < nb; ++j)
                out[i * (m + 1) + 1 + j] = bi[j];
        }
        free(bd);
        free(bi);
    }
}
