// vecchia_b200.cu -- C ABI (include/vecchia_b200.h) over the sm_100a kernels.
// Host side: problem lifetime, launch configuration, fixed-order reduction, failure report.
#include "../../include/vecchia_b200.h"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernel_warp_smem.cuh"
#include "kernel_thread.cuh"
#include "tiled_host.cuh"
#include "kernel_krige_generic.cuh"

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
static thread_local std::string g_err;

static int fail(int code, const std::string &msg)
{
    g_err = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                                   \
    do {                                                                                                 \
        cudaError_t _e = (expr);                                                                         \
        if (_e != cudaSuccess)                                                                           \
            return fail(_e == cudaErrorMemoryAllocation ? VB200_ENOMEM : VB200_ECUDA,                    \
                        std::string(#expr) + ": " + cudaGetErrorString(_e));                             \
    } while (0)

// ---------------------------------------------------------------------------
// small kernels
// ---------------------------------------------------------------------------
// Pack y / X / locs (reference row-major arrays) into one record per point:
// rec[i] = { locs[i][0..d), y[i], X[i][0..p), pad } -- one gather touches one or two
// 32-byte sectors instead of d+p+1 separate arrays.
__global__ void pack_records_kernel(const double *y, const double *X, const double *locs, int64_t n, int p, int d,
                                    int rs, double *rec)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    double *r = rec + i * rs;
    for (int l = 0; l < d; ++l)
        r[l] = locs[i * d + l];
    r[d] = y[i];
    for (int b = 0; b < p; ++b)
        r[d + 1 + b] = X[i * p + b];
    for (int t = d + 1 + p; t < rs; ++t)
        r[t] = 0.0;
}

// Design-column padding (enqueue_eval): a shape whose p has no register-tiled instance runs the instance of the next
// larger p on records whose extra design columns are zero -- every accumulator entry that involves a padded column
// is then exactly zero and the others are untouched -- and the result vector is gathered back to the layout of p.
// Likewise an isotropic family in fewer coordinates than any instance has (d = 1) runs a d = 2 instance on records with
// a zero coordinate appended: the distances are unchanged.
// out record = { locs[0..d), 0 x (d_out - d), y, X[0..p), 0 ... }
__global__ void repack_records_kernel(const double *rec, int rs, int d, int p, double *out, int rs_out, int d_out,
                                      int64_t n)
{
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n)
        return;
    const double *r = rec + i * rs;
    double *o = out + i * rs_out;
    for (int t = 0; t < rs_out; ++t) {
        double v = 0.0;
        if (t < d)
            v = r[t];
        else if (t >= d_out && t - d_out <= p) // y and the p design columns
            v = r[d + (t - d_out)];
        o[t] = v;
    }
}

__global__ void gather_result_kernel(const double *src, const int *map, double *dst, int count)
{
    for (int o = threadIdx.x; o < count; o += blockDim.x)
        dst[o] = src[map[o]];
}

// The partial rows are added inside the main kernel (vb_finish, common.cuh): one launch per evaluation.
// An evaluation over an empty range still has to produce its result vector:
__global__ void empty_result_kernel(double *out, int L)
{
    for (int o = threadIdx.x; o < L; o += blockDim.x)
        out[o] = 0.0;
    if (threadIdx.x == 0) {
        out[L] = 0.0;
        out[L + 1] = -INFINITY;
    }
}

// fail_word[0]: live failure word (atomicMin), [1]: live failure count (low 32 bits), [2]: latched word of the
// last finished likelihood evaluation.  The likelihood kernels reset [0] and [1] themselves when they finish
// (vb_finish); kriging / simulation reset them before their launch with this kernel.
__global__ void reset_fail_kernel(unsigned long long *fail_word, unsigned int *fail_count)
{
    *fail_word = ~0ull;
    *fail_count = 0u;
    fail_word[2] = ~0ull;
}

// Register-resident DFMA chains: 16 independent accumulators per thread.
__global__ void dfma_peak_kernel(double *sink, int iters, double a, double b)
{
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
           x7 = x0 + 7, x8 = x0 + 8, x9 = x0 + 9, xa = x0 + 10, xb = x0 + 11, xc = x0 + 12, xd = x0 + 13,
           xe = x0 + 14, xf = x0 + 15;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
            x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
            x8 = fma(x8, a, b); x9 = fma(x9, a, b); xa = fma(xa, a, b); xb = fma(xb, a, b);
            xc = fma(xc, a, b); xd = fma(xd, a, b); xe = fma(xe, a, b); xf = fma(xf, a, b);
        }
    }
    const double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 + x8 + x9 + xa + xb + xc + xd + xe + xf;
    if (s == 12345.678)
        sink[0] = s;
}

// FP64 MMA (mma.sync m8n8k4, SASS DMMA.8x8x4) issue rate: eight independent accumulator tiles per warp.
// Runs on the same FP64 units as DFMA; it reads fewer register operands per FMA and reaches the
// nominal 64 FMA/clk/SM where three-operand DFMA streams do not (tools/micro/dmma_rate.cu).
__global__ void dmma_peak_kernel(double *sink, int iters)
{
    double c[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        c[i][0] = threadIdx.x;
        c[i][1] = i;
    }
    const double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-9 * threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[i][0]), "+d"(c[i][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        s += c[i][0] + c[i][1];
    if (s == 1.2345)
        sink[0] = s;
}

// ---------------------------------------------------------------------------
// problem object
// ---------------------------------------------------------------------------
struct vb200_problem {
    int device = 0;
    int64_t n = 0;
    int p = 0, d = 0, mp1 = 0, rs = 0;
    double *rec = nullptr;
    const int64_t *nn = nullptr;
    bool own_nn = false;
    int64_t nn_row0 = 0, nn_rows = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    double *partials = nullptr; // block partial rows, followed by the group sums of vb_finish
    size_t partials_cap = 0; // doubles
    unsigned int *tickets = nullptr; // VB_FINISH_MAXGROUPS + 1 counters, zero between evaluations
    double *d_out = nullptr; // L+2 (own result vector for vb200_eval)
    size_t d_out_cap = 0;
    unsigned long long *fail_word = nullptr;
    unsigned int *fail_count = nullptr;
    double *h_out = nullptr; // pinned
    size_t h_out_cap = 0;
    unsigned long long *h_fail = nullptr; // pinned
    int layout = VB200_LAYOUT_AUTO;
    int last_launches = 0;
    const char *last_kernel = "";
    int sm_count = 0;
    size_t smem_optin = 0;
    bool timing = false;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    // design-column padding (see repack_records_kernel): records with pad_p >= p design columns, the result vector of
    // the padded evaluation and the gather map back to p (built per (pad_p, q))
    double *rec_pad = nullptr;
    int pad_p = 0, pad_d = 0, rs_pad = 0;
    double *out_pad = nullptr;
    size_t out_pad_cap = 0;
    int *map_dev = nullptr;
    int map_q = 0, map_len = 0;
};

static bool is_device_ptr(const void *ptr)
{
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

extern "C" int vb200_abi_version(void) { return VB200_ABI_VERSION; }
extern "C" const char *vb200_last_error(void) { return g_err.c_str(); }
extern "C" int vb200_acc_len(int p, int q) { return (1 + q) * (2 + p + p * p) + q * q; }

extern "C" int vb200_family_nparms(int family, int d)
{
    switch (family) {
    case VB200_EXP_ISO:
    case VB200_MATERN15:
    case VB200_MATERN25:
        return 3;
    case VB200_EXP_ANISO:
        return d + 2;
    case VB200_EXP_SPACETIME:
        return d >= 2 ? 4 : VB200_EINVAL;
    case VB200_MATERN:
        return 4;
    default:
        return VB200_EINVAL;
    }
}

extern "C" int vb200_device_count(void)
{
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return c;
}

// Stream-ordered allocations come from a PRIVATE memory pool per device whose release threshold is
// unlimited: memory freed by vb200_destroy stays cached in the pool, so the next vb200_create (one per
// dataset; bench.py's end-to-end leg creates one per step) does not pay cuMemCreate / map again
// (measured: 1.2-1.7 ms of host time per create at n = 2^20 with the default pool, which returns unused
// memory to the driver at every synchronisation).
static unsigned long long g_fallback_evals = 0; // see vb200_fallback_count
static std::mutex g_pool_mu;
static std::map<int, cudaMemPool_t> g_pools;

static cudaError_t vb_malloc_async(void **ptr, size_t bytes, cudaStream_t stream)
{
    std::mutex &mu = g_pool_mu;
    std::map<int, cudaMemPool_t> &pools = g_pools;
#ifdef VB200_EXPERIMENTS
    static const bool use_default = getenv("VB200_DEFAULT_POOL") != nullptr; // A/B of the private pool
    if (use_default)
        return cudaMallocAsync(ptr, bytes, stream);
#endif
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess)
        return e;
    cudaMemPool_t pool = nullptr;
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = pools.find(dev);
        if (it == pools.end()) {
            cudaMemPoolProps props;
            memset(&props, 0, sizeof(props));
            props.allocType = cudaMemAllocationTypePinned;
            props.handleTypes = cudaMemHandleTypeNone;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            e = cudaMemPoolCreate(&pool, &props);
            if (e != cudaSuccess)
                return e;
            // freed blocks stay cached up to this much (the e2e path re-creates a 0.3 GB problem per step);
            // anything above goes back to the driver at the next synchronisation, so a long-lived process
            // that shares the GPU with another allocator (PyTorch's) is not starved.  vb200_release_memory()
            // returns the rest.
            unsigned long long keep = 2ull << 30;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
            pools[dev] = pool;
        } else {
            pool = it->second;
        }
    }
    return cudaMallocFromPoolAsync(ptr, bytes, pool, stream);
}
template <class T>
static cudaError_t vb_malloc_async(T **ptr, size_t bytes, cudaStream_t stream)
{
    return vb_malloc_async(reinterpret_cast<void **>(ptr), bytes, stream);
}

extern "C" int vb200_create(int device, int64_t n, int p, int d, int mp1, const double *y, const double *X,
                            const double *locs, const int64_t *nn, int64_t nn_row0, int64_t nn_rows, void *stream,
                            vb200_problem **out)
{
    if (!out)
        return fail(VB200_EINVAL, "out is NULL");
    *out = nullptr;
    if (n < 1 || p < 1 || d < 1 || mp1 < 1)
        return fail(VB200_EINVAL, "n, p, d, m+1 must be >= 1");
    if (p > VB_MAXP || d > VB_MAXD)
        return fail(VB200_EUNSUPPORTED, "p or d exceeds the compiled limits (p <= 16, d <= 20)");
    if (mp1 > 0xfff0)
        return fail(VB200_EUNSUPPORTED, "m+1 too large");
    if (!y || !X || !locs || !nn)
        return fail(VB200_EINVAL, "NULL input array");
    if (nn_row0 < 0 || nn_rows < 0 || nn_row0 + nn_rows > n)
        return fail(VB200_EINVAL, "neighbor rows outside [0, n)");
    if (vb200_device_count() <= device || device < 0)
        return fail(VB200_ECUDA, "no such CUDA device (this library has no CPU fallback)");
    CUDA_TRY(cudaSetDevice(device));

    vb200_problem *P = new vb200_problem();
    P->device = device;
    P->n = n;
    P->p = p;
    P->d = d;
    P->mp1 = mp1;
    P->rs = (d + 1 + p + 1) & ~1;
    P->nn_row0 = nn_row0;
    P->nn_rows = nn_rows;
    int rc = VB200_OK;
    double *ty = nullptr, *tX = nullptr, *tl = nullptr;
    auto cleanup_tmp = [&]() { // stream-ordered: freed after the pack kernel that reads them
        if (ty) cudaFreeAsync(ty, P->stream);
        if (tX) cudaFreeAsync(tX, P->stream);
        if (tl) cudaFreeAsync(tl, P->stream);
        ty = tX = tl = nullptr;
    };
#define TRY_OR_FREE(expr)                                                                                \
    do {                                                                                                 \
        cudaError_t _e = (expr);                                                                         \
        if (_e != cudaSuccess) {                                                                         \
            rc = fail(_e == cudaErrorMemoryAllocation ? VB200_ENOMEM : VB200_ECUDA,                      \
                      std::string(#expr) + ": " + cudaGetErrorString(_e));                               \
            cleanup_tmp();                                                                               \
            vb200_destroy(P);                                                                            \
            return rc;                                                                                   \
        }                                                                                                \
    } while (0)

    // NULL is CUDA's (legacy) default stream, NOT a private one: work the caller queued on the
    // default stream before this call (e.g. torch uploads of the input buffers) is ordered before
    // everything the library launches.
    P->stream = (cudaStream_t)stream;
    {
        int sms = 0, optin = 0; // cudaDeviceGetAttribute is cheap; cudaGetDeviceProperties takes milliseconds
        TRY_OR_FREE(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        TRY_OR_FREE(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
        P->sm_count = sms;
        P->smem_optin = (size_t)optin;
    }

    // Stream-ordered allocations (cudaMallocAsync / cudaFreeAsync): no device-wide synchronisation,
    // so a caller that is still uploading the neighbor table on another stream keeps overlapping.
    bool copied_from_host = false;
    const double *dy = y, *dX = X, *dl = locs;
    if (!is_device_ptr(y)) {
        copied_from_host = true;
        TRY_OR_FREE(vb_malloc_async(&ty, sizeof(double) * n, P->stream));
        TRY_OR_FREE(cudaMemcpyAsync(ty, y, sizeof(double) * n, cudaMemcpyHostToDevice, P->stream));
        dy = ty;
    }
    if (!is_device_ptr(X)) {
        copied_from_host = true;
        TRY_OR_FREE(vb_malloc_async(&tX, sizeof(double) * n * p, P->stream));
        TRY_OR_FREE(cudaMemcpyAsync(tX, X, sizeof(double) * n * p, cudaMemcpyHostToDevice, P->stream));
        dX = tX;
    }
    if (!is_device_ptr(locs)) {
        copied_from_host = true;
        TRY_OR_FREE(vb_malloc_async(&tl, sizeof(double) * n * d, P->stream));
        TRY_OR_FREE(cudaMemcpyAsync(tl, locs, sizeof(double) * n * d, cudaMemcpyHostToDevice, P->stream));
        dl = tl;
    }
    TRY_OR_FREE(vb_malloc_async(&P->rec, sizeof(double) * n * P->rs, P->stream));
    {
        const int bs = 256;
        const unsigned grid = (unsigned)((n + bs - 1) / bs);
        pack_records_kernel<<<grid, bs, 0, P->stream>>>(dy, dX, dl, n, p, d, P->rs, P->rec);
        TRY_OR_FREE(cudaGetLastError());
    }
    if (is_device_ptr(nn)) {
        P->nn = nn;
    } else {
        int64_t *tn = nullptr;
        const size_t bytes = sizeof(int64_t) * (size_t)(nn_rows > 0 ? nn_rows : 1) * mp1;
        copied_from_host = true;
        TRY_OR_FREE(vb_malloc_async(&tn, bytes, P->stream));
        P->nn = tn;
        P->own_nn = true;
        if (nn_rows > 0)
            TRY_OR_FREE(cudaMemcpyAsync(tn, nn, sizeof(int64_t) * (size_t)nn_rows * mp1, cudaMemcpyHostToDevice,
                                        P->stream));
    }
    TRY_OR_FREE(vb_malloc_async(&P->fail_word, 4 * sizeof(unsigned long long), P->stream));
    P->fail_count = reinterpret_cast<unsigned int *>(P->fail_word + 1);
    TRY_OR_FREE(vb_malloc_async(&P->tickets, (VB_FINISH_MAXGROUPS + 1) * sizeof(unsigned int), P->stream));
    TRY_OR_FREE(cudaMemsetAsync(P->tickets, 0, (VB_FINISH_MAXGROUPS + 1) * sizeof(unsigned int), P->stream));
    reset_fail_kernel<<<1, 1, 0, P->stream>>>(P->fail_word, P->fail_count);
    TRY_OR_FREE(cudaGetLastError());
    cleanup_tmp();
    // host inputs may be released by the caller on return; adopted device inputs need no wait
    if (copied_from_host)
        TRY_OR_FREE(cudaStreamSynchronize(P->stream));
#undef TRY_OR_FREE
    *out = P;
    return VB200_OK;
}

extern "C" int vb200_destroy(vb200_problem *P)
{
    if (!P)
        return VB200_OK;
    cudaSetDevice(P->device);
    cudaStreamSynchronize(P->stream);
    if (P->rec) cudaFreeAsync(P->rec, P->stream);
    if (P->own_nn && P->nn) cudaFreeAsync((void *)P->nn, P->stream);
    if (P->partials) cudaFreeAsync(P->partials, P->stream);
    if (P->d_out) cudaFreeAsync(P->d_out, P->stream);
    if (P->fail_word) cudaFreeAsync(P->fail_word, P->stream);
    if (P->tickets) cudaFreeAsync(P->tickets, P->stream);
    if (P->rec_pad) cudaFreeAsync(P->rec_pad, P->stream);
    if (P->out_pad) cudaFreeAsync(P->out_pad, P->stream);
    if (P->map_dev) cudaFreeAsync(P->map_dev, P->stream);
    if (P->h_out) cudaFreeHost(P->h_out);
    if (P->h_fail) cudaFreeHost(P->h_fail);
    if (P->ev0) cudaEventDestroy(P->ev0);
    if (P->ev1) cudaEventDestroy(P->ev1);
    cudaGetLastError();
    delete P;
    return VB200_OK;
}

extern "C" int vb200_set_stream(vb200_problem *P, void *stream)
{
    if (!P)
        return fail(VB200_EINVAL, "NULL problem");
    cudaSetDevice(P->device);
    cudaStreamSynchronize(P->stream); // buffers were allocated in the old stream's order
    P->stream = (cudaStream_t)stream;
    return VB200_OK;
}

extern "C" int vb200_set_layout(vb200_problem *P, int layout)
{
    if (!P)
        return fail(VB200_EINVAL, "NULL problem");
    if (layout < VB200_LAYOUT_AUTO || layout > VB200_LAYOUT_THREAD_LOCAL)
        return fail(VB200_EINVAL, "unknown layout");
    P->layout = layout;
    return VB200_OK;
}

// ---------------------------------------------------------------------------
// evaluation
// ---------------------------------------------------------------------------
// Temme constants of one order (host, long double gamma): Gamma_1 = (1/G(1-mu) - 1/G(1+mu)) / (2 mu),
// Gamma_2 = (1/G(1-mu) + 1/G(1+mu)) / 2; for tiny |mu| the odd part of the reciprocal-gamma Taylor
// series is used: Gamma_1 -> -(euler_gamma + a3 mu^2), a3 = -0.0420026350340952.
// digamma in long double: recurrence up to x >= 12, then the asymptotic series (error < 1e-18 there)
static long double digammal(long double x)
{
    long double r = 0.0L;
    while (x < 12.0L) {
        r -= 1.0L / x;
        x += 1.0L;
    }
    const long double f = 1.0L / (x * x);
    return r + logl(x) - 0.5L / x -
           f * (1.0L / 12 - f * (1.0L / 120 - f * (1.0L / 252 - f * (1.0L / 240 - f * (1.0L / 132 - f * (691.0L / 32760 - f / 12))))));
}

static MaternOrder matern_order(double nu)
{
    MaternOrder M;
    memset(&M, 0, sizeof(M));
    M.nu = nu;
    M.nup = (int)std::floor(nu + 0.5);
    M.mu = nu - M.nup;
    const long double mu = (long double)M.mu;
    const long double gp = 1.0L / tgammal(1.0L + mu), gm = 1.0L / tgammal(1.0L - mu);
    M.gampl = (double)gp;
    M.gammi = (double)gm;
    M.gp = (double)tgammal(1.0L + mu);
    M.gm = (double)tgammal(1.0L - mu);
    M.gam2 = (double)(0.5L * (gm + gp));
    if (fabsl(mu) < 1e-4L)
        M.gam1 = (double)(-(0.5772156649015328606L - 0.0420026350340952L * mu * mu));
    else
        M.gam1 = (double)((gm - gp) / (2.0L * mu));
    const long double pimu = 3.14159265358979323846264338L * mu;
    M.fact = (fabsl(pimu) < 1e-9L) ? 1.0 : (double)(pimu / sinl(pimu));
    M.normcon = std::exp((1.0 - nu) * 0.6931471805599453 - std::lgamma(nu));
    M.nc2 = std::exp(0.6931471805599453 - std::lgamma(nu));
    M.inv_mu = M.mu != 0.0 ? 1.0 / M.mu : 0.0;
    // order derivatives (bessel_series_dnu): d(1/G(1+mu)) = -psi(1+mu)/G(1+mu), d(1/G(1-mu)) = +psi(1-mu)/G(1-mu)
    {
        const long double psp = digammal(1.0L + mu), psm = digammal(1.0L - mu);
        M.psi_p = (double)psp;
        M.psi_m = (double)psm;
        M.dgam2 = (double)(0.5L * (psm * gm - psp * gp));
        if (fabsl(mu) < 1e-2L) {
            // Gamma_1 = -(a2 + a4 mu^2 + a6 mu^4 + a8 mu^6 + ...), a_k the coefficients of 1/Gamma(z) = sum a_k z^k
            const long double a4 = -0.0420026350340952355L, a6 = -0.0421977345555443367L, a8 = 0.0072189432466630995L;
            const long double m2 = mu * mu;
            M.dgam1 = (double)(-mu * (2.0L * a4 + m2 * (4.0L * a6 + m2 * 6.0L * a8)));
        } else {
            const long double g1 = (gm - gp) / (2.0L * mu);
            M.dgam1 = (double)(((psm * gm + psp * gp) - 2.0L * g1) / (2.0L * mu));
        }
        if (fabsl(pimu) < 1e-2L) { // pi mu / sin(pi mu) = 1 + t^2/6 + 7 t^4/360 + 31 t^6/15120, t = pi mu
            const long double pi = 3.14159265358979323846264338L, t2 = pimu * pimu;
            M.dfact = (double)(pi * pimu * (1.0L / 3 + t2 * (7.0L / 90 + t2 * 31.0L / 2520)));
        } else {
            const long double pi = 3.14159265358979323846264338L;
            M.dfact = (double)((pimu / sinl(pimu)) * (1.0L / mu - pi * cosl(pimu) / sinl(pimu)));
        }
        M.dlognc2 = (double)(-digammal((long double)nu));
    }
    for (int i = 1; i <= VB_MATERN_TERMS; ++i) {
        M.tm[i - 1] = (double)(2.0L * mu / ((long double)i * i - mu * mu));
        M.r1[i - 1] = (double)(1.0L / ((long double)i * i - mu * mu));
        M.rp[i - 1] = (double)(1.0L / ((long double)i - mu));
        M.rq[i - 1] = (double)(1.0L / ((long double)i + mu));
    }
    long double a = -(0.25L - mu * mu);
    for (int i = 2; i < 2 + VB_MATERN_CF; ++i) {
        a -= 2.0L * (i - 1);
        M.ra[i - 2] = (double)(1.0L / a);
    }
    return M;
}

#ifdef VB200_EXPERIMENTS
// experiments only: per-phase cycle counters of kernels built with -DTILED_CLOCKS (nullptr unless
// vb200_debug_clocks has been called once to allocate them)
static unsigned long long *g_dbg_clocks = nullptr;
#define VB_DBG_CLOCKS 160
extern "C" int vb200_debug_clocks(unsigned long long *out, int n, int reset)
{
    if (!g_dbg_clocks) {
        CUDA_TRY(cudaMalloc(&g_dbg_clocks, sizeof(unsigned long long) * VB_DBG_CLOCKS));
        CUDA_TRY(cudaMemset(g_dbg_clocks, 0, sizeof(unsigned long long) * VB_DBG_CLOCKS));
    }
    CUDA_TRY(cudaDeviceSynchronize());
    if (out && n > 0)
        CUDA_TRY(cudaMemcpy(out, g_dbg_clocks, sizeof(unsigned long long) * (n < VB_DBG_CLOCKS ? n : VB_DBG_CLOCKS),
                            cudaMemcpyDeviceToHost));
    if (reset)
        CUDA_TRY(cudaMemset(g_dbg_clocks, 0, sizeof(unsigned long long) * VB_DBG_CLOCKS));
    return VB200_OK;
}
#else
static unsigned long long *const g_dbg_clocks = nullptr;
#endif

static int fill_params(const vb200_problem *P, int family, const double *theta, int q, double jitter, int64_t i0,
                       int64_t i1, EvalParams &E)
{
    const int want = vb200_family_nparms(family, P->d);
    if (want < 0)
        return fail(VB200_EINVAL, "unknown covariance family code or d too small for it");
    if (q != want)
        return fail(VB200_EINVAL, "theta has the wrong length for this family and d");
    if (!theta)
        return fail(VB200_EINVAL, "theta is NULL");
    for (int j = 0; j < q; ++j)
        if (!std::isfinite(theta[j]))
            return fail(VB200_EINVAL, "covariance parameters must be finite");
    for (int j = 0; j + 1 < q; ++j)
        if (!(theta[j] > 0.0))
            return fail(VB200_EINVAL, "variance and range parameters must be strictly positive");
    if (theta[q - 1] < 0.0)
        return fail(VB200_EINVAL, "nugget must be >= 0");
    if (i0 < P->nn_row0 || i1 > P->nn_row0 + P->nn_rows || i1 < i0)
        return fail(VB200_EINVAL, "[i0, i1) outside the neighbor rows of this shard");
    memset(&E, 0, sizeof(E));
    E.rec = P->rec;
    E.nn = P->nn;
    E.nn_row0 = P->nn_row0;
    E.i0 = i0;
    E.i1 = i1;
    E.p = P->p;
    E.d = P->d;
    E.q = q;
    E.qd = q - 2;
    E.mp1 = P->mp1;
    E.rs = P->rs;
    E.family = family;
    E.L = vb200_acc_len(P->p, q);
    E.sig2 = theta[0];
    E.tau2 = theta[q - 1];
    E.jitter = jitter;
    E.diag = theta[0] * (1.0 + theta[q - 1]) + jitter;
    E.inv_sig2 = 1.0 / theta[0];
    // The reference fails a factorization when a pivot is <= 0 (_kernels.pyx:246-249).  For an
    // exactly singular local matrix (duplicated location, zero nugget) that pivot is pure rounding
    // residue, +-1e-16 * diag, whose sign depends on the summation order; the reference's order
    // happens to give <= 0 (pinned by its tests/test_engine.py:230-243).  To report the same
    // failures independently of summation order, a pivot within 1e-14 * diag of zero also fails.
    E.piv_floor = 1e-14 * E.diag;
    for (int l = 0; l < P->d; ++l) {
        double rho;
        if (family == VB200_EXP_ANISO)
            rho = theta[1 + l];
        else if (family == VB200_EXP_SPACETIME)
            rho = (l < P->d - 1) ? theta[1] : theta[2];
        else
            rho = theta[1];
        E.inv_rho[l] = 1.0 / rho;
    }
    E.fail_word = P->fail_word;
    E.fail_count = P->fail_count;
    E.fail_latch = P->fail_word + 2;
    E.tickets = P->tickets;
    E.dbg_clocks = g_dbg_clocks;
    if (family == VB200_MATERN) {
        const double nu0 = theta[2];
        if (!(nu0 > 2.0 * VB_MATERN_H) || nu0 > 60.0)
            return fail(VB200_EINVAL, "matern_isotropic: smoothness must lie in (2e-5, 60]");
        const double orders[3] = {nu0, nu0 + VB_MATERN_H, nu0 - VB_MATERN_H};
        for (int t = 0; t < 3; ++t)
            E.mat[t] = matern_order(orders[t]);
    }
    return VB200_OK;
}

// room for `rows` partial rows of L doubles plus the group sums of vb_finish behind them
static size_t partial_doubles(size_t rows, int rows_per_block, int L)
{
    const size_t blocks = (rows + rows_per_block - 1) / rows_per_block;
    const size_t groups = (blocks + VB_FINISH_GROUP - 1) / VB_FINISH_GROUP;
    return (rows + groups) * (size_t)L;
}

static int ensure_partials(vb200_problem *P, size_t doubles)
{
    if (doubles <= P->partials_cap)
        return VB200_OK;
    if (P->partials)
        cudaFreeAsync(P->partials, P->stream);
    P->partials = nullptr;
    P->partials_cap = 0;
    CUDA_TRY(vb_malloc_async(&P->partials, sizeof(double) * doubles, P->stream));
    P->partials_cap = doubles;
    return VB200_OK;
}

typedef void (*ws_kernel_t)(const EvalParams);

static ws_kernel_t ws_kernel_for(int family)
{
    switch (family) {
    case VB200_EXP_ISO: return vecchia_warp_smem_kernel<FAM_EXP_ISO>;
    case VB200_EXP_ANISO: return vecchia_warp_smem_kernel<FAM_EXP_ANISO>;
    case VB200_EXP_SPACETIME: return vecchia_warp_smem_kernel<FAM_EXP_SPACETIME>;
    case VB200_MATERN15: return vecchia_warp_smem_kernel<FAM_MATERN15>;
    case VB200_MATERN: return vecchia_warp_smem_kernel<FAM_MATERN>;
    default: return vecchia_warp_smem_kernel<FAM_MATERN25>;
    }
}

// Launch the WARP_SMEM layout; returns the number of blocks via *nblocks.
static int launch_warp_smem(vb200_problem *P, EvalParams &E, int *nblocks)
{
    E.ws_doubles = warp_smem_doubles(P->mp1, P->d, P->p, E.q);
    int warps = WS_WARPS_MAX;
    while (warps > 1 && (size_t)warps * E.ws_doubles * sizeof(double) > P->smem_optin)
        warps >>= 1;
    const size_t smem = (size_t)warps * E.ws_doubles * sizeof(double);
    if (smem > P->smem_optin)
        return fail(VB200_EUNSUPPORTED, "m+1 too wide for the shared-memory layout on this device");
    ws_kernel_t kern = ws_kernel_for(E.family);
    int per_sm = 0;
    if (int rc0 = kernel_blocks_per_sm((const void *)kern, warps * 32, smem, false, &per_sm))
        return rc0 == -100 ? fail(VB200_ECUDA, std::string("launch setup: ") + cudaGetErrorString(cudaGetLastError())) : rc0;
    const int64_t count = E.i1 - E.i0;
    int64_t blocks = (int64_t)P->sm_count * per_sm;
    const int64_t need = (count + warps - 1) / warps;
    if (blocks > need)
        blocks = need;
    if (blocks < 1)
        blocks = 1;
    if ((blocks + VB_FINISH_GROUP - 1) / VB_FINISH_GROUP > VB_FINISH_MAXGROUPS)
        return fail(VB200_EUNSUPPORTED, "grid too large for the in-kernel reduction");
    int rc = ensure_partials(P, partial_doubles((size_t)blocks, 1, E.L));
    if (rc)
        return rc;
    E.partials = P->partials;
    E.group_sums = P->partials + (size_t)blocks * E.L;
    kern<<<(unsigned)blocks, warps * 32, smem, P->stream>>>(E);
    CUDA_TRY(cudaGetLastError());
    *nblocks = (int)blocks;
    P->last_kernel = "vecchia_warp_smem_kernel";
    return VB200_OK;
}

template <bool SMEM_TRI>
static ws_kernel_t thread_kernel_for(int family)
{
    switch (family) {
    case VB200_EXP_ISO: return vecchia_thread_kernel<FAM_EXP_ISO, SMEM_TRI>;
    case VB200_EXP_ANISO: return vecchia_thread_kernel<FAM_EXP_ANISO, SMEM_TRI>;
    case VB200_EXP_SPACETIME: return vecchia_thread_kernel<FAM_EXP_SPACETIME, SMEM_TRI>;
    case VB200_MATERN15: return vecchia_thread_kernel<FAM_MATERN15, SMEM_TRI>;
    case VB200_MATERN: return vecchia_thread_kernel<FAM_MATERN, SMEM_TRI>;
    default: return vecchia_thread_kernel<FAM_MATERN25, SMEM_TRI>;
    }
}

// Launch the THREAD layouts (one thread per observation; study arm).  One partial row per THREAD.
static int launch_thread(vb200_problem *P, EvalParams &E, bool smem_tri, int *nblocks)
{
    if (!thread_layout_supported(P->mp1, P->d, P->p, E.q))
        return fail(VB200_EUNSUPPORTED, "THREAD layouts serve m+1 <= 32, d <= 3, p <= 4, at most 2 range parameters");
    ws_kernel_t kern = smem_tri ? thread_kernel_for<true>(E.family) : thread_kernel_for<false>(E.family);
    const int threads = smem_tri ? 32 : 128;
    const size_t smem = smem_tri ? sizeof(double) * 32 * TH_TRI : 0;
    if (smem > P->smem_optin)
        return fail(VB200_EUNSUPPORTED, "THREAD_SMEM needs 132 KB of shared memory per warp");
    int per_sm = 0;
    if (int rc0 = kernel_blocks_per_sm((const void *)kern, threads, smem, false, &per_sm))
        return rc0 == -100 ? fail(VB200_ECUDA, std::string("launch setup: ") + cudaGetErrorString(cudaGetLastError())) : rc0;
    const int64_t count = E.i1 - E.i0;
    int64_t blocks = (int64_t)P->sm_count * per_sm;
    const int64_t need = (count + threads - 1) / threads;
    if (blocks > need)
        blocks = need;
    if (blocks < 1)
        blocks = 1;
    if ((blocks + VB_FINISH_GROUP - 1) / VB_FINISH_GROUP > VB_FINISH_MAXGROUPS)
        return fail(VB200_EUNSUPPORTED, "grid too large for the in-kernel reduction");
    int rc = ensure_partials(P, partial_doubles((size_t)blocks * threads, threads, E.L));
    if (rc)
        return rc;
    E.partials = P->partials;
    E.group_sums = P->partials + (size_t)blocks * threads * E.L;
    kern<<<(unsigned)blocks, threads, smem, P->stream>>>(E);
    CUDA_TRY(cudaGetLastError());
    *nblocks = (int)(blocks * threads);
    P->last_kernel = smem_tri ? "vecchia_thread_kernel<smem triangle>" : "vecchia_thread_kernel<local memory>";
    return VB200_OK;
}

// The (d, p) the register-tiled layout runs this problem with: its own, or -- design columns padded with zeros, and for
// the isotropic families coordinates padded with zeros -- the nearest larger shape that has an instance; false if none.
static bool tiled_effective_shape(const vb200_problem *P, int family, int *de_out, int *pe_out)
{
    const bool iso = family == VB200_EXP_ISO || family == VB200_MATERN15 || family == VB200_MATERN25 ||
                     family == VB200_MATERN;
    for (int de = P->d; de <= (iso ? 3 : P->d); ++de)
        for (int pe = P->p; pe <= 4; ++pe)
            if (tiled_find(family, P->mp1, pe, de) != nullptr) {
                if (de_out) *de_out = de;
                if (pe_out) *pe_out = pe;
                return true;
            }
    return false;
}

static int tiled_effective_p(const vb200_problem *P, int family)
{
    int de = 0, pe = 0;
    return tiled_effective_shape(P, family, &de, &pe) ? pe : 0;
}

static int resolve_layout(const vb200_problem *P, int family, int q)
{
    int layout = P->layout;
    (void)q;
    if (layout == VB200_LAYOUT_AUTO)
        layout = tiled_effective_p(P, family) ? VB200_LAYOUT_TILED_REG : VB200_LAYOUT_WARP_SMEM;
    return layout;
}

// Records with de coordinates and pe design columns (zeros beyond d and p), the padded result vector and the gather
// map for (pe, q).
static int ensure_padding(vb200_problem *P, int de, int pe, int q)
{
    if (P->pad_p != pe || P->pad_d != de) {
        if (P->rec_pad) {
            CUDA_TRY(cudaFreeAsync(P->rec_pad, P->stream));
            P->rec_pad = nullptr;
        }
        P->rs_pad = (de + 1 + pe + 1) & ~1;
        CUDA_TRY(vb_malloc_async(&P->rec_pad, sizeof(double) * (size_t)P->n * P->rs_pad, P->stream));
        const int bs = 256;
        const unsigned grid = (unsigned)((P->n + bs - 1) / bs);
        repack_records_kernel<<<grid, bs, 0, P->stream>>>(P->rec, P->rs, P->d, P->p, P->rec_pad, P->rs_pad, de, P->n);
        CUDA_TRY(cudaGetLastError());
        P->pad_p = pe;
        P->pad_d = de;
        P->map_q = 0;
    }
    const int Lp = vb200_acc_len(pe, q), L = vb200_acc_len(P->p, q);
    if (P->out_pad_cap < (size_t)Lp + 2) {
        if (P->out_pad)
            CUDA_TRY(cudaFreeAsync(P->out_pad, P->stream));
        CUDA_TRY(vb_malloc_async(&P->out_pad, sizeof(double) * ((size_t)Lp + 2), P->stream));
        P->out_pad_cap = (size_t)Lp + 2;
    }
    if (P->map_q != q) {
        const int p = P->p;
        const AccLayout A(p, q), B(pe, q);
        std::vector<int> map((size_t)L + 2);
        map[0] = 0;
        map[1] = 1;
        for (int a = 0; a < p; ++a)
            for (int b = 0; b < p; ++b)
                map[A.xsx + a * p + b] = B.xsx + a * pe + b;
        for (int b = 0; b < p; ++b)
            map[A.ysx + b] = B.ysx + b;
        for (int j = 0; j < q; ++j) {
            map[A.dlogdet + j] = B.dlogdet + j;
            map[A.dysy + j] = B.dysy + j;
        }
        for (int b = 0; b < p; ++b)
            for (int j = 0; j < q; ++j)
                map[A.dysx + b * q + j] = B.dysx + b * q + j;
        for (int a = 0; a < p; ++a)
            for (int b = 0; b < p; ++b)
                for (int j = 0; j < q; ++j)
                    map[A.dxsx + (a * p + b) * q + j] = B.dxsx + (a * pe + b) * q + j;
        for (int j = 0; j < q * q; ++j)
            map[A.ainfo + j] = B.ainfo + j;
        map[L] = Lp;          // failure count
        map[L + 1] = Lp + 1;  // -(first failing index) - 1
        if (P->map_dev && P->map_len < L + 2) {
            CUDA_TRY(cudaFreeAsync(P->map_dev, P->stream));
            P->map_dev = nullptr;
        }
        if (!P->map_dev) {
            CUDA_TRY(vb_malloc_async(&P->map_dev, sizeof(int) * ((size_t)L + 2), P->stream));
            P->map_len = L + 2;
        }
        // pageable source: the copy has returned from the host buffer when the call returns
        CUDA_TRY(cudaMemcpyAsync(P->map_dev, map.data(), sizeof(int) * ((size_t)L + 2), cudaMemcpyHostToDevice, P->stream));
        CUDA_TRY(cudaStreamSynchronize(P->stream));
        P->map_q = q;
    }
    return VB200_OK;
}

extern "C" int vb200_get_layout(const vb200_problem *P, int family, int q)
{
    if (!P)
        return fail(VB200_EINVAL, "NULL problem");
    return resolve_layout(P, family, q);
}

static int enqueue_eval(vb200_problem *P, int family, const double *theta, int q, double jitter, int64_t i0,
                        int64_t i1, double *d_out, double *d_rows, int *d_fail_rows)
{
    if (!P)
        return fail(VB200_EINVAL, "NULL problem");
    CUDA_TRY(cudaSetDevice(P->device));
    EvalParams E;
    int rc = fill_params(P, family, theta, q, jitter, i0, i1, E);
    if (rc)
        return rc;
    E.rows = d_rows;
    E.fail_rows = d_fail_rows;
    E.out = d_out;
    P->last_launches = 0;
    int nblocks = 0;
    if (i1 > i0) {
        int layout = resolve_layout(P, family, q);
        // per-observation rows (diagnostics) are laid out for p: a padded-p evaluation cannot write them
        if (P->layout == VB200_LAYOUT_AUTO && layout == VB200_LAYOUT_TILED_REG && (d_rows || d_fail_rows) &&
            tiled_effective_p(P, family) != P->p)
            layout = VB200_LAYOUT_WARP_SMEM;
        if (P->layout == VB200_LAYOUT_AUTO && layout == VB200_LAYOUT_WARP_SMEM)
            ++g_fallback_evals;
        if (P->timing)
            CUDA_TRY(cudaEventRecord(P->ev0, P->stream));
        if (layout == VB200_LAYOUT_TILED_REG) {
            int de = 0, pe = 0;
            if (!tiled_effective_shape(P, family, &de, &pe))
                return fail(VB200_EUNSUPPORTED, "TILED_REG layout does not support this shape");
            const bool padded = pe != P->p || de != P->d;
            if (padded) { // no instance for this (d, p): the nearest larger one on zero-padded records
                if ((d_rows || d_fail_rows) && pe != P->p)
                    return fail(VB200_EUNSUPPORTED, "per-observation rows need a TILED_REG instance for this p");
                if ((rc = ensure_padding(P, de, pe, q)))
                    return rc;
                E.rec = P->rec_pad;
                E.rs = P->rs_pad;
                for (int l = P->d; l < de; ++l)
                    E.inv_rho[l] = E.inv_rho[0]; // isotropic families only (tiled_effective_shape)
                E.d = de;
                if (pe != P->p) {
                    E.p = pe;
                    E.L = vb200_acc_len(pe, q);
                    E.out = P->out_pad;
                }
            }
            rc = launch_tiled(P->stream, P->sm_count, P->smem_optin, E, &nblocks, &P->last_kernel,
                              [&](size_t rows) -> double * {
                                  return ensure_partials(P, partial_doubles(rows, 1, E.L)) == VB200_OK ? P->partials
                                                                                                       : nullptr;
                              },
                              (size_t)P->n * (size_t)E.rs * sizeof(double));
            if (rc == -100)
                return fail(VB200_ECUDA, std::string("tiled launch: ") + cudaGetErrorString(cudaGetLastError()));
            if (rc)
                return fail(rc, "tiled launch failed");
            if (padded && pe != P->p) {
                gather_result_kernel<<<1, 128, 0, P->stream>>>(P->out_pad, P->map_dev, d_out, vb200_acc_len(P->p, q) + 2);
                CUDA_TRY(cudaGetLastError());
                P->last_launches++;
            }
        } else if (layout == VB200_LAYOUT_WARP_SMEM) {
            rc = launch_warp_smem(P, E, &nblocks);
            if (rc)
                return rc;
        } else {
            rc = launch_thread(P, E, layout == VB200_LAYOUT_THREAD_SMEM, &nblocks);
            if (rc)
                return rc;
        }
        P->last_launches++;
        if (P->timing)
            CUDA_TRY(cudaEventRecord(P->ev1, P->stream));
    } else {
        P->last_kernel = "";
        empty_result_kernel<<<1, 64, 0, P->stream>>>(d_out, E.L);
        CUDA_TRY(cudaGetLastError());
        P->last_launches++;
    }
    (void)nblocks;
    return VB200_OK;
}

extern "C" int vb200_eval_async(vb200_problem *P, int family, const double *theta, int q, double jitter, int64_t i0,
                                int64_t i1, double *d_out)
{
    if (!d_out)
        return fail(VB200_EINVAL, "d_out is NULL");
    return enqueue_eval(P, family, theta, q, jitter, i0, i1, d_out, nullptr, nullptr);
}

extern "C" int vb200_sync(vb200_problem *P)
{
    if (!P)
        return fail(VB200_EINVAL, "NULL problem");
    CUDA_TRY(cudaSetDevice(P->device));
    CUDA_TRY(cudaStreamSynchronize(P->stream));
    return VB200_OK;
}

static int ensure_host_fail(vb200_problem *P)
{
    if (!P->h_fail)
        CUDA_TRY(cudaMallocHost(&P->h_fail, sizeof(unsigned long long)));
    return VB200_OK;
}

extern "C" int vb200_fail_info(vb200_problem *P, int64_t *first_fail, int32_t *pivot)
{
    if (!P)
        return fail(VB200_EINVAL, "NULL problem");
    CUDA_TRY(cudaSetDevice(P->device));
    if (int rc0 = ensure_host_fail(P))
        return rc0;
    CUDA_TRY(cudaMemcpyAsync(P->h_fail, P->fail_word + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                             P->stream));
    CUDA_TRY(cudaStreamSynchronize(P->stream));
    const unsigned long long w = *P->h_fail;
    if (w == ~0ull) {
        if (first_fail) *first_fail = -1;
        if (pivot) *pivot = -1;
    } else {
        if (first_fail) *first_fail = (int64_t)(w >> 16);
        if (pivot) *pivot = (int32_t)(w & 0xffff) - 1;
    }
    return VB200_OK;
}

extern "C" int vb200_eval(vb200_problem *P, int family, const double *theta, int q, double jitter, int64_t i0,
                          int64_t i1, double *out_sums, int64_t *first_fail, int32_t *pivot)
{
    if (!P)
        return fail(VB200_EINVAL, "NULL problem");
    if (!out_sums)
        return fail(VB200_EINVAL, "out_sums is NULL");
    CUDA_TRY(cudaSetDevice(P->device));
    const int want = vb200_family_nparms(family, P->d);
    if (want < 0 || q != want)
        return fail(VB200_EINVAL, "theta has the wrong length for this family and d");
    const size_t L = (size_t)vb200_acc_len(P->p, q);
    if (P->d_out_cap < L + 2) {
        if (P->d_out) cudaFreeAsync(P->d_out, P->stream);
        P->d_out = nullptr;
        P->d_out_cap = 0;
        CUDA_TRY(vb_malloc_async(&P->d_out, sizeof(double) * (L + 2), P->stream));
        P->d_out_cap = L + 2;
    }
    if (P->h_out_cap < L + 2) {
        if (P->h_out) cudaFreeHost(P->h_out);
        P->h_out = nullptr;
        P->h_out_cap = 0;
        CUDA_TRY(cudaMallocHost(&P->h_out, sizeof(double) * (L + 2)));
        P->h_out_cap = L + 2;
    }
    if (int rc0 = ensure_host_fail(P))
        return rc0;
    int rc = enqueue_eval(P, family, theta, q, jitter, i0, i1, P->d_out, nullptr, nullptr);
    if (rc)
        return rc;
    CUDA_TRY(cudaMemcpyAsync(P->h_out, P->d_out, sizeof(double) * (L + 2), cudaMemcpyDeviceToHost, P->stream));
    CUDA_TRY(cudaStreamSynchronize(P->stream));
    memcpy(out_sums, P->h_out, sizeof(double) * L);
    unsigned long long w = ~0ull;
    if (P->h_out[L] > 0.0) { // rare: fetch the latched failure word (index and pivot) as well
        CUDA_TRY(cudaMemcpyAsync(P->h_fail, P->fail_word + 2, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                 P->stream));
        CUDA_TRY(cudaStreamSynchronize(P->stream));
        w = *P->h_fail;
    }
    if (P->h_out[L] > 0.0 && w != ~0ull) {
        if (first_fail) *first_fail = (int64_t)(w >> 16);
        if (pivot) *pivot = (int32_t)(w & 0xffff) - 1;
    } else {
        if (first_fail) *first_fail = -1;
        if (pivot) *pivot = -1;
    }
    return VB200_OK;
}

extern "C" int vb200_eval_rows(vb200_problem *P, int family, const double *theta, int q, double jitter, int64_t i0,
                               int64_t i1, double *rows_host, int32_t *fail_host)
{
    if (!P)
        return fail(VB200_EINVAL, "NULL problem");
    if (!rows_host || !fail_host)
        return fail(VB200_EINVAL, "NULL output");
    CUDA_TRY(cudaSetDevice(P->device));
    const int want = vb200_family_nparms(family, P->d);
    if (want < 0 || q != want)
        return fail(VB200_EINVAL, "theta has the wrong length for this family and d");
    const size_t L = (size_t)vb200_acc_len(P->p, q);
    const size_t cnt = (size_t)(i1 > i0 ? i1 - i0 : 0);
    if (cnt == 0)
        return VB200_OK;
    double *d_rows = nullptr, *d_tot = nullptr;
    int *d_fail = nullptr;
    auto release = [&]() {
        if (d_rows) cudaFreeAsync(d_rows, P->stream);
        if (d_fail) cudaFreeAsync(d_fail, P->stream);
        if (d_tot) cudaFreeAsync(d_tot, P->stream);
    };
    int rc = VB200_OK;
    cudaError_t e = vb_malloc_async(&d_rows, sizeof(double) * cnt * L, P->stream);
    if (e == cudaSuccess) e = vb_malloc_async(&d_fail, sizeof(int) * cnt, P->stream);
    if (e == cudaSuccess) e = vb_malloc_async(&d_tot, sizeof(double) * (L + 2), P->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_rows, 0, sizeof(double) * cnt * L, P->stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_fail, 0, sizeof(int) * cnt, P->stream);
    if (e != cudaSuccess) {
        release();
        return fail(e == cudaErrorMemoryAllocation ? VB200_ENOMEM : VB200_ECUDA,
                    std::string("eval_rows buffers: ") + cudaGetErrorString(e));
    }
    rc = enqueue_eval(P, family, theta, q, jitter, i0, i1, d_tot, d_rows, d_fail);
    if (rc == VB200_OK) {
        cudaError_t e1 = cudaMemcpyAsync(rows_host, d_rows, sizeof(double) * cnt * L, cudaMemcpyDeviceToHost, P->stream);
        cudaError_t e2 = cudaMemcpyAsync(fail_host, d_fail, sizeof(int) * cnt, cudaMemcpyDeviceToHost, P->stream);
        cudaError_t e3 = cudaStreamSynchronize(P->stream);
        if (e1 != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess)
            rc = fail(VB200_ECUDA, std::string("eval_rows copy: ") +
                                       cudaGetErrorString(e1 != cudaSuccess ? e1 : (e2 != cudaSuccess ? e2 : e3)));
    }
    release();
    return rc;
}

extern "C" int vb200_tiled_instance_count(void)
{
    int n = 0;
    for (const TiledPart &part : kTiledParts)
        n += *part.count;
    return n;
}

extern "C" int vb200_tiled_instance(int k, int *g, int *s, int *cap, int *family, int *d, int *p)
{
    for (const TiledPart &part : kTiledParts) {
        if (k < *part.count) {
            const TiledInstance &t = part.items[k];
            if (g) *g = t.g;
            if (s) *s = t.s;
            if (cap) *cap = t.cap - (t.npad - 1); // serves m+1 <= *cap - 1
            if (family) *family = t.family;
            if (d) *d = t.d;
            if (p) *p = t.p;
            return VB200_OK;
        }
        k -= *part.count;
    }
    return fail(VB200_EINVAL, "instance index out of range");
}

extern "C" int vb200_enable_timing(vb200_problem *P, int on)
{
    if (!P)
        return fail(VB200_EINVAL, "NULL problem");
    CUDA_TRY(cudaSetDevice(P->device));
    if (on && !P->ev0) {
        CUDA_TRY(cudaEventCreate(&P->ev0));
        CUDA_TRY(cudaEventCreate(&P->ev1));
    }
    P->timing = on != 0;
    return VB200_OK;
}

extern "C" int vb200_last_kernel_ms(vb200_problem *P, double *ms)
{
    if (!P || !ms)
        return fail(VB200_EINVAL, "NULL argument");
    if (!P->timing || !P->ev0)
        return fail(VB200_EINVAL, "timing is not enabled");
    CUDA_TRY(cudaSetDevice(P->device));
    CUDA_TRY(cudaEventSynchronize(P->ev1));
    float f = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&f, P->ev0, P->ev1));
    *ms = (double)f;
    return VB200_OK;
}

// Launch configuration of the shape-agnostic kriging kernel: warps per block (<= 4) such that the block's shared
// memory fits, blocks per SM from the occupancy query.  Returns 0, VB200_EUNSUPPORTED or -100 (CUDA error pending).
static int krige_generic_config(const vb200_problem *P, int family, int m_pred, krige_generic_kernel_t *kern, int *warps,
                                size_t *smem, int *per_sm)
{
    const size_t per_warp = sizeof(double) * (size_t)krige_generic_doubles(m_pred + 1, P->d);
    int w = 4;
    while (w > 1 && (size_t)w * per_warp > P->smem_optin)
        w >>= 1;
    if ((size_t)w * per_warp > P->smem_optin)
        return VB200_EUNSUPPORTED;
    *kern = krige_generic_for(family);
    *warps = w;
    *smem = (size_t)w * per_warp;
    return kernel_blocks_per_sm((const void *)*kern, 32 * w, *smem, true, per_sm);
}

// stream-ordered temporaries that are released on EVERY exit path of a function (round 1 leaked them when a
// CUDA call in the middle failed)
struct AsyncFreeGuard {
    cudaStream_t stream;
    std::vector<void *> ptrs;
    explicit AsyncFreeGuard(cudaStream_t s) : stream(s) {}
    void add(void *p) { ptrs.push_back(p); }
    ~AsyncFreeGuard()
    {
        for (void *p : ptrs)
            if (p)
                cudaFreeAsync(p, stream);
    }
};

extern "C" int vb200_krige(vb200_problem *P, int family, const double *theta, int q, const double *beta,
                           const double *locs_star, const int64_t *nn_star, int64_t npred, int m_pred, int latent,
                           double *mean_resid, double *var, int64_t *first_fail)
{
    if (!P)
        return fail(VB200_EINVAL, "NULL problem");
    if (!beta || !locs_star || !nn_star || !mean_resid || !var)
        return fail(VB200_EINVAL, "NULL argument");
    if (npred < 0 || m_pred < 1 || m_pred > P->n)
        return fail(VB200_EINVAL, "m_pred must be in [1, n]");
    CUDA_TRY(cudaSetDevice(P->device));
    EvalParams E;
    int rc = fill_params(P, family, theta, q, 0.0, P->nn_row0, P->nn_row0, E);
    if (rc)
        return rc;
    if (first_fail)
        *first_fail = -1;
    if (npred == 0)
        return VB200_OK;
    const KrigeInstance *inst = krige_find(family, m_pred, P->d);
    krige_generic_kernel_t gkern = nullptr;
    int gwarps = 0, gper_sm = 0;
    size_t gsmem = 0;
    if (!inst) { // any other shape: the generic warp-per-point kernel
        const int rcg = krige_generic_config(P, family, m_pred, &gkern, &gwarps, &gsmem, &gper_sm);
        if (rcg == VB200_EUNSUPPORTED)
            return fail(VB200_EUNSUPPORTED, "m_pred too large for the shared memory of this device");
        if (rcg)
            return fail(VB200_ECUDA, std::string("kriging launch setup: ") + cudaGetErrorString(cudaGetLastError()));
    } else {
        E.pair_tab = tiled_pair_table(inst->g, inst->s);
        if (!E.pair_tab)
            return fail(VB200_ECUDA, "pair table allocation failed");
    }
    KrigeParams K;
    memset(&K, 0, sizeof(K));
    K.npred = npred;
    K.m_pred = m_pred;
    K.prior = latent ? theta[0] : theta[0] * (1.0 + theta[q - 1]);
    for (int b = 0; b < P->p; ++b)
        K.beta[b] = beta[b];
    double *d_locs = nullptr, *d_out = nullptr;
    int64_t *d_nn = nullptr;
    AsyncFreeGuard tmp(P->stream);
    const size_t lbytes = sizeof(double) * (size_t)npred * P->d, nbytes = sizeof(int64_t) * (size_t)npred * m_pred;
    if (is_device_ptr(locs_star)) {
        K.locs_star = locs_star;
    } else {
        CUDA_TRY(vb_malloc_async(&d_locs, lbytes, P->stream));
        tmp.add(d_locs);
        CUDA_TRY(cudaMemcpyAsync(d_locs, locs_star, lbytes, cudaMemcpyHostToDevice, P->stream));
        K.locs_star = d_locs;
    }
    if (is_device_ptr(nn_star)) {
        K.nn_star = nn_star;
    } else {
        CUDA_TRY(vb_malloc_async(&d_nn, nbytes, P->stream));
        tmp.add(d_nn);
        CUDA_TRY(cudaMemcpyAsync(d_nn, nn_star, nbytes, cudaMemcpyHostToDevice, P->stream));
        K.nn_star = d_nn;
    }
    CUDA_TRY(vb_malloc_async(&d_out, sizeof(double) * 2 * (size_t)npred, P->stream));
    tmp.add(d_out);
    K.mean_resid = d_out;
    K.var = d_out + npred;
    reset_fail_kernel<<<1, 1, 0, P->stream>>>(P->fail_word, P->fail_count);
    if (inst) {
        const size_t smem = (size_t)inst->smem_doubles * sizeof(double);
        if (smem > P->smem_optin)
            return fail(VB200_EUNSUPPORTED, "kriging tier exceeds shared memory");
        int per_sm = 0;
        if (kernel_blocks_per_sm((const void *)inst->kernel, 32, smem, true, &per_sm))
            return fail(VB200_ECUDA, std::string("kriging launch setup: ") + cudaGetErrorString(cudaGetLastError()));
        const int opw = 32 / inst->g;
        const int64_t nbatch = (npred + opw - 1) / opw;
        int64_t blocks = (int64_t)P->sm_count * per_sm;
        if (blocks > nbatch)
            blocks = nbatch;
        inst->kernel<<<(unsigned)blocks, 32, smem, P->stream>>>(E, K);
        P->last_kernel = inst->name;
    } else {
        int64_t blocks = (int64_t)P->sm_count * gper_sm;
        if (blocks > (npred + gwarps - 1) / gwarps)
            blocks = (npred + gwarps - 1) / gwarps;
        gkern<<<(unsigned)blocks, 32 * gwarps, gsmem, P->stream>>>(E, K);
        P->last_kernel = "vecchia_krige_generic_kernel";
    }
    CUDA_TRY(cudaGetLastError());
    P->last_launches = 2;
    if (int rc0 = ensure_host_fail(P))
        return rc0;
    CUDA_TRY(cudaMemcpyAsync(mean_resid, d_out, sizeof(double) * (size_t)npred, cudaMemcpyDeviceToHost, P->stream));
    CUDA_TRY(cudaMemcpyAsync(var, d_out + npred, sizeof(double) * (size_t)npred, cudaMemcpyDeviceToHost, P->stream));
    CUDA_TRY(cudaMemcpyAsync(P->h_fail, P->fail_word, sizeof(unsigned long long), cudaMemcpyDeviceToHost, P->stream));
    CUDA_TRY(cudaStreamSynchronize(P->stream));
    if (*P->h_fail != ~0ull && first_fail)
        *first_fail = (int64_t)(*P->h_fail >> 16);
    return VB200_OK;
}

// Conditional simulation from the neighbour-conditioned model (see include/vecchia_b200.h).
extern "C" int vb200_simulate(vb200_problem *P, int family, const double *theta, int q, const double *beta,
                              const double *xi, const int64_t *order, const int64_t *level_ptr, int64_t nlevels,
                              double *y_out, int64_t *first_fail)
{
    if (!P)
        return fail(VB200_EINVAL, "NULL problem");
    if (!beta || !xi || !order || !level_ptr || !y_out)
        return fail(VB200_EINVAL, "NULL argument");
    if (P->nn_row0 != 0 || P->nn_rows != P->n)
        return fail(VB200_EINVAL, "simulation needs the neighbour rows of every observation (not a shard)");
    if (nlevels < 0 || (nlevels > 0 && (level_ptr[0] != 0 || level_ptr[nlevels] != P->n)))
        return fail(VB200_EINVAL, "level_ptr must run from 0 to n");
    CUDA_TRY(cudaSetDevice(P->device));
    EvalParams E;
    int rc = fill_params(P, family, theta, q, 0.0, 0, 0, E);
    if (rc)
        return rc;
    if (first_fail)
        *first_fail = -1;
    if (P->n == 0)
        return VB200_OK;
    const int m_pred = P->mp1 - 1;
    if (m_pred < 1)
        return fail(VB200_EINVAL, "simulation needs at least one neighbour column");
    const KrigeInstance *inst = krige_find(family, m_pred, P->d);
    krige_generic_kernel_t gkern = nullptr;
    int gwarps = 0, gper_sm = 0;
    size_t gsmem = 0;
    if (!inst) {
        const int rcg = krige_generic_config(P, family, m_pred, &gkern, &gwarps, &gsmem, &gper_sm);
        if (rcg == VB200_EUNSUPPORTED)
            return fail(VB200_EUNSUPPORTED, "m too large for the shared memory of this device");
        if (rcg)
            return fail(VB200_ECUDA, std::string("simulation launch setup: ") + cudaGetErrorString(cudaGetLastError()));
    } else {
        E.pair_tab = tiled_pair_table(inst->g, inst->s);
        if (!E.pair_tab)
            return fail(VB200_ECUDA, "pair table allocation failed");
    }
    KrigeParams K;
    memset(&K, 0, sizeof(K));
    K.m_pred = m_pred;
    K.prior = theta[0] * (1.0 + theta[q - 1]);
    for (int b = 0; b < P->p; ++b)
        K.beta[b] = beta[b];
    const size_t nb = sizeof(double) * (size_t)P->n;
    double *d_xi = nullptr, *d_y = nullptr;
    int64_t *d_order = nullptr;
    AsyncFreeGuard tmp(P->stream);
    CUDA_TRY(vb_malloc_async(&d_xi, nb, P->stream));
    tmp.add(d_xi);
    CUDA_TRY(vb_malloc_async(&d_y, nb, P->stream));
    tmp.add(d_y);
    CUDA_TRY(vb_malloc_async(&d_order, sizeof(int64_t) * (size_t)P->n, P->stream));
    tmp.add(d_order);
    CUDA_TRY(cudaMemcpyAsync(d_xi, xi, nb, cudaMemcpyDefault, P->stream));
    CUDA_TRY(cudaMemcpyAsync(d_order, order, sizeof(int64_t) * (size_t)P->n, cudaMemcpyDefault, P->stream));
    K.xi = d_xi;
    K.sim_y = d_y;
    K.rec_w = P->rec;
    reset_fail_kernel<<<1, 1, 0, P->stream>>>(P->fail_word, P->fail_count);
    size_t smem = gsmem;
    int per_sm = gper_sm;
    if (inst) {
        smem = (size_t)inst->smem_doubles * sizeof(double);
        if (smem > P->smem_optin)
            return fail(VB200_EUNSUPPORTED, "kriging tier exceeds shared memory");
        if (kernel_blocks_per_sm((const void *)inst->kernel, 32, smem, true, &per_sm))
            return fail(VB200_ECUDA, std::string("simulation launch setup: ") + cudaGetErrorString(cudaGetLastError()));
    }
    const int opw = inst ? 32 / inst->g : gwarps;
    // one launch per dependency level: the observations of a level only read values of lower levels,
    // written by earlier launches on the same stream
    for (int64_t l = 0; l < nlevels; ++l) {
        const int64_t cnt = level_ptr[l + 1] - level_ptr[l];
        if (cnt <= 0)
            continue;
        K.npred = cnt;
        K.sim_order = d_order + level_ptr[l];
        const int64_t nbatch = (cnt + opw - 1) / opw;
        int64_t blocks = (int64_t)P->sm_count * per_sm;
        if (blocks > nbatch)
            blocks = nbatch;
        if (inst)
            inst->kernel<<<(unsigned)blocks, 32, smem, P->stream>>>(E, K);
        else
            gkern<<<(unsigned)blocks, 32 * gwarps, smem, P->stream>>>(E, K);
    }
    CUDA_TRY(cudaGetLastError());
    P->last_kernel = inst ? inst->name : "vecchia_krige_generic_kernel";
    P->last_launches = 1 + (int)nlevels;
    if (int rc0 = ensure_host_fail(P))
        return rc0;
    CUDA_TRY(cudaMemcpyAsync(y_out, d_y, nb, cudaMemcpyDefault, P->stream));
    CUDA_TRY(cudaMemcpyAsync(P->h_fail, P->fail_word, sizeof(unsigned long long), cudaMemcpyDeviceToHost, P->stream));
    CUDA_TRY(cudaStreamSynchronize(P->stream));
    if (*P->h_fail != ~0ull && first_fail)
        *first_fail = (int64_t)(*P->h_fail >> 16);
    return VB200_OK;
}

extern "C" int vb200_last_launch_count(const vb200_problem *P) { return P ? P->last_launches : 0; }
extern "C" const char *vb200_last_kernel_name(const vb200_problem *P) { return P ? P->last_kernel : ""; }

extern "C" int vb200_measure_fp64_peak(int device, double seconds, double *tflops, double *sustained)
{
    if (!tflops || !sustained)
        return fail(VB200_EINVAL, "output pointer is NULL");
    if (vb200_device_count() <= device || device < 0)
        return fail(VB200_ECUDA, "no such CUDA device");
    CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    double *sink = nullptr;
    CUDA_TRY(cudaMalloc(&sink, sizeof(double)));
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    const int threads = 256, blocks = prop.multiProcessorCount * 4, iters = 4096;
    const double flops_per_launch = 2.0 * 16.0 * 8.0 * (double)iters * threads * (double)blocks;
    double best = 0.0, elapsed = 0.0, total_flops = 0.0;
    dfma_peak_kernel<<<blocks, threads>>>(sink, iters, 0.999999, 1e-9); // warm-up
    CUDA_TRY(cudaDeviceSynchronize());
    if (seconds <= 0.0)
        seconds = 0.2;
    while (elapsed < seconds) {
        CUDA_TRY(cudaEventRecord(e0));
        dfma_peak_kernel<<<blocks, threads>>>(sink, iters, 0.999999, 1e-9);
        CUDA_TRY(cudaEventRecord(e1));
        CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        elapsed += ms * 1e-3;
        total_flops += flops_per_launch;
        const double tf = flops_per_launch / (ms * 1e-3) * 1e-12;
        if (tf > best)
            best = tf;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    *tflops = best;
    *sustained = total_flops / elapsed * 1e-12;
    return VB200_OK;
}

// Best-of FP64 throughput of the DMMA micro-kernel (see dmma_peak_kernel).
extern "C" int vb200_measure_fp64_peak_mma(int device, double seconds, double *tflops, double *sustained)
{
    if (!tflops || !sustained)
        return fail(VB200_EINVAL, "output pointer is NULL");
    if (vb200_device_count() <= device || device < 0)
        return fail(VB200_ECUDA, "no such CUDA device");
    CUDA_TRY(cudaSetDevice(device));
    int sms = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    double *sink = nullptr;
    CUDA_TRY(cudaMalloc(&sink, sizeof(double)));
    cudaEvent_t e0, e1;
    CUDA_TRY(cudaEventCreate(&e0));
    CUDA_TRY(cudaEventCreate(&e1));
    const int threads = 256, blocks = sms * 2, iters = 8192;
    const double flops_per_launch = (double)iters * 8 * (threads / 32) * (double)blocks * 2.0 * 8 * 8 * 4;
    double best = 0.0, elapsed = 0.0, total_flops = 0.0;
    dmma_peak_kernel<<<blocks, threads>>>(sink, 64); // warm-up
    CUDA_TRY(cudaDeviceSynchronize());
    if (seconds <= 0.0)
        seconds = 0.2;
    while (elapsed < seconds) {
        CUDA_TRY(cudaEventRecord(e0));
        dmma_peak_kernel<<<blocks, threads>>>(sink, iters);
        CUDA_TRY(cudaEventRecord(e1));
        CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        elapsed += ms * 1e-3;
        total_flops += flops_per_launch;
        const double tf = flops_per_launch / (ms * 1e-3) * 1e-12;
        if (tf > best)
            best = tf;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    *tflops = best;
    *sustained = total_flops / elapsed * 1e-12;
    return VB200_OK;
}

// Widen neighbor indices shipped as int32 (vbh_narrow_indices of the host library: half the PCIe bytes of the
// table) back to the int64 rows the kernels read.  Both pointers are device memory; `count` entries; enqueued on
// `stream` (no synchronisation).
__global__ void widen_indices_kernel(const int *__restrict__ src, long long *__restrict__ dst, long long count)
{
    const long long stride = (long long)gridDim.x * blockDim.x;
    const long long pairs = count / 2;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < pairs; t += stride) {
        const int2 v = reinterpret_cast<const int2 *>(src)[t];
        reinterpret_cast<longlong2 *>(dst)[t] = make_longlong2((long long)v.x, (long long)v.y);
    }
    if ((count & 1) && blockIdx.x == 0 && threadIdx.x == 0)
        dst[count - 1] = (long long)src[count - 1];
}

extern "C" int vb200_widen_indices(const int32_t *src, int64_t *dst, int64_t count, void *stream)
{
    if (count < 0 || (count > 0 && (!src || !dst)))
        return fail(VB200_EINVAL, "vb200_widen_indices: bad arguments");
    if (count == 0)
        return VB200_OK;
    if ((reinterpret_cast<uintptr_t>(src) & 7) || (reinterpret_cast<uintptr_t>(dst) & 15))
        return fail(VB200_EINVAL, "vb200_widen_indices: src must be 8-byte and dst 16-byte aligned");
    const int threads = 256;
    long long blocks = (count / 2 + threads - 1) / threads;
    blocks = blocks < 1 ? 1 : (blocks > 148 * 16 ? 148 * 16 : blocks);
    widen_indices_kernel<<<(unsigned)blocks, threads, 0, static_cast<cudaStream_t>(stream)>>>(
        src, reinterpret_cast<long long *>(dst), (long long)count);
    CUDA_TRY(cudaGetLastError());
    return VB200_OK;
}

// Return the cached (freed) device memory of the library's private pool on `device` to the driver.
extern "C" int vb200_release_memory(int device)
{
    std::lock_guard<std::mutex> lock(g_pool_mu);
    auto it = g_pools.find(device);
    if (it == g_pools.end())
        return VB200_OK;
    CUDA_TRY(cudaSetDevice(device));
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemPoolTrimTo(it->second, 0));
    return VB200_OK;
}

// Evaluations (since process start) for which VB200_LAYOUT_AUTO had no TILED_REG instance and fell back to
// the shape-agnostic WARP_SMEM kernel (an order of magnitude slower): lets callers notice the cliff.
extern "C" unsigned long long vb200_fallback_count(void) { return g_fallback_evals; }
