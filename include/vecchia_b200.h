/*
 * vecchia_b200.h -- C ABI of the B200 (sm_100a) Vecchia likelihood core.
 *
 * This is the drop-in boundary for ONE path of the reference package
 * (`vecchiagp`, /root/reference/pkg/src/vecchiagp): the per-observation hot
 * loop behind `engine.run`.  Every entry point below replaces a piece of the
 * reference's runner seam; file:line citations are relative to
 * /root/reference/pkg/src/vecchiagp/.
 *
 *   reference interface                                   replaced by
 *   ----------------------------------------------------  -----------------------
 *   RUNNERS[backend](y, X, locs_work, nn_idx, theta,      vb200_create (inputs, once)
 *       kcode, jitter, slots, fail, i0, i1, workers, cap)  + vb200_eval / vb200_eval_async
 *       engine/__init__.py:237-245, _kernels.pyx:412-429     (theta, jitter, [i0,i1))
 *   _alloc_slots + _reduce (n-leading slots, host sum)     in-kernel fixed-order reduction;
 *       engine/__init__.py:141-170                           the L totals come back directly
 *   fail[i] = pivot+1, lowest failing index wins           first_fail / pivot out-parameters
 *       _kernels.pyx:384-386,427-429; __init__.py:246-247
 *   kernel_code 0/1 (covariance.py:33-35)                  vb200_family codes below
 *
 * Conventions
 *   - plain pointers and sizes only; no torch / C++ types cross this boundary;
 *   - array layouts are the reference's: y (n,), X (n,p) C-order, locs (n,d)
 *     C-order (already in working coordinates, i.e. after
 *     CovarianceFamily.prepare_locs, covariance.py:143-152), nn int64
 *     (rows, m+1) with -1 padding, column 0 = the observation itself
 *     (preprocess.py:95-118);
 *   - the accumulator vector has L = (1+q)(2+p+p^2) + q^2 doubles in the
 *     C order of the reference's slot arrays (engine/__init__.py:141-152):
 *     logdet, ysy, xsx[p][p], ysx[p], dlogdet[q], dysy[q], dysx[p][q],
 *     dxsx[p][p][q], ainfo[q][q];
 *   - every function returns 0 on success or a negative VB200_E* code;
 *     vb200_last_error() gives the message for the calling thread;
 *   - a numerically failed factorization is DATA, not an error: the call
 *     returns 0 with *first_fail = lowest failing observation index and
 *     *pivot = zero-based failing pivot IN THE REFERENCE'S LOCAL FRAME; the sums
 *     are then unspecified (the reference returns none either);
 *   - there is no CPU fallback: without a CUDA device every compute entry point
 *     fails with VB200_ECUDA.
 */
#ifndef VECCHIA_B200_H
#define VECCHIA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VB200_ABI_VERSION 1

/* error codes */
#define VB200_OK 0
#define VB200_EINVAL (-1)   /* bad argument (shape, family, theta arity, range) */
#define VB200_ECUDA (-2)    /* CUDA runtime error / no device */
#define VB200_ENOMEM (-3)   /* device or host allocation failed */
#define VB200_EUNSUPPORTED (-4) /* shape exceeds what the kernels support (m+1 too wide) */

/* covariance families.  Codes 0/1 are the reference's kernel codes
 * (covariance.py:33-35); the rest are extensions. theta layout:
 *   EXP_ISO / MATERN15 / MATERN25 : [variance, range, nugget]              (q = 3)
 *   EXP_ANISO                     : [variance, range_1..range_d, nugget]   (q = d+2)
 *   EXP_SPACETIME                 : [variance, range_space, range_time, nugget] (q = 4),
 *                                   time is the LAST coordinate
 *   MATERN                        : [variance, range, smoothness, nugget]  (q = 4): general-order Matern
 *                                   variance 2^(1-nu)/Gamma(nu) x^nu K_nu(x), x = r/range; the smoothness
 *                                   derivative is a central difference of step 1e-5
 * The nugget is relative: diag = variance*(1+nugget) + jitter (_kernels.pyx:34-50). */
enum vb200_family {
    VB200_EXP_ISO = 0,
    VB200_EXP_ANISO = 1,
    VB200_EXP_SPACETIME = 2,
    VB200_MATERN15 = 3,
    VB200_MATERN25 = 4,
    VB200_MATERN = 5
};

/* kernel layouts (the north-star layout study); AUTO picks the fastest that supports the shape */
enum vb200_layout {
    VB200_LAYOUT_AUTO = 0,
    VB200_LAYOUT_WARP_SMEM = 1,   /* warp per observation, matrices in shared memory (any shape) */
    VB200_LAYOUT_TILED_REG = 2,   /* sub-warp lane groups, rows register-resident (m+1 <= 64) */
    VB200_LAYOUT_THREAD_SMEM = 3, /* thread per observation (the paper's layout), packed triangle of K staged in
                                   * shared memory; study arm only, m+1 <= 32, d <= 3, p <= 4 */
    VB200_LAYOUT_THREAD_LOCAL = 4 /* thread per observation, every matrix thread-local (local memory), as GpGpU does */
};

typedef struct vb200_problem vb200_problem; /* opaque: device-resident inputs of one dataset shard */

/* ---- introspection (no device needed) ---------------------------------- */
int vb200_abi_version(void);
const char *vb200_last_error(void);
int vb200_acc_len(int p, int q);             /* L */
int vb200_family_nparms(int family, int d);  /* q, or VB200_EINVAL */
int vb200_device_count(void);                /* 0 when no usable CUDA device */

/* ---- problem lifetime --------------------------------------------------- */
/*
 * Upload (or adopt) the inputs of one shard.  `nn` holds rows
 * [nn_row0, nn_row0 + nn_rows) of the neighbor table; y / X / locs always hold
 * all n points (row i only references indices <= i, preprocess.py:99-101).
 * Each of y, X, locs, nn may be a HOST pointer (copied to the device here) or
 * a DEVICE pointer on `device` (adopted without a copy; the caller keeps it
 * alive until vb200_destroy -- this is how torch-allocated buffers are passed).
 * `stream` is a cudaStream_t; NULL is CUDA's default stream.  Device buffers passed in must be
 * ready in stream order on `stream` (the library launches everything there).
 * Replaces the array arguments of the reference runners (_kernels.pyx:392-393).
 */
int vb200_create(int device, int64_t n, int p, int d, int mp1,
                 const double *y, const double *X, const double *locs,
                 const int64_t *nn, int64_t nn_row0, int64_t nn_rows,
                 void *stream, vb200_problem **out);
int vb200_destroy(vb200_problem *prob);
int vb200_set_stream(vb200_problem *prob, void *stream);
int vb200_set_layout(vb200_problem *prob, int layout);
int vb200_get_layout(const vb200_problem *prob, int family, int q); /* layout AUTO resolves to */

/* ---- evaluation --------------------------------------------------------- */
/*
 * Totals of the L accumulators over observations [i0, i1) (which must lie in
 * the shard's nn rows), written to HOST memory; synchronises the stream.
 * Rows with fewer than m+1 live entries are processed with their true size
 * (engine/__init__.py:236-239).  Replaces run_sequential + RUNNERS[backend] +
 * _reduce (engine/__init__.py:233-248).
 */
int vb200_eval(vb200_problem *prob, int family, const double *theta, int q, double jitter,
               int64_t i0, int64_t i1, double *out_sums, int64_t *first_fail, int32_t *pivot);

/*
 * Asynchronous form for multi-GPU use: enqueues the evaluation on the problem's
 * stream and leaves L+2 doubles in DEVICE memory at d_out:
 *   d_out[0..L)  totals,
 *   d_out[L]     number of failed observations (0.0 on success),
 *   d_out[L+1]   -(lowest failing index) - 1 when any failed, else -inf  (so a
 *                MAX all-reduce of this slot, or of the whole vector's last slot,
 *                yields the globally lowest failing index).
 * The [0..L] prefix is combined across ranks with one SUM all-reduce.
 * vb200_fail_info returns the local first failure and its pivot (synchronises).
 */
int vb200_eval_async(vb200_problem *prob, int family, const double *theta, int q, double jitter,
                     int64_t i0, int64_t i1, double *d_out);
int vb200_sync(vb200_problem *prob);
int vb200_fail_info(vb200_problem *prob, int64_t *first_fail, int32_t *pivot);

/* per-observation rows (i1-i0, L) into DEVICE or HOST memory -- the analogue of the
 * reference's slot arrays, for tests and diagnostics (engine/__init__.py:141-152). */
int vb200_eval_rows(vb200_problem *prob, int family, const double *theta, int q, double jitter,
                    int64_t i0, int64_t i1, double *rows_host, int32_t *fail_host);

/* ---- kriging ------------------------------------------ */
/*
 * Nearest-neighbour kriging at `npred` new points from the training data held by `prob`; replaces
 * the per-point loop of the reference's predict.krige (predict.py:77-89).  locs_star (npred, d) are
 * WORKING coordinates, nn_star (npred, m_pred) int64 training indices (any order; -1 pads the tail) --
 * both host or device pointers.  beta (p) are the mean parameters: the kernel forms the residuals
 * y - X beta itself.  Outputs (host, npred each): mean_resid = conditional mean of the residual at the
 * point (the caller adds x*' beta), var = prior - k*' K^-1 k* with prior = variance (latent != 0) or
 * variance*(1+nugget); var is NOT clamped (the reference clamps at 0 before the square root,
 * predict.py:88).  *first_fail = lowest point index whose neighbour covariance failed to factor
 * (the reference raises NotPositiveDefinite(pivot=-1), predict.py:82-85), else -1.
 * Kernels exist for d in {2,3} and m_pred <= 62; otherwise VB200_EUNSUPPORTED.
 */
int vb200_krige(vb200_problem *prob, int family, const double *theta, int q, const double *beta,
                const double *locs_star, const int64_t *nn_star, int64_t npred, int m_pred, int latent,
                double *mean_resid, double *var, int64_t *first_fail);

/* ---- conditional simulation ------------------------------ */
/*
 * Draw y from the neighbour-conditioned model itself; replaces the sequential loop of the reference's
 * oracle.simulate_nn_gp (oracle.py:102-140): y_i = x_i' beta + E[r_i | y of its neighbours] +
 * sqrt(max(var_i, 0)) xi_i with var_i = variance*(1+nugget) - k' K^-1 k.  `prob` must hold the neighbour
 * rows of ALL n observations; xi (n) are the standard normal draws (the reference uses
 * numpy.random.Generator(PCG64(seed)).standard_normal(n): generate them on the host for identical
 * output).  Observation i only depends on observations of lower dependency LEVEL (level = 1 + max level of
 * its neighbours), so the device runs one launch per level: order (n) lists the observations by (level,
 * index), level_ptr (nlevels + 1) delimits the levels (vbh_dependency_levels of the host library builds
 * both).  y_out (n, host or device) receives the draw, and the response held by `prob` is REPLACED by it,
 * so the likelihood of the simulated field can be evaluated on the same handle.  Host or device pointers
 * for xi / order; level_ptr is read on the host.  *first_fail as in vb200_krige.
 */
int vb200_simulate(vb200_problem *prob, int family, const double *theta, int q, const double *beta,
                   const double *xi, const int64_t *order, const int64_t *level_ptr, int64_t nlevels,
                   double *y_out, int64_t *first_fail);

/* number of kernel launches the last vb200_eval* call enqueued, and the name of the
 * main kernel variant (for bench.py's gpu_launches / roofline bookkeeping) */
int vb200_last_launch_count(const vb200_problem *prob);
const char *vb200_last_kernel_name(const vb200_problem *prob);

/* Enumerate the compiled TILED_REG kernel instances (for tests and tooling): instance k serves
 * `family` with exactly d coordinates and p design columns, for any m+1 <= cap-1 (cap = rows of the packed
 * local triangle: lanes_per_obs * rows_per_lane minus the instance's static padding rows beyond the first). */
int vb200_tiled_instance_count(void);
int vb200_tiled_instance(int k, int *lanes_per_obs, int *rows_per_lane, int *cap, int *family, int *d, int *p);

/* CUDA-event timing of the MAIN kernel only (not the reset / reduction launches): enable,
 * evaluate, then read the duration of the last main-kernel launch in milliseconds
 * (synchronises on the closing event).  Used by bench.py for roofline.achieved. */
int vb200_enable_timing(vb200_problem *prob, int on);
int vb200_last_kernel_ms(vb200_problem *prob, double *ms);

/* ---- housekeeping --------------------------------------------------------- */
/* The library's stream-ordered allocations come from a private memory pool per device that keeps up to
 * 2 GiB of freed memory cached (so re-creating a problem per step does not pay the driver's map/unmap);
 * this returns the cached memory of `device` to the driver (synchronises the device). */
int vb200_release_memory(int device);
/* Upload helper for the neighbor table (the largest input: 8(m+1) bytes per observation, and the end-to-end path
 * is bound by its PCIe copy): a host caller may narrow the int64 indices of a dataset with n < 2^31 points to int32
 * (vbh_narrow_indices in libvecchia_host.so), copy half the bytes, and have the device widen them in place of the
 * rows vb200_create was given.  src / dst are DEVICE pointers (8- / 16-byte aligned), enqueued on `stream`. */
int vb200_widen_indices(const int32_t *src, int64_t *dst, int64_t count, void *stream);
/* Number of evaluations since process start for which VB200_LAYOUT_AUTO found no TILED_REG instance and ran
 * the shape-agnostic WARP_SMEM kernel instead (roughly 10x slower): 0 means every evaluation took the fast path. */
unsigned long long vb200_fallback_count(void);

/* ---- measurement helper -------------------------------------------------- */
/* FP64 FMA throughput of `device` in TFLOP/s (2 flops per DFMA) from a register-resident
 * DFMA micro-kernel timed with CUDA events for about `seconds`: *burst = best single
 * launch, *sustained = all launches / total time.  MEASURED_PEAKS.json has no FP64
 * entry, so bench.py measures the roofline denominator itself. */
int vb200_measure_fp64_peak(int device, double seconds, double *burst_tflops, double *sustained_tflops);
/* The same through the FP64 MMA instruction (mma.sync m8n8k4, SASS DMMA): it issues on the same FP64
 * units and reaches their nominal rate, so bench.py takes max(DFMA, DMMA) as the roofline denominator
 * and records both. */
int vb200_measure_fp64_peak_mma(int device, double seconds, double *burst_tflops, double *sustained_tflops);

#ifdef __cplusplus
}
#endif
#endif /* VECCHIA_B200_H */
