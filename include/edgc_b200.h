/*
 * edgc_b200.h — C ABI of libedgc_b200.so, the B200 (sm_100a) implementation of
 * the EDGC data-parallel hot path.
 *
 * The reference (arxiv 2511.10333, /root/reference/pkg/src/edgc) is a pure
 * Python + NumPy package with no FFI; its drop-in boundary is the Python API
 * re-exported at pkg/src/edgc/__init__.py:15-85.  The Python package
 * paper_2511_10333_b200 mirrors that API name for name and binds the entry
 * points below with ctypes.  Each entry point names the
 * reference interface it replaces.
 *
 * Conventions
 *   - extern "C", plain pointers and sizes, no C++ or torch types.
 *   - Pointers documented as "device" are CUDA device pointers; `stream` is a
 *     cudaStream_t passed as void*.  Every call is asynchronous on `stream`.
 *   - Every function returns an edgc_status; EDGC_OK == 0.  Errors detected
 *     on the device (non-finite input, degenerate sample, bin overflow) are
 *     written to caller-provided device status words and surface when the
 *     caller synchronises (the Python layer raises the reference's exception
 *     there, before any state is committed — see DESIGN.md "raise before
 *     mutate").
 *   - No entry point allocates device memory: callers pass a workspace sized
 *     by the matching *_workspace_bytes query.
 *   - Matrices are row-major fp32, flat index = row * n + col (the reference's
 *     ravel order, entropy.py:74).  Factors are row-major [rows x r].
 */
#ifndef EDGC_B200_H
#define EDGC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EDGC_ABI_VERSION 1

typedef enum {
    EDGC_OK = 0,
    EDGC_EINVAL = 1,        /* ValueError: shape / rank / beta / argument     */
    EDGC_ENONFINITE = 2,    /* ValueError: compressor.py:107-108              */
    EDGC_EDEGENERATE = 3,   /* DegenerateInputError: errors.py:8-9            */
    EDGC_ECUDA = 4,         /* CUDA runtime error (see edgc_last_error)       */
    EDGC_ETOOMANYBINS = 6,  /* ValueError raised by np.histogram (NumPy 2.3.5) */
    EDGC_ECAPACITY = 7,     /* caller buffer too small; retry with more        */
    EDGC_EDRAWS = 8         /* sample plan ran out of pre-generated draws      */
} edgc_status;

int edgc_abi_version(void);
/* Message for the last non-OK status returned on the calling thread. */
const char *edgc_last_error(void);
/* Number of kernels this library has launched in the process so far. */
int64_t edgc_launch_count(void);

/* ------------------------------------------------------------------------
 * Sample plan — replaces np.random.default_rng(seed).choice(N, count,
 * replace=False, shuffle=False) at entropy.py:78 (subsample_entries,
 * entropy.py:67-79).  Bit-exact with NumPy 2.3.5 for N < 2^31.
 * The PCG64 words are default_rng(seed).bit_generator.state (host NumPy
 * derives them from the seed; SeedSequence hashing is init-time scalar work).
 * ---------------------------------------------------------------------- */
typedef struct {
    uint64_t state_hi, state_lo, inc_hi, inc_lo;
    int64_t n_elems;   /* N = m * n                       */
    int64_t count;     /* ceil(beta * N); 1 <= count < N  */
    int32_t *idx;      /* device out [count], NumPy order ([1] with EDGC_PLAN_BITMAP_ONLY) */
    uint32_t *bitmap;  /* optional device out [ceil(N/32)] membership bits
                          (bit e set iff e is sampled; the caller zeroes it) or NULL */
    int64_t flags;     /* EDGC_PLAN_* */
} edgc_plan_desc;
/* Only the membership bitmap (required) and idx[0] (one sampled element, the
 * Gaussian estimator's shift: NumPy's first sample for Floyd plans, its last for
 * tail-shuffle plans) are produced: the set, not the order. */
#define EDGC_PLAN_BITMAP_ONLY 1
/* The plans are on the caller's critical path (built inline, not ahead on a side
 * stream): spread the sequential walk over all SMs instead of packing it onto few. */
#define EDGC_PLAN_LATENCY 2

int64_t edgc_sample_plan_workspace_bytes(const edgc_plan_desc *plans, int n_plans);
/* status_dev: device int32[n_plans]; nonzero = EDGC_EDRAWS for that plan. */
int edgc_sample_plan(const edgc_plan_desc *plans, int n_plans, int32_t *status_dev,
                     void *ws, int64_t ws_bytes, void *stream);

/* out[i] = src[idx[i]] (or src[i] when idx == NULL).  dtype: 0 = fp32, 1 = fp64.
 * Replaces flat[idx] at entropy.py:79. */
int edgc_gather(int src_dtype, const void *src, const int32_t *idx, int64_t count,
                int dst_dtype, void *dst, void *stream);

/* ------------------------------------------------------------------------
 * Gaussian plug-in entropy — replaces entropy_gaussian_plugin
 * (entropy.py:82-90): ln(std(ddof=1)) + 0.5 ln(2 pi e), fp64 reduction,
 * fused with the gather through idx.  Batched over layers for
 * EntropyTracker.observe (entropy.py:168-177).
 * ---------------------------------------------------------------------- */
typedef struct {
    const void *src;        /* fp32 or fp64 (src_dtype), device                       */
    const int32_t *idx;     /* device [count] or NULL (contiguous src)                */
    int64_t count;
    const uint32_t *bitmap; /* optional: stream src[0..n_elems) and keep the elements
                               whose bit is set (the set the plan's idx enumerates);
                               idx must then be given (its first entry is the shift) */
    int64_t n_elems;
} edgc_gauss_desc;

int64_t edgc_entropy_gaussian_workspace_bytes(const edgc_gauss_desc *descs, int n);
/* h_out: device double[n]; status_dev: device int32[n] (EDGC_EINVAL < 2 samples,
 * EDGC_EDEGENERATE zero variance). */
int edgc_entropy_gaussian(int src_dtype, const edgc_gauss_desc *descs, int n, double *h_out,
                          int32_t *status_dev, void *ws, int64_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------
 * Histogram entropy — replaces entropy_histogram (entropy.py:93-107) with
 * np.histogram(x, bins="fd") (fixed_bins == 0) or bins=<int> (fixed_bins > 0).
 * Bin edges and counts are bit-exact with NumPy 2.3.5.
 * inv_cbrt_n must be (double)count ** (-1.0/3.0) computed on the host (same
 * libm pow as NumPy's `x.size ** (-1.0 / 3.0)`).
 * result_dev: device double[5] = {H, first_edge, last_edge, width, nbins}.
 * counts_dev: device int64[bins_cap]; edges_dev (optional) double[bins_cap+1].
 * status_dev: device int32[1]: EDGC_EDEGENERATE (zero range), EDGC_EINVAL
 * (< 2 samples), EDGC_ETOOMANYBINS, EDGC_ECAPACITY (nbins > bins_cap; nbins
 * is still reported in result_dev[4]).
 * ---------------------------------------------------------------------- */
int64_t edgc_entropy_histogram_workspace_bytes(int64_t count);
int edgc_entropy_histogram(int dtype, const void *samples, int64_t count, double inv_cbrt_n,
                           int64_t fixed_bins, int64_t bins_cap, int64_t *counts_dev,
                           double *edges_dev, double *result_dev, int32_t *status_dev,
                           void *ws, int64_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------
 * Low-rank compression with error feedback — replaces compress
 * (compressor.py:94-123), batched over the bucket set as train_toy calls it
 * per (worker, layer) (grad_source.py:389-397).
 *
 * Residual representation: the reference stores residual = work - p q^T
 * (compressor.py:112).  Here the state keeps w (= last step's work) and the
 * last factor pair (p_res, q_res); residual = w - p_res q_res^T is formed on
 * the fly inside the next pass 1 (same arithmetic, never materialised).
 * r_res == 0 means "residual is w" (initial state: w = 0).
 * ---------------------------------------------------------------------- */
typedef struct {
    const float *g;       /* m x n gradient (ld_g)                              */
    float *w;             /* m x n error-feedback base, in/out (ld n)          */
    const float *p_res;   /* m x r_res (ld r_res) or NULL                       */
    const float *q_res;   /* n x r_res (ld r_res) or NULL                       */
    float *q_warm;        /* n x r (ld ld_q): warm start in, next warm start out */
    const float *basis;   /* n x r (ld ld_q): fresh columns, compressor.py:63-66 */
    float *p_out;         /* m x r (ld r): orthonormal P (dead columns = 0)     */
    float *q_out;         /* n x r (ld r): W^T P, dead columns reseeded         */
    double *precond;      /* state, r_cap x r_cap (ld ld_s) upper-triangular warm-start
                             preconditioner, identity at creation; NULL = none.  Any
                             such right factor leaves MGS(w q_warm) unchanged; the
                             library keeps it equal to the last step's transform so
                             the one-sweep Q = Z T path stays well conditioned.  */
    int64_t m, n, ld_g;
    int32_t r, r_res, ld_q, ld_s;
} edgc_compress_desc;

/* Persistent plan: descriptors and tile tables are uploaded into the
 * workspace once (bind, synchronous); run only launches kernels, so it can be
 * captured in a CUDA graph and replayed every step.  edgc_compress below is
 * create + bind + run + destroy in one call. */
typedef struct edgc_compress_plan edgc_compress_plan;
int edgc_compress_plan_create(const edgc_compress_desc *descs, int n, edgc_compress_plan **out);
int64_t edgc_compress_plan_workspace_bytes(const edgc_compress_plan *plan);
int edgc_compress_plan_bind(edgc_compress_plan *plan, void *ws, int64_t ws_bytes, void *stream);
/* phases: bit mask of the EDGC_PHASE_* steps to launch (EDGC_PHASE_ALL for a
 * full step); running them in order in separate calls is equivalent. */
enum {
    EDGC_PHASE_PASS1 = 1,     /* error feedback + P_raw partials (clears status) */
    EDGC_PHASE_FACTOR = 2,    /* P_raw reduce + CholQR2 -> P                     */
    EDGC_PHASE_PASS2 = 4,     /* Q partials = w^T P                               */
    EDGC_PHASE_FINALIZE = 8,  /* Q reduce, dead-column reseed, warm start        */
    EDGC_PHASE_ALL = 15
};
int edgc_compress_plan_run(edgc_compress_plan *plan, double col_tol, int32_t *status_dev, int phases,
                           void *stream);
void edgc_compress_plan_destroy(edgc_compress_plan *plan);

/* Fused sampled-iteration statistics (EntropyTracker.observe, entropy.py:168-177,
 * with the Gaussian plug-in on worker 0's raw gradients): pass 1 already streams
 * every raw gradient element, so on a sampled iteration it can also accumulate
 * the fp64 shifted sums {sum (x-K), sum (x-K)^2} of the elements whose
 * membership bit is set (K = the first sample, as edgc_entropy_gaussian).
 * sample_slots: partial slots per matrix, 0 when some matrix of the plan is
 * off the Z path (the caller then uses edgc_entropy_gaussian).
 * set_sampling arms the NEXT run that includes EDGC_PHASE_PASS1: descs[k] for
 * every matrix of the plan (bitmap NULL = not sampled), partials_dev =
 * double[n][slots][2], zeroed by the caller (a matrix writes only the slots
 * of its own CTAs).  edgc_entropy_gaussian_partials
 * reduces the slots in fixed order into h_out / status_dev as
 * edgc_entropy_gaussian does (counts_dev: int64[n] sample counts). */
typedef struct {
    const uint32_t *bitmap;   /* device membership bits [ceil(m*n/32)] (row-major flat index)  */
    const int32_t *first;     /* device: flat index of the first sample (the shift's element) */
} edgc_sample_desc;
int64_t edgc_compress_plan_sample_slots(const edgc_compress_plan *plan);
int edgc_compress_plan_set_sampling(edgc_compress_plan *plan, const edgc_sample_desc *descs, int n,
                                    double *partials_dev, void *stream);
int edgc_entropy_gaussian_partials(const double *partials_dev, int64_t slots, const int64_t *counts_dev, int n,
                                   double *h_out, int32_t *status_dev, void *stream);

int64_t edgc_compress_workspace_bytes(const edgc_compress_desc *descs, int n);
/* col_tol: relative dead-column tolerance (reference: 1e-12 at fp64,
 * compressor.py:23; see DESIGN.md for the fp32 value).
 * status_dev: device int32[n], bit 0 = non-finite work.  Pass 1 rewrites w in
 * place, so a flagged matrix's state is poisoned: callers that need the
 * reference's raise-before-mutate contract run edgc_check_work_finite first
 * (the Python API does; the bucket engine raises DivergenceError instead, as
 * train_toy does at grad_source.py:381-383).  Factors of a flagged matrix
 * are not written. */
int edgc_compress(const edgc_compress_desc *descs, int n, double col_tol, int32_t *status_dev,
                  void *ws, int64_t ws_bytes, void *stream);

/* ------------------------------------------------------------------------
 * (Averaged) reconstruction — replaces decompress (compressor.py:126-133) and
 * the data-parallel average of decompressed gradients (grad_source.py:
 * 404-408): out = scale * sum_{w < n_ranks} P_w Q_w^T, summed in rank order.
 * ---------------------------------------------------------------------- */
typedef struct {
    const float *p;         /* rank w's P at p + w * p_rank_stride (m x r, ld r) */
    const float *q;         /* rank w's Q at q + w * q_rank_stride (n x r, ld r) */
    float *out;             /* m x n (ld_out)                                     */
    int64_t m, n, ld_out;
    int64_t p_rank_stride, q_rank_stride;
    int32_t r, n_ranks;
    float scale;            /* 1 / n_ranks                                        */
    int32_t pad_;
} edgc_recon_desc;

typedef struct edgc_recon_plan edgc_recon_plan;
int edgc_recon_plan_create(const edgc_recon_desc *descs, int n, edgc_recon_plan **out);
int64_t edgc_recon_plan_workspace_bytes(const edgc_recon_plan *plan);
int edgc_recon_plan_bind(edgc_recon_plan *plan, void *ws, int64_t ws_bytes, void *stream);
int edgc_recon_plan_run(edgc_recon_plan *plan, void *stream);
void edgc_recon_plan_destroy(edgc_recon_plan *plan);

/* Device-initiated all-gather over NVLink (replaces the NCCL all-gather in front
 * of edgc_recon_plan_run, grad_source.py:404-408): every rank's packed factor
 * buffer and int64 flag array are mapped into every process by CUDA IPC.
 * edgc_p2p_signal publishes "my factors of step *counter_dev + 1 are complete"
 * into slot `me` of every rank's flags (peer_flags_dev[w] = rank w's flags as
 * mapped here; release, system scope) and advances the device counter;
 * edgc_p2p_pull waits until each rank's slot in its own flags reaches the counter
 * (acquire) and copies rank w's n floats from bases_dev[w] into gathered[w n ..)
 * -- the gathered layout the reconstruction plans read.  The step number lives on
 * the device, so the pair can be captured in a CUDA graph. */
int edgc_p2p_pull(const float *const *bases_dev, float *gathered, int64_t n, int nranks,
                  const int64_t *flags_dev, const int64_t *counter_dev, void *stream);
int edgc_p2p_signal(int64_t *const *peer_flags_dev, int me, int nranks, int64_t *counter_dev, void *stream);
/* The 64-byte cudaIpcMemHandle of the allocation holding device pointer ptr,
 * and ptr's byte offset in it; map a peer process's allocation into this
 * process on the current device, peer access enabled; and unmap it. */
int edgc_ipc_handle(const void *ptr, void *handle64, int64_t *offset);
int edgc_ipc_open(const void *handle64, void **ptr);
int edgc_ipc_close(void *ptr);

int64_t edgc_reconstruct_workspace_bytes(const edgc_recon_desc *descs, int n);
int edgc_reconstruct(const edgc_recon_desc *descs, int n, void *ws, int64_t ws_bytes, void *stream);

/* residual = w - p_res q_res^T (CompressorState.residual, compressor.py:112). */
int edgc_residual(const float *w, const float *p_res, const float *q_res, int32_t r_res,
                  int64_t m, int64_t n, float *e_out, void *stream);

/* flag_dev (int32, device) |= 1 if any (g + w - p_res q_res^T) is non-finite:
 * the work-matrix check of compressor.py:106-108, run before any state change. */
int edgc_check_work_finite(const float *g, int64_t ld_g, const float *w, const float *p_res,
                           const float *q_res, int32_t r_res, int64_t m, int64_t n,
                           int32_t *flag_dev, void *stream);

/* flag_dev |= 1 if any x[i] (fp32 dtype 0 / fp64 dtype 1) is non-finite
 * (GradientMatrix validation, matrix_core.py:30-38). */
int edgc_check_finite(int dtype, const void *x, int64_t count, int32_t *flag_dev, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* EDGC_B200_H */
