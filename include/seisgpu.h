/*
 * seisgpu.h -- C ABI of libseisgpu.so, the B200 (sm_100a) hot path of
 * Anderson-accelerated FWI / LSRTM (arXiv:2008.11778).
 *
 * The reference package (seisopt, pure Python) has no native layer; its
 * "plugin API" for this path is the duck-typed objective protocol
 * (seisopt/optim/problems.py:1-5) and the module functions below it.  Each
 * entry point here replaces one reference routine, named in its comment as
 * seisopt/<file>:<line>.  A ctypes shim (paper_2008_11778_b200/_lib.py) binds
 * these symbols and re-exposes the reference's Python signatures.
 *
 * Conventions
 *  - Plain pointers and sizes only.  "dev" pointers are CUDA device pointers
 *    on the handle's device; "host" pointers are ordinary host memory.
 *  - Element type of every wavefield / gather / model buffer is the handle's
 *    dtype (SG_F32 -> float, SG_F64 -> double) unless stated.
 *  - Arrays are C-order.  Physical grid (nz, nx), x fastest
 *    (seisopt/grid.py:5).  Gathers are (shots, nt, n_rec), time-major
 *    (seisopt/wavesim.py:74).
 *  - Every call returns 0 (SG_OK) or an SG_ERR_* code; sg_last_error() holds
 *    the message (thread-local).  The shim maps codes to the reference's
 *    exceptions: SG_ERR_ARG -> ValueError, SG_ERR_STABILITY ->
 *    StabilityError (seisopt/wavesim.py:41), SG_ERR_EMPTY -> EmptyWindowError
 *    (seisopt/optim/qr.py:18), SG_ERR_MODEL -> "model is not positive and
 *    finite" (seisopt/gradients.py:312-331).
 *  - Work is enqueued on the stream set by sg_set_stream (default: the
 *    legacy default stream).  Calls that return host scalars synchronise.
 */
#ifndef SEISGPU_H
#define SEISGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_OK 0
#define SG_ERR_ARG 1
#define SG_ERR_STABILITY 2
#define SG_ERR_EMPTY 3
#define SG_ERR_CUDA 4
#define SG_ERR_OOM 5
#define SG_ERR_MODEL 6
#define SG_ERR_STATE 7

#define SG_F32 4
#define SG_F64 8

/* forward-wavefield reconstruction for gradients / Born adjoints */
#define SG_RECON_FULL 0       /* whole acceleration history in HBM */
#define SG_RECON_CHECKPOINT 1 /* state checkpoints + segment recompute (bitwise) */
#define SG_RECON_AUTO 2       /* FULL when it fits, else (fp32, >= 2^20 padded cells)
                                 BOUNDARY when >= 8 shots
                                 per batch fit, else CHECKPOINT */
#define SG_RECON_BOUNDARY 3   /* boundary saving: u on the sponge frame every step +
                                 final state; the adjoint runs the forward backwards
                                 in the undamped interior (fused into its step) */

typedef struct sg_desc {
  int32_t nz, nx;                    /* physical grid, seisopt/grid.py:35-61 */
  int32_t pad_top, pad_bottom;       /* PadSpec, seisopt/wavesim.py:108-123 */
  int32_t pad_left, pad_right;
  int32_t nt;                        /* time steps, seisopt/grid.py:123 */
  int32_t n_shots;                   /* sources in the geometry */
  int32_t n_rec;                     /* receivers */
  int32_t dtype;                     /* SG_F32 | SG_F64 */
  int32_t order;                     /* 2 (seisopt 5-point) | 8 (BASELINE configs) */
  int32_t recon;                     /* SG_RECON_* */
  int32_t batch;                     /* max shots per launch, 0 = auto (memory) */
  int32_t checkpoint_every;          /* CHECKPOINT interval, 0 = auto (~sqrt(nt)) */
  int32_t device;                    /* CUDA ordinal */
  int32_t use_graphs;                /* capture time loops in CUDA graphs (1) */
  int32_t group;                     /* shots per CTA group, 0 = auto */
  int32_t step_mode;                 /* 0 = auto (one step per launch), 1 = one
                                        step, 2 = two steps per launch (fp32,
                                        temporally blocked) */
  int32_t chains;                    /* concurrent half-batch chains per sweep:
                                        0 = auto (2), 1 .. 4 */
  int32_t resident;                  /* fp32 cluster-resident whole-sweep kernels
                                        (one thread-block cluster per shot, field
                                        in shared memory, one launch per sweep) for
                                        grids that fit: 1 = on; 0 = auto and -1 =
                                        off both use the one-step kernels (the
                                        resident ones measured slower on B200) */
  double dx, dz, dt;                 /* metres, seconds */
  double cfl_safety;                 /* SimConfig.cfl_safety, seisopt/wavesim.py:57 */
  double mem_budget_bytes;           /* 0 = 50% of free device memory */
} sg_desc;

typedef struct sg_handle sg_handle;
typedef struct sg_aa sg_aa;

const char* sg_last_error(void);
int sg_version(void);
/* Build options compiled into this library: SG_BUILD_EXPERIMENTAL = the
 * opt-in two-step (desc.step_mode = 2) and cluster-resident (desc.resident)
 * kernels, measured slower than the one-step kernels on B200 and left out of
 * the default build (-DSG_EXPERIMENTAL=1 adds them). */
#define SG_BUILD_EXPERIMENTAL 1
int sg_build_flags(void);

/* ---- propagator context: replaces seisopt.wavesim.Workspace
 *      (seisopt/wavesim.py:183-214), built once per geometry rather than per
 *      call ------------------------------------------------------------------ */
int sg_create(const sg_desc* desc, sg_handle** out);
int sg_destroy(sg_handle* h);
int sg_set_stream(sg_handle* h, void* cuda_stream);

/* Sponge profiles pz (nzp) and px (nxp); damp = outer(pz, px)
 * (seisopt/wavesim.py:150-165).  host f64. */
int sg_set_sponge(sg_handle* h, const double* pz, const double* px);

/* Bilinear taps from seisopt/wavesim.py:168-180, computed host-side by the
 * shim (bit-identical restatement) and passed through unchanged:
 * rows/cols (4, n) int32 padded-grid indices, weights (4, n) f64.  Source
 * weights are pre-multiplied by nothing; src_scale = 1/(dx dz)
 * (seisopt/wavesim.py:214).  host pointers. */
int sg_set_geometry(sg_handle* h, const int32_t* src_rows, const int32_t* src_cols,
                    const double* src_w, const int32_t* rec_rows,
                    const int32_t* rec_cols, const double* rec_w, double src_scale);

/* Source wavelet amplitudes (nt) f64 host, seisopt/grid.py:158-176. */
int sg_set_wavelet(sg_handle* h, const double* amp);

/* Squared slowness m (nz, nx), device pointer, element type m_dtype
 * (SG_F32|SG_F64).  Validates positivity/finiteness (SG_ERR_MODEL,
 * seisopt/gradients.py:312-316) and the CFL bound (SG_ERR_STABILITY,
 * seisopt/wavesim.py:187-193; 8th order scaled by sqrt(4/6.5016)), then
 * forms 1/m on the padded grid (seisopt/wavesim.py:200-201).  Synchronises. */
int sg_set_model(sg_handle* h, const void* m_dev, int32_t m_dtype);

/* ---- sweeps --------------------------------------------------------------- */

/* Forward-model shots [shot0, shot0+count): gathers_dev (count, nt, n_rec).
 * Replaces fwi_synthetic, seisopt/gradients.py:98-115 (each shot one
 * _forward_sweep, seisopt/wavesim.py:259-304, keep_accel=False). */
int sg_fwi_synthetic(sg_handle* h, int32_t shot0, int32_t count, void* gathers_dev);

/* Forward + trapezoidal L2 misfit against observed (count, nt, n_rec) dev;
 * *misfit_host = 1/2 dt sum_t w_t sum_r (f-g)^2 summed over the shots.
 * Replaces FwiObjective.value -> fwi_synthetic + misfit_l2,
 * seisopt/gradients.py:318-326, :70-79. */
int sg_fwi_misfit(sg_handle* h, int32_t shot0, int32_t count, const void* observed_dev,
                  double* misfit_host);

/* Misfit and exact adjoint-state gradient over shots [shot0, shot0+count).
 * grad_dev (nz, nx) receives fold_pad(sum_s image_s) of these shots
 * (seisopt/gradients.py:118-155; fold seisopt/wavesim.py:135-147).  With
 * accumulate != 0 the gradient is added to grad_dev.  Synchronises. */
int sg_fwi_gradient(sg_handle* h, int32_t shot0, int32_t count, const void* observed_dev,
                    double* misfit_host, void* grad_dev, int32_t accumulate);

/* Born modelling about the current model as background
 * (BornKernel, seisopt/gradients.py:158-220).
 *  sg_born_forward : data_dev (count, nt, n_rec) = L m_r for m_r (nz, nx) dev
 *                    (seisopt/gradients.py:191-205).
 *  sg_born_adjoint : image_dev (nz, nx) = L^T data (seisopt/gradients.py:207-220).
 *  sg_lsrtm_gradient: J = 1/2 ||L m_r - d_r||^2, grad = L^T (L m_r - d_r)
 *                    (seisopt/gradients.py:253-277).
 * The background acceleration history is cached in HBM when it fits
 * (sg_born_cache), otherwise recomputed (lock-step forward, checkpointed
 * adjoint). */
int sg_born_cache(sg_handle* h, int32_t shot0, int32_t count, int32_t enable);
/* Shots whose background history is cached: a prefix of the requested range
 * sized to the free device memory (the rest is recomputed per apply). */
int sg_born_cached(sg_handle* h, int32_t* shot0, int32_t* count);
int sg_born_forward(sg_handle* h, int32_t shot0, int32_t count, const void* m_r_dev,
                    void* data_dev);
int sg_born_adjoint(sg_handle* h, int32_t shot0, int32_t count, const void* data_dev,
                    void* image_dev, int32_t accumulate);
int sg_lsrtm_gradient(sg_handle* h, int32_t shot0, int32_t count, const void* m_r_dev,
                      const void* d_r_dev, double* value_host, void* grad_dev,
                      int32_t accumulate);
/* LSRTM objective value only: *value_host = 1/2 ||L m_r - d_r||^2 over shots
 * [shot0, shot0+count) (LsrtmObjective.value / residual_norm,
 * seisopt/gradients.py:351-369) -- Born forward with the residual reduced in
 * fp64 on the device; no Born data leave it.  Synchronises. */
int sg_lsrtm_misfit(sg_handle* h, int32_t shot0, int32_t count, const void* m_r_dev,
                    const void* d_r_dev, double* value_host);

/* Single-shot forward with the full acceleration history returned
 * (forward_solve with keep_history, seisopt/wavesim.py:354-378):
 * gather_dev (nt, n_rec), accel_dev (nt, nzp, nxp) padded grid. */
int sg_forward_history(sg_handle* h, int32_t shot, void* gather_dev, void* accel_dev);

/* Adjoint sweep of one data set returning v_n (adjoint_solve,
 * seisopt/wavesim.py:414-430): ybar_dev (nt, n_rec), v_dev (nt, nzp, nxp). */
int sg_adjoint_history(sg_handle* h, const void* ybar_dev, void* v_dev);

/* Diagnostics: shots per batch chosen, reconstruction mode in use, bytes held. */
int sg_query(sg_handle* h, int32_t* batch, int32_t* recon, double* device_bytes);

/* Concurrent shot chains a sweep over `count` shots runs as (desc.chains). */
int sg_chains(sg_handle* h, int32_t count);

/* Cluster-resident sweep plan (desc.resident): out[6] = {in use (0/1), CTAs per
 * cluster, padded columns per CTA, threads per CTA, clusters resident at once,
 * adjoint shared-memory bytes per CTA}.  Plans on first use. */
int sg_resident_plan(sg_handle* h, int32_t* out);

/* Times `reps` steps of one step kernel (0 = forward+history store,
 * 1 = adjoint+imaging, 2 = forward no history; 3 / 4 = the two-step forward /
 * adjoint kernels, two time steps per launch; 5 / 6 = the boundary-saving
 * reverse+adjoint and band-storing forward kernels) over `count` shots with
 * CUDA events on the handle's stream, launched as the sweeps launch them
 * (sg_chains concurrent chains); *ms_per_launch = mean time per step. */
int sg_time_step_kernel(sg_handle* h, int32_t which, int32_t count, int32_t reps,
                        float* ms_per_launch);

/* Device time of the phases of the last sg_fwi_gradient call, summed over
 * its shot batches (CUDA events on the handle's stream): ms_out[4] = {forward
 * sweep, residual + injection, adjoint sweep with imaging, image reduction}.
 * Synchronises on the recorded events. */
int sg_phase_times(sg_handle* h, float* ms_out);

/* Number of kernel launches this handle (or AA window) has issued. */
int64_t sg_launch_count(void);

/* NaN/Inf guard: the number of non-finite entries in the gradient
 * or image the last sg_fwi_gradient / sg_lsrtm_gradient / sg_born_adjoint on
 * this handle wrote (counted on the device while folding the result).  The
 * reference raises nothing for a diverged sweep; the Python layer turns a
 * non-zero count into a RuntimeWarning.  No reference counterpart. */
int sg_last_nonfinite(sg_handle* h, int64_t* count);

/* The library's own memcheck.  With SG_REDZONE=1 in the environment when the
 * library is loaded, every device allocation of a handle or AA window carries
 * 64 KB guard zones of 0xFF bytes (NaN in fp32 and fp64) on both sides: an
 * out-of-bounds read poisons the results, an out-of-bounds write is counted
 * here.  bad_bytes = guard bytes found modified (allocations already freed
 * plus all live ones), allocations = guarded allocations made so far (0: the
 * mode is off).  poke != 0 first overwrites one guard byte of a live
 * allocation (self-test of the detection).  No reference counterpart. */
int sg_redzone_check(int64_t* bad_bytes, int64_t* allocations, int32_t poke);

/* ---- Anderson acceleration window on the device -------------------------
 * Replaces AAWindow / SlidingQR / aa_weights / aa_step
 * (seisopt/optim/anderson.py:55-148, seisopt/optim/qr.py:22-104) by a
 * ring buffer of residual / G differences plus a fp64 Gram matrix updated
 * with one fused pass per push; the m x m least-squares solve runs on the
 * host in fp64 and reproduces the reference's window decisions
 * (append-after-first-push, drop when ncols > memory, rank safeguard
 * min|diag R| <= 1e-12 ||R||_F, zero basis for dependent columns).
 * Windows the fp64 Gram cannot resolve (a Cholesky pivot with
 * rho^2 <= 1e-10 ||a||^2) are re-factored by a device thin QR with CGS2
 * appends in fp64 -- the reference's own append_column
 * (seisopt/optim/qr.py:34-60) -- and solved with its Q^T f and explicit
 * residual (qr.py:82-95). */
int sg_aa_create(int64_t n, int32_t memory, int32_t dtype, int32_t device, sg_aa** out);
int sg_aa_destroy(sg_aa* a);
int sg_aa_set_stream(sg_aa* a, void* cuda_stream);
/* N-sharded window (the standalone AA step on several GPUs shards
 * N): each rank's window holds its slice of the N-vectors.  Every quantity
 * the window reads back from the device -- Gram rows <df, dF_i>, projections
 * <f_k, dF_i>, squared norms, the QR fallback's dots -- is a plain sum over
 * the N entries, so `fn` only has to sum a small host buffer of doubles
 * (<= 2m + 3 values) over the ranks in place (an all-reduce; 0 = success).
 * gamma, alpha, the window decisions and the rank safeguard are then
 * identical on every rank, as the replicated reference window's would be
 * (seisopt/optim/anderson.py:55-123).  NULL restores the single-rank window. */
typedef int (*sg_reduce_fn)(double* buf, int32_t n, void* ctx);
int sg_aa_set_reducer(sg_aa* a, sg_reduce_fn fn, void* ctx);
int sg_aa_clear(sg_aa* a);                                   /* anderson.py:77-78 */
int sg_aa_push(sg_aa* a, const void* p_dev, const void* g_dev); /* anderson.py:80-112 */
int sg_aa_m_k(sg_aa* a);                                     /* anderson.py:69-71 */
/* gamma (m_k), alpha (m_k+1), residual norm: anderson.py:115-123, :41-52 */
int sg_aa_weights(sg_aa* a, double* gamma_host, double* alpha_host, double* resid_host,
                  int32_t* m_k_host);
/* p_out = G_k - sum gamma_i dG_i (beta == 1) or the alpha blend
 * (anderson.py:126-148). gamma/alpha from sg_aa_weights (host). */
int sg_aa_step(sg_aa* a, double beta, const double* gamma_host, const double* alpha_host,
               void* p_out_dev);
/* ||f_k||_2 (anderson.py:329) */
int sg_aa_fk_norm(sg_aa* a, double* out_host);
/* QR policy: 0 = Gram with the device-QR fallback (default), 1 = always the
 * device QR (SlidingQR semantics for every window). */
int sg_aa_set_qr(sg_aa* a, int32_t mode);
/* Whether the current window's R came from the device QR; QR passes run. */
int sg_aa_qr_info(sg_aa* a, int32_t* active_host, int64_t* passes_host);

/* Device vector helpers for the optimizer loop (anderson.py:322, :362-370):
 *  sg_vec_axpby      : z = a x + b y  (a == 1: z = x + b y, i.e. p - eta g)
 *  sg_vec_lerp       : z = x + lam (y - x)            (blend candidate, :369)
 *  sg_vec_blend_dots : out = {<g, pbar - p>, <g, ptil - pbar>}  (:363-364)
 *  sg_vec_stats      : out = {min, max, max|x|, ||x||_2, nonfinite count}
 * All device pointers of `dtype`, length n, fp64 accumulation. */
int sg_vec_axpby(int64_t n, int32_t dtype, double a, const void* x, double b, const void* y,
                 void* z, void* cuda_stream);
int sg_vec_lerp(int64_t n, int32_t dtype, const void* x, const void* y, double lam, void* z,
                void* cuda_stream);
int sg_vec_blend_dots(int64_t n, int32_t dtype, const void* g, const void* p,
                      const void* pbar, const void* ptil, double* out_host,
                      void* cuda_stream);
int sg_vec_stats(int64_t n, int32_t dtype, const void* x, double* out_host,
                 void* cuda_stream);

/* Krylov / quasi-Newton vector kernels (seisopt/krylov.py:130-190 Arnoldi
 * projections and updates, seisopt/optim/quasi_newton.py:36-55 two-loop
 * recursion), one pass over k <= 32 device vectors of `dtype`, length n;
 * xs is a HOST array of k device pointers.
 *  sg_vec_multi_dot  : out_host[i] = <x_i, y> (i < k), out_host[k] = <y, y>
 *                      (fp64 accumulation, fixed-order block sums)
 *  sg_vec_multi_axpy : z = y + sum_i coef_host[i] x_i (y may be NULL: z = sum),
 *                      fp64 per element; z may alias y or one of the x_i */
int sg_vec_multi_dot(int64_t n, int32_t dtype, int32_t k, const void* const* xs,
                     const void* y, double* out_host, void* cuda_stream);
int sg_vec_multi_axpy(int64_t n, int32_t dtype, int32_t k, const double* coef_host,
                      const void* const* xs, const void* y, void* z, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif /* SEISGPU_H */
