/*
 * vpetabc.h -- C ABI of libvpetabc.so, the B200 (sm_100a) implementation of the
 * data-parallel hot path of vPET-ABC (arxiv 2603.14859): voxelwise rejection ABC.
 *
 * Citation key: P:n = line n of the paper's LaTeX source, with the
 * equation / algorithm label; S:n = SPEC.md line n; DESIGN.md Rk = reading k.
 *
 * What one call of abc_run_voxels computes (Alg. 1 "Vectorized Voxelwise Rejection
 * ABC"):
 *   line 1-2  draws i = 0..N-1 of (model m_i, theta_i) from the priors
 *   line 3    model curves s_i = frame averages of the model TAC
 *   line 4    D_ji = rho(y_j, s_i) for every voxel j
 *   line 5    per voxel the n smallest D_ji (top-n) or
 *             every draw with D_ji <= eps
 *   then      posterior summaries: model probabilities, the
 *             preferred model (>50 %), conditional mean / SD / quantiles
 *              and K_i = K1 k3/(k2+k3).
 * Results equal those of the FP64 CPU oracle (oracle/) on the same inputs: the
 * GPU ranks draws with an FP32 pass whose error is bounded, then re-scores every
 * candidate near the acceptance boundary in FP64 exactly as the oracle does
 * (DESIGN.md "Exactness").
 *
 * Conventions
 *   Ownership:  every input is caller-owned and copied (or only read) during the
 *               call; outputs are caller-allocated; the context is library-owned
 *               and released by abc_destroy.
 *   Errors:     status codes only; nothing is thrown and nothing exits across the
 *               ABI.  abc_last_error(ctx) describes the last failure on ctx and is
 *               valid until the next call on ctx.
 *   Threading:  a context is bound to one device and is not re-entrant; use one
 *               context per device / host thread.
 *   State:      abc_init -> {abc_set_input_function, abc_set_frames} (any order,
 *               repeatable) -> abc_run_voxels* ; running before both are set gives
 *               ABC_E_STATE.
 *   Units:      time in minutes, rates in 1/min, activity in any consistent unit.
 *   Multi-GPU:  the ABI is per device; voxel sharding and NCCL live above it
 *               (paper_2603_14859_b200/distributed.py).
 */
#ifndef VPETABC_H
#define VPETABC_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define VPETABC_ABI_VERSION 2  /* 2: abc_stats.n_fallback_exact, abc_reduce_accepted, n <= 15360 */
#define ABC_MAX_P 8       /* parameter columns per draw (2TCM family uses 5, RT family 7) */
#define ABC_MAX_MODELS 4  /* M */
#define ABC_MAX_L 128     /* frames per TAC */

typedef enum {
  ABC_OK = 0,
  ABC_E_ARG = 1,          /* invalid argument (see each function) */
  ABC_E_STATE = 2,        /* input function or frames not set */
  ABC_E_NOMEM = 3,        /* device memory for this call exceeds what is free; nothing allocated */
  ABC_E_CUDA = 4,         /* a CUDA runtime error; abc_last_error has the CUDA message */
  ABC_E_UNSUPPORTED = 5   /* valid request outside what this build supports */
} abc_status;

/* Forward models.  Parameter columns:
 *   2TCM family:  [K1, k2, k3, k4, Vb]            -- IRR forces k4 = 0
 *   RT family:  [R1, k2, k2a, gamma, tD, tP, alpha]
 *                            -- MRTM forces gamma = 0; tD, tP, alpha do not exist
 *                               for MRTM (their summaries are NaN).  Column 5 is drawn as
 *                               the offset tP - tD ~ U(lo[5], hi[5]) and reported as
 *                               tP = tD + offset (R8).
 * All models of one context must be of the same family. */
typedef enum { ABC_2TCM_IRR = 0, ABC_2TCM_REV = 1, ABC_MRTM = 2, ABC_LPNTPET = 3 } abc_model_kind;

/* Discrepancy (Alg.1 l.4): WL2: D = sum_f w_f (y_f - s_f)^2 (north star);
 * L1: D = sum_f w_f |y_f - s_f|.  Exactly the oracle's FP64 value. */
typedef enum { ABC_DIST_L1 = 1, ABC_DIST_WL2 = 2 } abc_distance;

/* Acceptance: TOPN keeps the n smallest by (D, draw index) (ties -> lower
 * index); EPS keeps every draw with D <= epsilon. */
typedef enum { ABC_ACCEPT_TOPN = 0, ABC_ACCEPT_EPS = 1 } abc_accept;

/* Input function.  PWL: knots (t_k, c_k), t_0 = 0, t strictly increasing, linear in
 * between, held at c_last after the last knot (IDIF "frame-wise mean"; R1).
 * FENG: value[6] = (beta1, beta2, beta3, kappa1, kappa2, kappa3) of P:204-207, kappas > 0.
 * 2TCM: the input is the plasma curve C_p (= C_wb).  RT models: the input is the
 * reference-region TAC C_r and must be PWL. */
typedef enum { ABC_INPUT_PWL = 0, ABC_INPUT_FENG = 1 } abc_input_kind;

/* abc_config.flags */
#define ABC_FLAG_TIMING 0x1u     /* record per-stage CUDA-event times (abc_get_stats) */
#define ABC_FLAG_EXACT 0x2u      /* skip the FP32 pass: exact FP64 scan for every voxel (slow) */
#define ABC_FLAG_COUNT_WORK 0x4u /* count executed frame updates of the FP32 pass */
#define ABC_FLAG_NO_PRUNE 0x8u   /* FP32 pass evaluates all frames of every pair (A/B only) */
#define ABC_FLAG_NO_REORDER 0x10u/* FP32 pass keeps the acquisition frame order (A/B only) */
#define ABC_FLAG_NO_TREE 0x20u   /* FP32 pass scans every draw in index order, no bounds (A/B only) */
#define ABC_FLAG_DENSE_TC 0x40u  /* replace the FP32 pass by the dense shared-bank tensor-core
                                    distance (y.s cross term on tcgen05, BF16x3 split; WL2, TOPN,
                                    L <= 48, n <= 2032, else ABC_E_UNSUPPORTED).  Same certified results;
                                    evaluates every pair (SURVEY.md §8f-1, A/B comparison) */
#define ABC_FLAG_FORCE_FALLBACK 0x80u /* test hook: certification rejects every voxel, so every
                                    voxel takes the uncertified-voxel path (seeded FP64 collector,
                                    DESIGN.md §3); results must be unchanged */

/* abc_run_voxels ptr_flags */
#define ABC_PTR_TACS_DEVICE 0x1u /* tacs is a device pointer on ctx's device */
#define ABC_PTR_OUT_DEVICE 0x2u  /* every abc_result array is a device pointer */

typedef struct abc_model_spec {
  int32_t kind;           /* abc_model_kind */
  uint32_t reserved0;     /* must be 0 */
  uint64_t n_draws;       /* N_m >= 1: this model owns the contiguous draw-index block
                             [sum_{k<m} N_k, sum_{k<=m} N_k)  (Alg.1 l.1; R7) */
  float lo[ABC_MAX_P];    /* uniform prior U(lo, hi) per column; lo == hi fixes the column */
  float hi[ABC_MAX_P];
} abc_model_spec;

typedef struct abc_config {
  uint32_t struct_size;   /* = sizeof(abc_config) (376) */
  uint32_t n_models;      /* M, 1..ABC_MAX_MODELS */
  uint64_t seed;          /* Philox4x32-10 key (R7) */
  int32_t device;         /* CUDA device ordinal */
  int32_t distance;       /* abc_distance */
  int32_t accept;         /* abc_accept */
  uint32_t n_accept;      /* n for TOPN: 1 <= n <= N, n <= 15360 (n = floor(N p)) */
  double epsilon;         /* tolerance h for EPS, >= 0 */
  double lpnt_step_min;   /* lp-ntPET integrator step delta (min); <= 0 selects 0.05 */
  uint32_t flags;         /* ABC_FLAG_* */
  uint32_t reserved1;     /* must be 0 */
  abc_model_spec model[ABC_MAX_MODELS];
} abc_config;

/* Caller-allocated outputs (row-major).  A NULL pointer means "not produced".
 * P = 5 for the 2TCM family, 7 for the RT family; M = n_models. */
typedef struct abc_result {
  float* prob;          /* J x M   count_m / n_acc (NaN if nothing accepted)             */
  int32_t* preferred;   /* J       argmax_m count_m, ties -> lowest m (= the >50 % rule of
                                   P:282 for M = 2 with model 0 the simpler model); -1 if none */
  uint32_t* count;      /* J x M   accepted draws per model                                */
  float* mean;          /* J x P   mean of each column over the accepted draws of the
                                   preferred model; NaN if the column does not exist */
  float* sd;            /* J x P   SD, ddof = 1 (NaN if < 2 draws)                          */
  float* q;             /* J x P x 3  type-7 quantiles at 2.5/50/97.5 % (TOPN only, else NaN) */
  float* ki_mean;       /* J       K_i = K1 k3/(k2+k3) per accepted draw (2TCM only)  */
  float* ki_sd;         /* J                                                                 */
  float* ki_q;          /* J x 3   (TOPN only)                                               */
  uint64_t* acc_idx;    /* J x n   accepted draw indices sorted by (D, index) (TOPN only)    */
  double* acc_dist;     /* J x n   their FP64 discrepancies (TOPN only)                      */
} abc_result;

/* Per-call statistics of the last abc_run_voxels on ctx (times need ABC_FLAG_TIMING). */
typedef struct abc_stats {
  uint32_t struct_size;       /* = sizeof(abc_stats) */
  uint32_t gpu_launches;      /* kernels launched by the last run */
  uint64_t n_voxels;
  uint64_t n_draws;
  uint64_t n_fallback;        /* voxels whose FP32 pass could not be certified (re-run exactly) */
  uint64_t n_fallback_exact;  /* of these, voxels re-run by the exact heap scan (the others by the
                                 seeded GPU-wide collector) */
  uint64_t frame_updates;     /* executed FP32 frame updates of draw evaluations (ABC_FLAG_COUNT_WORK) */
  uint64_t bound_updates;     /* executed FP32 frame updates of (super-)tile lower bounds (idem) */
  uint32_t lp;                /* padded frame count of the FP32 pass */
  uint32_t heap_k;            /* candidates kept per voxel by the FP32 pass */
  double ms_h2d, ms_bank, ms_order, ms_scan, ms_certify, ms_fallback, ms_d2h, ms_total;
} abc_stats;

typedef struct abc_ctx abc_ctx; /* opaque, library-owned */

/* Create a context on cfg->device.  ABC_E_ARG: struct_size mismatch, M out of range,
 * mixed model families, N_m = 0, N = sum N_m >= 2^32, lo > hi or non-finite bounds,
 * 2TCM with lo[k3] <= 0 (R3), unknown distance/accept, TOPN with n = 0,
 * n > N or n > 15360, EPS with epsilon < 0 or NaN, reserved fields != 0.
 * ABC_E_CUDA: the device cannot be selected.  *out is NULL on failure. */
abc_status abc_init(const abc_config* cfg, abc_ctx** out);

/* Set the input function (host arrays, copied).  kind = ABC_INPUT_PWL: t_min[n], value[n],
 * n >= 1, t_min[0] == 0, strictly increasing, finite.  kind = ABC_INPUT_FENG: value[6]
 * (t_min ignored, n == 6), finite, kappas > 0; ABC_E_UNSUPPORTED for RT models. */
abc_status abc_set_input_function(abc_ctx* ctx, int32_t kind, const double* t_min,
                                  const double* value, uint32_t n);

/* Set the frame schedule (host arrays, copied): L frames [start, start + dur), start >= 0,
 * dur > 0, non-overlapping and increasing (start[f+1] >= start[f] + dur[f]), 1 <= L <= 128.
 * weight (FP32, > 0, finite) may be NULL for w = 1 (R6). */
abc_status abc_set_frames(abc_ctx* ctx, const double* start_min, const double* dur_min,
                          const float* weight, uint32_t L);

/* Run Alg. 1 for J voxels.  tacs: J x L FP32 row-major (frame-contiguous per voxel), host
 * or device per ptr_flags; negative values allowed.  Non-finite values -> ABC_E_ARG: the
 * kernels that follow the on-device finite check skip their work (the call returns in about
 * the time of the bank stage) and the output arrays are left unspecified.
 * J = 0 is a no-op.  The work is ordered on the context's stream (abc_set_stream); the call
 * returns after the results are complete, for host and device outputs alike (it ends with a
 * synchronisation of that stream, which also reads the status flags of the run).
 * ABC_E_NOMEM if the bank (2 x N x L FP32), the per-voxel state and the staging buffers
 * do not fit in free device memory (checked before allocating).  ABC_E_UNSUPPORTED if a
 * kernel's shared-memory need exceeds the device's opt-in maximum. */
abc_status abc_run_voxels(abc_ctx* ctx, const float* tacs, uint64_t J, uint32_t ptr_flags,
                          abc_result* out);

/* Model selection only: prob (J x M) and preferred (J). */
abc_status abc_model_select(abc_ctx* ctx, const float* tacs, uint64_t J, uint32_t ptr_flags,
                            float* prob, int32_t* preferred);

/* Order the context's work on a caller stream (a cudaStream_t; NULL = the library's own
 * stream).  The stream must belong to ctx's device and outlive its use. */
abc_status abc_set_stream(abc_ctx* ctx, void* cuda_stream);

/* Block until the context's stream is idle. */
abc_status abc_sync(abc_ctx* ctx);

/* Copy the statistics of the last run (stats->struct_size must be set). */
abc_status abc_get_stats(const abc_ctx* ctx, abc_stats* stats);

/* Copy rows [first, first + count) of the simulation bank of the last run (Alg.1 l.3, the
 * N x L matrix X of P:150, FP32, acquisition frame order) to host memory out[count * L].
 * ABC_E_STATE before the first run; ABC_E_ARG if the rows are out of range. */
abc_status abc_get_bank(const abc_ctx* ctx, float* out, uint64_t first, uint64_t count);

/* Patlak K_i map (the clinical reference K_i image of P:282; Patlak 1983; SURVEY.md §8f-4;
 * DESIGN.md R18).  For each voxel, the least-squares line z = K_i x + V0 through the frames
 * whose mid-time t_f >= t_star_min, with x_f = (int_0^{t_f} C_in) / Cp_f, z_f = y_f / Cp_f and
 * Cp_f the frame average of the context's input function (FP64).  tacs: J x L FP32 (host, or
 * device with ABC_PTR_TACS_DEVICE); ki, intercept (may be NULL): J FP32 (host, or device with
 * ABC_PTR_OUT_DEVICE).  NaN when fewer than two frames qualify.  ABC_E_STATE before the input
 * function and frames are set; ABC_E_ARG for NULL tacs/ki or a non-finite t_star_min.  Blocks until
 * the outputs are complete. */
abc_status abc_patlak(abc_ctx* ctx, const float* tacs, uint64_t J, double t_star_min, uint32_t ptr_flags,
                      float* ki, float* intercept);

/* Simulated-draw noise (the P:218-220 observation model applied to the draws, as
 * SPEC S:301 does; R17).  From the next run on, each bank value becomes
 *   s_if = RN32(v_f + ell sigma_f z_if),  sigma_f = sqrt(max(v_f, 0) e^{-lambda t_f} / dt_f) e^{lambda t_f},
 * v_f the FP64 frame average, t_f the frame mid-time, lambda = ln 2 / half_life_min, and z_if a
 * standard normal from Box-Muller on Philox4x32-10(ctr = {i_lo, i_hi, 2 + f/2, 'VPET'}, key = seed)
 * (words x0..x3: ua = u53(x0, x1), ub = u53(x2, x3), u53(a, b) = ((a:b) >> 11 + 1/2) 2^-53;
 * z = sqrt(-2 ln ua) cos(2 pi ub) for even f, sin(2 pi ub) for odd f).  ell = 0 (the default)
 * is the noise-free method.  ABC_E_ARG: ell < 0 or non-finite, half_life_min <= 0 or NaN
 * (+inf = no decay correction). */
abc_status abc_set_sim_noise(abc_ctx* ctx, double ell, double half_life_min);

/* Response-function 95 % credible envelope (Fig. 1).  For voxel j
 * and time t_min[k]: the type-7 2.5/50/97.5 % quantiles, over the voxel's accepted draws of an
 * lp-ntPET model, of the response function
 *     r(t) = k2a(t)/k2a = 1 + (gamma/k2a) g(t; tD, tP, alpha)      (eq:Bt P:90-94)
 * with g the peak-normalised gamma variate (R4), in FP64 from the FP32 draws.  Draws of
 * other models are skipped (R16); a voxel without lp-ntPET draws gets NaN.
 * acc_idx: J x n_acc draw indices (e.g. abc_result.acc_idx of a TOPN run); host, or device if
 * ptr_flags has ABC_PTR_TACS_DEVICE.  t_min: T times (host, finite).  q: J x T x 3 FP32,
 * caller-allocated; host, or device if ptr_flags has ABC_PTR_OUT_DEVICE.  1 <= n_acc <= 4096,
 * 1 <= T <= 1024, else ABC_E_ARG; ABC_E_ARG also for an index >= N (detected on device, after
 * the work).  ABC_E_UNSUPPORTED if ctx has no lp-ntPET model.  Blocks until q is complete. */
abc_status abc_response_envelope(abc_ctx* ctx, const uint64_t* acc_idx, uint64_t J, uint32_t n_acc,
                                 const double* t_min, uint32_t T, uint32_t ptr_flags, float* q);

/* Posterior summaries of given accepted lists (the reduction step of P:177-180, P:282 alone;
 * SURVEY.md §8f-3).  For voxel j the first n_use entries of row j of acc_idx (J x n_acc draw
 * indices, row-major) are reduced exactly as abc_run_voxels reduces its accepted set: counts,
 * probabilities, preferred model, conditional mean / SD / type-7 quantiles, K_i.  A top-n row of
 * abc_run_voxels is sorted by (D, index), so its prefix of length n' IS the top-n' accepted set of
 * the same run: one run at the largest n gives every smaller n of a pilot sweep.
 * acc_idx: host, or device with ABC_PTR_TACS_DEVICE.  out: as for abc_run_voxels (host, or device
 * with ABC_PTR_OUT_DEVICE); out->acc_idx (J x n_use) receives the prefix; out->acc_dist must be
 * NULL.  Needs only abc_init (the prior).  ABC_E_ARG: n_use == 0, n_use > n_acc, n_use > 4096,
 * acc_dist != NULL, or an index >= N (detected on device after the work).  Blocks until done. */
abc_status abc_reduce_accepted(abc_ctx* ctx, const uint64_t* acc_idx, uint64_t J, uint32_t n_acc, uint32_t n_use,
                               uint32_t ptr_flags, abc_result* out);

const char* abc_last_error(const abc_ctx* ctx);
void abc_destroy(abc_ctx* ctx);
uint32_t abc_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* VPETABC_H */
