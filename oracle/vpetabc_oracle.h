/*
 * vpetabc_oracle.h -- CPU ORACLE for the vPET-ABC hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This library is the plain, slow, obviously-correct FP64 definition of what the
 * GPU path computes.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It shares NO code, header,
 * helper or table generator with the CUDA library under paper_2603_14859_b200/.
 *
 * Citation key: P:n = PAPER.md line n (arxiv 2603.14859 LaTeX source);
 *               S:n = SPEC.md line n; SURVEY §8c = the readings adopted in DESIGN.md.
 *
 * It exports the same C entry points as the product ABI (abc_init, ...,
 * abc_run_voxels, abc_model_select) so that the same driver can run either, plus
 * oracle_* entry points used by the pin tests.  Host pointers only.
 *
 * Parity-pinned functions (tests/test_oracle_pins.py):
 *   philox KATs, uniform mapping, 2TCM (PWL + Feng) vs ODE/quadrature, step-input
 *   closed form, K1=0 limit, Patlak slope, MRTM == lp-ntPET(gamma=0), gamma
 *   variate examples, distance examples, top-n vs brute force, eps->inf prior
 *   moments, eps->0 concentration, reduction examples.
 * Parity unpinned: lp-ntPET (gamma>0) against the true ODE solution beyond grid
 *   refinement and the S:93 integral-identity residual (no closed form exists).
 */
#ifndef VPETABC_ORACLE_H
#define VPETABC_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define ABC_MAX_P 8
#define ABC_MAX_MODELS 4
#define ABC_MAX_L 128

typedef enum { ABC_OK = 0, ABC_E_ARG = 1, ABC_E_STATE = 2, ABC_E_NOMEM = 3,
               ABC_E_CUDA = 4, ABC_E_UNSUPPORTED = 5 } abc_status;
typedef enum { ABC_2TCM_IRR = 0, ABC_2TCM_REV = 1, ABC_MRTM = 2, ABC_LPNTPET = 3 } abc_model_kind;
typedef enum { ABC_DIST_L1 = 1, ABC_DIST_WL2 = 2 } abc_distance;
typedef enum { ABC_ACCEPT_TOPN = 0, ABC_ACCEPT_EPS = 1 } abc_accept;
typedef enum { ABC_INPUT_PWL = 0, ABC_INPUT_FENG = 1 } abc_input_kind;

typedef struct abc_model_spec {
  int32_t kind;          /* abc_model_kind */
  uint32_t reserved0;
  uint64_t n_draws;      /* N_m: contiguous index block of the draws of this model */
  float lo[ABC_MAX_P];   /* uniform prior bounds per parameter column */
  float hi[ABC_MAX_P];
} abc_model_spec;

typedef struct abc_config {
  uint32_t struct_size;
  uint32_t n_models;
  uint64_t seed;
  int32_t device;
  int32_t distance;
  int32_t accept;
  uint32_t n_accept;
  double epsilon;
  double lpnt_step_min;
  uint32_t flags;
  uint32_t reserved1;
  abc_model_spec model[ABC_MAX_MODELS];
} abc_config;

typedef struct abc_result {
  float* prob;        /* J x M */
  int32_t* preferred; /* J */
  uint32_t* count;    /* J x M */
  float* mean;        /* J x P */
  float* sd;          /* J x P */
  float* q;           /* J x P x 3 */
  float* ki_mean;     /* J */
  float* ki_sd;       /* J */
  float* ki_q;        /* J x 3 */
  uint64_t* acc_idx;  /* J x n (top-n only) */
  double* acc_dist;   /* J x n (top-n only) */
} abc_result;

typedef struct abc_ctx abc_ctx;

abc_status abc_init(const abc_config* cfg, abc_ctx** out);
abc_status abc_set_input_function(abc_ctx* ctx, int32_t kind, const double* t_min,
                                  const double* value, uint32_t n);
abc_status abc_set_frames(abc_ctx* ctx, const double* start_min, const double* dur_min,
                          const float* weight, uint32_t L);
abc_status abc_run_voxels(abc_ctx* ctx, const float* tacs, uint64_t J, uint32_t ptr_flags,
                          abc_result* out);
abc_status abc_model_select(abc_ctx* ctx, const float* tacs, uint64_t J, uint32_t ptr_flags,
                            float* prob, int32_t* preferred);
/* Response-function 95 % CrI envelope (Fig. 1): J x T x 3 quantiles of
 * 1 + gamma/k2a g(t) over each voxel's accepted lp-ntPET draws (host pointers only). */
/* Simulated-draw noise (P:218-220 model on the draws): ell = 0 disables. */
abc_status abc_set_sim_noise(abc_ctx* ctx, double ell, double half_life_min);
/* the standard normal z_if of draw i, frame f (Box-Muller on Philox; see abc_set_sim_noise) */
double oracle_std_normal(uint64_t seed, uint64_t i, uint32_t f);
/* Patlak K_i and intercept per voxel from the frames with mid-time >= t_star (R18). */
abc_status abc_patlak(abc_ctx* ctx, const float* tacs, uint64_t J, double t_star_min, uint32_t ptr_flags,
                      float* ki, float* intercept);
abc_status abc_response_envelope(abc_ctx* ctx, const uint64_t* acc_idx, uint64_t J, uint32_t n_acc,
                                 const double* t_min, uint32_t T, uint32_t ptr_flags, float* q);
const char* abc_last_error(const abc_ctx* ctx);
void abc_destroy(abc_ctx* ctx);

/* ---- oracle-only entry points (pins) ---- */
void oracle_set_threads(int n);
int oracle_get_threads(void);
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
float oracle_uniform(uint32_t x);
/* draw i of the configured prior: model index, parameter columns (P_family of them) */
abc_status oracle_draw(const abc_ctx* ctx, uint64_t i, int32_t* model, float* theta);
/* FP64 frame averages (before RN32) of model `kind` at theta, on ctx's input and frames */
abc_status oracle_simulate(const abc_ctx* ctx, int32_t kind, const float* theta, double* value);
/* RN32 bank: N x L floats, row i = draw i */
abc_status oracle_bank(const abc_ctx* ctx, float* bank);
double oracle_distance(int32_t dist, const float* y, const float* s, const float* w, uint32_t L);
double oracle_gamma_variate(double tD, double tP, double alpha, double t);
double oracle_feng(const double* bk, double t);
double oracle_quantile7(const double* sorted_x, uint32_t n, double q);
uint32_t oracle_family_width(int32_t kind);

#ifdef __cplusplus
}
#endif
#endif
