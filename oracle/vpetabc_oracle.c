/*
 * vpetabc_oracle.c -- plain FP64 CPU ORACLE of voxelwise rejection ABC (vPET-ABC).
 *
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py.  Never by the product path.
 * Shares no code with paper_2603_14859_b200/csrc (the CUDA library).
 *
 * What it computes, step by step, in the order of Alg. 1:
 *   1. prior draw (Alg.1 l.1-2; priors eq:prior2 P:272-277):
 *        Philox4x32-10 counter-based uniforms -> theta (FP32, fmaf)
 *   2. model curve (Alg.1 l.3): FP64 frame averages of the model TAC,
 *        2TCM eq:2TCM/eq:2TCM_op as the bi-exponential impulse response
 *        convolved with the input (Feng P:204-207 closed form, or a piecewise-linear
 *        IDIF P:269 by exact recurrences); MRTM / lp-ntPET eq:lp-ntPET, eq:Bt;
 *        then rounded to FP32 (the method's FP32 TAC).
 *   3. discrepancy (Alg.1 l.4): D = sum_f w_f (y_f - s_f)^2 (weighted L2,
 *        north star) or sum_f w_f |y_f - s_f| (L1), in FP64.
 *   4. acceptance (Alg.1 l.5): full sort by (D, index), keep
 *        the first n; or eps mode {i : D_i <= eps}.
 *   5. posterior reduction: per-model counts and
 *        probabilities, preferred model (>50 %, tie -> model 0), conditional mean,
 *        SD (ddof=1), type-7 quantiles, K_i = K1 k3/(k2+k3) per accepted draw.
 * Paper-silent points follow the readings listed in DESIGN.md ("Readings").
 * Compile with -ffp-contract=off: every FP64 operation below is rounded as written.
 */
#include "vpetabc_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u
#define CTR_TAG 0x56504554u /* "VPET" */

struct abc_ctx {
  abc_config cfg;
  int have_input, have_frames;
  int32_t input_kind;
  double feng[6];
  double* kt; /* input knots (PWL) */
  double* kc;
  uint32_t nk;
  uint32_t L;
  double* fs; /* frame start */
  double* fd; /* frame duration */
  float* w;   /* weights (1 if NULL given) */
  int prepared;      /* draw-independent grids below are valid */
  struct grid_s* gc; /* coarse grid: input knots U frame bounds */
  struct grid_s* gf; /* fine grid (lp-ntPET): {k delta} U knots U frame bounds */
  double noise_ell, noise_lam; /* simulated-draw noise (abc_set_sim_noise); ell = 0: none */
  char err[256];
};

static int g_threads = 0;
void oracle_set_threads(int n) { g_threads = n; }
int oracle_get_threads(void) {
#ifdef _OPENMP
  return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
  return 1;
#endif
}

static abc_status fail(abc_ctx* c, abc_status s, const char* msg) {
  if (c) snprintf(c->err, sizeof c->err, "%s", msg);
  return s;
}

/* ------------------------------------------------------------------------- */
/* 1. Prior draw.  Philox4x32-10 (Salmon et al., SC'11), 10 rounds.           */
/* ------------------------------------------------------------------------- */
void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int r = 0; r < 10; ++r) {
    if (r > 0) { k0 += PHILOX_W0; k1 += PHILOX_W1; }
    uint64_t p0 = (uint64_t)PHILOX_M0 * (uint64_t)c0;
    uint64_t p1 = (uint64_t)PHILOX_M1 * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* u = (2*(x>>9)+1) * 2^-24, exactly representable, strictly inside (0,1). */
float oracle_uniform(uint32_t x) {
  uint32_t m = ((x >> 9) << 1) | 1u;
  return (float)m * (1.0f / 16777216.0f);
}

uint32_t oracle_family_width(int32_t kind) {
  return (kind == ABC_MRTM || kind == ABC_LPNTPET) ? 7u : 5u;
}

static uint64_t total_draws(const abc_config* c) {
  uint64_t n = 0;
  for (uint32_t m = 0; m < c->n_models; ++m) n += c->model[m].n_draws;
  return n;
}

/* Alg.1 l.1: model indicator.  Reading: stratified contiguous blocks of N_m draws. */
static int32_t model_of(const abc_config* c, uint64_t i) {
  uint64_t off = 0;
  for (uint32_t m = 0; m < c->n_models; ++m) {
    off += c->model[m].n_draws;
    if (i < off) return (int32_t)m;
  }
  return -1;
}

/* Alg.1 l.2: theta_k = fmaf(hi_k - lo_k, u_k, lo_k); u_k from Philox block k/4, word k%4.
 * IRR: k4 := 0.  MRTM: gamma := 0.  lp-ntPET/MRTM: column 5 is drawn as the
 * offset tP - tD and reported as tP = tD + offset (FP32 add) (reading). */
static void draw_theta(const abc_config* c, uint64_t i, int32_t* model, float* th) {
  int32_t m = model_of(c, i);
  *model = m;
  const abc_model_spec* ms = &c->model[m];
  uint32_t P = oracle_family_width(ms->kind);
  uint32_t key[2] = {(uint32_t)c->seed, (uint32_t)(c->seed >> 32)};
  uint32_t r[8];
  for (uint32_t b = 0; b < 2; ++b) {
    uint32_t ctr[4] = {(uint32_t)i, (uint32_t)(i >> 32), b, CTR_TAG};
    oracle_philox4x32_10(ctr, key, r + 4 * b);
  }
  for (uint32_t k = 0; k < ABC_MAX_P; ++k) th[k] = 0.0f;
  for (uint32_t k = 0; k < P; ++k) {
    float u = oracle_uniform(r[k]);
    float span = ms->hi[k] - ms->lo[k];
    th[k] = fmaf(span, u, ms->lo[k]);
  }
  if (ms->kind == ABC_2TCM_IRR) th[3] = 0.0f;
  if (ms->kind == ABC_MRTM) th[3] = 0.0f;
  if (ms->kind == ABC_MRTM || ms->kind == ABC_LPNTPET) th[5] = th[4] + th[5];
}

abc_status oracle_draw(const abc_ctx* ctx, uint64_t i, int32_t* model, float* theta) {
  if (!ctx || i >= total_draws(&ctx->cfg)) return ABC_E_ARG;
  draw_theta(&ctx->cfg, i, model, theta);
  return ABC_OK;
}

/* ------------------------------------------------------------------------- */
/* 2. Forward model.  phi-functions of the exact exponential integrals.       */
/*   phi1(x) = (1-e^-x)/x, psi(x) = (x-1+e^-x)/x^2,                            */
/*   chi(x) = phi1 - psi = (1-e^-x(1+x))/x^2, omega(x) = (x^2/2-1+e^-x(1+x))/x^3 */
/*   Series below x = 0.5:  phi1 = sum (-x)^k/(k+1)!, psi = sum (-x)^k/(k+2)!,   */
/*   chi = sum (-x)^k (k+1)/(k+2)!, omega = sum (-x)^k (k+2)/(k+3)!.            */
/* ------------------------------------------------------------------------- */
#define SERIES_CUT 0.5
#define SERIES_TERMS 24

static double fact(int n) {
  double f = 1.0;
  for (int i = 2; i <= n; ++i) f *= (double)i;
  return f;
}
static double phi1(double x) {
  if (x < SERIES_CUT) {
    double s = 0.0, p = 1.0;
    for (int k = 0; k < SERIES_TERMS; ++k) { s += p / fact(k + 1); p *= -x; }
    return s;
  }
  return -expm1(-x) / x;
}
static double psi(double x) {
  if (x < SERIES_CUT) {
    double s = 0.0, p = 1.0;
    for (int k = 0; k < SERIES_TERMS; ++k) { s += p / fact(k + 2); p *= -x; }
    return s;
  }
  return (x - 1.0 + exp(-x)) / (x * x);
}
static double chi(double x) {
  if (x < SERIES_CUT) {
    double s = 0.0, p = 1.0;
    for (int k = 0; k < SERIES_TERMS; ++k) { s += p * (double)(k + 1) / fact(k + 2); p *= -x; }
    return s;
  }
  return (-expm1(-x) - x * exp(-x)) / (x * x);
}
static double omega(double x) {
  if (x < SERIES_CUT) {
    double s = 0.0, p = 1.0;
    for (int k = 0; k < SERIES_TERMS; ++k) { s += p * (double)(k + 2) / fact(k + 3); p *= -x; }
    return s;
  }
  return (0.5 * x * x - 1.0 + exp(-x) * (1.0 + x)) / (x * x * x);
}

/* --- Piecewise-linear input on an augmented grid (input knots U frame bounds) --- */
typedef struct grid_s { double* t; double* c; int* seg_frame; uint32_t n; } grid_t;

static double pwl_value(const double* kt, const double* kc, uint32_t nk, double t) {
  /* linear interpolation through the knots; beyond the last knot hold the last value */
  if (t >= kt[nk - 1]) return kc[nk - 1];
  for (uint32_t k = 0; k + 1 < nk; ++k) {
    if (t >= kt[k] && t <= kt[k + 1]) {
      if (t == kt[k]) return kc[k];
      if (t == kt[k + 1]) return kc[k + 1];
      double a = (t - kt[k]) / (kt[k + 1] - kt[k]);
      return kc[k] + (kc[k + 1] - kc[k]) * a;
    }
  }
  return kc[nk - 1];
}

static int cmp_double(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* Frame of the segment [t0,t1] (fully inside one frame) or -1 (gap). */
static int frame_of_segment(const abc_ctx* c, double t0, double t1) {
  for (uint32_t f = 0; f < c->L; ++f)
    if (t0 >= c->fs[f] && t1 <= c->fs[f] + c->fd[f]) return (int)f;
  return -1;
}

/* sorted union of `extra` time points and {0, frame starts, frame ends}, deduplicated */
static grid_t make_grid(const abc_ctx* c, const double* extra, uint32_t n_extra) {
  uint32_t cap = n_extra + 2 * c->L + 1;
  double* t = (double*)malloc(sizeof(double) * cap);
  uint32_t n = 0;
  double tend = c->fs[c->L - 1] + c->fd[c->L - 1];
  t[n++] = 0.0;
  for (uint32_t i = 0; i < n_extra; ++i)
    if (extra[i] <= tend) t[n++] = extra[i];
  for (uint32_t f = 0; f < c->L; ++f) { t[n++] = c->fs[f]; t[n++] = c->fs[f] + c->fd[f]; }
  qsort(t, n, sizeof(double), cmp_double);
  uint32_t m = 0;
  for (uint32_t i = 0; i < n; ++i)
    if (m == 0 || t[i] != t[m - 1]) t[m++] = t[i];
  grid_t g;
  g.t = t;
  g.n = m;
  g.c = (double*)malloc(sizeof(double) * m);
  for (uint32_t i = 0; i < m; ++i) g.c[i] = pwl_value(c->kt, c->kc, c->nk, t[i]);
  g.seg_frame = (int*)malloc(sizeof(int) * m);
  for (uint32_t i = 0; i + 1 < m; ++i) g.seg_frame[i] = frame_of_segment(c, t[i], t[i + 1]);
  return g;
}
static void free_grid(grid_t* g) { free(g->t); free(g->c); free(g->seg_frame); }


/* S_f(a) = int_frame (C (x) e^{-a.})(t) dt for every frame, for a PWL C on grid g.
 * Exact recurrences for a linear input on each segment [t_k, t_k+h], x = a h:
 *   I_{k+1} = e^{-x} I_k + h [c_k chi(x) + c_{k+1} psi(x)]
 *   int_seg I = h phi1(x) I_k + h^2 [c_{k+1} psi(x) - (c_{k+1}-c_k) omega(x)]   */
static void conv_frame_integrals_pwl(const abc_ctx* c, const grid_t* g, double a, double* S) {
  for (uint32_t f = 0; f < c->L; ++f) S[f] = 0.0;
  double I = 0.0;
  for (uint32_t k = 0; k + 1 < g->n; ++k) {
    double h = g->t[k + 1] - g->t[k];
    double x = a * h;
    double ck = g->c[k], ck1 = g->c[k + 1];
    double seg = h * phi1(x) * I + h * h * (ck1 * psi(x) - (ck1 - ck) * omega(x));
    int f = g->seg_frame[k];
    if (f >= 0) S[f] += seg;
    I = exp(-x) * I + h * (ck * chi(x) + ck1 * psi(x));
  }
}

/* int_frame C dt for the PWL C (trapezoid, exact for PWL) */
static void frame_integrals_pwl(const abc_ctx* c, const grid_t* g, double* A) {
  for (uint32_t f = 0; f < c->L; ++f) A[f] = 0.0;
  for (uint32_t k = 0; k + 1 < g->n; ++k) {
    int f = g->seg_frame[k];
    if (f >= 0) A[f] += 0.5 * (g->t[k + 1] - g->t[k]) * (g->c[k] + g->c[k + 1]);
  }
}

/* --- Feng input: C(t) = (b1 t - b2 - b3) e^{-k1 t} + b2 e^{-k2 t} + b3 e^{-k3 t} --- */
double oracle_feng(const double* bk, double t) {
  return (bk[0] * t - bk[1] - bk[2]) * exp(-bk[3] * t) + bk[1] * exp(-bk[4] * t) +
         bk[2] * exp(-bk[5] * t);
}
/* E(a,k,t) = int_0^t e^{-k u} e^{-a(t-u)} du = t e^{-min(a,k) t} phi1(|a-k| t) */
static double convE(double a, double k, double t) {
  double mn = a < k ? a : k;
  return t * exp(-mn * t) * phi1(fabs(a - k) * t);
}
/* Et(a,k,t) = int_0^t u e^{-k u} e^{-a(t-u)} du
 *   = t^2 e^{-k t} psi((a-k) t)        if a >= k
 *   = t^2 e^{-a t} chi((k-a) t)        if a <  k                                  */
static double convEt(double a, double k, double t) {
  if (a >= k) return t * t * exp(-k * t) * psi((a - k) * t);
  return t * t * exp(-a * t) * chi((k - a) * t);
}
/* G(x) = int_ts^te e^{-x t} dt = e^{-x ts} (te-ts) phi1(x (te-ts)) */
static double Gint(double x, double ts, double te) { return exp(-x * ts) * (te - ts) * phi1(x * (te - ts)); }
/* int_ts^te E dt, from E' = e^{-k t} - a E = e^{-a t} - k E: divide by the larger rate */
static double intE(double a, double k, double ts, double te) {
  double dE = convE(a, k, te) - convE(a, k, ts);
  if (a >= k) return (Gint(k, ts, te) - dE) / a;
  return (Gint(a, ts, te) - dE) / k;
}
/* int_ts^te Et dt, from Et' = E - k Et */
static double intEt(double a, double k, double ts, double te) {
  double dEt = convEt(a, k, te) - convEt(a, k, ts);
  return (intE(a, k, ts, te) - dEt) / k;
}
/* int_frame (C_Feng (x) e^{-a.}) dt */
static double feng_conv_frame(const double* bk, double a, double ts, double te) {
  return bk[0] * intEt(a, bk[3], ts, te) - (bk[1] + bk[2]) * intE(a, bk[3], ts, te) +
         bk[1] * intE(a, bk[4], ts, te) + bk[2] * intE(a, bk[5], ts, te);
}
/* int_frame C_Feng dt; int t e^{-k t} = (ts e^{-k ts} - te e^{-k te})/k + G(k)/k */
static double feng_frame(const double* bk, double ts, double te) {
  double k1 = bk[3];
  double tint = (ts * exp(-k1 * ts) - te * exp(-k1 * te)) / k1 + Gint(k1, ts, te) / k1;
  return bk[0] * tint - (bk[1] + bk[2]) * Gint(k1, ts, te) + bk[1] * Gint(bk[4], ts, te) +
         bk[2] * Gint(bk[5], ts, te);
}

/* 2TCM (eq:2TCM P:69-74, eq:2TCM_op P:75-80, C_wb = C_p P:80).  Impulse response
 * h(t) = K1/(a2-a1) [(k3+k4-a1) e^{-a1 t} + (a2-k3-k4) e^{-a2 t}], with
 * s = k2+k3+k4, r = sqrt(s^2 - 4 k2 k4) written as sqrt((k2-k4)^2 + k3 (k3 + 2(k2+k4))),
 * a2 = (s+r)/2, a1 = 2 k2 k4 / (s+r).
 * value_f = [(1-Vb)(c1 S_f(a1) + c2 S_f(a2)) + Vb int_frame C_p] / dt_f            */
static void sim_2tcm(const abc_ctx* c, const float* th, double* out) {
  double K1 = th[0], k2 = th[1], k3 = th[2], k4 = th[3], Vb = th[4];
  double s = k2 + k3 + k4;
  double r = sqrt((k2 - k4) * (k2 - k4) + k3 * (k3 + 2.0 * (k2 + k4)));
  double a2 = 0.5 * (s + r);
  double a1 = (s + r) > 0.0 ? 2.0 * k2 * k4 / (s + r) : 0.0;
  double c1 = K1 * (k3 + k4 - a1) / (a2 - a1);
  double c2 = K1 * (a2 - k3 - k4) / (a2 - a1);
  uint32_t L = c->L;
  double S1[ABC_MAX_L], S2[ABC_MAX_L], A[ABC_MAX_L];
  if (c->input_kind == ABC_INPUT_FENG) {
    for (uint32_t f = 0; f < L; ++f) {
      double ts = c->fs[f], te = c->fs[f] + c->fd[f];
      S1[f] = feng_conv_frame(c->feng, a1, ts, te);
      S2[f] = feng_conv_frame(c->feng, a2, ts, te);
      A[f] = feng_frame(c->feng, ts, te);
    }
  } else {
    conv_frame_integrals_pwl(c, c->gc, a1, S1);
    conv_frame_integrals_pwl(c, c->gc, a2, S2);
    frame_integrals_pwl(c, c->gc, A);
  }
  for (uint32_t f = 0; f < L; ++f)
    out[f] = ((1.0 - Vb) * (c1 * S1[f] + c2 * S2[f]) + Vb * A[f]) / c->fd[f];
}

/* MRTM (eq:lp-ntPET with gamma = 0): z = C_t - R1 C_r solves
 * z' = (k2 - R1 k2a) C_r - k2a z, z(0) = 0, so
 * value_f = R1 avg_f(C_r) + (k2 - R1 k2a) S_f(k2a) / dt_f                           */
static void sim_mrtm(const abc_ctx* c, const float* th, double* out) {
  double R1 = th[0], k2 = th[1], k2a = th[2];
  double S[ABC_MAX_L], A[ABC_MAX_L];
  conv_frame_integrals_pwl(c, c->gc, k2a, S);
  frame_integrals_pwl(c, c->gc, A);
  for (uint32_t f = 0; f < c->L; ++f) out[f] = (R1 * A[f] + (k2 - R1 * k2a) * S[f]) / c->fd[f];
}

/* gamma variate (eq:Bt), peak-normalised (reading):
 * g = 0 for t <= tD, else x^alpha e^{alpha (1-x)}, x = (t-tD)/(tP-tD)               */
double oracle_gamma_variate(double tD, double tP, double alpha, double t) {
  if (t <= tD) return 0.0;
  double x = (t - tD) / (tP - tD);
  return pow(x, alpha) * exp(alpha * (1.0 - x));
}

/* lp-ntPET (eq:lp-ntPET, eq:Bt).  Differentiated form with z = C_t - R1 C_r:
 *   z' = (k2 - R1 a(t)) C_r - a(t) z,  a(t) = k2a + gamma g(t),  z(0) = 0.
 * Reading: on the grid {k delta} U knots U frame bounds, a(t) is frozen at
 * each substep midpoint (abar) and the forcing f = (k2 - R1 abar) C_r is linear on the
 * substep; the substep is then integrated exactly with the same recurrences as above. */
static void sim_lpntpet(const abc_ctx* c, const float* th, double* out) {
  double R1 = th[0], k2 = th[1], k2a = th[2], gam = th[3], tD = th[4], tP = th[5], al = th[6];
  uint32_t L = c->L;
  const grid_t* gp = c->gf;
  double Z[ABC_MAX_L], A[ABC_MAX_L];
  for (uint32_t f = 0; f < L; ++f) Z[f] = 0.0;
  frame_integrals_pwl(c, gp, A);
  double z = 0.0;
  for (uint32_t k = 0; k + 1 < gp->n; ++k) {
    double t0 = gp->t[k], t1 = gp->t[k + 1], h = t1 - t0;
    double tm = 0.5 * (t0 + t1);
    double abar = k2a + gam * oracle_gamma_variate(tD, tP, al, tm);
    double x = abar * h;
    double fk = (k2 - R1 * abar) * gp->c[k];
    double fk1 = (k2 - R1 * abar) * gp->c[k + 1];
    double seg = h * phi1(x) * z + h * h * (fk1 * psi(x) - (fk1 - fk) * omega(x));
    int f = gp->seg_frame[k];
    if (f >= 0) Z[f] += seg;
    z = exp(-x) * z + h * (fk * chi(x) + fk1 * psi(x));
  }
  for (uint32_t f = 0; f < L; ++f) out[f] = (Z[f] + R1 * A[f]) / c->fd[f];
}

/* Build the draw-independent grids once (not thread safe; called before parallel loops). */
static void unprepare(abc_ctx* c) {
  if (c->gc) { free_grid(c->gc); free(c->gc); c->gc = NULL; }
  if (c->gf) { free_grid(c->gf); free(c->gf); c->gf = NULL; }
  c->prepared = 0;
}
static void prepare(abc_ctx* c) {
  if (c->prepared) return;
  unprepare(c);
  if (c->input_kind == ABC_INPUT_PWL) {
    c->gc = (grid_t*)malloc(sizeof(grid_t));
    *c->gc = make_grid(c, c->kt, c->nk);
    double delta = c->cfg.lpnt_step_min > 0.0 ? c->cfg.lpnt_step_min : 0.05;
    double tend = c->fs[c->L - 1] + c->fd[c->L - 1];
    uint32_t nu = 0;
    while ((double)nu * delta < tend) ++nu;
    uint32_t ne = nu + c->nk;
    double* extra = (double*)malloc(sizeof(double) * ne);
    for (uint32_t k = 0; k < nu; ++k) extra[k] = (double)k * delta;
    for (uint32_t k = 0; k < c->nk; ++k) extra[nu + k] = c->kt[k];
    c->gf = (grid_t*)malloc(sizeof(grid_t));
    *c->gf = make_grid(c, extra, ne);
    free(extra);
  }
  c->prepared = 1;
}

static void simulate(const abc_ctx* c, int32_t kind, const float* th, double* out) {
  switch (kind) {
    case ABC_2TCM_IRR:
    case ABC_2TCM_REV: sim_2tcm(c, th, out); break;
    case ABC_MRTM: sim_mrtm(c, th, out); break;
    default: sim_lpntpet(c, th, out); break;
  }
}

abc_status oracle_simulate(const abc_ctx* ctx, int32_t kind, const float* theta, double* value) {
  if (!ctx || !ctx->have_input || !ctx->have_frames) return ABC_E_STATE;
  int rt = (kind == ABC_MRTM || kind == ABC_LPNTPET);
  if (rt && ctx->input_kind != ABC_INPUT_PWL) return ABC_E_UNSUPPORTED;
  prepare((abc_ctx*)ctx);
  simulate(ctx, kind, theta, value);
  return ABC_OK;
}

/* Alg.1 l.1-3: the N x L matrix X, each value rounded to FP32 (RN). */
/* Simulated-draw noise (P:218-220's model on the draws, as S:301; R17):
 *   s = RN32(v + ell sigma z),  sigma = sqrt(max(v,0) e^{-lambda t} / dt) e^{lambda t},  t = frame mid,
 *   z = Box-Muller of Philox4x32-10(ctr = {i_lo, i_hi, 2 + f/2, 'VPET'}, key = seed):
 *   ua = u53(x0,x1), ub = u53(x2,x3), z = sqrt(-2 ln ua) cos(2 pi ub) (even f) | sin(2 pi ub) (odd f). */
static double u53(uint32_t a, uint32_t b) {
  uint64_t m = (((uint64_t)a << 32) | b) >> 11;
  return (double)m * 0x1p-53 + 0x1p-54;
}
double oracle_std_normal(uint64_t seed, uint64_t i, uint32_t f) {
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t ctr[4] = {(uint32_t)i, (uint32_t)(i >> 32), 2u + f / 2u, CTR_TAG};
  uint32_t x[4];
  oracle_philox4x32_10(ctr, key, x);
  double ua = u53(x[0], x[1]), ub = u53(x[2], x[3]);
  double r = sqrt(-2.0 * log(ua));
  double ang = 6.283185307179586 * ub;
  return r * ((f & 1u) ? sin(ang) : cos(ang));
}
static float noisy_value(const abc_ctx* c, uint64_t i, uint32_t f, double v) {
  if (c->noise_ell == 0.0) return (float)v;
  double z = oracle_std_normal(c->cfg.seed, i, f);
  double tm = c->fs[f] + 0.5 * c->fd[f];
  double e = exp(c->noise_lam * tm);
  double sig = sqrt(fmax(v, 0.0) / e / c->fd[f]) * e;
  return (float)(v + c->noise_ell * sig * z);
}

abc_status abc_set_sim_noise(abc_ctx* c, double ell, double half_life_min) {
  if (!c) return ABC_E_ARG;
  if (!isfinite(ell) || ell < 0.0) return fail(c, ABC_E_ARG, "noise level must be finite and >= 0");
  if (!(half_life_min > 0.0)) return fail(c, ABC_E_ARG, "half-life must be > 0 (may be +inf)");
  c->noise_ell = ell;
  c->noise_lam = log(2.0) / half_life_min;
  return ABC_OK;
}

abc_status oracle_bank(const abc_ctx* ctx, float* bank) {
  if (!ctx || !ctx->have_input || !ctx->have_frames) return ABC_E_STATE;
  prepare((abc_ctx*)ctx);
  uint64_t N = total_draws(&ctx->cfg);
  uint32_t L = ctx->L;
  long long NN = (long long)N;
#pragma omp parallel for schedule(dynamic, 256) num_threads(oracle_get_threads())
  for (long long i = 0; i < NN; ++i) {
    int32_t m;
    float th[ABC_MAX_P];
    double v[ABC_MAX_L];
    draw_theta(&ctx->cfg, (uint64_t)i, &m, th);
    simulate(ctx, ctx->cfg.model[m].kind, th, v);
    for (uint32_t f = 0; f < L; ++f) bank[(uint64_t)i * L + f] = noisy_value(ctx, (uint64_t)i, f, v[f]);
  }
  return ABC_OK;
}

/* ------------------------------------------------------------------------- */
/* 3. Discrepancy (Alg.1 l.4), FP64, frame order 0..L-1, no contraction.  */
/* ------------------------------------------------------------------------- */
double oracle_distance(int32_t dist, const float* y, const float* s, const float* w, uint32_t L) {
  double D = 0.0;
  for (uint32_t f = 0; f < L; ++f) {
    double wf = w ? (double)w[f] : 1.0;
    double d = (double)y[f] - (double)s[f];
    if (dist == ABC_DIST_L1) D = D + wf * fabs(d);
    else D = D + wf * (d * d);
  }
  return D;
}

/* ------------------------------------------------------------------------- */
/* 5. Reduction helpers                                                       */
/* ------------------------------------------------------------------------- */
/* type-7 quantile (linear interpolation of order statistics), x sorted ascending */
double oracle_quantile7(const double* x, uint32_t n, double q) {
  double h = (double)(n - 1) * q;
  uint32_t lo = (uint32_t)floor(h);
  if (lo + 1 >= n) return x[n - 1];
  return x[lo] + (h - (double)lo) * (x[lo + 1] - x[lo]);
}

/* ------------------------------------------------------------------------- */
/* API                                                                        */
/* ------------------------------------------------------------------------- */
abc_status abc_init(const abc_config* cfg, abc_ctx** out) {
  if (!cfg || !out) return ABC_E_ARG;
  *out = NULL;
  if (cfg->struct_size != sizeof(abc_config)) return ABC_E_ARG;
  if (cfg->n_models < 1 || cfg->n_models > ABC_MAX_MODELS) return ABC_E_ARG;
  int fam = -1;
  for (uint32_t m = 0; m < cfg->n_models; ++m) {
    const abc_model_spec* ms = &cfg->model[m];
    if (ms->kind < ABC_2TCM_IRR || ms->kind > ABC_LPNTPET) return ABC_E_ARG;
    int f = (ms->kind >= ABC_MRTM);
    if (fam >= 0 && f != fam) return ABC_E_ARG;
    fam = f;
    if (ms->n_draws == 0) return ABC_E_ARG;
    for (uint32_t k = 0; k < oracle_family_width(ms->kind); ++k)
      if (!(ms->lo[k] <= ms->hi[k]) || !isfinite(ms->lo[k]) || !isfinite(ms->hi[k])) return ABC_E_ARG;
  }
  uint64_t N = total_draws(cfg);
  if (N >= (1ull << 32)) return ABC_E_ARG;
  if (cfg->distance != ABC_DIST_L1 && cfg->distance != ABC_DIST_WL2) return ABC_E_ARG;
  if (cfg->accept == ABC_ACCEPT_TOPN) {
    if (cfg->n_accept == 0 || cfg->n_accept > N) return ABC_E_ARG;
  } else if (cfg->accept == ABC_ACCEPT_EPS) {
    if (!(cfg->epsilon >= 0.0)) return ABC_E_ARG;
  } else {
    return ABC_E_ARG;
  }
  abc_ctx* c = (abc_ctx*)calloc(1, sizeof(abc_ctx));
  if (!c) return ABC_E_NOMEM;
  c->cfg = *cfg;
  *out = c;
  return ABC_OK;
}

abc_status abc_set_input_function(abc_ctx* c, int32_t kind, const double* t, const double* v, uint32_t n) {
  if (!c) return ABC_E_ARG;
  if (kind == ABC_INPUT_FENG) {
    if (!v || n != 6) return fail(c, ABC_E_ARG, "FENG input needs value[6]");
    for (int i = 0; i < 6; ++i)
      if (!isfinite(v[i])) return fail(c, ABC_E_ARG, "non-finite Feng parameter");
    if (!(v[3] > 0 && v[4] > 0 && v[5] > 0)) return fail(c, ABC_E_ARG, "Feng rates must be > 0");
    if (c->cfg.model[0].kind >= ABC_MRTM) return fail(c, ABC_E_UNSUPPORTED, "reference models need a PWL C_r");
    memcpy(c->feng, v, sizeof(double) * 6);
  } else if (kind == ABC_INPUT_PWL) {
    if (!t || !v || n < 1) return fail(c, ABC_E_ARG, "PWL input needs knots");
    if (t[0] != 0.0) return fail(c, ABC_E_ARG, "first knot must be at t=0");
    for (uint32_t k = 0; k < n; ++k) {
      if (!isfinite(t[k]) || !isfinite(v[k])) return fail(c, ABC_E_ARG, "non-finite knot");
      if (k > 0 && !(t[k] > t[k - 1])) return fail(c, ABC_E_ARG, "knot times must increase");
    }
    free(c->kt); free(c->kc);
    c->kt = (double*)malloc(sizeof(double) * n);
    c->kc = (double*)malloc(sizeof(double) * n);
    memcpy(c->kt, t, sizeof(double) * n);
    memcpy(c->kc, v, sizeof(double) * n);
    c->nk = n;
  } else {
    return fail(c, ABC_E_ARG, "unknown input kind");
  }
  c->input_kind = kind;
  c->have_input = 1;
  unprepare(c);
  return ABC_OK;
}

abc_status abc_set_frames(abc_ctx* c, const double* st, const double* du, const float* w, uint32_t L) {
  if (!c) return ABC_E_ARG;
  if (!st || !du || L < 1 || L > ABC_MAX_L) return fail(c, ABC_E_ARG, "bad frame arrays");
  for (uint32_t f = 0; f < L; ++f) {
    if (!isfinite(st[f]) || !isfinite(du[f]) || !(du[f] > 0.0) || st[f] < 0.0)
      return fail(c, ABC_E_ARG, "frame durations must be > 0, starts >= 0");
    if (f > 0 && st[f] < st[f - 1] + du[f - 1]) return fail(c, ABC_E_ARG, "frames overlap");
    if (w && !(w[f] > 0.0f && isfinite(w[f]))) return fail(c, ABC_E_ARG, "weights must be > 0");
  }
  free(c->fs); free(c->fd); free(c->w);
  c->fs = (double*)malloc(sizeof(double) * L);
  c->fd = (double*)malloc(sizeof(double) * L);
  c->w = (float*)malloc(sizeof(float) * L);
  memcpy(c->fs, st, sizeof(double) * L);
  memcpy(c->fd, du, sizeof(double) * L);
  for (uint32_t f = 0; f < L; ++f) c->w[f] = w ? w[f] : 1.0f;
  c->L = L;
  c->have_frames = 1;
  unprepare(c);
  return ABC_OK;
}

typedef struct { double D; uint32_t i; } dpair;
static int cmp_pair(const void* a, const void* b) {
  const dpair* x = (const dpair*)a;
  const dpair* y = (const dpair*)b;
  if (x->D < y->D) return -1;
  if (x->D > y->D) return 1;
  return (x->i > y->i) - (x->i < y->i);
}
static int cmp_dbl(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}

/* mean, sd (ddof=1), type-7 quantiles of v[0..c-1] (in accepted order) */
static void summarise(double* v, uint32_t c, float* mean, float* sd, float* q3) {
  if (c == 0) {
    if (mean) *mean = NAN;
    if (sd) *sd = NAN;
    if (q3) q3[0] = q3[1] = q3[2] = NAN;
    return;
  }
  double s = 0.0;
  for (uint32_t a = 0; a < c; ++a) s += v[a];
  double mu = s / (double)c;
  double ss = 0.0;
  for (uint32_t a = 0; a < c; ++a) ss += (v[a] - mu) * (v[a] - mu);
  if (mean) *mean = (float)mu;
  if (sd) *sd = c >= 2 ? (float)sqrt(ss / (double)(c - 1)) : NAN;
  if (q3) {
    qsort(v, c, sizeof(double), cmp_dbl);
    q3[0] = (float)oracle_quantile7(v, c, 0.025);
    q3[1] = (float)oracle_quantile7(v, c, 0.5);
    q3[2] = (float)oracle_quantile7(v, c, 0.975);
  }
}

/* column k exists in model kind? (MRTM has no tD, tP, alpha) */
static int column_exists(int32_t kind, uint32_t k) {
  if (kind == ABC_MRTM) return k <= 3;
  return k < oracle_family_width(kind);
}

/* Reduce one voxel's accepted list acc[0..na-1] (draw indices, in accepted order). */
static void reduce_voxel(const abc_ctx* c, const uint32_t* acc, uint32_t na, uint64_t j, abc_result* o) {
  const abc_config* cfg = &c->cfg;
  uint32_t M = cfg->n_models;
  uint32_t P = oracle_family_width(cfg->model[0].kind);
  uint32_t cnt[ABC_MAX_MODELS] = {0, 0, 0, 0};
  for (uint32_t a = 0; a < na; ++a) {
    int32_t m = model_of(cfg, acc[a]);
    cnt[m]++;
  }
  int32_t pref = -1;
  if (na > 0) {
    pref = 0;
    for (uint32_t m = 1; m < M; ++m)
      if (cnt[m] > cnt[pref]) pref = (int32_t)m;
  }
  for (uint32_t m = 0; m < M; ++m) {
    if (o->count) o->count[j * M + m] = cnt[m];
    if (o->prob) o->prob[j * M + m] = na ? (float)((double)cnt[m] / (double)na) : NAN;
  }
  if (o->preferred) o->preferred[j] = pref;
  int want_q = cfg->accept == ABC_ACCEPT_TOPN;
  uint32_t cp = pref >= 0 ? cnt[pref] : 0;
  double* v = (double*)malloc(sizeof(double) * (cp ? cp : 1));
  int32_t kind = pref >= 0 ? cfg->model[pref].kind : cfg->model[0].kind;
  for (uint32_t k = 0; k < P; ++k) {
    uint32_t n = 0;
    if (pref >= 0 && column_exists(kind, k)) {
      for (uint32_t a = 0; a < na; ++a) {
        int32_t m;
        float th[ABC_MAX_P];
        draw_theta(cfg, acc[a], &m, th);
        if (m == pref) v[n++] = (double)th[k];
      }
    }
    float mu, sd, q3[3];
    summarise(v, n, &mu, &sd, q3);
    if (o->mean) o->mean[j * P + k] = mu;
    if (o->sd) o->sd[j * P + k] = sd;
    if (o->q) {
      for (int t = 0; t < 3; ++t) o->q[(j * P + k) * 3 + t] = want_q ? q3[t] : NAN;
    }
  }
  /* K_i = K1 k3 / (k2 + k3) per accepted draw of the preferred 2TCM model */
  uint32_t n = 0;
  if (pref >= 0 && (kind == ABC_2TCM_IRR || kind == ABC_2TCM_REV)) {
    for (uint32_t a = 0; a < na; ++a) {
      int32_t m;
      float th[ABC_MAX_P];
      draw_theta(cfg, acc[a], &m, th);
      if (m == pref) v[n++] = (double)th[0] * (double)th[2] / ((double)th[1] + (double)th[2]);
    }
  }
  float mu, sd, q3[3];
  summarise(v, n, &mu, &sd, q3);
  if (o->ki_mean) o->ki_mean[j] = mu;
  if (o->ki_sd) o->ki_sd[j] = sd;
  if (o->ki_q)
    for (int t = 0; t < 3; ++t) o->ki_q[j * 3 + t] = want_q ? q3[t] : NAN;
  free(v);
}

abc_status abc_run_voxels(abc_ctx* c, const float* tacs, uint64_t J, uint32_t ptr_flags, abc_result* o) {
  if (!c || !o) return ABC_E_ARG;
  if (!c->have_input || !c->have_frames) return fail(c, ABC_E_STATE, "input function and frames must be set");
  if (ptr_flags != 0) return fail(c, ABC_E_UNSUPPORTED, "oracle takes host pointers only");
  if (J == 0) return ABC_OK;
  if (!tacs) return fail(c, ABC_E_ARG, "tacs is NULL");
  uint32_t L = c->L;
  for (uint64_t e = 0; e < J * L; ++e)
    if (!isfinite(tacs[e])) return fail(c, ABC_E_ARG, "non-finite TAC value");
  if (c->cfg.model[0].kind >= ABC_MRTM && c->input_kind != ABC_INPUT_PWL)
    return fail(c, ABC_E_UNSUPPORTED, "reference models need a PWL C_r");
  uint64_t N = total_draws(&c->cfg);
  float* bank = (float*)malloc(sizeof(float) * N * L);
  if (!bank) return fail(c, ABC_E_NOMEM, "bank allocation failed");
  oracle_bank(c, bank);
  const float* w = c->w;
  int dist = c->cfg.distance;
  int topn = c->cfg.accept == ABC_ACCEPT_TOPN;
  uint32_t n = c->cfg.n_accept;
  double eps = c->cfg.epsilon;
  int nthr = oracle_get_threads();
  long long JJ = (long long)J;
  int oom = 0;
#pragma omp parallel num_threads(nthr)
  {
    dpair* Dp = (dpair*)malloc(sizeof(dpair) * N);
    uint32_t* acc = (uint32_t*)malloc(sizeof(uint32_t) * N);
    if (!Dp || !acc) {
#pragma omp atomic write
      oom = 1;
    } else {
#pragma omp for schedule(dynamic, 1)
      for (long long j = 0; j < JJ; ++j) {
        const float* y = tacs + (uint64_t)j * L;
        for (uint64_t i = 0; i < N; ++i) {
          Dp[i].D = oracle_distance(dist, y, bank + i * L, w, L);
          Dp[i].i = (uint32_t)i;
        }
        uint32_t na = 0;
        if (topn) {
          qsort(Dp, N, sizeof(dpair), cmp_pair);
          for (uint32_t a = 0; a < n; ++a) acc[a] = Dp[a].i;
          na = n;
          for (uint32_t a = 0; a < n; ++a) {
            if (o->acc_idx) o->acc_idx[(uint64_t)j * n + a] = Dp[a].i;
            if (o->acc_dist) o->acc_dist[(uint64_t)j * n + a] = Dp[a].D;
          }
        } else {
          for (uint64_t i = 0; i < N; ++i)
            if (Dp[i].D <= eps) acc[na++] = (uint32_t)i;
        }
        reduce_voxel(c, acc, na, (uint64_t)j, o);
      }
    }
    free(Dp);
    free(acc);
  }
  free(bank);
  if (oom) return fail(c, ABC_E_NOMEM, "per-thread distance buffer allocation failed");
  return ABC_OK;
}

abc_status abc_model_select(abc_ctx* c, const float* tacs, uint64_t J, uint32_t ptr_flags, float* prob,
                            int32_t* preferred) {
  abc_result r;
  memset(&r, 0, sizeof r);
  r.prob = prob;
  r.preferred = preferred;
  return abc_run_voxels(c, tacs, J, ptr_flags, &r);
}

/* Response-function credible envelope (Fig. 1).  For voxel j and time t_k: the
 * type-7 2.5/50/97.5 % quantiles, over the voxel's accepted lp-ntPET draws, of
 *   r(t) = k2a(t)/k2a = 1 + (gamma/k2a) g(t; tD, tP, alpha)          (eq:Bt P:90-94)
 * with g the peak-normalised gamma variate above (R4).  Draws of other models are
 * skipped (the envelope is that of "the lp-ntPET model", Fig. 1; R16); NaN when a voxel
 * has none.  acc_idx: J x n_acc (host); q: J x T x 3 (host).  Plain loops, FP64, qsort. */
abc_status abc_response_envelope(abc_ctx* c, const uint64_t* acc_idx, uint64_t J, uint32_t n_acc,
                                 const double* t, uint32_t T, uint32_t ptr_flags, float* q) {
  if (!c) return ABC_E_ARG;
  if (ptr_flags != 0) return fail(c, ABC_E_ARG, "the oracle takes host pointers only");
  if (J == 0) return ABC_OK;
  if (!acc_idx || !t || !q || n_acc == 0 || T == 0 || T > 1024) return fail(c, ABC_E_ARG, "bad envelope arguments");
  int has_lp = 0;
  for (uint32_t m = 0; m < c->cfg.n_models; ++m) has_lp |= c->cfg.model[m].kind == ABC_LPNTPET;
  if (!has_lp) return fail(c, ABC_E_UNSUPPORTED, "no lp-ntPET model in the context");
  for (uint32_t k = 0; k < T; ++k)
    if (!isfinite(t[k])) return fail(c, ABC_E_ARG, "non-finite time");
  const uint64_t N = total_draws(&c->cfg);
  for (uint64_t e = 0; e < J * n_acc; ++e)
    if (acc_idx[e] >= N) return fail(c, ABC_E_ARG, "draw index out of range");
  double* v = (double*)malloc(sizeof(double) * n_acc);
  float(*th)[ABC_MAX_P] = malloc(sizeof(float) * ABC_MAX_P * n_acc);
  if (!v || !th) {
    free(v);
    free(th);
    return fail(c, ABC_E_NOMEM, "envelope buffers");
  }
  for (uint64_t j = 0; j < J; ++j) {
    uint32_t cnt = 0;
    for (uint32_t a = 0; a < n_acc; ++a) {
      int32_t m;
      float x[ABC_MAX_P];
      draw_theta(&c->cfg, acc_idx[j * n_acc + a], &m, x);
      if (c->cfg.model[m].kind != ABC_LPNTPET) continue;
      for (uint32_t k = 0; k < ABC_MAX_P; ++k) th[cnt][k] = x[k];
      ++cnt;
    }
    for (uint32_t k = 0; k < T; ++k) {
      float* o = q + (j * T + k) * 3;
      if (cnt == 0) {
        o[0] = o[1] = o[2] = NAN;
        continue;
      }
      for (uint32_t a = 0; a < cnt; ++a) {
        /* columns: R1, k2, k2a, gamma, tD, tP, alpha */
        double ratio = (double)th[a][3] / (double)th[a][2];
        v[a] = 1.0 + ratio * oracle_gamma_variate(th[a][4], th[a][5], th[a][6], t[k]);
      }
      qsort(v, cnt, sizeof(double), cmp_dbl);
      o[0] = (float)oracle_quantile7(v, cnt, 0.025);
      o[1] = (float)oracle_quantile7(v, cnt, 0.5);
      o[2] = (float)oracle_quantile7(v, cnt, 0.975);
    }
  }
  free(v);
  free(th);
  return ABC_OK;
}

/* Patlak graphical analysis (the clinical K_i reference of P:282, Patlak 1983; SURVEY §8f-4;
 * DESIGN.md R18).  For the frames with mid-time t_f >= t_star:
 *   Cp_f = int_frame Cp / dt_f (frame average of the input), X_f = int_0^{t_f} Cp,
 *   x_f = X_f / Cp_f,  z_f = y_f / Cp_f,
 * and the ordinary least-squares line z = K_i x + V0 (centred two-pass formulas, FP64).
 * NaN when fewer than two frames qualify.  Host pointers only. */
static double input_at(const abc_ctx* c, double t) {
  return c->input_kind == ABC_INPUT_FENG ? oracle_feng(c->feng, t) : pwl_value(c->kt, c->kc, c->nk, t);
}
static double input_integral(const abc_ctx* c, double t0, double t1) {
  if (c->input_kind == ABC_INPUT_FENG) return feng_frame(c->feng, t0, t1);
  /* piecewise linear: trapezoids between t0, the knots inside (t0, t1), and t1 (exact) */
  double s = 0.0, a = t0, va = input_at(c, t0);
  for (uint32_t k = 0; k < c->nk; ++k) {
    if (c->kt[k] <= t0) continue;
    if (c->kt[k] >= t1) break;
    double vb = c->kc[k];
    s += 0.5 * (c->kt[k] - a) * (va + vb);
    a = c->kt[k];
    va = vb;
  }
  s += 0.5 * (t1 - a) * (va + input_at(c, t1));
  return s;
}
abc_status abc_patlak(abc_ctx* c, const float* tacs, uint64_t J, double t_star, uint32_t ptr_flags, float* ki,
                      float* intercept) {
  if (!c) return ABC_E_ARG;
  if (!c->have_input || !c->have_frames) return fail(c, ABC_E_STATE, "input function and frames must be set");
  if (ptr_flags != 0) return fail(c, ABC_E_ARG, "the oracle takes host pointers only");
  if (J == 0) return ABC_OK;
  if (!tacs || !ki || !isfinite(t_star)) return fail(c, ABC_E_ARG, "bad Patlak arguments");
  uint32_t L = c->L;
  double* x = (double*)malloc(sizeof(double) * L);
  double* cp = (double*)malloc(sizeof(double) * L);
  int* use = (int*)malloc(sizeof(int) * L);
  uint32_t m = 0;
  for (uint32_t f = 0; f < L; ++f) {
    double tm = c->fs[f] + 0.5 * c->fd[f];
    use[f] = tm >= t_star;
    cp[f] = input_integral(c, c->fs[f], c->fs[f] + c->fd[f]) / c->fd[f];
    x[f] = input_integral(c, 0.0, tm) / cp[f];
    m += use[f];
  }
  for (uint64_t j = 0; j < J; ++j) {
    double slope = NAN, icpt = NAN;
    if (m >= 2) {
      double xb = 0.0, zb = 0.0;
      for (uint32_t f = 0; f < L; ++f)
        if (use[f]) {
          xb += x[f];
          zb += (double)tacs[j * L + f] / cp[f];
        }
      xb /= m;
      zb /= m;
      double sxx = 0.0, sxz = 0.0;
      for (uint32_t f = 0; f < L; ++f)
        if (use[f]) {
          double dx = x[f] - xb, dz = (double)tacs[j * L + f] / cp[f] - zb;
          sxx += dx * dx;
          sxz += dx * dz;
        }
      if (sxx > 0.0) {
        slope = sxz / sxx;
        icpt = zb - slope * xb;
      }
    }
    ki[j] = (float)slope;
    if (intercept) intercept[j] = (float)icpt;
  }
  free(x);
  free(cp);
  free(use);
  return ABC_OK;
}

const char* abc_last_error(const abc_ctx* c) { return c ? c->err : "null context"; }

void abc_destroy(abc_ctx* c) {
  if (!c) return;
  unprepare(c);
  free(c->kt); free(c->kc); free(c->fs); free(c->fd); free(c->w);
  free(c);
}
