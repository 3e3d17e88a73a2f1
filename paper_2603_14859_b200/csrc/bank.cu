// bank.cu -- K1: simulation bank (Alg. 1 lines 1-3).
//
// Each thread simulates one draw in FP64 and stores the frame averages rounded to FP32
// (the method's FP32 TAC):
//   2TCM (eq:2TCM P:69-74, eq:2TCM_op P:75-80, C_wb = C_p P:80):
//     h(t) = c1 e^{-a1 t} + c2 e^{-a2 t},  a2 = (s+r)/2, a1 = 2 k2 k4/(s+r),
//     s = k2+k3+k4, r^2 = (k2-k4)^2 + k3 (k3 + 2 (k2+k4)),
//     c1 = K1 (k3+k4-a1)/(a2-a1), c2 = K1 (a2-k3-k4)/(a2-a1),
//     value_f = [(1-Vb)(c1 S_f(a1) + c2 S_f(a2)) + Vb int_f C_p] / dt_f,
//     S_f(a) = int_f (C_p (x) e^{-a.}) dt: exact recurrences on the PWL grid, or the Feng
//     closed form.
//   MRTM (eq:lp-ntPET with gamma = 0): value_f = [R1 int_f C_r + (k2 - R1 k2a) S_f(k2a)]/dt_f.
//   (/ dt_f is applied as * RN64(1/dt_f), rounded on the host.)
// The FP64 values are not bit-identical to the oracle's: besides the host-rounded 1/dt_f, nvcc
// contracts a*b+c into DFMA here (default -fmad=true), the phi functions use a series below 0.5
// (the oracle uses closed forms / expm1) and the device exp differs from glibc's in the last ulp.
// All of these are a few FP64 ulps, so RN32 of a frame value flips only when the value lies within
// that distance of an FP32 rounding boundary (measured: < 1e-4 of bank entries, test_gpu_parity);
// DESIGN.md §3 counts such flips among the parity-exempt boundary cases.
//   lp-ntPET (eq:lp-ntPET, eq:Bt): z = C_t - R1 C_r, z' = (k2 - R1 a) C_r - a z,
//     a(t) = k2a + gamma g(t) frozen at each substep midpoint (R4).
#include <cfloat>

#include "common.cuh"

namespace vpet {

namespace {

// Optional simulated-draw noise (abc_set_sim_noise; P:218-220 noise model applied to
// the draws as in S:301; R17): value_f + ell sigma_f z_if with
//   sigma_f = sqrt(max(value_f, 0) / e / dt_f) e,  e = exp(lambda t_f),  t_f = start_f + dt_f / 2,
//   z_if = Box-Muller of Philox4x32-10(ctr = {i_lo, i_hi, 2 + f/2, 'VPET'}, key = seed):
//   ua = u53(x0, x1), ub = u53(x2, x3), z = sqrt(-2 ln ua) (cos | sin)(2 pi ub) for even | odd f.
// FP64, no contraction, then RN32.  ell = 0: exactly the noise-free RN32 value.
struct DrawId {
  uint64_t i;
  uint32_t s0, s1;
};
__device__ __forceinline__ double u53(uint32_t a, uint32_t b) {
  const uint64_t m = ((uint64_t(a) << 32) | b) >> 11;
  return __dadd_rn(__dmul_rn(double(m), 1.1102230246251565e-16), 5.551115123125783e-17);  // (m + 1/2) 2^-53
}
__device__ __forceinline__ float emit_noisy(const Tables& T, const DrawId& d, int f, double v) {
  uint32_t x[4];
  philox10(uint32_t(d.i), uint32_t(d.i >> 32), 2u + uint32_t(f) / 2u, kCtrTag, d.s0, d.s1, x);
  const double ua = u53(x[0], x[1]), ub = u53(x[2], x[3]);
  const double r = sqrt(__dmul_rn(-2.0, log(ua)));
  const double ang = __dmul_rn(6.283185307179586, ub);
  const double z = __dmul_rn(r, (f & 1) ? sin(ang) : cos(ang));
  const double tm = __dadd_rn(T.fs[f], __dmul_rn(0.5, T.fdur[f]));
  const double e = exp(__dmul_rn(T.noise_lam, tm));
  const double sig = __dmul_rn(sqrt(__ddiv_rn(__ddiv_rn(fmax(v, 0.0), e), T.fdur[f])), e);
  return __double2float_rn(__dadd_rn(v, __dmul_rn(__dmul_rn(T.noise_ell, sig), z)));
}
// NZ = false (ell = 0): a single rounding; the noisy variant is a separate kernel instance
template <bool NZ>
__device__ __forceinline__ float emit(const Tables& T, const DrawId& d, int f, double v) {
  if constexpr (NZ) return emit_noisy(T, d, f, v);
  else return __double2float_rn(v);
}

struct FrameAcc {
  int cur = -1;
  double A = 0.0, B = 0.0;
};

// ---- piecewise-linear input on a grid: both rates of the 2TCM at once ----
template <bool NZ>
__device__ void sim_2tcm_pwl(const Tables& T, const DrawId& D, double a1, double a2, double c1, double c2, double Vb,
                             float* out) {
  double I1 = 0.0, I2 = 0.0;
  Phi P0{}, P1{}, Q0{}, Q1{};
  FrameAcc fa;
  auto flush = [&](int f) {
    double v = ((1.0 - Vb) * (c1 * fa.A + c2 * fa.B) + Vb * T.favg_in[f]) * T.finv[f];
    out[f] = emit<NZ>(T, D, f, v);
  };
  for (uint32_t k = 0; k + 1 < T.G; ++k) {
    double t0 = T.gt[k], t1 = T.gt[k + 1];
    double h = t1 - t0;
    double ck = T.gc[k], ck1 = T.gc[k + 1];
    int f = T.gframe[k];
    // phi(a h) depends on the draw only through a: reuse it across segments of equal length h
    // (bit-identical to recomputing; the cache schedule is the same for every draw)
    const uint32_t code = T.gcode[k];
    const uint32_t slot = code & 3u;
    if (code & 0x80u) {
      Phi np = phi_all(a1 * h), nq = phi_all(a2 * h);
      if (slot == 0) { P0 = np; Q0 = nq; } else { P1 = np; Q1 = nq; }
    }
    // slot is warp-uniform (one schedule for all draws): branch instead of selecting 10 doubles
    auto body = [&](const Phi& p, const Phi& q) {
      double dc = ck1 - ck;
      double s1 = h * p.p1 * I1 + h * h * (ck1 * p.ps - dc * p.om);
      double s2 = h * q.p1 * I2 + h * h * (ck1 * q.ps - dc * q.om);
      if (f != fa.cur) {
        if (fa.cur >= 0) flush(fa.cur);
        fa.cur = f;
        fa.A = 0.0;
        fa.B = 0.0;
      }
      fa.A += s1;
      fa.B += s2;
      I1 = p.e * I1 + h * (ck * p.ch + ck1 * p.ps);
      I2 = q.e * I2 + h * (ck * q.ch + ck1 * q.ps);
    };
    if (slot == 0) body(P0, Q0);
    else body(P1, Q1);
  }
  if (fa.cur >= 0) flush(fa.cur);
}

// ---- irreversible 2TCM (k4 = 0, so a1 = 0): the a1 = 0 frame integrals S_f(0) do not depend on the
// draw; they are precomputed once per grid (s0_table_kernel, the same FP64 operations as the a1
// half of sim_2tcm_pwl) and only the a2 recurrence runs per draw ----
template <bool NZ>
__device__ void sim_2tcm_pwl_irr(const Tables& T, const DrawId& D, double a2, double c1, double c2, double Vb,
                                 float* out) {
  double I2 = 0.0;
  Phi Q0{}, Q1{};
  FrameAcc fa;
  auto flush = [&](int f) {
    double v = ((1.0 - Vb) * (c1 * T.s0[f] + c2 * fa.B) + Vb * T.favg_in[f]) * T.finv[f];
    out[f] = emit<NZ>(T, D, f, v);
  };
  for (uint32_t k = 0; k + 1 < T.G; ++k) {
    double t0 = T.gt[k], t1 = T.gt[k + 1];
    double h = t1 - t0;
    double ck = T.gc[k], ck1 = T.gc[k + 1];
    int f = T.gframe[k];
    const uint32_t code = T.gcode[k];
    const uint32_t slot = code & 3u;
    if (code & 0x80u) {
      Phi nq = phi_all(a2 * h);
      if (slot == 0) Q0 = nq; else Q1 = nq;
    }
    auto body = [&](const Phi& q) {
      double dc = ck1 - ck;
      double s2 = h * q.p1 * I2 + h * h * (ck1 * q.ps - dc * q.om);
      if (f != fa.cur) {
        if (fa.cur >= 0) flush(fa.cur);
        fa.cur = f;
        fa.B = 0.0;
      }
      fa.B += s2;
      I2 = q.e * I2 + h * (ck * q.ch + ck1 * q.ps);
    };
    if (slot == 0) body(Q0);
    else body(Q1);
  }
  if (fa.cur >= 0) flush(fa.cur);
}

__global__ void s0_table_kernel(const Tables T, double* s0) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double I1 = 0.0;
  Phi P0{}, P1{};
  int cur = -1;
  double A = 0.0;
  const double a1 = 0.0;
  for (uint32_t k = 0; k + 1 < T.G; ++k) {
    double t0 = T.gt[k], t1 = T.gt[k + 1];
    double h = t1 - t0;
    double ck = T.gc[k], ck1 = T.gc[k + 1];
    int f = T.gframe[k];
    const uint32_t code = T.gcode[k];
    const uint32_t slot = code & 3u;
    if (code & 0x80u) {
      Phi np = phi_all(a1 * h);
      if (slot == 0) P0 = np; else P1 = np;
    }
    const Phi& p = slot == 0 ? P0 : P1;
    double dc = ck1 - ck;
    double s1 = h * p.p1 * I1 + h * h * (ck1 * p.ps - dc * p.om);
    if (f != cur) {
      if (cur >= 0) s0[cur] = A;
      cur = f;
      A = 0.0;
    }
    A += s1;
    I1 = p.e * I1 + h * (ck * p.ch + ck1 * p.ps);
  }
  if (cur >= 0) s0[cur] = A;
}

// ---- Feng input: closed forms of e^{-a t} (x) {e^{-k t}, t e^{-k t}} and their integrals ----
__device__ inline double convE(double a, double k, double t) {
  double mn = fmin(a, k);
  return t * exp(-mn * t) * phi1_only(fabs(a - k) * t);
}
__device__ inline double convEt(double a, double k, double t) {
  if (a >= k) {
    Phi p = phi_all((a - k) * t);
    return t * t * exp(-k * t) * p.ps;
  }
  Phi p = phi_all((k - a) * t);
  return t * t * exp(-a * t) * p.ch;
}
__device__ inline double Gexp(double x, double ts, double te) {
  double d = te - ts;
  return exp(-x * ts) * d * phi1_only(x * d);
}
// int_ts^te E dt via E' = e^{-k t} - a E = e^{-a t} - k E (divide by the larger rate)
__device__ inline double intE(double a, double k, double ts, double te) {
  double dE = convE(a, k, te) - convE(a, k, ts);
  return (a >= k) ? (Gexp(k, ts, te) - dE) / a : (Gexp(a, ts, te) - dE) / k;
}
// int Et via Et' = E - k Et
__device__ inline double intEt(double a, double k, double ts, double te) {
  double dEt = convEt(a, k, te) - convEt(a, k, ts);
  return (intE(a, k, ts, te) - dEt) / k;
}
__device__ inline double feng_conv(const double* b, double a, double ts, double te) {
  return b[0] * intEt(a, b[3], ts, te) - (b[1] + b[2]) * intE(a, b[3], ts, te) + b[1] * intE(a, b[4], ts, te) +
         b[2] * intE(a, b[5], ts, te);
}

template <bool NZ>
__device__ void sim_2tcm_feng(const Tables& T, const DrawId& D, double a1, double a2, double c1, double c2, double Vb, float* out) {
  for (uint32_t f = 0; f < T.L; ++f) {
    double ts = T.fs[f], te = T.fe[f];
    double S1 = feng_conv(T.fb, a1, ts, te);
    double S2 = feng_conv(T.fb, a2, ts, te);
    double v = ((1.0 - Vb) * (c1 * S1 + c2 * S2) + Vb * T.favg_in[f]) * T.finv[f];
    out[f] = emit<NZ>(T, D, f, v);
  }
}

template <bool NZ>
__device__ void sim_mrtm(const Tables& T, const DrawId& D, double R1, double k2, double k2a, float* out) {
  double I = 0.0;
  FrameAcc fa;
  double kf = k2 - R1 * k2a;
  Phi P0{}, P1{};
  auto flush = [&](int f) { out[f] = emit<NZ>(T, D, f, (R1 * T.favg_in[f] + kf * fa.A) * T.finv[f]); };
  for (uint32_t k = 0; k + 1 < T.G; ++k) {
    double h = T.gt[k + 1] - T.gt[k];
    double ck = T.gc[k], ck1 = T.gc[k + 1];
    int f = T.gframe[k];
    const uint32_t code = T.gcode[k];
    const uint32_t slot = code & 3u;
    if (code & 0x80u) {
      Phi np = phi_all(k2a * h);
      if (slot == 0) P0 = np; else P1 = np;
    }
    auto body = [&](const Phi& p) {  // slot is warp-uniform: branch, not select
      double s = h * p.p1 * I + h * h * (ck1 * p.ps - (ck1 - ck) * p.om);
      if (f != fa.cur) {
        if (fa.cur >= 0) flush(fa.cur);
        fa.cur = f;
        fa.A = 0.0;
      }
      fa.A += s;
      I = p.e * I + h * (ck * p.ch + ck1 * p.ps);
    };
    if (slot == 0) body(P0);
    else body(P1);
  }
  if (fa.cur >= 0) flush(fa.cur);
}

template <bool NZ>
__device__ void sim_lpntpet(const Tables& T, const DrawId& D, const float* th, float* out) {
  double R1 = th[0], k2 = th[1], k2a = th[2], gam = th[3], tD = th[4], tP = th[5], al = th[6];
  double inv = 1.0 / (tP - tD);
  double z = 0.0;
  FrameAcc fa;
  auto flush = [&](int f) { out[f] = emit<NZ>(T, D, f, (fa.A + R1 * T.favg_in[f]) * T.finv[f]); };
  for (uint32_t k = 0; k + 1 < T.GF; ++k) {
    double t0 = T.ft[k], t1 = T.ft[k + 1];
    double h = t1 - t0;
    double tm = 0.5 * (t0 + t1);
    double g = 0.0;
    if (tm > tD) {
      double x = (tm - tD) * inv;
      g = exp(al * (log(x) + 1.0 - x));  // x^alpha e^{alpha (1-x)}
    }
    double ab = k2a + gam * g;
    Phi p = phi_all(ab * h);
    double kf = k2 - R1 * ab;
    double fk = kf * T.fc[k], fk1 = kf * T.fc[k + 1];
    double s = h * p.p1 * z + h * h * (fk1 * p.ps - (fk1 - fk) * p.om);
    int f = T.fframe[k];
    if (f != fa.cur) {
      if (fa.cur >= 0) flush(fa.cur);
      fa.cur = f;
      fa.A = 0.0;
    }
    fa.A += s;
    z = p.e * z + h * (fk * p.ch + fk1 * p.ps);
  }
  if (fa.cur >= 0) flush(fa.cur);
}

template <bool NZ>
__global__ void __launch_bounds__(128) bank_kernel(const BankParams p, const PriorDev prior) {
  uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= p.N) return;
  float th[ABC_MAX_P];
  int m = draw_theta(prior, i, th);
  int kind = prior.m[m].kind;
  float* out = p.bank + i * p.T.LS;
  const Tables& T = p.T;
  const DrawId D{i, prior.seed_lo, prior.seed_hi};
  if (kind <= ABC_2TCM_REV) {
    double K1 = th[0], k2 = th[1], k3 = th[2], k4 = th[3], Vb = th[4];
    double s = k2 + k3 + k4;
    double r = sqrt((k2 - k4) * (k2 - k4) + k3 * (k3 + 2.0 * (k2 + k4)));
    double a2 = 0.5 * (s + r);
    double a1 = (s + r) > 0.0 ? 2.0 * k2 * k4 / (s + r) : 0.0;
    double den = a2 - a1;
    double c1 = K1 * (k3 + k4 - a1) / den;
    double c2 = K1 * (a2 - k3 - k4) / den;
    if (T.feng) sim_2tcm_feng<NZ>(T, D, a1, a2, c1, c2, Vb, out);
    else if (a1 == 0.0 && T.s0) sim_2tcm_pwl_irr<NZ>(T, D, a2, c1, c2, Vb, out);
    else sim_2tcm_pwl<NZ>(T, D, a1, a2, c1, c2, Vb, out);
  } else if (kind == ABC_MRTM) {
    sim_mrtm<NZ>(T, D, th[0], th[1], th[2], out);
  } else {
    sim_lpntpet<NZ>(T, D, th, out);
  }
  for (uint32_t f = T.L; f < T.LS; ++f) out[f] = 0.0f;
}

__global__ void fill_u32_kernel(uint32_t* p, uint32_t v, uint64_t n) {
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += uint64_t(gridDim.x) * blockDim.x)
    p[e] = v;
}

}  // namespace

void launch_bank(const BankParams& p, const PriorDev& prior, cudaStream_t st) {
  uint64_t blocks = (p.N + 127) / 128;
  if (p.T.noise_ell != 0.0) bank_kernel<true><<<unsigned(blocks), 128, 0, st>>>(p, prior);
  else bank_kernel<false><<<unsigned(blocks), 128, 0, st>>>(p, prior);
}

void launch_s0_table(const Tables& T, double* s0, cudaStream_t st) { s0_table_kernel<<<1, 32, 0, st>>>(T, s0); }

void launch_fill_u32(uint32_t* p, uint32_t v, uint64_t n, cudaStream_t st) {
  fill_u32_kernel<<<148, 256, 0, st>>>(p, v, n);
}

}  // namespace vpet
