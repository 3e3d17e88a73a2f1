// api.cu -- host runtime and C ABI of libvpetabc.so (see include/vpetabc.h).
//
// Owns the per-device context: validated configuration, draw-independent time grids and
// frame tables (built here in FP64), device buffers (reused across calls), the stream, and
// the launch sequence of one abc_run_voxels call:
//   K0  finite check of the TACs
//   K1  bank: N draws simulated in FP64, stored RN32            (Alg.1 l.1-3)
//   K1b frame spread + scan order; K1c negated prescaled copy
//   K2  FP32 pass: fused distance + per-voxel selection        (Alg.1 l.4-5)
//   K3  FP64 certification, K4 posterior reduction
//   K5  exact FP64 scan of uncertified voxels, then K3/K4 on them
// Nothing runs on the CPU except validation and table construction.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

using namespace vpet;

namespace {

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) cap = bytes;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
};

uint32_t family_width(int kind) { return kind >= ABC_MRTM ? 7u : 5u; }

enum Stage { EV_START, EV_H2D, EV_BANK, EV_ORDER, EV_SCAN, EV_CERT, EV_FB, EV_D2H, EV_N };

}  // namespace

struct abc_ctx {
  abc_config cfg{};
  int dev = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  std::string err;
  uint64_t N = 0;
  uint32_t P = 5, M = 1;
  PriorDev prior{};
  // input
  bool have_input = false, have_frames = false;
  int input_kind = ABC_INPUT_PWL;
  double feng[6] = {0, 0, 0, 0, 0, 0};
  double noise_ell = 0.0, noise_lam = 0.0;  // abc_set_sim_noise
  std::vector<double> kt, kc;
  // frames
  uint32_t L = 0;
  std::vector<double> fs, fd;
  std::vector<float> w;
  bool unit_w = true;
  // device tables
  bool dirty = true;
  uint32_t G = 0, GF = 0;
  DevBuf d_finv;  // [L] 1 / frame duration (the bank multiplies instead of dividing)
  DevBuf d_s0;    // [L] S_f(0) of the PWL grid (irreversible 2TCM draws)
  bool have_s0 = false;
  DevBuf d_cwd;  // [L] sqrt(w_f) in FP64 (rotated scan basis)
  DevBuf d_fdur, d_fs, d_fe, d_favg, d_w, d_wsc, d_gt, d_gc, d_gframe, d_gcode, d_ft, d_fc, d_fframe;
  // work buffers
  DevBuf d_prior, bank, bankp, var, fmean, perm, wsp, heap, heap_cnt, tacs, fb_list, fb_len, work, hd, hidx, mom, flag, outs;
  DevBuf cov, pcs, pminmax, keys, keys_alt, vals, order, idxmap, sort_temp, tbounds, sbounds, hbounds, tau_glob, queue;
  DevBuf rotq, ytr, gbox;  // rotated scan basis: [L][LP] FP64 rotation, [J][LP] voxel coordinates, [2][LP] bank box
  DevBuf vkeys, vkeys_alt, vvals, vorder, vslot, vsort_temp, item_log;
  DevBuf fb_tau, cl_d, cl_i, cl_cnt, fb2_list, fb2_len;  // fallback tiers (certify.cu)
  DevBuf dBt, dS2, dAt, dY2;  // ABC_FLAG_DENSE_TC operands (dense_tc.cu)
  DevBuf env_idx, env_t, env_q;  // abc_response_envelope staging
  DevBuf proj;                   // [N][kNPC] bank projections (order stage)
  DevBuf pat_ab;                 // abc_patlak frame coefficients [2][L]
  abc_stats stats{};
  bool bank_valid = false;
  uint64_t mem_sig[6] = {~0ull, 0, 0, 0, 0, 0};  // (J, N, flags, ptr_flags, n, L) of the last passed memory check
  bool dist_wl2() const { return cfg.distance == ABC_DIST_WL2; }
  uint32_t bank_L = 0;
  cudaEvent_t ev[EV_N] = {};
  cudaStream_t copy = nullptr;       // host->device TAC copies, overlapped with the bank / order stages
  cudaEvent_t tacs_ready = nullptr;
  cudaStream_t aux = nullptr;        // the order stage's basis computation, overlapped with its sorts
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  static constexpr int kOutChunks = 4;  // host outputs: K4 in chunks, each chunk's D2H overlapping the next
  cudaEvent_t ev_chunk[kOutChunks] = {};
  bool ev_ok = false;
  int num_sms = 148;
};

namespace {

abc_status fail(abc_ctx* c, abc_status s, const std::string& m) {
  if (c) c->err = m;
  return s;
}

abc_status cuda_fail(abc_ctx* c, cudaError_t e, const char* where) {
  return fail(c, ABC_E_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(call)                                                 \
  do {                                                           \
    cudaError_t e_ = (call);                                     \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call);     \
  } while (0)

template <class T>
cudaError_t upload(DevBuf& b, const std::vector<T>& v) {
  cudaError_t e = b.ensure(sizeof(T) * (v.empty() ? 1 : v.size()));
  if (e != cudaSuccess) return e;
  if (v.empty()) return cudaSuccess;
  return cudaMemcpy(b.p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice);
}

// PWL interpolation through the knots, held after the last knot (R1).
double pwl_at(const std::vector<double>& kt, const std::vector<double>& kc, double t) {
  if (t >= kt.back()) return kc.back();
  size_t k = size_t(std::upper_bound(kt.begin(), kt.end(), t) - kt.begin()) - 1;  // kt[k] <= t < kt[k+1]
  double a = (t - kt[k]) / (kt[k + 1] - kt[k]);
  return kc[k] + (kc[k + 1] - kc[k]) * a;
}

// sorted, de-duplicated union of {0}, `extra` (<= tend), frame starts and ends
std::vector<double> make_grid(const abc_ctx* c, const std::vector<double>& extra) {
  double tend = c->fs[c->L - 1] + c->fd[c->L - 1];
  std::vector<double> t;
  t.reserve(extra.size() + 2 * c->L + 1);
  t.push_back(0.0);
  for (double x : extra)
    if (x <= tend) t.push_back(x);
  for (uint32_t f = 0; f < c->L; ++f) {
    t.push_back(c->fs[f]);
    t.push_back(c->fs[f] + c->fd[f]);
  }
  std::sort(t.begin(), t.end());
  t.erase(std::unique(t.begin(), t.end()), t.end());
  return t;
}

std::vector<int> segment_frames(const abc_ctx* c, const std::vector<double>& t) {
  std::vector<int> sf(t.size() > 1 ? t.size() - 1 : 1, -1);
  uint32_t f = 0;
  for (size_t k = 0; k + 1 < t.size(); ++k) {
    while (f < c->L && t[k] >= c->fs[f] + c->fd[f]) ++f;
    if (f < c->L && t[k] >= c->fs[f] && t[k + 1] <= c->fs[f] + c->fd[f]) sf[k] = int(f);
  }
  return sf;
}

// int_ts^te of the Feng curve, closed form
double feng_frame_integral(const double* b, double ts, double te) {
  auto G = [](double x, double a, double z) {  // int_a^z e^{-x t} dt
    double d = z - a;
    double ph = (x * d == 0.0) ? 1.0 : -std::expm1(-x * d) / (x * d);
    return std::exp(-x * a) * d * ph;
  };
  double k1 = b[3];
  double tint = (ts * std::exp(-k1 * ts) - te * std::exp(-k1 * te)) / k1 + G(k1, ts, te) / k1;
  return b[0] * tint - (b[1] + b[2]) * G(k1, ts, te) + b[1] * G(b[4], ts, te) + b[2] * G(b[5], ts, te);
}

Tables make_tables(const abc_ctx* c, uint32_t LS);

abc_status build_tables(abc_ctx* ctx) {
  if (!ctx->dirty) return ABC_OK;
  const uint32_t L = ctx->L;
  std::vector<double> fe(L), favg(L, 0.0);
  for (uint32_t f = 0; f < L; ++f) fe[f] = ctx->fs[f] + ctx->fd[f];
  std::vector<double> gt{0.0, 1.0}, gc{0.0, 0.0}, ft{0.0, 1.0}, fc{0.0, 0.0};
  std::vector<int> gfr{-1}, ffr{-1};
  if (ctx->input_kind == ABC_INPUT_PWL) {
    gt = make_grid(ctx, ctx->kt);
    gc.resize(gt.size());
    for (size_t k = 0; k < gt.size(); ++k) gc[k] = pwl_at(ctx->kt, ctx->kc, gt[k]);
    gfr = segment_frames(ctx, gt);
    for (size_t k = 0; k + 1 < gt.size(); ++k)
      if (gfr[k] >= 0) favg[gfr[k]] += 0.5 * (gt[k + 1] - gt[k]) * (gc[k] + gc[k + 1]);
    bool lpnt = false;
    for (uint32_t m = 0; m < ctx->M; ++m) lpnt |= ctx->cfg.model[m].kind == ABC_LPNTPET;
    if (lpnt) {
      double delta = ctx->cfg.lpnt_step_min > 0.0 ? ctx->cfg.lpnt_step_min : 0.05;
      double tend = fe[L - 1];
      std::vector<double> extra;
      for (uint64_t k = 0; double(k) * delta < tend; ++k) extra.push_back(double(k) * delta);
      for (double x : ctx->kt) extra.push_back(x);
      ft = make_grid(ctx, extra);
      if (ft.size() > 4000000) return fail(ctx, ABC_E_UNSUPPORTED, "lp-ntPET grid too fine");
      fc.resize(ft.size());
      for (size_t k = 0; k < ft.size(); ++k) fc[k] = pwl_at(ctx->kt, ctx->kc, ft[k]);
      ffr = segment_frames(ctx, ft);
    }
  } else {
    for (uint32_t f = 0; f < L; ++f) favg[f] = feng_frame_integral(ctx->feng, ctx->fs[f], fe[f]);
  }
  std::vector<float> wsc(L);
  for (uint32_t f = 0; f < L; ++f) {
    if (ctx->unit_w) wsc[f] = 1.0f;
    else if (ctx->cfg.distance == ABC_DIST_WL2) wsc[f] = float(std::sqrt(double(ctx->w[f])));
    else wsc[f] = ctx->w[f];
  }
  CK(upload(ctx->d_fdur, ctx->fd));
  {
    std::vector<double> finv(ctx->fd.size());
    for (size_t f = 0; f < finv.size(); ++f) finv[f] = 1.0 / ctx->fd[f];
    CK(upload(ctx->d_finv, finv));
  }
  CK(upload(ctx->d_fs, ctx->fs));
  CK(upload(ctx->d_fe, fe));
  CK(upload(ctx->d_favg, favg));
  CK(upload(ctx->d_w, ctx->w));
  CK(upload(ctx->d_wsc, wsc));
  {
    std::vector<double> cwd(L);
    for (uint32_t f = 0; f < L; ++f) cwd[f] = ctx->unit_w ? 1.0 : std::sqrt(double(ctx->w[f]));
    CK(upload(ctx->d_cwd, cwd));
  }
  CK(upload(ctx->d_gt, gt));
  CK(upload(ctx->d_gc, gc));
  CK(upload(ctx->d_gframe, gfr));
  {  // phi cache codes: an LRU of kPhiSlots segment lengths, simulated here (the grid is shared)
    std::vector<uint8_t> code(gt.size() > 1 ? gt.size() - 1 : 1, 0x80);
    double slot_h[kPhiSlots];
    int age[kPhiSlots];
    for (int c = 0; c < kPhiSlots; ++c) { slot_h[c] = -1.0; age[c] = -1; }
    for (size_t k = 0; k + 1 < gt.size(); ++k) {
      const double h = gt[k + 1] - gt[k];  // the device computes the same difference
      int hit = -1;
      for (int c = 0; c < kPhiSlots; ++c)
        if (slot_h[c] == h) hit = c;
      if (hit >= 0) {
        code[k] = uint8_t(hit);
      } else {
        int v = 0;
        for (int c = 1; c < kPhiSlots; ++c)
          if (age[c] < age[v]) v = c;
        slot_h[v] = h;
        hit = v;
        code[k] = uint8_t(0x80 | v);
      }
      age[hit] = int(k);
    }
    CK(upload(ctx->d_gcode, code));
  }
  CK(upload(ctx->d_ft, ft));
  CK(upload(ctx->d_fc, fc));
  CK(upload(ctx->d_fframe, ffr));
  CK(ctx->d_prior.ensure(sizeof(PriorDev)));
  CK(cudaMemcpy(ctx->d_prior.p, &ctx->prior, sizeof(PriorDev), cudaMemcpyHostToDevice));
  ctx->G = uint32_t(gt.size());
  ctx->GF = uint32_t(ft.size());
  ctx->have_s0 = false;
  if (ctx->input_kind == ABC_INPUT_PWL && ctx->cfg.model[0].kind <= ABC_2TCM_REV) {
    CK(ctx->d_s0.ensure(sizeof(double) * L));
    CK(cudaMemset(ctx->d_s0.p, 0, sizeof(double) * L));
    Tables T = make_tables(ctx, (L + 3) & ~3u);
    T.s0 = nullptr;
    launch_s0_table(T, ctx->d_s0.as<double>(), nullptr);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());  // the context's stream does not synchronise with the legacy stream
    ctx->have_s0 = true;
  }
  ctx->dirty = false;
  return ABC_OK;
}

Tables make_tables(const abc_ctx* c, uint32_t LS) {
  Tables T{};
  T.L = c->L;
  T.LS = LS;
  T.fdur = c->d_fdur.as<double>();
  T.finv = c->d_finv.as<double>();
  T.fs = c->d_fs.as<double>();
  T.fe = c->d_fe.as<double>();
  T.favg_in = c->d_favg.as<double>();
  T.w = c->d_w.as<float>();
  T.G = c->G;
  T.gt = c->d_gt.as<double>();
  T.gc = c->d_gc.as<double>();
  T.gframe = c->d_gframe.as<int>();
  T.gcode = c->d_gcode.as<uint8_t>();
  T.GF = c->GF;
  T.ft = c->d_ft.as<double>();
  T.fc = c->d_fc.as<double>();
  T.fframe = c->d_fframe.as<int>();
  T.feng = c->input_kind == ABC_INPUT_FENG;
  T.noise_ell = c->noise_ell;
  T.noise_lam = c->noise_lam;
  for (int k = 0; k < 6; ++k) T.fb[k] = c->feng[k];
  T.s0 = c->have_s0 ? c->d_s0.as<double>() : nullptr;
  return T;
}

// Rigorous |D32 - D| bound of the FP32 pass, doubled for margin.
ErrBound error_bound(const abc_ctx* c, uint32_t LP) {
  const double u = std::ldexp(1.0, -24);
  const double g = LP * u / (1.0 - LP * u);
  ErrBound e{0, 0, 0, 0};
  if (c->cfg.distance == ABC_DIST_WL2) {
    if (c->unit_w) {
      e.a = 2.0 * (g + 3.0 * u);
    } else {
      e.a = 2.0 * (g + 6.1 * u);
      e.b = 2.0 * 4.1 * u;
      e.c = 2.0 * 16.5 * u * u;
    }
  } else {
    if (c->unit_w) {
      e.a = 2.0 * (g + 2.0 * u);
    } else {
      e.a = 2.0 * (g + 3.1 * u);
      e.d = 2.0 * 2.1 * u;
    }
  }
  return e;
}

// Rotated scan basis (WL2): scan coordinates y'_k = RN32(sum_f Q_fk sqrt(w_f) y_f)
// and s'_k likewise (FP64 sums), ||Q^T Q - I||_2 <= e_Q = kRotEps.  With a = y' - s' (reals) and
// v = sqrt(w)(y - s), D = |v|^2:  |a - Q^T v| <= u (|y'| + |s'|) (1 + 1e-12) <= u' (2 sqrt(Y2) + sqrt(D)),
// u' = u sqrt(1 + e_Q) (1 + 1e-12), so |A - D| <= (e_Q + 2u' + u'^2) D + (4u' + 4u'^2) sqrt(Y2 D) + 4u'^2 Y2
// for A = |a|^2; the FP32 pass on (y', s') is the unit-weight WL2 case, |D32 - A| <= (g_L + 3u) A.
// Combined, with margin: (g_L + 6u + e_Q) D + 4.1u sqrt(Y2 D) + 16.5u^2 Y2, doubled like the others.
ErrBound rotated_error_bound(uint32_t LP) {
  const double u = std::ldexp(1.0, -24);
  const double g = LP * u / (1.0 - LP * u);
  ErrBound e{0, 0, 0, 0};
  e.a = 2.0 * (g + 6.1 * u + kRotEps);
  e.b = 2.0 * 4.1 * u;
  e.c = 2.0 * 16.5 * u * u;
  return e;
}

// Rigorous |D' - D| bound of the dense dot form (ABC_FLAG_DENSE_TC, dense_tc.cu),
// doubled for margin.  With a = fl(ws y), b = fl(ws s), Z = sum w (|y| + |s|)^2 <= 4 Y2 + 4 sqrt(Y2 D) + D:
//   prescaling        |sum (a-b)^2 - D| <= (2u + u^2) D + 2u sqrt(D Z) + u^2 Z
//   Y2, S2 in FP32    gamma_{L+1} (sum a^2 + sum b^2)
//   G on tcgen05      (3.01 * 2^-18 [dropped split terms] + 144 * 2^-23 [FP32 accumulation, any
//                     order, truncating adds]) sum |a b|
//   final fadd, ffma  u (Y2 + S2) + u |D'|
// all <= C Z + 2u D + 2u sqrt(D Z), C = gamma_{L+1} + 2u + c_G (+ u^2 terms absorbed).
ErrBound dense_error_bound(uint32_t L) {
  const double u = std::ldexp(1.0, -24);
  const double g = (L + 1) * u / (1.0 - (L + 1) * u);
  const double cG = 3.01 * std::ldexp(1.0, -18) + 144.0 * std::ldexp(1.0, -23);
  const double C = g + 2.0 * u + cG + 4.0 * u * u;
  ErrBound e{0, 0, 0, 0};
  e.a = 2.0 * (C + 4.0 * u);
  e.b = 2.0 * (4.0 * C + 4.0 * u);
  e.c = 2.0 * 4.0 * C;
  return e;
}

}  // namespace

namespace vpet {
cudaError_t ensure_smem_attr(const void* func, size_t bytes) {
  if (bytes <= 32 * 1024) return cudaSuccess;  // + static shared memory stays under the 48 KB default
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;  // (function, device) -> opted-in bytes
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{func, dev}];
  if (have >= bytes) return cudaSuccess;
  int optin = 0;
  e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  if (e != cudaSuccess) return e;
  cudaFuncAttributes fa{};
  e = cudaFuncGetAttributes(&fa, func);
  if (e != cudaSuccess) return e;
  if (bytes + fa.sharedSizeBytes <= 48 * 1024) {
    have = bytes;
    return cudaSuccess;
  }
  if (bytes + fa.sharedSizeBytes > size_t(optin)) return cudaErrorInvalidValue;
  e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
  if (e == cudaSuccess) have = bytes;
  return e;
}

// host outputs of at least this many voxels are reduced and copied back in chunks (overlap)
constexpr uint64_t kChunkedOutMin = 1u << 18;

// padded frame counts with a compiled FP32-pass instance (scan_kernels.cuh VPET_LP_LIST)
static const uint32_t kLPs[] = {8, 12, 16, 20, 24, 28, 32, 36, 40, 44, 48, 56, 64, 80, 96, 128};
bool scan_supported(uint32_t LP) {
  for (uint32_t v : kLPs)
    if (v == LP) return true;
  return false;
}
uint32_t scan_lp_for(uint32_t L) {
  for (uint32_t v : kLPs)
    if (L <= v) return v;
  return 0;
}
}  // namespace vpet

namespace {

// 16-B loads, four in flight per thread (the TAC buffer is cudaMalloc- or user-aligned to 16 B when
// its size allows; otherwise the scalar loop covers everything)
__global__ void __launch_bounds__(256) finite_check_kernel(const float* x, uint64_t n, int* flag) {
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x, nt = uint64_t(gridDim.x) * blockDim.x;
  bool bad = false;
  uint64_t done = 0;
  if ((reinterpret_cast<uintptr_t>(x) & 15u) == 0) {
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const uint64_t n4 = n / 4;
    for (uint64_t e = tid; e < n4; e += 4 * nt) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = e + u * nt < n4 ? __ldcs(x4 + e + u * nt) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 4; ++u) bad |= !(isfinite(v[u].x) && isfinite(v[u].y) && isfinite(v[u].z) && isfinite(v[u].w));
    }
    done = n4 * 4;
  }
  for (uint64_t e = done + tid; e < n; e += nt) bad |= !isfinite(x[e]);
  if (bad) *flag = 1;
}

}  // namespace

extern "C" {

uint32_t abc_abi_version(void) { return VPETABC_ABI_VERSION; }

abc_status abc_init(const abc_config* cfg, abc_ctx** out) {
  if (!out) return ABC_E_ARG;
  *out = nullptr;
  if (!cfg || cfg->struct_size != sizeof(abc_config)) return ABC_E_ARG;
  if (cfg->n_models < 1 || cfg->n_models > ABC_MAX_MODELS) return ABC_E_ARG;
  if (cfg->reserved1 != 0) return ABC_E_ARG;
  uint64_t N = 0;
  int fam = -1;
  for (uint32_t m = 0; m < cfg->n_models; ++m) {
    const abc_model_spec& ms = cfg->model[m];
    if (ms.kind < ABC_2TCM_IRR || ms.kind > ABC_LPNTPET || ms.reserved0 != 0 || ms.n_draws == 0) return ABC_E_ARG;
    int f = ms.kind >= ABC_MRTM;
    if (fam >= 0 && f != fam) return ABC_E_ARG;
    fam = f;
    for (uint32_t k = 0; k < family_width(ms.kind); ++k)
      if (!std::isfinite(ms.lo[k]) || !std::isfinite(ms.hi[k]) || !(ms.lo[k] <= ms.hi[k])) return ABC_E_ARG;
    if (ms.kind <= ABC_2TCM_REV && !(ms.lo[2] > 0.0f)) return ABC_E_ARG;  // r > 0 (R3)
    if (ms.kind == ABC_LPNTPET && !(ms.lo[5] > 0.0f)) return ABC_E_ARG;   // tP > tD
    N += ms.n_draws;
  }
  if (N >= (1ull << 32)) return ABC_E_ARG;
  if (cfg->distance != ABC_DIST_L1 && cfg->distance != ABC_DIST_WL2) return ABC_E_ARG;
  if (cfg->accept == ABC_ACCEPT_TOPN) {
    if (cfg->n_accept == 0 || cfg->n_accept > N || cfg->n_accept > kMaxAccept) return ABC_E_ARG;
  } else if (cfg->accept == ABC_ACCEPT_EPS) {
    if (!(cfg->epsilon >= 0.0)) return ABC_E_ARG;
  } else {
    return ABC_E_ARG;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg->device < 0 || cfg->device >= ndev) return ABC_E_CUDA;
  if (cudaSetDevice(cfg->device) != cudaSuccess) return ABC_E_CUDA;
  abc_ctx* c = new (std::nothrow) abc_ctx();
  if (!c) return ABC_E_NOMEM;
  c->cfg = *cfg;
  c->dev = cfg->device;
  if (cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, cfg->device) != cudaSuccess) c->num_sms = 148;
  c->N = N;
  c->M = cfg->n_models;
  c->P = family_width(cfg->model[0].kind);
  c->prior.M = c->M;
  c->prior.seed_lo = uint32_t(cfg->seed);
  c->prior.seed_hi = uint32_t(cfg->seed >> 32);
  uint64_t off = 0;
  for (uint32_t m = 0; m < c->M; ++m) {
    ModelDev& md = c->prior.m[m];
    const abc_model_spec& ms = cfg->model[m];
    md.kind = ms.kind;
    md.P = family_width(ms.kind);
    md.begin = off;
    off += ms.n_draws;
    md.end = off;
    for (int k = 0; k < ABC_MAX_P; ++k) {
      md.lo[k] = ms.lo[k];
      md.span[k] = ms.hi[k] - ms.lo[k];  // FP32 subtraction (theta = fmaf(span, u, lo))
    }
  }
  for (uint32_t m = c->M; m < ABC_MAX_MODELS; ++m) c->prior.m[m].begin = ~0ull;
  if (cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking) != cudaSuccess) {
    delete c;
    return ABC_E_CUDA;
  }
  c->stream = c->own;
  if (cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->tacs_ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      [&] {
        for (auto& e : c->ev_chunk)
          if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return true;
        return false;
      }()) {
    cudaStreamDestroy(c->own);
    delete c;
    return ABC_E_CUDA;
  }
  c->ev_ok = true;
  for (int k = 0; k < EV_N; ++k)
    if (cudaEventCreate(&c->ev[k]) != cudaSuccess) c->ev_ok = false;
  c->stats.struct_size = sizeof(abc_stats);
  *out = c;
  return ABC_OK;
}

abc_status abc_set_input_function(abc_ctx* ctx, int32_t kind, const double* t, const double* v, uint32_t n) {
  if (!ctx) return ABC_E_ARG;
  if (kind == ABC_INPUT_FENG) {
    if (!v || n != 6) return fail(ctx, ABC_E_ARG, "FENG input needs value[6]");
    for (int k = 0; k < 6; ++k)
      if (!std::isfinite(v[k])) return fail(ctx, ABC_E_ARG, "non-finite Feng parameter");
    if (!(v[3] > 0 && v[4] > 0 && v[5] > 0)) return fail(ctx, ABC_E_ARG, "Feng rates must be > 0");
    if (ctx->cfg.model[0].kind >= ABC_MRTM) return fail(ctx, ABC_E_UNSUPPORTED, "reference models need a PWL C_r");
    std::memcpy(ctx->feng, v, sizeof ctx->feng);
  } else if (kind == ABC_INPUT_PWL) {
    if (!t || !v || n < 1) return fail(ctx, ABC_E_ARG, "PWL input needs knots");
    if (t[0] != 0.0) return fail(ctx, ABC_E_ARG, "first knot must be at t = 0");
    for (uint32_t k = 0; k < n; ++k) {
      if (!std::isfinite(t[k]) || !std::isfinite(v[k])) return fail(ctx, ABC_E_ARG, "non-finite knot");
      if (k > 0 && !(t[k] > t[k - 1])) return fail(ctx, ABC_E_ARG, "knot times must increase");
    }
    ctx->kt.assign(t, t + n);
    ctx->kc.assign(v, v + n);
  } else {
    return fail(ctx, ABC_E_ARG, "unknown input kind");
  }
  ctx->input_kind = kind;
  ctx->have_input = true;
  ctx->dirty = true;
  return ABC_OK;
}

abc_status abc_set_frames(abc_ctx* ctx, const double* st, const double* du, const float* wt, uint32_t L) {
  if (!ctx) return ABC_E_ARG;
  if (!st || !du || L < 1 || L > ABC_MAX_L) return fail(ctx, ABC_E_ARG, "need 1..128 frames");
  for (uint32_t f = 0; f < L; ++f) {
    if (!std::isfinite(st[f]) || !std::isfinite(du[f]) || !(du[f] > 0.0) || st[f] < 0.0)
      return fail(ctx, ABC_E_ARG, "frame durations must be > 0 and starts >= 0");
    if (f > 0 && st[f] < st[f - 1] + du[f - 1]) return fail(ctx, ABC_E_ARG, "frames overlap or are not increasing");
    if (wt && !(wt[f] > 0.0f && std::isfinite(wt[f]))) return fail(ctx, ABC_E_ARG, "weights must be finite and > 0");
  }
  ctx->fs.assign(st, st + L);
  ctx->fd.assign(du, du + L);
  ctx->w.assign(L, 1.0f);
  ctx->unit_w = true;
  if (wt) {
    for (uint32_t f = 0; f < L; ++f) {
      ctx->w[f] = wt[f];
      if (wt[f] != 1.0f) ctx->unit_w = false;
    }
  }
  ctx->L = L;
  ctx->have_frames = true;
  ctx->dirty = true;
  return ABC_OK;
}

abc_status abc_set_stream(abc_ctx* ctx, void* s) {
  if (!ctx) return ABC_E_ARG;
  ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own;
  return ABC_OK;
}

abc_status abc_sync(abc_ctx* ctx) {
  if (!ctx) return ABC_E_ARG;
  CK(cudaSetDevice(ctx->dev));
  CK(cudaStreamSynchronize(ctx->stream));
  return ABC_OK;
}

abc_status abc_get_stats(const abc_ctx* ctx, abc_stats* s) {
  if (!ctx || !s || s->struct_size != sizeof(abc_stats)) return ABC_E_ARG;
  *s = ctx->stats;
  return ABC_OK;
}

abc_status abc_run_voxels(abc_ctx* ctx, const float* tacs, uint64_t J, uint32_t ptr_flags, abc_result* out) {
  if (!ctx || !out) return ABC_E_ARG;
  if (!ctx->have_input || !ctx->have_frames) return fail(ctx, ABC_E_STATE, "input function and frames must be set");
  if (ptr_flags & ~(ABC_PTR_TACS_DEVICE | ABC_PTR_OUT_DEVICE)) return fail(ctx, ABC_E_ARG, "unknown ptr_flags");
  if (ctx->cfg.model[0].kind >= ABC_MRTM && ctx->input_kind != ABC_INPUT_PWL)
    return fail(ctx, ABC_E_UNSUPPORTED, "reference models need a PWL C_r");
  if (J >= (1ull << 32)) return fail(ctx, ABC_E_ARG, "J must be < 2^32");
  abc_stats& S = ctx->stats;
  std::memset(&S, 0, sizeof S);
  S.struct_size = sizeof(abc_stats);
  S.n_voxels = J;
  S.n_draws = ctx->N;
  if (J == 0) return ABC_OK;
  if (!tacs) return fail(ctx, ABC_E_ARG, "tacs is NULL");
  static const bool host_dbg = getenv("VPET_HOST_TIMING") != nullptr;
  auto hnow = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const double h0 = hnow();
  double h1 = 0, h2 = 0, h3 = 0;
  CK(cudaSetDevice(ctx->dev));
  abc_status bs = build_tables(ctx);
  if (bs != ABC_OK) return bs;
  const double h_tab = hnow();

  const cudaStream_t st = ctx->stream;
  const uint64_t N = ctx->N;
  const uint32_t L = ctx->L, LS = (L + 3) & ~3u, M = ctx->M, P = ctx->P;
  const uint32_t LP = scan_lp_for(L);
  const bool eps = ctx->cfg.accept == ABC_ACCEPT_EPS;
  const bool exact = (ctx->cfg.flags & ABC_FLAG_EXACT) && !eps;
  const bool timing = (ctx->cfg.flags & ABC_FLAG_TIMING) && ctx->ev_ok;
  const bool count_work = (ctx->cfg.flags & ABC_FLAG_COUNT_WORK) != 0;
  const bool dense = (ctx->cfg.flags & ABC_FLAG_DENSE_TC) && !exact;
  if (dense && (eps || !ctx->dist_wl2() || L > 48 || 2 * (4 * uint64_t(ctx->cfg.n_accept) + 64) > kLargeMaxCand))
    return fail(ctx, ABC_E_UNSUPPORTED, "ABC_FLAG_DENSE_TC needs WL2, top-n acceptance, L <= 48 and n <= 2032");
  const uint32_t n = ctx->cfg.n_accept;
  uint32_t K = 0;
  if (!eps) {
    // dense mode: a wider candidate band, since its dot-form error bound is ~1e-4 of ||y||^2 (vs ~u D)
    // FP32 pass: K = n + slack candidates per part.  The K-th smallest D32 is the pruning threshold, so
    // a small slack prunes harder; the slack (>= 1) only has to keep D_(K) above D_(n) + err for the
    // certification: 4 draws left no uncertified voxel on the 4.44M-voxel TB volume
    // (slack 2: 30 voxels; slack 1: 187 on the 1/32 slab set), and an uncertified voxel costs ~0.25 ms
    // in the fallback collector.
    static const uint64_t slack = getenv("VPET_KSLACK") ? uint64_t(std::max(1, atoi(getenv("VPET_KSLACK")))) : 4;  // tuning knob
    uint64_t k = dense ? 4 * uint64_t(n) + 64 : uint64_t(n) + std::max<uint64_t>(slack, n / 16);
    if (dense) k = (k + 7) & ~7ull;
    if (getenv("VPET_KROUND")) k = (k + 7) & ~7ull;  // tuning knob: round-1 behaviour
    K = uint32_t(std::min<uint64_t>(k, N));
  }
  S.lp = LP;
  S.heap_k = K;

  // ---- memory plan (checked before allocating) ----
  const bool host_tacs = !(ptr_flags & ABC_PTR_TACS_DEVICE);
  const bool host_out = !(ptr_flags & ABC_PTR_OUT_DEVICE);
  struct OutDesc {
    void* user;
    size_t bytes;
  };
  OutDesc od[11] = {
      {out->prob, 4 * J * M},       {out->preferred, 4 * J},      {out->count, 4 * J * M},
      {out->mean, 4 * J * P},       {out->sd, 4 * J * P},         {out->q, 12 * J * P},
      {out->ki_mean, 4 * J},        {out->ki_sd, 4 * J},          {out->ki_q, 12 * J},
      {eps ? nullptr : out->acc_idx, 8 * J * n}, {eps ? nullptr : out->acc_dist, 8 * J * n}};
  size_t out_bytes = 0;
  for (auto& d : od)
    if (d.user && host_out) out_bytes += (d.bytes + 255) & ~size_t(255);
  size_t need = 0;
  need += sizeof(float) * N * LS;                        // exact bank
  if (!exact && !dense) need += sizeof(float) * N * LP;  // scan bank
  if (dense) need += dense_bank_bytes(N) + dense_voxel_bytes(J) + 4 * J;
  const bool tree = !exact && !dense && !(ctx->cfg.flags & ABC_FLAG_NO_TREE) && N < (1ull << 31);
  const uint64_t ntile = (N + kTile - 1) / kTile, nsuper = (ntile + kSuper - 1) / kSuper;
  // rotated scan basis: WL2, tree mode, frame reordering allowed, LP <= 96 (shared
  // memory of the basis and rotation kernels)
  static const bool rot_env = getenv("VPET_ROT") ? atoi(getenv("VPET_ROT")) != 0 : true;  // tuning knob
  // and enough pairs to amortise the basis (config 2, 1e4 TACs x 2e5 draws: +12 ms of order stage
  // for -2 ms of scan; the TB volume: 4.4e13 pairs)
  // (n = 1e4 of config 5 is faster in the frame basis: 1015 vs 1144 ms of scan; n = 1e3: 148 vs 137)
  const bool rotated = rot_env && tree && ctx->dist_wl2() && !(ctx->cfg.flags & ABC_FLAG_NO_REORDER) && LP <= 96 &&
                       ((double(J) * double(N) >= 1e11 && K <= 4096) || getenv("VPET_ROT_ALWAYS"));
  const size_t sort_tmp = tree ? order_sort_temp_bytes(N) : 0;
  // draw-range split of the tree scan (interleaved super-tiles): balances heavy voxels over SMs
  uint32_t nparts = 1;
  // parts share the draws of a voxel between SMs; each keeps its own K candidates, so large n uses
  // fewer parts (certification holds all parts' candidates of a voxel in shared memory)
  // The parts also balance the persistent scan over the SMs: with few voxel tiles per CTA slot
  // more parts keep every SM busy, with many the parts only duplicate heap fills and threshold
  // traffic.  Measured best on the TB phantom with the rotated scan (CTA slots = SMs x 8): 4-6 parts
  // at 1.8 voxel tiles per slot (1/16 slab set), 2 at 7.3 (1/4) and at 29 (the whole volume: 170 ms
  // vs 173 with 1 part and 178 with 3; the frame-basis kernel wanted 6 / 4 / 3).
  if (tree && !eps) {
    if (K <= 512) {
      const double tiles_per_slot = double((J + 127) / 128) / double(std::max(1, ctx->num_sms) * 8);
      nparts = tiles_per_slot < 2.0 ? 6u : (tiles_per_slot < 4.0 ? 4u : 2u);
    } else {
      nparts = 2 * K <= kLargeMaxCand ? 2u : 1u;
    }
  }
  if (tree && eps) nparts = 6u;
  if (const char* e = getenv("VPET_NPARTS")) nparts = uint32_t(std::max(1, atoi(e)));  // tuning knob
  // hyper-tiles of hs super-tiles: the unit of the work split and of the best-first order; at most
  // kHyperSort per part
  uint32_t hs = 16;
  if (const char* e = getenv("VPET_HS")) hs = uint32_t(std::max(1, atoi(e)));  // tuning knob
  {
    const uint64_t need_hs = (nsuper + uint64_t(kHyperSort) * nparts - 1) / (uint64_t(kHyperSort) * nparts);
    if (need_hs > hs) hs = uint32_t(need_hs);
  }
  const uint64_t nhyper = (nsuper + hs - 1) / hs;
  if (nparts > nhyper) nparts = uint32_t(nhyper);
  if (nparts == 0) nparts = 1;
  if (dense) nparts = 2;  // the two column halves of each draw tile (dense_tc.cu)
  const size_t vsort_tmp = tree ? voxel_sort_temp_bytes(J) : 0;
  if (tree) need += N * (8 + 8 + 4 + 4 + 4 + 4 * kNPC) + 16 + sort_tmp + sizeof(float) * 2 * LP * (ntile + nsuper + nhyper);
  if (tree) need += 28 * J + vsort_tmp;
  if (rotated) need += sizeof(double) * L * LP + sizeof(float) * J * LP;
  if (!eps) need += (size_t(8) * heap_stride(std::max<uint32_t>(K, 1)) + 4) * J * nparts + 4 * J;  // heaps
  need += size_t(12) * J * (n ? n : 1);                  // exact heaps (last-resort fallback)
  // fallback collector lists: cl_cap (the certification capacity) entries for up to cl_voxels voxels
  uint32_t cl_cap = 32, cl_voxels = 0;
  if (!eps && !exact) {
    ReduceParams tmp{};
    tmp.K = K;
    tmp.nparts = dense ? 2u : ((tree) ? nparts : 1u);
    tmp.n = n;
    cl_cap = certify_capacity(tmp);
    const uint64_t by_mem = (uint64_t(256) << 20) / (12ull * cl_cap);
    cl_voxels = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(J, by_mem)));
    need += size_t(12) * cl_cap * cl_voxels + 4 * size_t(cl_voxels) + 12 * J + 16;
  }
  if (eps) need += sizeof(Fix128) * J * nparts * M * MOMW;
  if (host_tacs) need += sizeof(float) * J * L;
  need += out_bytes + 8 * J + (64u << 20);
  // the device-memory query is skipped when this exact shape passed it before (all buffers exist)
  const uint64_t sig[6] = {J, N, ctx->cfg.flags, ptr_flags, n, L};
  if (!std::equal(sig, sig + 6, ctx->mem_sig)) {
    size_t free_b = 0, total_b = 0;
    CK(cudaMemGetInfo(&free_b, &total_b));
    size_t have = free_b + ctx->bank.cap + ctx->bankp.cap + ctx->heap.cap + ctx->hd.cap + ctx->hidx.cap + ctx->tacs.cap +
                  ctx->outs.cap + ctx->mom.cap;
    if (need > have) return fail(ctx, ABC_E_NOMEM, "device memory: need " + std::to_string(need >> 20) + " MiB");
  }

  CK(ctx->bank.ensure(sizeof(float) * N * LS));
  if (!exact && !dense) CK(ctx->bankp.ensure(sizeof(float) * N * LP));
  if (dense) {
    const uint64_t Npad = (N + 255) / 256 * 256, Jpad = (J + 127) / 128 * 128;
    CK(ctx->dBt.ensure(Npad * 144 * 2));
    CK(ctx->dS2.ensure(Npad * 4));
    CK(ctx->dAt.ensure(Jpad * 144 * 2));
    CK(ctx->dY2.ensure(Jpad * 4));
    CK(ctx->tau_glob.ensure(4 * J));
  }
  CK(ctx->var.ensure(sizeof(double) * kMaxLP));
  CK(ctx->fmean.ensure(sizeof(double) * kMaxLP));
  if (tree) {
    CK(ctx->cov.ensure(sizeof(double) * kMaxLP * kMaxLP));
    CK(ctx->pcs.ensure(sizeof(float) * kNPC * kMaxLP));
    CK(ctx->pminmax.ensure(sizeof(unsigned int) * 2 * kNPC));
    CK(ctx->keys.ensure(8 * N));
    CK(ctx->proj.ensure(sizeof(float) * kNPC * N));
    CK(ctx->keys_alt.ensure(8 * N));
    CK(ctx->vals.ensure(4 * N));
    CK(ctx->order.ensure(4 * N));
    CK(ctx->idxmap.ensure(4 * (N + 4)));
    CK(ctx->sort_temp.ensure(sort_tmp));
    CK(ctx->tbounds.ensure(sizeof(float) * 2 * LP * ntile));
    CK(ctx->sbounds.ensure(sizeof(float) * 2 * LP * nsuper));
    CK(ctx->hbounds.ensure(sizeof(float) * 2 * LP * nhyper));
    CK(ctx->tau_glob.ensure(4 * J));
    CK(ctx->queue.ensure(16));
    if (rotated) {
      CK(ctx->rotq.ensure(sizeof(double) * L * LP));
      CK(ctx->ytr.ensure(sizeof(float) * J * LP));
      CK(ctx->gbox.ensure(sizeof(float) * 2 * LP));
    }
    CK(ctx->vkeys.ensure(8 * J));
    CK(ctx->vkeys_alt.ensure(8 * J));
    CK(ctx->vvals.ensure(4 * J));
    CK(ctx->vorder.ensure(4 * J));
    CK(ctx->vslot.ensure(4 * J));
    CK(ctx->vsort_temp.ensure(vsort_tmp));
  }
  CK(ctx->perm.ensure(sizeof(int) * kMaxLP));
  CK(ctx->wsp.ensure(sizeof(float) * kMaxLP));
  if (!eps) {
    CK(ctx->heap.ensure(size_t(8) * J * nparts * heap_stride(std::max<uint32_t>(K, 1))));
    CK(ctx->heap_cnt.ensure(4 * J * nparts));
    CK(ctx->hd.ensure(sizeof(double) * J * n));
    CK(ctx->hidx.ensure(sizeof(uint32_t) * J * n));
  } else {
    CK(ctx->mom.ensure(sizeof(Fix128) * J * nparts * M * MOMW));
  }
  CK(ctx->fb_list.ensure(4 * J));
  CK(ctx->fb_len.ensure(16));
  if (cl_voxels) {
    CK(ctx->fb_tau.ensure(8 * J));
    CK(ctx->cl_d.ensure(size_t(8) * cl_cap * cl_voxels));
    CK(ctx->cl_i.ensure(size_t(4) * cl_cap * cl_voxels));
    CK(ctx->cl_cnt.ensure(size_t(4) * cl_voxels));
    CK(ctx->fb2_list.ensure(4 * J));
    CK(ctx->fb2_len.ensure(16));
  }
  CK(ctx->work.ensure(32));
  CK(ctx->flag.ensure(16));
  if (host_tacs) CK(ctx->tacs.ensure(sizeof(float) * J * L));
  if (out_bytes) CK(ctx->outs.ensure(out_bytes));

  std::copy(sig, sig + 6, ctx->mem_sig);
  const double h_alloc = hnow();

  // device-side result pointers
  abc_result dout = *out;
  if (eps) {
    dout.acc_idx = nullptr;
    dout.acc_dist = nullptr;
  }
  if (host_out) {
    char* base = ctx->outs.as<char>();
    void** fields[11] = {(void**)&dout.prob,    (void**)&dout.preferred, (void**)&dout.count,
                         (void**)&dout.mean,    (void**)&dout.sd,        (void**)&dout.q,
                         (void**)&dout.ki_mean, (void**)&dout.ki_sd,     (void**)&dout.ki_q,
                         (void**)&dout.acc_idx, (void**)&dout.acc_dist};
    size_t off = 0;
    for (int k = 0; k < 11; ++k) {
      if (od[k].user) {
        *fields[k] = base + off;
        off += (od[k].bytes + 255) & ~size_t(255);
      } else {
        *fields[k] = nullptr;
      }
    }
  }

  uint32_t launches = 0;
  bool outs_copied = false;  // host outputs already copied chunk by chunk (K4 overlap)
  auto rec = [&](int k) {
    if (timing) cudaEventRecord(ctx->ev[k], st);
  };
  h1 = hnow();
  rec(EV_START);
  const float* d_tacs = tacs;
  if (host_tacs) {
    // the copy runs on its own stream, overlapped with the bank and bank-order stages (which do
    // not read the TACs); the compute stream joins it before the first TAC reader.  ctx->tacs is
    // free: the previous call ended with a stream synchronisation.
    CK(cudaEventRecord(ctx->tacs_ready, st));
    CK(cudaStreamWaitEvent(ctx->copy, ctx->tacs_ready, 0));
    CK(cudaMemcpyAsync(ctx->tacs.p, tacs, sizeof(float) * J * L, cudaMemcpyHostToDevice, ctx->copy));
    CK(cudaEventRecord(ctx->tacs_ready, ctx->copy));
    d_tacs = ctx->tacs.as<float>();
  }
  rec(EV_H2D);
  CK(cudaMemsetAsync(ctx->flag.p, 0, 16, st));
  CK(cudaMemsetAsync(ctx->fb_len.p, 0, 16, st));
  if (cl_voxels) {
    CK(cudaMemsetAsync(ctx->fb2_len.p, 0, 16, st));
    CK(cudaMemsetAsync(ctx->cl_cnt.p, 0, size_t(4) * cl_voxels, st));
  }
  CK(cudaMemsetAsync(ctx->work.p, 0, 32, st));
  bool joined = false;
  auto join_tacs = [&]() -> cudaError_t {  // before the first kernel that reads the TACs
    if (joined) return cudaSuccess;
    joined = true;
    if (host_tacs) {
      cudaError_t e = cudaStreamWaitEvent(st, ctx->tacs_ready, 0);
      if (e != cudaSuccess) return e;
    }
    finite_check_kernel<<<148 * 8, 256, 0, st>>>(d_tacs, J * L, ctx->flag.as<int>());
    ++launches;
    return cudaGetLastError();
  };

  // K1: bank
  BankParams bp{make_tables(ctx, LS), N, ctx->bank.as<float>()};
  launch_bank(bp, ctx->prior, st);
  ++launches;
  ctx->bank_valid = true;
  ctx->bank_L = L;
  rec(EV_BANK);

  const ErrBound eb = dense ? dense_error_bound(L) : (rotated ? rotated_error_bound(LP) : error_bound(ctx, LP));
  if (!exact && !dense) {
    OrderParams op{};
    op.bank = ctx->bank.as<float>();
    op.N = N;
    op.L = L;
    op.LS = LS;
    op.LP = LP;
    op.wsc = ctx->d_wsc.as<float>();
    op.var = ctx->var.as<double>();
    op.mean = ctx->fmean.as<double>();
    op.perm = ctx->perm.as<int>();
    op.wsp = ctx->wsp.as<float>();
    op.bankp = ctx->bankp.as<float>();
    op.reorder = !(ctx->cfg.flags & ABC_FLAG_NO_REORDER);
    op.tree = tree;
    if (tree) {
      op.cov = ctx->cov.as<double>();
      op.pcs = ctx->pcs.as<float>();
      op.pminmax = ctx->pminmax.as<unsigned int>();
      op.proj = ctx->proj.as<float>();
      op.keys = ctx->keys.as<unsigned long long>();
      op.keys_alt = ctx->keys_alt.as<unsigned long long>();
      op.vals = ctx->vals.as<uint32_t>();
      op.order = ctx->order.as<uint32_t>();
      op.idxmap = ctx->idxmap.as<uint32_t>();
      op.sort_temp = ctx->sort_temp.p;
      op.sort_temp_bytes = sort_tmp;
      op.tbounds = ctx->tbounds.as<float>();
      op.sbounds = ctx->sbounds.as<float>();
      op.hbounds = ctx->hbounds.as<float>();
      op.hs = hs;
      op.nhyper = nhyper;
      if (rotated) {
        op.rotq = ctx->rotq.as<double>();
        op.cw = ctx->d_cwd.as<double>();
        op.gbox = ctx->gbox.as<float>();
        op.aux = ctx->aux;
        op.ev_fork = ctx->ev_fork;
        op.ev_join = ctx->ev_join;
      }
    }
    CK(launch_order(op, st, &launches));
    if (tree) {
      CK(join_tacs());
      VoxelOrderParams vp{};
      vp.tacs = d_tacs;
      vp.J = J;
      vp.L = L;
      vp.LP = LP;
      vp.perm = ctx->perm.as<int>();
      vp.wsp = ctx->wsp.as<float>();
      vp.mean = ctx->fmean.as<double>();
      vp.pcs = ctx->pcs.as<float>();
      vp.pminmax = ctx->pminmax.as<unsigned int>();
      vp.keys = ctx->vkeys.as<unsigned long long>();
      vp.keys_alt = ctx->vkeys_alt.as<unsigned long long>();
      vp.vals = ctx->vvals.as<uint32_t>();
      vp.vorder = ctx->vorder.as<uint32_t>();
      vp.vslot = ctx->vslot.as<uint32_t>();
      vp.sort_temp = ctx->vsort_temp.p;
      vp.sort_temp_bytes = vsort_tmp;
      CK(launch_voxel_order(vp, st, &launches));
      if (rotated) {
        CK(launch_voxel_rotate(d_tacs, J, L, LP, ctx->rotq.as<double>(), ctx->ytr.as<float>(), st));
        ++launches;
      }
    }
  }
  CK(join_tacs());
  rec(EV_ORDER);

  if (dense) {
    DenseParams dp{};
    dp.Bt = ctx->dBt.as<uint16_t>();
    dp.S2 = ctx->dS2.as<float>();
    dp.At = ctx->dAt.as<uint16_t>();
    dp.Y2 = ctx->dY2.as<float>();
    dp.N = N;
    dp.J = J;
    dp.L = L;
    dp.K = K;
    dp.heap = ctx->heap.as<unsigned long long>();
    dp.heap_cnt = ctx->heap_cnt.as<uint32_t>();
    dp.tau_glob = ctx->tau_glob.as<unsigned int>();
    dp.bad = ctx->flag.as<int>();
    launch_fill_u32(ctx->tau_glob.as<uint32_t>(), 0x7f800000u, J, st);
    ++launches;
    CK(launch_dense(dp, ctx->bank.as<float>(), LS, d_tacs, ctx->d_wsc.as<float>(), st, &launches));
  } else if (!exact) {
    ScanParams sp{};
    sp.bankp = ctx->bankp.as<float>();
    sp.N = N;
    sp.tacs = d_tacs;
    sp.J = J;
    sp.L = L;
    sp.perm = ctx->perm.as<int>();
    sp.wsp = ctx->wsp.as<float>();
    sp.K = K;
    sp.heap = ctx->heap.as<unsigned long long>();
    sp.heap_cnt = ctx->heap_cnt.as<uint32_t>();
    sp.prune = !(ctx->cfg.flags & ABC_FLAG_NO_PRUNE);
    sp.work = ctx->work.as<unsigned long long>();
    sp.eps_mode = eps;
    sp.eps = ctx->cfg.epsilon;
    sp.w = ctx->d_w.as<float>();
    sp.bank = ctx->bank.as<float>();
    sp.LS = LS;
    sp.dist = ctx->cfg.distance;
    sp.unit_w = ctx->unit_w;
    sp.mom = eps ? ctx->mom.as<Fix128>() : nullptr;
    sp.eb = eb;
    sp.prior_g = ctx->d_prior.as<PriorDev>();
    sp.M = M;
    sp.bad = ctx->flag.as<int>();
    if (tree) {
      sp.idxmap = ctx->idxmap.as<uint32_t>();
      sp.tbounds = ctx->tbounds.as<float>();
      sp.sbounds = ctx->sbounds.as<float>();
      sp.hbounds = ctx->hbounds.as<float>();
      sp.nhyper = nhyper;
      sp.hs = hs;
      sp.ntile = ntile;
      sp.nsuper = nsuper;
      sp.tau_glob = eps ? nullptr : ctx->tau_glob.as<unsigned int>();
      sp.queue = ctx->queue.as<unsigned int>();
      sp.vorder = ctx->vorder.as<uint32_t>();
      sp.ytr = rotated ? ctx->ytr.as<float>() : nullptr;
      sp.gbox = rotated ? ctx->gbox.as<float>() : nullptr;
      if (!eps) launch_fill_u32(ctx->tau_glob.as<uint32_t>(), 0x7f800000u, J, st);
      CK(cudaMemsetAsync(ctx->queue.p, 0, 16, st));
      launches += eps ? 0 : 1;
    }
    sp.nparts = nparts;
    sp.bound_work = ctx->work.as<unsigned long long>() + 1;
    if (eps) CK(cudaMemsetAsync(ctx->mom.p, 0, sizeof(Fix128) * J * nparts * M * MOMW, st));
    // diagnostics: per-item timeline of the tree scan (env VPET_ITEMLOG=<file>)
    const char* ilog = tree ? getenv("VPET_ITEMLOG") : nullptr;
    const uint64_t nitems_dbg = ((J + 127) / 128) * nparts + 64;
    if (ilog) {
      CK(ctx->item_log.ensure(32 * nitems_dbg));
      CK(cudaMemsetAsync(ctx->item_log.p, 0, 32 * nitems_dbg, st));
      sp.item_log = ctx->item_log.as<unsigned long long>();
    }
    CK(ctx->dist_wl2() ? launch_scan_wl2(sp, LP, count_work, tree, st) : launch_scan_l1(sp, LP, count_work, tree, st));
    ++launches;
    if (ilog) {
      std::vector<unsigned long long> hl(4 * nitems_dbg);
      CK(cudaMemcpyAsync(hl.data(), ctx->item_log.p, 32 * nitems_dbg, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (FILE* fp = fopen(ilog, "wb")) {
        fwrite(hl.data(), 8, hl.size(), fp);
        fclose(fp);
      }
    }
  }
  rec(EV_SCAN);

  ReduceParams rp{};
  rp.K = K;
  rp.nparts = ((tree || dense) && !eps) ? nparts : 1;
  rp.tau_glob = ((tree || dense) && !eps) ? ctx->tau_glob.as<unsigned int>() : nullptr;
  rp.vslot = tree ? ctx->vslot.as<uint32_t>() : nullptr;  // tau_glob is slot-indexed in tree mode
  rp.heap = ctx->heap.as<unsigned long long>();
  rp.heap_cnt = ctx->heap_cnt.as<uint32_t>();
  rp.hd = ctx->hd.as<double>();
  rp.hidx = ctx->hidx.as<uint32_t>();
  rp.J = J;
  rp.n = n;
  rp.bank = ctx->bank.as<float>();
  rp.N = N;
  rp.L = L;
  rp.LS = LS;
  rp.LP = LP;
  rp.tacs = d_tacs;
  rp.w = ctx->d_w.as<float>();
  rp.dist = ctx->cfg.distance;
  rp.unit_w = ctx->unit_w;
  rp.eb = eb;
  rp.prior = ctx->prior;
  rp.P = P;
  rp.fb_list = ctx->fb_list.as<uint32_t>();
  rp.fb_len = ctx->fb_len.as<uint32_t>();
  rp.force_fb = (ctx->cfg.flags & ABC_FLAG_FORCE_FALLBACK) ? 1 : 0;
  rp.bad = ctx->flag.as<int>();
  // K3 / K4 split (warp layout only): the certification kernels write sorted accepted lists, one
  // reduction kernel then summarises every voxel (smaller kernels: fewer instruction-cache misses)
  static const bool split_env = getenv("VPET_SPLIT") ? atoi(getenv("VPET_SPLIT")) != 0 : true;  // tuning knob
  const bool split = split_env && !eps && certify_capacity(rp) <= kWarpCertifyMax;
  static const bool reg_sort_env = getenv("VPET_REG_SORT") ? atoi(getenv("VPET_REG_SORT")) != 0 : true;  // tuning knob
  rp.reg_sort = reg_sort_env ? 1 : 0;
  if (split) {
    rp.list_only = 1;
    rp.acc_i = ctx->hidx.as<uint32_t>();
    rp.acc_d = ctx->hd.as<double>();
  }
  if (cl_voxels) {
    rp.fb_tau = ctx->fb_tau.as<double>();
    rp.cl_d = ctx->cl_d.as<double>();
    rp.cl_i = ctx->cl_i.as<uint32_t>();
    rp.cl_cnt = ctx->cl_cnt.as<uint32_t>();
    rp.cl_cap = cl_cap;
    rp.cl_voxels = cl_voxels;
    rp.fb2_list = ctx->fb2_list.as<uint32_t>();
    rp.fb2_len = ctx->fb2_len.as<uint32_t>();
  }
  rp.out = dout;

  ExactParams xp{};
  xp.bank = ctx->bank.as<float>();
  xp.N = N;
  xp.L = L;
  xp.LS = LS;
  xp.tacs = d_tacs;
  xp.w = ctx->d_w.as<float>();
  xp.dist = ctx->cfg.distance;
  xp.n = n;
  xp.J = J;
  xp.hd = ctx->hd.as<double>();
  xp.hi = ctx->hidx.as<uint32_t>();
  xp.bad = ctx->flag.as<int>();

  if (eps) {
    EpsReduceParams ep{ctx->mom.as<Fix128>(), nparts, J, ctx->prior, P, dout};
    launch_eps_reduce(ep, st);
    ++launches;
    rec(EV_CERT);
    rec(EV_FB);
  } else if (exact) {
    launch_exact_scan(xp, st);
    rp.exact = 1;
    rp.list = nullptr;
    rp.list_len = nullptr;
    rec(EV_CERT);
    CK(launch_certify_reduce(rp, st));
    launches += 2;
    if (split) {
      CK(launch_reduce_accepted_lists(rp, ctx->hidx.as<uint32_t>(), ctx->hd.as<double>(), ctx->flag.as<int>(), st));
      ++launches;
    }
    rec(EV_FB);
  } else {
    rp.exact = 0;
    rp.list = nullptr;
    rp.list_len = nullptr;
    CK(launch_certify_reduce(rp, st));
    ++launches;
    rec(EV_CERT);
    // uncertified voxels (device-side list, no host sync).  Tier 2: every draw with D64 <= the seed
    // (the n-th FP64 distance among the voxel's candidates, >= tau64) is collected by a GPU-wide
    // FP64 scan, then sorted and reduced.  Tier 3 (seed unknown or list overflow): exact heap scan.
    ReduceParams rc = rp;
    rc.force_fb = 0;
    if (cl_voxels) {
      CollectParams cp{};
      cp.bank = ctx->bank.as<float>();
      cp.N = N;
      cp.L = L;
      cp.LS = LS;
      cp.tacs = d_tacs;
      cp.w = ctx->d_w.as<float>();
      cp.dist = ctx->cfg.distance;
      cp.list = ctx->fb_list.as<uint32_t>();
      cp.list_len = ctx->fb_len.as<uint32_t>();
      cp.tau = ctx->fb_tau.as<double>();
      cp.cap_voxels = cl_voxels;
      cp.cap = cl_cap;
      cp.nchunk = 2048;
      cp.cnt = ctx->cl_cnt.as<uint32_t>();
      cp.cd = ctx->cl_d.as<double>();
      cp.ci = ctx->cl_i.as<uint32_t>();
      cp.bad = ctx->flag.as<int>();
      launch_fallback_collect(cp, st);
      rc.exact = 2;
      rc.list = ctx->fb_list.as<uint32_t>();
      rc.list_len = ctx->fb_len.as<uint32_t>();
      rc.fb_list = nullptr;
      CK(launch_certify_reduce(rc, st));
      launches += 2;
      xp.list = ctx->fb2_list.as<uint32_t>();
      xp.list_len = ctx->fb2_len.as<uint32_t>();
    } else {
      xp.list = ctx->fb_list.as<uint32_t>();
      xp.list_len = ctx->fb_len.as<uint32_t>();
    }
    launch_exact_scan(xp, st);
    ReduceParams rx = rc;
    rx.exact = 1;
    rx.list = xp.list;
    rx.list_len = xp.list_len;
    rx.fb_list = nullptr;
    CK(launch_certify_reduce(rx, st));
    launches += 2;
    if (split && host_out && J >= kChunkedOutMin) {
      // K4 for every voxel, in chunks of voxels: the device-to-host copy of a chunk's outputs runs on
      // the copy stream while K4 reduces the next chunk (the copies are joined before the call ends)
      const int nch = abc_ctx::kOutChunks;
      const uint64_t per = (J + nch - 1) / nch;
      void* srcs[11] = {dout.prob, dout.preferred, dout.count, dout.mean, dout.sd, dout.q,
                        dout.ki_mean, dout.ki_sd, dout.ki_q, dout.acc_idx, dout.acc_dist};
      for (int c = 0; c < nch; ++c) {
        const uint64_t v0 = uint64_t(c) * per, nv = std::min<uint64_t>(per, J - std::min<uint64_t>(J, v0));
        if (nv == 0) break;
        ReduceParams rq = rp;
        rq.J = nv;
        abc_result& o = rq.out;
        if (o.prob) o.prob += v0 * M;
        if (o.preferred) o.preferred += v0;
        if (o.count) o.count += v0 * M;
        if (o.mean) o.mean += v0 * P;
        if (o.sd) o.sd += v0 * P;
        if (o.q) o.q += v0 * P * 3;
        if (o.ki_mean) o.ki_mean += v0;
        if (o.ki_sd) o.ki_sd += v0;
        if (o.ki_q) o.ki_q += v0 * 3;
        if (o.acc_idx) o.acc_idx += v0 * n;
        if (o.acc_dist) o.acc_dist += v0 * n;
        CK(launch_reduce_accepted_lists(rq, ctx->hidx.as<uint32_t>() + v0 * n, ctx->hd.as<double>() + v0 * n,
                                        ctx->flag.as<int>(), st));
        ++launches;
        CK(cudaEventRecord(ctx->ev_chunk[c], st));
        CK(cudaStreamWaitEvent(ctx->copy, ctx->ev_chunk[c], 0));
        for (int k = 0; k < 11; ++k) {
          if (!od[k].user || !srcs[k]) continue;
          const size_t row = od[k].bytes / J;
          CK(cudaMemcpyAsync(static_cast<char*>(od[k].user) + v0 * row, static_cast<char*>(srcs[k]) + v0 * row, nv * row,
                             cudaMemcpyDeviceToHost, ctx->copy));
        }
      }
      CK(cudaEventRecord(ctx->ev_join, ctx->copy));
      CK(cudaStreamWaitEvent(st, ctx->ev_join, 0));
      outs_copied = true;
    } else if (split) {  // K4 for every voxel (certified or from a fallback tier)
      CK(launch_reduce_accepted_lists(rp, ctx->hidx.as<uint32_t>(), ctx->hd.as<double>(), ctx->flag.as<int>(), st));
      ++launches;
    }
    rec(EV_FB);
  }
  CK(cudaGetLastError());
  if (host_out && !outs_copied) {
    void* srcs[11] = {dout.prob, dout.preferred, dout.count, dout.mean, dout.sd, dout.q,
                      dout.ki_mean, dout.ki_sd, dout.ki_q, dout.acc_idx, dout.acc_dist};
    for (int k = 0; k < 11; ++k)
      if (od[k].user && srcs[k]) CK(cudaMemcpyAsync(od[k].user, srcs[k], od[k].bytes, cudaMemcpyDeviceToHost, st));
  }
  rec(EV_D2H);
  h2 = hnow();
  int h_flag = 0;
  uint32_t h_fb = 0, h_fb2 = 0;
  unsigned long long h_work[2] = {0, 0};
  CK(cudaMemcpyAsync(&h_flag, ctx->flag.p, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&h_fb, ctx->fb_len.p, 4, cudaMemcpyDeviceToHost, st));
  if (cl_voxels && !exact && !eps) CK(cudaMemcpyAsync(&h_fb2, ctx->fb2_len.p, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(h_work, ctx->work.p, 16, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  h3 = hnow();
  if (host_dbg) fprintf(stderr, "host: tables %.3f plan+alloc %.3f prep %.3f enqueue %.3f wait %.3f ms\n", h_tab - h0, h_alloc - h_tab, h1 - h_alloc, h2 - h1, h3 - h2);
  S.gpu_launches = launches;
  S.n_fallback = h_fb;
  S.n_fallback_exact = cl_voxels ? h_fb2 : h_fb;
  if (getenv("VPET_UNION_STATS") || getenv("VPET_PUSH_STATS") || getenv("VPET_TRAV_STATS")) {  // diagnostic counters of a VPET_UNION_STATS build (scan_kernels.cuh)
    unsigned long long u[2] = {0, 0};
    CK(cudaMemcpy(u, static_cast<unsigned long long*>(ctx->work.p) + 2, 16, cudaMemcpyDeviceToHost));
    unsigned long long w1 = 0;
    CK(cudaMemcpy(&w1, static_cast<unsigned long long*>(ctx->work.p) + 1, 8, cudaMemcpyDeviceToHost));
    fprintf(stderr, "diag counters: work[1]>>32 %llu, work[2] %llu, work[3] %llu (union: evaluated / alive voxel-lane "
            "tiles; push: pushes in work[3]; trav: super-tiles checked / passed / tiles loaded)\n", w1 >> 32, u[0], u[1]);
  }
  S.frame_updates = h_work[0];
  S.bound_updates = h_work[1];
  if (timing) {
    auto ms = [&](int a, int b) {
      float x = 0.0f;
      cudaEventElapsedTime(&x, ctx->ev[a], ctx->ev[b]);
      return double(x);
    };
    S.ms_h2d = ms(EV_START, EV_H2D);
    S.ms_bank = ms(EV_H2D, EV_BANK);
    S.ms_order = ms(EV_BANK, EV_ORDER);
    S.ms_scan = ms(EV_ORDER, EV_SCAN);
    S.ms_certify = ms(EV_SCAN, EV_CERT);
    S.ms_fallback = ms(EV_CERT, EV_FB);
    S.ms_d2h = ms(EV_FB, EV_D2H);
    S.ms_total = ms(EV_START, EV_D2H);
  }
  if (h_flag) return fail(ctx, ABC_E_ARG, "non-finite TAC value");
  return ABC_OK;
}

abc_status abc_model_select(abc_ctx* ctx, const float* tacs, uint64_t J, uint32_t ptr_flags, float* prob,
                            int32_t* preferred) {
  abc_result r;
  std::memset(&r, 0, sizeof r);
  r.prob = prob;
  r.preferred = preferred;
  return abc_run_voxels(ctx, tacs, J, ptr_flags, &r);
}

// int_t0^t1 of the input function (host, FP64): Feng closed form, or exact trapezoids of the PWL
// curve between t0, the knots inside and t1 (held at the last value after the last knot).
static double input_integral_host(const abc_ctx* c, double t0, double t1) {
  if (c->input_kind == ABC_INPUT_FENG) return feng_frame_integral(c->feng, t0, t1);
  double s = 0.0, a = t0, va = pwl_at(c->kt, c->kc, t0);
  for (size_t k = 0; k < c->kt.size(); ++k) {
    if (c->kt[k] <= t0) continue;
    if (c->kt[k] >= t1) break;
    s += 0.5 * (c->kt[k] - a) * (va + c->kc[k]);
    a = c->kt[k];
    va = c->kc[k];
  }
  return s + 0.5 * (t1 - a) * (va + pwl_at(c->kt, c->kc, t1));
}

abc_status abc_patlak(abc_ctx* ctx, const float* tacs, uint64_t J, double t_star_min, uint32_t ptr_flags, float* ki,
                      float* intercept) {
  if (!ctx) return ABC_E_ARG;
  if (!ctx->have_input || !ctx->have_frames) return fail(ctx, ABC_E_STATE, "input function and frames must be set");
  if (ptr_flags & ~(ABC_PTR_TACS_DEVICE | ABC_PTR_OUT_DEVICE)) return fail(ctx, ABC_E_ARG, "unknown ptr_flags");
  if (J == 0) return ABC_OK;
  if (!tacs || !ki || !std::isfinite(t_star_min)) return fail(ctx, ABC_E_ARG, "bad Patlak arguments");
  const uint32_t L = ctx->L;
  // frame coefficients (draw- and voxel-independent): centred OLS as two dot products
  std::vector<double> cp(L), x(L), ab(2 * L, 0.0);
  uint32_t m = 0, f0 = L;
  for (uint32_t f = 0; f < L; ++f) {
    const double tm = ctx->fs[f] + 0.5 * ctx->fd[f];
    cp[f] = input_integral_host(ctx, ctx->fs[f], ctx->fs[f] + ctx->fd[f]) / ctx->fd[f];
    x[f] = input_integral_host(ctx, 0.0, tm) / cp[f];
    if (tm >= t_star_min) {
      ++m;
      f0 = std::min(f0, f);
    }
  }
  double xb = 0.0, sxx = 0.0;
  for (uint32_t f = 0; f < L; ++f)
    if (ctx->fs[f] + 0.5 * ctx->fd[f] >= t_star_min) xb += x[f];
  xb = m ? xb / m : 0.0;
  for (uint32_t f = 0; f < L; ++f)
    if (ctx->fs[f] + 0.5 * ctx->fd[f] >= t_star_min) sxx += (x[f] - xb) * (x[f] - xb);
  const bool valid = m >= 2 && sxx > 0.0;
  for (uint32_t f = 0; f < L; ++f)
    if (valid && ctx->fs[f] + 0.5 * ctx->fd[f] >= t_star_min) {
      ab[f] = (x[f] - xb) / (sxx * cp[f]);
      ab[L + f] = 1.0 / (double(m) * cp[f]);
    }
  CK(cudaSetDevice(ctx->dev));
  const cudaStream_t st = ctx->stream;
  CK(upload(ctx->pat_ab, ab));
  const float* d_tacs = tacs;
  if (!(ptr_flags & ABC_PTR_TACS_DEVICE)) {
    CK(ctx->tacs.ensure(sizeof(float) * J * L));
    CK(cudaMemcpyAsync(ctx->tacs.p, tacs, sizeof(float) * J * L, cudaMemcpyHostToDevice, st));
    d_tacs = ctx->tacs.as<float>();
  }
  const bool dev_out = ptr_flags & ABC_PTR_OUT_DEVICE;
  float* d_ki = ki;
  float* d_ic = intercept;
  if (!dev_out) {
    CK(ctx->env_q.ensure(8 * J));
    d_ki = ctx->env_q.as<float>();
    d_ic = intercept ? d_ki + J : nullptr;
  }
  PatlakParams pp{d_tacs, J, L, f0 < L ? f0 : 0, ctx->pat_ab.as<double>(), ctx->pat_ab.as<double>() + L, xb,
                  valid ? 1 : 0, d_ki, d_ic};
  launch_patlak(pp, st);
  CK(cudaGetLastError());
  if (!dev_out) {
    CK(cudaMemcpyAsync(ki, d_ki, 4 * J, cudaMemcpyDeviceToHost, st));
    if (intercept) CK(cudaMemcpyAsync(intercept, d_ic, 4 * J, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  return ABC_OK;
}

abc_status abc_set_sim_noise(abc_ctx* ctx, double ell, double half_life_min) {
  if (!ctx) return ABC_E_ARG;
  if (!std::isfinite(ell) || ell < 0.0) return fail(ctx, ABC_E_ARG, "noise level must be finite and >= 0");
  if (!(half_life_min > 0.0)) return fail(ctx, ABC_E_ARG, "half-life must be > 0 (may be +inf)");
  ctx->noise_ell = ell;
  ctx->noise_lam = std::log(2.0) / half_life_min;
  return ABC_OK;
}

abc_status abc_response_envelope(abc_ctx* ctx, const uint64_t* acc_idx, uint64_t J, uint32_t n_acc,
                                 const double* t_min, uint32_t T, uint32_t ptr_flags, float* q) {
  if (!ctx) return ABC_E_ARG;
  if (ptr_flags & ~(ABC_PTR_TACS_DEVICE | ABC_PTR_OUT_DEVICE)) return fail(ctx, ABC_E_ARG, "unknown ptr_flags");
  if (J == 0) return ABC_OK;
  if (!acc_idx || !t_min || !q || n_acc == 0 || n_acc > 4096 || T == 0 || T > 1024)
    return fail(ctx, ABC_E_ARG, "bad envelope arguments");
  bool has_lp = false;
  for (uint32_t m = 0; m < ctx->M; ++m) has_lp |= ctx->prior.m[m].kind == ABC_LPNTPET;
  if (!has_lp) return fail(ctx, ABC_E_UNSUPPORTED, "no lp-ntPET model in the context");
  for (uint32_t k = 0; k < T; ++k)
    if (!std::isfinite(t_min[k])) return fail(ctx, ABC_E_ARG, "non-finite time");
  CK(cudaSetDevice(ctx->dev));
  const cudaStream_t st = ctx->stream;
  const bool dev_idx = ptr_flags & ABC_PTR_TACS_DEVICE, dev_out = ptr_flags & ABC_PTR_OUT_DEVICE;
  const uint64_t* d_idx = acc_idx;
  if (!dev_idx) {
    CK(ctx->env_idx.ensure(8 * J * n_acc));
    CK(cudaMemcpyAsync(ctx->env_idx.p, acc_idx, 8 * J * n_acc, cudaMemcpyHostToDevice, st));
    d_idx = ctx->env_idx.as<uint64_t>();
  }
  CK(ctx->env_t.ensure(8 * T));
  CK(cudaMemcpyAsync(ctx->env_t.p, t_min, 8 * T, cudaMemcpyHostToDevice, st));
  float* d_q = q;
  if (!dev_out) {
    CK(ctx->env_q.ensure(12 * J * T));
    d_q = ctx->env_q.as<float>();
  }
  CK(ctx->flag.ensure(16));
  CK(cudaMemsetAsync(ctx->flag.p, 0, 16, st));
  EnvelopeParams ep{d_idx, J, ctx->N, n_acc, T, ctx->env_t.as<double>(), ctx->prior, d_q, ctx->flag.as<int>()};
  CK(launch_response_envelope(ep, st));
  if (!dev_out) CK(cudaMemcpyAsync(q, d_q, 12 * J * T, cudaMemcpyDeviceToHost, st));
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, ctx->flag.p, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (bad) return fail(ctx, ABC_E_ARG, "draw index out of range");
  return ABC_OK;
}

abc_status abc_reduce_accepted(abc_ctx* ctx, const uint64_t* acc_idx, uint64_t J, uint32_t n_acc, uint32_t n_use,
                               uint32_t ptr_flags, abc_result* out) {
  if (!ctx || !out) return ABC_E_ARG;
  if (ptr_flags & ~(ABC_PTR_TACS_DEVICE | ABC_PTR_OUT_DEVICE)) return fail(ctx, ABC_E_ARG, "unknown ptr_flags");
  if (J == 0) return ABC_OK;
  if (!acc_idx || n_acc == 0 || n_use == 0 || n_use > n_acc || n_use > 4096)
    return fail(ctx, ABC_E_ARG, "need 1 <= n_use <= n_acc, n_use <= 4096");
  if (out->acc_dist) return fail(ctx, ABC_E_ARG, "acc_dist is not produced by abc_reduce_accepted");
  CK(cudaSetDevice(ctx->dev));
  const cudaStream_t st = ctx->stream;
  const uint32_t M = ctx->M, P = ctx->P;
  const bool dev_idx = ptr_flags & ABC_PTR_TACS_DEVICE, host_out = !(ptr_flags & ABC_PTR_OUT_DEVICE);
  const uint64_t* d_idx = acc_idx;
  if (!dev_idx) {
    CK(ctx->env_idx.ensure(8 * J * n_acc));
    CK(cudaMemcpyAsync(ctx->env_idx.p, acc_idx, 8 * J * n_acc, cudaMemcpyHostToDevice, st));
    d_idx = ctx->env_idx.as<uint64_t>();
  }
  struct OutDesc { void* user; size_t bytes; };
  OutDesc od[10] = {{out->prob, 4 * J * M},       {out->preferred, 4 * J},  {out->count, 4 * J * M},
                    {out->mean, 4 * J * P},       {out->sd, 4 * J * P},     {out->q, 12 * J * P},
                    {out->ki_mean, 4 * J},        {out->ki_sd, 4 * J},      {out->ki_q, 12 * J},
                    {out->acc_idx, 8 * J * n_use}};
  abc_result dout = *out;
  if (host_out) {
    size_t tot = 0;
    for (auto& d : od) if (d.user) tot += (d.bytes + 255) & ~size_t(255);
    CK(ctx->env_q.ensure(tot ? tot : 16));
    void** fields[10] = {(void**)&dout.prob, (void**)&dout.preferred, (void**)&dout.count, (void**)&dout.mean,
                         (void**)&dout.sd,   (void**)&dout.q,         (void**)&dout.ki_mean, (void**)&dout.ki_sd,
                         (void**)&dout.ki_q, (void**)&dout.acc_idx};
    size_t off = 0;
    for (int k = 0; k < 10; ++k) {
      *fields[k] = od[k].user ? ctx->env_q.as<char>() + off : nullptr;
      if (od[k].user) off += (od[k].bytes + 255) & ~size_t(255);
    }
  }
  CK(ctx->flag.ensure(16));
  CK(cudaMemsetAsync(ctx->flag.p, 0, 16, st));
  ReduceParams rp{};
  rp.J = J;
  rp.n = n_use;
  rp.N = ctx->N;
  rp.prior = ctx->prior;
  rp.P = P;
  rp.out = dout;
  CK(launch_reduce_list(rp, d_idx, n_acc, ctx->flag.as<int>(), st));
  if (host_out) {
    void* srcs[10] = {dout.prob, dout.preferred, dout.count, dout.mean, dout.sd, dout.q,
                      dout.ki_mean, dout.ki_sd, dout.ki_q, dout.acc_idx};
    for (int k = 0; k < 10; ++k)
      if (od[k].user) CK(cudaMemcpyAsync(od[k].user, srcs[k], od[k].bytes, cudaMemcpyDeviceToHost, st));
  }
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, ctx->flag.p, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (bad) return fail(ctx, ABC_E_ARG, "draw index out of range");
  return ABC_OK;
}

abc_status abc_get_bank(const abc_ctx* ctx_c, float* out, uint64_t first, uint64_t count) {
  abc_ctx* ctx = const_cast<abc_ctx*>(ctx_c);
  if (!ctx || !out) return ABC_E_ARG;
  if (!ctx->bank_valid) return fail(ctx, ABC_E_STATE, "no bank: run first");
  if (first > ctx->N || count > ctx->N - first) return fail(ctx, ABC_E_ARG, "bank rows out of range");
  CK(cudaSetDevice(ctx->dev));
  const uint32_t LS = (ctx->bank_L + 3) & ~3u;
  CK(cudaMemcpy2D(out, sizeof(float) * ctx->bank_L, ctx->bank.as<float>() + first * LS, sizeof(float) * LS,
                  sizeof(float) * ctx->bank_L, count, cudaMemcpyDeviceToHost));
  return ABC_OK;
}

const char* abc_last_error(const abc_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void abc_destroy(abc_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->dev);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  DevBuf* bufs2[] = {&ctx->fmean, &ctx->cov, &ctx->pcs, &ctx->pminmax, &ctx->keys, &ctx->keys_alt, &ctx->vals,
                     &ctx->order, &ctx->idxmap, &ctx->sort_temp, &ctx->tbounds, &ctx->sbounds, &ctx->hbounds, &ctx->tau_glob, &ctx->rotq, &ctx->ytr, &ctx->gbox,
                     &ctx->queue, &ctx->vkeys, &ctx->vkeys_alt, &ctx->vvals, &ctx->vorder, &ctx->vslot, &ctx->vsort_temp, &ctx->item_log,
                     &ctx->dBt, &ctx->dS2, &ctx->dAt, &ctx->dY2,
                     &ctx->env_idx, &ctx->env_t, &ctx->env_q, &ctx->proj, &ctx->pat_ab,
                     &ctx->fb_tau, &ctx->cl_d, &ctx->cl_i, &ctx->cl_cnt, &ctx->fb2_list, &ctx->fb2_len};
  for (DevBuf* b : bufs2) b->release();
  DevBuf* bufs[] = {&ctx->d_finv, &ctx->d_s0, &ctx->d_prior, &ctx->d_fdur, &ctx->d_fs,  &ctx->d_fe,   &ctx->d_favg, &ctx->d_w,        &ctx->d_wsc, &ctx->d_cwd,
                    &ctx->d_gt,   &ctx->d_gc,  &ctx->d_gframe, &ctx->d_gcode, &ctx->d_ft, &ctx->d_fc,       &ctx->d_fframe,
                    &ctx->bank,   &ctx->bankp, &ctx->var,    &ctx->perm,   &ctx->wsp,        &ctx->heap,
                    &ctx->heap_cnt, &ctx->tacs, &ctx->fb_list, &ctx->fb_len, &ctx->work,     &ctx->hd,
                    &ctx->hidx,   &ctx->mom,   &ctx->flag,   &ctx->outs};
  for (DevBuf* b : bufs) b->release();
  for (int k = 0; k < EV_N; ++k)
    if (ctx->ev[k]) cudaEventDestroy(ctx->ev[k]);
  if (ctx->own) cudaStreamDestroy(ctx->own);
  if (ctx->copy) cudaStreamDestroy(ctx->copy);
  if (ctx->aux) cudaStreamDestroy(ctx->aux);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  for (auto& e : ctx->ev_chunk)
    if (e) cudaEventDestroy(e);
  if (ctx->tacs_ready) cudaEventDestroy(ctx->tacs_ready);
  delete ctx;
}

}  // extern "C"
