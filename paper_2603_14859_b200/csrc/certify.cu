// certify.cu -- K3 certification + K4 posterior reduction, the exact FP64 scan used as the
// fallback (and as ABC_FLAG_EXACT), and the eps-mode reduction.
//
// K3 (warp per voxel): the FP32 pass left K = n + slack candidates (D32, i) per voxel.  Each is
// re-scored in FP64 exactly as the oracle scores it (acquisition frame order, no contraction),
// sorted by (D64, i) (ties -> lower index) and the first n kept.  The selection is
// certified when every draw the FP32 pass excluded -- all have D32 >= tauK32, the largest kept
// D32 -- provably has D > tau64 = the n-th D64:  tauK32 > tau64 + err(tau64) with err the
// rigorous FP32 error bound.  Uncertified voxels go to the exact scan.
// K4: per-model counts and probabilities, the preferred model (>50 %, P:282;
// ties -> model 0), conditional mean, SD (ddof 1) and type-7 quantiles of every column over
// the accepted draws of the preferred model, and K_i = K1 k3/(k2+k3).
#include <cfloat>
#include <cstdlib>

#include "common.cuh"

namespace vpet {
namespace {

// FP64 distance of one candidate, term by term in acquisition frame order as the oracle computes
// it (no contraction).  The bank row is read as float4 (rows are LS = L rounded up to 4 floats,
// 16-B aligned; w is a 16-B aligned device array): a quarter of the divergent row loads.
__device__ __forceinline__ double exact_distance_v(const float* y, const float* s, const float* w, uint32_t L,
                                                   int dist) {
  const float4* s4 = reinterpret_cast<const float4*>(s);
  const float4* w4 = reinterpret_cast<const float4*>(w);
  double D = 0.0;
  auto term = [&](float yv, float sv, float wv) {
    const double d = __dsub_rn(double(yv), double(sv));
    const double t = (dist == ABC_DIST_L1) ? fabs(d) : __dmul_rn(d, d);
    D = __dadd_rn(D, __dmul_rn(double(wv), t));
  };
  uint32_t f = 0;
#pragma unroll 2
  for (; f + 4 <= L; f += 4) {
    const float4 sv = __ldg(s4 + f / 4), wv = __ldg(w4 + f / 4);
    term(__ldg(y + f), sv.x, wv.x);
    term(__ldg(y + f + 1), sv.y, wv.y);
    term(__ldg(y + f + 2), sv.z, wv.z);
    term(__ldg(y + f + 3), sv.w, wv.w);
  }
  for (; f < L; ++f) term(__ldg(y + f), __ldg(s + f), __ldg(w + f));
  return D;
}

__device__ __forceinline__ bool pair_gt(double a, uint32_t ia, double b, uint32_t ib) {
  return a > b || (a == b && ia > ib);
}

// Append voxel v to the fallback list with the seed threshold tau (see ReduceParams).
__device__ __forceinline__ void push_fb(const ReduceParams& p, uint32_t v, double tau) {
  const uint32_t pos = atomicAdd(p.fb_len, 1u);
  p.fb_list[pos] = v;
  if (p.fb_tau) p.fb_tau[pos] = tau;
}
__device__ __forceinline__ void push_fb2(const ReduceParams& p, uint32_t v) { p.fb2_list[atomicAdd(p.fb2_len, 1u)] = v; }

// bitonic sort of (key, idx) pairs, ascending, n2 a power of two, one warp
__device__ void warp_sort_pairs(double* key, uint32_t* idx, uint32_t n2, int lane) {
  for (uint32_t size = 2; size <= n2; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = lane; i < n2; i += 32) {
        uint32_t j = i ^ stride;
        if (j > i) {
          bool asc = (i & size) == 0;
          double a = key[i], b = key[j];
          uint32_t ia = idx[i], ib = idx[j];
          bool swap = asc ? pair_gt(a, ia, b, ib) : pair_gt(b, ib, a, ia);
          if (swap) {
            key[i] = b; key[j] = a;
            idx[i] = ib; idx[j] = ia;
          }
        }
      }
      __syncwarp();
    }
  }
}

__device__ void warp_sort_keys(double* key, uint32_t n2, int lane) {
  for (uint32_t size = 2; size <= n2; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t i = lane; i < n2; i += 32) {
        uint32_t j = i ^ stride;
        if (j > i) {
          bool asc = (i & size) == 0;
          double a = key[i], b = key[j];
          if (asc ? (a > b) : (a < b)) {
            key[i] = b;
            key[j] = a;
          }
        }
      }
      __syncwarp();
    }
  }
}

// Register bitonic sorts of 32 * E elements (element g = e * 32 + lane), ascending.
template <int E, bool PAIRS>
__device__ __forceinline__ void warp_sort_reg(double (&k)[E], uint32_t (&ix)[E], int lane) {
#pragma unroll
  for (uint32_t size = 2; size <= 32u * E; size <<= 1) {
#pragma unroll
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 32) {
        const uint32_t es = stride / 32;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int e2 = e ^ int(es);
          if (e2 > e) {
            const uint32_t g = uint32_t(e) * 32 + lane;
            const bool asc = (g & size) == 0;
            const bool gt = PAIRS ? pair_gt(k[e], ix[e], k[e2], ix[e2]) : (k[e] > k[e2]);
            if (gt == asc) {
              double t = k[e]; k[e] = k[e2]; k[e2] = t;
              uint32_t u = ix[e]; ix[e] = ix[e2]; ix[e2] = u;
            }
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const uint32_t g = uint32_t(e) * 32 + lane;
          const double ok = __shfl_xor_sync(0xffffffffu, k[e], stride);
          const uint32_t oi = __shfl_xor_sync(0xffffffffu, ix[e], stride);
          const bool lower = (lane & stride) == 0;
          const bool asc = (g & size) == 0;
          // the lower position keeps the smaller element when ascending
          const bool mine_gt = PAIRS ? pair_gt(k[e], ix[e], ok, oi) : (k[e] > ok);
          const bool other_gt = PAIRS ? pair_gt(ok, oi, k[e], ix[e]) : (ok > k[e]);
          const bool take = (lower == asc) ? mine_gt : other_gt;
          if (take) { k[e] = ok; ix[e] = oi; }
        }
      }
    }
  }
}

template <int E>
__device__ void warp_sort_regs(double* key, uint32_t* idx, int lane) {
  double k[E];
  uint32_t ix[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    k[e] = key[e * 32 + lane];
    ix[e] = idx ? idx[e * 32 + lane] : 0u;
  }
  __syncwarp();
  if (idx) warp_sort_reg<E, true>(k, ix, lane);
  else warp_sort_reg<E, false>(k, ix, lane);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    key[e * 32 + lane] = k[e];
    if (idx) idx[e * 32 + lane] = ix[e];
  }
  __syncwarp();
}

// Sort n2 (power of two) smem keys (and indices if idx) ascending: registers for n2 <= 64.
__device__ void warp_sort_any(double* key, uint32_t* idx, uint32_t n2, int lane) {
  if (n2 <= 32) {
    double k[1];
    uint32_t ix[1];
    const bool in = uint32_t(lane) < n2;
    k[0] = in ? key[lane] : __longlong_as_double(0x7ff0000000000000ll);
    ix[0] = (in && idx) ? idx[lane] : 0xffffffffu;
    __syncwarp();
    if (idx) warp_sort_reg<1, true>(k, ix, lane);
    else warp_sort_reg<1, false>(k, ix, lane);
    if (in) {  // padding (+inf, 0xffffffff) sorts last and is never stored back
      key[lane] = k[0];
      if (idx) idx[lane] = ix[0];
    }
    __syncwarp();
  } else if (n2 == 64) {
    warp_sort_regs<2>(key, idx, lane);
  } else if (idx) {
    warp_sort_pairs(key, idx, n2, lane);
  } else {
    warp_sort_keys(key, n2, lane);
  }
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

__device__ __forceinline__ double quantile7(const double* x, uint32_t c, double q) {
  double h = double(c - 1) * q;
  uint32_t lo = uint32_t(floor(h));
  if (lo + 1 >= c) return x[c - 1];
  return x[lo] + (h - double(lo)) * (x[lo + 1] - x[lo]);
}

__device__ __forceinline__ bool column_exists(int kind, uint32_t k) {
  if (kind == ABC_MRTM) return k <= 3;
  return k < ((kind >= ABC_MRTM) ? 7u : 5u);
}

// Ascending bitonic sort of one value per lane across the warp; returns this lane's sorted value.
template <typename T>
__device__ __forceinline__ T warp_sort32(T x, int lane) {
#pragma unroll
  for (uint32_t size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      const T o = __shfl_xor_sync(0xffffffffu, x, stride);
      const bool lower = (uint32_t(lane) & stride) == 0, asc = (uint32_t(lane) & size) == 0;
      if ((lower == asc) ? (x > o) : (o > x)) x = o;
    }
  }
  return x;
}

// Reduce the sorted accepted list (ci[0..n)) of voxel v.  sc: np2 doubles of scratch.
__device__ void reduce_topn(const ReduceParams& p, uint64_t v, const uint32_t* ci, const double* cd, double* sc,
                            uint32_t np2, int lane) {
  const uint32_t n = p.n;
  const uint32_t M = p.prior.M;
  const abc_result& o = p.out;
  for (uint32_t a = lane; a < n; a += 32) {
    if (o.acc_idx) o.acc_idx[v * n + a] = ci[a];
    if (o.acc_dist && cd) o.acc_dist[v * n + a] = cd[a];
  }
  uint32_t cnt[ABC_MAX_MODELS] = {0, 0, 0, 0};
  for (uint32_t base = 0; base < n; base += 32) {
    uint32_t a = base + lane;
    int m = (a < n) ? model_index(p.prior, ci[a]) : -1;
#pragma unroll
    for (int k = 0; k < ABC_MAX_MODELS; ++k) cnt[k] += __popc(__ballot_sync(0xffffffffu, m == k));
  }
  int pref = 0;
  for (uint32_t m = 1; m < M; ++m)
    if (cnt[m] > cnt[pref]) pref = int(m);
  if (lane == 0) {
    for (uint32_t m = 0; m < M; ++m) {
      if (o.count) o.count[v * M + m] = cnt[m];
      if (o.prob) o.prob[v * M + m] = float(double(cnt[m]) / double(n));
    }
    if (o.preferred) o.preferred[v] = pref;
  }
  const int kind = p.prior.m[pref].kind;
  const uint32_t c = cnt[pref];
  const bool tcm = kind <= ABC_2TCM_REV;
  const float NANF = __int_as_float(0x7fc00000);
  // n <= 32: each lane draws the parameters of its accepted draw once, for all columns
  // n <= 32: each lane draws the parameters of its accepted draw once, for all columns
  const bool small = n <= 32;
  float thr[ABC_MAX_P];
  bool mine0 = false;
  uint32_t bal0 = 0;
  if (small) {
    mine0 = uint32_t(lane) < n && model_index(p.prior, ci[lane]) == pref;
    if (mine0) draw_theta(p.prior, ci[lane], thr);
    bal0 = __ballot_sync(0xffffffffu, mine0);
  }
  for (uint32_t k = 0; k <= p.P; ++k) {  // column P = K_i
    const bool is_ki = (k == p.P);
    if (is_ki && !tcm) {
      if (lane == 0) {
        if (o.ki_mean) o.ki_mean[v] = NANF;
        if (o.ki_sd) o.ki_sd[v] = NANF;
        if (o.ki_q) for (int t = 0; t < 3; ++t) o.ki_q[v * 3 + t] = NANF;
      }
      continue;
    }
    bool exists = c > 0 && (is_ki || column_exists(kind, k));
    float mean = NANF, sd = NANF, q3[3] = {NANF, NANF, NANF};
    if (exists) {
      uint32_t npos = 0;
      double sum = 0.0;
      if (small && p.reg_sort) {
        // n <= 32, one value per lane: sums by warp_sum (same order as below), the order statistics
        // by a register bitonic sort across the lanes -- FP32 for the parameter columns (the
        // values ARE FP32; half the shuffles of FP64), FP64 for K_i; +inf pads the other lanes
        const double x = !mine0 ? 0.0
                         : (is_ki ? double(thr[0]) * double(thr[2]) / (double(thr[1]) + double(thr[2])) : double(thr[k]));
        const double mu = warp_sum(x) / double(c);
        const double ss = warp_sum(mine0 ? (x - mu) * (x - mu) : 0.0);
        double xs;
        if (is_ki) {
          xs = warp_sort32<double>(mine0 ? x : __longlong_as_double(0x7ff0000000000000ll), lane);
        } else {
          xs = double(warp_sort32<float>(mine0 ? thr[k] : __int_as_float(0x7f800000), lane));
        }
        mean = float(mu);
        sd = c >= 2 ? float(sqrt(ss / double(c - 1))) : NANF;
        const double qs[3] = {0.025, 0.5, 0.975};
#pragma unroll
        for (int t = 0; t < 3; ++t) {
          const double h = double(c - 1) * qs[t];
          const uint32_t lo = uint32_t(floor(h));
          const uint32_t hi = lo + 1 < c ? lo + 1 : lo;
          const double xl = __shfl_sync(0xffffffffu, xs, int(lo));
          const double xh = __shfl_sync(0xffffffffu, xs, int(hi));
          q3[t] = float(lo + 1 < c ? xl + (h - double(lo)) * (xh - xl) : xl);
        }
      } else {
      if (small) {
        if (mine0) {
          double x = is_ki ? double(thr[0]) * double(thr[2]) / (double(thr[1]) + double(thr[2])) : double(thr[k]);
          sc[__popc(bal0 & ((1u << lane) - 1u))] = x;
          sum += x;
        }
        npos = __popc(bal0);
      }
      for (uint32_t base = 0; !small && base < n; base += 32) {
        uint32_t a = base + lane;
        bool mine = a < n && model_index(p.prior, ci[a]) == pref;
        uint32_t bal = __ballot_sync(0xffffffffu, mine);
        if (mine) {
          float th[ABC_MAX_P];
          draw_theta(p.prior, ci[a], th);
          double x = is_ki ? double(th[0]) * double(th[2]) / (double(th[1]) + double(th[2])) : double(th[k]);
          uint32_t pos = npos + __popc(bal & ((1u << lane) - 1u));
          sc[pos] = x;
          sum += x;
        }
        npos += __popc(bal);
      }
      sum = warp_sum(sum);
      double mu = sum / double(c);
      __syncwarp();
      double ss = 0.0;
      for (uint32_t a = lane; a < c; a += 32) ss += (sc[a] - mu) * (sc[a] - mu);
      ss = warp_sum(ss);
      uint32_t cp2 = 32;  // sort only the occupied power of two of this model's c values
      while (cp2 < c) cp2 <<= 1;
      for (uint32_t a = c + lane; a < cp2; a += 32) sc[a] = __longlong_as_double(0x7ff0000000000000ll);
      __syncwarp();
      warp_sort_any(sc, nullptr, cp2, lane);
      mean = float(mu);
      sd = c >= 2 ? float(sqrt(ss / double(c - 1))) : NANF;
      q3[0] = float(quantile7(sc, c, 0.025));
      q3[1] = float(quantile7(sc, c, 0.5));
      q3[2] = float(quantile7(sc, c, 0.975));
      __syncwarp();
      }
    }
    if (lane == 0) {
      if (is_ki) {
        if (o.ki_mean) o.ki_mean[v] = mean;
        if (o.ki_sd) o.ki_sd[v] = sd;
        if (o.ki_q) for (int t = 0; t < 3; ++t) o.ki_q[v * 3 + t] = q3[t];
      } else {
        if (o.mean) o.mean[v * p.P + k] = mean;
        if (o.sd) o.sd[v * p.P + k] = sd;
        if (o.q) for (int t = 0; t < 3; ++t) o.q[(v * p.P + k) * 3 + t] = q3[t];
      }
    }
  }
}

#ifndef CERT_MINB
#define CERT_MINB 4  // 4 CTAs of 8 warps per SM (<= 64 registers)
#endif
__global__ void __launch_bounds__(256, CERT_MINB) certify_reduce_kernel(const ReduceParams p, uint32_t Kp, uint32_t np2, uint32_t wpc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const uint32_t w = threadIdx.x >> 5;
  const size_t per_warp = size_t(Kp) * 12 + size_t(np2) * 8;
  double* cd = reinterpret_cast<double*>(smem_raw + per_warp * w);
  double* sc = cd + Kp;
  uint32_t* ci = reinterpret_cast<uint32_t*>(sc + np2);
  if (p.bad && *p.bad) return;  // non-finite TACs: no results (ABC_E_ARG)
  const uint64_t len = p.list_len ? uint64_t(*p.list_len) : p.J;
  const uint64_t nwarps = uint64_t(gridDim.x) * wpc;
  const double DINF = __longlong_as_double(0x7ff0000000000000ll);
  for (uint64_t e = uint64_t(blockIdx.x) * wpc + w; e < len; e += nwarps) {
    const uint64_t v = p.list ? p.list[e] : e;
    const float* y = p.tacs + v * p.L;
    uint32_t cnt;
    float tK = __int_as_float(0x7f800000);
    if (p.exact == 2) {  // the draws with D64 <= fb_tau collected for this fallback entry
      cnt = e < p.cl_voxels ? p.cl_cnt[e] : 0xffffffffu;
      if (!(p.fb_tau[e] < DINF) || cnt > p.cl_cap || cnt > Kp || cnt < p.n) {
        if (lane == 0) push_fb2(p, uint32_t(v));
        continue;
      }
      for (uint32_t a = lane; a < Kp; a += 32) {
        cd[a] = a < cnt ? p.cl_d[e * p.cl_cap + a] : DINF;
        ci[a] = a < cnt ? p.cl_i[e * p.cl_cap + a] : 0xffffffffu;
      }
    } else if (p.exact) {
      cnt = p.n;
      for (uint32_t a = lane; a < Kp; a += 32) {
        cd[a] = a < cnt ? p.hd[v * p.n + a] : DINF;
        ci[a] = a < cnt ? p.hidx[v * p.n + a] : 0xffffffffu;
      }
    } else {
      // Candidates: the keys of all parts' heaps with D32 <= B, where B bounds the D32 of every
      // draw the FP32 pass excluded (tau_glob in tree mode, the heap root in flat mode).
      const uint32_t S = p.nparts;
      float B = __int_as_float(0x7f800000);
      uint64_t total = 0;
      for (uint32_t q = 0; q < S; ++q) total += p.heap_cnt[v * S + q];
      if (p.tau_glob) {
        B = __uint_as_float(p.tau_glob[p.vslot ? p.vslot[v] : v]);
      } else if (p.heap_cnt[v] >= p.K) {
        float tmax = 0.0f;
        for (uint32_t a = lane; a < p.K; a += 32)
          tmax = fmaxf(tmax, __uint_as_float(uint32_t(p.heap[v * heap_stride(p.K) + kHeapOff + a] >> 32)));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
        B = tmax;
      }
      const bool complete = (total == p.N);  // every draw was kept: nothing excluded
      if (!complete && !(B < __int_as_float(0x7f800000))) {  // no finite bound (non-finite D32s)
        if (lane == 0) push_fb(p, uint32_t(v), DINF);
        continue;
      }
      uint32_t nc = 0;  // warp-uniform candidate count
      for (uint32_t q = 0; q < S; ++q) {
        const uint32_t cq = p.heap_cnt[v * S + q];
        const unsigned long long* h = p.heap + (v * S + q) * heap_stride(p.K) + kHeapOff;
        for (uint32_t base = 0; base < cq; base += 32) {
          uint32_t a = base + lane;
          unsigned long long key = a < cq ? h[a] : ~0ull;
          bool take = a < cq && __uint_as_float(uint32_t(key >> 32)) <= B;
          uint32_t bal = __ballot_sync(0xffffffffu, take);
          if (take) {
            uint32_t pos = nc + __popc(bal & ((1u << lane) - 1u));
            if (pos < Kp) ci[pos] = uint32_t(key & 0xffffffffull);
          }
          nc += __popc(bal);
        }
      }
      if (nc > Kp || nc < p.n) {  // capacity (or a degenerate bound): exact path
        if (lane == 0) push_fb(p, uint32_t(v), DINF);
        continue;
      }
      __syncwarp();
      for (uint32_t a = lane; a < Kp; a += 32) {
        if (a < nc) {
          cd[a] = exact_distance_v(y, p.bank + uint64_t(ci[a]) * p.LS, p.w, p.L, p.dist);
        } else {
          cd[a] = DINF;
          ci[a] = 0xffffffffu;
        }
      }
      tK = complete ? __int_as_float(0x7f800000) : B;
      cnt = nc;
    }
    __syncwarp();
    {
      uint32_t kp = 32;  // sort only the occupied power of two
      while (kp < cnt) kp <<= 1;
      warp_sort_any(cd, ci, kp < Kp ? kp : Kp, lane);
    }
    if (!p.exact && (tK < __int_as_float(0x7f800000) || p.force_fb)) {
      double Y2 = 0.0, Y1 = 0.0;
      for (uint32_t f = lane; f < p.L; f += 32) {
        double yv = __ldg(y + f), wv = __ldg(p.w + f);
        Y2 += wv * yv * yv;
        Y1 += wv * fabs(yv);
      }
      Y2 = warp_sum(Y2);
      Y1 = warp_sum(Y1);
      double t64 = cd[p.n - 1];
      double err = p.eb.a * t64 + p.eb.b * sqrt(Y2 * t64) + p.eb.c * Y2 + p.eb.d * Y1;
      bool ok = !p.force_fb && double(tK) > t64 + err;
      if (!ok) {  // t64 >= tau64: every accepted draw has D64 <= t64 (the collector's seed)
        if (lane == 0) push_fb(p, uint32_t(v), t64);
        continue;
      }
    }
    if (p.list_only) {  // K3 only: the (D, i)-sorted accepted list; K4 runs once for all voxels
      for (uint32_t a = lane; a < p.n; a += 32) {
        p.acc_i[v * p.n + a] = ci[a];
        p.acc_d[v * p.n + a] = cd[a];
      }
    } else {
      reduce_topn(p, v, ci, cd, sc, np2, lane);
    }
    __syncwarp();
  }
}

// =============================================================================================
// Large-n certification + reduction (K3/K4 for n up to kMaxAccept): one CTA of kLT threads per
// voxel, candidates in shared memory (up to kLargeMaxCand (D64, i) pairs = 196 KB), a CTA-wide
// bitonic sort of the candidates by (D64, i), and a CTA-wide sort of each column's values for the
// type-7 quantiles.  Same arithmetic and same
// certification test as the warp path (certify_reduce_kernel); only the parallel layout differs.
// =============================================================================================
constexpr int kLT = 512;

// Ascending bitonic sort of n2 (power of two) (key, idx) pairs by (key, idx), whole CTA.
__device__ void cta_sort_pairs(double* key, uint32_t* idx, uint32_t n2) {
  for (uint32_t size = 2; size <= n2; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t t = threadIdx.x; t < n2 / 2; t += blockDim.x) {
        const uint32_t i = 2 * t - (t & (stride - 1)), j = i + stride;
        const bool asc = (i & size) == 0;
        const double a = key[i], b = key[j];
        const uint32_t ia = idx[i], ib = idx[j];
        if (pair_gt(a, ia, b, ib) == asc) {
          key[i] = b; key[j] = a;
          idx[i] = ib; idx[j] = ia;
        }
      }
      __syncthreads();
    }
  }
}

// Ascending bitonic sort of n2 (power of two) doubles, whole CTA.
__device__ void cta_sort_keys(double* key, uint32_t n2) {
  for (uint32_t size = 2; size <= n2; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      for (uint32_t t = threadIdx.x; t < n2 / 2; t += blockDim.x) {
        const uint32_t i = 2 * t - (t & (stride - 1)), j = i + stride;
        const double a = key[i], b = key[j];
        if ((a > b) == ((i & size) == 0)) {
          key[i] = b;
          key[j] = a;
        }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ double cta_sum(double x, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  x = warp_sum(x);
  __syncthreads();
  if (lane == 0) red[warp] = x;
  __syncthreads();
  double t = 0.0;
  for (int w = 0; w < int(blockDim.x >> 5); ++w) t += red[w];  // fixed order: deterministic
  return t;
}

// theta columns of the Philox block that holds column k (one Philox4x32-10 call): block 0 = columns
// 0-3, block 1 = columns 4-7; same values as draw_theta (common.cuh).
__device__ __forceinline__ void theta_block(const PriorDev& pr, uint64_t i, int m, uint32_t blk, float th[ABC_MAX_P]) {
  const ModelDev& md = pr.m[m];
  uint32_t w[4];
  philox10(uint32_t(i), uint32_t(i >> 32), blk, kCtrTag, pr.seed_lo, pr.seed_hi, w);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int k = int(blk) * 4 + q;
    th[k] = (k < (int)md.P) ? fmaf(md.span[k], u01(w[q]), md.lo[k]) : 0.0f;
  }
  if (blk == 0 && (md.kind == ABC_2TCM_IRR || md.kind == ABC_MRTM)) th[3] = 0.0f;
  if (blk == 1 && md.kind >= ABC_MRTM) th[5] = __fadd_rn(th[4], th[5]);
}

__global__ void __launch_bounds__(kLT, 2) certify_large_kernel(const ReduceParams p, uint32_t Kp) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* cd = reinterpret_cast<double*>(smem_raw);          // [Kp] D64 (later: uint64 value keys)
  uint32_t* ci = reinterpret_cast<uint32_t*>(cd + Kp);       // [Kp] draw indices
  uint32_t* sc = ci + Kp;                                    // [16] counters / broadcasts
  double* red = reinterpret_cast<double*>(sc + 16);          // [kLT / 32]
  if (p.bad && *p.bad) return;
  const int lane = threadIdx.x & 31;
  const uint64_t len = p.list_len ? uint64_t(*p.list_len) : p.J;
  const double DINF = __longlong_as_double(0x7ff0000000000000ll);
  const float NANF = __int_as_float(0x7fc00000);
  const abc_result& o = p.out;
  for (uint64_t e = blockIdx.x; e < len; e += gridDim.x) {
    const uint64_t v = p.list ? p.list[e] : e;
    const float* y = p.tacs + v * p.L;
    uint32_t cnt = 0;
    float tK = __int_as_float(0x7f800000);
    if (p.exact == 2) {  // the draws with D64 <= fb_tau collected for this fallback entry
      cnt = e < p.cl_voxels ? p.cl_cnt[e] : 0xffffffffu;
      if (!(p.fb_tau[e] < DINF) || cnt > p.cl_cap || cnt > Kp || cnt < p.n) {
        if (threadIdx.x == 0) push_fb2(p, uint32_t(v));
        __syncthreads();
        continue;
      }
      for (uint32_t a = threadIdx.x; a < Kp; a += kLT) {
        cd[a] = a < cnt ? p.cl_d[e * p.cl_cap + a] : DINF;
        ci[a] = a < cnt ? p.cl_i[e * p.cl_cap + a] : 0xffffffffu;
      }
    } else if (p.exact) {
      cnt = p.n;
      for (uint32_t a = threadIdx.x; a < Kp; a += kLT) {
        cd[a] = a < cnt ? p.hd[v * p.n + a] : DINF;
        ci[a] = a < cnt ? p.hidx[v * p.n + a] : 0xffffffffu;
      }
    } else {
      const uint32_t S = p.nparts;
      float B = __int_as_float(0x7f800000);
      uint64_t total = 0;
      for (uint32_t q = 0; q < S; ++q) total += p.heap_cnt[v * S + q];
      if (p.tau_glob) {
        B = __uint_as_float(p.tau_glob[p.vslot ? p.vslot[v] : v]);
      } else if (p.heap_cnt[v] >= p.K) {  // flat mode: the root of the single heap is its maximum
        B = __uint_as_float(uint32_t(p.heap[v * heap_stride(p.K) + kHeapOff] >> 32));
      }
      const bool complete = (total == p.N);
      bool to_fb = !complete && !(B < __int_as_float(0x7f800000));
      if (!to_fb) {
        if (threadIdx.x == 0) sc[0] = 0;
        __syncthreads();
        for (uint32_t q = 0; q < S; ++q) {
          const uint32_t cq = p.heap_cnt[v * S + q];
          const unsigned long long* h = p.heap + (v * S + q) * heap_stride(p.K) + kHeapOff;
          for (uint32_t a = threadIdx.x; a < cq; a += kLT) {
            const unsigned long long key = h[a];
            if (__uint_as_float(uint32_t(key >> 32)) <= B) {
              const uint32_t pos = atomicAdd(&sc[0], 1u);
              if (pos < Kp) ci[pos] = uint32_t(key & 0xffffffffull);
            }
          }
        }
        __syncthreads();
        cnt = sc[0];
        to_fb = cnt > Kp || cnt < p.n;
      }
      if (to_fb) {
        if (threadIdx.x == 0) push_fb(p, uint32_t(v), DINF);
        __syncthreads();
        continue;
      }
      for (uint32_t a = threadIdx.x; a < Kp; a += kLT) {
        if (a < cnt) {
          cd[a] = exact_distance_v(y, p.bank + uint64_t(ci[a]) * p.LS, p.w, p.L, p.dist);
        } else {
          cd[a] = DINF;
          ci[a] = 0xffffffffu;
        }
      }
      tK = complete ? __int_as_float(0x7f800000) : B;
    }
    __syncthreads();
    {
      uint32_t kp = 2;
      while (kp < cnt) kp <<= 1;
      cta_sort_pairs(cd, ci, kp < Kp ? kp : Kp);
    }
    if (!p.exact && (tK < __int_as_float(0x7f800000) || p.force_fb)) {
      double Y2 = 0.0, Y1 = 0.0;
      for (uint32_t f = threadIdx.x; f < p.L; f += kLT) {
        const double yv = __ldg(y + f), wv = __ldg(p.w + f);
        Y2 += wv * yv * yv;
        Y1 += wv * fabs(yv);
      }
      Y2 = cta_sum(Y2, red);
      Y1 = cta_sum(Y1, red);
      const double t64 = cd[p.n - 1];
      const double err = p.eb.a * t64 + p.eb.b * sqrt(Y2 * t64) + p.eb.c * Y2 + p.eb.d * Y1;
      if (p.force_fb || !(double(tK) > t64 + err)) {
        if (threadIdx.x == 0) push_fb(p, uint32_t(v), t64);
        __syncthreads();
        continue;
      }
    }
    // ---- K4: reduce the accepted (D, i)-sorted list ci[0..n) ----
    const uint32_t n = p.n, M = p.prior.M;
    for (uint32_t a = threadIdx.x; a < n; a += kLT) {
      if (o.acc_idx) o.acc_idx[v * n + a] = ci[a];
      if (o.acc_dist) o.acc_dist[v * n + a] = cd[a];
    }
    if (threadIdx.x < ABC_MAX_MODELS) sc[4 + threadIdx.x] = 0;
    __syncthreads();
    for (uint32_t a = threadIdx.x; a < n; a += kLT) atomicAdd(&sc[4 + model_index(p.prior, ci[a])], 1u);
    __syncthreads();
    uint32_t cntm[ABC_MAX_MODELS];
    for (int m = 0; m < ABC_MAX_MODELS; ++m) cntm[m] = sc[4 + m];
    int pref = 0;
    for (uint32_t m = 1; m < M; ++m)
      if (cntm[m] > cntm[pref]) pref = int(m);
    if (threadIdx.x == 0) {
      for (uint32_t m = 0; m < M; ++m) {
        if (o.count) o.count[v * M + m] = cntm[m];
        if (o.prob) o.prob[v * M + m] = float(double(cntm[m]) / double(n));
      }
      if (o.preferred) o.preferred[v] = pref;
    }
    const int kind = p.prior.m[pref].kind;
    const uint32_t c = cntm[pref];
    const bool tcm = kind <= ABC_2TCM_REV;
    double* xv = cd;  // the distances are written out: reuse the space for the column values
    uint32_t np2 = 2;
    while (np2 < n) np2 <<= 1;
    __syncthreads();
    for (uint32_t k = 0; k <= p.P; ++k) {  // column P = K_i
      const bool is_ki = (k == p.P);
      float mean = NANF, sd = NANF, q3[3] = {NANF, NANF, NANF};
      const bool exists = c > 0 && (is_ki ? tcm : column_exists(kind, k));
      if (exists) {
        const uint32_t blk = (is_ki || k < 4) ? 0u : 1u;
        double sum = 0.0;
        for (uint32_t a = threadIdx.x; a < np2; a += kLT) {
          double x = DINF;  // other models (and padding) sort last
          if (a < n) {
            const uint32_t i = ci[a];
            if (model_index(p.prior, i) == pref) {
              float th[ABC_MAX_P];
              theta_block(p.prior, i, pref, blk, th);
              x = is_ki ? double(th[0]) * double(th[2]) / (double(th[1]) + double(th[2])) : double(th[k]);
              sum += x;
            }
          }
          xv[a] = x;
        }
        const double mu = cta_sum(sum, red) / double(c);
        double ss = 0.0;
        for (uint32_t a = threadIdx.x; a < n; a += kLT)
          if (xv[a] != DINF) ss += (xv[a] - mu) * (xv[a] - mu);
        ss = cta_sum(ss, red);
        mean = float(mu);
        sd = c >= 2 ? float(sqrt(ss / double(c - 1))) : NANF;
        cta_sort_keys(xv, np2);
        q3[0] = float(quantile7(xv, c, 0.025));
        q3[1] = float(quantile7(xv, c, 0.5));
        q3[2] = float(quantile7(xv, c, 0.975));
      }
      if (threadIdx.x == 0) {
        if (is_ki) {
          if (o.ki_mean) o.ki_mean[v] = mean;
          if (o.ki_sd) o.ki_sd[v] = sd;
          if (o.ki_q) for (int t = 0; t < 3; ++t) o.ki_q[v * 3 + t] = q3[t];
        } else {
          if (o.mean) o.mean[v * p.P + k] = mean;
          if (o.sd) o.sd[v * p.P + k] = sd;
          if (o.q) for (int t = 0; t < 3; ++t) o.q[(v * p.P + k) * 3 + t] = q3[t];
        }
      }
      __syncthreads();
    }
    (void)lane;
  }
}

// ---- exact FP64 scan: thread per voxel, max-heap of (D64, i) of size n, prefix pruning ----
__device__ __noinline__ double exact_push(double* hd, uint32_t* hi, uint32_t n, uint32_t& cnt, double D, uint32_t idx) {
  if (cnt < n) {
    uint32_t pos = cnt++;
    while (pos > 0) {
      uint32_t par = (pos - 1) >> 1;
      if (pair_gt(D, idx, hd[par], hi[par])) {  // new key above its parent: move parent down
        hd[pos] = hd[par];
        hi[pos] = hi[par];
        pos = par;
      } else {
        break;
      }
    }
    hd[pos] = D;
    hi[pos] = idx;
  } else {
    uint32_t pos = 0;
    for (;;) {
      uint32_t l = 2 * pos + 1;
      if (l >= n) break;
      uint32_t c = l;
      if (l + 1 < n && pair_gt(hd[l + 1], hi[l + 1], hd[l], hi[l])) c = l + 1;
      if (!pair_gt(hd[c], hi[c], D, idx)) break;
      hd[pos] = hd[c];
      hi[pos] = hi[c];
      pos = c;
    }
    hd[pos] = D;
    hi[pos] = idx;
  }
  return cnt >= n ? hd[0] : __longlong_as_double(0x7ff0000000000000ll);
}

// Warp per voxel: lane l scores draws l, l + 32, ... in FP64 (operation for operation as the
// oracle), with prefix pruning against the warp-uniform threshold tau (the n-th smallest (D, i) so
// far: prefix sums of non-negative terms only grow, so a prefix >= tau means D >= tau).  Survivors
// are pushed by their own lane, one lane at a time in lane order, into the voxel's max-heap of the
// n smallest (D64, i); the new root is then broadcast.  The heap holds exactly the n smallest keys
// of the draws seen, so the result does not depend on the interleaving.
__global__ void __launch_bounds__(256) exact_scan_kernel(const ExactParams p) {
  if (p.bad && *p.bad) return;  // non-finite TACs: no results (ABC_E_ARG)
  const int lane = threadIdx.x & 31;
  const uint64_t len = p.list_len ? uint64_t(*p.list_len) : p.J;
  const uint64_t nwarps = uint64_t(gridDim.x) * (blockDim.x >> 5);
  const double DINF = __longlong_as_double(0x7ff0000000000000ll);
  for (uint64_t e = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; e < len; e += nwarps) {
    const uint64_t v = p.list ? p.list[e] : e;
    const float* y = p.tacs + v * p.L;
    double* hd = p.hd + v * p.n;
    uint32_t* hi = p.hi + v * p.n;
    uint32_t cnt = 0;  // warp-uniform
    double tau = DINF;
    uint32_t tau_i = 0xffffffffu;  // index of the root: keys compare as (D, i)
    for (uint64_t base = 0; base < p.N; base += 32) {
      const uint64_t i = base + lane;
      double D = DINF;
      bool cand = false;
      if (i < p.N) {
        const float* s = p.bank + i * p.LS;
        D = 0.0;
        bool rej = false;
        for (uint32_t f = 0; f < p.L; ++f) {
          double d = __dsub_rn(double(__ldg(y + f)), double(__ldg(s + f)));
          double t = (p.dist == ABC_DIST_L1) ? fabs(d) : __dmul_rn(d, d);
          D = __dadd_rn(D, __dmul_rn(double(__ldg(p.w + f)), t));
          if (D > tau) { rej = true; break; }  // prefix > tau => D > tau (D == tau decided by index)
        }
        cand = !rej && (cnt < p.n || pair_gt(tau, tau_i, D, uint32_t(i)));
      }
      uint32_t bal = __ballot_sync(0xffffffffu, cand);
      while (bal) {
        const int src = __ffs(bal) - 1;
        bal &= bal - 1;
        if (lane == src && (cnt < p.n || pair_gt(tau, tau_i, D, uint32_t(i)))) {
          exact_push(hd, hi, p.n, cnt, D, uint32_t(i));
        }
        __syncwarp();
        cnt = __shfl_sync(0xffffffffu, cnt, src);
        if (cnt >= p.n) {
          tau = hd[0];
          tau_i = hi[0];
        }
        __syncwarp();
      }
    }
  }
}

// ---- eps mode: moments -> summaries (thread per voxel) ----
__global__ void eps_reduce_kernel(const EpsReduceParams p) {
  uint64_t v = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (v >= p.J) return;
  const uint32_t M = p.prior.M;
  const abc_result& o = p.out;
  const float NANF = __int_as_float(0x7fc00000);
  // sum the parts' fixed-point sums (exact), then convert once
  auto total = [&](uint32_t m, uint32_t slot) {
    Fix128 a = 0;
    for (uint32_t q = 0; q < p.nparts; ++q) a += p.mom[((v * p.nparts + q) * M + m) * MOMW + slot];
    return from_fix(a);
  };
  double tot = 0.0;
  int pref = -1;
  double best = -1.0;
  for (uint32_t m = 0; m < M; ++m) {
    double c = total(m, 0);
    tot += c;
    if (c > best) { best = c; pref = int(m); }
  }
  if (tot == 0.0) pref = -1;
  for (uint32_t m = 0; m < M; ++m) {
    double c = total(m, 0);
    if (o.count) o.count[v * M + m] = uint32_t(c);
    if (o.prob) o.prob[v * M + m] = tot > 0.0 ? float(c / tot) : NANF;
  }
  if (o.preferred) o.preferred[v] = pref;
  int kind = pref >= 0 ? p.prior.m[pref].kind : p.prior.m[0].kind;
  const uint32_t pm = pref >= 0 ? uint32_t(pref) : 0u;
  double c = pref >= 0 ? total(pm, 0) : 0.0;
  for (uint32_t k = 0; k < p.P; ++k) {
    float mean = NANF, sd = NANF;
    if (c > 0.0 && column_exists(kind, k)) {
      double lo = p.prior.m[pref].lo[k];
      double s1 = total(pm, 1 + 2 * k), s2 = total(pm, 2 + 2 * k);
      mean = float(lo + s1 / c);
      if (c >= 2.0) sd = float(sqrt(fmax(s2 - s1 * s1 / c, 0.0) / (c - 1.0)));
    }
    if (o.mean) o.mean[v * p.P + k] = mean;
    if (o.sd) o.sd[v * p.P + k] = sd;
    if (o.q) for (int t = 0; t < 3; ++t) o.q[(v * p.P + k) * 3 + t] = NANF;
  }
  float km = NANF, ks = NANF;
  if (c > 0.0 && kind <= ABC_2TCM_REV) {
    double s1 = total(pm, 1 + 2 * ABC_MAX_P), s2 = total(pm, 2 + 2 * ABC_MAX_P);
    km = float(s1 / c);
    if (c >= 2.0) ks = float(sqrt(fmax(s2 - s1 * s1 / c, 0.0) / (c - 1.0)));
  }
  if (o.ki_mean) o.ki_mean[v] = km;
  if (o.ki_sd) o.ki_sd[v] = ks;
  if (o.ki_q) for (int t = 0; t < 3; ++t) o.ki_q[v * 3 + t] = NANF;
}

// ---- posterior summaries of given accepted lists (abc_reduce_accepted) ----------------------
// Warp per voxel: the first n_use indices of the voxel's list (e.g. a top-n list sorted by (D, i):
// its prefix IS the top-n_use set of the same run, SURVEY §8f-3 "truncation of one max-n run")
// are reduced exactly as K4 reduces a certified list.
template <typename IdxT>
__global__ void reduce_list_kernel(const ReduceParams p, const IdxT* idx, const double* dist, uint32_t n_acc, uint32_t np2,
                                   uint32_t wpc, int* bad) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const uint32_t w = threadIdx.x >> 5;
  const size_t per_warp = size_t(np2) * 12;
  double* sc = reinterpret_cast<double*>(smem_raw + per_warp * w);
  uint32_t* ci = reinterpret_cast<uint32_t*>(sc + np2);
  if (p.bad && *p.bad) return;
  for (uint64_t v = uint64_t(blockIdx.x) * wpc + w; v < p.J; v += uint64_t(gridDim.x) * wpc) {
    for (uint32_t a = lane; a < p.n; a += 32) {
      const uint64_t i = idx[v * n_acc + a];
      if (i >= p.N) atomicExch(bad, 1);
      ci[a] = uint32_t(i < p.N ? i : 0);
    }
    __syncwarp();
    reduce_topn(p, v, ci, dist ? dist + v * n_acc : nullptr, sc, np2, lane);
    __syncwarp();
  }
}

// ---- K4, thread per voxel (n <= 32, the accepted lists of the K3/K4 split) -------------------
// One thread summarises one voxel: per column, the accepted draws' values (the preferred model's;
// +inf for the others and for the padding) go to the thread's own 8-byte slots of shared memory
// ([a][thread]: conflict-free), come back into registers, are sorted by a fixed 32-element bitonic network
// (static register indices, fmin/fmax) and written back for the type-7 order statistics.  Sums run
// sequentially in accepted-list order, in FP64.  Roughly a tenth of the warp-per-voxel version's
// warp instructions (a warp summarises 32 voxels at once instead of one).
constexpr int kRT = 128;  // threads per block of the thread-per-voxel reduction

template <typename T>
__device__ __forceinline__ void sort32_regs(T (&r)[32]) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int l = i ^ j;
        if (l > i) {
          const T a = r[i], b = r[l];
          const T lo = a < b ? a : b, hi = a < b ? b : a;
          if ((i & k) == 0) { r[i] = lo; r[l] = hi; } else { r[i] = hi; r[l] = lo; }
        }
      }
    }
  }
}

// this thread's 32 column entries live in its own 8-byte slots of smem_d[a][thread] (an FP32
// value in the first half of the slot: FP32 and FP64 columns never overlap another thread's)
template <typename T>
__device__ __forceinline__ T& col_at(double* slot0, uint32_t a) {
  return *reinterpret_cast<T*>(slot0 + a * kRT);
}

template <typename T>
__device__ __forceinline__ void column_summary(double* col, uint32_t c, double sum, double ss, float& mean, float& sd,
                                               float (&q3)[3]) {
  // first c entries finite
  T r[32];
#pragma unroll
  for (int a = 0; a < 32; ++a) r[a] = col_at<T>(col, a);
  sort32_regs<T>(r);
#pragma unroll
  for (int a = 0; a < 32; ++a) col_at<T>(col, a) = r[a];
  const double mu = sum / double(c);
  mean = float(mu);
  sd = c >= 2 ? float(sqrt(ss / double(c - 1))) : __int_as_float(0x7fc00000);
  const double qs[3] = {0.025, 0.5, 0.975};
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    const double h = double(c - 1) * qs[t];
    const uint32_t lo = uint32_t(floor(h));
    const double xl = double(col_at<T>(col, lo));
    q3[t] = float(lo + 1 < c ? xl + (h - double(lo)) * (double(col_at<T>(col, lo + 1)) - xl) : xl);
  }
}

template <typename IdxT>
__global__ void __launch_bounds__(kRT) reduce_thread_kernel(const ReduceParams p, const IdxT* __restrict__ idx,
                                                             const double* __restrict__ dist, uint32_t n_acc, int* bad) {
  __shared__ double smem_d[32 * kRT];  // per-thread columns [a][thread] (FP64 for K_i, FP32 aliases it)
  if (p.bad && *p.bad) return;
  const uint64_t v = uint64_t(blockIdx.x) * kRT + threadIdx.x;
  if (v >= p.J) return;
  const uint32_t n = p.n, M = p.prior.M;
  const abc_result& o = p.out;
  const IdxT* li = idx + v * n_acc;
  uint32_t cnt[ABC_MAX_MODELS] = {0, 0, 0, 0};
  for (uint32_t a = 0; a < n; ++a) {
    uint64_t i = uint64_t(li[a]);
    if (i >= p.N) {
      atomicExch(bad, 1);
      i = 0;
    }
    cnt[model_index(p.prior, i)] += 1;
    if (o.acc_idx) o.acc_idx[v * n + a] = i;
    if (o.acc_dist && dist) o.acc_dist[v * n + a] = dist[v * n_acc + a];
  }
  int pref = 0;
  for (uint32_t m = 1; m < M; ++m)
    if (cnt[m] > cnt[pref]) pref = int(m);
  for (uint32_t m = 0; m < M; ++m) {
    if (o.count) o.count[v * M + m] = cnt[m];
    if (o.prob) o.prob[v * M + m] = float(double(cnt[m]) / double(n));
  }
  if (o.preferred) o.preferred[v] = pref;
  const int kind = p.prior.m[pref].kind;
  const uint32_t c = cnt[pref];
  const bool tcm = kind <= ABC_2TCM_REV;
  const float NANF = __int_as_float(0x7fc00000);
  double* col = smem_d + threadIdx.x;  // this thread's slots [a * kRT]
  for (uint32_t k = 0; k <= p.P; ++k) {  // column P = K_i
    const bool is_ki = (k == p.P);
    const bool exists = c > 0 && (is_ki ? tcm : column_exists(kind, k));
    float mean = NANF, sd = NANF, q3[3] = {NANF, NANF, NANF};
    if (exists) {
      const uint32_t blk = (is_ki || k < 4) ? 0u : 1u;
      double sum = 0.0;
      for (uint32_t a = 0; a < 32; ++a) {
        double x = __longlong_as_double(0x7ff0000000000000ll);
        if (a < n) {
          const uint64_t i = uint64_t(li[a]) < p.N ? uint64_t(li[a]) : 0ull;
          if (model_index(p.prior, i) == pref) {
            float th[ABC_MAX_P];
            theta_block(p.prior, i, pref, blk, th);
            x = is_ki ? double(th[0]) * double(th[2]) / (double(th[1]) + double(th[2])) : double(th[k]);
            sum += x;
          }
        }
        if (is_ki) col_at<double>(col, a) = x;
        else col_at<float>(col, a) = float(x);
      }
      const double mu = sum / double(c);
      double ss = 0.0;
      for (uint32_t a = 0; a < n; ++a) {
        const double x = is_ki ? col_at<double>(col, a) : double(col_at<float>(col, a));
        if (x != __longlong_as_double(0x7ff0000000000000ll)) ss += (x - mu) * (x - mu);
      }
      if (is_ki) column_summary<double>(col, c, sum, ss, mean, sd, q3);
      else column_summary<float>(col, c, sum, ss, mean, sd, q3);
    }
    if (is_ki) {
      if (o.ki_mean) o.ki_mean[v] = mean;
      if (o.ki_sd) o.ki_sd[v] = sd;
      if (o.ki_q) for (int t = 0; t < 3; ++t) o.ki_q[v * 3 + t] = q3[t];
    } else {
      if (o.mean) o.mean[v * p.P + k] = mean;
      if (o.sd) o.sd[v * p.P + k] = sd;
      if (o.q) for (int t = 0; t < 3; ++t) o.q[(v * p.P + k) * 3 + t] = q3[t];
    }
  }
}

uint32_t next_pow2(uint32_t x) {
  uint32_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// ---- response-function credible envelope (Fig. 1) --------------------------------
// r(t) = 1 + (gamma/k2a) g(t; tD, tP, alpha) per accepted lp-ntPET draw, g the peak-normalised
// gamma variate (eq:Bt P:90-94, R4); type-7 quantiles across the draws per time.
// Operation for operation as the oracle (no FMA contraction).
__device__ __forceinline__ double gamma_variate_d(double tD, double tP, double alpha, double t) {
  if (t <= tD) return 0.0;
  const double x = __ddiv_rn(__dsub_rn(t, tD), __dsub_rn(tP, tD));
  return __dmul_rn(pow(x, alpha), exp(__dmul_rn(alpha, __dsub_rn(1.0, x))));
}

__global__ void response_envelope_kernel(const EnvelopeParams p, uint32_t np2, uint32_t wpc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const uint32_t w = threadIdx.x >> 5;
  const size_t per_warp = size_t(np2) * 28;
  double* sc = reinterpret_cast<double*>(smem_raw + per_warp * w);  // [np2] values at one time
  float4* prm = reinterpret_cast<float4*>(sc + np2);                 // [np2] (gamma, k2a, tD, tP)
  float* pal = reinterpret_cast<float*>(prm + np2);                  // [np2] alpha
  const float NANF = __int_as_float(0x7fc00000);
  for (uint64_t v = uint64_t(blockIdx.x) * wpc + w; v < p.J; v += uint64_t(gridDim.x) * wpc) {
    uint32_t cnt = 0;
    for (uint32_t base = 0; base < p.n_acc; base += 32) {
      const uint32_t a = base + lane;
      bool mine = false;
      float th[ABC_MAX_P];
      if (a < p.n_acc) {
        const uint64_t i = p.acc_idx[v * p.n_acc + a];
        if (i >= p.N) {
          atomicExch(p.bad, 1);
        } else if (p.prior.m[model_index(p.prior, i)].kind == ABC_LPNTPET) {
          draw_theta(p.prior, i, th);
          mine = true;
        }
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, mine);
      if (mine) {
        const uint32_t pos = cnt + __popc(bal & ((1u << lane) - 1u));
        prm[pos] = make_float4(th[3], th[2], th[4], th[5]);
        pal[pos] = th[6];
      }
      cnt += __popc(bal);
    }
    __syncwarp();
    uint32_t kp = 32;
    while (kp < cnt) kp <<= 1;
    for (uint32_t k = 0; k < p.T; ++k) {
      float* o = p.q + (v * p.T + k) * 3;
      if (cnt == 0) {
        if (lane == 0) o[0] = o[1] = o[2] = NANF;
        continue;
      }
      const double tk = p.t[k];
      for (uint32_t a = lane; a < kp; a += 32) {
        double r = __longlong_as_double(0x7ff0000000000000ll);
        if (a < cnt) {
          const float4 x = prm[a];
          const double ratio = __ddiv_rn(double(x.x), double(x.y));
          r = __dadd_rn(1.0, __dmul_rn(ratio, gamma_variate_d(x.z, x.w, pal[a], tk)));
        }
        sc[a] = r;
      }
      __syncwarp();
      warp_sort_any(sc, nullptr, kp, lane);
      if (lane == 0) {
        o[0] = float(quantile7(sc, cnt, 0.025));
        o[1] = float(quantile7(sc, cnt, 0.5));
        o[2] = float(quantile7(sc, cnt, 0.975));
      }
      __syncwarp();
    }
  }
}

}  // namespace

size_t certify_large_smem(uint32_t Kp) { return size_t(Kp) * 12 + 16 * 4 + (kLT / 32) * 8; }

uint32_t certify_candidates_pow2(const ReduceParams& p) {
  if (p.exact == 2) return p.cl_cap;  // collected fallback lists (a power of two)
  return next_pow2(p.exact ? p.n : (p.K * p.nparts > p.n ? p.K * p.nparts : p.n));
}

uint32_t certify_capacity(const ReduceParams& p) {
  const uint32_t Kp = certify_candidates_pow2(p);
  return Kp < 32 ? 32 : Kp;
}

// Fallback collector (see CollectParams): warp item w = (entry e, chunk c) scans draws
// [N c / nchunk, N (c + 1) / nchunk) lane-strided, FP64 in acquisition order with prefix pruning
// against the fixed seed tau[e] (prefix sums only grow: a prefix > tau means D > tau).
__global__ void __launch_bounds__(256) fallback_collect_kernel(const CollectParams p) {
  if (p.bad && *p.bad) return;
  const uint32_t len = min(*p.list_len, p.cap_voxels);
  const int lane = threadIdx.x & 31;
  const uint64_t nw = uint64_t(gridDim.x) * (blockDim.x >> 5);
  const uint64_t items = uint64_t(len) * p.nchunk;
  for (uint64_t it = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; it < items; it += nw) {
    const uint32_t e = uint32_t(it / p.nchunk), c = uint32_t(it % p.nchunk);
    const double tau = p.tau[e];
    if (!(tau < __longlong_as_double(0x7ff0000000000000ll))) continue;
    const float* y = p.tacs + uint64_t(p.list[e]) * p.L;
    const uint64_t i0 = p.N * c / p.nchunk, i1 = p.N * (c + 1) / p.nchunk;
    for (uint64_t i = i0 + lane; i < i1; i += 32) {
      const float* s = p.bank + i * p.LS;
      double D = 0.0;
      bool rej = false;
      for (uint32_t f = 0; f < p.L; ++f) {
        const double d = __dsub_rn(double(__ldg(y + f)), double(__ldg(s + f)));
        const double t = (p.dist == ABC_DIST_L1) ? fabs(d) : __dmul_rn(d, d);
        D = __dadd_rn(D, __dmul_rn(double(__ldg(p.w + f)), t));
        if (D > tau) { rej = true; break; }
      }
      if (!rej) {
        const uint32_t pos = atomicAdd(p.cnt + e, 1u);
        if (pos < p.cap) {
          p.cd[uint64_t(e) * p.cap + pos] = D;
          p.ci[uint64_t(e) * p.cap + pos] = uint32_t(i);
        }
      }
    }
  }
}

void launch_fallback_collect(const CollectParams& p, cudaStream_t st) {
  fallback_collect_kernel<<<148 * 8, 256, 0, st>>>(p);
}

cudaError_t launch_certify_reduce(const ReduceParams& p, cudaStream_t st) {
  uint32_t Kp = certify_candidates_pow2(p);
  if (Kp < 32) Kp = 32;
  if (Kp > kWarpCertifyMax) {  // large n: one CTA per voxel, candidates and sorts CTA-wide
    if (Kp > kLargeMaxCand) return cudaErrorInvalidValue;
    const size_t smem = certify_large_smem(Kp);
    cudaError_t e = ensure_smem_attr((const void*)certify_large_kernel, smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    int occ = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, certify_large_kernel, kLT, smem);
    uint64_t blocks = uint64_t(nsm) * uint64_t(occ > 0 ? occ : 1);
    if (blocks > p.J) blocks = p.J;
    if (blocks == 0) blocks = 1;
    certify_large_kernel<<<unsigned(blocks), kLT, smem, st>>>(p, Kp);
    return cudaGetLastError();
  }
  uint32_t np2 = next_pow2(p.n);
  if (np2 < 32) np2 = 32;
  size_t per_warp = size_t(Kp) * 12 + size_t(np2) * 8;
  uint32_t wpc = 8;
  while (wpc > 1 && per_warp * wpc > 96 * 1024) wpc >>= 1;
  size_t smem = per_warp * wpc;
  cudaError_t e = ensure_smem_attr((const void*)certify_reduce_kernel, smem);
  if (e != cudaSuccess) return e;
  uint64_t work = p.list ? p.J : p.J;  // upper bound on list length
  uint64_t blocks = (work + wpc - 1) / wpc;
  if (blocks > 148ull * 64) blocks = 148ull * 64;
  if (blocks == 0) blocks = 1;
  certify_reduce_kernel<<<unsigned(blocks), wpc * 32, smem, st>>>(p, Kp, np2, wpc);
  return cudaGetLastError();
}

void launch_exact_scan(const ExactParams& p, cudaStream_t st) {
  uint64_t blocks = (p.J + 7) / 8;  // 8 warps per CTA, one voxel per warp
  if (blocks > 148ull * 8) blocks = 148ull * 8;
  if (blocks == 0) blocks = 1;
  exact_scan_kernel<<<unsigned(blocks), 256, 0, st>>>(p);
}

void launch_eps_reduce(const EpsReduceParams& p, cudaStream_t st) {
  uint64_t blocks = (p.J + 127) / 128;
  if (blocks == 0) return;
  eps_reduce_kernel<<<unsigned(blocks), 128, 0, st>>>(p);
}

template <typename IdxT>
static cudaError_t launch_reduce_list_t(const ReduceParams& p, const IdxT* idx, const double* dist, uint32_t n_acc,
                                        int* bad, cudaStream_t st) {
  // n <= 32: thread per voxel (reduce_thread_kernel); else warp per voxel (reduce_list_kernel)
  static const bool thread_env = getenv("VPET_REDUCE_THREAD") ? atoi(getenv("VPET_REDUCE_THREAD")) != 0 : true;  // tuning knob
  if (thread_env && p.n <= 32) {
    const uint64_t blocks = (p.J + kRT - 1) / kRT;
    reduce_thread_kernel<IdxT><<<unsigned(blocks > 0 ? blocks : 1), kRT, 0, st>>>(p, idx, dist, n_acc, bad);
    return cudaGetLastError();
  }
  uint32_t np2 = next_pow2(p.n);
  if (np2 < 32) np2 = 32;
  const size_t per_warp = size_t(np2) * 12;
  uint32_t wpc = 8;
  while (wpc > 1 && per_warp * wpc > 96 * 1024) wpc >>= 1;
  const size_t smem = per_warp * wpc;
  cudaError_t e = ensure_smem_attr((const void*)reduce_list_kernel<IdxT>, smem);
  if (e != cudaSuccess) return e;
  uint64_t blocks = (p.J + wpc - 1) / wpc;
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  if (blocks == 0) blocks = 1;
  reduce_list_kernel<IdxT><<<unsigned(blocks), wpc * 32, smem, st>>>(p, idx, dist, n_acc, np2, wpc, bad);
  return cudaGetLastError();
}

cudaError_t launch_reduce_list(const ReduceParams& p, const uint64_t* idx, uint32_t n_acc, int* bad, cudaStream_t st) {
  return launch_reduce_list_t<uint64_t>(p, idx, nullptr, n_acc, bad, st);
}

cudaError_t launch_reduce_accepted_lists(const ReduceParams& p, const uint32_t* idx, const double* dist, int* bad,
                                         cudaStream_t st) {
  return launch_reduce_list_t<uint32_t>(p, idx, dist, p.n, bad, st);
}

cudaError_t launch_response_envelope(const EnvelopeParams& p, cudaStream_t st) {
  uint32_t np2 = next_pow2(p.n_acc);
  if (np2 < 32) np2 = 32;
  const size_t per_warp = size_t(np2) * 28;
  uint32_t wpc = 8;
  while (wpc > 1 && per_warp * wpc > 96 * 1024) wpc >>= 1;
  const size_t smem = per_warp * wpc;
  cudaError_t e = ensure_smem_attr((const void*)response_envelope_kernel, smem);
  if (e != cudaSuccess) return e;
  uint64_t blocks = (p.J + wpc - 1) / wpc;
  if (blocks > 148ull * 32) blocks = 148ull * 32;
  if (blocks == 0) blocks = 1;
  response_envelope_kernel<<<unsigned(blocks), wpc * 32, smem, st>>>(p, np2, wpc);
  return cudaGetLastError();
}

}  // namespace vpet
