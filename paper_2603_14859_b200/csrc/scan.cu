// scan.cu -- K2: the FP32 pass of Alg. 1 lines 4-5, fused distance + selection.
//
// One thread owns R voxels; their prescaled TACs (y~_k = wsp_k * y_perm(k)) live in registers
// as float2 pairs.  The CTA streams the negated, prescaled, scan-ordered bank
// (bankp[i][k] = -wsp_k s_{i,perm(k)}) through a 4-stage shared-memory ring filled by
// cp.async.bulk (TMA bulk copies, mbarrier complete_tx).  For every draw i and voxel:
//     d = y~ + bankp_i        (FADD2, two frames per instruction)
//     acc = fma(d, d, acc)    (FFMA2; WL2)      or   acc += |d|  (L1)
// Frames are visited in descending-spread order and, after every chunk of CH frames, the
// warp stops the draw when no lane's partial sum is below its pruning threshold.  Partial
// sums of non-negative terms are monotone under rounding, so a pruned draw provably has
// D32 >= tau and the pruned pass accepts exactly the draws the full pass would.
// Top-n mode keeps the K = n + slack smallest (D32, i) keys per voxel in a global max-heap;
// K3 (certify.cu) re-scores them in FP64.  Eps mode re-scores every draw with
// D32 <= eps + err(eps) inline in FP64 and accumulates posterior moments.
#include <cfloat>
#include <cstdio>

#include "common.cuh"

namespace vpet {
namespace {

constexpr int NT = 256;
constexpr int NW = NT / 32;
constexpr int NST = 4;
constexpr int CH = 8;

template <int LP>
struct ScanShape {
  static constexpr int R = (LP <= 48) ? 2 : 1;
  static constexpr int T = (LP <= 48) ? 64 : 32;
  static constexpr int MINB = (LP * R <= 96) ? 2 : 1;
  static constexpr size_t SMEM = size_t(NST) * T * LP * 4 + NST * 8 + NST * 4 + 16;
};

__device__ __forceinline__ uint32_t smem_u32(const void* ptr) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(ptr));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Max-heap of K keys (D32 bits << 32 | draw index) per voxel, in global memory.  Returns
// (new count, new threshold bits).  Rare: ~K (1 + ln(N/K)) calls per voxel.
__device__ __noinline__ uint2 heap_push(unsigned long long* h, uint32_t K, uint32_t cnt, unsigned long long key) {
  if (cnt < K) {
    uint32_t pos = cnt++;
    while (pos > 0) {
      uint32_t par = (pos - 1) >> 1;
      unsigned long long pk = h[par];
      if (pk >= key) break;
      h[pos] = pk;
      pos = par;
    }
    h[pos] = key;
  } else {
    uint32_t pos = 0;
    for (;;) {
      uint32_t l = 2 * pos + 1;
      if (l >= K) break;
      uint32_t c = l;
      unsigned long long hc = h[l];
      if (l + 1 < K) {
        unsigned long long hr = h[l + 1];
        if (hr > hc) { c = l + 1; hc = hr; }
      }
      if (hc <= key) break;
      h[pos] = hc;
      pos = c;
    }
    h[pos] = key;
  }
  float tau = (cnt >= K) ? __uint_as_float(uint32_t(h[0] >> 32)) : __int_as_float(0x7f800000);
  return make_uint2(cnt, __float_as_uint(tau));
}

// Exact FP64 discrepancy in acquisition order, operation for operation as the oracle.
__device__ __forceinline__ double exact_distance(const float* y, const float* s, const float* w, uint32_t L,
                                                 int dist) {
  double D = 0.0;
  for (uint32_t f = 0; f < L; ++f) {
    double d = __dsub_rn(double(y[f]), double(__ldg(s + f)));
    double t = (dist == ABC_DIST_L1) ? fabs(d) : __dmul_rn(d, d);
    D = __dadd_rn(D, __dmul_rn(double(__ldg(w + f)), t));
  }
  return D;
}

// Eps mode: exact re-score of a candidate; accepted draws update the voxel's moment sums.
__device__ __noinline__ void eps_candidate(const float* yrow, const float* bank, uint32_t LS, const float* w,
                                           uint32_t L, int dist, double eps, double* mom, const PriorDev* prior,
                                           uint64_t i) {
  double D = exact_distance(yrow, bank + i * LS, w, L, dist);
  if (!(D <= eps)) return;
  float th[ABC_MAX_P];
  int m = draw_theta(*prior, i, th);
  const ModelDev& md = prior->m[m];
  double* s = mom + size_t(m) * MOMW;
  s[0] += 1.0;
  for (uint32_t k = 0; k < md.P; ++k) {
    double x = double(th[k]) - double(md.lo[k]);
    s[1 + 2 * k] += x;
    s[2 + 2 * k] += x * x;
  }
  if (md.kind <= ABC_2TCM_REV) {
    double ki = double(th[0]) * double(th[2]) / (double(th[1]) + double(th[2]));
    s[1 + 2 * ABC_MAX_P] += ki;
    s[2 + 2 * ABC_MAX_P] += ki * ki;
  }
}

template <int LP, int DIST, bool COUNT>
__global__ void __launch_bounds__(NT, ScanShape<LP>::MINB) scan_kernel(const ScanParams p) {
  constexpr int R = ScanShape<LP>::R;
  constexpr int T = ScanShape<LP>::T;
  constexpr int NCH = (LP + CH - 1) / CH;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stage = reinterpret_cast<float*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + size_t(NST) * T * LP * 4);
  int* arrivals = reinterpret_cast<int*>(full + NST);

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const uint64_t N = p.N;
  const uint32_t ntile = uint32_t((N + T - 1) / T);

  const float* __restrict__ bankp = p.bankp;
  auto issue = [=](uint32_t tt, int ss) {
    uint64_t i0 = uint64_t(tt) * T;
    uint32_t nd = uint32_t((N - i0) < uint64_t(T) ? (N - i0) : uint64_t(T));
    uint32_t bytes = nd * LP * 4u;
    mbar_expect_tx(&full[ss], bytes);
    bulk_g2s(stage + size_t(ss) * T * LP, bankp + i0 * LP, bytes, &full[ss]);
  };

  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      arrivals[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    for (uint32_t s = 0; s < uint32_t(NST) && s < ntile; ++s) issue(s, int(s));
  }

  // ---- voxel state in registers ----
  float2 y[R][LP / 2];
  float tau[R], tp[R];
  uint32_t cnt[R];
  uint64_t vox[R];
  const float INF = __int_as_float(0x7f800000);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    uint64_t v = uint64_t(blockIdx.x) * (NT * R) + uint64_t(r) * NT + tid;
    vox[r] = v;
    bool valid = v < p.J;
    const float* yr = p.tacs + (valid ? v : 0) * p.L;
#pragma unroll
    for (int k = 0; k < LP; k += 2) {
      int s0 = __ldg(p.perm + k), s1 = __ldg(p.perm + k + 1);
      float a = (valid && s0 >= 0) ? __fmul_rn(__ldg(p.wsp + k), __ldg(yr + s0)) : 0.0f;
      float b = (valid && s1 >= 0) ? __fmul_rn(__ldg(p.wsp + k + 1), __ldg(yr + s1)) : 0.0f;
      y[r][k / 2] = make_float2(a, b);
    }
    cnt[r] = 0;
    if (!p.eps_mode) {
      tau[r] = valid ? INF : -INF;
    } else {
      double Y2 = 0.0, Y1 = 0.0;
      if (valid) {
        for (uint32_t f = 0; f < p.L; ++f) {
          double yv = yr[f], wv = __ldg(p.w + f);
          Y2 += wv * yv * yv;
          Y1 += wv * fabs(yv);
        }
      }
      double err = p.eb.a * p.eps + p.eb.b * sqrt(Y2 * p.eps) + p.eb.c * Y2 + p.eb.d * Y1;
      // candidates: D32 <= eps + err(eps)  <=>  D32 < next float above it
      tau[r] = valid ? nextafterf(__double2float_ru(p.eps + err), INF) : -INF;
    }
    tp[r] = (p.prune || !valid) ? tau[r] : INF;
  }

  unsigned long long work = 0;
  for (uint32_t t = 0; t < ntile; ++t) {
    const int s = int(t % NST);
    mbar_wait(&full[s], (t / NST) & 1u);
    const float* sb = stage + size_t(s) * T * LP;
    const uint64_t rem = N - uint64_t(t) * T;
    const uint32_t nd = uint32_t(rem < uint64_t(T) ? rem : uint64_t(T));
    const uint64_t ibase = uint64_t(t) * T;
    for (uint32_t d = 0; d < nd; ++d) {
      const float* sr = sb + d * LP;
      float2 acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) acc[r] = make_float2(0.0f, 0.0f);
      bool go = true;
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        if (go) {
#pragma unroll
          for (int q = c * CH; q < ((c + 1) * CH < LP ? (c + 1) * CH : LP); q += 4) {
            const float4 s4 = *reinterpret_cast<const float4*>(sr + q);
            const float2 sa = make_float2(s4.x, s4.y);
            const float2 sc = make_float2(s4.z, s4.w);
#pragma unroll
            for (int r = 0; r < R; ++r) {
              float2 d0 = __fadd2_rn(y[r][q / 2], sa);
              float2 d1 = __fadd2_rn(y[r][q / 2 + 1], sc);
              if (DIST == ABC_DIST_WL2) {
                acc[r] = __ffma2_rn(d0, d0, acc[r]);
                acc[r] = __ffma2_rn(d1, d1, acc[r]);
              } else {
                acc[r].x = __fadd_rn(acc[r].x, fabsf(d0.x));
                acc[r].y = __fadd_rn(acc[r].y, fabsf(d0.y));
                acc[r].x = __fadd_rn(acc[r].x, fabsf(d1.x));
                acc[r].y = __fadd_rn(acc[r].y, fabsf(d1.y));
              }
            }
          }
          if (COUNT) work += uint64_t(((c + 1) * CH < LP ? (c + 1) * CH : LP) - c * CH) * R;
          if (c < NCH - 1) {
            bool alive = false;
#pragma unroll
            for (int r = 0; r < R; ++r) alive |= (__fadd_rn(acc[r].x, acc[r].y) < tp[r]);
            go = __any_sync(0xffffffffu, alive);
          }
        }
      }
      if (go) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float D = __fadd_rn(acc[r].x, acc[r].y);
          if (D < tau[r]) {
            uint64_t i = ibase + d;
            if (!p.eps_mode) {
              unsigned long long key = (static_cast<unsigned long long>(__float_as_uint(D)) << 32) | uint32_t(i);
              uint2 st = heap_push(p.heap + vox[r] * p.K, p.K, cnt[r], key);
              cnt[r] = st.x;
              tau[r] = __uint_as_float(st.y);
              if (p.prune) tp[r] = tau[r];
            } else {
              eps_candidate(p.tacs + vox[r] * p.L, p.bank, p.LS, p.w, p.L, p.dist, p.eps,
                            p.mom + vox[r] * (size_t(p.M) * MOMW), p.prior_g, i);
            }
          }
        }
      }
    }
    // release the stage; the last warp to finish it refills it with tile t + NST
    __syncwarp();
    if (lane == 0) {
      __threadfence_block();
      int old = atomicAdd(&arrivals[s], 1);
      if (old == NW - 1) {
        atomicExch(&arrivals[s], 0);
        uint32_t tn = t + NST;
        if (tn < ntile) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(tn, s);
        }
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (vox[r] < p.J && !p.eps_mode) p.heap_cnt[vox[r]] = cnt[r];
  if (COUNT) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) work += __shfl_xor_sync(0xffffffffu, work, o);
    if (lane == 0) atomicAdd(p.work, work);
  }
}

template <int LP, int DIST, bool COUNT>
cudaError_t launch_one(const ScanParams& p, cudaStream_t st) {
  using S = ScanShape<LP>;
  auto kern = scan_kernel<LP, DIST, COUNT>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(S::SMEM));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  uint64_t per_cta = uint64_t(NT) * S::R;
  unsigned grid = unsigned((p.J + per_cta - 1) / per_cta);
  kern<<<grid, NT, S::SMEM, st>>>(p);
  return cudaGetLastError();
}

#define VPET_LP_LIST(X) X(8) X(12) X(16) X(20) X(24) X(28) X(32) X(36) X(40) X(44) X(48) X(56) X(64) X(72) X(80) X(96) X(112) X(128)

}  // namespace

bool scan_supported(uint32_t LP) {
#define X(v) if (LP == v) return true;
  VPET_LP_LIST(X)
#undef X
  return false;
}

uint32_t scan_lp_for(uint32_t L) {
#define X(v) if (L <= v) return v;
  VPET_LP_LIST(X)
#undef X
  return 0;
}

cudaError_t launch_scan(const ScanParams& p, uint32_t LP, int count_work, cudaStream_t st) {
#define X(v)                                                                                  \
  if (LP == v) {                                                                              \
    if (p.dist == ABC_DIST_WL2)                                                               \
      return count_work ? launch_one<v, ABC_DIST_WL2, true>(p, st) : launch_one<v, ABC_DIST_WL2, false>(p, st); \
    return count_work ? launch_one<v, ABC_DIST_L1, true>(p, st) : launch_one<v, ABC_DIST_L1, false>(p, st);     \
  }
  VPET_LP_LIST(X)
#undef X
  return cudaErrorInvalidValue;
}

}  // namespace vpet
