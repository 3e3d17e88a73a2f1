// scan_kernels.cuh -- K2: the FP32 pass of Alg. 1 lines 4-5, fused distance +
// per-voxel selection.  Included by scan_wl2.cu / scan_l1.cu (one distance each).
//
// One thread owns R voxels; their prescaled TACs (y~_k = wsp_k * y_perm(k)) live in registers as
// float2 pairs.  The CTA streams tiles of the negated, prescaled, scan-order bank
// (bankp[j][k] = -wsp_k s_{i(j), perm(k)}) through a 4-stage shared-memory ring filled by
// cp.async.bulk (TMA bulk copies completing on mbarriers).  For every draw and voxel:
//     d = y~ + bankp_j          (FADD2: two frames per instruction)
//     acc = fma(d, d, acc)      (FFMA2, WL2)     or    acc += |d|   (L1)
// Frames are visited in descending-spread order; after every chunk of CH frames the warp drops
// the draw if no lane's partial sum is below its threshold (prefix sums of non-negative terms
// are monotone under rounding, so this is exact).
//
// Two variants:
//   scan_flat_kernel  draws in index order, every tile of the bank (ABC_FLAG_NO_TREE).
//   scan_tree_kernel  draws in Morton order of their principal-axis projections (order.cu);
//                     per tile and per super-tile of ST tiles the per-frame [min, max] of bankp
//                     gives, with the same FP32 chain, a lower bound LB32 <= D32 of every draw
//                     inside (|fl(y + b)| >= gap by monotone rounding), so a (super-)tile whose
//                     LB32 >= threshold for all lanes of a warp is skipped by that warp, and one
//                     skipped by all warps is never loaded.  Each warp first scans the super-tile
//                     closest to its mean TAC (seeding) so thresholds drop early.
// Top-n mode keeps the K = n + slack smallest (D32, i) keys per voxel in a global max-heap and K3
// re-scores them in FP64; eps mode re-scores every draw with D32 <= eps + err(eps) inline.
#pragma once
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace vpet {
namespace scan {

#ifndef VPET_NT
#define VPET_NT 64
#endif
#ifndef VPET_NST
#define VPET_NST 2
#endif
constexpr int NT = VPET_NT;   // threads per CTA (the warps of a CTA share tile loads)
constexpr int NW = NT / 32;
constexpr int NST = VPET_NST;  // TMA ring stages
#ifndef VPET_CH
#define VPET_CH 0
#endif
constexpr int CH = VPET_CH;  // frames per pruning chunk of a draw evaluation (multiple of 4); 0 = LP (one chunk)
// Chunk of a draw evaluation: the whole row when two voxels share a lane (LP <= 48): a row is then
// evaluated for 64 voxels, one of which nearly always keeps it alive past a 16-frame chunk (rows ran
// 31 of 36 frames on the TB volume), so the intermediate votes cost more than they save (scan -9.5 %
// with 12-frame bound chunks).  16 frames for the one-voxel-per-lane layouts.
template <int LP>
__host__ __device__ constexpr int chd() { return CH > 0 ? CH : (LP <= 48 ? LP : 16); }
#ifndef VPET_CHB
#define VPET_CHB 12
#endif
constexpr int CHB = VPET_CHB;  // frames per pruning chunk of a box lower bound (multiple of 4)
constexpr int T = kTile;
#ifndef VPET_REFRESH
#define VPET_REFRESH 0  // pull tau_glob every VPET_REFRESH + 1 super-tiles
#endif
#ifndef VPET_REFRESH_ROT
#define VPET_REFRESH_ROT 3  // rotated kernel: every 4th super-tile and hyper-tile (the per-tile refresh
#endif                      // stays): scan 140 -> 136 ms on the TB volume
#ifndef VPET_HREFRESH_ROT
#define VPET_HREFRESH_ROT 3
#endif
#ifndef VPET_HREFRESH
#define VPET_HREFRESH 0  // and every VPET_HREFRESH + 1 hyper-tiles
#endif
#ifndef VPET_TREFRESH
#define VPET_TREFRESH 2  // and before every evaluated tile (1: pipelined load, 2: immediate)
#endif
#ifndef VPET_RREFRESH
#define VPET_RREFRESH 0  // and every VPET_RREFRESH rows inside a tile (0: off)
#endif
#ifndef VPET_HEAD
#define VPET_HEAD 12  // rotated basis: coordinates evaluated before a row's first test (multiple of 4)
#endif
constexpr int kHead = VPET_HEAD;
#ifndef VPET_BOXHEAD
#define VPET_BOXHEAD 4  // coordinates of a box tested before its tail bound (<= kHead: rv starts at kHead);
                        // measured 12 / 4 against 8 / 8: scan 144 -> 140 ms (16 / 4: 144, 16 / 8: 147)
#endif
constexpr int kBoxHead = VPET_BOXHEAD;
static_assert(kBoxHead <= kHead && kBoxHead % 4 == 0, "the box head test must not overlap rv's coordinates");
#ifndef VPET_SHEAP
#define VPET_SHEAP 0  // keep the top of each candidate heap in shared memory (tree scan)
#endif
#ifndef VPET_SSORT
#define VPET_SSORT 1
#endif

template <int LP>
struct Shape {
#ifndef VPET_R
#define VPET_R 0  // voxels per lane: 0 = 2 for LP <= 48, else 1
#endif
  static constexpr int R = VPET_R > 0 ? VPET_R : ((LP <= 48) ? 2 : 1);
#ifdef VPET_MINB
  static constexpr int MINB = VPET_MINB;
#else
  static constexpr int MINB = ((LP * R <= 96) ? 16 : 8) / NW;
#endif
#ifdef VPET_MINB_ROT
  static constexpr int MINB_ROT = VPET_MINB_ROT;
#else
  static constexpr int MINB_ROT = MINB * 7 / 8 > 0 ? MINB * 7 / 8 : 1;  // the rotated path's extra state
#endif
  static constexpr size_t STAGE_FLOATS = size_t(T) * LP;
  // prefetched boxes of one super-tile: its own [lo; hi] then its kSuper tiles' (double buffered)
  static constexpr size_t BOXB_FLOATS = size_t(kSuper + 1) * 2 * LP;
  // the TMA ring; the best-first sort scratch aliases it (used only while the ring is idle)
  static constexpr size_t RING_BYTES = size_t(NST) * STAGE_FLOATS * 4;
  static constexpr size_t SCRATCH_BYTES = size_t(kHyperSort) * NW * 12 + kHyperSort / 8;
#ifndef VPET_ALIAS
#define VPET_ALIAS 1
#endif
  static constexpr size_t REGION = VPET_ALIAS ? ((RING_BYTES > SCRATCH_BYTES ? RING_BYTES : SCRATCH_BYTES) + 15) & ~size_t(15)
                                              : ((RING_BYTES + SCRATCH_BYTES) + 15) & ~size_t(15);
  // top of each voxel's candidate heap (root + its 8 children) kept in shared memory per item
  static constexpr int KTOP = 9;
  static constexpr size_t HTOP_BYTES = VPET_SHEAP ? size_t(NT) * R * KTOP * 8 : 0;
  static constexpr size_t RV_BYTES = size_t(NT) * R * 4;  // rotated basis: tail bounds per thread
  static constexpr size_t SMEM = REGION + size_t(NST) * T * 4 + NST * 8 + NST * 4 + NW * 4 + NW * LP * 4 + 16 + 64 +
                                 size_t(kHyperSort) * 8 + 2 * BOXB_FLOATS * 4 + 16 + 16 + HTOP_BYTES + 16 + RV_BYTES + 16;

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

// 8-ary max-heap of K keys (D32 bits << 32 | draw index) per (voxel, part), in global memory
// (layout: common.cuh heap_stride).  The caller pushes only keys below the root of a full heap
// (D < taup).  A push touches <= 2 levels for K <= 72: one 64-B group of children per level.
// Returns (new count, new threshold bits).
#ifndef VPET_HEAP_INLINE
#define VPET_HEAP_INLINE 0
#endif
#if VPET_HEAP_INLINE
#define VPET_HEAP_ATTR __forceinline__
#else
#define VPET_HEAP_ATTR __noinline__
#endif
static __device__ VPET_HEAP_ATTR uint2 heap_push(unsigned long long* hb, uint32_t K, uint32_t cnt, unsigned long long key) {
  unsigned long long* h = hb + kHeapOff;
  unsigned long long root;
  if (cnt < K) {
    uint32_t pos = cnt++;
    while (pos > 0) {
      uint32_t par = (pos - 1) >> 3;
      unsigned long long pk = h[par];
      if (pk >= key) break;
      h[pos] = pk;
      pos = par;
    }
    h[pos] = key;
    if (cnt < K) return make_uint2(cnt, 0x7f800000u);
    root = pos == 0 ? key : h[0];  // heap just became full
  } else {
    uint32_t pos = 0;
    root = key;
    for (;;) {
      const uint32_t c0 = 8 * pos + 1;
      if (c0 >= K) break;
      const ulonglong2* g = reinterpret_cast<const ulonglong2*>(h + c0);
      const ulonglong2 q0 = g[0], q1 = g[1], q2 = g[2], q3 = g[3];
      const unsigned long long ch[8] = {q0.x, q0.y, q1.x, q1.y, q2.x, q2.y, q3.x, q3.y};
      unsigned long long m = 0;
      uint32_t mj = 0;
#pragma unroll
      for (uint32_t j = 0; j < 8; ++j)
        if (c0 + j < K && ch[j] > m) { m = ch[j]; mj = j; }
      if (m <= key) break;
      if (pos == 0) root = m;  // the largest child of the root becomes the root
      h[pos] = m;
      pos = c0 + mj;
    }
    h[pos] = key;
  }
  return make_uint2(cnt, uint32_t(root >> 32));
}

// Same heap with nodes 0..8 (the root and its 8 children) in shared memory at byte address ts.
__device__ __forceinline__ unsigned long long lds64(uint32_t a) {
  unsigned long long v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts64(uint32_t a, unsigned long long v) {
  asm volatile("st.shared.u64 [%0], %1;" ::"r"(a), "l"(v) : "memory");
}
static __device__ __noinline__ uint2 heap_push_s(unsigned long long* hb, uint32_t ts, uint32_t K, uint32_t cnt,
                                                 unsigned long long key) {
  unsigned long long* h = hb + kHeapOff;
  auto ld = [&](uint32_t i) { return i < 9 ? lds64(ts + 8 * i) : h[i]; };
  auto st = [&](uint32_t i, unsigned long long v) {
    if (i < 9) sts64(ts + 8 * i, v);
    else h[i] = v;
  };
  unsigned long long root;
  if (cnt < K) {
    uint32_t pos = cnt++;
    while (pos > 0) {
      uint32_t par = (pos - 1) >> 3;
      unsigned long long pk = ld(par);
      if (pk >= key) break;
      st(pos, pk);
      pos = par;
    }
    st(pos, key);
    if (cnt < K) return make_uint2(cnt, 0x7f800000u);
    root = pos == 0 ? key : lds64(ts);
  } else {
    // level 1 (shared memory)
    unsigned long long m = 0;
    uint32_t mj = 0;
#pragma unroll
    for (uint32_t j = 0; j < 8; ++j) {
      const unsigned long long c = lds64(ts + 8 * (1 + j));
      if (1 + j < K && c > m) { m = c; mj = j; }
    }
    if (m <= key) {
      sts64(ts, key);
      root = key;
    } else {
      sts64(ts, m);
      root = m;
      uint32_t pos = 1 + mj;
      for (;;) {  // levels >= 2 (global memory)
        const uint32_t c0 = 8 * pos + 1;
        if (c0 >= K) break;
        const ulonglong2* g = reinterpret_cast<const ulonglong2*>(h + c0);
        const ulonglong2 q0 = g[0], q1 = g[1], q2 = g[2], q3 = g[3];
        const unsigned long long ch[8] = {q0.x, q0.y, q1.x, q1.y, q2.x, q2.y, q3.x, q3.y};
        unsigned long long mm = 0;
        uint32_t mjj = 0;
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j)
          if (c0 + j < K && ch[j] > mm) { mm = ch[j]; mjj = j; }
        if (mm <= key) break;
        st(pos, mm);
        pos = c0 + mjj;
      }
      st(pos, key);
    }
  }
  return make_uint2(cnt, uint32_t(root >> 32));
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

// Eps mode: exact re-score of a candidate; accepted draws update the voxel's moment sums of this
// part (mom points at [M][MOMW] of (voxel, part): one owner thread at a time, no atomics).
static __device__ __noinline__ void eps_candidate(const float* yrow, const float* bank, uint32_t LS, const float* w,
                                           uint32_t L, int dist, double eps, Fix128* mom, const PriorDev* prior,
                                           uint64_t i) {
  double D = exact_distance(yrow, bank + i * LS, w, L, dist);
  if (!(D <= eps)) return;
  float th[ABC_MAX_P];
  int m = draw_theta(*prior, i, th);
  const ModelDev& md = prior->m[m];
  Fix128* s = mom + size_t(m) * MOMW;
  s[0] += Fix128(1) << kFixFrac;
  for (uint32_t k = 0; k < md.P; ++k) {
    double x = double(th[k]) - double(md.lo[k]);
    s[1 + 2 * k] += to_fix(x);
    s[2 + 2 * k] += to_fix(x * x);
  }
  if (md.kind <= ABC_2TCM_REV) {
    double ki = double(th[0]) * double(th[2]) / (double(th[1]) + double(th[2]));
    s[1 + 2 * ABC_MAX_P] += to_fix(ki);
    s[2 + 2 * ABC_MAX_P] += to_fix(ki * ki);
  }
}

// tau_glob is indexed by scan-order slot (a warp's 32 lanes read 32 consecutive words: one request)
#ifndef VPET_WARP_CONTIG
#define VPET_WARP_CONTIG 1
#endif
constexpr uint32_t kSlotStride = VPET_WARP_CONTIG ? 32u : uint32_t(NT);

// Per-thread voxel state.
template <int LP, int R>
struct Voxels {
  float2 y[R][LP / 2];
  float tau[R];   // threshold: min(own heap root, shared tau_glob) (top-n) / eps bound; prunes too
  float taup[R];  // own (part) heap root, +inf until the heap is full
  uint32_t cnt[R];
  uint32_t vox[R];  // voxel index (>= J for an empty slot)
  uint32_t slot0;   // scan-order slot of voxel 0; voxel r sits at slot0 + r * kSlotStride
  float rv[R];      // rotated basis: lower bound on the coordinates >= kHead of every draw's D32 terms
};

template <int LP, int R, bool ROT = false>
__device__ __forceinline__ void load_voxels(const ScanParams& p, Voxels<LP, R>& V, int tid, uint64_t vtile) {
  const float INF = __int_as_float(0x7f800000);
#pragma unroll
  for (int r = 0; r < R; ++r) {
#ifndef VPET_WARP_CONTIG
#define VPET_WARP_CONTIG 1
#endif
    // a warp's 32 R voxels are one contiguous run of the voxel order (the most similar TACs: a tile
    // is evaluated for all of them once its bound is alive for one)
    const uint64_t slot = VPET_WARP_CONTIG ? vtile * (NT * R) + uint64_t(tid >> 5) * (32 * R) + uint64_t(r) * 32 + (tid & 31)
                                           : vtile * (NT * R) + uint64_t(r) * NT + tid;
    if (r == 0) V.slot0 = uint32_t(slot);
    bool valid = slot < p.J;
    uint64_t v = (valid && p.vorder) ? uint64_t(__ldg(p.vorder + slot)) : slot;
    V.vox[r] = uint32_t(v);
    const float* yr = p.tacs + (valid ? v : 0) * p.L;
    if (p.ytr) {  // rotated basis: the voxel's scan coordinates were computed by voxel_rotate_kernel
      const float4* yt = reinterpret_cast<const float4*>(p.ytr + (valid ? v : 0) * uint64_t(LP));
#pragma unroll
      for (int k = 0; k < LP; k += 4) {
        const float4 q = valid ? __ldg(yt + k / 4) : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        V.y[r][k / 2] = make_float2(q.x, q.y);
        V.y[r][k / 2 + 1] = make_float2(q.z, q.w);
      }
    } else {
#pragma unroll
      for (int k = 0; k < LP; k += 2) {
        int s0 = __ldg(p.perm + k), s1 = __ldg(p.perm + k + 1);
        float a = (valid && s0 >= 0) ? __fmul_rn(__ldg(p.wsp + k), __ldg(yr + s0)) : 0.0f;
        float b = (valid && s1 >= 0) ? __fmul_rn(__ldg(p.wsp + k + 1), __ldg(yr + s1)) : 0.0f;
        V.y[r][k / 2] = make_float2(a, b);
      }
    }
    V.rv[r] = 0.0f;
    if (ROT && valid) {
      // sum over the tail coordinates of the squared gap to the whole bank's box, the same FP32
      // gap as bound_chunk (so every row's term is >= it), squares and sum in FP64, rounded down
      double t = 0.0;
#pragma unroll
      for (int k = kHead; k < LP; k += 2) {
        const float2 yk = V.y[r][k / 2];
        const float lo0 = __ldg(p.gbox + k), hi0 = __ldg(p.gbox + LP + k);
        const float lo1 = __ldg(p.gbox + k + 1), hi1 = __ldg(p.gbox + LP + k + 1);
        const float g0 = fmaxf(fmaxf(__fadd_rn(yk.x, lo0), -__fadd_rn(yk.x, hi0)), 0.0f);
        const float g1 = fmaxf(fmaxf(__fadd_rn(yk.y, lo1), -__fadd_rn(yk.y, hi1)), 0.0f);
        t += double(g0) * double(g0) + double(g1) * double(g1);
      }
      V.rv[r] = __double2float_rd(t * (1.0 - 1e-14));
    }
    V.cnt[r] = 0;
    V.taup[r] = INF;
    if (!p.eps_mode) {
      V.tau[r] = valid ? INF : -INF;
      if (valid && p.tau_glob) V.tau[r] = fminf(V.tau[r], __uint_as_float(__ldcg(p.tau_glob + slot)));
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
      V.tau[r] = valid ? nextafterf(__double2float_ru(p.eps + err), INF) : -INF;
    }
  }
}

// Per-voxel accumulator of the FP32 pass: float2 chains (even / odd frames).  VPET_ACC2 = 1 uses two
// float2 chains (frames 4q, 4q+1 and 4q+2, 4q+3): half the dependent FFMA2 latency per chunk, two
// more registers per voxel.  Every chain only grows (non-negative terms, monotone rounding), so any
// prefix total is <= the final D32 (exact pruning), and the total is a sum of the L terms in a
// tree of height < L (the gamma_L error bound holds).
#ifndef VPET_ACC2
#define VPET_ACC2 0
#endif
struct Acc {
  float2 a;
#if VPET_ACC2
  float2 b;
#endif
};
__device__ __forceinline__ void acc_zero(Acc& c) {
  c.a = make_float2(0.0f, 0.0f);
#if VPET_ACC2
  c.b = make_float2(0.0f, 0.0f);
#endif
}
__device__ __forceinline__ float acc_total(const Acc& c) {
#if VPET_ACC2
  return __fadd_rn(__fadd_rn(c.a.x, c.a.y), __fadd_rn(c.b.x, c.b.y));
#else
  return __fadd_rn(c.a.x, c.a.y);
#endif
}
__device__ __forceinline__ float2& acc_second(Acc& c) {
#if VPET_ACC2
  return c.b;
#else
  return c.a;
#endif
}

// Row / box sources.  Shared-memory rows are addressed by their 32-bit shared address and read with
// ld.shared (a generic pointer made the compiler re-derive the shared window base -- S2UR of the
// cluster CTA id -- inside the row loop).  Volatile: never moved above the ring's mbarrier wait.
__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
struct SmemSrc {
  uint32_t a;  // shared address of element 0
  __device__ __forceinline__ float4 ld(int q) const { return lds4(a + 4u * uint32_t(q)); }
  __device__ __forceinline__ SmemSrc off(int q) const { return SmemSrc{a + 4u * uint32_t(q)}; }
};
struct GmemSrc {
  const float* p;  // global memory, read-only during the scan
  __device__ __forceinline__ float4 ld(int q) const { return __ldg(reinterpret_cast<const float4*>(p + q)); }
  __device__ __forceinline__ GmemSrc off(int q) const { return GmemSrc{p + q}; }
};

// Chunk [c*CH, min((c+1)*CH, LP)) of the distance of R voxels to one bank row (scan order).
template <int LP, int R, int DIST, int C, class Src>
__device__ __forceinline__ void dist_chunk(const Voxels<LP, R>& V, const Src sr, Acc (&acc)[R]) {
#pragma unroll
  constexpr int CD = chd<LP>();
  for (int q = C * CD; q < ((C + 1) * CD < LP ? (C + 1) * CD : LP); q += 4) {
    const float4 s4 = sr.ld(q);
    const float2 sa = make_float2(s4.x, s4.y);
    const float2 sc = make_float2(s4.z, s4.w);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float2 d0 = __fadd2_rn(V.y[r][q / 2], sa);
      float2 d1 = __fadd2_rn(V.y[r][q / 2 + 1], sc);
      if (DIST == ABC_DIST_WL2) {
        acc[r].a = __ffma2_rn(d0, d0, acc[r].a);
        acc_second(acc[r]) = __ffma2_rn(d1, d1, acc_second(acc[r]));
      } else {
        acc[r].a.x = __fadd_rn(acc[r].a.x, fabsf(d0.x));
        acc[r].a.y = __fadd_rn(acc[r].a.y, fabsf(d0.y));
        acc_second(acc[r]).x = __fadd_rn(acc_second(acc[r]).x, fabsf(d1.x));
        acc_second(acc[r]).y = __fadd_rn(acc_second(acc[r]).y, fabsf(d1.y));
      }
    }
  }
}

// Same chunk of the lower bound against a box [lo, hi] of bankp values (shared memory for the
// prefetched super-tile / tile boxes, global memory for the hyper-tile boxes).
template <int LP, int R, int DIST, int C, class Src>
__device__ __forceinline__ void bound_chunk(const Voxels<LP, R>& V, const Src lo, const Src hi, Acc (&acc)[R]) {
#pragma unroll
  for (int q = C * CHB; q < ((C + 1) * CHB < LP ? (C + 1) * CHB : LP); q += 4) {
    const float4 l4 = lo.ld(q);
    const float4 h4 = hi.ld(q);
    const float2 la = make_float2(l4.x, l4.y), lc = make_float2(l4.z, l4.w);
    const float2 ha = make_float2(h4.x, h4.y), hc = make_float2(h4.z, h4.w);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      // d = fl(y + b) for b in [lo, hi]:  fl(y + lo) <= d <= fl(y + hi)  =>  |d| >= gap
      float2 a0 = __fadd2_rn(V.y[r][q / 2], la), b0 = __fadd2_rn(V.y[r][q / 2], ha);
      float2 a1 = __fadd2_rn(V.y[r][q / 2 + 1], lc), b1 = __fadd2_rn(V.y[r][q / 2 + 1], hc);
      float2 g0 = make_float2(fmaxf(fmaxf(a0.x, -b0.x), 0.0f), fmaxf(fmaxf(a0.y, -b0.y), 0.0f));
      float2 g1 = make_float2(fmaxf(fmaxf(a1.x, -b1.x), 0.0f), fmaxf(fmaxf(a1.y, -b1.y), 0.0f));
      if (DIST == ABC_DIST_WL2) {
        acc[r].a = __ffma2_rn(g0, g0, acc[r].a);
        acc_second(acc[r]) = __ffma2_rn(g1, g1, acc_second(acc[r]));
      } else {
        acc[r].a.x = __fadd_rn(acc[r].a.x, g0.x);
        acc[r].a.y = __fadd_rn(acc[r].a.y, g0.y);
        acc_second(acc[r]).x = __fadd_rn(acc_second(acc[r]).x, g1.x);
        acc_second(acc[r]).y = __fadd_rn(acc_second(acc[r]).y, g1.y);
      }
    }
  }
}

template <int LP, int R>
__device__ __forceinline__ bool any_alive(const Voxels<LP, R>& V, const Acc (&acc)[R], bool noprune) {
  bool alive = noprune;
#pragma unroll
  for (int r = 0; r < R; ++r) alive |= (acc_total(acc[r]) < V.tau[r]);
  return __any_sync(0xffffffffu, alive);
}

// Unrolled chunk loop with warp-uniform early exit after each chunk.
template <int LP, int R, int DIST, bool BOUND, int C>
struct Chunks {
  static constexpr int CHX = BOUND ? CHB : chd<LP>();
  static constexpr int NCH = (LP + CHX - 1) / CHX;
  template <class Src>
  __device__ __forceinline__ static bool run(const Voxels<LP, R>& V, const Src a, const Src b, Acc (&acc)[R],
                                             unsigned long long& work, bool noprune) {
    if (BOUND) bound_chunk<LP, R, DIST, C>(V, a, b, acc);
    else dist_chunk<LP, R, DIST, C>(V, a, acc);
    work += uint64_t(((C + 1) * CHX < LP ? (C + 1) * CHX : LP) - C * CHX) * R;
    if (!any_alive<LP, R>(V, acc, noprune)) return false;
    if constexpr (C + 1 < NCH) return Chunks<LP, R, DIST, BOUND, C + 1>::run(V, a, b, acc, work, noprune);
    return true;
  }
};

// Evaluate one bank row (scan order) against the thread's voxels; insert survivors.
#ifndef VPET_COUNT_PUSH
#define VPET_COUNT_PUSH 0  // tuning: count heap pushes instead of frame updates
#endif
#ifndef VPET_PUSHCHECK
#define VPET_PUSHCHECK 0  // re-read the shared threshold before a heap push
#endif
// Insert the survivors of draw i (full D32 in acc) into the lanes' candidate heaps.
template <int LP, int R, bool COUNT, bool SH>
__device__ __forceinline__ void finish_row(const ScanParams& p, Voxels<LP, R>& V, const Acc (&acc)[R], uint64_t i,
                                           uint32_t part, unsigned long long& work, uint32_t htop_s) {
#pragma unroll
  for (int r = 0; r < R; ++r) {
    float D = acc_total(acc[r]);
    if (VPET_PUSHCHECK && D < V.tau[r] && !p.eps_mode && p.tau_glob)
      V.tau[r] = fminf(V.tau[r], __uint_as_float(__ldcg(p.tau_glob + V.slot0 + uint32_t(r) * kSlotStride)));
    if (D < V.tau[r]) {
      if (!p.eps_mode) {
        unsigned long long key = (static_cast<unsigned long long>(__float_as_uint(D)) << 32) | uint32_t(i);
        if (COUNT && VPET_COUNT_PUSH) work += 1;
        unsigned long long* hb = p.heap + (uint64_t(V.vox[r]) * p.nparts + part) * heap_stride(p.K);
        uint2 st = SH ? heap_push_s(hb, htop_s + uint32_t(r) * NT * 72u, p.K, V.cnt[r], key)
                      : heap_push(hb, p.K, V.cnt[r], key);
#ifdef VPET_PUSH_STATS
        atomicAdd(p.work + 3, 1ull);
#endif
        V.cnt[r] = st.x;
        V.taup[r] = __uint_as_float(st.y);
        if (p.tau_glob && st.y != 0x7f800000u) atomicMin(p.tau_glob + V.slot0 + uint32_t(r) * kSlotStride, st.y);
        V.tau[r] = fminf(V.tau[r], V.taup[r]);
      } else {
        eps_candidate(p.tacs + uint64_t(V.vox[r]) * p.L, p.bank, p.LS, p.w, p.L, p.dist, p.eps,
                      p.mom + (uint64_t(V.vox[r]) * p.nparts + part) * (size_t(p.M) * MOMW), p.prior_g, i);
      }
    }
  }
}

template <int LP, int R, int DIST, bool COUNT, bool SH = false>
__device__ __forceinline__ void eval_row(const ScanParams& p, Voxels<LP, R>& V, const SmemSrc sr, uint64_t i,
                                         uint32_t part, unsigned long long& work, uint32_t htop_s = 0) {
  Acc acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc_zero(acc[r]);
  unsigned long long w = 0;
  bool go = Chunks<LP, R, DIST, false, 0>::run(V, sr, sr, acc, w, !p.prune);
  if (COUNT && !VPET_COUNT_PUSH) work += w;
  if (go) finish_row<LP, R, COUNT, SH>(p, V, acc, i, part, work, htop_s);
}

// Coordinates [Q0, Q1) of the distance of R voxels to one bank row (scan order).
template <int LP, int R, int DIST, int Q0, int Q1, class Src>
__device__ __forceinline__ void dist_range(const Voxels<LP, R>& V, const Src sr, Acc (&acc)[R]) {
#pragma unroll
  for (int q = Q0; q < Q1; q += 4) {
    const float4 s4 = sr.ld(q);
    const float2 sa = make_float2(s4.x, s4.y);
    const float2 sc = make_float2(s4.z, s4.w);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float2 d0 = __fadd2_rn(V.y[r][q / 2], sa);
      float2 d1 = __fadd2_rn(V.y[r][q / 2 + 1], sc);
      acc[r].a = __ffma2_rn(d0, d0, acc[r].a);
      acc_second(acc[r]) = __ffma2_rn(d1, d1, acc_second(acc[r]));
    }
  }
}

// Rotated basis (WL2): the first kHead coordinates, then a warp test against th = RU(RU(tau k) - rv),
// rv the voxel's tail bound, k = 1 + 2 (LP + kHead + 4) u: a row is dropped when every lane's
// prefix total is >= th, which implies D32 >= tau (the prefix is a FP32 sum of
// kHead / 2 + 1 roundings per chain, the rest of D32 adds terms >= the gaps summed in rv, and the
// whole sum rounds by at most (1 - u)^(LP / 2 + 1)).  th is computed per tile from the tau of the
// tile's start (a larger, older tau only keeps more rows).
constexpr float rot_tau_factor(int LP) { return 1.0f + float(2 * (LP + kHead + 4)) * 5.9604644775390625e-8f; }
template <int LP, int R>
__device__ __forceinline__ void rot_thresholds(const ScanParams& p, const Voxels<LP, R>& V, uint32_t rv_s, float (&th)[R]) {
#pragma unroll
  for (int r = 0; r < R; ++r) {
    float rv;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(rv) : "r"(rv_s + uint32_t(r) * NT * 4u));
    th[r] = p.prune ? __fsub_ru(__fmul_ru(V.tau[r], rot_tau_factor(LP)), rv) : __int_as_float(0x7f800000);
  }
}
template <int LP, int R, int DIST, bool COUNT, bool SH = false>
__device__ __forceinline__ void eval_row_rot(const ScanParams& p, Voxels<LP, R>& V, const SmemSrc sr, uint32_t i_a,
                                             uint32_t part, unsigned long long& work, uint32_t htop_s,
                                             const float (&th)[R]) {
  Acc acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc_zero(acc[r]);
  dist_range<LP, R, DIST, 0, kHead>(V, sr, acc);
  bool alive = false;
#pragma unroll
  for (int r = 0; r < R; ++r) alive |= acc_total(acc[r]) < th[r];
  const bool go = __any_sync(0xffffffffu, alive);
  if (COUNT && !VPET_COUNT_PUSH) work += uint64_t(kHead) * R;
  if (!go) return;
  dist_range<LP, R, DIST, kHead, LP>(V, sr, acc);
  if (COUNT && !VPET_COUNT_PUSH) work += uint64_t(LP - kHead) * R;
  uint32_t i;  // the draw index, read from the ring only for rows that pass the test
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(i) : "r"(i_a));
  finish_row<LP, R, COUNT, SH>(p, V, acc, i, part, work, htop_s);
}

// Two consecutive rows (at shared addresses ra, ra + 4 LP): both heads, one vote for the pair,
// then each row that passes its own vote is finished as in eval_row_rot.
#ifndef VPET_RPAIR
#define VPET_RPAIR 1
#endif
template <int LP, int R, int DIST, bool COUNT, bool SH = false>
__device__ __forceinline__ void eval_pair_rot(const ScanParams& p, Voxels<LP, R>& V, uint32_t ra, uint32_t ia,
                                              uint32_t part, unsigned long long& work, uint32_t htop_s,
                                              const float (&th)[R]) {
  Acc aa[R], ab[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    acc_zero(aa[r]);
    acc_zero(ab[r]);
  }
  const SmemSrc sa{ra}, sb{ra + 4u * LP};
  dist_range<LP, R, DIST, 0, kHead>(V, sa, aa);
  dist_range<LP, R, DIST, 0, kHead>(V, sb, ab);
  bool la = false, lb = false;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    la |= acc_total(aa[r]) < th[r];
    lb |= acc_total(ab[r]) < th[r];
  }
  if (COUNT && !VPET_COUNT_PUSH) work += 2ull * kHead * R;
  if (!__any_sync(0xffffffffu, la || lb)) return;
  if (__any_sync(0xffffffffu, la)) {
    dist_range<LP, R, DIST, kHead, LP>(V, sa, aa);
    if (COUNT && !VPET_COUNT_PUSH) work += uint64_t(LP - kHead) * R;
    uint32_t i;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(i) : "r"(ia));
    finish_row<LP, R, COUNT, SH>(p, V, aa, i, part, work, htop_s);
  }
  if (__any_sync(0xffffffffu, lb)) {
    dist_range<LP, R, DIST, kHead, LP>(V, sb, ab);
    if (COUNT && !VPET_COUNT_PUSH) work += uint64_t(LP - kHead) * R;
    uint32_t i;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(i) : "r"(ia + 4u));
    finish_row<LP, R, COUNT, SH>(p, V, ab, i, part, work, htop_s);
  }
}

// Two rows at once: their first chunks run interleaved (twice the independent FMA chains, one
// pair of votes), then each survivor continues alone.  Row B's first-chunk test may use the
// threshold from before row A's inserts: a larger threshold only keeps more, so this is exact.
template <int LP, int R, int DIST, bool COUNT, bool SH = false>
__device__ __forceinline__ void eval_pair(const ScanParams& p, Voxels<LP, R>& V, const SmemSrc sa, uint64_t ia,
                                          const SmemSrc sb, uint64_t ib, uint32_t part, unsigned long long& work,
                                          uint32_t htop_s = 0) {
  constexpr int NCH = (LP + chd<LP>() - 1) / chd<LP>();
  Acc aa[R], ab[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    acc_zero(aa[r]);
    acc_zero(ab[r]);
  }
  dist_chunk<LP, R, DIST, 0>(V, sa, aa);
  dist_chunk<LP, R, DIST, 0>(V, sb, ab);
  unsigned long long w = 2ull * uint64_t((chd<LP>() < LP ? chd<LP>() : LP)) * R;
  bool ga = any_alive<LP, R>(V, aa, !p.prune);
  bool gb = any_alive<LP, R>(V, ab, !p.prune);
  if constexpr (NCH > 1) {
    if (ga) ga = Chunks<LP, R, DIST, false, 1>::run(V, sa, sa, aa, w, !p.prune);
  }
  if (COUNT && !VPET_COUNT_PUSH) work += w;
  if (ga) finish_row<LP, R, COUNT, SH>(p, V, aa, ia, part, work, htop_s);
  w = 0;
  if constexpr (NCH > 1) {
    if (gb) gb = Chunks<LP, R, DIST, false, 1>::run(V, sb, sb, ab, w, !p.prune);
  }
  if (COUNT && !VPET_COUNT_PUSH) work += w;
  if (gb) finish_row<LP, R, COUNT, SH>(p, V, ab, ib, part, work, htop_s);
}

// Pull the other parts' progress on the shared thresholds.
template <int LP, int R>
__device__ __forceinline__ void refresh_tau(const ScanParams& p, Voxels<LP, R>& V) {
  if (p.eps_mode || !p.tau_glob) return;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (V.vox[r] < p.J) {
      float g = __uint_as_float(__ldcg(p.tau_glob + V.slot0 + uint32_t(r) * kSlotStride));
      V.tau[r] = fminf(V.tau[r], g);
    }
  }
}

// Split refresh: issue the loads (early), apply them (late).
template <int LP, int R>
__device__ __forceinline__ void refresh_issue(const ScanParams& p, const Voxels<LP, R>& V, float (&g)[R]) {
#pragma unroll
  for (int r = 0; r < R; ++r)
    g[r] = (!p.eps_mode && p.tau_glob && V.vox[r] < p.J) ? __uint_as_float(__ldcg(p.tau_glob + V.slot0 + uint32_t(r) * kSlotStride))
                                                          : __int_as_float(0x7f800000);
}
template <int LP, int R>
__device__ __forceinline__ void refresh_apply(Voxels<LP, R>& V, const float (&g)[R]) {
#pragma unroll
  for (int r = 0; r < R; ++r) V.tau[r] = fminf(V.tau[r], g[r]);
}

// Software-pipelined variant: apply the value loaded at the previous call, issue the next load.
template <int LP, int R>
__device__ __forceinline__ void refresh_tau_pipe(const ScanParams& p, Voxels<LP, R>& V, float (&gpend)[R]) {
  if (p.eps_mode || !p.tau_glob) return;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    V.tau[r] = fminf(V.tau[r], gpend[r]);
    if (V.vox[r] < p.J) gpend[r] = __uint_as_float(__ldcg(p.tau_glob + V.slot0 + uint32_t(r) * kSlotStride));
  }
}

template <int LP, int R, int DIST>
__device__ __forceinline__ bool box_alive(const Voxels<LP, R>& V, const GmemSrc box, unsigned long long& work) {
  Acc acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc_zero(acc[r]);
  return Chunks<LP, R, DIST, true, 0>::run(V, box, box.off(LP), acc, work, false);
}
template <int LP, int R, int DIST>
__device__ __forceinline__ bool box_alive(const Voxels<LP, R>& V, const SmemSrc box, unsigned long long& work) {
  Acc acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc_zero(acc[r]);
  return Chunks<LP, R, DIST, true, 0>::run(V, box, box.off(LP), acc, work, false);
}

// Coordinates [Q0, Q1) of the box lower bound (WL2), as bound_chunk.
template <int LP, int R, int Q0, int Q1, class Src>
__device__ __forceinline__ void bound_range(const Voxels<LP, R>& V, const Src lo, const Src hi, Acc (&acc)[R]) {
#pragma unroll
  for (int q = Q0; q < Q1; q += 4) {
    const float4 l4 = lo.ld(q);
    const float4 h4 = hi.ld(q);
    const float2 la = make_float2(l4.x, l4.y), lc = make_float2(l4.z, l4.w);
    const float2 ha = make_float2(h4.x, h4.y), hc = make_float2(h4.z, h4.w);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      float2 a0 = __fadd2_rn(V.y[r][q / 2], la), b0 = __fadd2_rn(V.y[r][q / 2], ha);
      float2 a1 = __fadd2_rn(V.y[r][q / 2 + 1], lc), b1 = __fadd2_rn(V.y[r][q / 2 + 1], hc);
      float2 g0 = make_float2(fmaxf(fmaxf(a0.x, -b0.x), 0.0f), fmaxf(fmaxf(a0.y, -b0.y), 0.0f));
      float2 g1 = make_float2(fmaxf(fmaxf(a1.x, -b1.x), 0.0f), fmaxf(fmaxf(a1.y, -b1.y), 0.0f));
      acc[r].a = __ffma2_rn(g0, g0, acc[r].a);
      acc_second(acc[r]) = __ffma2_rn(g1, g1, acc_second(acc[r]));
    }
  }
}

// Rotated basis: the box's first kHead coordinates tested against th (as eval_row_rot: every
// draw of the box then has D32 >= tau), then the whole lower bound against tau.
template <int LP, int R, class Src>
__device__ __forceinline__ bool box_alive_rot(const Voxels<LP, R>& V, const Src box, const float (&th)[R],
                                              unsigned long long& work) {
  Acc acc[R];
#pragma unroll
  for (int r = 0; r < R; ++r) acc_zero(acc[r]);
  bound_range<LP, R, 0, kBoxHead>(V, box, box.off(LP), acc);
  work += uint64_t(kBoxHead) * R;
  bool alive = false;
#pragma unroll
  for (int r = 0; r < R; ++r) alive |= acc_total(acc[r]) < th[r];
  if (!__any_sync(0xffffffffu, alive)) return false;
  bound_range<LP, R, kBoxHead, LP>(V, box, box.off(LP), acc);
  work += uint64_t(LP - kBoxHead) * R;
  alive = false;
#pragma unroll
  for (int r = 0; r < R; ++r) alive |= acc_total(acc[r]) < V.tau[r];
  return __any_sync(0xffffffffu, alive);
}

// th[r] = RU(RU(tau k) - rv) (eval_row_rot), +inf without pruning
template <int LP, int R>
__device__ __forceinline__ void rot_thresholds(const ScanParams& p, const Voxels<LP, R>& V, uint32_t rv_s, float (&th)[R]);

template <int LP, int R>
__device__ __forceinline__ void store_counts(const ScanParams& p, const Voxels<LP, R>& V, uint32_t part,
                                             const unsigned long long* htop = nullptr) {
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (V.vox[r] < p.J && !p.eps_mode) {
      const uint64_t row = uint64_t(V.vox[r]) * p.nparts + part;
      p.heap_cnt[row] = V.cnt[r];
      if (htop) {  // write the shared-memory top of the heap back (certify reads the whole heap)
        unsigned long long* h = p.heap + row * heap_stride(p.K) + kHeapOff;
        const unsigned long long* t = htop + size_t(r) * NT * 9;
        const uint32_t nt = V.cnt[r] < 9u ? V.cnt[r] : 9u;
        for (uint32_t j = 0; j < nt; ++j) h[j] = t[j];
      }
    }
}

__device__ __forceinline__ void finish_counts(const ScanParams& p, unsigned long long work, unsigned long long bwork,
                                              int lane, bool count) {
  if (count) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      work += __shfl_xor_sync(0xffffffffu, work, o);
      bwork += __shfl_xor_sync(0xffffffffu, bwork, o);
    }
    if (lane == 0) {
      atomicAdd(p.work, work);
      if (p.bound_work) atomicAdd(p.bound_work, bwork);
    }
  }
}

// =============================================================================================
// Flat scan: every tile, index order (ABC_FLAG_NO_TREE, and N >= 2^31).
// =============================================================================================
template <int LP, int DIST, bool COUNT>
__global__ void __launch_bounds__(NT, Shape<LP>::MINB) scan_flat_kernel(const ScanParams p) {
  constexpr int R = Shape<LP>::R;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stage = reinterpret_cast<float*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + NST * (Shape<LP>::STAGE_FLOATS * 4 + T * 4));
  int* arrivals = reinterpret_cast<int*>(full + NST);
  if (p.bad && *p.bad) return;  // non-finite TACs: the call fails with ABC_E_ARG, skip the work
  const int tid = threadIdx.x, lane = tid & 31;
  const uint64_t N = p.N;
  const uint32_t ntile = uint32_t((N + T - 1) / T);
  const float* __restrict__ bankp = p.bankp;
  auto issue = [=](uint32_t tt, int ss) {
    uint64_t i0 = uint64_t(tt) * T;
    uint32_t nd = uint32_t((N - i0) < uint64_t(T) ? (N - i0) : uint64_t(T));
    mbar_expect_tx(&full[ss], nd * LP * 4u);
    bulk_g2s(stage + size_t(ss) * Shape<LP>::STAGE_FLOATS, bankp + i0 * LP, nd * LP * 4u, &full[ss]);
  };
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      arrivals[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0)
    for (uint32_t s = 0; s < uint32_t(NST) && s < ntile; ++s) issue(s, int(s));
  Voxels<LP, R> V;
  load_voxels<LP, R>(p, V, tid, blockIdx.x);
  unsigned long long work = 0;
  for (uint32_t t = 0; t < ntile; ++t) {
    const int s = int(t % NST);
    mbar_wait(&full[s], (t / NST) & 1u);
    const float* sb = stage + size_t(s) * Shape<LP>::STAGE_FLOATS;
    const uint64_t rem = N - uint64_t(t) * T;
    const uint32_t nd = uint32_t(rem < uint64_t(T) ? rem : uint64_t(T));
    const uint64_t ibase = uint64_t(t) * T;
    for (uint32_t d = 0; d < nd; ++d) eval_row<LP, R, DIST, COUNT>(p, V, SmemSrc{smem_u32(sb) + 4u * d * LP}, ibase + d, 0u, work);
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
  store_counts<LP, R>(p, V, 0u);
  finish_counts(p, work, 0ull, lane, COUNT);
}

// Ascending bitonic sort of P2 (a power of two) keys in shared memory by the whole CTA (NTH threads).
template <int NTH>
__device__ __forceinline__ void cta_bitonic(unsigned long long* key, uint32_t P2, int tid) {
  for (uint32_t kk = 2; kk <= P2; kk <<= 1) {
    for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
      for (uint32_t i = tid; i < P2; i += NTH) {
        const uint32_t l = i ^ jj;
        if (l > i) {
          const unsigned long long a = key[i], b = key[l];
          if ((a > b) == ((i & kk) == 0)) { key[i] = b; key[l] = a; }
        }
      }
      __syncthreads();
    }
  }
}

// Best-first visiting order of n boxes for the CTA: each warp ranks the boxes by the lower bound of
// its mean TAC (lbs[w][k]); the CTA order alternates between the warps' rankings (warp 0's best,
// warp 1's best, warp 0's second, ...) skipping boxes already taken and warps without voxels.
// keys: [NW * kHyperSort] scratch; order: [kHyperSort] output; vis: [kHyperSort / 32] scratch.
template <int NTH>
__device__ __forceinline__ void best_first_n(const float* lbs, uint32_t n, unsigned long long* keys, uint32_t* order,
                                             uint32_t* vis, int tid) {
  constexpr int NW = NTH / 32;
  uint32_t P2 = 1;
  while (P2 < n) P2 <<= 1;
  for (uint32_t e = tid; e < NW * P2; e += NTH) {
    const uint32_t w = e / P2, k = e % P2;
    const uint32_t lbb = k < n ? __float_as_uint(lbs[w * kHyperSort + k]) : 0x7fffffffu;
    keys[e] = (static_cast<unsigned long long>(w) << 62) | (static_cast<unsigned long long>(lbb) << 16) | k;
  }
  for (uint32_t e = tid; e < kHyperSort / 32; e += NTH) vis[e] = 0u;
  __syncthreads();
  cta_bitonic<NTH>(keys, NW * P2, tid);
  if (tid == 0) {
    uint32_t ptr[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) ptr[w] = 0;
    uint32_t q = 0, turn = 0;
    while (q < n) {
      bool took = false;
      for (int a = 0; a < NW && !took; ++a) {
        const uint32_t w = (turn + a) % NW;
        while (ptr[w] < n) {
          const unsigned long long kk = keys[w * P2 + ptr[w]];
          const uint32_t k = uint32_t(kk & 0xffffu), lbb = uint32_t((kk >> 16) & 0x7fffffffu);
          if (lbb >= 0x7f800000u) { ptr[w] = n; break; }  // warp without voxels (or no bound)
          if ((vis[k >> 5] >> (k & 31)) & 1u) { ++ptr[w]; continue; }
          vis[k >> 5] |= 1u << (k & 31);
          order[q++] = k;
          ++ptr[w];
          took = true;
          break;
        }
      }
      if (!took) {  // every ranking exhausted: append the rest in index order
        for (uint32_t k = 0; k < n; ++k)
          if (!((vis[k >> 5] >> (k & 31)) & 1u)) order[q++] = k;
        break;
      }
      turn = (turn + 1) % NW;
    }
  }
  __syncthreads();
}

// Lower bound of a mean TAC (shared memory, LP frames) against a box [lo; hi] (global memory).
template <int LP>
__device__ __forceinline__ float mean_lb(const float* yb, const float* lo) {
  const float* hi = lo + LP;
  float lb = 0.0f;
  for (int f = 0; f < LP; f += 4) {
    const float4 l4 = __ldg(reinterpret_cast<const float4*>(lo + f));
    const float4 h4 = __ldg(reinterpret_cast<const float4*>(hi + f));
    const float l[4] = {l4.x, l4.y, l4.z, l4.w}, h[4] = {h4.x, h4.y, h4.z, h4.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float g = fmaxf(fmaxf(yb[f + u] + l[u], -(yb[f + u] + h[u])), 0.0f);
      lb = fmaf(g, g, lb);
    }
  }
  return lb;
}

// =============================================================================================
// Tree scan: Morton-ordered bank, hyper-tile / super-tile / tile bounds, best-first order.
// =============================================================================================
template <int LP, int DIST, bool COUNT, bool ROT = false>
__global__ void __launch_bounds__(NT, ROT ? Shape<LP>::MINB_ROT : Shape<LP>::MINB) scan_tree_kernel(const ScanParams p) {
  constexpr int R = Shape<LP>::R;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* stage = reinterpret_cast<float*>(smem_raw);  // [NST][STAGE_FLOATS] TMA ring
  // best-first sort scratch, aliasing the ring (the ring is idle whenever an order is computed)
  unsigned long long* okeys = reinterpret_cast<unsigned long long*>(
      smem_raw + (VPET_ALIAS ? 0 : Shape<LP>::RING_BYTES));  // [NW][kHyperSort]
  float* hlb = reinterpret_cast<float*>(okeys + NW * kHyperSort);               // [NW][kHyperSort]
  uint32_t* vis = reinterpret_cast<uint32_t*>(hlb + NW * kHyperSort);           // [kHyperSort / 32]
  unsigned char* after = smem_raw + Shape<LP>::REGION;
  uint32_t* sidx = reinterpret_cast<uint32_t*>(after);
  uint64_t* full = reinterpret_cast<uint64_t*>(after + NST * T * 4);
  int* arrivals = reinterpret_cast<int*>(full + NST);
  uint32_t* wmask = reinterpret_cast<uint32_t*>(arrivals + NST);
  float* ybar = reinterpret_cast<float*>(wmask + NW);
  int* s_item = reinterpret_cast<int*>(ybar + NW * LP);
  // 16-B aligned sub-buffers, addressed as smem_raw + offset (so the compiler keeps the shared
  // address space and emits LDS, not generic loads, for the prefetched boxes)
  auto align16 = [&](const void* q) { return (size_t(static_cast<const unsigned char*>(q) - smem_raw) + 15) & ~size_t(15); };
  uint32_t* horder = reinterpret_cast<uint32_t*>(smem_raw + align16(s_item + 4));  // [kHyperSort] hyper-tile order
  uint32_t* sorder = horder + kHyperSort;                                            // [kHyperSort] super-tile order
  constexpr size_t BXF = Shape<LP>::BOXB_FLOATS;
  float* bbuf = reinterpret_cast<float*>(smem_raw + align16(sorder + kHyperSort));  // [2][BXF]
  uint64_t* bbar = reinterpret_cast<uint64_t*>(bbuf + 2 * BXF);                    // [2]
  const uint32_t stage_a = smem_u32(stage), bbuf_a = smem_u32(bbuf);  // 32-bit shared addresses
  const uint32_t sidx_a = smem_u32(sidx);
  unsigned long long* htop = reinterpret_cast<unsigned long long*>(smem_raw + align16(bbar + 2));  // [R][NT][9]
  unsigned long long* htop_t = VPET_SHEAP ? htop + threadIdx.x * 9 : nullptr;
  const uint32_t htop_s = smem_u32(htop) + uint32_t(threadIdx.x) * 72u;  // this thread's heap tops (bytes)
  // rotated basis: this thread's tail bounds rv[R] ([R][NT] floats after the heap tops)
  const uint32_t rv_s = uint32_t(align16(reinterpret_cast<unsigned char*>(htop) + Shape<LP>::HTOP_BYTES)) +
                        smem_u32(smem_raw) + uint32_t(threadIdx.x) * 4u;

  if (p.bad && *p.bad) return;  // non-finite TACs: the call fails with ABC_E_ARG, skip the work
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t N = p.N;
  const float* __restrict__ bankp = p.bankp;
  const uint32_t* __restrict__ idxmap = p.idxmap;
  auto issue = [=](uint64_t tt, int ss) {
    uint64_t i0 = tt * T;
    uint32_t nd = uint32_t((N - i0) < uint64_t(T) ? (N - i0) : uint64_t(T));
    uint32_t ndp = (nd + 3u) & ~3u;  // idxmap is padded to a multiple of 4 entries (16-B copies)
    mbar_expect_tx(&full[ss], nd * LP * 4u + ndp * 4u);
    bulk_g2s(stage + size_t(ss) * Shape<LP>::STAGE_FLOATS, bankp + i0 * LP, nd * LP * 4u, &full[ss]);
    bulk_g2s(sidx + ss * T, idxmap + i0, ndp * 4u, &full[ss]);
  };
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      arrivals[s] = 0;
    }
    mbar_init(&bbar[0], 1);
    mbar_init(&bbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint32_t bcount = 0;  // super-tile box buffers consumed (CTA-uniform)
  auto prefetch_boxes = [&](uint64_t sx, uint32_t b) {
    const uint64_t a0 = sx * kSuper;
    const uint64_t a1 = (a0 + kSuper < p.ntile) ? a0 + kSuper : p.ntile;
    const uint32_t sbytes = 2 * LP * 4, tbytes = uint32_t(a1 - a0) * 2 * LP * 4;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&bbar[b], sbytes + tbytes);
    bulk_g2s(bbuf + b * BXF, p.sbounds + sx * 2 * LP, sbytes, &bbar[b]);
    bulk_g2s(bbuf + b * BXF + 2 * LP, p.tbounds + a0 * 2 * LP, tbytes, &bbar[b]);
  };
  const uint32_t S = p.nparts;
  const uint64_t nvt = (p.J + uint64_t(NT) * R - 1) / (uint64_t(NT) * R);
  const uint64_t nitems = nvt * S;
  unsigned long long work = 0, bwork = 0;
  uint32_t consumed = 0;  // ring position (persists across items)

  // Persistent CTA: pull (voxel tile, part) items; parts of a tile are adjacent in the queue so
  // they run concurrently on different SMs and tighten each other's thresholds via tau_glob.
  for (;;) {
    if (tid == 0) *s_item = int(atomicAdd(p.queue, 1u));
    __syncthreads();
    const uint64_t item = uint64_t(uint32_t(*s_item));
    __syncthreads();
    if (item >= nitems) break;
#ifndef VPET_QORDER
#define VPET_QORDER 3
#endif
    // queue order of voxel tiles (the voxel order is PC1-major Morton): 3 = both ends of the PC1
    // range first, alternating (0, last, 1, last-1, ...).  The extremes are the long items: high
    // activity (thresholds grow with the noise) and near-zero TACs (where the prior puts
    // many draws); longest-first scheduling of the persistent queue shortens the tail.
    // 0 = Morton order, 1 = reversed, 2 = strided.
    const uint64_t nvt_ = nvt;
    uint64_t vt = item / S;
    if (VPET_QORDER == 1) vt = nvt_ - 1 - vt;
    if (VPET_QORDER == 2) vt = (vt * 613ull) % nvt_;
    if (VPET_QORDER == 3) vt = (vt & 1) ? nvt_ - 1 - (vt >> 1) : (vt >> 1);  // both ends first
    const uint32_t part = uint32_t(item % S);
    unsigned long long t_item0 = 0;
    if (p.item_log && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_item0));
    const uint64_t nsub = (p.nhyper > part) ? (p.nhyper - part + S - 1) / S : 0;  // hyper-tiles of this part
    Voxels<LP, R> V;
    load_voxels<LP, R, ROT>(p, V, tid, vt);
    if constexpr (ROT) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(rv_s + uint32_t(r) * NT * 4u), "f"(V.rv[r]) : "memory");
    }

    // ---- best-first order of this part's hyper-tiles: key = min over warps of the lower bound of
    // the warp's mean TAC against the hyper-tile box (a heuristic order; exactness does not depend
    // on it).  Sorted in shared memory (bitonic), then scanned in that order.
    bool wvalid;
    {
      int nvalid = 0;
#pragma unroll
      for (int r = 0; r < R; ++r) nvalid += (V.vox[r] < p.J);
      nvalid = __reduce_add_sync(0xffffffffu, nvalid);
      wvalid = nvalid > 0;
      float inv = nvalid > 0 ? 1.0f / float(nvalid) : 0.0f;
#pragma unroll
      for (int k = 0; k < LP / 2; ++k) {
        float2 sm = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (V.vox[r] < p.J) { sm.x += V.y[r][k].x; sm.y += V.y[r][k].y; }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          sm.x += __shfl_xor_sync(0xffffffffu, sm.x, o);
          sm.y += __shfl_xor_sync(0xffffffffu, sm.y, o);
        }
        if (lane == 0) {
          ybar[wid * LP + 2 * k] = sm.x * inv;
          ybar[wid * LP + 2 * k + 1] = sm.y * inv;
        }
      }
      __syncwarp();
      for (uint64_t k = lane; k < nsub; k += 32) {
        const float lb = mean_lb<LP>(ybar + wid * LP, p.hbounds + (part + k * S) * 2 * LP);
        hlb[wid * kHyperSort + k] = wvalid ? lb : __int_as_float(0x7f800000);
      }
    }
    __syncthreads();
    best_first_n<NT>(hlb, uint32_t(nsub), okeys, horder, vis, tid);

    uint32_t it = 0;
    float gpend[R];
#pragma unroll
    for (int r = 0; r < R; ++r) gpend[r] = __int_as_float(0x7f800000);
    for (uint32_t q = 0; q < nsub; ++q) {
      const uint64_t h = part + uint64_t(horder[q]) * S;
      if ((q & uint32_t(ROT ? VPET_HREFRESH_ROT : VPET_HREFRESH)) == 0) refresh_tau<LP, R>(p, V);
      bool halive;
      if constexpr (ROT) {
        float thh[R];
        rot_thresholds<LP, R>(p, V, rv_s, thh);
        halive = box_alive_rot<LP, R>(V, GmemSrc{p.hbounds + h * 2 * LP}, thh, bwork);
      } else {
        halive = box_alive<LP, R, DIST>(V, GmemSrc{p.hbounds + h * 2 * LP}, bwork);
      }
      if (!__syncthreads_or(halive)) continue;
      const uint64_t s0 = h * p.hs;
      const uint32_t ns = uint32_t(((s0 + p.hs < p.nsuper) ? s0 + p.hs : p.nsuper) - s0);
      const bool ssort = VPET_SSORT && ns <= uint32_t(kHyperSort);
      if (ssort) {  // best-first order of the super-tiles inside the hyper-tile
        for (uint32_t k = lane; k < ns; k += 32)
          hlb[wid * kHyperSort + k] =
              wvalid ? mean_lb<LP>(ybar + wid * LP, p.sbounds + (s0 + k) * 2 * LP) : __int_as_float(0x7f800000);
        __syncthreads();
        best_first_n<NT>(hlb, ns, okeys, sorder, vis, tid);
      }
      for (uint32_t u = 0; u < ns; ++u, ++it) {
      const uint64_t s = s0 + (ssort ? sorder[u] : u);
      // boxes of this super-tile (and its tiles) arrive by TMA; the next one's are requested now
      const uint32_t cur = bcount & 1u;
      if (tid == 0) {
        if (u == 0) prefetch_boxes(s, cur);
        if (u + 1 < ns) prefetch_boxes(s0 + (ssort ? sorder[u + 1] : u + 1), cur ^ 1u);
      }
      {
        constexpr uint32_t kRef = ROT ? VPET_REFRESH_ROT : VPET_REFRESH;
        if ((it & kRef) == kRef) refresh_tau<LP, R>(p, V);
      }
      mbar_wait(&bbar[cur], (bcount >> 1) & 1u);
      ++bcount;
      // super-tile bound
      const uint32_t sbx_a = bbuf_a + cur * uint32_t(BXF) * 4u;  // shared address of the boxes
      float ths[R];
      if constexpr (ROT) rot_thresholds<LP, R>(p, V, rv_s, ths);
      bool alive;
      if constexpr (ROT) alive = halive && box_alive_rot<LP, R>(V, SmemSrc{sbx_a}, ths, bwork);
      else alive = halive && box_alive<LP, R, DIST>(V, SmemSrc{sbx_a}, bwork);
#ifdef VPET_TRAV_STATS
      if (tid == 0) atomicAdd(p.work + 1, 1ull << 32);  // super-tiles bound-checked (high word of bound_work)
#endif
      if (!__syncthreads_or(alive)) continue;
      // tile bounds -> per-warp masks
      const uint64_t t0 = s * kSuper;
      const uint64_t t1 = (t0 + kSuper < p.ntile) ? t0 + kSuper : p.ntile;
      uint32_t mask = 0;
      if (alive) {
        for (uint64_t t = t0; t < t1; ++t)
          if (ROT ? box_alive_rot<LP, R>(V, SmemSrc{sbx_a + 4u * uint32_t(2 * LP + (t - t0) * 2 * LP)}, ths, bwork)
                  : box_alive<LP, R, DIST>(V, SmemSrc{sbx_a + 4u * uint32_t(2 * LP + (t - t0) * 2 * LP)}, bwork))
            mask |= 1u << uint32_t(t - t0);
      }
#ifdef VPET_UNION_STATS
      // diagnostic: voxel-lanes a warp evaluates per tile (R x 32) vs those whose own complete tile
      // bound is below their threshold (the work a per-(tile, voxel) schedule would do)
      if (COUNT && alive) {
        unsigned long long ev = 0, al = 0;
        for (uint32_t b = 0; b < uint32_t(t1 - t0); ++b) {
          if (!((mask >> b) & 1u)) continue;
          Acc acc[R];
#pragma unroll
          for (int r = 0; r < R; ++r) acc_zero(acc[r]);
          unsigned long long dummy = 0;
          const SmemSrc bx{sbx_a + 4u * uint32_t(2 * LP + b * 2 * LP)};
          Chunks<LP, R, DIST, true, 0>::run(V, bx, bx.off(LP), acc, dummy, true);
          int c = 0;
#pragma unroll
          for (int r = 0; r < R; ++r) c += (acc_total(acc[r]) < V.tau[r]) ? 1 : 0;
          c = __reduce_add_sync(0xffffffffu, c);
          ev += uint64_t(R) * 32u;
          al += uint64_t(c);
        }
        if (lane == 0) {
          atomicAdd(p.work + 2, ev);
          atomicAdd(p.work + 3, al);
        }
      }
#endif
      if (lane == 0) wmask[wid] = mask;
      __syncthreads();
      uint32_t cm = 0;
#pragma unroll
      for (int w = 0; w < NW; ++w) cm |= wmask[w];
      const uint32_t mym = wmask[wid];
      const uint32_t nal = __popc(cm);
#ifdef VPET_TRAV_STATS
      // diagnostic: super-tiles that passed the super bound (per CTA) and tiles loaded (per CTA)
      if (tid == 0) {
        atomicAdd(p.work + 2, 1ull);
        atomicAdd(p.work + 3, 1ull * nal);
      }
#endif
      if (tid == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        uint32_t m = cm;
        for (uint32_t q = 0; q < nal && q < uint32_t(NST); ++q) {
          uint32_t b = __ffs(m) - 1;
          m &= m - 1;
          issue(t0 + b, int((consumed + q) % NST));
        }
      }
      uint32_t rest = cm;
      for (uint32_t q = 0; q < nal; ++q) {
        const uint32_t b = __ffs(rest) - 1;
        rest &= rest - 1;
        const uint64_t t = t0 + b;
        const uint32_t g = consumed + q;
        const int st = int(g % NST);
        // every warp observes every phase of the ring (parity waits are only unambiguous when no
        // phase is skipped), then only the warps whose lanes can improve evaluate the tile
        // VPET_TREFRESH 3: the shared-threshold load is issued before the ring wait, so its L2 round
        // trip overlaps the wait (the value is as fresh as mode 2's up to the wait time)
        float gnow[R];
        if (VPET_TREFRESH == 3 && ((mym >> b) & 1u)) refresh_issue<LP, R>(p, V, gnow);
        mbar_wait(&full[st], (g / NST) & 1u);
        if ((mym >> b) & 1u) {
          if (VPET_TREFRESH == 1) refresh_tau_pipe<LP, R>(p, V, gpend);
          if (VPET_TREFRESH == 2) refresh_tau<LP, R>(p, V);
          if (VPET_TREFRESH == 3) refresh_apply<LP, R>(V, gnow);
          const uint32_t sb_a = stage_a + uint32_t(st) * uint32_t(Shape<LP>::STAGE_FLOATS) * 4u;
          float th[R];  // rotated basis: per-tile row threshold (eval_row_rot)
          if constexpr (ROT) rot_thresholds<LP, R>(p, V, rv_s, th);
          const uint32_t* si = sidx + st * T;
          const uint32_t si_a = sidx_a + 4u * uint32_t(st * T);  // shared address of si
          const uint64_t rem = N - t * T;
          const uint32_t nd = uint32_t(rem < uint64_t(T) ? rem : uint64_t(T));
#ifndef VPET_PAIR
#define VPET_PAIR 0
#endif
          uint32_t d = 0;
          // VPET_TREFRESH 4: the shared-threshold load is issued here and applied after the first
          // kTrefreshRows rows, so its L2 round trip hides behind their evaluation (those rows use
          // the threshold of the previous tile: larger, so they only keep more -- still exact)
          constexpr uint32_t kTrefreshRows = 4;
          if (VPET_TREFRESH == 4) {
            float gnow4[R];
            refresh_issue<LP, R>(p, V, gnow4);
            const uint32_t d0 = nd < kTrefreshRows ? nd : kTrefreshRows;
            for (; d < d0; ++d)
              {
              if constexpr (ROT) eval_row_rot<LP, R, DIST, COUNT, VPET_SHEAP != 0>(p, V, SmemSrc{sb_a + 4u * d * LP}, si_a + 4u * d, part, work, htop_s, th);
              else eval_row<LP, R, DIST, COUNT, VPET_SHEAP != 0>(p, V, SmemSrc{sb_a + 4u * d * LP}, si[d], part, work, htop_s);
            }
            refresh_apply<LP, R>(V, gnow4);
          }
          if (VPET_PAIR)
            for (; d + 1 < nd; d += 2)
              eval_pair<LP, R, DIST, COUNT, VPET_SHEAP != 0>(p, V, SmemSrc{sb_a + 4u * d * LP}, si[d],
                                                              SmemSrc{sb_a + 4u * (d + 1) * LP}, si[d + 1],
                                                              part, work, htop_s);
          if constexpr (ROT) {
            // row addresses as induction variables (keeps the shared base out of the loop)
            uint32_t ra = sb_a + 4u * d * LP, ia = si_a + 4u * d;
            if (VPET_RPAIR)
              for (; d + 1 < nd; d += 2, ra += 8u * LP, ia += 8u)
                eval_pair_rot<LP, R, DIST, COUNT, VPET_SHEAP != 0>(p, V, ra, ia, part, work, htop_s, th);
            for (; d < nd; ++d, ra += 4u * LP, ia += 4u)
              eval_row_rot<LP, R, DIST, COUNT, VPET_SHEAP != 0>(p, V, SmemSrc{ra}, ia, part, work, htop_s, th);
          } else {
            for (; d < nd; ++d)
              eval_row<LP, R, DIST, COUNT, VPET_SHEAP != 0>(p, V, SmemSrc{sb_a + 4u * d * LP}, si[d], part, work, htop_s);
          }
        }
        __syncwarp();
        if (lane == 0) {
          __threadfence_block();
          int old = atomicAdd(&arrivals[st], 1);
          if (old == NW - 1) {
            atomicExch(&arrivals[st], 0);
            if (q + NST < nal) {
              uint32_t m = rest;  // tiles after q; the (NST-1)-th of them is q + NST
              for (int kk = 0; kk < NST - 1; ++kk) m &= m - 1;
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              issue(t0 + (__ffs(m) - 1), st);
            }
          }
        }
      }
      consumed += nal;
      }
    }
    store_counts<LP, R>(p, V, part, htop_t);
    if (p.item_log && tid == 0) {
      unsigned long long t1, smid;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      uint32_t sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      smid = sm;
      p.item_log[item * 4 + 0] = t_item0;
      p.item_log[item * 4 + 1] = t1;
      p.item_log[item * 4 + 2] = smid;
      p.item_log[item * 4 + 3] = vt;
    }
  }
  finish_counts(p, work, bwork, lane, COUNT);
}

template <int LP, int DIST, bool COUNT, bool TREE, bool ROT = false>
cudaError_t launch_one(const ScanParams& p, cudaStream_t st) {
  using S = Shape<LP>;
  auto kern = TREE ? scan_tree_kernel<LP, DIST, COUNT, ROT> : scan_flat_kernel<LP, DIST, COUNT>;
  {
    cudaError_t e = ensure_smem_attr((const void*)kern, S::SMEM);
    if (e != cudaSuccess) return e;
  }
  uint64_t per_cta = uint64_t(NT) * S::R;
  uint64_t nvt = (p.J + per_cta - 1) / per_cta;
  uint64_t grid = nvt;
  if (TREE) {  // persistent: one CTA per resident slot, items pulled from p.queue
    int dev = 0, nsm = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, NT, S::SMEM);
    if (getenv("VPET_SHOW_OCC")) fprintf(stderr, "scan LP=%d smem=%zu occupancy=%d CTAs/SM\n", LP, S::SMEM, occ);
    uint64_t slots = uint64_t(nsm) * uint64_t(occ > 0 ? occ : 1);
    uint64_t items = nvt * p.nparts;
    grid = items < slots ? items : slots;
  }
  kern<<<unsigned(grid), NT, S::SMEM, st>>>(p);
  return cudaGetLastError();
}

#define VPET_LP_LIST(X) X(8) X(12) X(16) X(20) X(24) X(28) X(32) X(36) X(40) X(44) X(48) X(56) X(64) X(80) X(96) X(128)

template <int DIST>
cudaError_t launch_dist(const ScanParams& p, uint32_t LP, int count_work, int tree, cudaStream_t st) {
  // rotated basis (p.ytr): WL2, kHead < LP (api.cu selects it only for WL2)
  const bool rot = p.ytr != nullptr;
#define X(v)                                                                          \
  if (LP == v) {                                                                      \
    if constexpr (DIST == ABC_DIST_WL2 && v > kHead) {                                \
      if (tree && rot)                                                                \
        return count_work ? launch_one<v, DIST, true, true, true>(p, st) : launch_one<v, DIST, false, true, true>(p, st); \
    }                                                                                 \
    if (tree) return count_work ? launch_one<v, DIST, true, true>(p, st) : launch_one<v, DIST, false, true>(p, st); \
    return count_work ? launch_one<v, DIST, true, false>(p, st) : launch_one<v, DIST, false, false>(p, st);         \
  }
  VPET_LP_LIST(X)
#undef X
  return cudaErrorInvalidValue;
}

}  // namespace scan
}  // namespace vpet
