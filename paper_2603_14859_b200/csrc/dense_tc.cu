// dense_tc.cu -- K6: the optional shared-bank tensor-core distance (ABC_FLAG_DENSE_TC).
//
// North star: "an optional shared-simulation-bank mode, where ||y-s||^2 is expanded and the y.s
// cross term becomes a voxels x draws x frames contraction on tensor cores, used only if it
// measurably beats the fused FP32 path".  Alg. 1 l.4-5 for every
// (voxel, draw) pair, without pruning:
//     D'_ji = Y2_j + S2_i - 2 G_ji,   a = fl(ws y), b = fl(ws s), ws = RN32(sqrt(w_f)),
//     Y2 = sum a^2, S2 = sum b^2 (FP32),  G = a.b on tcgen05 (kind::f16, BF16 x 3 split, FP32 acc):
//     a = a_hi + a_lo (+ r, |r| <= 2^-18 |a|),  G ~ a_hi.b_hi + a_hi.b_lo + a_lo.b_hi,
//     i.e. one K = 144 contraction of [a_hi | a_hi | a_lo] with [b_hi | b_lo | b_hi].
// The epilogue (tcgen05.ld from TMEM) forms D', keeps the K smallest (D', i) per voxel in the same
// 8-ary candidate heaps as K2 (two parts: the two column halves of each draw tile), and K3
// certifies them in FP64 with the dot-form error bound (api.cu dense_error_bound).
//
// Tiles: one CTA = 128 voxels (UMMA M = 128, one TMEM lane each) against draw tiles of 256
// (UMMA N = 256); two FP32 accumulators of 256 TMEM columns (512 allocated) so the MMA of tile t
// overlaps the epilogue of tile t - 1.  Operands are stored in HBM already in the no-swizzle
// K-major core-matrix layout (8 rows x 16 B), so one cp.async.bulk per tile lands them in shared
// memory exactly as the smem descriptors describe them.
#include <cuda_bf16.h>

#include <algorithm>

#include "common.cuh"
#include "scan_kernels.cuh"  // heap_push, mbarrier and bulk-copy helpers

namespace vpet {
namespace dense {

constexpr int LMAX = 48;        // frames (padded) per split
constexpr int KD = 3 * LMAX;    // 144: contraction length
constexpr int KC = KD / 8;      // 18 core-matrix columns
constexpr int BM = 128;         // voxels per CTA
constexpr int BN = 256;         // draws per tile
constexpr int NTH = 256;        // 8 warps: warp w reads TMEM lanes 32 (w % 4) .., column half w / 4
constexpr uint32_t A_BYTES = BM * KD * 2;
constexpr uint32_t B_BYTES = BN * KD * 2;
constexpr uint32_t CAND_BYTES = 8 * NTH * 8;  // 8 candidate slots per thread ([slot][thread])
constexpr uint32_t SMEM = A_BYTES + 2 * B_BYTES + CAND_BYTES + 64;
constexpr uint32_t TMEM_COLS = 512;

// element offset of (row, k) in a tile of R rows: core matrix (row / 8, k / 8), K-chunk-major
__host__ __device__ inline uint32_t tile_off(uint32_t R, uint32_t row, uint32_t k) {
  return (((k >> 3) * (R >> 3) + (row >> 3)) * 8 + (row & 7)) * 8 + (k & 7);
}

// ---- operand preparation -------------------------------------------------------------------
// Bank side: row i -> [b_hi | b_lo | b_hi] (frames f < L, zero padded), S2[i] = sum b^2 (FP32).
// Rows i >= N (tail of the last tile) are zero with S2 = +inf, so D' = +inf is never kept.
__global__ void prep_bank_kernel(const float* __restrict__ bank, uint64_t N, uint64_t Npad, uint32_t L, uint32_t LS,
                                 const float* __restrict__ wsc, uint16_t* __restrict__ Bt, float* __restrict__ S2) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < Npad; i += uint64_t(gridDim.x) * blockDim.x) {
    const bool valid = i < N;
    __nv_bfloat16 hi[LMAX], lo[LMAX];
    float s2 = 0.0f;
#pragma unroll
    for (int f = 0; f < LMAX; ++f) {
      float b = (valid && f < int(L)) ? __fmul_rn(__ldg(wsc + f), __ldg(bank + i * LS + f)) : 0.0f;
      s2 = __fmaf_rn(b, b, s2);
      hi[f] = __float2bfloat16_rn(b);
      lo[f] = __float2bfloat16_rn(__fsub_rn(b, __bfloat162float(hi[f])));
    }
    S2[i] = valid ? s2 : __int_as_float(0x7f800000);
    uint16_t* tile = Bt + (i / BN) * (size_t(BN) * KD);
    const uint32_t r = uint32_t(i % BN);
#pragma unroll
    for (int c = 0; c < KC; ++c) {
      __align__(16) __nv_bfloat16 v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int k = c * 8 + e;
        v[e] = k < LMAX ? hi[k] : (k < 2 * LMAX ? lo[k - LMAX] : hi[k - 2 * LMAX]);
      }
      *reinterpret_cast<uint4*>(tile + tile_off(BN, r, c * 8)) = *reinterpret_cast<const uint4*>(v);
    }
  }
}

// Voxel side: slot j -> [a_hi | a_hi | a_lo], Y2[j] = sum a^2 (FP32).
__global__ void prep_voxel_kernel(const float* __restrict__ tacs, uint64_t J, uint64_t Jpad, uint32_t L,
                                  const float* __restrict__ wsc, uint16_t* __restrict__ At, float* __restrict__ Y2) {
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < Jpad; j += uint64_t(gridDim.x) * blockDim.x) {
    const bool valid = j < J;
    __nv_bfloat16 hi[LMAX], lo[LMAX];
    float y2 = 0.0f;
#pragma unroll
    for (int f = 0; f < LMAX; ++f) {
      float a = (valid && f < int(L)) ? __fmul_rn(__ldg(wsc + f), __ldg(tacs + j * L + f)) : 0.0f;
      y2 = __fmaf_rn(a, a, y2);
      hi[f] = __float2bfloat16_rn(a);
      lo[f] = __float2bfloat16_rn(__fsub_rn(a, __bfloat162float(hi[f])));
    }
    Y2[j] = y2;
    uint16_t* tile = At + (j / BM) * (size_t(BM) * KD);
    const uint32_t r = uint32_t(j % BM);
#pragma unroll
    for (int c = 0; c < KC; ++c) {
      __align__(16) __nv_bfloat16 v[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int k = c * 8 + e;
        v[e] = k < 2 * LMAX ? hi[k % LMAX] : lo[k - 2 * LMAX];
      }
      *reinterpret_cast<uint4*>(tile + tile_off(BM, r, c * 8)) = *reinterpret_cast<const uint4*>(v);
    }
  }
}

// ---- tcgen05 helpers ---------------------------------------------------------------------------
// Shared-memory matrix descriptor, no swizzle, K-major: LBO = byte stride between the two K core
// matrices of one MMA (K = 16), SBO = byte stride between 8-row groups; version 1 (sm_100).
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3fffu);
  d |= uint64_t((lbo >> 4) & 0x3fffu) << 16;
  d |= uint64_t((sbo >> 4) & 0x3fffu) << 32;
  d |= uint64_t(1) << 46;  // version (Blackwell)
  return d;                // base offset 0, legacy LBO mode, layout SWIZZLE_NONE (0)
}
// Instruction descriptor: D = F32, A = B = BF16, both K-major, N = 256, M = 128.
constexpr uint32_t kIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(kIdesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   scan::smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---- main kernel -------------------------------------------------------------------------------
__global__ void __launch_bounds__(NTH, 1) dense_tc_kernel(const DenseParams p) {
  if (p.bad && *p.bad) return;  // non-finite TACs: the call fails with ABC_E_ARG
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* sA = smem;
  unsigned char* sB = smem + A_BYTES;  // [2][B_BYTES]
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + A_BYTES + 2 * B_BYTES);  // barA, full[2], done[2]
  uint64_t* barA = bars;
  uint64_t* full = bars + 1;
  uint64_t* done = bars + 3;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(bars + 5);
  unsigned long long* sbuf = reinterpret_cast<unsigned long long*>(smem + A_BYTES + 2 * B_BYTES + 64);

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int q = wid & 3, half = wid >> 2;
  const uint64_t vb = blockIdx.x;
  const uint64_t ntile = p.ntile;

  if (tid == 0) {
    scan::mbar_init(barA, 1);
    for (int s = 0; s < 2; ++s) {
      scan::mbar_init(&full[s], 1);
      scan::mbar_init(&done[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (wid == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(scan::smem_u32(s_tmem)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *s_tmem;

  auto issue_b = [&](uint64_t t, int s) {
    scan::mbar_expect_tx(&full[s], B_BYTES);
    scan::bulk_g2s(sB + size_t(s) * B_BYTES, p.Bt + t * (size_t(BN) * KD), B_BYTES, &full[s]);
  };
  if (tid == 0) {
    scan::mbar_expect_tx(barA, A_BYTES);
    scan::bulk_g2s(sA, p.At + vb * (size_t(BM) * KD), A_BYTES, barA);
    issue_b(0, 0);
    if (ntile > 1) issue_b(1, 1);
  }

  // this thread's voxel (TMEM lane 32 q + lane) and heap part (column half)
  const uint64_t v = vb * BM + uint64_t(q) * 32 + lane;
  const bool valid = v < p.J;
  const float INF = __int_as_float(0x7f800000);
  const float y2 = valid ? p.Y2[v] : 0.0f;
  float tau = valid ? INF : -INF, taup = INF;
  uint32_t cnt = 0;
  unsigned long long* hb = p.heap + (v * 2 + uint64_t(half)) * heap_stride(p.K);

  const uint32_t a_base = scan::smem_u32(sA), b_base = scan::smem_u32(sB);
  for (uint64_t t = 0; t <= ntile; ++t) {
    if (tid == 0 && t < ntile) {  // MMA of tile t into accumulator t % 2
      const int s = int(t & 1);
      if (t == 0) scan::mbar_wait(barA, 0);
      scan::mbar_wait(&full[s], uint32_t(t >> 1) & 1u);
      tc_fence_after();
#pragma unroll
      for (int k = 0; k < KD / 16; ++k) {
        const uint64_t da = smem_desc(a_base + uint32_t(k) * 2u * (BM * 16u), BM * 16u, 128u);
        const uint64_t db = smem_desc(b_base + uint32_t(s) * B_BYTES + uint32_t(k) * 2u * (BN * 16u), BN * 16u, 128u);
        mma_bf16(tbase + uint32_t(s) * BN, da, db, k > 0 ? 1u : 0u);
      }
      mma_commit(&done[s]);
    }
    if (t >= 1) {  // epilogue of tile u = t - 1
      const uint64_t u = t - 1;
      const int s = int(u & 1);
      scan::mbar_wait(&done[s], uint32_t(u >> 1) & 1u);
      tc_fence_after();
      if (tid == 0 && u + 2 < ntile) {  // the MMA has consumed stage s: refill it with tile u + 2
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue_b(u + 2, s);
      }
      if (valid && p.tau_glob) tau = fminf(tau, __uint_as_float(__ldcg(p.tau_glob + v)));
      const uint64_t i0 = u * BN + uint64_t(half) * (BN / 2);
#pragma unroll 1
      for (int c = 0; c < BN / 2 / 32; ++c) {
        uint32_t g[32];
        __syncwarp();  // tcgen05.ld is warp-collective: reconverge after the heap pushes
        tmem_ld32(tbase + (uint32_t(q * 32) << 16) + uint32_t(s) * BN + uint32_t(half) * (BN / 2) + uint32_t(c) * 32u,
                  g);
        const float4* s2p = reinterpret_cast<const float4*>(p.S2 + i0 + uint64_t(c) * 32);
        float4 s4[8];
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) s4[j4] = __ldg(s2p + j4);
        // D' = fl(fl(Y2 + S2) - 2 G) (clamped at 0 below), in place of G
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const float s2v[4] = {s4[j4].x, s4[j4].y, s4[j4].z, s4[j4].w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            g[j4 * 4 + e] = __float_as_uint(__fmaf_rn(-2.0f, __uint_as_float(g[j4 * 4 + e]), __fadd_rn(y2, s2v[e])));
        }
        // fast path: one vote per 8 columns on the minimum; most groups hold no candidate
#pragma unroll
        for (int grp = 0; grp < 4; ++grp) {
          float m = __uint_as_float(g[grp * 8]);
#pragma unroll
          for (int e = 1; e < 8; ++e) m = fminf(m, __uint_as_float(g[grp * 8 + e]));
          if (!__any_sync(0xffffffffu, fmaxf(m, 0.0f) < tau)) continue;
          // slow path: compact this lane's candidates into its shared-memory slots, then push them
          // with the warp in lockstep (rounds = the largest per-lane count, not the sum)
          uint32_t nb = 0;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float D = fmaxf(__uint_as_float(g[grp * 8 + e]), 0.0f);
            if (D < tau) {
              const uint32_t i = uint32_t(i0 + uint64_t(c) * 32 + uint64_t(grp * 8 + e));
              sbuf[nb * NTH + tid] = (static_cast<unsigned long long>(__float_as_uint(D)) << 32) | i;
              ++nb;
            }
          }
          const uint32_t rounds = __reduce_max_sync(0xffffffffu, nb);
          for (uint32_t k = 0; k < rounds; ++k) {
            if (k < nb) {
              const unsigned long long key = sbuf[k * NTH + tid];
              if (__uint_as_float(uint32_t(key >> 32)) < tau) {
                const uint2 st = scan::heap_push(hb, p.K, cnt, key);
                cnt = st.x;
                taup = __uint_as_float(st.y);
                if (p.tau_glob && st.y != 0x7f800000u) atomicMin(p.tau_glob + v, st.y);
                tau = fminf(tau, taup);
              }
            }
          }
        }
      }
      tc_fence_before();
    }
    __syncthreads();  // accumulator u % 2 is free for the MMA of tile u + 2
  }
  if (valid) p.heap_cnt[v * 2 + uint64_t(half)] = cnt;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (wid == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(TMEM_COLS));
}

}  // namespace dense

uint64_t dense_bank_bytes(uint64_t N) {
  const uint64_t Npad = (N + dense::BN - 1) / dense::BN * dense::BN;
  return Npad * dense::KD * 2 + Npad * 4;
}
uint64_t dense_voxel_bytes(uint64_t J) {
  const uint64_t Jpad = (J + dense::BM - 1) / dense::BM * dense::BM;
  return Jpad * dense::KD * 2 + Jpad * 4;
}

cudaError_t launch_dense(DenseParams p, const float* bank, uint32_t LS, const float* tacs, const float* wsc,
                         cudaStream_t st, uint32_t* launches) {
  using namespace dense;
  if (p.L > uint32_t(LMAX)) return cudaErrorInvalidValue;
  const uint64_t Npad = (p.N + BN - 1) / BN * BN;
  const uint64_t Jpad = (p.J + BM - 1) / BM * BM;
  p.ntile = Npad / BN;
  prep_bank_kernel<<<unsigned(std::min<uint64_t>((Npad + 255) / 256, 148 * 16)), 256, 0, st>>>(
      bank, p.N, Npad, p.L, LS, wsc, p.Bt, p.S2);
  prep_voxel_kernel<<<unsigned(std::min<uint64_t>((Jpad + 255) / 256, 148 * 16)), 256, 0, st>>>(
      tacs, p.J, Jpad, p.L, wsc, p.At, p.Y2);
  {
    cudaError_t e = ensure_smem_attr((const void*)dense_tc_kernel, SMEM);
    if (e != cudaSuccess) return e;
  }
  dense_tc_kernel<<<unsigned(Jpad / BM), NTH, SMEM, st>>>(p);
  if (launches) *launches += 3;
  return cudaGetLastError();
}

}  // namespace vpet
