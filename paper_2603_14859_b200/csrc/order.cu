// order.cu -- K1b/K1c: the scan-order copy of the bank and its bounding-box hierarchy.
//
// The FP32 pass visits frames in descending-spread order (frame_var/frame_perm) and draws in a
// locality-preserving order: each draw's prescaled curve is projected on the top NPC principal
// axes of the bank (covariance + power iteration), quantised on an isotropic grid and sorted by
// its Morton code.  Consecutive draws are then close in TAC space, so the per-frame bounding
// boxes of tiles of T draws (and of super-tiles of ST tiles) are tight and give exact lower
// bounds on the FP32 discrepancy of every draw inside them (scan_tree.cu).  The order only
// changes which draws are looked at first; selection is by (D, original index) keys.

#include <cstdlib>

#include "common.cuh"

namespace vpet {
namespace {

// ---- per-frame mean and spread of the prescaled bank over a strided sample ----
__global__ void __launch_bounds__(1024) frame_stats_kernel(const OrderParams p) {
  uint32_t f = blockIdx.x;
  uint64_t stride = p.N > 65536 ? p.N / 65536 : 1;
  uint64_t ns = (p.N + stride - 1) / stride;
  double s1 = 0.0, s2 = 0.0;
  double sc = p.wsc[f];
  for (uint64_t j = threadIdx.x; j < ns; j += blockDim.x) {
    double x = sc * double(p.bank[j * stride * p.LS + f]);
    s1 += x;
    s2 += x * x;
  }
  for (int o = 16; o > 0; o >>= 1) {
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
    s2 += __shfl_xor_sync(0xffffffffu, s2, o);
  }
  __shared__ double r1[32], r2[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) {
    r1[wid] = s1;
    r2[wid] = s2;
  }
  __syncthreads();
  if (wid == 0) {
    const int nw = int(blockDim.x >> 5);
    s1 = lane < nw ? r1[lane] : 0.0;
    s2 = lane < nw ? r2[lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) {
      double m = s1 / double(ns);
      p.var[f] = fmax(s2 / double(ns) - m * m, 0.0);
      p.mean[f] = m;
    }
  }
}

// ---- descending-spread permutation (stable), padded with -1: thread f places frame f at its
// rank (frames of larger spread, or of equal spread and lower index, go first) ----
__global__ void __launch_bounds__(kMaxLP) frame_perm_kernel(const OrderParams p) {
  __shared__ int order[kMaxLP];
  const uint32_t f = threadIdx.x;
  if (f < p.L) {
    uint32_t rank = f;
    if (p.reorder) {
      const double vf = p.var[f];
      rank = 0;
      for (uint32_t g = 0; g < p.L; ++g) {
        const double vg = p.var[g];
        rank += (vg > vf || (vg == vf && g < f)) ? 1u : 0u;
      }
    }
    order[rank] = int(f);
  }
  __syncthreads();
  for (uint32_t k = f; k < p.LP; k += blockDim.x) {
    int src = k < p.L ? order[k] : -1;
    p.perm[k] = src;
    p.wsp[k] = src >= 0 ? p.wsc[src] : 0.0f;
  }
  if (f == 0 && p.tree && p.pminmax)  // projection range accumulators (order-preserving uint of float)
    for (int c = 0; c < kNPC; ++c) {
      p.pminmax[2 * c] = 0xffffffffu;
      p.pminmax[2 * c + 1] = 0u;
    }
}

// ---- covariance of the prescaled bank (scan order), one block per (row, col) pair ----
__global__ void __launch_bounds__(256) cov_kernel(const OrderParams p) {
  uint32_t a = blockIdx.x, b = blockIdx.y;
  if (b < a) return;
  int fa = p.perm[a], fb = p.perm[b];
  uint64_t stride = p.N > 16384 ? p.N / 16384 : 1;
  uint64_t ns = (p.N + stride - 1) / stride;
  double s = 0.0;
  if (fa >= 0 && fb >= 0) {
    double ma = p.mean[fa], mb = p.mean[fb], ca = p.wsc[fa], cb = p.wsc[fb];
    for (uint64_t j = threadIdx.x; j < ns; j += blockDim.x) {
      const float* row = p.bank + j * stride * p.LS;
      s += (ca * double(row[fa]) - ma) * (cb * double(row[fb]) - mb);
    }
  }
  __shared__ double r[256];
  r[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) r[threadIdx.x] += r[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double c = r[0] / double(ns);
    p.cov[a * p.LP + b] = c;
    p.cov[b * p.LP + a] = c;
  }
}

// ---- top-NPC eigenvectors by power iteration with deflation (one block) ----
// ---- first kNPC principal axes of the covariance: power iteration with deflation, one warp;
// stops when the direction changes by < 1e-9 (eigen-gaps of a bank are large) or after 100 steps ----
__global__ void __launch_bounds__(32) pca_kernel(const OrderParams p) {
  extern __shared__ double C[];  // [LP][LP] working copy (p.cov stays intact for rot_kernel)
  __shared__ double v[kMaxLP], w[kMaxLP];
  const uint32_t LP = p.LP;
  const int lane = threadIdx.x;
  double* Cm = C;
  for (uint32_t e = lane; e < LP * LP; e += 32) C[e] = p.cov[e];
  __syncwarp();
  auto wsum = [](double x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
  };
  for (int c = 0; c < kNPC; ++c) {
    for (uint32_t k = lane; k < LP; k += 32) v[k] = 1.0 + 0.001 * double((k * 7919u + c * 104729u) % 97u);
    __syncwarp();
    for (int it = 0; it < 100; ++it) {
      double ss = 0.0;
      for (uint32_t k = lane; k < LP; k += 32) {
        double s = 0.0;
        for (uint32_t g = 0; g < LP; ++g) s += Cm[k * LP + g] * v[g];
        w[k] = s;
        ss += s * s;
      }
      ss = wsum(ss);
      const double nrm = ss > 0.0 ? 1.0 / sqrt(ss) : 0.0;
      double dd = 0.0;
      __syncwarp();
      for (uint32_t k = lane; k < LP; k += 32) {
        const double nv = w[k] * nrm;
        dd += (nv - v[k]) * (nv - v[k]);
        v[k] = nv;
      }
      dd = wsum(dd);
      __syncwarp();
      if (dd < 1e-18) break;
    }
    // eigenvalue and deflation
    double lam = 0.0;
    for (uint32_t k = lane; k < LP; k += 32) {
      double s = 0.0;
      for (uint32_t g = 0; g < LP; ++g) s += Cm[k * LP + g] * v[g];
      lam += v[k] * s;
    }
    lam = wsum(lam);
    __syncwarp();
    for (uint32_t e = lane; e < LP * LP; e += 32) Cm[e] -= lam * v[e / LP] * v[e % LP];
    for (uint32_t k = lane; k < LP; k += 32) p.pcs[c * LP + k] = float(v[k]);
    __syncwarp();
  }
}

// ---- rotated scan basis (WL2, tree mode, LP <= kRotMaxLP): eigenvectors of the covariance of
// the prescaled bank by cyclic Jacobi (round-robin parallel ordering: LP / 2 disjoint rotations
// per round), one block; columns in descending eigenvalue order.  Out: rotq[f][k] = Q[a][k] * cw[f]
// for the real frames f = perm[a].  The bank's curves span few directions (2TCM: ~4 carry all
// the variance), so in this basis a tile's box is thin in every coordinate.
// Exactness does not rest on Q being eigenvectors, only on its orthogonality, which is checked:
// LP * max|Q^T Q - I| > kRotEps falls back to Q = I. ----
constexpr uint32_t kRotMaxLP = 96;  // shared memory: rot_kernel 2 LP^2 doubles, permute LP L doubles + rows
__global__ void __launch_bounds__(256) rot_kernel(const OrderParams p) {
  extern __shared__ double rsm[];
  const uint32_t n = p.LP;  // a multiple of 4
  double* A = rsm;          // [n][n]
  double* V = rsm + n * n;  // [n][n]
  __shared__ double cs_c[kRotMaxLP / 2], cs_s[kRotMaxLP / 2];
  __shared__ int pp[kRotMaxLP / 2], pq[kRotMaxLP / 2];
  __shared__ double red[2][8];
  __shared__ int rank[kRotMaxLP];
  __shared__ int stop;
  const uint32_t tid = threadIdx.x, nt = blockDim.x;
  for (uint32_t e = tid; e < n * n; e += nt) {
    A[e] = p.cov[e];
    V[e] = (e / n == e % n) ? 1.0 : 0.0;
  }
  __syncthreads();
  auto block_sum2 = [&](double x, double y, double& sx, double& sy) {
    for (int o = 16; o > 0; o >>= 1) {
      x += __shfl_xor_sync(0xffffffffu, x, o);
      y += __shfl_xor_sync(0xffffffffu, y, o);
    }
    if ((tid & 31) == 0) {
      red[0][tid >> 5] = x;
      red[1][tid >> 5] = y;
    }
    __syncthreads();
    sx = 0.0;
    sy = 0.0;
    for (uint32_t w = 0; w < nt / 32; ++w) {
      sx += red[0][w];
      sy += red[1][w];
    }
    __syncthreads();
  };
  for (int sweep = 0; sweep < 12; ++sweep) {  // a good basis suffices: exactness needs only orthogonality
    double off = 0.0, dia = 0.0;
    for (uint32_t e = tid; e < n * n; e += nt) {
      const double a = A[e];
      if (e / n == e % n) dia += a * a;
      else off += a * a;
    }
    block_sum2(off, dia, off, dia);
    if (off <= 1e-20 * dia || off == 0.0) break;
    for (uint32_t r = 0; r + 1 < n; ++r) {
      if (tid < n / 2) {
        // round-robin: position 0 holds index 0, position i >= 1 holds ((i - 1 + r) mod (n - 1)) + 1
        auto at = [&](uint32_t pos) { return pos == 0 ? 0u : ((pos - 1 + r) % (n - 1)) + 1; };
        uint32_t a = at(tid), b = at(n - 1 - tid);
        if (a > b) { const uint32_t t = a; a = b; b = t; }
        const double apq = A[a * n + b];
        double c = 1.0, sn = 0.0;
        if (fabs(apq) > 1e-300) {
          const double th = (A[b * n + b] - A[a * n + a]) / (2.0 * apq);
          const double t = fabs(th) > 1e150 ? 0.5 / th : copysign(1.0, th) / (fabs(th) + sqrt(th * th + 1.0));
          c = 1.0 / sqrt(t * t + 1.0);
          sn = t * c;
        }
        cs_c[tid] = c;
        cs_s[tid] = sn;
        pp[tid] = int(a);
        pq[tid] = int(b);
      }
      __syncthreads();
      for (uint32_t e = tid; e < (n / 2) * n; e += nt) {  // columns of A and V
        const uint32_t k = e / n, i = e % n;
        const uint32_t a = uint32_t(pp[k]), b = uint32_t(pq[k]);
        const double c = cs_c[k], sn = cs_s[k];
        const double x = A[i * n + a], y = A[i * n + b];
        A[i * n + a] = c * x - sn * y;
        A[i * n + b] = sn * x + c * y;
        const double u = V[i * n + a], v = V[i * n + b];
        V[i * n + a] = c * u - sn * v;
        V[i * n + b] = sn * u + c * v;
      }
      __syncthreads();
      for (uint32_t e = tid; e < (n / 2) * n; e += nt) {  // rows of A
        const uint32_t k = e / n, j = e % n;
        const uint32_t a = uint32_t(pp[k]), b = uint32_t(pq[k]);
        const double c = cs_c[k], sn = cs_s[k];
        const double x = A[a * n + j], y = A[b * n + j];
        A[a * n + j] = c * x - sn * y;
        A[b * n + j] = sn * x + c * y;
      }
      __syncthreads();
    }
  }
  // descending eigenvalue order (stable)
  if (tid < n) {
    const double lk = A[tid * n + tid];
    int rk = 0;
    for (uint32_t j = 0; j < n; ++j) {
      const double lj = A[j * n + j];
      rk += (lj > lk || (lj == lk && j < tid)) ? 1 : 0;
    }
    rank[tid] = rk;
  }
  if (tid == 0) stop = 0;
  __syncthreads();
  // orthogonality defect of V (columns permute without changing it)
  double md = 0.0;
  for (uint32_t e = tid; e < n * n; e += nt) {
    const uint32_t i = e / n, j = e % n;
    double d = 0.0;
    for (uint32_t a = 0; a < n; ++a) d = fma(V[a * n + i], V[a * n + j], d);
    md = fmax(md, fabs(d - (i == j ? 1.0 : 0.0)));
  }
  for (int o = 16; o > 0; o >>= 1) md = fmax(md, __shfl_xor_sync(0xffffffffu, md, o));
  if ((tid & 31) == 0 && double(n) * md + 1e-14 > kRotEps) atomicExch(&stop, 1);
  __syncthreads();
  // a failed check (never seen) falls back to Q = I: exactly orthogonal, the frame basis
  const bool ok = stop == 0;
  for (uint32_t e = tid; e < p.L * n; e += nt) {
    const uint32_t a = e / n, k = e % n;  // scan position a (a real frame: a < L), eigen-column k
    const int f = p.perm[a];
    const double q = ok ? V[a * n + k] : (a == k ? 1.0 : 0.0);
    if (f >= 0) p.rotq[uint32_t(f) * n + (ok ? uint32_t(rank[k]) : k)] = q * p.cw[f];
  }
}

__device__ __forceinline__ unsigned int f2ord(float x) {
  unsigned int u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned int u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// Projection of bank rows on the principal axes, in acquisition frame order (float4 row loads):
// pr_c = sum_f bank[i][f] coef[c][f] - off[c], coef[c][perm[k]] = wsp[k] pc[c][k],
// off[c] = sum_k mean[perm[k]] pc[c][k].  (A heuristic ordering key: exactness does not depend on it.)
struct ProjSmem {
  float coef[kNPC][kMaxLP];
  float off[kNPC];
};

__device__ void proj_setup(const OrderParams& p, ProjSmem& s) {
  for (uint32_t e = threadIdx.x; e < kNPC * kMaxLP; e += blockDim.x) (&s.coef[0][0])[e] = 0.0f;
  __syncthreads();
  for (uint32_t k = threadIdx.x; k < p.LP; k += blockDim.x) {
    const int src = p.perm[k];
    if (src >= 0)
      for (int c = 0; c < kNPC; ++c) s.coef[c][src] = p.wsp[k] * p.pcs[c * p.LP + k];
  }
  if (threadIdx.x < kNPC) {
    float o = 0.0f;
    for (uint32_t k = 0; k < p.LP; ++k)
      if (p.perm[k] >= 0) o = fmaf(float(p.mean[p.perm[k]]), p.pcs[threadIdx.x * p.LP + k], o);
    s.off[threadIdx.x] = o;
  }
  __syncthreads();
}

__device__ __forceinline__ void project(const OrderParams& p, const ProjSmem& s, uint64_t i, float pr[kNPC]) {
  const float4* row = reinterpret_cast<const float4*>(p.bank + i * p.LS);
#pragma unroll
  for (int c = 0; c < kNPC; ++c) pr[c] = -s.off[c];
  for (uint32_t q = 0; q < p.LS / 4; ++q) {
    const float4 x = __ldg(row + q);
#pragma unroll
    for (int c = 0; c < kNPC; ++c) {
      const float* cf = s.coef[c] + 4 * q;
      pr[c] = fmaf(x.x, cf[0], pr[c]);
      pr[c] = fmaf(x.y, cf[1], pr[c]);
      pr[c] = fmaf(x.z, cf[2], pr[c]);
      pr[c] = fmaf(x.w, cf[3], pr[c]);
    }
  }
}

__global__ void __launch_bounds__(256) proj_minmax_kernel(const OrderParams p) {
  __shared__ ProjSmem sm;
  proj_setup(p, sm);
  float lo[kNPC], hi[kNPC];
#pragma unroll
  for (int c = 0; c < kNPC; ++c) { lo[c] = 3.0e38f; hi[c] = -3.0e38f; }
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < p.N; i += uint64_t(gridDim.x) * blockDim.x) {
    float pr[kNPC];
    project(p, sm, i, pr);
#pragma unroll
    for (int c = 0; c < kNPC; ++c) { lo[c] = fminf(lo[c], pr[c]); hi[c] = fmaxf(hi[c], pr[c]); }
    // kept for key_kernel (one pass over the bank instead of two)
    if constexpr (kNPC == 4) reinterpret_cast<float4*>(p.proj)[i] = make_float4(pr[0], pr[1], pr[2], pr[3]);
    else
      for (int c = 0; c < kNPC; ++c) p.proj[i * kNPC + c] = pr[c];
  }
#pragma unroll
  for (int c = 0; c < kNPC; ++c) {
    for (int o = 16; o > 0; o >>= 1) {
      lo[c] = fminf(lo[c], __shfl_xor_sync(0xffffffffu, lo[c], o));
      hi[c] = fmaxf(hi[c], __shfl_xor_sync(0xffffffffu, hi[c], o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(p.pminmax + 2 * c, f2ord(lo[c]));
      atomicMax(p.pminmax + 2 * c + 1, f2ord(hi[c]));
    }
  }
}

// bank Morton grid: scale of principal axes 2..4 relative to the isotropic grid, and whether the
// first axis takes the most significant bit of each 4-bit group
#ifndef VPET_BANKS
#define VPET_BANKS 1.0f
#endif
#ifndef VPET_MBITS
#define VPET_MBITS 16  // Morton bits per principal axis of the bank order
#endif
constexpr int kMBits = (VPET_MBITS * kNPC <= 64) ? VPET_MBITS : 64 / kNPC;
// insert kNPC - 1 zero bits between the low kMBits bits of x (kNPC-dimensional Morton)
__device__ __forceinline__ unsigned long long spread_npc(unsigned long long x) {
  unsigned long long r = 0;
#pragma unroll
  for (int b = 0; b < kMBits; ++b) r |= ((x >> b) & 1ull) << (kNPC * b);
  return r;
}
#ifndef VPET_BANK_MSB
#define VPET_BANK_MSB 0
#endif
// Space-filling curve of the draw order: VPET_HILBERT = 1 Hilbert (12 % fewer executed frame updates
// than Morton on the TB slab set, scan -2 %), 0 Morton (Z-order).
// A Hilbert curve has no long jumps at cell boundaries, so a run of consecutive keys (a tile of 32
// draws, a warp of 64 voxels) covers a more compact region: tighter tile boxes, more similar
// voxels per warp (the order is free for exactness).
#ifndef VPET_HILBERT
#define VPET_HILBERT 1
#endif
#ifndef VPET_HILBERT_VOX
#define VPET_HILBERT_VOX 0  // the voxel order stays Morton: the scan's queue takes voxel tiles from both
                            // ends of the PC1-major Morton range first (the long items); a Hilbert voxel
                            // order cut 3 % more work but lost that longest-first schedule (+30 % scan)
#endif
// Skilling's transpose form of the n-dimensional Hilbert index (J. Skilling, "Programming the
// Hilbert curve", AIP Conf. Proc. 707, 2004): coordinates X[n] of b bits -> the transposed index,
// bit-interleaved with X[0] the most significant bit of each group of n.
template <int n, int b>
__device__ __forceinline__ unsigned long long hilbert_key(uint32_t (&X)[n]) {
  const uint32_t M = 1u << (b - 1);
  for (uint32_t Q = M; Q > 1; Q >>= 1) {  // inverse undo
    const uint32_t P = Q - 1;
#pragma unroll
    for (int i = 0; i < n; ++i) {
      if (X[i] & Q) {
        X[0] ^= P;
      } else {
        const uint32_t t = (X[0] ^ X[i]) & P;
        X[0] ^= t;
        X[i] ^= t;
      }
    }
  }
#pragma unroll
  for (int i = 1; i < n; ++i) X[i] ^= X[i - 1];  // Gray encode
  uint32_t t = 0;
  for (uint32_t Q = M; Q > 1; Q >>= 1)
    if (X[n - 1] & Q) t ^= Q - 1;
#pragma unroll
  for (int i = 0; i < n; ++i) X[i] ^= t;
  unsigned long long key = 0;
  for (int bit = b - 1; bit >= 0; --bit)
#pragma unroll
    for (int i = 0; i < n; ++i) key = (key << 1) | ((X[i] >> bit) & 1u);
  return key;
}
__device__ __forceinline__ unsigned long long spread4(unsigned long long x) {
  // insert 3 zero bits between the low 16 bits of x (4-D Morton)
  unsigned long long r = 0;
#pragma unroll
  for (int b = 0; b < 16; ++b) r |= ((x >> b) & 1ull) << (4 * b);
  return r;
}

__global__ void __launch_bounds__(256) key_kernel(const OrderParams p) {
  __shared__ ProjSmem sm;
  __shared__ float sm_lo[kNPC], sm_scale;
  proj_setup(p, sm);
  if (threadIdx.x == 0) {
    float rng = 0.0f;
    for (int c = 0; c < kNPC; ++c) {
      sm_lo[c] = ord2f(p.pminmax[2 * c]);
      rng = fmaxf(rng, ord2f(p.pminmax[2 * c + 1]) - sm_lo[c]);
    }
    sm_scale = rng > 0.0f ? float((1u << kMBits) - 1u) / rng : 0.0f;  // isotropic grid, kMBits on the widest axis
  }
  __syncthreads();
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < p.N; i += uint64_t(gridDim.x) * blockDim.x) {
    float pr[kNPC];
    if constexpr (kNPC == 4) {
      const float4 v = reinterpret_cast<const float4*>(p.proj)[i];
      pr[0] = v.x; pr[1] = v.y; pr[2] = v.z; pr[3] = v.w;
    } else {
      for (int c = 0; c < kNPC; ++c) pr[c] = p.proj[i * kNPC + c];
    }
    unsigned long long key = 0;
    uint32_t X[kNPC];
#pragma unroll
    for (int c = 0; c < kNPC; ++c) {
      const float sc = c == 0 ? sm_scale : sm_scale * VPET_BANKS;
      float q = fminf(fmaxf((pr[c] - sm_lo[c]) * sc, 0.0f), float((1u << kMBits) - 1u));
      X[c] = uint32_t(q);
      if (!VPET_HILBERT) key |= spread_npc((unsigned long long)q) << (VPET_BANK_MSB ? kNPC - 1 - c : c);
    }
    if (VPET_HILBERT) key = hilbert_key<kNPC, kMBits>(X);
    p.keys[i] = key;
    p.vals[i] = uint32_t(i);
  }
}

// Rotated coordinates of one curve x (L floats, shared memory) into out (LP floats): RN32 of the FP64
// sums over the frames, in blocks of KB coordinates (one pass over x per block), negated if NEG.
template <int KB, bool NEG>
__device__ __forceinline__ uint32_t rotate_blocks(const float* x, const double* q, uint32_t L, uint32_t LP, uint32_t k0,
                                                  float* out) {
  for (; k0 + KB <= LP; k0 += KB) {
    double acc[KB];
#pragma unroll
    for (int u = 0; u < KB; ++u) acc[u] = 0.0;
    for (uint32_t f = 0; f < L; ++f) {
      const double xf = double(x[f]);
      const double2* qf = reinterpret_cast<const double2*>(q + f * LP + k0);
#pragma unroll
      for (int u = 0; u < KB / 2; ++u) {
        const double2 c = qf[u];
        acc[2 * u] = fma(c.x, xf, acc[2 * u]);
        acc[2 * u + 1] = fma(c.y, xf, acc[2 * u + 1]);
      }
    }
#pragma unroll
    for (int u = 0; u < KB; ++u) out[k0 + u] = NEG ? -__double2float_rn(acc[u]) : __double2float_rn(acc[u]);
  }
  return k0;
}
template <bool NEG>
__device__ __forceinline__ void rotate_curve(const float* x, const double* q, uint32_t L, uint32_t LP, float* out) {
  uint32_t k0 = rotate_blocks<12, NEG>(x, q, L, LP, 0, out);
  rotate_blocks<4, NEG>(x, q, L, LP, k0, out);
}

// ---- scan-order copy fused with the tile bounds, one warp per tile of kTile rows:
// bankp[j][k] = -(wsp[k] * bank[order[j]][perm[k]]), idxmap[j] = order[j], and (tree mode)
// tbounds[t] = per-frame [min, max] of the tile's bankp rows.  Raw rows are gathered with
// coalesced 16-B loads into shared memory, then written out frame-contiguous. ----
constexpr int kPermWarps = 4;
__global__ void __launch_bounds__(32 * kPermWarps) permute_kernel(const OrderParams p) {
  extern __shared__ double psm_d[];  // rotated basis: [L][LP] rotq; then [kPermWarps][kTile][max(LS, LP) + 1] floats
  __shared__ int sperm[kMaxLP];
  __shared__ float swsp[kMaxLP];
  __shared__ uint32_t sidx[kPermWarps][kTile];
  for (uint32_t k = threadIdx.x; k < p.LP; k += blockDim.x) {
    sperm[k] = p.perm[k];
    swsp[k] = p.wsp[k];
  }
  const double* srot = psm_d;
  if (p.rotq)
    for (uint32_t e = threadIdx.x; e < p.L * p.LP; e += blockDim.x) psm_d[e] = p.rotq[e];
  float* psm = reinterpret_cast<float*>(psm_d + (p.rotq ? p.L * p.LP : 0));
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint32_t LS = p.LS, Q = LS / 4, stride = (LS > p.LP ? LS : p.LP) + 1;
  float* rows = psm + size_t(wid) * kTile * stride * (p.rotq ? 2 : 1);
  const uint64_t ntile = (p.N + kTile - 1) / kTile;
  for (uint64_t t = uint64_t(blockIdx.x) * kPermWarps + wid; t < ntile; t += uint64_t(gridDim.x) * kPermWarps) {
    const uint64_t j0 = t * kTile;
    const uint32_t nr = uint32_t((p.N - j0) < uint64_t(kTile) ? (p.N - j0) : uint64_t(kTile));
    uint32_t myi = 0;
    if (uint32_t(lane) < nr) {
      myi = p.order ? p.order[j0 + lane] : uint32_t(j0 + lane);
      if (p.idxmap) p.idxmap[j0 + lane] = myi;
    }
    if (lane < kTile) sidx[wid][lane] = myi;
    __syncwarp();
    // gather: element e = (row e / Q, float4 e % Q); eight independent 16-B loads in flight per lane
    for (uint32_t e0 = lane; e0 < nr * Q; e0 += 32 * 8) {
      float4 x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t e = e0 + 32u * u;
        if (e < nr * Q)
          x[u] = __ldg(reinterpret_cast<const float4*>(p.bank + uint64_t(sidx[wid][e / Q]) * LS) + e % Q);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t e = e0 + 32u * u;
        if (e < nr * Q) {
          float* d = rows + (e / Q) * stride + 4 * (e % Q);
          d[0] = x[u].x; d[1] = x[u].y; d[2] = x[u].z; d[3] = x[u].w;
        }
      }
    }
    __syncwarp();
    const uint32_t QP = p.LP / 4;
    float4* dst = reinterpret_cast<float4*>(p.bankp + j0 * p.LP);
    if (p.rotq) {
      // rotated basis: lane r computes row r's LP coordinates, RN32 of FP64 sums over the frames,
      // into its own row of rows (overwritten in place after the whole row is read), negated
      float* orows = rows + kTile * stride;  // [kTile][stride] rotated rows of this warp
      if (uint32_t(lane) < nr) rotate_curve<true>(rows + lane * stride, srot, p.L, p.LP, orows + lane * stride);
      __syncwarp();
      for (uint32_t q = lane; q < nr * QP; q += 32) {
        const float* row = orows + (q / QP) * stride + 4 * (q % QP);
        dst[q] = make_float4(row[0], row[1], row[2], row[3]);
      }
      if (p.tree && p.tbounds)
        for (uint32_t k = lane; k < p.LP; k += 32) {
          float lo = 3.0e38f, hi = -3.0e38f;
          for (uint32_t r = 0; r < nr; ++r) {
            const float v = orows[r * stride + k];
            lo = fminf(lo, v);
            hi = fmaxf(hi, v);
          }
          p.tbounds[(t * 2 + 0) * p.LP + k] = lo;
          p.tbounds[(t * 2 + 1) * p.LP + k] = hi;
        }
      __syncwarp();
      continue;
    }
    // the tile's nr x LP block of bankp is contiguous (LP % 4 == 0): 16-B stores, lane q writes
    // frames 4(q % QP) .. +3 of row q / QP
    for (uint32_t q = lane; q < nr * QP; q += 32) {
      const float* row = rows + (q / QP) * stride;
      const uint32_t k = 4 * (q % QP);
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int src = sperm[k + u];
        v[u] = src >= 0 ? -__fmul_rn(swsp[k + u], row[src]) : 0.0f;
      }
      dst[q] = make_float4(v[0], v[1], v[2], v[3]);
    }
    if (p.tree && p.tbounds)
      for (uint32_t k = lane; k < p.LP; k += 32) {
        const int src = sperm[k];
        const float ws = swsp[k];
        float lo = 3.0e38f, hi = -3.0e38f;
        for (uint32_t r = 0; r < nr; ++r) {
          const float v = src >= 0 ? -__fmul_rn(ws, rows[r * stride + src]) : 0.0f;
          lo = fminf(lo, v);
          hi = fmaxf(hi, v);
        }
        p.tbounds[(t * 2 + 0) * p.LP + k] = lo;
        p.tbounds[(t * 2 + 1) * p.LP + k] = hi;
      }
    __syncwarp();
  }
}

__global__ void __launch_bounds__(128) super_bounds_kernel(const OrderParams p, uint64_t ntile) {
  uint64_t s = blockIdx.x;
  uint64_t t0 = s * kSuper;
  uint64_t t1 = t0 + kSuper < ntile ? t0 + kSuper : ntile;
  for (uint32_t k = threadIdx.x; k < p.LP; k += blockDim.x) {
    float lo = 3.0e38f, hi = -3.0e38f;
    for (uint64_t t = t0; t < t1; ++t) {
      lo = fminf(lo, p.tbounds[(t * 2 + 0) * p.LP + k]);
      hi = fmaxf(hi, p.tbounds[(t * 2 + 1) * p.LP + k]);
    }
    p.sbounds[(s * 2 + 0) * p.LP + k] = lo;
    p.sbounds[(s * 2 + 1) * p.LP + k] = hi;
  }
}

__global__ void __launch_bounds__(128) hyper_bounds_kernel(const OrderParams p, uint64_t nsup) {
  uint64_t h = blockIdx.x;
  uint64_t s0 = h * p.hs;
  uint64_t s1 = s0 + p.hs < nsup ? s0 + p.hs : nsup;
  for (uint32_t k = threadIdx.x; k < p.LP; k += blockDim.x) {
    float lo = 3.0e38f, hi = -3.0e38f;
    for (uint64_t s = s0; s < s1; ++s) {
      lo = fminf(lo, p.sbounds[(s * 2 + 0) * p.LP + k]);
      hi = fmaxf(hi, p.sbounds[(s * 2 + 1) * p.LP + k]);
    }
    p.hbounds[(h * 2 + 0) * p.LP + k] = lo;
    p.hbounds[(h * 2 + 1) * p.LP + k] = hi;
  }
}

// whole-bank box of the scan coordinates (rotated basis: the tail bound of each voxel), one block
__global__ void __launch_bounds__(128) global_box_kernel(const OrderParams p) {
  for (uint32_t k = threadIdx.x; k < p.LP; k += blockDim.x) {
    float lo = 3.0e38f, hi = -3.0e38f;
    for (uint64_t h = 0; h < p.nhyper; ++h) {
      lo = fminf(lo, p.hbounds[(h * 2 + 0) * p.LP + k]);
      hi = fmaxf(hi, p.hbounds[(h * 2 + 1) * p.LP + k]);
    }
    p.gbox[k] = lo;
    p.gbox[p.LP + k] = hi;
  }
}

// Voxel scan order.  VPET_VOXKEY = 1: first-principal-axis projection; D = 2 or 4: D-dimensional
// Morton code of the projection on the first D principal axes, on the bank's isotropic grid.
#ifndef VPET_VOXKEY
#define VPET_VOXKEY 4  // rotated scan: 4 axes on an isotropic grid (3 axes, 0.25 scale: +6 % scan)
#endif
#ifndef VPET_VOXS
#define VPET_VOXS 1.0f
#endif
#ifndef VPET_VOXS3
#define VPET_VOXS3 VPET_VOXS  // scale of the third and fourth axes
#endif
constexpr int kVoxDims = VPET_VOXKEY;
constexpr int kVoxAxisBits = kVoxDims == 1 ? 32 : (kVoxDims == 2 ? 16 : (kVoxDims == 3 ? 20 : 15));
constexpr int kVoxBits = kVoxDims * kVoxAxisBits;

__device__ __forceinline__ unsigned long long spread_d(unsigned long long x) {
  unsigned long long r = 0;
#pragma unroll
  for (int b = 0; b < kVoxAxisBits; ++b) r |= ((x >> b) & 1ull) << (kVoxDims * b);
  return r;
}

__global__ void __launch_bounds__(256) voxel_key_kernel(const VoxelOrderParams p) {
  __shared__ float sm_mu[kMaxLP], sm_wsp[kMaxLP], sm_pc[kNPC * kMaxLP];
  __shared__ int sm_perm[kMaxLP];
  __shared__ float sm_lo[kNPC], sm_scale;
  for (uint32_t k = threadIdx.x; k < p.LP; k += blockDim.x) {
    int src = p.perm[k];
    sm_perm[k] = src;
    sm_wsp[k] = p.wsp[k];
    sm_mu[k] = src >= 0 ? float(p.mean[src]) : 0.0f;
  }
  for (uint32_t e = threadIdx.x; e < kNPC * p.LP; e += blockDim.x) sm_pc[e] = p.pcs[e];
  if (threadIdx.x == 0) {
    float rng = 0.0f;
    for (int c = 0; c < kNPC; ++c) {
      sm_lo[c] = ord2f(p.pminmax[2 * c]);
      rng = fmaxf(rng, ord2f(p.pminmax[2 * c + 1]) - sm_lo[c]);
    }
    const float top = float((1u << (kVoxDims == 1 ? 15 : kVoxAxisBits)) - 1u);
    sm_scale = rng > 0.0f ? top / rng : 0.0f;
  }
  __syncthreads();
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < p.J; j += uint64_t(gridDim.x) * blockDim.x) {
    const float* y = p.tacs + j * p.L;
    float pr[kVoxDims];
#pragma unroll
    for (int c = 0; c < kVoxDims; ++c) pr[c] = 0.0f;
    for (uint32_t k = 0; k < p.LP; ++k) {
      int src = sm_perm[k];
      if (src < 0) break;
      const float x = sm_wsp[k] * __ldg(y + src) - sm_mu[k];
#pragma unroll
      for (int c = 0; c < kVoxDims; ++c) pr[c] = fmaf(x, sm_pc[c * p.LP + k], pr[c]);
    }
    unsigned long long key = 0;
    if (kVoxDims == 1) {
      key = f2ord(pr[0]);
    } else {
      const float top = float((1u << kVoxAxisBits) - 1u);
      uint32_t X[kVoxDims];
#pragma unroll
      for (int c = 0; c < kVoxDims; ++c) {
        const float sc = c == 0 ? sm_scale : (c == 1 ? sm_scale * VPET_VOXS : sm_scale * VPET_VOXS3);
        const float q = fminf(fmaxf((pr[c] - sm_lo[c]) * sc, 0.0f), top);
        X[c] = uint32_t(q);
        if (!VPET_HILBERT_VOX) key |= spread_d((unsigned long long)q) << (kVoxDims - 1 - c);
      }
      if (VPET_HILBERT_VOX) key = hilbert_key<kVoxDims, kVoxAxisBits>(X);
    }
    p.keys[j] = key;
    p.vals[j] = uint32_t(j);
  }
}

// ---- rotated voxel coordinates: thread per voxel, ytr[j][k] = RN32(sum_f rotq[f][k] y_f); the
// block's TAC rows are staged in shared memory with coalesced loads (odd row stride) ----
constexpr int kVR = 128;
__global__ void __launch_bounds__(kVR) voxel_rotate_kernel(const float* __restrict__ tacs, uint64_t J, uint32_t L,
                                                           uint32_t LP, const double* __restrict__ rotq,
                                                           float* __restrict__ ytr) {
  extern __shared__ double vq[];  // [L][LP] rotq, then [kVR][ys] TAC rows, then [kVR][LP + 1] outputs
  const uint32_t ys = L | 1u, os = LP + 1;
  float* yb = reinterpret_cast<float*>(vq + L * LP);
  float* ob = yb + kVR * ys;
  for (uint32_t e = threadIdx.x; e < L * LP; e += kVR) vq[e] = rotq[e];
  for (uint64_t base = uint64_t(blockIdx.x) * kVR; base < J; base += uint64_t(gridDim.x) * kVR) {
    const uint32_t nb = uint32_t(J - base < uint64_t(kVR) ? J - base : uint64_t(kVR));
    __syncthreads();
    const float* src = tacs + base * L;
    for (uint32_t e = threadIdx.x; e < nb * L; e += kVR) {
      const uint32_t v = e / L;
      yb[v * ys + (e - v * L)] = __ldcs(src + e);
    }
    __syncthreads();
    if (threadIdx.x < nb) rotate_curve<false>(yb + threadIdx.x * ys, vq, L, LP, ob + threadIdx.x * os);
    __syncthreads();
    float* dst = ytr + base * LP;  // the block's rows are contiguous: coalesced stores
    for (uint32_t e = threadIdx.x; e < nb * LP; e += kVR) {
      const uint32_t v = e / LP;
      dst[e] = ob[v * os + (e - v * LP)];
    }
  }
}

__global__ void vslot_kernel(const uint32_t* __restrict__ vorder, uint64_t J, uint32_t* __restrict__ vslot) {
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < J; j += uint64_t(gridDim.x) * blockDim.x)
    vslot[vorder[j]] = uint32_t(j);
}

}  // namespace

cudaError_t launch_voxel_rotate(const float* tacs, uint64_t J, uint32_t L, uint32_t LP, const double* rotq, float* ytr,
                                cudaStream_t st) {
  if (LP > kRotMaxLP) return cudaErrorInvalidValue;
  const size_t smem = sizeof(double) * L * LP + sizeof(float) * kVR * ((L | 1u) + LP + 1);
  cudaError_t e = ensure_smem_attr((const void*)voxel_rotate_kernel, smem);
  if (e != cudaSuccess) return e;
  voxel_rotate_kernel<<<148 * 4, kVR, smem, st>>>(tacs, J, L, LP, rotq, ytr);
  return cudaGetLastError();
}

size_t voxel_sort_temp_bytes(uint64_t J) { return radix_temp_bytes(J); }

cudaError_t launch_voxel_order(const VoxelOrderParams& p, cudaStream_t st, uint32_t* launches) {
  voxel_key_kernel<<<148 * 4, 256, 0, st>>>(p);
  *launches += 1;
  cudaError_t e = radix_sort_pairs(p.sort_temp, p.sort_temp_bytes, p.keys, p.keys_alt, p.vals, p.vorder, p.J, 0,
                                   kVoxBits, st, launches);
  if (e != cudaSuccess) return e;
  if (p.vslot) {
    vslot_kernel<<<148 * 4, 256, 0, st>>>(p.vorder, p.J, p.vslot);
    *launches += 1;
  }
  return cudaGetLastError();
}

size_t order_sort_temp_bytes(uint64_t N) { return radix_temp_bytes(N); }

cudaError_t launch_order(const OrderParams& p, cudaStream_t st, uint32_t* launches) {
  frame_stats_kernel<<<p.L, 1024, 0, st>>>(p);
  frame_perm_kernel<<<1, kMaxLP, 0, st>>>(p);
  *launches += 2;
  OrderParams q = p;
  if (p.tree) {
    cudaMemsetAsync(p.cov, 0, sizeof(double) * p.LP * p.LP, st);
    cov_kernel<<<dim3(p.LP, p.LP), 256, 0, st>>>(p);
    *launches += 2;
    if (p.rotq) {  // needs cov only; with an aux stream it overlaps proj / key / sort
      if (p.LP > kRotMaxLP) return cudaErrorInvalidValue;
      const size_t rs = sizeof(double) * 2 * p.LP * p.LP;
      cudaError_t er = ensure_smem_attr((const void*)rot_kernel, rs);
      if (er != cudaSuccess) return er;
      cudaStream_t rst = st;
      if (p.aux) {
        cudaEventRecord(p.ev_fork, st);
        cudaStreamWaitEvent(p.aux, p.ev_fork, 0);
        rst = p.aux;
      }
      rot_kernel<<<1, 256, rs, rst>>>(p);
      if (p.aux) cudaEventRecord(p.ev_join, p.aux);
      *launches += 1;
    }
    {
      const size_t cs = sizeof(double) * p.LP * p.LP;
      cudaError_t ec = ensure_smem_attr((const void*)pca_kernel, cs);
      if (ec != cudaSuccess) return ec;
      pca_kernel<<<1, 32, cs, st>>>(p);
    }
    proj_minmax_kernel<<<148 * 4, 256, 0, st>>>(p);
    key_kernel<<<148 * 8, 256, 0, st>>>(p);
    *launches += 2;
    // the lowest 8 key bits (the two finest levels of the curve) are not sorted: one radix pass
    // less, same scan time (Morton, measured: 0 / 8 / 16 bits -> scan 19.6 / 19.5 / 20.3 ms; with
    // the Hilbert order 24 unsorted bits double the scan); the order is free.
    // Tuning knob VPET_SORT_LO.
    static const int lo_bit = getenv("VPET_SORT_LO") ? atoi(getenv("VPET_SORT_LO")) : 8;
    cudaError_t e = radix_sort_pairs(p.sort_temp, p.sort_temp_bytes, p.keys, p.keys_alt, p.vals, p.order, p.N, lo_bit,
                                     kNPC * kMBits, st, launches);
    if (e != cudaSuccess) return e;
  } else {
    q.order = nullptr;
  }
  {
    if (!p.tree) q.rotq = nullptr;
    if (q.rotq && p.aux) cudaStreamWaitEvent(st, p.ev_join, 0);
    const size_t psmem = sizeof(float) * kPermWarps * kTile * ((p.LS > p.LP ? p.LS : p.LP) + 1) * (q.rotq ? 2 : 1) +
                         (q.rotq ? sizeof(double) * p.L * p.LP : 0);
    cudaError_t ea = ensure_smem_attr((const void*)permute_kernel, psmem);
    if (ea != cudaSuccess) return ea;
    permute_kernel<<<148 * 8, 32 * kPermWarps, psmem, st>>>(q);
    *launches += 1;
  }
  if (p.tree) {
    uint64_t ntile = (p.N + kTile - 1) / kTile;
    uint64_t nsup = (ntile + kSuper - 1) / kSuper;
    super_bounds_kernel<<<unsigned(nsup), 128, 0, st>>>(p, ntile);
    hyper_bounds_kernel<<<unsigned(p.nhyper), 128, 0, st>>>(p, nsup);
    *launches += 2;
    if (p.rotq && p.gbox) {
      global_box_kernel<<<1, 128, 0, st>>>(p);
      *launches += 1;
    }
  }
  return cudaGetLastError();
}

}  // namespace vpet
