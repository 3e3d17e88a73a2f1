// common.cuh -- device-side building blocks shared by the kernels of libvpetabc.so.
// (Independent of oracle/: nothing here is shared with the CPU oracle.)
#pragma once
#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/vpetabc.h"

namespace vpet {

constexpr uint32_t kCtrTag = 0x56504554u;  // "VPET": 4th Philox counter word (R7)
constexpr int kMaxLP = 128;
#ifndef VPET_NPC
#define VPET_NPC 4
#endif
constexpr int kNPC = VPET_NPC;  // principal axes used for the draw order (order.cu)
#ifndef VPET_TILE
#define VPET_TILE 32
#endif
#ifndef VPET_SUPER
#define VPET_SUPER 8
#endif
constexpr int kTile = VPET_TILE;    // draws per tile (bounding box + TMA transfer unit)
constexpr int kSuper = VPET_SUPER;  // tiles per super-tile (<= 32: one bit per tile in a mask)
constexpr int kMaxGrid = 8192;  // max points of a draw-independent time grid
// ---------------------------------------------------------------------------------------
// Eps-mode moment sums in 128-bit fixed point (kFixFrac fractional bits).  Each accepted draw's
// value is rounded once to the grid 2^-62 (deterministically, per draw); integer sums are then
// exact and associative, so the result does not depend on the order in which the FP32 pass
// visits the draws (which depends on the voxel's CTA-mates, i.e. on the sharding).
// Range: |value| < 2^53, sums < 2^64 (count <= 2^32, values < 2^31): < 2^126.
// ---------------------------------------------------------------------------------------
typedef __int128 Fix128;
constexpr int kFixFrac = 62;
__host__ __device__ inline Fix128 to_fix(double v) {
  const double ip = trunc(v);
  const double r = v - ip;  // exact, |r| < 1
#ifdef __CUDA_ARCH__
  const long long f = __double2ll_rn(r * 4611686018427387904.0);  // r 2^62 (exact scaling)
#else
  const long long f = llrint(r * 4611686018427387904.0);
#endif
  return (Fix128((long long)ip) << kFixFrac) + Fix128(f);
}
__host__ __device__ inline double from_fix(Fix128 a) {
  const long long hi = (long long)(a >> kFixFrac);  // floor
  const unsigned long long lo = (unsigned long long)(a & ((Fix128(1) << kFixFrac) - 1));
  return double(hi) + double(lo) * 2.168404344971008868e-19;  // 2^-62
}

// ---------------------------------------------------------------------------------------
// Prior draw (Alg.1 l.1-2): Philox4x32-10 keyed by the seed, counter
// {i_lo, i_hi, block, 'VPET'}; u = (2*(x>>9)+1) 2^-24; theta = fmaf(hi-lo, u, lo).
// ---------------------------------------------------------------------------------------
__host__ __device__ inline void philox10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                                         uint32_t k1, uint32_t out[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
#ifdef __CUDA_ARCH__
    uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
#else
    uint64_t p0 = 0xD2511F53ull * c0, p1 = 0xCD9E8D57ull * c2;
    uint32_t hi0 = uint32_t(p0 >> 32), lo0 = uint32_t(p0), hi1 = uint32_t(p1 >> 32), lo1 = uint32_t(p1);
#endif
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

__host__ __device__ inline float u01(uint32_t x) {
  return float(((x >> 9) << 1) | 1u) * 5.9604644775390625e-8f;  // * 2^-24 (exact)
}

// Model / prior description in device-friendly form (constant memory).
struct ModelDev {
  int32_t kind;
  uint32_t P;          // columns of the family (5 or 7)
  uint64_t begin, end; // draw-index block [begin, end)
  float lo[ABC_MAX_P], span[ABC_MAX_P];  // span = fl32(hi - lo)
};
struct PriorDev {
  uint32_t M;
  uint32_t seed_lo, seed_hi;
  ModelDev m[ABC_MAX_MODELS];
};

__host__ __device__ inline int model_index(const PriorDev& pr, uint64_t i) {
  int m = 0;
#pragma unroll
  for (int k = 1; k < ABC_MAX_MODELS; ++k)
    if (k < (int)pr.M && i >= pr.m[k].begin) m = k;
  return m;
}

// theta columns of draw i (P columns; IRR k4 := 0, MRTM gamma := 0, RT column 5 = tD + offset)
__host__ __device__ inline int draw_theta(const PriorDev& pr, uint64_t i, float th[ABC_MAX_P]) {
  int m = model_index(pr, i);
  const ModelDev& md = pr.m[m];
  uint32_t w[8];
  philox10(uint32_t(i), uint32_t(i >> 32), 0u, kCtrTag, pr.seed_lo, pr.seed_hi, w);
  philox10(uint32_t(i), uint32_t(i >> 32), 1u, kCtrTag, pr.seed_lo, pr.seed_hi, w + 4);
#pragma unroll
  for (int k = 0; k < ABC_MAX_P; ++k) th[k] = (k < (int)md.P) ? fmaf(md.span[k], u01(w[k]), md.lo[k]) : 0.0f;
  if (md.kind == ABC_2TCM_IRR || md.kind == ABC_MRTM) th[3] = 0.0f;
#ifdef __CUDA_ARCH__
  if (md.kind >= ABC_MRTM) th[5] = __fadd_rn(th[4], th[5]);
#else
  if (md.kind >= ABC_MRTM) th[5] = th[4] + th[5];
#endif
  return m;
}

// ---------------------------------------------------------------------------------------
// Exponential-integral phi functions (exact integration of a linear input against e^{-a t}
// over a step of length h, x = a h):
//   p1 = (1-e^-x)/x, ps = (x-1+e^-x)/x^2, ch = p1 - ps = (1-e^-x(1+x))/x^2,
//   om = (x^2/2-1+e^-x(1+x))/x^3;  e = e^-x.
// Series (Horner, 18 terms) below x = 0.5, closed forms above.
// ---------------------------------------------------------------------------------------
struct Phi {
  double e, p1, ps, ch, om;
};

__device__ inline Phi phi_all(double x) {
  Phi r;
  if (x == 0.0) {
    r.e = 1.0; r.p1 = 1.0; r.ps = 0.5; r.ch = 0.5; r.om = 1.0 / 3.0;
  } else if (x < 0.5) {
    // coefficients: p1: 1/(k+1)!, ps: 1/(k+2)!, om: (k+2)/(k+3)!, alternating in x.
    double p1 = 0.0, ps = 0.0, om = 0.0;
    double f1 = 1.0 / 6402373705728000.0;  // 1/18!
    double f2 = f1 / 19.0, f3 = f2 / 20.0;  // 1/19!, 1/20!
#pragma unroll
    for (int k = 17; k >= 0; --k) {
      // f1 = 1/(k+1)!, f2 = 1/(k+2)!, f3 = 1/(k+3)!
      p1 = fma(p1, -x, f1);
      ps = fma(ps, -x, f2);
      om = fma(om, -x, double(k + 2) * f3);
      f3 = f2; f2 = f1; f1 = f1 * double(k + 1);
    }
    r.p1 = p1; r.ps = ps; r.om = om;
    r.ch = p1 - ps;           // ~1/2: no cancellation
    r.e = fma(-x, p1, 1.0);   // 1 - x p1 = e^-x; x p1 <= 0.4
  } else {
    double e = exp(-x);
    double em1 = 1.0 - e;     // e <= 0.61: no cancellation
    double ix = 1.0 / x;
    r.e = e;
    r.p1 = em1 * ix;
    r.ps = (x - em1) * ix * ix;
    r.ch = (em1 - x * e) * ix * ix;
    r.om = (0.5 * x * x - em1 + x * e) * ix * ix * ix;
  }
  return r;
}

// (1 - e^-x)/x for x >= 0; expm1 keeps full relative accuracy as x -> 0.
__device__ inline double phi1_only(double x) { return x == 0.0 ? 1.0 : -expm1(-x) / x; }

// ---------------------------------------------------------------------------------------
// Launch-side helpers
// ---------------------------------------------------------------------------------------
constexpr int kPhiSlots = 2;  // per-rate cache of phi(a h) for recently seen segment lengths h
struct Tables {
  // frames (acquisition order)
  uint32_t L, LS;          // frames, padded stride of the exact bank
  const double* fdur;      // [L]
  const double* finv;      // [L] 1 / fdur (host-rounded)
  const double* fs;        // [L] starts
  const double* fe;        // [L] ends
  const double* favg_in;   // [L] int_frame C_in dt (draw independent)
  const float* w;          // [L] weights (1 if none)
  // coarse grid (PWL input U frame bounds)
  uint32_t G;
  const double* gt;        // [G]
  const double* gc;        // [G] input value at grid points
  const int* gframe;       // [G-1] frame of segment k or -1
  const uint8_t* gcode;    // [G-1] phi cache code of segment k: bit 7 = recompute, bits 0-1 = slot
  // fine grid (lp-ntPET)
  uint32_t GF;
  const double* ft;
  const double* fc;
  const int* fframe;
  // Feng input
  int feng;
  double fb[6];
  // simulated-draw noise (abc_set_sim_noise): ell = 0 disables
  double noise_ell, noise_lam;
  // [L] S_f(0) = frame integrals of the rate-0 convolution on the coarse grid (PWL input): the
  // draw-independent half of an irreversible 2TCM draw (launch_s0_table); nullptr = not available
  const double* s0;
};

struct BankParams {
  Tables T;
  uint64_t N;
  float* bank;  // [N][LS] RN32 frame averages, acquisition order, zero padded
};

void launch_bank(const BankParams& p, const PriorDev& prior, cudaStream_t st);
void launch_s0_table(const Tables& T, double* s0, cudaStream_t st);

struct OrderParams {
  const float* bank;  // [N][LS]
  uint64_t N;
  uint32_t L, LS, LP;
  const float* wsc;   // [L] prescale factor per frame (sqrt(w) for WL2, w for L1, 1 if unit)
  double* var;        // [L] scratch: spread of the prescaled frame
  double* mean;       // [L] scratch: mean of the prescaled frame
  int* perm;          // [LP] out: source frame of scan position k (-1 = pad)
  float* wsp;         // [LP] out: prescale factor of scan position k (0 for pad)
  float* bankp;       // [N][LP] out: -(wsp[k] * bank[order[j]][perm[k]])
  int reorder;
  // locality order + bounds (tree mode)
  int tree;
  double* cov;        // [LP][LP]
  float* pcs;         // [kNPC][LP]
  unsigned int* pminmax;  // [kNPC][2] ordered-int min/max of the projections
  float* proj;            // [N][kNPC] principal-axis projections (written by proj_minmax, read by key)
  unsigned long long* keys;      // [N]
  unsigned long long* keys_alt;  // [N]
  uint32_t* vals;     // [N]
  uint32_t* order;    // [N] sorted position -> draw index
  uint32_t* idxmap;   // [N] out: draw index of scan row j
  void* sort_temp;
  size_t sort_temp_bytes;
  float* tbounds;     // [ntile][2][LP] per-tile min/max of bankp
  float* sbounds;     // [nsuper][2][LP]
  float* hbounds;     // [nhyper][2][LP] (hyper-tile = hs consecutive super-tiles)
  uint32_t hs;
  uint64_t nhyper;
  // rotated scan basis (WL2, tree mode): rotq != nullptr selects it
  double* rotq;         // [L][LP] out: rotq[f][k] = Q[a][k] sqrt(w_f), f = perm[a]; scan coordinate k = sum_f rotq[f][k] x_f
  const double* cw;     // [L] sqrt(w_f) in FP64 (1 for unit weights)
  float* gbox;          // [2][LP] out (rotated basis): min / max of bankp over all draws
  cudaStream_t aux;     // if set: the basis (rot_kernel) runs on it, overlapped with the draw-order sort
  cudaEvent_t ev_fork, ev_join;
};
cudaError_t launch_order(const OrderParams& p, cudaStream_t st, uint32_t* launches);
// Rotated voxel coordinates ytr[j][k] = RN32(sum_f rotq[f][k] y_f) (FP64 sums), k < LP.
cudaError_t launch_voxel_rotate(const float* tacs, uint64_t J, uint32_t L, uint32_t LP, const double* rotq, float* ytr,
                                cudaStream_t st);
// ||Q^T Q - I||_2 assumed by the rotated-basis error bound (checked on device; Q = I otherwise)
constexpr double kRotEps = 1e-10;
size_t order_sort_temp_bytes(uint64_t N);

// Voxel order for the tree scan: voxels sorted by the projection of their prescaled TAC on the
// bank's first principal axis, so a warp's voxels have similar TACs (smaller alive-tile unions).
struct VoxelOrderParams {
  const float* tacs;  // [J][L]
  uint64_t J;
  uint32_t L, LP;
  const int* perm;
  const float* wsp;
  const double* mean;  // [L] prescaled frame means (acquisition order)
  const float* pcs;    // [kNPC][LP]
  const unsigned int* pminmax;  // [2 kNPC] bank projection range (order-preserving uint of float)
  unsigned long long* keys;
  unsigned long long* keys_alt;
  uint32_t* vals;
  uint32_t* vorder;   // out [J]
  uint32_t* vslot;    // out [J]: vslot[vorder[j]] = j
  void* sort_temp;
  size_t sort_temp_bytes;
};
size_t voxel_sort_temp_bytes(uint64_t J);
// Stable LSD radix sort of (u64 key, u32 value) pairs on key bits [lo_bit, hi_bit) (radix.cu).
// keys / keys_alt are overwritten (ping-pong); the sorted values land in vals_out.
size_t radix_temp_bytes(uint64_t n);
cudaError_t radix_sort_pairs(void* temp, size_t temp_bytes, unsigned long long* keys, unsigned long long* keys_alt,
                             const uint32_t* vals_in, uint32_t* vals_out, uint64_t n, int lo_bit, int hi_bit,
                             cudaStream_t st, uint32_t* launches);
cudaError_t launch_voxel_order(const VoxelOrderParams& p, cudaStream_t st, uint32_t* launches);

// Rigorous bound on |D32 - D| for the FP32 pass:
//   err(D) = a D + b sqrt(Y2 D) + c Y2 + d Y1,  Y2 = sum_f w_f y_f^2, Y1 = sum_f w_f |y_f|.
struct ErrBound {
  double a, b, c, d;
};

struct ScanParams {
  const float* bankp;   // [N][LP] negated prescaled bank in scan order
  uint64_t N;
  const float* tacs;    // [J][L]
  uint64_t J;
  uint32_t L;
  const int* perm;      // [LP]
  const float* wsp;     // [LP]
  uint32_t K;           // heap capacity per voxel (top-n mode)
  unsigned long long* heap;  // [J][nparts][heap_stride(K)] keys (D32 bits << 32 | idx), 8-ary heaps
  uint32_t* heap_cnt;   // [J]
  int prune;
  unsigned long long* work;  // frame-update counter (COUNT)
  // eps mode
  int eps_mode;
  double eps;
  const float* w;       // [L] weights (acquisition order), for inline FP64 rescoring
  const float* bank;    // [N][LS] exact bank
  uint32_t LS;
  int dist;             // ABC_DIST_*
  int unit_w;
  Fix128* mom;          // [J][nparts][M][MOMW] eps-mode moment sums (fixed point, one owner per slot)
  ErrBound eb;
  const PriorDev* prior_g;  // device copy of the prior (eps-mode slow path)
  uint32_t M;
  // tree mode
  const uint32_t* idxmap;   // [N] draw index of scan row j
  const float* tbounds;     // [ntile][2][LP]
  const float* sbounds;     // [nsuper][2][LP]
  const float* hbounds;     // [nhyper][2][LP]
  uint64_t ntile, nsuper, nhyper;
  uint32_t hs;              // super-tiles per hyper-tile
  unsigned long long* bound_work;  // LB frame-evaluation counter (COUNT)
  // work split: item = (voxel tile, part); part p owns hyper-tiles h = p (mod nparts) and its own
  // heap [J][nparts][K]; tau_glob[v] = min over parts of their heap thresholds (shared pruning)
  uint32_t nparts;
  unsigned int* tau_glob;   // [J] float bits (positive), atomicMin; indexed by scan slot (vorder position)
  unsigned int* queue;      // work-queue counter (zeroed per run)
  unsigned long long* item_log;  // diagnostics (env VPET_ITEMLOG): [item][4] = start ns, end ns, SM, voxel tile
  const uint32_t* vorder;   // [J] voxel processed in slot j (tree mode) or nullptr (identity)
  const int* bad;           // set by the finite check when a TAC value is not finite: skip all work
  const float* ytr;         // [J][LP] rotated voxel coordinates (rotated basis) or nullptr (frame basis)
  const float* gbox;        // [2][LP] rotated basis: min / max over the whole scan bank (tail bounds)
};
// Candidate heaps: 8-ary max-heaps; node i lives at slot i + kHeapOff of a (voxel, part) row of
// heap_stride(K) keys, so the 8 children of node i (slots 8i + 8 .. 8i + 15) are one 64-B group.
constexpr uint32_t kHeapOff = 7;
__host__ __device__ inline uint32_t heap_stride(uint32_t K) { return (K + kHeapOff + 7u) & ~7u; }
#ifndef VPET_HSORTMAX
#define VPET_HSORTMAX 256
#endif
constexpr int kHyperSort = VPET_HSORTMAX;  // max hyper-tiles per part (best-first order sorted in shared memory)
constexpr int MOMW = 2 + 2 * ABC_MAX_P + 2;  // count, (S1,S2) x P, (KS1, KS2), pad
cudaError_t launch_scan(const ScanParams& p, uint32_t LP, int count_work, int tree, cudaStream_t st);
cudaError_t launch_scan_wl2(const ScanParams& p, uint32_t LP, int count_work, int tree, cudaStream_t st);
cudaError_t launch_scan_l1(const ScanParams& p, uint32_t LP, int count_work, int tree, cudaStream_t st);
bool scan_supported(uint32_t LP);
uint32_t scan_lp_for(uint32_t L);

struct ExactParams {
  const float* bank;  // [N][LS]
  uint64_t N;
  uint32_t L, LS;
  const float* tacs;  // [J][L]
  const float* w;     // [L]
  int dist;
  uint32_t n;
  const uint32_t* list;  // voxel list (nullptr = all voxels 0..J-1)
  const uint32_t* list_len;  // device count (nullptr = J)
  uint64_t J;
  double* hd;         // [J][n] exact heap distances
  uint32_t* hi;       // [J][n] exact heap indices
  const int* bad;     // non-finite TACs: skip all work
};
void launch_exact_scan(const ExactParams& p, cudaStream_t st);

struct ReduceParams {
  // candidates
  int exact;                    // 1: candidates from the exact heap (no certification)
  const unsigned long long* heap;  // fast mode: [J][nparts][heap_stride(K)]
  const uint32_t* heap_cnt;        // [J][nparts]
  uint32_t K;
  uint32_t nparts;
  const unsigned int* tau_glob;    // [J] by scan slot (tree mode, via vslot) or voxel, or nullptr: bound B on excluded draws' D32
  const uint32_t* vslot;           // [J] scan slot of voxel v (tree mode) or nullptr (identity)
  const double* hd;             // exact mode
  const uint32_t* hidx;
  const uint32_t* list;         // voxel list or nullptr
  const uint32_t* list_len;
  uint64_t J;
  uint32_t n;
  // data
  const float* bank;  // [N][LS]
  uint64_t N;
  uint32_t L, LS, LP;
  const float* tacs;
  const float* w;
  int dist;
  int unit_w;
  ErrBound eb;
  PriorDev prior;
  uint32_t P;
  // fallback output
  uint32_t* fb_list;
  uint32_t* fb_len;
  int force_fb;       // ABC_FLAG_FORCE_FALLBACK: treat every voxel as uncertified (test hook)
  const int* bad;     // non-finite TACs: skip all work
  // fallback tiers.  An uncertified voxel is appended to fb_list with fb_tau = the
  // n-th smallest FP64 distance among its candidates (an upper bound on the exact tau64; +inf if
  // unknown).  exact == 2: the candidates are the draws with D64 <= fb_tau collected for fb_list
  // entry e by the fallback collector (cl_*); a voxel that cannot use them goes to fb2_list (exact
  // heap scan, exact == 1).
  double* fb_tau;            // [J] per fb_list entry
  const double* cl_d;        // [cl_voxels][cl_cap]
  const uint32_t* cl_i;      // [cl_voxels][cl_cap]
  const uint32_t* cl_cnt;    // [cl_voxels]
  uint32_t cl_cap, cl_voxels;
  uint32_t* fb2_list;
  uint32_t* fb2_len;
  // list_only: the certification (warp layout) writes each voxel's (D, i)-sorted accepted list to
  // acc_i / acc_d ([J][n]) instead of reducing it; launch_reduce_accepted_lists reduces them all
  int list_only;
  uint32_t* acc_i;
  double* acc_d;
  int reg_sort;  // n <= 32: order statistics by register sorts across the lanes (K4)
  // results (device pointers, may be null)
  abc_result out;
};
cudaError_t launch_certify_reduce(const ReduceParams& p, cudaStream_t st);
// candidate capacity (a power of two >= 32) of the certification of p
uint32_t certify_capacity(const ReduceParams& p);
// Fallback collector: for fb_list entry e < min(*list_len, cap_voxels) with finite tau[e], every draw
// with D64 <= tau[e] (FP64, operation for operation as the oracle; prefix pruning) is appended to
// entry e's list (cnt[e] counts all of them, at most cap are stored).  The N draws of a voxel are
// split into nchunk warp items spread over the whole GPU.
struct CollectParams {
  const float* bank;  // [N][LS]
  uint64_t N;
  uint32_t L, LS;
  const float* tacs;
  const float* w;
  int dist;
  const uint32_t* list;
  const uint32_t* list_len;
  const double* tau;
  uint32_t cap_voxels, cap, nchunk;
  uint32_t* cnt;
  double* cd;
  uint32_t* ci;
  const int* bad;
};
void launch_fallback_collect(const CollectParams& p, cudaStream_t st);
// Certification layouts: warp per voxel while the candidate set (a power of two) is <= kWarpCertifyMax,
// else one CTA per voxel with up to kLargeMaxCand candidates in shared memory (196 KB).
constexpr uint32_t kWarpCertifyMax = 2048;
constexpr uint32_t kLargeMaxCand = 16384;
constexpr uint32_t kMaxAccept = 15360;  // n_accept cap: n + n/16 slack <= kLargeMaxCand (one part)
// K4 on given accepted lists (abc_reduce_accepted): the first p.n of n_acc indices per voxel.
cudaError_t launch_reduce_list(const ReduceParams& p, const uint64_t* idx, uint32_t n_acc, int* bad, cudaStream_t st);
// K4 over the accepted lists written by list_only certification (u32 indices, FP64 distances).
cudaError_t launch_reduce_accepted_lists(const ReduceParams& p, const uint32_t* idx, const double* dist, int* bad,
                                         cudaStream_t st);

// Response-function envelope (Fig. 1): abc_response_envelope.
struct EnvelopeParams {
  const uint64_t* acc_idx;  // [J][n_acc]
  uint64_t J, N;
  uint32_t n_acc, T;
  const double* t;          // [T] minutes
  PriorDev prior;
  float* q;                 // [J][T][3]
  int* bad;                 // set when an index is >= N
};
cudaError_t launch_response_envelope(const EnvelopeParams& p, cudaStream_t st);

// Patlak K_i map (patlak.cu): abc_patlak.
struct PatlakParams {
  const float* tacs;   // [J][L]
  uint64_t J;
  uint32_t L, f0;      // frames f0.. carry the coefficients (the others are 0)
  const double* a;     // [L] slope weights
  const double* b;     // [L] mean-of-z weights
  double xbar;
  int valid;           // >= 2 late frames with spread in x
  float* ki;           // [J]
  float* intercept;    // [J] or nullptr
};
void launch_patlak(const PatlakParams& p, cudaStream_t st);

struct EpsReduceParams {
  const Fix128* mom;    // [J][nparts][M][MOMW]
  uint32_t nparts;
  uint64_t J;
  PriorDev prior;
  uint32_t P;
  abc_result out;
};
void launch_eps_reduce(const EpsReduceParams& p, cudaStream_t st);

void launch_fill_u32(uint32_t* p, uint32_t v, uint64_t n, cudaStream_t st);
// Opt `func` in to `bytes` of dynamic shared memory on the CURRENT device (the attribute is per
// device; cached per (function, device), thread-safe).  Returns the CUDA error of the opt-in, or
// cudaErrorInvalidValue when `bytes` exceeds the device's opt-in maximum.
cudaError_t ensure_smem_attr(const void* func, size_t bytes);

// K6 (dense_tc.cu): shared-bank tensor-core distance, ABC_FLAG_DENSE_TC (WL2, top-n, L <= 48).
// Operands live in HBM pre-tiled in the UMMA no-swizzle K-major core-matrix layout (bf16 bits).
struct DenseParams {
  uint16_t* Bt;             // [Npad/256][256 x 144] bank operand [b_hi | b_lo | b_hi]
  float* S2;                // [Npad] sum b^2 (FP32; +inf for padding rows)
  uint16_t* At;             // [Jpad/128][128 x 144] voxel operand [a_hi | a_hi | a_lo]
  float* Y2;                // [Jpad] sum a^2 (FP32)
  uint64_t N, J, ntile;
  uint32_t L, K;
  unsigned long long* heap;  // [J][2][heap_stride(K)]: part = column half of each draw tile
  uint32_t* heap_cnt;        // [J][2]
  unsigned int* tau_glob;    // [J]
  const int* bad;            // non-finite TACs: skip all work
};
uint64_t dense_bank_bytes(uint64_t N);
uint64_t dense_voxel_bytes(uint64_t J);
cudaError_t launch_dense(DenseParams p, const float* bank, uint32_t LS, const float* tacs, const float* wsc,
                         cudaStream_t st, uint32_t* launches);

}  // namespace vpet
