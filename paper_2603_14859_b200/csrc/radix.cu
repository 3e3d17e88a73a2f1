// radix.cu -- stable LSD radix sort of (u64 key, u32 value) pairs on a bit range, used by the order
// stage for the draw order (Hilbert keys of the bank's principal projections) and the voxel order
// (Morton keys).  8-bit digits; per pass three kernels:
//   hist     per tile of RT = 4096 elements (RB threads x RI items) a 256-bin digit histogram,
//            stored digit-major: counts[d * ntiles + tile];
//   scan     one warp per digit: exclusive prefix of the digit's counts over the tiles, and the
//            digit total;
//   scatter  per tile: digit bases = exclusive scan of the 256 totals + the tile's prefix, a stable
//            rank within the tile from __match_any_sync over 32-element rounds (warp-local counts
//            per digit, then an exclusive scan of the warps' counts), the tile sorted by digit in
//            shared memory, then written out so that each digit's run is a contiguous store.
// Element e of a tile is (warp w, round k, lane l) -> tile * RT + w * RI * 32 + k * 32 + l, so the
// ranks follow the input order: the sort is stable (equal keys keep their input order).
#include "common.cuh"

namespace vpet {
namespace {

constexpr int RB = 256;          // threads per block
constexpr int RI = 8;            // items per thread
constexpr int RT = RB * RI;      // elements per tile
constexpr int RW = RB / 32;      // warps per block

__device__ __forceinline__ uint32_t tile_elem(int w, int k, int lane) {
  return uint32_t(w * RI * 32 + k * 32 + lane);
}

__global__ void __launch_bounds__(RB) radix_hist_kernel(const unsigned long long* __restrict__ keys, uint64_t n, int shift,
                                                        uint32_t* __restrict__ counts, uint32_t ntiles) {
  __shared__ uint32_t h[256];
  for (int i = threadIdx.x; i < 256; i += RB) h[i] = 0u;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t base = uint64_t(blockIdx.x) * RT;
#pragma unroll 4
  for (int k = 0; k < RI; ++k) {
    const uint64_t e = base + tile_elem(w, k, lane);
    if (e < n) atomicAdd(&h[uint32_t(__ldg(keys + e) >> shift) & 255u], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += RB) counts[uint64_t(d) * ntiles + blockIdx.x] = h[d];
}

// one warp per digit: in-place exclusive prefix over the tiles, and the digit's total
__global__ void __launch_bounds__(256) radix_scan_kernel(uint32_t* __restrict__ counts, uint32_t ntiles,
                                                         uint32_t* __restrict__ totals) {
  const int lane = threadIdx.x & 31;
  const uint32_t d = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (d >= 256) return;
  uint32_t* c = counts + uint64_t(d) * ntiles;
  uint32_t carry = 0;
  for (uint32_t b0 = 0; b0 < ntiles; b0 += 32) {
    const uint32_t b = b0 + lane;
    const uint32_t v = b < ntiles ? c[b] : 0u;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (b < ntiles) c[b] = carry + x - v;
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) totals[d] = carry;
}

__global__ void __launch_bounds__(RB) radix_scatter_kernel(const unsigned long long* __restrict__ kin,
                                                           const uint32_t* __restrict__ vin,
                                                           unsigned long long* __restrict__ kout,
                                                           uint32_t* __restrict__ vout, uint64_t n, int shift,
                                                           const uint32_t* __restrict__ counts, uint32_t ntiles,
                                                           const uint32_t* __restrict__ totals) {
  __shared__ uint32_t base[256];
  __shared__ uint32_t wcnt[RW][256];
  __shared__ uint32_t tcnt[256], toff[256];
  __shared__ unsigned long long sk[RT];
  __shared__ uint32_t sv[RT];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  // digit bases: exclusive scan of the 256 totals (warp 0, 8 digits per lane) + this tile's prefix
  if (w == 0) {
    uint32_t t[8], s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      t[q] = totals[lane * 8 + q];
      s += t[q];
    }
    uint32_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    uint32_t run = x - s;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int d = lane * 8 + q;
      base[d] = run + counts[uint64_t(d) * ntiles + blockIdx.x];
      run += t[q];
    }
  }
  for (int i = threadIdx.x; i < RW * 256; i += RB) (&wcnt[0][0])[i] = 0u;
  const uint64_t t0 = uint64_t(blockIdx.x) * RT;
  unsigned long long key[RI];
  uint32_t val[RI];
  uint32_t dig[RI];
#pragma unroll
  for (int k = 0; k < RI; ++k) {
    const uint64_t e = t0 + tile_elem(w, k, lane);
    const bool ok = e < n;
    key[k] = ok ? __ldg(kin + e) : 0ull;
    val[k] = ok ? __ldg(vin + e) : 0u;
    dig[k] = ok ? uint32_t(key[k] >> shift) & 255u : 0x100u + uint32_t(lane);  // padding: unique, never written
  }
  __syncthreads();
  // pass 1: per-warp digit counts
#pragma unroll
  for (int k = 0; k < RI; ++k) {
    const uint32_t peers = __match_any_sync(0xffffffffu, dig[k]);
    if (dig[k] < 256u && lane == __ffs(peers) - 1) wcnt[w][dig[k]] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // exclusive scan of the warps' counts per digit (warp order = input order); tcnt keeps the last
  // warp's own count so that the tile total is wcnt[RW - 1][d] + tcnt[d]
  for (int d = threadIdx.x; d < 256; d += RB) {
    uint32_t run = 0;
#pragma unroll
    for (int q = 0; q < RW; ++q) {
      const uint32_t c = wcnt[q][d];
      wcnt[q][d] = run;
      run += c;
    }
    tcnt[d] = run - wcnt[RW - 1][d];
  }
  __syncthreads();
  // tile-local digit offsets: exclusive scan over the digits of the tile's counts
  if (w == 0) {
    uint32_t c[8], s = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int d = lane * 8 + q;
      c[q] = wcnt[RW - 1][d] + tcnt[d];  // exclusive over warps + the last warp's own count = tile count
      s += c[q];
    }
    uint32_t x = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    uint32_t run = x - s;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      toff[lane * 8 + q] = run;
      run += c[q];
    }
  }
  __syncthreads();
  // pass 2: stable tile-local ranks -> the tile sorted in shared memory
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int k = 0; k < RI; ++k) {
    const uint32_t peers = __match_any_sync(0xffffffffu, dig[k]);
    if (dig[k] < 256u) {
      const uint32_t d = dig[k];
      const uint32_t lp = toff[d] + wcnt[w][d] + __popc(peers & lt);
      sk[lp] = key[k];
      sv[lp] = val[k];
    }
    __syncwarp();
    if (dig[k] < 256u && lane == __ffs(peers) - 1) wcnt[w][dig[k]] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // write out in tile-sorted order: runs of one digit go to consecutive global positions
  const uint32_t nv = uint32_t(n - t0 < uint64_t(RT) ? n - t0 : uint64_t(RT));
  for (uint32_t j = threadIdx.x; j < nv; j += RB) {
    const unsigned long long kk = sk[j];
    const uint32_t d = uint32_t(kk >> shift) & 255u;
    const uint64_t pos = uint64_t(base[d]) + (j - toff[d]);
    kout[pos] = kk;
    vout[pos] = sv[j];
  }
}

uint32_t radix_tiles(uint64_t n) { return uint32_t((n + RT - 1) / RT); }

}  // namespace

size_t radix_temp_bytes(uint64_t n) {
  const uint64_t nt = radix_tiles(n > 0 ? n : 1);
  return 4 * n + 4 * 256 * nt + 4 * 256 + 256;
}

// Sort (keys, vals_in) by key bits [lo_bit, hi_bit), stable.  keys and keys_alt are overwritten
// (ping-pong); the sorted values are written to vals_out (vals_in is not modified).
cudaError_t radix_sort_pairs(void* temp, size_t temp_bytes, unsigned long long* keys, unsigned long long* keys_alt,
                             const uint32_t* vals_in, uint32_t* vals_out, uint64_t n, int lo_bit, int hi_bit,
                             cudaStream_t st, uint32_t* launches) {
  if (n == 0) return cudaSuccess;
  if (temp_bytes < radix_temp_bytes(n)) return cudaErrorInvalidValue;
  const uint32_t nt = radix_tiles(n);
  uint32_t* vtmp = static_cast<uint32_t*>(temp);
  uint32_t* counts = vtmp + n;
  uint32_t* totals = counts + uint64_t(256) * nt;
  const int D = (hi_bit - lo_bit + 7) / 8;
  const unsigned long long* kin = keys;
  const uint32_t* vin = vals_in;
  for (int p = 0; p < D; ++p) {
    const int shift = lo_bit + 8 * p;
    unsigned long long* kout = (p % 2 == 0) ? keys_alt : keys;
    uint32_t* vout = ((D - 1 - p) % 2 == 0) ? vals_out : vtmp;
    radix_hist_kernel<<<nt, RB, 0, st>>>(kin, n, shift, counts, nt);
    radix_scan_kernel<<<32, 256, 0, st>>>(counts, nt, totals);
    radix_scatter_kernel<<<nt, RB, 0, st>>>(kin, vin, kout, vout, n, shift, counts, nt, totals);
    kin = kout;
    vin = vout;
  }
  if (launches) *launches += 3 * D;
  return cudaGetLastError();
}

}  // namespace vpet
