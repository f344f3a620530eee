// sort.cu -- hand-written device primitives for the report paths: an LSD
// radix sort of 64-bit keys, stream compaction of flagged indices and of
// distinct keys (RaceState::reported in std::set order, mckg_sort_triples;
// the deadlocked-block list of K4, mckg_scan_stuck).  No library kernels.
//
// Radix sort: 8-bit digits; per pass a tile of 4096 keys per CTA (8 warps x
// 16 rows x 32 lanes, row-major inside each warp's 512-key segment):
//   1. tile_hist: digit histogram of every tile, stored digit-major
//      ([digit][tile]), so one exclusive scan gives each (digit, tile) its
//      global base;
//   2. the scan;
//   3. tile_scatter: per-warp digit counts, a prefix over the warps, then
//      every key at base + (earlier warps) + (earlier rows of its warp) +
//      (lower lanes of its row with the same digit, __match_any_sync): a
//      stable scatter.
#include "common.cuh"
#include "sort.cuh"

namespace mckg {
namespace {

constexpr uint32_t RT = 256;            // threads per tile
constexpr uint32_t RW = RT / 32;        // warps
constexpr uint32_t RROWS = 16;          // rows of 32 keys per warp
constexpr uint32_t RTILE = RT * RROWS;  // keys per tile
constexpr uint32_t RBINS = 256;

__device__ __forceinline__ uint32_t digit(unsigned long long k, uint32_t shift) {
  return (uint32_t)(k >> shift) & (RBINS - 1);
}

__global__ void __launch_bounds__(RT) tile_hist_kernel(const unsigned long long* keys, uint64_t n, uint32_t shift,
                                                       uint32_t ntiles, uint32_t* hist) {
  __shared__ uint32_t h[RBINS];
  h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t t0 = (uint64_t)blockIdx.x * RTILE;
  for (uint32_t i = threadIdx.x; i < RTILE; i += RT) {
    const uint64_t g = t0 + i;
    if (g < n) atomicAdd(&h[digit(keys[g], shift)], 1u);
  }
  __syncthreads();
  hist[(size_t)threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];
}

__global__ void __launch_bounds__(RT) tile_scatter_kernel(const unsigned long long* in, unsigned long long* out,
                                                          uint64_t n, uint32_t shift, uint32_t ntiles,
                                                          const uint64_t* base) {
  __shared__ uint32_t wc[RW][RBINS];   // per-warp digit counts, then exclusive per-warp starts
  __shared__ uint64_t tb[RBINS];       // this tile's global base per digit
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  for (uint32_t i = threadIdx.x; i < RW * RBINS; i += RT) wc[i / RBINS][i % RBINS] = 0;
  tb[threadIdx.x] = base[(size_t)threadIdx.x * ntiles + blockIdx.x];
  __syncthreads();
  const uint64_t seg = (uint64_t)blockIdx.x * RTILE + (uint64_t)warp * (RROWS * 32);
  unsigned long long k[RROWS];
  uint32_t rank[RROWS];
#pragma unroll
  for (uint32_t r = 0; r < RROWS; ++r) {
    const uint64_t g = seg + r * 32 + lane;
    const bool in_range = g < n;
    k[r] = in_range ? in[g] : 0ull;
    const uint32_t d = in_range ? digit(k[r], shift) : RBINS + lane;  // out-of-range: unique dummies
    const uint32_t peers = __match_any_sync(0xFFFFFFFFu, d);
    const uint32_t before = __popc(peers & ((1u << lane) - 1u));
    uint32_t prior = 0;
    if (in_range) prior = wc[warp][d];  // keys of this digit in the warp's earlier rows
    __syncwarp();
    if (in_range && before == 0) wc[warp][d] = prior + __popc(peers);
    __syncwarp();
    rank[r] = prior + before;
  }
  __syncthreads();
  // exclusive prefix over the warps, per digit (thread = digit)
  {
    uint32_t acc = 0;
    for (uint32_t w = 0; w < RW; ++w) {
      const uint32_t c = wc[w][threadIdx.x];
      wc[w][threadIdx.x] = acc;
      acc += c;
    }
  }
  __syncthreads();
#pragma unroll
  for (uint32_t r = 0; r < RROWS; ++r) {
    const uint64_t g = seg + r * 32 + lane;
    if (g >= n) continue;
    const uint32_t d = digit(k[r], shift);
    out[tb[d] + wc[warp][d] + rank[r]] = k[r];
  }
}

// ---- exclusive scan of 32-bit counts into 64-bit offsets (three kernels) ----
constexpr uint32_t SCT = 1024;

__global__ void scan_reduce_kernel(const uint32_t* in, uint64_t n, uint64_t* tile_sum) {
  __shared__ uint64_t ws[32];
  const uint64_t i = (uint64_t)blockIdx.x * SCT + threadIdx.x;
  uint64_t v = i < n ? in[i] : 0u;
  for (int d = 16; d; d >>= 1) v += __shfl_down_sync(0xFFFFFFFFu, v, d);
  if ((threadIdx.x & 31u) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint64_t s = ws[threadIdx.x];
    for (int d = 16; d; d >>= 1) s += __shfl_down_sync(0xFFFFFFFFu, s, d);
    if (threadIdx.x == 0) tile_sum[blockIdx.x] = s;
  }
}

// in-place exclusive scan of n tile sums by one CTA
__global__ void scan_carry_kernel(uint64_t* sums, uint64_t n) {
  __shared__ uint64_t ws[32];
  __shared__ uint64_t carry;
  if (threadIdx.x == 0) carry = 0;
  for (uint64_t c0 = 0; c0 < n; c0 += SCT) {
    __syncthreads();
    const uint64_t i = c0 + threadIdx.x;
    const uint64_t v = i < n ? sums[i] : 0u;
    uint64_t x = v;
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, x, d);
      if ((threadIdx.x & 31u) >= (uint32_t)d) x += y;
    }
    if ((threadIdx.x & 31u) == 31u) ws[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      uint64_t w = ws[threadIdx.x];
      for (int d = 1; d < 32; d <<= 1) {
        const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, w, d);
        if (threadIdx.x >= (uint32_t)d) w += y;
      }
      ws[threadIdx.x] = w;
    }
    __syncthreads();
    const uint64_t excl = carry + (threadIdx.x >= 32 ? ws[(threadIdx.x >> 5) - 1] : 0u) + x - v;
    if (i < n) sums[i] = excl;
    __syncthreads();
    if (threadIdx.x == SCT - 1) carry = excl + v;
  }
}

__global__ void scan_fix_kernel(const uint32_t* in, uint64_t n, const uint64_t* tile_off, uint64_t* out) {
  __shared__ uint64_t ws[32];
  const uint64_t i = (uint64_t)blockIdx.x * SCT + threadIdx.x;
  const uint64_t v = i < n ? in[i] : 0u;
  uint64_t x = v;
  for (int d = 1; d < 32; d <<= 1) {
    const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, x, d);
    if ((threadIdx.x & 31u) >= (uint32_t)d) x += y;
  }
  if ((threadIdx.x & 31u) == 31u) ws[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    uint64_t w = ws[threadIdx.x];
    for (int d = 1; d < 32; d <<= 1) {
      const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, w, d);
      if (threadIdx.x >= (uint32_t)d) w += y;
    }
    ws[threadIdx.x] = w;
  }
  __syncthreads();
  const uint64_t excl = tile_off[blockIdx.x] + (threadIdx.x >= 32 ? ws[(threadIdx.x >> 5) - 1] : 0u) + x - v;
  if (i < n) out[i] = excl;
  if (i + 1 == n) out[n] = excl + v;
}

// flags of the first key of every run of equal keys (sorted input)
__global__ void head_flags_kernel(const unsigned long long* k, uint64_t n, uint32_t* f) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    f[i] = (i == 0 || k[i] != k[i - 1]) ? 1u : 0u;
}

__global__ void gather_keys_kernel(const unsigned long long* k, const uint32_t* f, const uint64_t* pos, uint64_t n,
                                   unsigned long long* out, unsigned long long* n_out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (f[i]) out[pos[i]] = k[i];
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_out = pos[n];
}

__global__ void gather_index_kernel(const uint8_t* f, const uint64_t* pos, uint64_t n, uint32_t first,
                                    uint32_t* out, uint32_t* n_out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (f[i]) out[pos[i]] = first + (uint32_t)i;
  if (blockIdx.x == 0 && threadIdx.x == 0) *n_out = (uint32_t)pos[n];
}

__global__ void u8_to_u32_kernel(const uint8_t* f, uint64_t n, uint32_t* o) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    o[i] = f[i] ? 1u : 0u;
}

uint32_t grid_of(uint64_t n) {
  const uint64_t want = (n + 255) / 256, cap = (uint64_t)sm_count() * 8;
  return (uint32_t)(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace

cudaError_t exclusive_scan_u32(const uint32_t* in, uint64_t n, uint64_t* out, cudaStream_t s, uint32_t* launches) {
  const uint64_t tiles = (n + SCT - 1) / SCT;
  PoolGuard pg(s);
  uint64_t* ts = nullptr;
  cudaError_t e = pg.alloc(&ts, (tiles ? tiles : 1) * sizeof(uint64_t));
  if (e != cudaSuccess) return e;
  if (n == 0) {
    e = cudaMemsetAsync(out, 0, sizeof(uint64_t), s);
  } else {
    scan_reduce_kernel<<<(uint32_t)tiles, SCT, 0, s>>>(in, n, ts);
    scan_carry_kernel<<<1, SCT, 0, s>>>(ts, tiles);
    scan_fix_kernel<<<(uint32_t)tiles, SCT, 0, s>>>(in, n, ts, out);
    e = cudaGetLastError();
    if (launches) *launches += 3;
  }
  return e;
}

cudaError_t radix_sort_u64(unsigned long long* keys, unsigned long long* tmp, uint64_t n, uint32_t bits,
                           cudaStream_t s, uint32_t* launches) {
  if (n < 2) return cudaSuccess;
  const uint32_t ntiles = (uint32_t)((n + RTILE - 1) / RTILE);
  PoolGuard pg(s);
  uint32_t* hist = nullptr;
  uint64_t* base = nullptr;
  cudaError_t e;
  if ((e = pg.alloc(&hist, (size_t)RBINS * ntiles * sizeof(uint32_t))) != cudaSuccess) return e;
  if ((e = pg.alloc(&base, ((size_t)RBINS * ntiles + 1) * sizeof(uint64_t))) != cudaSuccess) return e;
  unsigned long long *src = keys, *dst = tmp;
  uint32_t passes = 0;
  for (uint32_t shift = 0; shift < bits; shift += 8, ++passes) {
    tile_hist_kernel<<<ntiles, RT, 0, s>>>(src, n, shift, ntiles, hist);
    if ((e = exclusive_scan_u32(hist, (uint64_t)RBINS * ntiles, base, s, launches)) != cudaSuccess) break;
    tile_scatter_kernel<<<ntiles, RT, 0, s>>>(src, dst, n, shift, ntiles, base);
    if ((e = cudaGetLastError()) != cudaSuccess) break;
    if (launches) *launches += 2;
    unsigned long long* t = src;
    src = dst;
    dst = t;
  }
  if (e == cudaSuccess && src != keys) e = cudaMemcpyAsync(keys, src, n * sizeof(unsigned long long),
                                                           cudaMemcpyDeviceToDevice, s);
  return e;
}

cudaError_t unique_sorted_u64(const unsigned long long* sorted, uint64_t n, unsigned long long* out,
                              unsigned long long* n_out, cudaStream_t s, uint32_t* launches) {
  PoolGuard pg(s);
  uint32_t* f = nullptr;
  uint64_t* pos = nullptr;
  cudaError_t e;
  if ((e = pg.alloc(&f, (n ? n : 1) * sizeof(uint32_t))) != cudaSuccess) return e;
  if ((e = pg.alloc(&pos, (n + 1) * sizeof(uint64_t))) != cudaSuccess) return e;
  head_flags_kernel<<<grid_of(n), 256, 0, s>>>(sorted, n, f);
  if ((e = exclusive_scan_u32(f, n, pos, s, launches)) == cudaSuccess) {
    gather_keys_kernel<<<grid_of(n), 256, 0, s>>>(sorted, f, pos, n, out, n_out);
    e = cudaGetLastError();
    if (launches) *launches += 2;
  }
  return e;
}

cudaError_t select_flagged_index(const uint8_t* flags, uint64_t n, uint32_t first, uint32_t* out, uint32_t* n_out,
                                 cudaStream_t s, uint32_t* launches) {
  PoolGuard pg(s);
  uint32_t* f = nullptr;
  uint64_t* pos = nullptr;
  cudaError_t e;
  if ((e = pg.alloc(&f, (n ? n : 1) * sizeof(uint32_t))) != cudaSuccess) return e;
  if ((e = pg.alloc(&pos, (n + 1) * sizeof(uint64_t))) != cudaSuccess) return e;
  u8_to_u32_kernel<<<grid_of(n), 256, 0, s>>>(flags, n, f);
  if ((e = exclusive_scan_u32(f, n, pos, s, launches)) == cudaSuccess) {
    gather_index_kernel<<<grid_of(n), 256, 0, s>>>(flags, pos, n, first, out, n_out);
    e = cudaGetLastError();
    if (launches) *launches += 2;
  }
  return e;
}

}  // namespace mckg
