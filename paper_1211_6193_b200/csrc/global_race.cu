// global_race.cu -- K3/K6: cross-block global-memory race detection
// (BASELINE config 5; not a reference
// interface -- see include/mckg.h).
//
// Multi-GPU dataflow (paper_1211_6193_b200/global_race.py drives it):
//   1. every rank holds the records of its shard of simulated blocks;
//   2. K3 `mckg_partition_global` buckets them by owner rank (address-range
//      partition: GPU g owns [g*A/P, (g+1)*A/P)), counts first;
//   3. the buckets travel with one NCCL all-to-all(v) over NVLink;
//   4. K6 `mckg_detect_global` on each rank: every record is expanded into the
//      4-byte words it touches, (word, record) pairs are radix-sorted by word
//      (CUB), and one thread per pair scans its word's run: X races on the
//      bytes it shares with an EARLIER (sweep, bid, tid) access Y of ANOTHER
//      BLOCK where X or Y writes (racecheck.cpp:24-32 with thread -> block).
//      Racing (byte, line) keys are appended, then sorted + uniqued; the first
//      racing timestamp per line is min-reduced per CTA, then globally.
#include <cub/cub.cuh>

#include "common.cuh"

namespace mckg {
namespace {

__device__ __forceinline__ unsigned long long sm64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t ga_addr(uint64_t a) { return a & 0xFFFFFFFFFFull; }
__device__ __forceinline__ uint32_t ga_len(uint64_t a) { return (uint32_t)((a >> 40) & 0xFu); }
__device__ __forceinline__ uint32_t ga_write(uint64_t a) { return (uint32_t)((a >> 44) & 1u); }
__device__ __forceinline__ uint32_t ga_tid(uint64_t a) { return (uint32_t)((a >> 45) & 0x7FFu); }
__device__ __forceinline__ int32_t ga_line(uint64_t a, uint32_t b) {
  return (int32_t)(((b >> 24) << 8) | (uint32_t)((a >> 56) & 0xFFu));
}

__global__ void gen_c5_kernel(mckg_gaccess* ev, uint32_t blk0, uint32_t n_blocks, uint32_t n_total,
                              unsigned long long seed) {
  const unsigned long long per = MCKG_C5_EVENTS_PER_BLOCK;
  const unsigned long long total = (unsigned long long)n_blocks * per;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long r = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; r < total; r += stride) {
    const unsigned long long i = (unsigned long long)blk0 * per + r;
    const uint32_t b = (uint32_t)(i / per), j = (uint32_t)(i % per);
    const uint32_t tid = j % 256u, k = j / 256u;
    const unsigned long long h = sm64(seed + i);
    const uint32_t write = (uint32_t)(h & 1u);
    const bool redirect = ((h >> 32) % 10000u) < 100u;
    const uint32_t tb = redirect ? (b + 1u) % n_total : b;
    const uint64_t addr = (uint64_t)tb * MCKG_C5_RANGE + (uint64_t)(tid * 16u + k) * 8u;
    const int32_t line = 200 + (int32_t)(k % 4u);
    mckg_gaccess g;
    g.a = (addr & 0xFFFFFFFFFFull) | (4ull << 40) | ((unsigned long long)write << 44) |
          ((unsigned long long)tid << 45) | ((unsigned long long)((uint32_t)line & 0xFFu) << 56);
    g.sweep = k;
    g.b = (b & 0xFFFFFFu) | ((((uint32_t)line >> 8) & 0xFFu) << 24);
    ev[r] = g;
  }
}

// ---- K3: owner partition ----
__device__ __forceinline__ uint32_t owner_of(uint64_t a, uint32_t P, unsigned long long space) {
  const uint32_t o = (uint32_t)((ga_addr(a) * P) / space);
  return o < P ? o : P - 1;
}

constexpr uint32_t TILE = 4096;  // records per scatter tile (256 threads x 16)

__global__ void owner_hist_kernel(const mckg_gaccess* ev, uint64_t n, uint32_t P, unsigned long long space,
                                  unsigned long long* counts) {
  __shared__ unsigned int h[64];
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u;
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x; i0 < n; i0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    const uint32_t o = i < n ? owner_of(ev[i].a, P, space) : 0xFFFFFFFFu;
    const uint32_t grp = __match_any_sync(0xFFFFFFFFu, o);  // warp-aggregated
    if (o != 0xFFFFFFFFu && lane == (uint32_t)(__ffs(grp) - 1)) atomicAdd(&h[o], (unsigned)__popc(grp));
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < P; i += blockDim.x)
    if (h[i]) atomicAdd(counts + i, (unsigned long long)h[i]);
}

// One tile of TILE records per CTA iteration: per-owner tile counts in shared
// memory (warp-aggregated), one global reservation per (tile, owner), then
// every record lands at base + its rank inside the tile.
__global__ void owner_scatter_kernel(const mckg_gaccess* ev, uint64_t n, uint32_t P, unsigned long long space,
                                     const unsigned long long* counts, unsigned long long* cursor,
                                     mckg_gaccess* out) {
  __shared__ unsigned long long base[64];
  __shared__ unsigned long long tbase[64];
  __shared__ unsigned int tcnt[64];
  if (threadIdx.x == 0) {
    unsigned long long s = 0;
    for (uint32_t r = 0; r < P; ++r) {
      base[r] = s;
      s += counts[r];
    }
  }
  const uint32_t lane = threadIdx.x & 31u;
  constexpr uint32_t PER = TILE / 256;
  for (uint64_t t0 = blockIdx.x * (uint64_t)TILE; t0 < n; t0 += (uint64_t)gridDim.x * TILE) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) tcnt[i] = 0;
    __syncthreads();
    uint32_t o[PER], pos[PER];
#pragma unroll
    for (uint32_t k = 0; k < PER; ++k) {
      const uint64_t i = t0 + (uint64_t)k * 256 + threadIdx.x;
      o[k] = i < n ? owner_of(ev[i].a, P, space) : 0xFFFFFFFFu;
      const uint32_t grp = __match_any_sync(0xFFFFFFFFu, o[k]);
      const int leader = __ffs(grp) - 1;
      uint32_t b = 0;
      if (o[k] != 0xFFFFFFFFu && lane == (uint32_t)leader) b = atomicAdd(&tcnt[o[k]], (unsigned)__popc(grp));
      b = __shfl_sync(0xFFFFFFFFu, b, leader);
      pos[k] = b + __popc(grp & ((1u << lane) - 1u));
    }
    __syncthreads();
    for (uint32_t r = threadIdx.x; r < P; r += blockDim.x)
      tbase[r] = tcnt[r] ? atomicAdd(cursor + r, (unsigned long long)tcnt[r]) : 0ull;
    __syncthreads();
#pragma unroll
    for (uint32_t k = 0; k < PER; ++k) {
      const uint64_t i = t0 + (uint64_t)k * 256 + threadIdx.x;
      if (i < n) out[base[o[k]] + tbase[o[k]] + pos[k]] = ev[i];
    }
  }
}

// ---- K6: detection ----
__device__ __forceinline__ uint32_t words_of(uint64_t a) {
  const uint64_t addr = ga_addr(a);
  const uint32_t len = ga_len(a);
  if (len == 0) return 0;
  return (uint32_t)(((addr + len - 1) >> 2) - (addr >> 2) + 1);
}

__global__ void word_count_kernel(const mckg_gaccess* ev, uint64_t n, uint32_t* nw) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    nw[i] = words_of(ev[i].a);
}

__global__ void word_emit_kernel(const mckg_gaccess* ev, uint64_t n, const uint32_t* off, uint64_t addr_lo,
                                 unsigned long long* keys, uint32_t* vals) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t a = ev[i].a;
    const uint32_t k = words_of(a);
    const uint64_t w0 = (ga_addr(a) - addr_lo) >> 2;
    for (uint32_t q = 0; q < k; ++q) {
      keys[off[i] + q] = w0 + q;
      vals[off[i] + q] = (uint32_t)i;
    }
  }
}

constexpr uint32_t LT = 64;

__global__ void scan_runs_kernel(const mckg_gaccess* ev, const unsigned long long* keys, const uint32_t* vals,
                                 uint64_t m, uint64_t addr_lo, unsigned long long* out, unsigned long long cap,
                                 unsigned long long* n_out, unsigned long long* line_first, uint32_t* status) {
  __shared__ uint32_t s_line[LT];
  __shared__ unsigned long long s_ts[LT];
  for (uint32_t i = threadIdx.x; i < LT; i += blockDim.x) {
    s_line[i] = 0xFFFFFFFFu;
    s_ts[i] = ~0ull;
  }
  __syncthreads();
  for (uint64_t e0 = blockIdx.x * (uint64_t)blockDim.x; e0 < m; e0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = e0 + threadIdx.x;
    if (e < m) {
      const unsigned long long w = keys[e];
      // a word touched by one access only cannot race: skip without loading
      const bool single = (e == 0 || keys[e - 1] != w) && (e + 1 >= m || keys[e + 1] != w);
      if (single) continue;
      const mckg_gaccess X = ev[vals[e]];
      const uint32_t xbid = X.b & 0xFFFFFFu, xtid = ga_tid(X.a);
      const unsigned long long xts = ts_key(X.sweep, xbid, xtid);
      const bool xw = ga_write(X.a);
      const uint64_t wb = addr_lo + (w << 2);  // byte address of the word
      const uint64_t xa = ga_addr(X.a);
      // X's bytes inside this word, as a 4-bit mask
      const uint64_t lo = xa > wb ? xa : wb, hi = (xa + ga_len(X.a)) < wb + 4 ? (xa + ga_len(X.a)) : wb + 4;
      const uint32_t xm = ((1u << (uint32_t)(hi - lo)) - 1u) << (uint32_t)(lo - wb);
      uint32_t raced = 0;
      // the run of this word: walk both directions
      for (int dir = -1; dir <= 1; dir += 2) {
        for (uint64_t f = e + dir; f < m && (raced & xm) != xm; f += dir) {
          if (keys[f] != w) break;
          const mckg_gaccess Y = ev[vals[f]];
          const uint32_t ybid = Y.b & 0xFFFFFFu;
          if (ybid == xbid || !(xw || ga_write(Y.a))) continue;
          if (ts_key(Y.sweep, ybid, ga_tid(Y.a)) >= xts) continue;
          const uint64_t ya = ga_addr(Y.a);
          const uint64_t ylo = ya > wb ? ya : wb, yhi = (ya + ga_len(Y.a)) < wb + 4 ? (ya + ga_len(Y.a)) : wb + 4;
          if (ylo >= yhi) continue;
          raced |= (((1u << (uint32_t)(yhi - ylo)) - 1u) << (uint32_t)(ylo - wb)) & xm;
        }
      }
      if (raced) {
        const int32_t line = ga_line(X.a, X.b);
        for (uint32_t q = 0; q < 4; ++q) {
          if (!((raced >> q) & 1u)) continue;
          const unsigned long long i = atomicAdd(n_out, 1ull);
          if (i < cap)
            out[i] = ((unsigned long long)((wb + q) & 0xFFFFFFFFFFull) << 16) | ((uint32_t)line & 0xFFFFu);
          else
            atomicOr(status, (uint32_t)MCKG_ST_OVERFLOW);
        }
        if ((uint32_t)line < MCKG_MAX_LINES) {
          uint32_t h = (uint32_t)line & (LT - 1);
          bool done = false;
          for (uint32_t p = 0; p < LT && !done; ++p) {
            uint32_t v = s_line[h];
            if (v == 0xFFFFFFFFu) {
              const uint32_t old = atomicCAS(s_line + h, 0xFFFFFFFFu, (uint32_t)line);
              v = old == 0xFFFFFFFFu ? (uint32_t)line : old;
            }
            if (v == (uint32_t)line) {
              atomicMin(s_ts + h, xts);
              done = true;
            }
            h = (h + 1) & (LT - 1);
          }
          if (!done) atomicMin(line_first + line, xts);
        } else {
          atomicOr(status, (uint32_t)MCKG_ST_RANGE);
        }
      }
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < LT; i += blockDim.x)
    if (s_line[i] != 0xFFFFFFFFu) atomicMin(line_first + s_line[i], s_ts[i]);
}

__global__ void decode_races_kernel(const unsigned long long* k, const unsigned long long* n_dev,
                                    mckg_grace* out, uint64_t cap) {
  const uint64_t n = *n_dev;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n && i < cap;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long v = k[i];
    out[i] = mckg_grace{v >> 16, (int32_t)(v & 0xFFFFu), 0};
  }
}

uint32_t grid_for(uint64_t n, uint32_t per_sm = 8) {
  const uint64_t want = (n + 255) / 256;
  const uint64_t cap = (uint64_t)sm_count() * per_sm;
  return (uint32_t)(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace
}  // namespace mckg

using namespace mckg;

extern "C" int mckg_gen_c5(mckg_gaccess* events, uint32_t blk0, uint32_t n_blocks, uint32_t n_total,
                           uint64_t seed, void* stream) {
  if (!events || n_total == 0) {
    set_error("mckg_gen_c5: null buffer or empty grid");
    return MCKG_E_ARG;
  }
  const uint32_t grid = (uint32_t)sm_count() * 8u;
  gen_c5_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(events, blk0, n_blocks, n_total, seed);
  MCKG_CUDA_TRY(cudaGetLastError());
  note_launch(1, grid, 256, 0);
  return MCKG_OK;
}

extern "C" int mckg_partition_global(const mckg_gaccess* events, uint64_t n, uint32_t n_ranks,
                                     uint64_t addr_space, mckg_gaccess* out, uint64_t* counts, void* stream) {
  if ((!events && n) || (!out && n) || !counts || n_ranks == 0 || n_ranks > 64 || addr_space == 0) {
    set_error("mckg_partition_global: bad argument");
    return MCKG_E_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  keep_pool_memory();
  unsigned long long* cursor = nullptr;
  MCKG_CUDA_TRY(cudaMemsetAsync(counts, 0, n_ranks * sizeof(uint64_t), s));
  MCKG_CUDA_TRY(cudaMallocAsync(&cursor, n_ranks * sizeof(unsigned long long), s));
  MCKG_CUDA_TRY(cudaMemsetAsync(cursor, 0, n_ranks * sizeof(unsigned long long), s));
  if (n) {
    const uint32_t g = grid_for(n);
    owner_hist_kernel<<<g, 256, 0, s>>>(events, n, n_ranks, addr_space, (unsigned long long*)counts);
    const uint64_t tiles = (n + TILE - 1) / TILE;
    const uint32_t gs = (uint32_t)(tiles < (uint64_t)sm_count() * 8 ? tiles : (uint64_t)sm_count() * 8);
    owner_scatter_kernel<<<gs, 256, 0, s>>>(events, n, n_ranks, addr_space, (const unsigned long long*)counts,
                                            cursor, out);
    MCKG_CUDA_TRY(cudaGetLastError());
  }
  cudaFreeAsync(cursor, s);
  add_launches(2);
  return MCKG_OK;
}

extern "C" int mckg_detect_global(const mckg_gaccess* events, uint64_t n, uint64_t addr_lo, mckg_grace* races,
                                  uint64_t capacity, unsigned long long* n_races, unsigned long long* line_first,
                                  uint32_t* status, void* stream) {
  if ((!events && n) || !n_races || !line_first || !status || (!races && capacity)) {
    set_error("mckg_detect_global: null argument");
    return MCKG_E_ARG;
  }
  if (n >= (1ull << 32)) {
    set_error("mckg_detect_global: more than 2^32 records on one rank");
    return MCKG_E_RANGE;
  }
  cudaStream_t s = (cudaStream_t)stream;
  keep_pool_memory();
  MCKG_CUDA_TRY(cudaMemsetAsync(n_races, 0, sizeof(unsigned long long), s));
  if (n == 0) return MCKG_OK;
  uint32_t *nw = nullptr, *off = nullptr, *vals = nullptr, *vals2 = nullptr;
  unsigned long long *keys = nullptr, *keys2 = nullptr, *tmp_keys = nullptr, *uniq = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0, t2 = 0;
  uint32_t m32 = 0;
  const uint32_t g = grid_for(n);
  MCKG_CUDA_TRY(cudaMallocAsync(&nw, n * sizeof(uint32_t), s));
  MCKG_CUDA_TRY(cudaMallocAsync(&off, (n + 1) * sizeof(uint32_t), s));
  word_count_kernel<<<g, 256, 0, s>>>(events, n, nw);
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, nw, off, (int64_t)n + 0, s);
  MCKG_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, s));
  MCKG_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, nw, off, (int64_t)n, s));
  cudaFreeAsync(tmp, s);
  // total word entries m = off[n-1] + nw[n-1]
  uint32_t last[2];
  MCKG_CUDA_TRY(cudaMemcpyAsync(&last[0], off + (n - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  MCKG_CUDA_TRY(cudaMemcpyAsync(&last[1], nw + (n - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
  MCKG_CUDA_TRY(cudaStreamSynchronize(s));
  m32 = last[0] + last[1];
  const uint64_t m = m32;
  MCKG_CUDA_TRY(cudaMallocAsync(&keys, m * sizeof(unsigned long long), s));
  MCKG_CUDA_TRY(cudaMallocAsync(&keys2, m * sizeof(unsigned long long), s));
  MCKG_CUDA_TRY(cudaMallocAsync(&vals, m * sizeof(uint32_t), s));
  MCKG_CUDA_TRY(cudaMallocAsync(&vals2, m * sizeof(uint32_t), s));
  word_emit_kernel<<<g, 256, 0, s>>>(events, n, off, addr_lo, keys, vals);
  // word index < 2^38 (40-bit byte addresses)
  tmp_bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys, keys2, vals, vals2, (int64_t)m, 0, 38, s);
  MCKG_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, s));
  MCKG_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys, keys2, vals, vals2, (int64_t)m, 0, 38, s));
  cudaFreeAsync(tmp, s);
  // racing (byte, line) keys: at most 4 per word entry; capacity m/8 + 1M
  const unsigned long long cap = m / 8 + (1ull << 20);
  MCKG_CUDA_TRY(cudaMallocAsync(&tmp_keys, cap * sizeof(unsigned long long), s));
  unsigned long long* n_raw = nullptr;
  MCKG_CUDA_TRY(cudaMallocAsync(&n_raw, sizeof(unsigned long long), s));
  MCKG_CUDA_TRY(cudaMemsetAsync(n_raw, 0, sizeof(unsigned long long), s));
  scan_runs_kernel<<<grid_for(m), 256, 0, s>>>(events, keys2, vals2, m, addr_lo, tmp_keys, cap, n_raw, line_first,
                                               status);
  MCKG_CUDA_TRY(cudaGetLastError());
  unsigned long long nr = 0;
  MCKG_CUDA_TRY(cudaMemcpyAsync(&nr, n_raw, sizeof nr, cudaMemcpyDeviceToHost, s));
  MCKG_CUDA_TRY(cudaStreamSynchronize(s));
  if (nr > cap) nr = cap;
  if (nr) {
    MCKG_CUDA_TRY(cudaMallocAsync(&uniq, nr * sizeof(unsigned long long), s));
    tmp_bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, tmp_keys, uniq, (int64_t)nr, 0, 56, s);
    cub::DeviceSelect::Unique(nullptr, t2, uniq, tmp_keys, n_races, (int64_t)nr, s);
    tmp_bytes = tmp_bytes > t2 ? tmp_bytes : t2;
    MCKG_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, s));
    MCKG_CUDA_TRY(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, tmp_keys, uniq, (int64_t)nr, 0, 56, s));
    MCKG_CUDA_TRY(cub::DeviceSelect::Unique(tmp, tmp_bytes, uniq, tmp_keys, n_races, (int64_t)nr, s));
    cudaFreeAsync(tmp, s);
    if (capacity) decode_races_kernel<<<grid_for(nr), 256, 0, s>>>(tmp_keys, n_races, races, capacity);
    MCKG_CUDA_TRY(cudaGetLastError());
    cudaFreeAsync(uniq, s);
  }
  cudaFreeAsync(n_raw, s);
  cudaFreeAsync(tmp_keys, s);
  cudaFreeAsync(nw, s);
  cudaFreeAsync(off, s);
  cudaFreeAsync(keys, s);
  cudaFreeAsync(keys2, s);
  cudaFreeAsync(vals, s);
  cudaFreeAsync(vals2, s);
  add_launches(8);
  return MCKG_OK;
}
