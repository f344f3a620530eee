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
#include <vector>

#include "common.cuh"
#include "sort.cuh"

namespace mckg {
namespace {

__device__ __forceinline__ unsigned long long sm64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ uint64_t ga_addr(uint64_t a) { return a & 0xFFFFFFFFFFull; }
// a record's address word from its 16-byte image
__device__ __forceinline__ unsigned long long rec_a(const uint4& r) {
  return ((unsigned long long)r.y << 32) | r.x;
}
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

// ---- K6: detection (bucket partition + per-bucket filter and exact pass) ----
//
// Semantics (oracle/global_detector.c): records in timestamp order (sweep,
// bid, tid); X races on byte b iff X writes and an earlier access to b came
// from another block, or X reads and an earlier write to b came from another
// block (racecheck.cpp:24-32 with "thread" replaced by "block").  Per byte
// this needs only four minima over the timestamp keys, which embed the
// block: f1 = the earliest access, f2 = the earliest access from a block
// other than f1's, and w1 / w2 likewise over the writes.  X (block B, key t)
// then has an earlier access from another block iff (blk(f1) != B) or
// (f2 < t), and an earlier write from another block iff (blk(w1) != B and
// w1 < t) or (blk(w1) == B and w2 < t) -- no sort, no order of arrival.
//
// Dataflow, all hand-written:
//   1. the address span is estimated from a strided sample; buckets are
//      2^shift-byte address ranges sized for ~256 records;
//   2. bucket_count: a record counts in every bucket its bytes touch
//      (warp-aggregated atomics);
//   3. an exclusive scan of the counts (scan_* kernels);
//   4. bucket_scatter: re-read, write each record into its bucket(s);
//   5. bucket_detect, one CTA per bucket, tables in shared memory:
//      P1/P2/P3 the word filter of K2 (some accessing block per word, then
//      "a second block" and "a write" stamps) -> candidates; E1-E3 the four
//      per-byte minima over the candidates' bytes (any Y that X can race
//      with is a candidate too) -> racing (byte, line) pairs, deduplicated
//      per bucket (a byte lives in one bucket); first racing key per line.
//      A bucket beyond the shared-memory tables is redone by the same code
//      with tables in global memory sized for it (bucket_detect_big).
constexpr uint32_t BT = 256;      // threads per detect CTA
constexpr uint32_t BCAP = 1024;   // records of a shared-memory bucket
constexpr uint32_t BWS = 2048;    // word-table slots (shared)
constexpr uint32_t BCC = 128;     // candidates (shared)
constexpr uint32_t BBS = 512;     // candidate-byte slots (shared)
constexpr uint32_t BDS = 512;     // reported (byte, line) slots (shared)
constexpr uint32_t BLT = 32;      // line-first cache entries
constexpr unsigned long long KEMPTY = 0ull;
constexpr unsigned long long TSMAX = ~0ull;

__device__ __forceinline__ uint32_t ts_bid(unsigned long long ts) {
  return (uint32_t)(ts >> 11) & (MCKG_MAX_BID - 1);
}
__device__ __forceinline__ unsigned long long ga_ts(const mckg_gaccess& r) {
  return ts_key(r.sweep, r.b & 0xFFFFFFu, ga_tid(r.a));
}
__device__ __forceinline__ uint32_t hash64(unsigned long long k, uint32_t mask) {
  return (uint32_t)((k * 0x9E3779B97F4A7C15ull) >> 40) & mask;
}

// The tables of one bucket (shared memory or global memory).
struct BTab {
  unsigned long long* wkey;  // stamp << 41 | word address + 1
  uint32_t* wtag;            // some accessing block
  uint32_t* wflag;           // {second-block stamp u16, write stamp u16}
  uint32_t wmask;
  uint32_t* cand;            // candidate record indices
  uint32_t ccap;
  unsigned long long* bkey;  // stamp << 41 | byte address + 1
  unsigned long long* bmin;  // [4 * slots]: f1, f2, w1, w2
  uint32_t bmask;
  unsigned long long* dkey;  // reported (byte, line): stamp << 56 | (byte & 2^40-1) << 16 | line
  uint32_t dmask;
};

// open-addressing insert / find; keys carry the bucket stamp, so keys of
// other stamps read as empty.  Returns the slot, or ~0u when full.
__device__ __forceinline__ uint32_t tab_insert(unsigned long long* keys, uint32_t mask, unsigned long long key,
                                               uint32_t stamp_shift, bool* claimed) {
  const unsigned long long st = key >> stamp_shift;
  uint32_t h = hash64(key, mask);
  *claimed = false;
  for (uint32_t p = 0; p <= mask; ++p) {
    unsigned long long cur = keys[h];
    while ((cur >> stamp_shift) != st) {  // stale or empty: claim it
      const unsigned long long old = atomicCAS(keys + h, cur, key);
      if (old == cur) {
        *claimed = true;
        return h;
      }
      cur = old;
    }
    if (cur == key) return h;
    h = (h + 1) & mask;
  }
  return ~0u;
}

__device__ __forceinline__ uint32_t tab_find(const unsigned long long* keys, uint32_t mask, unsigned long long key) {
  uint32_t h = hash64(key, mask);
  for (uint32_t p = 0; p <= mask; ++p) {
    const unsigned long long cur = keys[h];
    if (cur == key) return h;
    h = (h + 1) & mask;
  }
  return ~0u;
}

struct BOut {
  mckg_grace* races;
  unsigned long long cap;
  unsigned long long* n;
  unsigned long long* line_first;
  uint32_t* status;
};

// One bucket [blo, bhi) of m records at R, by the CTA.  Returns false (all
// threads) when the tables overflow: the caller redoes the bucket with
// bigger ones.  stamp: 1..2^23, unique per bucket processed by this CTA.
__device__ bool detect_bucket(const mckg_gaccess* R, uint32_t m, uint64_t blo, uint64_t bhi, const BTab& T,
                              uint32_t stamp, const BOut& O, uint32_t* s_line, unsigned long long* s_lts,
                              uint32_t* s_cnt, uint32_t* s_flag) {
  const uint32_t t = threadIdx.x;
  const unsigned long long sk = (unsigned long long)stamp << 41;
  const uint32_t st16 = stamp & 0xFFFFu ? stamp & 0xFFFFu : 1u;
  if (t == 0) {
    s_cnt[0] = 0;
    *s_flag = 0;
  }
  __syncthreads();
  // P1: claim a slot per touched word, store some accessing block
  for (uint32_t i = t; i < m; i += blockDim.x) {
    const mckg_gaccess r = R[i];
    const uint64_t a = ga_addr(r.a);
    const uint32_t len = ga_len(r.a);
    const uint64_t b0 = a > blo ? a : blo, b1 = (a + len) < bhi ? (a + len) : bhi;
    for (uint64_t w = b0 >> 2; (w << 2) < b1; ++w) {
      bool cl;
      const uint32_t h = tab_insert(T.wkey, T.wmask, sk | (w + 1), 41, &cl);
      if (h == ~0u) {
        *s_flag = 1;
        break;
      }
      if (cl) T.wflag[h] = 0u;
      T.wtag[h] = r.b & 0xFFFFFFu;
    }
  }
  __syncthreads();
  if (*s_flag) return false;
  // P2: words touched by a second block; written words
  for (uint32_t i = t; i < m; i += blockDim.x) {
    const mckg_gaccess r = R[i];
    const uint64_t a = ga_addr(r.a);
    const uint32_t len = ga_len(r.a), bid = r.b & 0xFFFFFFu;
    const bool wr = ga_write(r.a);
    const uint64_t b0 = a > blo ? a : blo, b1 = (a + len) < bhi ? (a + len) : bhi;
    for (uint64_t w = b0 >> 2; (w << 2) < b1; ++w) {
      const uint32_t h = tab_find(T.wkey, T.wmask, sk | (w + 1));
      uint16_t* f = reinterpret_cast<uint16_t*>(T.wflag + h);
      if (T.wtag[h] != bid) f[0] = (uint16_t)st16;
      if (wr) f[1] = (uint16_t)st16;
    }
  }
  __syncthreads();
  // P3: candidates = records with a word touched by two blocks and written
  for (uint32_t i = t; i < m; i += blockDim.x) {
    const mckg_gaccess r = R[i];
    const uint64_t a = ga_addr(r.a);
    const uint32_t len = ga_len(r.a);
    const uint64_t b0 = a > blo ? a : blo, b1 = (a + len) < bhi ? (a + len) : bhi;
    bool c = false;
    for (uint64_t w = b0 >> 2; (w << 2) < b1; ++w)
      c |= T.wflag[tab_find(T.wkey, T.wmask, sk | (w + 1))] == (st16 | (st16 << 16));
    if (c) {
      const uint32_t k = atomicAdd(s_cnt, 1u);
      if (k < T.ccap) T.cand[k] = i; else *s_flag = 1;
    }
  }
  __syncthreads();
  if (*s_flag) return false;
  const uint32_t nc = s_cnt[0];
  if (nc == 0) return true;
  // E1: claim the candidates' bytes, initialise their minima
  for (uint32_t q = t; q < nc * 8u; q += blockDim.x) {
    const mckg_gaccess r = R[T.cand[q >> 3]];
    const uint64_t a = ga_addr(r.a) + (q & 7u);
    if ((q & 7u) >= ga_len(r.a) || a < blo || a >= bhi) continue;
    bool cl;
    const uint32_t h = tab_insert(T.bkey, T.bmask, sk | (a + 1), 41, &cl);
    if (h == ~0u) {
      *s_flag = 1;
      continue;
    }
    if (cl) {
      T.bmin[4 * h] = TSMAX;
      T.bmin[4 * h + 1] = TSMAX;
      T.bmin[4 * h + 2] = TSMAX;
      T.bmin[4 * h + 3] = TSMAX;
    }
  }
  __syncthreads();
  if (*s_flag) return false;
  // E2: f1 / w1, then E3: f2 / w2 (another block than f1's / w1's)
  for (int pass = 0; pass < 2; ++pass) {
    for (uint32_t q = t; q < nc * 8u; q += blockDim.x) {
      const mckg_gaccess r = R[T.cand[q >> 3]];
      const uint64_t a = ga_addr(r.a) + (q & 7u);
      if ((q & 7u) >= ga_len(r.a) || a < blo || a >= bhi) continue;
      const uint32_t h = tab_find(T.bkey, T.bmask, sk | (a + 1));
      const unsigned long long ts = ga_ts(r);
      const bool wr = ga_write(r.a);
      unsigned long long* mn = T.bmin + 4 * h;
      if (pass == 0) {
        atomicMin(mn, ts);
        if (wr) atomicMin(mn + 2, ts);
      } else {
        const uint32_t bid = r.b & 0xFFFFFFu;
        if (ts_bid(mn[0]) != bid) atomicMin(mn + 1, ts);
        if (wr && ts_bid(mn[2]) != bid) atomicMin(mn + 3, ts);
      }
    }
    __syncthreads();
  }
  // E4: racing bytes -> (byte, line) once per bucket; first key per line
  for (uint32_t q = t; q < nc * 8u; q += blockDim.x) {
    const mckg_gaccess r = R[T.cand[q >> 3]];
    const uint64_t a = ga_addr(r.a) + (q & 7u);
    if ((q & 7u) >= ga_len(r.a) || a < blo || a >= bhi) continue;
    const unsigned long long* mn = T.bmin + 4 * tab_find(T.bkey, T.bmask, sk | (a + 1));
    const unsigned long long ts = ga_ts(r);
    const uint32_t bid = r.b & 0xFFFFFFu;
    bool race;
    if (ga_write(r.a))
      race = ts_bid(mn[0]) != bid || mn[1] < ts;
    else
      race = (mn[2] != TSMAX && ts_bid(mn[2]) != bid && mn[2] < ts) || (ts_bid(mn[2]) == bid && mn[3] < ts);
    if (!race) continue;
    const int32_t line = ga_line(r.a, r.b);
    const unsigned long long dk =
        ((unsigned long long)(stamp & 0xFFu) << 56) | ((a & 0xFFFFFFFFFFull) << 16) | ((uint32_t)line & 0xFFFFu);
    bool fresh;
    // dedup keys: stamp in the top 8 bits (bucket-local tables; 0 = empty)
    const uint32_t h = tab_insert(T.dkey, T.dmask, dk, 56, &fresh);
    if (h == ~0u) {
      atomicOr(O.status, (uint32_t)MCKG_ST_DUP);
      fresh = true;
    }
    if (fresh) {
      const unsigned long long k = atomicAdd(O.n, 1ull);
      if (k < O.cap)
        O.races[k] = mckg_grace{a, line, 0};
      else
        atomicOr(O.status, (uint32_t)MCKG_ST_OVERFLOW);
    }
    // first racing key of the line: a CTA cache, global atomicMin otherwise
    const uint32_t l = (uint32_t)line;
    uint32_t hh = l & (BLT - 1);
    bool done = false;
    for (uint32_t p = 0; p < BLT && !done; ++p) {
      uint32_t v = s_line[hh];
      if (v == 0xFFFFFFFFu) {
        const uint32_t old = atomicCAS(s_line + hh, 0xFFFFFFFFu, l);
        v = old == 0xFFFFFFFFu ? l : old;
      }
      if (v == l) {
        atomicMin(s_lts + hh, ts);
        done = true;
      }
      hh = (hh + 1) & (BLT - 1);
    }
    if (!done) atomicMin(O.line_first + l, ts);
  }
  __syncthreads();
  return true;
}

// bucket b's byte range under the sampled span (edge buckets are open)
__device__ __forceinline__ void bucket_range(uint32_t b, uint32_t nb, uint32_t shift, uint64_t base, uint64_t* lo,
                                             uint64_t* hi) {
  *lo = b == 0 ? 0ull : base + ((uint64_t)b << shift);
  *hi = b + 1 >= nb ? ~0ull : base + ((uint64_t)(b + 1) << shift);
}

__device__ __forceinline__ uint32_t bucket_of(uint64_t a, uint32_t nb, uint32_t shift, uint64_t base) {
  if (a < base) return 0;
  const uint64_t q = (a - base) >> shift;
  return q >= nb ? nb - 1 : (uint32_t)q;
}

// min / max address over one record per stride-sized window, at a hashed
// position inside the window (a fixed position can alias the input's period)
__global__ void span_sample_kernel(const mckg_gaccess* ev, uint64_t n, uint64_t stride, unsigned long long* mm) {
  unsigned long long lo = ~0ull, hi = 0;
  for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w * stride < n;
       w += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t i = w * stride + sm64(w) % stride;
    if (i >= n) i = n - 1;
    const uint64_t a = ga_addr(ev[i].a);
    lo = a < lo ? a : lo;
    hi = a > hi ? a : hi;
  }
  // one atomic pair per warp (a single address hit by every thread serialises)
  for (int d = 16; d; d >>= 1) {
    const unsigned long long l = __shfl_xor_sync(0xFFFFFFFFu, lo, d), h = __shfl_xor_sync(0xFFFFFFFFu, hi, d);
    lo = l < lo ? l : lo;
    hi = h > hi ? h : hi;
  }
  if ((threadIdx.x & 31u) == 0) {
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
  }
}

__global__ void bucket_count_kernel(const mckg_gaccess* ev, uint64_t n, uint32_t nb, uint32_t shift, uint64_t base,
                                    uint32_t* cnt, uint32_t* status) {
  const uint32_t lane = threadIdx.x & 31u;
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x; i0 < n; i0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    uint32_t b0 = 0xFFFFFFFFu, b1 = 0xFFFFFFFFu;
    if (i < n) {
      const mckg_gaccess r = ev[i];
      const uint32_t len = ga_len(r.a);
      if ((r.b & 0xFFFFFFu) >= MCKG_MAX_BID || len - 1u >= MCKG_MAX_LEN) {
        atomicOr(status, (uint32_t)MCKG_ST_RANGE);
      } else {
        const uint64_t a = ga_addr(r.a);
        b0 = bucket_of(a, nb, shift, base);
        const uint32_t bl = bucket_of(a + len - 1u, nb, shift, base);
        if (bl != b0) b1 = bl;
      }
    }
    uint32_t g = __match_any_sync(0xFFFFFFFFu, b0);
    if (b0 != 0xFFFFFFFFu && lane == (uint32_t)(__ffs(g) - 1)) atomicAdd(cnt + b0, (uint32_t)__popc(g));
    if (__any_sync(0xFFFFFFFFu, b1 != 0xFFFFFFFFu) && b1 != 0xFFFFFFFFu) atomicAdd(cnt + b1, 1u);
  }
}

__global__ void bucket_scatter_kernel(const mckg_gaccess* ev, uint64_t n, uint32_t nb, uint32_t shift,
                                      uint64_t base, const uint64_t* off, uint32_t* cur, mckg_gaccess* out) {
  const uint32_t lane = threadIdx.x & 31u;
  for (uint64_t i0 = blockIdx.x * (uint64_t)blockDim.x; i0 < n; i0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i = i0 + threadIdx.x;
    uint32_t b0 = 0xFFFFFFFFu, b1 = 0xFFFFFFFFu;
    mckg_gaccess r{};
    if (i < n) {
      r = ev[i];
      const uint32_t len = ga_len(r.a);
      if ((r.b & 0xFFFFFFu) < MCKG_MAX_BID && len - 1u < MCKG_MAX_LEN) {
        const uint64_t a = ga_addr(r.a);
        b0 = bucket_of(a, nb, shift, base);
        const uint32_t bl = bucket_of(a + len - 1u, nb, shift, base);
        if (bl != b0) b1 = bl;
      }
    }
    const uint32_t g = __match_any_sync(0xFFFFFFFFu, b0);
    const int leader = __ffs(g) - 1;
    uint32_t p = 0;
    if (b0 != 0xFFFFFFFFu && lane == (uint32_t)leader) p = atomicAdd(cur + b0, (uint32_t)__popc(g));
    p = __shfl_sync(0xFFFFFFFFu, p, leader) + __popc(g & ((1u << lane) - 1u));
    if (b0 != 0xFFFFFFFFu) out[off[b0] + p] = r;
    if (b1 != 0xFFFFFFFFu) out[off[b1] + atomicAdd(cur + b1, 1u)] = r;
  }
}

// ---- the dense-span fast path: one warp per 2 KiB bucket ----
// Buckets of FB_WORDS words, direct-indexed tag arrays per warp (no hashing),
// races staged per warp and appended FB_STAGE at a time,
// the K2 word filter with __syncwarp between its phases, and the exact pass
// on <= 32 candidates (one per lane, same-word groups by __match_any_sync).
// A bucket with more than FB_MAX records, a record crossing a word, or more
// than 32 candidates is handed to the general kernel (bucket_detect_kernel).
constexpr uint32_t FB_SHIFT = 11;             // 2 KiB buckets
constexpr uint32_t FB_WORDS = 1u << (FB_SHIFT - 2);
constexpr uint32_t FB_ROWS = 16;               // records per lane
constexpr uint32_t FB_MAX = FB_ROWS * 32;
constexpr uint32_t FB_WARPS = 16;
constexpr int FB_BR = 2;                       // rows per load batch
constexpr uint32_t FB_STAGE = 128;             // staged races per warp
constexpr uint32_t FB_WARP_BYTES = FB_WORDS * 8 + 32 * 16 + FB_STAGE * 16;
constexpr uint32_t FB_SMEM = FB_WARPS * FB_WARP_BYTES;

struct LineCache {  // lane-owned first-racing-key cache of one warp
  uint32_t line;
  unsigned long long ts;
  uint32_t next;
};

__device__ __forceinline__ void lc_note(LineCache& C, unsigned long long* line_first, uint32_t L,
                                        unsigned long long T) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t own = __ballot_sync(0xFFFFFFFFu, C.line == L);
  if (own) {
    if (lane == (uint32_t)(__ffs(own) - 1) && T < C.ts) C.ts = T;
  } else {
    if (lane == C.next) {
      if (C.line != 0xFFFFFFFFu) atomicMin(line_first + C.line, C.ts);
      C.line = L;
      C.ts = T;
    }
    C.next = (C.next + 1u) & 31u;
  }
}

// appends a warp's staged races (one atomic per flush)
__device__ __forceinline__ void fb_flush(const BOut& O, const mckg_grace* stg, uint32_t n, uint32_t& flags) {
  const uint32_t lane = threadIdx.x & 31u;
  __syncwarp();
  if (n == 0) return;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(O.n, (unsigned long long)n);
  base = __shfl_sync(0xFFFFFFFFu, base, 0);
  for (uint32_t i = lane; i < n; i += 32) {
    if (base + i < O.cap)
      O.races[base + i] = stg[i];
    else
      flags |= MCKG_ST_OVERFLOW;
  }
  __syncwarp();
}

// Exact pass over a warp's batch of n <= 32 candidates (global record
// offsets in cl, from one or more buckets): lane per candidate X; X races on
// the bytes it shares with an earlier (timestamp) candidate Y of another
// block where X or Y writes; same-word groups by __match_any_sync (buckets
// are disjoint, so a word's candidates all sit in one bucket).  Racing
// (byte, line) pairs are reported once (the group of a (word, line) ORs its
// byte masks), staged per warp; the first racing key per line goes to the
// warp's line cache.
__device__ __noinline__ void fb_exact(const BOut& O, const uint4* cl, uint32_t nc,
                                      LineCache& C, mckg_grace* stg, uint32_t& nstg, uint32_t& flags) {
  const uint32_t lane = threadIdx.x & 31u;
  __syncwarp();
  if (nc == 0) return;
  const bool act = lane < nc;
  mckg_gaccess X{};
  if (act) {
    const uint4 r = cl[lane];
    X.a = rec_a(r);
    X.sweep = r.z;
    X.b = r.w;
  }
  const uint64_t xa = ga_addr(X.a);
  const unsigned long long xw = act ? (unsigned long long)(xa >> 2) : ~0ull - lane;
  const uint32_t xmask = act ? ((1u << ga_len(X.a)) - 1u) << (xa & 3u) : 0u;
  const unsigned long long xts = ga_ts(X);
  const uint32_t xbid = X.b & 0xFFFFFFu, xwr = ga_write(X.a);
  uint32_t rest = __match_any_sync(0xFFFFFFFFu, xw) & ~(1u << lane);
  uint32_t race = 0;
  while (__any_sync(0xFFFFFFFFu, rest != 0u)) {
    const uint32_t y = rest ? (uint32_t)__ffs(rest) - 1u : lane;
    rest &= rest - 1u;
    const uint32_t ymask = __shfl_sync(0xFFFFFFFFu, xmask, y), ybid = __shfl_sync(0xFFFFFFFFu, xbid, y),
                   ywr = __shfl_sync(0xFFFFFFFFu, xwr, y);
    const unsigned long long yts = __shfl_sync(0xFFFFFFFFu, xts, y);
    if (y != lane && yts < xts && ybid != xbid && (xwr | ywr)) race |= xmask & ymask;
  }
  const uint32_t rm = __ballot_sync(0xFFFFFFFFu, race != 0u);
  if (!rm) return;
  const uint32_t line = (uint32_t)ga_line(X.a, X.b);
  // first racing key per line
  for (uint32_t left = rm; left;) {
    const uint32_t L = __shfl_sync(0xFFFFFFFFu, line, __ffs(left) - 1);
    const bool in = race && line == L;
    const uint32_t mh = __reduce_min_sync(0xFFFFFFFFu, in ? (uint32_t)(xts >> 32) : ~0u);
    const uint32_t ml = __reduce_min_sync(0xFFFFFFFFu, in && (uint32_t)(xts >> 32) == mh ? (uint32_t)xts : ~0u);
    left &= ~__ballot_sync(0xFFFFFFFFu, in);
    lc_note(C, O.line_first, L, ((unsigned long long)mh << 32) | ml);
  }
  const unsigned long long gkey = race ? ((unsigned long long)(xa >> 2) << 16) | (line & 0xFFFFu) : ~0ull - lane;
  const uint32_t grp = __match_any_sync(0xFFFFFFFFu, gkey);
  // OR of the group's byte masks.  Not __reduce_or_sync(grp, ...): with a
  // different mask per group it runs once per distinct group (up to 32
  // serial redux), while groups here are mostly singletons -- this loop runs
  // (largest group - 1) shuffles
  uint32_t mine = race;
  for (uint32_t q = grp & ~(1u << lane); __any_sync(0xFFFFFFFFu, q != 0u);) {
    const uint32_t y = q ? (uint32_t)__ffs(q) - 1u : lane;
    q &= q - 1u;
    mine |= __shfl_sync(0xFFFFFFFFu, race, y);
  }
  const bool rep = race && (grp & rm & ((1u << lane) - 1u)) == 0u;
  const uint32_t cnt = rep ? __popc(mine) : 0u;
  uint32_t ci = cnt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, ci, d);
    if (lane >= (uint32_t)d) ci += t;
  }
  const uint32_t tot = __shfl_sync(0xFFFFFFFFu, ci, 31);
  if (nstg + tot > FB_STAGE) {
    fb_flush(O, stg, nstg, flags);
    nstg = 0;
  }
  if (tot > FB_STAGE) {  // more than a buffer at once: straight out
    unsigned long long base_o = 0;
    if (lane == 0) base_o = atomicAdd(O.n, (unsigned long long)tot);
    base_o = __shfl_sync(0xFFFFFFFFu, base_o, 0) + ci - cnt;
    if (rep)
      for (uint32_t q = mine; q; q &= q - 1u, ++base_o) {
        if (base_o < O.cap)
          O.races[base_o] = mckg_grace{(xa & ~3ull) + (uint32_t)(__ffs(q) - 1), (int32_t)line, 0};
        else
          flags |= MCKG_ST_OVERFLOW;
      }
    return;
  }
  if (rep) {
    uint32_t p = nstg + ci - cnt;
    for (uint32_t q = mine; q; q &= q - 1u, ++p)
      stg[p] = mckg_grace{(xa & ~3ull) + (uint32_t)(__ffs(q) - 1), (int32_t)line, 0};
  }
  nstg += tot;
  __syncwarp();
}

__global__ void __launch_bounds__(FB_WARPS * 32, 2) bucket_fast_kernel(const mckg_gaccess* recs, const uint64_t* off,
                                                                       uint32_t nb, uint64_t base, BOut O,
                                                                       uint32_t* big, uint32_t* nbig,
                                                                       uint32_t* next) {
  extern __shared__ __align__(16) uint8_t sm[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  uint32_t* tag = reinterpret_cast<uint32_t*>(sm + warp * FB_WARP_BYTES);
  uint32_t* flg = tag + FB_WORDS;
  uint4* cl = reinterpret_cast<uint4*>(flg + FB_WORDS);  // the candidate batch (records)
  mckg_grace* stg = reinterpret_cast<mckg_grace*>(cl + 32);  // staged races
  uint32_t nbatch = 0;                                          // warp-uniform
  uint32_t nstg = 0;                                          // warp-uniform
  for (uint32_t i = lane; i < FB_WORDS; i += 32) flg[i] = 0u;
  __syncwarp();
  LineCache C{0xFFFFFFFFu, ~0ull, 0u};
  uint32_t stamp = 0;
  uint32_t flags = 0;
  // buckets are claimed in chunks from a counter: a fixed stride can alias
  // the data's period (e.g. every other 32 KiB empty) and idle half the warps
  // (a chunk is 32 buckets: lane l holds bucket l's record range, so empty
  // and single-record buckets cost no memory round trip)
  constexpr uint32_t CH = 32;
  uint32_t b = 0, bend = 0;
  uint64_t lo0 = 0, lo1 = 0;  // lane l: off[b0 + l], off[b0 + l + 1]
  uint32_t b0 = 0;
  while (true) {
    if (b == bend) {
      uint32_t c0 = 0;
      if (lane == 0) c0 = atomicAdd(next, CH);
      b = b0 = __shfl_sync(0xFFFFFFFFu, c0, 0);
      bend = min(b + CH, nb);
      if (b >= nb) break;
      const uint32_t mine = b0 + lane;
      lo0 = mine < nb ? off[mine] : 0;
      lo1 = mine < nb ? off[mine + 1] : 0;
    }
    // the next bucket of the chunk with >= 2 records
    const uint32_t busy = __ballot_sync(0xFFFFFFFFu, b0 + lane >= b && b0 + lane < bend && lo1 - lo0 >= 2);
    if (!busy) {
      b = bend;
      continue;
    }
    const uint32_t bl = (uint32_t)__ffs(busy) - 1u;
    const uint32_t bb = b0 + bl;
    b = bb + 1;
    const uint64_t o0 = __shfl_sync(0xFFFFFFFFu, lo0, bl), o1 = __shfl_sync(0xFFFFFFFFu, lo1, bl);
    if (o1 - o0 <= 32u) {
      // small buckets skip the filter: a run of whole buckets (contiguous
      // records, disjoint words) of <= 32 records joins the exact batch --
      // the filter only prunes, fb_exact decides every pair itself
      if (nbatch + (uint32_t)(o1 - o0) > 32u) {
        fb_exact(O, cl, nbatch, C, stg, nstg, flags);
        nbatch = 0;
      }
      const uint32_t room = 32u - nbatch;
      const uint32_t fits = __ballot_sync(0xFFFFFFFFu, lane >= bl && b0 + lane < bend && lo1 - o0 <= room);
      const uint32_t r = __popc(fits);  // buckets bl .. bl + r - 1 (lo1 is monotonic)
      const uint64_t e = __shfl_sync(0xFFFFFFFFu, lo1, bl + r - 1u);
      const uint32_t len = (uint32_t)(e - o0);
      bool badr = false;
      uint4 rr = make_uint4(0, 0, 0, 0);
      if (lane < len) {
        rr = __ldg(reinterpret_cast<const uint4*>(recs) + o0 + lane);
        const uint64_t a64 = rec_a(rr);
        badr = (ga_addr(a64) & 3u) + ga_len(a64) > 4u;  // a word-contained record lies in its bucket
      }
      const uint32_t badm = __ballot_sync(0xFFFFFFFFu, badr);
      if (badm) {
        // hand the buckets holding crossing records to the general kernel;
        // the rest of the run is retried from the next bucket on
        const uint32_t p = (uint32_t)__ffs(badm) - 1u;  // first crossing record
        const uint32_t hb = __ffs(__ballot_sync(0xFFFFFFFFu, lane >= bl && lane < bl + r &&
                                                             lo0 - o0 <= p && p < lo1 - o0)) - 1u;
        if (lane == 0) big[atomicAdd(nbig, 1u)] = b0 + hb;
        b = b0 + hb + 1;
        if (hb > bl) {  // the buckets before it are clean
          const uint32_t clen = (uint32_t)(__shfl_sync(0xFFFFFFFFu, lo0, hb) - o0);
          if (lane < clen) cl[nbatch + lane] = rr;
          nbatch += clen;
        }
        __syncwarp();
        continue;
      }
      if (lane < len) cl[nbatch + lane] = rr;
      nbatch += len;
      b = b0 + bl + r;
      __syncwarp();
      continue;
    }
    if (o1 - o0 > FB_MAX) {
      if (lane == 0) big[atomicAdd(nbig, 1u)] = bb;
      continue;
    }
    const uint32_t m = (uint32_t)(o1 - o0);
    const mckg_gaccess* R = recs + o0;
    uint64_t blo, bhi;
    bucket_range(bb, nb, FB_SHIFT, base, &blo, &bhi);

    // load + pack: word (10 bits) | write << 10 | bid << 11 (rows of 32
    // records, FB_BR rows in flight ahead of the decode)
    uint32_t pk[FB_ROWS];
    bool bad = false;
    const uint4* R4 = reinterpret_cast<const uint4*>(R);
    uint4 buf[2][FB_BR];
#pragma unroll
    for (int q = 0; q < FB_BR; ++q) {
      const uint32_t i = (uint32_t)q * 32u + lane;
      buf[0][q] = i < m ? __ldg(R4 + i) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int h = 0; h < (int)(FB_ROWS / FB_BR); ++h) {
      if ((uint32_t)h * FB_BR * 32u < m) {  // warp-uniform
        if (h + 1 < (int)(FB_ROWS / FB_BR)) {
#pragma unroll
          for (int q = 0; q < FB_BR; ++q) {
            const uint32_t i = (uint32_t)((h + 1) * FB_BR + q) * 32u + lane;
            buf[(h + 1) & 1][q] = i < m ? __ldg(R4 + i) : make_uint4(0, 0, 0, 0);
          }
        }
#pragma unroll
        for (int q = 0; q < FB_BR; ++q) {
          const int j = h * FB_BR + q;
          const uint32_t i = (uint32_t)j * 32u + lane;
          const uint4 r = buf[h & 1][q];
          const unsigned long long a64 = ((unsigned long long)r.y << 32) | r.x;
          const uint64_t a = ga_addr(a64);
          const bool in = i < m;
          bad |= in && ((a & 3u) + ga_len(a64) > 4u || a < blo || a >= bhi);
          // the word index is swizzled (w ^ (w >> 5)): a row of records of
          // consecutive threads at a 32-word stride (one thread's 128 B run
          // per 4-byte slot) would otherwise land on one bank
          const uint32_t w = (uint32_t)((a - blo) >> 2);
          pk[j] = in ? (w ^ ((w >> 5) & 31u)) | (ga_write(a64) << 10) | ((r.w & 0x1FFFFFu) << 11) : 0xFFFFFFFFu;
        }
      } else {
#pragma unroll
        for (int q = 0; q < FB_BR; ++q) pk[h * FB_BR + q] = 0xFFFFFFFFu;
      }
    }
    if (__any_sync(0xFFFFFFFFu, bad)) {
      if (lane == 0) big[atomicAdd(nbig, 1u)] = bb;
      continue;
    }
    stamp = stamp == 0xFFFFu ? 1u : stamp + 1u;
    const uint32_t pat = stamp | (stamp << 16);
    // P1 / P2 / P3 (__syncwarp between them)
#pragma unroll
    for (int j = 0; j < (int)FB_ROWS; ++j)
      if (pk[j] != 0xFFFFFFFFu) tag[pk[j] & (FB_WORDS - 1)] = pk[j] >> 11;
    __syncwarp();
#pragma unroll
    for (int j = 0; j < (int)FB_ROWS; ++j) {
      const uint32_t x = pk[j];
      if (x == 0xFFFFFFFFu) continue;
      uint16_t* f = reinterpret_cast<uint16_t*>(flg + (x & (FB_WORDS - 1)));
      if (tag[x & (FB_WORDS - 1)] != (x >> 11)) f[0] = (uint16_t)stamp;
      if (x & 0x400u) f[1] = (uint16_t)stamp;
    }
    __syncwarp();
    uint32_t cm = 0;
#pragma unroll
    for (int j = 0; j < (int)FB_ROWS; ++j)
      if (pk[j] != 0xFFFFFFFFu && flg[pk[j] & (FB_WORDS - 1)] == pat) cm |= 1u << j;
    const uint32_t c = __popc(cm);
    uint32_t incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= (uint32_t)d) incl += t;
    }
    const uint32_t nc = __shfl_sync(0xFFFFFFFFu, incl, 31);
    if (nc == 0) continue;
    if (nc > 32u) {
      if (lane == 0) big[atomicAdd(nbig, 1u)] = bb;
      continue;
    }
    // the bucket's candidates join the warp's batch (exact pass per 32)
    if (nbatch + nc > 32u) {
      fb_exact(O, cl, nbatch, C, stg, nstg, flags);
      nbatch = 0;
    }
    uint32_t pos = nbatch + incl - c;
    for (uint32_t g = cm; g; g &= g - 1u) cl[pos++] = __ldg(R4 + (uint64_t)((__ffs(g) - 1) * 32u + lane));
    nbatch += nc;
    __syncwarp();
  }
  fb_exact(O, cl, nbatch, C, stg, nstg, flags);
  fb_flush(O, stg, nstg, flags);
  if (C.line != 0xFFFFFFFFu) atomicMin(O.line_first + C.line, C.ts);
  flags = __reduce_or_sync(0xFFFFFFFFu, flags);
  if (lane == 0 && flags) atomicOr(O.status, flags);
}

// ---- the in-place tile path (block-clustered inputs: a K1 log, C5) ----
// Records come grouped by simulated block and a block's accesses mostly fall
// in its own address range.  Instead of partitioning every record into
// address buckets (count: read; scatter: read + write; detect: read), tiles of
// TT consecutive records are checked where they lie:
//   pass 0 (tile_claim): a tile's window is TW consecutive 2 KiB buckets from
//     an anchor chosen on a sample of its records (the anchor covering most
//     samples); it claims the window buckets it occupies (claim[b] += 1).
//     Every other record of the tile (outside the window, crossing a word,
//     out of range) is FOREIGN: appended to the side list, its words marked
//     in a bitmap over the span;
//   pass 1: a record in its tile's window is OWN when its bucket was claimed
//     by that tile alone and its word is unmarked.  No record of another
//     tile touches an own record's word, so a tile whose own records all
//     come from one block has no race among them (races are cross-block);
//     otherwise they run the word filter of bucket_fast over the window's
//     TW x 512 words.  The rest (contested buckets, marked words) are MIXED
//     and join the side list.  Pass 0 leaves a 2-byte code per record (its
//     window word) and whether the tile's in-window records span blocks;
//     tile_mixed classifies single-block tiles from the codes alone (8 KiB
//     per tile instead of 64 KiB of records) and lists the others for
//     tile_detect, which re-reads them;
//   the side list (foreign + mixed, every record on their words) then runs
//     through the bucket pipeline.
// Each word is decided by exactly one of the two, so the race sets are
// disjoint and their union is the bucket pipeline's on the whole input.
// The window choice only moves records between the two routes.
constexpr uint32_t TT = 4096;                // records per tile
constexpr uint32_t TB = 512;                 // threads per tile CTA
constexpr uint32_t TR = TT / TB;             // records per thread
constexpr uint32_t TW = 16;                  // window buckets per tile
constexpr uint32_t TWW = TW * FB_WORDS;      // window words
constexpr uint32_t TS = 16;                  // anchor samples per tile
constexpr uint32_t TBW = FB_WORDS / 32;      // bitmap words per bucket
// pass-1 word table: bid (21 bits) | MULTI | WRITE (flags set by atomicOr)
constexpr uint32_t TAG_MULTI = 1u << 30, TAG_WRITE = 1u << 31;
// dynamic shared memory: the tile stage (TT records, filled by the bulk-copy
// engine one tile ahead); tile_multi's word table
constexpr uint32_t TC_SMEM = TT * 16;
constexpr uint32_t TD_SMEM = TT * 16;
constexpr uint32_t TM_SMEM = TWW * 4;

// the bucket of an in-span, word-contained record, else ~0u
__device__ __forceinline__ uint32_t tile_bucket(uint64_t a64, uint32_t bid, uint64_t base, uint32_t nbk) {
  const uint64_t a = ga_addr(a64);
  const uint32_t len = ga_len(a64);
  if (len == 0 || (a & 3u) + len > 4u || a < base || bid >= MCKG_MAX_BID) return ~0u;
  const uint64_t q = (a - base) >> FB_SHIFT;
  return q < nbk ? (uint32_t)q : ~0u;
}

// one tile into the stage (thread 0; the stage's readers are past a barrier)
__device__ __forceinline__ void tile_fetch(const mckg_gaccess* ev, uint64_t n, uint64_t t, void* stage,
                                           uint64_t* bar) {
  const uint64_t r0 = t * TT;
  const uint32_t bytes = (uint32_t)((n - r0 < TT ? n - r0 : TT) * sizeof(mckg_gaccess));
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_expect_tx(bar, bytes);
  bulk_g2s(stage, ev + r0, bytes, bar);
}


// The window slot of record r for a tile whose window starts at byte wbase
// and has jmax = min(TW, nbk - anchor) buckets, else ~0u -- exactly
// tile_bucket(r) - anchor < TW, in fewer instructions (the hot test of both
// passes).  *rel: the byte offset in the window.
__device__ __forceinline__ uint32_t win_slot(const uint4& r, uint64_t wbase, uint32_t jmax, uint32_t* rel) {
  const unsigned long long a = ((unsigned long long)(r.y & 0xFFu) << 32) | r.x;
  const uint32_t len = (r.y >> 8) & 0xFu;
  const uint64_t d = a - wbase;  // wraps high below the window
  const uint32_t dl = (uint32_t)d, j = dl >> FB_SHIFT;
  *rel = dl;
  const bool in = d < ((uint64_t)TW << FB_SHIFT) && j < jmax && len != 0u && (dl & 3u) + len <= 4u &&
                  (r.w & 0xFFFFFFu) < MCKG_MAX_BID;
  return in ? j : ~0u;
}

// This thread's slot among a tile's flagged records (bits of `fm`): a warp
// scan plus one shared-memory atomic per warp on the tile's counter.
__device__ __forceinline__ uint32_t side_slot(uint32_t fm, uint32_t* cnt) {
  const uint32_t lane = threadIdx.x & 31u;
  if (!__any_sync(0xFFFFFFFFu, fm != 0u)) return 0;
  const uint32_t c = __popc(fm);
  uint32_t incl = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t x = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if (lane >= (uint32_t)d) incl += x;
  }
  uint32_t wb = 0;
  if (lane == 31) wb = atomicAdd(cnt, incl);
  return __shfl_sync(0xFFFFFFFFu, wb, 31) + incl - c;
}

// The deferred write of this thread's flagged records of the tile at r0
// (re-read from ev: rare, L2-resident) to side[base + slot ...].
__device__ __forceinline__ void side_write(uint32_t fm, uint32_t slot, unsigned long long base,
                                           const mckg_gaccess* ev, uint64_t r0, mckg_gaccess* side) {
  unsigned long long p = base + slot;
  for (uint32_t q = fm; q; q &= q - 1u) side[p++] = ev[r0 + (uint64_t)((__ffs(q) - 1) * TB + threadIdx.x)];
}

// Pass 0, persistent: a CTA walks tiles blockIdx.x, + gridDim.x, ...; the
// next tile streams into the stage while this one is classified.  Two
// barriers per tile: the side-list base of a tile is taken after its second
// barrier and its records are written after the next tile's first.  Output
// per tile: win[t] = anchor | occupied-bucket mask << 32 (~0: no window).
__global__ void __launch_bounds__(TB, 2) tile_claim_kernel(const mckg_gaccess* ev, uint64_t n, uint64_t ntiles,
                                                           uint64_t base, uint32_t nbk, uint32_t* claim,
                                                           uint32_t* bits, unsigned long long* win,
                                                           mckg_gaccess* side, unsigned long long* nside,
                                                           uint16_t* code, uint8_t* tmulti) {
  extern __shared__ __align__(16) uint8_t sm[];
  const uint4* stage = reinterpret_cast<const uint4*>(sm);
  __shared__ uint32_t s_anchor, s_occ[2], s_cnt[2], s_bmin[2], s_bmax[2];
  __shared__ unsigned long long s_base[2];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t nwords = nbk * FB_WORDS;  // nbk < 2^23
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    s_occ[0] = s_occ[1] = 0;
    s_cnt[0] = s_cnt[1] = 0;
    s_bmin[0] = s_bmin[1] = ~0u;
    s_bmax[0] = s_bmax[1] = 0;
  }
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x < ntiles) tile_fetch(ev, n, blockIdx.x, sm, &bar);
  uint32_t pfm = 0, pslot = 0;  // the previous tile's foreign records (deferred)
  uint64_t pr0 = 0;
  uint32_t it = 0;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const uint32_t cb = it & 1u;
    const uint64_t r0 = t * TT;
    const uint32_t m = (uint32_t)(n - r0 < TT ? n - r0 : TT);
    mbar_wait(&bar, cb);
    if (threadIdx.x < 32) {
      // the anchor: of TS sampled buckets, the one whose TW-bucket window
      // covers most samples (ties: the lowest)
      const uint32_t si = lane * (TT / TS);
      uint32_t sb = ~0u;
      if (lane < TS && si < m) {
        const uint4 r = stage[si];
        sb = tile_bucket(rec_a(r), r.w & 0xFFFFFFu, base, nbk);
      }
      uint32_t cover = 0;
#pragma unroll
      for (uint32_t j = 0; j < TS; ++j) {
        const uint32_t u = __shfl_sync(0xFFFFFFFFu, sb, j);
        cover += (u != ~0u && u - sb < TW);
      }
      const uint32_t key = sb == ~0u ? 0u : (cover << 23) | ((1u << 23) - 1u - sb);
      const uint32_t best = __reduce_max_sync(0xFFFFFFFFu, key);
      if (lane == 0) s_anchor = best ? (1u << 23) - 1u - (best & ((1u << 23) - 1u)) : ~0u;
    }
    __syncthreads();  // #1: s_anchor; the previous tile's side base
    if (pfm) side_write(pfm, pslot, s_base[cb ^ 1u], ev, pr0, side);
    const uint32_t anchor = s_anchor;
    const uint64_t wbase = base + ((uint64_t)anchor << FB_SHIFT);
    const uint32_t jmax = anchor == ~0u ? 0u : min(TW, nbk - anchor);
    uint32_t fm = 0, occ = 0, bmin = ~0u, bmax = 0;
#pragma unroll
    for (uint32_t k = 0; k < TR; ++k) {
      const uint32_t i = k * TB + threadIdx.x;
      uint32_t c = 0xFFFFu;  // the record's pass-1 code: window word, or none
      if (i < m) {
        const uint4 r = stage[i];
        uint32_t rel;
        const uint32_t j = win_slot(r, wbase, jmax, &rel);
        if (j != ~0u) {
          occ |= 1u << j;
          // j << 9 | word in the bucket, its bitmap word x = c >> 5 swizzled
          // as pass 1 stores it (x ^ ((x >> 5) & 7))
          c = rel >> 2;
          c = ((c >> 5) ^ ((c >> 10) & 7u)) << 5 | (c & 31u);
          bmin = min(bmin, r.w & 0xFFFFFFu);
          bmax = max(bmax, r.w & 0xFFFFFFu);
        }
      }
      if (code) code[r0 + i] = (uint16_t)c;
      if (c != 0xFFFFu || i >= m) continue;
      const uint4 r = stage[i];
      const unsigned long long a64 = rec_a(r);
      fm |= 1u << k;
      // foreign: mark the words it touches (clipped to the span)
      const uint64_t a = ga_addr(a64);
      const uint32_t len = ga_len(a64) ? ga_len(a64) : 1u;
      if (a + len > base && a < base + ((uint64_t)nwords << 2)) {
        const uint32_t w0 = a < base ? 0u : (uint32_t)((a - base) >> 2);
        const uint64_t wl = (a + len - 1 - base) >> 2;
        const uint32_t w1 = wl < nwords ? (uint32_t)wl : nwords - 1u;
        for (uint32_t w = w0; w <= w1; ++w) atomicOr(bits + (w >> 5), 1u << (w & 31u));
      }
    }
    occ = __reduce_or_sync(0xFFFFFFFFu, occ);
    if (lane == 0 && occ) atomicOr(&s_occ[cb], occ);
    bmin = __reduce_min_sync(0xFFFFFFFFu, bmin);
    bmax = __reduce_max_sync(0xFFFFFFFFu, bmax);
    if (lane == 0 && bmin != ~0u) {
      atomicMin(&s_bmin[cb], bmin);
      atomicMax(&s_bmax[cb], bmax);
    }
    const uint32_t slot = side_slot(fm, &s_cnt[cb]);
    __syncthreads();  // #2: the stage is free; s_occ / s_cnt / s_bmin / s_bmax of this tile final
    if (threadIdx.x == 0) {
      if (t + gridDim.x < ntiles) tile_fetch(ev, n, t + gridDim.x, sm, &bar);
      s_base[cb] = s_cnt[cb] ? atomicAdd(nside, (unsigned long long)s_cnt[cb]) : 0ull;
      s_cnt[cb ^ 1u] = 0;  // the next tile's (last read before #2)
      s_occ[cb ^ 1u] = 0;
      s_bmin[cb ^ 1u] = ~0u;
      s_bmax[cb ^ 1u] = 0;
    }
    const uint32_t so = s_occ[cb];
    if (threadIdx.x == 32) win[t] = (anchor == ~0u || !so) ? ~0ull : ((unsigned long long)so << 32) | anchor;
    if (threadIdx.x == 64 && tmulti) tmulti[t] = s_bmin[cb] != s_bmax[cb] ? 1 : 0;
    if (threadIdx.x < TW && ((so >> threadIdx.x) & 1u)) atomicAdd(claim + anchor + threadIdx.x, 1u);
    pfm = fm;
    pslot = slot;
    pr0 = r0;
  }
  __syncthreads();
  if (pfm) side_write(pfm, pslot, s_base[(it - 1u) & 1u], ev, pr0, side);
}

// Pass 1, persistent like pass 0; the window metadata of a CTA's next tile
// (claims, word marks) is fetched while this one is checked.  A tile whose
// own records come from two or more blocks is listed for tile_multi_kernel
// (the word filter needs a 32 KiB table that would cost this kernel a CTA
// per SM).
__global__ void __launch_bounds__(TB, 3) tile_detect_kernel(const mckg_gaccess* ev, uint64_t n, uint64_t ntiles,
                                                            uint64_t base, uint32_t nbk, const uint32_t* claim,
                                                            const uint32_t* bits, const unsigned long long* win,
                                                            mckg_gaccess* side, unsigned long long* nside,
                                                            uint32_t* multi, uint32_t* nmulti,
                                                            const uint32_t* list, const uint32_t* nlist) {
  extern __shared__ __align__(16) uint8_t sm[];
  const uint4* stage = reinterpret_cast<const uint4*>(sm);
  __shared__ uint32_t s_anc[2], s_ok[2], s_bmin[2], s_bmax[2], s_cnt[2];
  __shared__ unsigned long long s_base[2];
  __shared__ uint32_t sbits[2][TW * TBW];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t lane = threadIdx.x & 31u;
  // the window metadata of tile t into buffer q (s_ok[q] is 0 on entry)
  // the tiles: every tile, or the listed ones
  const uint64_t cnt = list ? (uint64_t)*nlist : ntiles;
  auto tile = [&](uint64_t idx) -> uint64_t { return list ? (uint64_t)list[idx] : idx; };
  auto meta = [&](uint32_t q, uint64_t t) {
    const unsigned long long wv = win[t];
    const uint32_t anchor = (uint32_t)wv, occ = (uint32_t)(wv >> 32);
    if (threadIdx.x == 0) s_anc[q] = anchor;
    if (anchor == ~0u) return;
    if (threadIdx.x < TW && ((occ >> threadIdx.x) & 1u) && claim[anchor + threadIdx.x] == 1u)
      atomicOr(&s_ok[q], 1u << threadIdx.x);
    if (threadIdx.x < TW * TBW && ((occ >> (threadIdx.x / TBW)) & 1u))
      sbits[q][threadIdx.x] = bits[(uint64_t)anchor * TBW + threadIdx.x];
  };
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
    for (int q = 0; q < 2; ++q) {
      s_ok[q] = 0;
      s_cnt[q] = 0;
      s_bmin[q] = ~0u;
      s_bmax[q] = 0;
    }
  }
  __syncthreads();
  if (blockIdx.x < cnt) {
    if (threadIdx.x == 0) tile_fetch(ev, n, tile(blockIdx.x), sm, &bar);
    meta(0, tile(blockIdx.x));
  }
  uint32_t pmm = 0, pslot = 0;           // the previous tile's mixed records (deferred)
  uint64_t pr0 = 0;
  uint32_t it = 0;
  for (uint64_t idx = blockIdx.x; idx < cnt; idx += gridDim.x, ++it) {
    const uint64_t t = tile(idx);
    const uint32_t cb = it & 1u;
    const uint64_t r0 = t * TT;
    const uint32_t m = (uint32_t)(n - r0 < TT ? n - r0 : TT);
    mbar_wait(&bar, cb);
    __syncthreads();  // #1: this tile's metadata; the previous tile's side base
    if (pmm) side_write(pmm, pslot, s_base[cb ^ 1u], ev, pr0, side);
    if (threadIdx.x == 0) {  // the next tile's counters (last read before #1)
      s_ok[cb ^ 1u] = 0;
      s_cnt[cb ^ 1u] = 0;
      s_bmin[cb ^ 1u] = ~0u;
      s_bmax[cb ^ 1u] = 0;
    }
    const uint32_t anchor = s_anc[cb], ok = s_ok[cb];
    const uint64_t wbase = base + ((uint64_t)anchor << FB_SHIFT);
    const uint32_t jmax = anchor == ~0u ? 0u : min(TW, nbk - anchor);
    uint32_t bmin = ~0u, bmax = 0, mm = 0;
#pragma unroll
    for (uint32_t k = 0; k < TR; ++k) {
      const uint32_t i = k * TB + threadIdx.x;
      if (i >= m) continue;
      const uint4 r = stage[i];
      uint32_t rel;
      const uint32_t j = win_slot(r, wbase, jmax, &rel);
      if (j == ~0u) continue;  // foreign: sent in pass 0
      const uint32_t w = (rel >> 2) & (FB_WORDS - 1u);
      const uint32_t bid = r.w & 0xFFFFFFu;
      if (((ok >> j) & 1u) && !((sbits[cb][j * TBW + (w >> 5)] >> (w & 31u)) & 1u)) {
        bmin = min(bmin, bid);
        bmax = max(bmax, bid);
      } else {
        mm |= 1u << k;  // mixed
      }
    }
    bmin = __reduce_min_sync(0xFFFFFFFFu, bmin);
    bmax = __reduce_max_sync(0xFFFFFFFFu, bmax);
    if (lane == 0 && bmin != ~0u) {
      atomicMin(&s_bmin[cb], bmin);
      atomicMax(&s_bmax[cb], bmax);
    }
    const uint32_t slot = side_slot(mm, &s_cnt[cb]);
    __syncthreads();  // #2: the stage is free; this tile's counters final
    if (threadIdx.x == 0) {
      if (idx + gridDim.x < cnt) tile_fetch(ev, n, tile(idx + gridDim.x), sm, &bar);
      s_base[cb] = s_cnt[cb] ? atomicAdd(nside, (unsigned long long)s_cnt[cb]) : 0ull;
    }
    if (idx + gridDim.x < cnt) meta(cb ^ 1u, tile(idx + gridDim.x));
    pmm = mm;
    pslot = slot;
    pr0 = r0;
    if (threadIdx.x == 0 && s_bmin[cb] != ~0u && s_bmin[cb] != s_bmax[cb]) multi[atomicAdd(nmulti, 1u)] = (uint32_t)t;
  }
  __syncthreads();
  if (pmm) side_write(pmm, pslot, s_base[(it - 1u) & 1u], ev, pr0, side);
}

// Pass 1 without re-reading the records (the default): a warp per tile
// reads the tile's 2-byte codes from pass 0 (window word per record, 8 KiB
// per tile instead of 64 KiB of records) and sends its MIXED records to the
// side list -- exactly pass 1's classification.  A tile whose in-window
// records come from two or more blocks (tmulti) may have own records that
// race among themselves: it is listed for the full pass 1 (tile_detect on
// the list), which re-reads it.
constexpr uint32_t TQ = TT / 8 / 32;  // uint4 code groups per lane
__global__ void __launch_bounds__(TB, 4) tile_mixed_kernel(const mckg_gaccess* ev, uint64_t ntiles,
                                                           const uint32_t* claim, const uint32_t* bits,
                                                           const unsigned long long* win, const uint16_t* code,
                                                           const uint8_t* tmulti, mckg_gaccess* side,
                                                           unsigned long long* nside, uint32_t* full,
                                                           uint32_t* nfull) {
  __shared__ uint32_t sbits_all[TB / 32][TW * TBW];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  uint32_t* sb = sbits_all[warp];
  const uint4* c4 = reinterpret_cast<const uint4*>(code);
  for (uint64_t t = (uint64_t)blockIdx.x * (TB / 32) + warp; t < ntiles; t += (uint64_t)gridDim.x * (TB / 32)) {
    const unsigned long long wv = win[t];
    const uint32_t anchor = (uint32_t)wv, occ = (uint32_t)(wv >> 32);
    uint32_t mw[TQ / 4] = {};
    uint32_t c = 0, incl = 0;
    if (anchor != ~0u && tmulti[t]) {
      if (lane == 0) full[atomicAdd(nfull, 1u)] = (uint32_t)t;
    } else if (anchor != ~0u) {  // (no window: every record foreign, sent in pass 0)
      const bool own = lane < TW && ((occ >> lane) & 1u) && claim[anchor + lane] == 1u;
      const uint32_t ok = __ballot_sync(0xFFFFFFFFu, own);
#pragma unroll
      for (uint32_t q = 0; q < TW * TBW / 32; ++q) {
        const uint32_t x = q * 32u + lane;
        // word x of the window's bitmap, all-ones when its bucket is not
        // solely this tile's (so a set bit = MIXED), stored swizzled at
        // x ^ ((x >> 5) & 7): lanes holding records a fixed stride apart,
        // e.g. one per thread of a simulated block, hit 8 words of one bank
        // otherwise (pass 0's codes carry the swizzled index)
        if ((occ >> (x / TBW)) & 1u)
          sb[x ^ ((x >> 5) & 7u)] = ((ok >> (x / TBW)) & 1u) ? bits[(uint64_t)anchor * TBW + x] : ~0u;
      }
      __syncwarp();
      // lane l holds code groups g = q * 32 + l (records 8g .. 8g + 7)
#pragma unroll
      for (uint32_t q = 0; q < TQ; ++q) {
        const uint4 c = c4[t * (TT / 8) + q * 32u + lane];
        const uint32_t cc[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (uint32_t e = 0; e < 8; ++e) {
          const uint32_t v = (cc[e >> 1] >> (16 * (e & 1))) & 0xFFFFu;
          if (v == 0xFFFFu) continue;
          const uint32_t b = sb[v >> 5];
          mw[q >> 2] |= (__funnelshift_r(b, b, v) & 1u) << ((q & 3u) * 8u + e);
        }
      }
#pragma unroll
      for (uint32_t h = 0; h < TQ / 4; ++h) c += __popc(mw[h]);
      incl = c;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, d);
        if (lane >= (uint32_t)d) incl += y;
      }
    }
    const uint32_t tot = __shfl_sync(0xFFFFFFFFu, incl, 31);
    if (tot) {
      unsigned long long b = 0;
      if (lane == 31) b = atomicAdd(nside, (unsigned long long)tot);
      unsigned long long p = __shfl_sync(0xFFFFFFFFu, b, 31) + incl - c;
      const uint64_t r0 = t * TT;
#pragma unroll
      for (uint32_t h = 0; h < TQ / 4; ++h)
        for (uint32_t f = mw[h]; f; f &= f - 1u) {
          const uint32_t bit = (uint32_t)__ffs(f) - 1u, q = h * 4u + (bit >> 3), e = bit & 7u;
          side[p++] = ev[r0 + (uint64_t)(q * 32u + lane) * 8u + e];
        }
    }
    __syncwarp();  // sb is rewritten for the warp's next tile
  }
}

// The listed tiles of pass 1 (own records from two or more blocks): the own
// records again (same classification), then the word filter of bucket_fast
// over the window -- P1 last bid per word, P2 multi-block / write flags
// (atomicOr keeps the bid bits readable), P3 candidates -- and the exact pass
// (<= 32 candidates) or, past that, the tile's own records to the side list.
__global__ void __launch_bounds__(TB) tile_multi_kernel(const mckg_gaccess* ev, uint64_t n, uint64_t base,
                                                        uint32_t nbk, const uint32_t* claim, const uint32_t* bits,
                                                        const unsigned long long* win, const uint32_t* multi,
                                                        const uint32_t* nmulti, mckg_gaccess* side,
                                                        unsigned long long* nside, BOut O) {
  extern __shared__ __align__(16) uint8_t sm[];
  uint32_t* tag = reinterpret_cast<uint32_t*>(sm);
  __shared__ uint32_t s_ok, s_nc, s_cnt;
  __shared__ unsigned long long s_base;
  __shared__ uint32_t sbits[TW * TBW];
  __shared__ uint4 cl[32];
  __shared__ mckg_grace stg[FB_STAGE];
  LineCache C{0xFFFFFFFFu, ~0ull, 0u};  // warp 0's
  uint32_t nstg = 0, flags = 0;          // warp 0's
  const uint32_t nl = *nmulti;
  for (uint32_t li = blockIdx.x; li < nl; li += gridDim.x) {
    const uint64_t t = multi[li];
    const uint64_t r0 = t * TT;
    const uint32_t m = (uint32_t)(n - r0 < TT ? n - r0 : TT);
    const unsigned long long wv = win[t];
    const uint32_t anchor = (uint32_t)wv, occ = (uint32_t)(wv >> 32);
    if (threadIdx.x == 0) {
      s_ok = 0;
      s_nc = 0;
      s_cnt = 0;
    }
    __syncthreads();
    if (threadIdx.x < TW && ((occ >> threadIdx.x) & 1u) && claim[anchor + threadIdx.x] == 1u)
      atomicOr(&s_ok, 1u << threadIdx.x);
    if (threadIdx.x < TW * TBW && ((occ >> (threadIdx.x / TBW)) & 1u))
      sbits[threadIdx.x] = bits[(uint64_t)anchor * TBW + threadIdx.x];
    __syncthreads();
    const uint32_t ok = s_ok;
    const uint64_t wbase = base + ((uint64_t)anchor << FB_SHIFT);
    const uint32_t jmax = min(TW, nbk - anchor);
    uint32_t wp[TR], bp[TR];  // own: window word | write << 13, bid; else bp = ~0u
#pragma unroll
    for (uint32_t k = 0; k < TR; ++k) {
      const uint32_t i = k * TB + threadIdx.x;
      bp[k] = ~0u;
      wp[k] = 0;
      if (i >= m) continue;
      const uint4 r = reinterpret_cast<const uint4*>(ev + r0)[i];
      uint32_t rel;
      const uint32_t j = win_slot(r, wbase, jmax, &rel);
      if (j == ~0u) continue;
      const uint32_t w = (rel >> 2) & (FB_WORDS - 1u);
      if (((ok >> j) & 1u) && !((sbits[j * TBW + (w >> 5)] >> (w & 31u)) & 1u)) {
        wp[k] = (j * FB_WORDS + (w ^ ((w >> 5) & 31u))) | (((r.y >> 12) & 1u) << 13);
        bp[k] = r.w & 0xFFFFFFu;
      }
    }
#pragma unroll
    for (uint32_t k = 0; k < TR; ++k)
      if (bp[k] != ~0u) tag[wp[k] & (TWW - 1)] = bp[k];
    __syncthreads();
#pragma unroll
    for (uint32_t k = 0; k < TR; ++k) {
      if (bp[k] == ~0u) continue;
      const uint32_t x = wp[k] & (TWW - 1);
      const uint32_t f = ((tag[x] & (MCKG_MAX_BID - 1)) != bp[k] ? TAG_MULTI : 0u) | ((wp[k] & TWW) ? TAG_WRITE : 0u);
      if (f) atomicOr(tag + x, f);
    }
    __syncthreads();
    uint32_t cm = 0;
#pragma unroll
    for (uint32_t k = 0; k < TR; ++k)
      if (bp[k] != ~0u && (tag[wp[k] & (TWW - 1)] & (TAG_MULTI | TAG_WRITE)) == (TAG_MULTI | TAG_WRITE))
        cm |= 1u << k;
    const uint32_t c = __popc(cm);
    uint32_t pos = c ? atomicAdd(&s_nc, c) : 0u;
    for (uint32_t q = cm; q; q &= q - 1u, ++pos)
      if (pos < 32) cl[pos] = reinterpret_cast<const uint4*>(ev)[r0 + (uint64_t)((__ffs(q) - 1) * TB + threadIdx.x)];
    __syncthreads();
    const uint32_t nc = s_nc;
    if (nc > 32) {
      // too many candidates for one exact batch: the tile's own records join
      // the side list (all of them: every record on their words is here)
      uint32_t om = 0;
#pragma unroll
      for (uint32_t k = 0; k < TR; ++k) om |= (bp[k] != ~0u ? 1u : 0u) << k;
      const uint32_t os = side_slot(om, &s_cnt);
      __syncthreads();
      if (threadIdx.x == 0) s_base = atomicAdd(nside, (unsigned long long)s_cnt);
      __syncthreads();
      if (om) side_write(om, os, s_base, ev, r0, side);
    } else if (nc && threadIdx.x < 32) {
      fb_exact(O, cl, nc, C, stg, nstg, flags);
    }
    __syncthreads();  // tables reused by the next tile
  }
  if (threadIdx.x < 32) {
    fb_flush(O, stg, nstg, flags);
    if (C.line != 0xFFFFFFFFu) atomicMin(O.line_first + C.line, C.ts);
    flags = __reduce_or_sync(0xFFFFFFFFu, flags);
    if (threadIdx.x == 0 && flags) atomicOr(O.status, flags);
  }
}

// shared-memory layout of bucket_detect (bytes)
constexpr uint32_t BD_WKEY = 0;
constexpr uint32_t BD_WTAG = BD_WKEY + BWS * 8;
constexpr uint32_t BD_WFLAG = BD_WTAG + BWS * 4;
constexpr uint32_t BD_BKEY = BD_WFLAG + BWS * 4;
constexpr uint32_t BD_BMIN = BD_BKEY + BBS * 8;
constexpr uint32_t BD_DKEY = BD_BMIN + BBS * 32;
constexpr uint32_t BD_CAND = BD_DKEY + BDS * 8;
constexpr uint32_t BD_SMEM = BD_CAND + BCC * 4;

// One CTA per bucket (grid-stride); buckets over BCAP records or whose tables
// overflow go to the big list.
__global__ void __launch_bounds__(BT) bucket_detect_kernel(const mckg_gaccess* recs, const uint64_t* off, uint32_t nb,
                                                           uint32_t shift, uint64_t base, const uint32_t* list,
                                                           const uint32_t* nlist, BOut O, uint32_t* big,
                                                           uint32_t* nbig) {
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ uint32_t s_line[BLT];
  __shared__ unsigned long long s_lts[BLT];
  __shared__ uint32_t s_cnt[1], s_flag[1];
  BTab T;
  T.wkey = reinterpret_cast<unsigned long long*>(sm + BD_WKEY);
  T.wtag = reinterpret_cast<uint32_t*>(sm + BD_WTAG);
  T.wflag = reinterpret_cast<uint32_t*>(sm + BD_WFLAG);
  T.wmask = BWS - 1;
  T.bkey = reinterpret_cast<unsigned long long*>(sm + BD_BKEY);
  T.bmin = reinterpret_cast<unsigned long long*>(sm + BD_BMIN);
  T.bmask = BBS - 1;
  T.dkey = reinterpret_cast<unsigned long long*>(sm + BD_DKEY);
  T.dmask = BDS - 1;
  T.cand = reinterpret_cast<uint32_t*>(sm + BD_CAND);
  T.ccap = BCC;
  for (uint32_t i = threadIdx.x; i < BWS; i += BT) T.wkey[i] = KEMPTY;
  for (uint32_t i = threadIdx.x; i < BBS; i += BT) T.bkey[i] = KEMPTY;
  for (uint32_t i = threadIdx.x; i < BDS; i += BT) T.dkey[i] = KEMPTY;
  for (uint32_t i = threadIdx.x; i < BLT; i += BT) {
    s_line[i] = 0xFFFFFFFFu;
    s_lts[i] = ~0ull;
  }
  __syncthreads();
  uint32_t stamp = 0;
  const uint32_t nwork = list ? *nlist : nb;
  for (uint32_t jb = blockIdx.x; jb < nwork; jb += gridDim.x) {
    const uint32_t b = list ? list[jb] : jb;
    const uint64_t o0 = off[b], m = off[b + 1] - o0;
    if (m < 2) continue;  // a lone record cannot race
    if (m > BCAP) {
      if (threadIdx.x == 0) big[atomicAdd(nbig, 1u)] = b;
      continue;
    }
    // stamps 1..255 (the dedup keys keep 8 bits): re-clear the tables on wrap
    if (++stamp == 256u) {
      stamp = 1;
      for (uint32_t i = threadIdx.x; i < BWS; i += BT) T.wkey[i] = KEMPTY;
      for (uint32_t i = threadIdx.x; i < BBS; i += BT) T.bkey[i] = KEMPTY;
      for (uint32_t i = threadIdx.x; i < BDS; i += BT) T.dkey[i] = KEMPTY;
      __syncthreads();
    }
    uint64_t blo, bhi;
    bucket_range(b, nb, shift, base, &blo, &bhi);
    if (!detect_bucket(recs + o0, (uint32_t)m, blo, bhi, T, stamp, O, s_line, s_lts, s_cnt, s_flag)) {
      if (threadIdx.x == 0) big[atomicAdd(nbig, 1u)] = b;
      __syncthreads();
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < BLT; i += BT)
    if (s_line[i] != 0xFFFFFFFFu) atomicMin(O.line_first + s_line[i], s_lts[i]);
}

// One big bucket with tables in global memory (zeroed by the caller, stamp 1).
__global__ void __launch_bounds__(BT) bucket_detect_big_kernel(const mckg_gaccess* recs, const uint64_t* off,
                                                               uint32_t b, uint32_t nb, uint32_t shift, uint64_t base,
                                                               BTab T, BOut O) {
  __shared__ uint32_t s_line[BLT];
  __shared__ unsigned long long s_lts[BLT];
  __shared__ uint32_t s_cnt[1], s_flag[1];
  for (uint32_t i = threadIdx.x; i < BLT; i += BT) {
    s_line[i] = 0xFFFFFFFFu;
    s_lts[i] = ~0ull;
  }
  __syncthreads();
  const uint64_t o0 = off[b], m = off[b + 1] - o0;
  uint64_t blo, bhi;
  bucket_range(b, nb, shift, base, &blo, &bhi);
  if (!detect_bucket(recs + o0, (uint32_t)m, blo, bhi, T, 1u, O, s_line, s_lts, s_cnt, s_flag) && threadIdx.x == 0)
    atomicOr(O.status, (uint32_t)MCKG_ST_RANGE);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < BLT; i += BT)
    if (s_line[i] != 0xFFFFFFFFu) atomicMin(O.line_first + s_line[i], s_lts[i]);
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
  PoolGuard pg(s);
  unsigned long long* cursor = nullptr;
  MCKG_CUDA_TRY(cudaMemsetAsync(counts, 0, n_ranks * sizeof(uint64_t), s));
  MCKG_CUDA_TRY(pg.alloc(&cursor, n_ranks * sizeof(unsigned long long)));
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
  add_launches(2);
  return MCKG_OK;
}

namespace mckg {
namespace {

// the sampled address span of n records: {min, max} over a strided sample
int sample_span(const mckg_gaccess* events, uint64_t n, unsigned long long hm[2], cudaStream_t s,
                uint32_t& launches) {
  PoolGuard pg(s);
  unsigned long long* mm = nullptr;
  MCKG_CUDA_TRY(pg.alloc(&mm, 2 * sizeof(unsigned long long)));
  const unsigned long long init[2] = {~0ull, 0ull};
  MCKG_CUDA_TRY(cudaMemcpyAsync(mm, init, sizeof init, cudaMemcpyHostToDevice, s));
  const uint64_t stride = n > (1u << 16) ? n >> 16 : 1;
  span_sample_kernel<<<grid_for(n / stride), 256, 0, s>>>(events, n, stride, mm);
  ++launches;
  MCKG_CUDA_TRY(cudaMemcpyAsync(hm, mm, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
  MCKG_CUDA_TRY(cudaStreamSynchronize(s));
  return MCKG_OK;
}

// The bucket pipeline on n >= 1 records: span, count, scan, scatter, detect.
int detect_buckets(const mckg_gaccess* events, uint64_t n, const BOut& O, cudaStream_t s, uint32_t& launches,
                   const unsigned long long* span_in = nullptr) {
  unsigned long long hm[2];
  if (span_in) {  // a span known to the caller (buckets are open at both ends)
    hm[0] = span_in[0];
    hm[1] = span_in[1];
  } else if (int rc = sample_span(events, n, hm, s, launches)) {
    return rc;
  }
  uint32_t* status = O.status;
  // the sample can miss the extremes: the edge buckets are open, and a
  // margin keeps the top records out of one crowded last bucket
  const uint64_t base = hm[0] & ~0xFFFull;
  const uint64_t span = (hm[1] + 16 - base) + ((hm[1] - base) >> 6) + 65536;
  // dense spans: 4 KiB buckets for the warp-per-bucket kernel; sparse ones:
  // buckets sized for ~256 records, hashed tables only
  const bool dense = (span >> FB_SHIFT) + 1 <= 2 * n + 1024 && !(debug_flags() & 128u);
  uint32_t shift = FB_SHIFT;
  if (!dense) {
    const uint64_t want_nb = (n + 255) / 256;
    shift = 4;
    while (shift < 40 && (span >> shift) > want_nb) ++shift;
  }
  const uint32_t nb = (uint32_t)((span >> shift) + 1);
  // 2-4. count, scan, scatter
  PoolGuard pg(s);
  uint32_t *cnt = nullptr, *cur = nullptr, *big = nullptr;
  uint64_t* off = nullptr;
  mckg_gaccess* recs = nullptr;
  MCKG_CUDA_TRY(pg.alloc(&cnt, (size_t)nb * 4));
  MCKG_CUDA_TRY(pg.alloc(&cur, (size_t)nb * 4));
  MCKG_CUDA_TRY(pg.alloc(&off, ((size_t)nb + 1) * 8));
  MCKG_CUDA_TRY(pg.alloc(&big, ((size_t)nb + 1) * 4));
  MCKG_CUDA_TRY(cudaMemsetAsync(cnt, 0, (size_t)nb * 4, s));
  MCKG_CUDA_TRY(cudaMemsetAsync(cur, 0, (size_t)nb * 4, s));
  MCKG_CUDA_TRY(cudaMemsetAsync(big, 0, 4, s));
  const uint32_t g = grid_for(n, 16);
  bucket_count_kernel<<<g, 256, 0, s>>>(events, n, nb, shift, base, cnt, status);
  MCKG_CUDA_TRY(exclusive_scan_u32(cnt, nb, off, s, &launches));
  MCKG_CUDA_TRY(cudaGetLastError());
  // a record counts once per bucket it touches (at most two): 2n slots
  // bound the layout without waiting for the count
  MCKG_CUDA_TRY(pg.alloc(&recs, 2 * n * sizeof(mckg_gaccess)));
  bucket_scatter_kernel<<<g, 256, 0, s>>>(events, n, nb, shift, base, off, cur, recs);
  launches += 2;
  // 5. detection
  MCKG_CUDA_TRY(cudaFuncSetAttribute(bucket_detect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, BD_SMEM));
  MCKG_CUDA_TRY(cudaFuncSetAttribute(bucket_detect_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int per = 0;
  MCKG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, bucket_detect_kernel, BT, BD_SMEM));
  const uint32_t gd = (uint32_t)sm_count() * (uint32_t)(per > 0 ? per : 1);
  if (dense) {
    // warp per bucket; the buckets it hands back go to the general kernel
    uint32_t* mid = nullptr;
    MCKG_CUDA_TRY(pg.alloc(&mid, ((size_t)nb + 2) * 4));
    MCKG_CUDA_TRY(cudaMemsetAsync(mid, 0, 8, s));  // [0] handed-back buckets, [1] claim counter
    MCKG_CUDA_TRY(cudaFuncSetAttribute(bucket_fast_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FB_SMEM));
    MCKG_CUDA_TRY(cudaFuncSetAttribute(bucket_fast_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    int pf = 0;
    MCKG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pf, bucket_fast_kernel, FB_WARPS * 32, FB_SMEM));
    const uint32_t gf = (uint32_t)sm_count() * (uint32_t)(pf > 0 ? pf : 1);
    bucket_fast_kernel<<<gf, FB_WARPS * 32, FB_SMEM, s>>>(recs, off, nb, base, O, mid + 2, mid, mid + 1);
    bucket_detect_kernel<<<gd, BT, BD_SMEM, s>>>(recs, off, nb, shift, base, mid + 2, mid, O, big + 1, big);
    MCKG_CUDA_TRY(cudaGetLastError());
      launches += 2;
  } else {
    bucket_detect_kernel<<<gd < nb ? gd : nb, BT, BD_SMEM, s>>>(recs, off, nb, shift, base, nullptr, nullptr, O,
                                                                 big + 1, big);
    MCKG_CUDA_TRY(cudaGetLastError());
    ++launches;
  }
  uint32_t nbig = 0;
  MCKG_CUDA_TRY(cudaMemcpyAsync(&nbig, big, 4, cudaMemcpyDeviceToHost, s));
  MCKG_CUDA_TRY(cudaStreamSynchronize(s));
  if (nbig) {
    // the rare path: one bucket at a time, tables in global memory
    std::vector<uint32_t> bl(nbig);
    MCKG_CUDA_TRY(cudaMemcpy(bl.data(), big + 1, nbig * 4, cudaMemcpyDeviceToHost));
    for (uint32_t b : bl) {
      uint64_t ob[2];
      MCKG_CUDA_TRY(cudaMemcpy(ob, off + b, sizeof ob, cudaMemcpyDeviceToHost));
      const uint64_t m = ob[1] - ob[0];
      if (m > (1ull << 26)) {
        set_error("mckg_detect_global: more than 2^26 records in one address bucket");
        return MCKG_E_RANGE;
      }
      auto pow2 = [](uint64_t x) {
        uint64_t p = 64;
        while (p < x) p <<= 1;
        return p;
      };
      const uint64_t ws = pow2(6 * m), bs = pow2(16 * m), ds = pow2(16 * m);
      uint8_t* scratch = nullptr;
      const size_t cand_bytes = (m * 4 + 15) & ~(size_t)15;  // keeps the 8-byte tables aligned
      const size_t bytes = ws * 16 + cand_bytes + bs * 40 + ds * 8;
      PoolGuard sg(s);
      MCKG_CUDA_TRY(sg.alloc(&scratch, bytes));
      MCKG_CUDA_TRY(cudaMemsetAsync(scratch, 0, bytes, s));
      BTab T;
      T.wkey = reinterpret_cast<unsigned long long*>(scratch);
      T.wtag = reinterpret_cast<uint32_t*>(scratch + ws * 8);
      T.wflag = reinterpret_cast<uint32_t*>(scratch + ws * 12);
      T.wmask = (uint32_t)(ws - 1);
      T.cand = reinterpret_cast<uint32_t*>(scratch + ws * 16);
      T.ccap = (uint32_t)m;
      T.bkey = reinterpret_cast<unsigned long long*>(scratch + ws * 16 + cand_bytes);
      T.bmin = reinterpret_cast<unsigned long long*>(scratch + ws * 16 + cand_bytes + bs * 8);
      T.bmask = (uint32_t)(bs - 1);
      T.dkey = reinterpret_cast<unsigned long long*>(scratch + ws * 16 + cand_bytes + bs * 40);
      T.dmask = (uint32_t)(ds - 1);
      bucket_detect_big_kernel<<<1, BT, 0, s>>>(recs, off, b, nb, shift, base, T, O);
      MCKG_CUDA_TRY(cudaGetLastError());
      ++launches;
    }
  }
  return MCKG_OK;
}

// The tile path (see tile_claim_kernel): returns false (nothing launched
// that reports) when the span is too wide for its bitmap.
int detect_tiles(const mckg_gaccess* events, uint64_t n, const BOut& O, cudaStream_t s, uint32_t& launches,
                 bool& used) {
  used = false;
  unsigned long long hm[2];
  if (int rc = sample_span(events, n, hm, s, launches)) return rc;
  // window buckets live in the sampled span (records outside it are
  // foreign), widened on both sides: the sample can miss the extremes, and
  // the records it misses would otherwise all be foreign in one edge bucket
  const uint64_t margin = ((hm[1] - hm[0]) >> 6) + 65536;
  hm[0] = hm[0] > margin ? hm[0] - margin : 0;
  hm[1] = hm[1] + margin;
  const uint64_t base = hm[0] & ~(uint64_t)((1u << FB_SHIFT) - 1);
  const uint64_t nbk64 = ((hm[1] - base) >> FB_SHIFT) + 1;
  if (nbk64 >= (1ull << 23)) return MCKG_OK;  // >= 16 GiB: anchors keep 23 bits (the bitmap is span / 32)
  if (reinterpret_cast<uintptr_t>(events) & 15u) return MCKG_OK;  // the bulk copies need 16-byte alignment
  used = true;
  const uint32_t nbk = (uint32_t)nbk64;
  const uint64_t ntiles = (n + TT - 1) / TT;
  PoolGuard pg(s);
  uint32_t *claim = nullptr, *bits = nullptr;
  unsigned long long* win = nullptr;
  mckg_gaccess* side = nullptr;
  unsigned long long* nside = nullptr;
  MCKG_CUDA_TRY(pg.alloc(&claim, (size_t)nbk * 4));
  MCKG_CUDA_TRY(pg.alloc(&bits, (size_t)nbk * (FB_WORDS / 8)));
  MCKG_CUDA_TRY(pg.alloc(&win, (size_t)ntiles * 8));
  MCKG_CUDA_TRY(pg.alloc(&side, (size_t)n * sizeof(mckg_gaccess)));  // each record joins at most once
  MCKG_CUDA_TRY(pg.alloc(&nside, 8));
  MCKG_CUDA_TRY(cudaMemsetAsync(claim, 0, (size_t)nbk * 4, s));
  MCKG_CUDA_TRY(cudaMemsetAsync(bits, 0, (size_t)nbk * (FB_WORDS / 8), s));
  MCKG_CUDA_TRY(cudaMemsetAsync(nside, 0, 8, s));
  uint32_t* multi = nullptr;  // [ntiles] tiles for tile_multi, then their count
  MCKG_CUDA_TRY(pg.alloc(&multi, ((size_t)ntiles + 1) * 4));
  MCKG_CUDA_TRY(cudaMemsetAsync(multi + ntiles, 0, 4, s));
  // pass 1 from pass 0's codes (debug 1024: every tile re-read instead)
  const bool compact = !(debug_flags() & 1024u);
  uint16_t* code = nullptr;  // [ntiles * TT] window word per record
  uint8_t* tmulti = nullptr;  // [ntiles] in-window records from >= 2 blocks
  uint32_t* full = nullptr;  // [ntiles] tiles for the full pass 1, then their count
  if (compact) {
    MCKG_CUDA_TRY(pg.alloc(&code, (size_t)ntiles * TT * 2));
    MCKG_CUDA_TRY(pg.alloc(&tmulti, (size_t)ntiles));
    MCKG_CUDA_TRY(pg.alloc(&full, ((size_t)ntiles + 1) * 4));
    MCKG_CUDA_TRY(cudaMemsetAsync(full + ntiles, 0, 4, s));
  }
  MCKG_CUDA_TRY(cudaFuncSetAttribute(tile_claim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TC_SMEM));
  MCKG_CUDA_TRY(cudaFuncSetAttribute(tile_claim_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  MCKG_CUDA_TRY(cudaFuncSetAttribute(tile_detect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TD_SMEM));
  MCKG_CUDA_TRY(cudaFuncSetAttribute(tile_detect_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
  int pc = 0, pd = 0;
  MCKG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pc, tile_claim_kernel, TB, TC_SMEM));
  MCKG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pd, tile_detect_kernel, TB, TD_SMEM));
  const uint64_t gc = std::min<uint64_t>(ntiles, (uint64_t)sm_count() * (uint64_t)(pc > 0 ? pc : 1));
  const uint64_t gdt = std::min<uint64_t>(ntiles, (uint64_t)sm_count() * (uint64_t)(pd > 0 ? pd : 1));
  tile_claim_kernel<<<(unsigned)gc, TB, TC_SMEM, s>>>(events, n, ntiles, base, nbk, claim, bits, win, side, nside,
                                                      code, tmulti);
  if (compact) {
    int pm = 0;
    MCKG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&pm, tile_mixed_kernel, TB, 0));
    const uint64_t gm = std::min<uint64_t>((ntiles + TB / 32 - 1) / (TB / 32),
                                           (uint64_t)sm_count() * (uint64_t)(pm > 0 ? pm : 1));
    tile_mixed_kernel<<<(unsigned)gm, TB, 0, s>>>(events, ntiles, claim, bits, win, code, tmulti, side, nside, full,
                                                  full + ntiles);
    ++launches;
  }
  tile_detect_kernel<<<(unsigned)gdt, TB, TD_SMEM, s>>>(events, n, ntiles, base, nbk, claim, bits, win, side, nside,
                                                        multi, multi + ntiles, compact ? full : nullptr,
                                                        compact ? full + ntiles : nullptr);
  MCKG_CUDA_TRY(cudaFuncSetAttribute(tile_multi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TM_SMEM));
  tile_multi_kernel<<<(unsigned)gdt, TB, TM_SMEM, s>>>(events, n, base, nbk, claim, bits, win, multi, multi + ntiles,
                                                       side, nside, O);
  MCKG_CUDA_TRY(cudaGetLastError());
  launches += 3;
  unsigned long long ns = 0;
  MCKG_CUDA_TRY(cudaMemcpyAsync(&ns, nside, 8, cudaMemcpyDeviceToHost, s));
  MCKG_CUDA_TRY(cudaStreamSynchronize(s));
  int rc = ns ? detect_buckets(side, ns, O, s, launches, hm) : MCKG_OK;
  return rc;
}

}  // namespace
}  // namespace mckg

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
  (void)addr_lo;  // buckets follow the sampled span of the records themselves
  cudaStream_t s = (cudaStream_t)stream;
  keep_pool_memory();
  MCKG_CUDA_TRY(cudaMemsetAsync(n_races, 0, sizeof(unsigned long long), s));
  if (n == 0) return MCKG_OK;
  uint32_t launches = 0;
  const BOut O{races, capacity, n_races, line_first, status};
  // the tile path for large inputs (debug 512: always, 256: never)
  const uint32_t dbg = debug_flags();
  bool used = false;
  int rc = MCKG_OK;
  if (!(dbg & 256u) && (n >= (1ull << 20) || (dbg & 512u))) rc = detect_tiles(events, n, O, s, launches, used);
  if (rc == MCKG_OK && !used) rc = detect_buckets(events, n, O, s, launches);
  add_launches(launches);
  return rc;
}
