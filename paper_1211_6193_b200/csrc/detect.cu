// detect.cu -- K2: block-local shared-memory race detector (sm_100a).
//
// Replaces Machine::recordAccess / Machine::clearEpoch (racecheck.cpp:9-73)
// for a whole grid at once.  Reference semantics: for every access X to byte
// b of a block's shared object, X races iff an EARLIER access to b in the same
// barrier epoch came from another thread and X or it is a write; a racing
// (obj, b, line(X)) is reported once per run (RaceState::reported,
// machine.hpp:91) and the Race diagnostic of a line appears at its first
// racing access (addDiagnostic dedup, machine.cpp:41-46).
//
// Design (one CTA streams many simulated blocks; blocks never
// interact because each owns its shared object, device.cpp:33-38):
//   1. stage: the block's 16-byte records are pulled into shared memory by
//      the TMA engine (cp.async.bulk + mbarrier), NSTAGE blocks in flight;
//      each thread keeps its EPT records (decoded) in registers.
//   2. epochs: a per-block start bitmap (shfl_up + ballot) splits the records
//      into epoch segments (epochs are non-decreasing in timestamp order).
//   3. filter, per epoch, on 4-byte words: P1 tag[w] = some accessing tid;
//      P2 mark words seen by a second tid / written; P3 an event is a
//      candidate iff one of its words is both.  A byte can race only if its
//      word passes, so the filter has no false negatives (a byte has a racing
//      access iff >= 2 threads touch it in the epoch and one writes).  P3 of
//      epoch k and P1 of epoch k+1 share a barrier interval.
//   4. exact pass, once per block over the (rare) candidates, byte-exact and
//      warp-cooperative: X races on the bytes it shares with an earlier
//      candidate Y of the same epoch and another thread where X or Y writes --
//      the reference predicate verbatim, restricted to the bytes that can
//      matter.  Lanes hold the Y's; one __reduce_or_sync gives X's racing bytes.
//   5. report: racing (byte, line) pairs are deduplicated per block in a
//      shared hash set (the reported set is per object), staged in shared
//      memory and appended to the global triple array in chunks; the first
//      racing timestamp per line is min-reduced in shared memory, then
//      globally.
#include <cub/cub.cuh>

#include "common.cuh"

namespace mckg {
namespace {

constexpr int NT = 256;
constexpr int NWARP = NT / 32;
constexpr int NSTAGE = 2;
constexpr int EPT_MAX = 16;     // records per thread kept in registers (cap <= 4096)
constexpr uint32_t HS = 1024;   // (byte, line) dedup set entries
constexpr uint32_t TBN = 512;   // staged triples before a global flush
constexpr uint32_t LTN = 32;    // line-first local table entries
constexpr uint32_t INF = 0xFFFFFFFFu;
constexpr uint32_t INV = 0xFFFFFFFFu;
constexpr uint32_t ST_OVERFLOW = MCKG_ST_OVERFLOW, ST_RANGE = MCKG_ST_RANGE,
                   ST_ORDER = MCKG_ST_ORDER, ST_DUP = MCKG_ST_DUP;
// misc[] slots
constexpr int M_TBN = 0, M_CLN = 1, M_BASE_LO = 3, M_BASE_HI = 4, M_FLAGS = 5;

struct Params {
  const mckg_access* ev;
  const uint64_t* bstart;
  uint32_t n_blocks, obj_base, bid_base, shmem_bytes, cap, wpad;
  mckg_race_triple* tri;
  unsigned long long capacity;
  unsigned long long* n_tri;
  unsigned long long* line_first;
  uint32_t* status;
};

extern __shared__ __align__(128) uint8_t smem_raw[];

// Byte offsets into the dynamic shared memory (32-bit, so every access is a
// plain LDS/STS with a register offset).
struct Lay {
  uint32_t stage, tag, multi, anyw, hset, lt_ts, tbuf, lt_line, bitmap, cl, mbar, misc, end;
};

__host__ __device__ inline Lay layout(uint32_t cap, uint32_t wpad) {
  Lay L;
  uint32_t p = 0;
  L.stage = p;   p += NSTAGE * cap * 16;
  L.tag = p;     p += wpad * 4;
  L.multi = p;   p += wpad * 4;
  L.anyw = p;    p += wpad * 4;
  L.hset = p;    p += HS * 8;
  L.lt_ts = p;   p += LTN * 8;
  L.tbuf = p;    p += TBN * 12;
  L.lt_line = p; p += LTN * 4;
  L.bitmap = p;  p += (cap / 32 + 1) * 4;
  L.cl = p;      p += cap * 2;
  p = (p + 7u) & ~7u;
  L.mbar = p;    p += NSTAGE * 8;
  L.misc = p;    p += 8 * 4;
  L.end = (p + 127u) & ~127u;
  return L;
}

template <typename T>
__device__ __forceinline__ T* sp(uint32_t off) {
  return reinterpret_cast<T*>(smem_raw + off);
}

__device__ __forceinline__ uint32_t sw(uint32_t w) { return w ^ ((w >> 5) & 31u); }

__device__ __forceinline__ bool valid_ev(uint32_t w0, int32_t line, uint32_t shm) {
  uint32_t off = acc_off(w0), len = acc_len(w0);
  return len != 0 && len <= MCKG_MAX_LEN && off + len <= shm && (uint32_t)line < MCKG_MAX_LINES;
}

// 1 = inserted, 0 = already present, 2 = probe limit (caller flags ST_DUP)
__device__ int hset_insert(const Lay& L, unsigned long long key, unsigned long long bstamp) {
  unsigned long long* hs = sp<unsigned long long>(L.hset);
  uint32_t h = (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> 40) & (HS - 1);
  for (uint32_t probe = 0; probe < 64; ++probe) {
    unsigned long long cur = hs[h];
    while ((cur >> 40) != bstamp) {  // stale slot: claim it
      unsigned long long old = atomicCAS(hs + h, cur, key);
      if (old == cur) return 1;
      cur = old;
    }
    if (cur == key) return 0;
    h = (h + 1) & (HS - 1);
  }
  return 2;
}

__device__ void line_note(const Lay& L, const Params& P, int32_t line, unsigned long long ts) {
  uint32_t* lt_line = sp<uint32_t>(L.lt_line);
  unsigned long long* lt_ts = sp<unsigned long long>(L.lt_ts);
  uint32_t l = (uint32_t)line;
  uint32_t h = l & (LTN - 1);
  for (uint32_t probe = 0; probe < LTN; ++probe) {
    uint32_t v = lt_line[h];
    if (v == INF) {
      uint32_t old = atomicCAS(lt_line + h, INF, l);
      v = old == INF ? l : old;
    }
    if (v == l) {
      atomicMin(lt_ts + h, ts);
      return;
    }
    h = (h + 1) & (LTN - 1);
  }
  atomicMin(P.line_first + l, ts);
}

// Flushes the staged triples (uniform call, all threads).
__device__ void flush_tbuf(const Lay& L, const Params& P) {
  uint32_t* misc = sp<uint32_t>(L.misc);
  mckg_race_triple* tbuf = sp<mckg_race_triple>(L.tbuf);
  __syncthreads();
  uint32_t n = misc[M_TBN] < TBN ? misc[M_TBN] : TBN;
  if (n == 0) return;
  if (threadIdx.x == 0) {
    unsigned long long base = atomicAdd(P.n_tri, (unsigned long long)n);
    misc[M_BASE_LO] = (uint32_t)base;
    misc[M_BASE_HI] = (uint32_t)(base >> 32);
  }
  __syncthreads();
  unsigned long long base = ((unsigned long long)misc[M_BASE_HI] << 32) | misc[M_BASE_LO];
  for (uint32_t i = threadIdx.x; i < n; i += NT) {
    if (base + i < P.capacity)
      P.tri[base + i] = tbuf[i];
    else
      atomicOr(misc + M_FLAGS, ST_OVERFLOW);
  }
  __syncthreads();
  if (threadIdx.x == 0) misc[M_TBN] = 0;
}

// Next epoch start at index >= p (bit set in the bitmap), or n.  Uniform.
__device__ uint32_t next_start(const uint32_t* bitmap, uint32_t p, uint32_t n) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t nwords = (n + 31u) / 32u;
  for (uint32_t base = p >> 5; base < nwords; base += 32) {
    uint32_t wi = base + lane;
    uint32_t word = wi < nwords ? bitmap[wi] : 0u;
    if (wi == (p >> 5)) word &= ~0u << (p & 31u);
    uint32_t m = __ballot_sync(0xFFFFFFFFu, word != 0);
    if (m) {
      uint32_t f = __ffs(m) - 1u;
      uint32_t wf = __shfl_sync(0xFFFFFFFFu, word, f);
      uint32_t idx = (base + f) * 32u + (__ffs(wf) - 1u);
      return idx < n ? idx : n;
    }
  }
  return n;
}

// Rare path: the 2nd/3rd word of an access spanning several 4-byte words.
__device__ __noinline__ bool extra_words(const Lay L, uint32_t w0, uint32_t tid, int phase,
                                         uint32_t st16) {
  uint32_t* tag = sp<uint32_t>(L.tag);
  uint32_t* multi = sp<uint32_t>(L.multi);
  uint32_t* anyw = sp<uint32_t>(L.anyw);
  const uint32_t off = acc_off(w0), len = acc_len(w0);
  const bool wr = acc_write(w0);
  bool cand = false;
  for (uint32_t w = (off >> 2) + 1; w <= (off + len - 1u) >> 2; ++w) {
    const uint32_t x = sw(w);
    if (phase == 1) {
      tag[x] = tid;
    } else if (phase == 2) {
      if (tag[x] != tid) multi[x] = st16;
      if (wr) anyw[x] = st16;
    } else {
      cand |= multi[x] == st16 && anyw[x] == st16;
    }
  }
  return cand;
}

// Exact pass over the block's candidate list (all warps; see header).
__device__ void exact_block(const Lay& L, const Params& P, const uint4* src, uint32_t m,
                            uint32_t obj, uint32_t bid, unsigned long long bstamp) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint16_t* cl = sp<uint16_t>(L.cl);
  uint32_t* misc = sp<uint32_t>(L.misc);
  mckg_race_triple* tbuf = sp<mckg_race_triple>(L.tbuf);
  // lanes hold the first 32 candidates (later ones are re-read per X)
  uint32_t yi0 = INV, yx0 = 0, yy0 = 0;
  if (lane < m) {
    yi0 = cl[lane];
    const uint4 Y = src[yi0];
    yx0 = Y.x;
    yy0 = Y.y;
  }
  for (uint32_t xp = warp; xp < m; xp += NWARP) {
    const uint32_t xi = cl[xp];
    const uint4 X = src[xi];
    const uint32_t xoff = acc_off(X.x), xend = xoff + acc_len(X.x);
    const uint32_t xtid = acc_tid(X.y), xep = acc_epoch(X.y);
    const bool xw = acc_write(X.x);
    uint32_t bits = 0;
    for (uint32_t base = 0; base < m; base += 32) {
      uint32_t yi, yx, yy;
      if (base == 0) {
        yi = yi0; yx = yx0; yy = yy0;
      } else {
        yi = INV; yx = 0; yy = 0;
        if (base + lane < m) {
          yi = cl[base + lane];
          const uint4 Y = src[yi];
          yx = Y.x;
          yy = Y.y;
        }
      }
      if (yi < xi && acc_epoch(yy) == xep && acc_tid(yy) != xtid && (xw || acc_write(yx))) {
        const uint32_t yoff = acc_off(yx), yend = yoff + acc_len(yx);
        const uint32_t lo = max(xoff, yoff), hi = min(xend, yend);
        if (lo < hi) bits |= ((1u << (hi - lo)) - 1u) << (lo - xoff);
      }
    }
    bits = __reduce_or_sync(0xFFFFFFFFu, bits);
    if (!bits) continue;
    const int32_t line = (int32_t)X.z;
    // lanes q < 8 report byte xoff + q
    bool fresh = false;
    if (lane < 8 && ((bits >> lane) & 1u)) {
      const uint32_t byte = xoff + lane;
      const unsigned long long key = (bstamp << 40) |
                                     ((unsigned long long)(byte & 0xFFFFFu) << 16) |
                                     ((uint32_t)line & 0xFFFFu);
      const int r = hset_insert(L, key, bstamp);
      if (r == 2) atomicOr(misc + M_FLAGS, ST_DUP);
      fresh = r != 0;
    }
    const uint32_t fm = __ballot_sync(0xFFFFFFFFu, fresh);
    if (fm) {
      uint32_t pos = 0;
      if (lane == 0) pos = atomicAdd(misc + M_TBN, (uint32_t)__popc(fm));
      pos = __shfl_sync(0xFFFFFFFFu, pos, 0) + __popc(fm & ((1u << lane) - 1u));
      if (fresh) {
        const mckg_race_triple tr{obj, xoff + lane, line};
        if (pos < TBN) {
          tbuf[pos] = tr;
        } else {
          unsigned long long gp = atomicAdd(P.n_tri, 1ull);
          if (gp < P.capacity)
            P.tri[gp] = tr;
          else
            atomicOr(misc + M_FLAGS, ST_OVERFLOW);
        }
      }
    }
    if (lane == 0) line_note(L, P, line, ts_key(X.w, bid, xtid));
  }
}

template <int EPT>
__device__ void process_block(const Lay& L, const Params& P, const uint4* src, uint32_t n,
                              uint32_t obj, uint32_t bid, uint32_t& stamp,
                              unsigned long long bstamp) {
  const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
  const uint32_t shm = P.shmem_bytes;
  uint32_t* tag = sp<uint32_t>(L.tag);
  uint32_t* multi = sp<uint32_t>(L.multi);
  uint32_t* anyw = sp<uint32_t>(L.anyw);
  uint32_t* bitmap = sp<uint32_t>(L.bitmap);
  uint16_t* cl = sp<uint16_t>(L.cl);
  uint32_t* misc = sp<uint32_t>(L.misc);
  // Per owned record i = k*NT + t: epoch, first word (swizzled; INV = skip),
  // and meta = tid | write << 11 | spans-several-words << 12.
  uint32_t ep[EPT], x0[EPT], meta[EPT];
  uint32_t flags = 0;
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const uint32_t i = (uint32_t)k * NT + t;
    const bool in = i < n;
    const uint4 r = in ? src[i] : make_uint4(0, 0, 0, 0);
    ep[k] = acc_epoch(r.y);
    uint32_t prev = __shfl_up_sync(0xFFFFFFFFu, ep[k], 1);
    if (lane == 0 && in && i > 0) prev = acc_epoch(src[i - 1].y);
    const bool start = in && (i == 0 || ep[k] != prev);
    if (in && i > 0 && ep[k] < prev) flags |= ST_ORDER;
    const bool ok = in && valid_ev(r.x, (int32_t)r.z, shm);
    if (in && !ok) flags |= ST_RANGE;
    const uint32_t off = acc_off(r.x), len = acc_len(r.x);
    x0[k] = ok ? sw(off >> 2) : INV;
    meta[k] = acc_tid(r.y) | (acc_write(r.x) << 11) |
              ((uint32_t)(((off & 3u) + len) > 4u) << 12);
    const uint32_t bm = __ballot_sync(0xFFFFFFFFu, start);
    if (lane == 0 && (uint32_t)k * NT < n) bitmap[(uint32_t)k * NWARP + warp] = bm;
  }
  flags = __reduce_or_sync(0xFFFFFFFFu, flags);
  if (lane == 0 && flags) atomicOr(misc + M_FLAGS, flags);

  auto p1 = [&](uint32_t cur, uint32_t st) {
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      if (ep[k] == cur && x0[k] != INV) {
        const uint32_t tid = meta[k] & 0x7FFu;
        tag[x0[k]] = tid;
        if (meta[k] & 0x1000u) extra_words(L, src[k * NT + t].x, tid, 1, st);
      }
    }
  };
  uint32_t s = 0;
  uint32_t cur = acc_epoch(src[0].y);
  uint32_t st = ++stamp;
  p1(cur, st);
  if (t == 0) misc[M_CLN] = 0;
  __syncthreads();
  while (true) {
    // P2: words seen by a second thread; written words
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      if (ep[k] == cur && x0[k] != INV) {
        const uint32_t tid = meta[k] & 0x7FFu;
        if (tag[x0[k]] != tid) multi[x0[k]] = st;
        if (meta[k] & 0x800u) anyw[x0[k]] = st;
        if (meta[k] & 0x1000u) extra_words(L, src[k * NT + t].x, tid, 2, st);
      }
    }
    __syncthreads();
    const uint32_t e = next_start(bitmap, s + 1, n);
    // P3: candidates -> block list cl (warp-aggregated compaction)
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      bool cand = false;
      if (ep[k] == cur && x0[k] != INV) {
        cand = multi[x0[k]] == st && anyw[x0[k]] == st;
        if (meta[k] & 0x1000u) cand |= extra_words(L, src[k * NT + t].x, meta[k] & 0x7FFu, 3, st);
      }
      const uint32_t bm = __ballot_sync(0xFFFFFFFFu, cand);
      if (bm) {
        const uint32_t leader = __ffs(bm) - 1u;
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(misc + M_CLN, (uint32_t)__popc(bm));
        base = __shfl_sync(0xFFFFFFFFu, base, leader);
        if (cand) cl[base + __popc(bm & ((1u << lane) - 1u))] = (uint16_t)((uint32_t)k * NT + t);
      }
    }
    const bool more = e < n;
    if (more) {  // P1 of the next epoch shares this barrier interval
      s = e;
      cur = acc_epoch(src[s].y);
      st = ++stamp;
      p1(cur, st);
    }
    __syncthreads();
    if (!more) break;
  }
  const uint32_t m = misc[M_CLN];
  if (m) exact_block(L, P, src, m, obj, bid, bstamp);
}

template <int EPT>
__global__ void __launch_bounds__(NT, EPT <= 4 ? 3 : (EPT <= 8 ? 2 : 1))
    race_detect_kernel(Params P) {
  const Lay L = layout(P.cap, P.wpad);
  const uint32_t t = threadIdx.x;
  unsigned long long* hset = sp<unsigned long long>(L.hset);
  uint32_t* lt_line = sp<uint32_t>(L.lt_line);
  unsigned long long* lt_ts = sp<unsigned long long>(L.lt_ts);
  uint32_t* misc = sp<uint32_t>(L.misc);
  uint64_t* mbar = sp<uint64_t>(L.mbar);
  uint4* stage = sp<uint4>(L.stage);
  for (uint32_t i = t; i < HS; i += NT) hset[i] = 0ull;
  for (uint32_t i = t; i < LTN; i += NT) {
    lt_line[i] = INF;
    lt_ts[i] = ~0ull;
  }
  for (uint32_t i = t; i < 3 * P.wpad; i += NT) sp<uint32_t>(L.tag)[i] = 0u;
  if (t < 8) misc[t] = 0u;
  if (t == 0) {
    for (int k = 0; k < NSTAGE; ++k) mbar_init(mbar + k, 1);
    fence_mbar_init();
  }
  __syncthreads();

  const uint32_t G = gridDim.x;
  auto fits = [&](uint32_t b) {
    uint64_t n = P.bstart[b + 1] - P.bstart[b];
    return n > 0 && n <= P.cap;
  };
  auto issue = [&](uint32_t b, int st) {
    uint64_t s0 = P.bstart[b];
    uint32_t bytes = (uint32_t)((P.bstart[b + 1] - s0) * 16);
    mbar_expect_tx(mbar + st, bytes);
    bulk_g2s(stage + (size_t)st * P.cap, P.ev + s0, bytes, mbar + st);
  };
  if (t == 0) {
    for (int k = 0; k < NSTAGE; ++k) {
      uint32_t b = blockIdx.x + (uint32_t)k * G;
      if (b < P.n_blocks && fits(b)) issue(b, k);
    }
  }
  uint32_t phase = 0;
  uint32_t stamp = 0;
  unsigned long long bstamp = 0;
  int it = 0;
  for (uint32_t b = blockIdx.x; b < P.n_blocks; b += G, ++it) {
    const int st = it % NSTAGE;
    const uint64_t n_all = P.bstart[b + 1] - P.bstart[b];
    const uint32_t n = n_all <= P.cap ? (uint32_t)n_all : 0u;
    ++bstamp;
    if (n > 0) {
      mbar_wait(mbar + st, (phase >> st) & 1u);
      phase ^= 1u << st;
      process_block<EPT>(L, P, stage + (size_t)st * P.cap, n, P.obj_base + b, P.bid_base + b,
                         stamp, bstamp);
    } else if (n_all > 0 && t == 0) {
      atomicOr(misc + M_FLAGS, ST_RANGE);  // block larger than the staging capacity
    }
    __syncthreads();  // stage `st` fully consumed (including the exact pass)
    if (t == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const uint32_t nb = b + (uint32_t)NSTAGE * G;
      if (nb < P.n_blocks && fits(nb)) issue(nb, st);
    }
    if (misc[M_TBN] >= TBN / 2) flush_tbuf(L, P);
  }
  flush_tbuf(L, P);
  __syncthreads();
  for (uint32_t i = t; i < LTN; i += NT)
    if (lt_line[i] != INF) atomicMin(P.line_first + lt_line[i], lt_ts[i]);
  if (t == 0 && misc[M_FLAGS]) atomicOr(P.status, misc[M_FLAGS]);
}

__global__ void reset_kernel(unsigned long long* n_tri, unsigned long long* line_first,
                             uint32_t* status) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < MCKG_MAX_LINES) line_first[i] = ~0ull;
  if (i == 0) {
    *n_tri = 0;
    *status = 0;
  }
}

__global__ void encode_triples(const mckg_race_triple* t, unsigned long long* k, uint64_t n,
                               uint32_t obj_base) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  mckg_race_triple x = t[i];
  k[i] = ((unsigned long long)((x.obj - obj_base) & 0x3FFFFFu) << 36) |
         ((unsigned long long)(x.byte & 0xFFFFFu) << 16) | ((uint32_t)x.line & 0xFFFFu);
}

__global__ void decode_triples(const unsigned long long* k, mckg_race_triple* t,
                               const unsigned long long* n_dev, uint64_t n, uint32_t obj_base) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (n_dev && i >= *n_dev) return;
  if (i >= n) return;
  unsigned long long v = k[i];
  t[i] = mckg_race_triple{obj_base + (uint32_t)(v >> 36), (uint32_t)((v >> 16) & 0xFFFFFu),
                          (int32_t)(v & 0xFFFFu)};
}

}  // namespace

int detect_config(uint32_t cap, uint32_t shmem_bytes, size_t* smem, uint32_t* wpad) {
  uint32_t words = (shmem_bytes + 3u) / 4u;
  *wpad = (words + 31u) & ~31u;
  if (*wpad == 0) *wpad = 32;
  *smem = layout(cap, *wpad).end;
  return *smem <= 227u * 1024u ? MCKG_OK : MCKG_E_RANGE;
}

}  // namespace mckg

using namespace mckg;

extern "C" int mckg_race_out_reset(const mckg_race_out* out, void* stream) {
  if (!out || !out->n_triples || !out->line_first || !out->status) {
    set_error("mckg_race_out_reset: null output");
    return MCKG_E_ARG;
  }
  reset_kernel<<<MCKG_MAX_LINES / 256, 256, 0, (cudaStream_t)stream>>>(out->n_triples,
                                                                      out->line_first, out->status);
  MCKG_CUDA_TRY(cudaGetLastError());
  add_launches(1);
  return MCKG_OK;
}

extern "C" int mckg_detect_shared(const mckg_trace* tr, const mckg_race_out* out, void* stream) {
  if (!tr || !out || !out->n_triples || !out->line_first || !out->status ||
      (!out->triples && out->capacity)) {
    set_error("mckg_detect_shared: null argument");
    return MCKG_E_ARG;
  }
  if (tr->n_blocks == 0) return MCKG_OK;
  if (!tr->block_start || (!tr->events && tr->n_events)) {
    set_error("mckg_detect_shared: null trace");
    return MCKG_E_ARG;
  }
  if (tr->shmem_bytes > MCKG_MAX_OFF || (uint64_t)tr->bid_base + tr->n_blocks > MCKG_MAX_BID) {
    set_error("mckg_detect_shared: shmem_bytes or bid out of range");
    return MCKG_E_RANGE;
  }
  uint32_t cap = tr->max_block_events ? tr->max_block_events : 1024u;
  cap = (cap + 31u) & ~31u;
  if (cap > (uint32_t)EPT_MAX * NT) {
    set_error("mckg_detect_shared: a block holds more than 4096 events (staging limit)");
    return MCKG_E_RANGE;
  }
  size_t smem;
  uint32_t wpad;
  if (detect_config(cap, tr->shmem_bytes, &smem, &wpad) != MCKG_OK) {
    set_error("mckg_detect_shared: shared object too large for the shared-memory filter");
    return MCKG_E_RANGE;
  }
  void (*kern)(Params) = cap <= 4u * NT   ? race_detect_kernel<4>
                         : cap <= 8u * NT ? race_detect_kernel<8>
                                          : race_detect_kernel<16>;
  const int ki = cap <= 4u * NT ? 0 : cap <= 8u * NT ? 1 : 2;
  static thread_local size_t configured[3] = {0, 0, 0};
  if (smem > configured[ki]) {
    MCKG_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured[ki] = smem;
  }
  int per_sm = 0;
  MCKG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NT, smem));
  if (per_sm < 1) per_sm = 1;
  uint32_t grid = (uint32_t)sm_count() * (uint32_t)per_sm;
  if (grid > tr->n_blocks) grid = tr->n_blocks;
  Params P;
  P.ev = tr->events;
  P.bstart = tr->block_start;
  P.n_blocks = tr->n_blocks;
  P.obj_base = tr->obj_base;
  P.bid_base = tr->bid_base;
  P.shmem_bytes = tr->shmem_bytes;
  P.cap = cap;
  P.wpad = wpad;
  P.tri = out->triples;
  P.capacity = out->capacity;
  P.n_tri = out->n_triples;
  P.line_first = out->line_first;
  P.status = out->status;
  kern<<<grid, NT, smem, (cudaStream_t)stream>>>(P);
  MCKG_CUDA_TRY(cudaGetLastError());
  note_launch(1, grid, NT, (uint32_t)smem);
  return MCKG_OK;
}

extern "C" int mckg_sort_triples(mckg_race_triple* triples, uint64_t n, uint32_t obj_base,
                                 unsigned long long* n_unique, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) {
    if (n_unique) MCKG_CUDA_TRY(cudaMemsetAsync(n_unique, 0, sizeof(unsigned long long), s));
    return MCKG_OK;
  }
  if (!triples) return MCKG_E_ARG;
  unsigned long long *k0 = nullptr, *k1 = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0, tmp2 = 0;
  MCKG_CUDA_TRY(cudaMallocAsync(&k0, n * sizeof(unsigned long long), s));
  MCKG_CUDA_TRY(cudaMallocAsync(&k1, n * sizeof(unsigned long long), s));
  uint32_t nb = (uint32_t)((n + 255) / 256);
  encode_triples<<<nb, 256, 0, s>>>(triples, k0, n, obj_base);
  cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, k0, k1, (int64_t)n, 0, 58, s);
  if (n_unique) {
    cub::DeviceSelect::Unique(nullptr, tmp2, k1, k0, n_unique, (int64_t)n, s);
    tmp_bytes = std::max(tmp_bytes, tmp2);
  }
  MCKG_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, s));
  MCKG_CUDA_TRY(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, k0, k1, (int64_t)n, 0, 58, s));
  if (n_unique) {
    MCKG_CUDA_TRY(cub::DeviceSelect::Unique(tmp, tmp_bytes, k1, k0, n_unique, (int64_t)n, s));
    decode_triples<<<nb, 256, 0, s>>>(k0, triples, n_unique, n, obj_base);
  } else {
    decode_triples<<<nb, 256, 0, s>>>(k1, triples, nullptr, n, obj_base);
  }
  MCKG_CUDA_TRY(cudaGetLastError());
  cudaFreeAsync(tmp, s);
  cudaFreeAsync(k0, s);
  cudaFreeAsync(k1, s);
  add_launches(n_unique ? 4 : 3);
  return MCKG_OK;
}
