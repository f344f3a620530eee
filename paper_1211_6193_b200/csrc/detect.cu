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

#ifndef MCKG_K2_NSTAGE
#define MCKG_K2_NSTAGE 3
#endif
#ifndef MCKG_K2_MINB
#define MCKG_K2_MINB 3
#endif

namespace mckg {
namespace {

constexpr int NT = 256;
constexpr int NWARP = NT / 32;
constexpr int NSTAGE = MCKG_K2_NSTAGE;
constexpr int EPT_MAX = 16;     // records per thread kept in registers (cap <= 4096)
constexpr uint32_t HS = 512;    // (byte, line) dedup set entries
constexpr uint32_t TBN = 256;   // staged triples before a global flush
constexpr uint32_t LTN = 32;    // line-first local table entries
constexpr uint32_t INF = 0xFFFFFFFFu;
constexpr uint32_t INV = 0xFFFFFFFFu;
constexpr uint32_t ST_OVERFLOW = MCKG_ST_OVERFLOW, ST_RANGE = MCKG_ST_RANGE,
                   ST_ORDER = MCKG_ST_ORDER, ST_DUP = MCKG_ST_DUP;
// misc[] slots
constexpr int M_TBN = 0, M_CLN = 1, M_NSEG = 2, M_BASE_LO = 3, M_BASE_HI = 4, M_FLAGS = 5;

struct Params {
  const mckg_access* ev;
  const uint64_t* bstart;
  uint32_t n_blocks, obj_base, bid_base, shmem_bytes, cap, wpad;
  mckg_race_triple* tri;
  unsigned long long capacity;
  unsigned long long* n_tri;
  unsigned long long* line_first;
  uint32_t* status;
  uint32_t debug;  // experiments only (MCKG_DEBUG): 1 skip exact, 2 skip filter, 8/16 stop early (bisection)
};

extern __shared__ __align__(128) uint8_t smem_raw[];
// fixed-size per-CTA state (static shared memory: compile-time addresses)
__shared__ unsigned long long s_hset[HS];
__shared__ unsigned long long s_lt_ts[LTN];
__shared__ mckg_race_triple s_tbuf[TBN];
__shared__ uint32_t s_lt_line[LTN];
__shared__ uint32_t s_misc[16];
__shared__ uint32_t s_info[2][4];  // per cl buffer: n, b, m
__shared__ uint64_t s_full_cl[2], s_free_cl[2];
__shared__ uint64_t s_mbar[NSTAGE];

// Byte offsets of the size-dependent state in the dynamic shared memory.
struct Lay {
  uint32_t tag, multi, anyw, bitmap, cl, seg, stage, end;
};

__host__ __device__ inline Lay layout(uint32_t cap, uint32_t wpad) {
  Lay L;
  uint32_t p = 0;
  L.tag = p;     p += wpad * 4;
  L.multi = p;   p += wpad * 4;
  L.anyw = p;    p += wpad * 4;
  L.bitmap = p;  p += (cap / 32 + 1) * 4;
  L.cl = p;      p += 2 * cap * 2;
  L.seg = p;     p += (cap + 2) * 2;
  p = (p + 127u) & ~127u;
  L.stage = p;   p += NSTAGE * cap * 16;
  L.end = p;
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
  unsigned long long* hs = s_hset;
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
  uint32_t* lt_line = s_lt_line;
  unsigned long long* lt_ts = s_lt_ts;
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



// ---- 32-bit shared-window accessors (plain LDS/STS, predicated stores) ----
__device__ __forceinline__ uint32_t lds(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts_if(bool p, uint32_t a, uint32_t v) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n}" ::"r"(a),
      "r"(v), "r"((uint32_t)p)
      : "memory");
}

// Barrier among the NT filter threads only (the exact warp runs decoupled).
__device__ __forceinline__ void fsync() { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); }

// Rare path: the 2nd/3rd word of an access spanning several 4-byte words.
__device__ __noinline__ bool extra_words(uint32_t tag_base, uint32_t d1, uint32_t d2, uint32_t w0,
                                         uint32_t tid, int phase, uint32_t st) {
  const uint32_t off = acc_off(w0), len = acc_len(w0);
  const bool wr = acc_write(w0);
  bool cand = false;
  for (uint32_t w = (off >> 2) + 1; w <= (off + len - 1u) >> 2; ++w) {
    const uint32_t a = tag_base + sw(w) * 4u;
    if (phase == 1) {
      sts_if(true, a, tid);
    } else if (phase == 2) {
      sts_if(lds(a) != tid, a + d1, st);
      sts_if(wr, a + d2, st);
    } else {
      cand |= lds(a + d1) == st && lds(a + d2) == st;
    }
  }
  return cand;
}

// Epoch segment starts from the start bitmap, in order (warp 0 only).
__device__ void build_segments(const Lay& L, uint32_t n) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t* bitmap = sp<uint32_t>(L.bitmap);
  uint16_t* seg = sp<uint16_t>(L.seg);
  const uint32_t nwords = (n + 31u) / 32u;
  uint32_t total = 0;
  for (uint32_t base = 0; base < nwords; base += 32) {
    uint32_t word = base + lane < nwords ? bitmap[base + lane] : 0u;
    const uint32_t c = __popc(word);
    uint32_t incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= (uint32_t)d) incl += v;
    }
    uint32_t pos = total + incl - c;
    while (word) {
      const uint32_t b = __ffs(word) - 1u;
      seg[pos++] = (uint16_t)((base + lane) * 32u + b);
      word &= word - 1u;
    }
    total += __shfl_sync(0xFFFFFFFFu, incl, 31);
  }
  if (lane == 0) {
    seg[total] = (uint16_t)n;
    s_misc[M_NSEG] = total;
  }
}

// Per-lane cache of first racing timestamps by line (exact warp only; lane l
// owns one entry), flushed to the global line table on eviction / at exit.
struct ExactState {
  uint32_t lc_line;
  unsigned long long lc_ts;
  uint32_t lc_next;  // uniform: next slot to allocate
  uint32_t tbn;      // uniform: staged triples in s_tbuf
};

__device__ __forceinline__ unsigned long long shfl64(unsigned long long v, int src) {
  return ((unsigned long long)__shfl_sync(0xFFFFFFFFu, (uint32_t)(v >> 32), src) << 32) |
         __shfl_sync(0xFFFFFFFFu, (uint32_t)v, src);
}

__device__ void line_cache_put(ExactState& E, const Params& P, bool leader, uint32_t line,
                               unsigned long long ts) {
  const uint32_t lane = threadIdx.x & 31u;
  for (uint32_t lm = __ballot_sync(0xFFFFFFFFu, leader); lm; lm &= lm - 1u) {
    const int src = __ffs(lm) - 1;
    const uint32_t L = __shfl_sync(0xFFFFFFFFu, line, src);
    const unsigned long long T = shfl64(ts, src);
    const uint32_t own = __ballot_sync(0xFFFFFFFFu, E.lc_line == L);
    if (own) {
      if (lane == (uint32_t)(__ffs(own) - 1) && T < E.lc_ts) E.lc_ts = T;
    } else {
      if (lane == E.lc_next) {
        if (E.lc_line != INF) atomicMin(P.line_first + E.lc_line, E.lc_ts);
        E.lc_line = L;
        E.lc_ts = T;
      }
      E.lc_next = (E.lc_next + 1u) & 31u;
    }
  }
}

// Flushes the staged triples (exact warp only).
__device__ void flush_tbuf(ExactState& E, const Params& P) {
  const uint32_t lane = threadIdx.x & 31u;
  __syncwarp();
  const uint32_t n = E.tbn;
  if (n == 0) return;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(P.n_tri, (unsigned long long)n);
  base = __shfl_sync(0xFFFFFFFFu, base, 0);
  for (uint32_t i = lane; i < n; i += 32) {
    if (base + i < P.capacity)
      P.tri[base + i] = s_tbuf[i];
    else
      atomicOr(s_misc + M_FLAGS, ST_OVERFLOW);
  }
  __syncwarp();
  E.tbn = 0;
}

// Appends k (warp-uniform) triples per `emit` lane: bytes b0..b0+k-1.
__device__ void append_triples(ExactState& E, const Params& P, bool emit, uint32_t obj,
                               uint32_t b0, uint32_t k, int32_t line) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t em = __ballot_sync(0xFFFFFFFFu, emit);
  if (!em) return;
  const uint32_t need = k * __popc(em);
  if (E.tbn + need > TBN) flush_tbuf(E, P);
  const uint32_t pre = k * __popc(em & ((1u << lane) - 1u));
  if (emit)
    for (uint32_t q = 0; q < k; ++q) s_tbuf[E.tbn + pre + q] = mckg_race_triple{obj, b0 + q, line};
  __syncwarp();
  E.tbn += need;
}

// Exact pass over a block's candidate list, run by the dedicated exact warp:
// lane-per-X, each lane scans every candidate Y (broadcast loads).
__device__ void exact_block(ExactState& E, const Lay& L, const Params& P, const uint4* src,
                            const uint16_t* cl, uint32_t m, uint32_t obj, uint32_t bid,
                            unsigned long long bstamp) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t* misc = s_misc;
  for (uint32_t xb = 0; xb < m; xb += 32u) {
    const uint32_t xp = xb + lane;
    const bool act = xp < m;
    const uint32_t xi = act ? cl[xp] : 0u;
    const uint4 X = src[xi];
    const uint32_t xlen = acc_len(X.x);
    const uint32_t xoff = acc_off(X.x), xend = xoff + xlen;
    const uint32_t xtid = acc_tid(X.y), xep = acc_epoch(X.y);
    const bool xw = acc_write(X.x);
    uint32_t bits = 0;
#pragma unroll 4
    for (uint32_t j = 0; j < m; ++j) {
      const uint32_t yi = cl[j];
      const uint2 Y = *reinterpret_cast<const uint2*>(src + yi);
      const uint32_t yoff = acc_off(Y.x), yend = yoff + acc_len(Y.x);
      const uint32_t lo = max(xoff, yoff), hi = min(xend, yend);
      const bool hit = yi < xi && acc_epoch(Y.y) == xep && acc_tid(Y.y) != xtid &&
                       (xw || acc_write(Y.x)) && lo < hi;
      if (hit) bits |= ((1u << (hi - lo)) - 1u) << (lo - xoff);
    }
    if (!act) bits = 0;
    const bool racing = bits != 0;
    if (!__any_sync(0xFFFFFFFFu, racing)) continue;
    const int32_t line = (int32_t)X.z;
    const unsigned long long ts = ts_key(X.w, bid, xtid);
    // first racing timestamp per line: min within the warp, then the cache
    const uint32_t rm = __ballot_sync(0xFFFFFFFFu, racing);
    const uint32_t gm = __match_any_sync(0xFFFFFFFFu, racing ? (uint32_t)line : (0x80000000u | lane));
    unsigned long long mn = ts;
    for (uint32_t tmp = rm; tmp; tmp &= tmp - 1u) {
      const int s = __ffs(tmp) - 1;
      const unsigned long long v = shfl64(ts, s);
      if ((gm >> s) & 1u) mn = v < mn ? v : mn;
    }
    line_cache_put(E, P, racing && lane == (uint32_t)(__ffs(gm) - 1), (uint32_t)line, mn);
    // reported triples, deduplicated per block
    const bool simple = m <= 32u &&
        __all_sync(0xFFFFFFFFu, !racing || (xlen == 4u && (xoff & 3u) == 0u && bits == 0xFu));
    if (simple) {
      // whole aligned words: (word, line) identifies the 4 bytes exactly
      const uint32_t km = __match_any_sync(0xFFFFFFFFu, racing ? ((xoff >> 2) | ((uint32_t)line << 18))
                                                                : (0xFFFFFFFFu - lane));
      const bool lead = racing && lane == (uint32_t)(__ffs(km) - 1);
      append_triples(E, P, lead, obj, xoff, 4u, line);
    } else {
      for (uint32_t q = 0; q < MCKG_MAX_LEN; ++q) {
        bool fresh = false;
        if ((bits >> q) & 1u) {
          const uint32_t byte = xoff + q;
          const unsigned long long key = (bstamp << 40) |
                                         ((unsigned long long)(byte & 0xFFFFFu) << 16) |
                                         ((uint32_t)line & 0xFFFFu);
          const int r = hset_insert(L, key, bstamp);
          if (r == 2) atomicOr(misc + M_FLAGS, ST_DUP);
          fresh = r != 0;
        }
        append_triples(E, P, fresh, obj, xoff + q, 1u, line);
      }
    }
  }
}

template <int EPT>
__device__ void process_block(const Lay& L, const Params& P, const uint4* src, uint32_t n,
                              uint16_t* cl, uint32_t* clcount, uint32_t& stamp) {
  const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
  const uint32_t shm = P.shmem_bytes;
  const uint32_t tag_base = smem_u32(smem_raw) + L.tag;
  const uint32_t d1 = L.multi - L.tag, d2 = L.anyw - L.tag;
  uint32_t* bitmap = sp<uint32_t>(L.bitmap);
  const uint16_t* seg = sp<uint16_t>(L.seg);
  uint32_t* misc = s_misc;
  // Per owned record i = k*NT + t: epoch (INV = absent or invalid), shared
  // address of its first word's tag, meta = tid | write << 11 | spans << 12.
  uint32_t ep[EPT], xa[EPT], meta[EPT];
  uint32_t flags = 0, mw = 0;
  const uint32_t cur0 = acc_epoch(src[0].y);
#pragma unroll
  for (int k = 0; k < EPT; ++k) {
    const uint32_t i = (uint32_t)k * NT + t;
    const bool in = i < n;
    const uint4 r = in ? src[i] : make_uint4(0, 0, 0, 0);
    const uint32_t e = acc_epoch(r.y);
    uint32_t prev = __shfl_up_sync(0xFFFFFFFFu, e, 1);
    if (lane == 0 && in && i > 0) prev = acc_epoch(src[i - 1].y);
    const bool start = in && (i == 0 || e != prev);
    if (in && i > 0 && e < prev) flags |= ST_ORDER;
    const uint32_t off = acc_off(r.x), len = acc_len(r.x);
    const bool ok = in && (len - 1u) < MCKG_MAX_LEN && off + len <= shm &&
                    ((uint32_t)r.z >> 16) == 0u;
    if (in && !ok) flags |= ST_RANGE;
    ep[k] = ok ? e : INV;
    xa[k] = tag_base + (ok ? sw(off >> 2) * 4u : 0u);
    const uint32_t spans = ok && ((off & 3u) + len) > 4u;
    meta[k] = acc_tid(r.y) | (acc_write(r.x) << 11) | (spans << 12);
    mw |= spans;
    const uint32_t bm = __ballot_sync(0xFFFFFFFFu, start);
    if (lane == 0 && (uint32_t)k * NT < n) bitmap[(uint32_t)k * NWARP + warp] = bm;
    // P1 of the first epoch, fused with the load
    sts_if(ep[k] == cur0, xa[k], meta[k] & 0x7FFu);
  }
  flags = __reduce_or_sync(0xFFFFFFFFu, flags);
  if (lane == 0 && flags) atomicOr(misc + M_FLAGS, flags);
  const bool wmw = __any_sync(0xFFFFFFFFu, mw);  // warp has multi-word accesses
  uint32_t st = ++stamp;
  if (wmw) {
    for (int k = 0; k < EPT; ++k)
      if (ep[k] == cur0 && (meta[k] & 0x1000u))
        extra_words(tag_base, d1, d2, src[k * NT + t].x, meta[k] & 0x7FFu, 1, st);
  }
  if (t == 0) *clcount = 0;
  fsync();
  if (P.debug & 8u) return;   // experiment: load + bitmap + first P1 only
  if (warp == 0) build_segments(L, n);
  if (P.debug & 16u) {        // experiment: + epoch segmentation
    fsync();
    return;
  }
  uint32_t cur = cur0;
  uint32_t sidx = 0;
  while (true) {
    // P2: words seen by a second thread; written words
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const bool a = ep[k] == cur;
      const uint32_t tg = lds(xa[k]);
      sts_if(a && tg != (meta[k] & 0x7FFu), xa[k] + d1, st);
      sts_if(a && (meta[k] & 0x800u), xa[k] + d2, st);
    }
    if (wmw) {
      for (int k = 0; k < EPT; ++k)
        if (ep[k] == cur && (meta[k] & 0x1000u))
          extra_words(tag_base, d1, d2, src[k * NT + t].x, meta[k] & 0x7FFu, 2, st);
    }
    fsync();
    const uint32_t e = seg[sidx + 1];
    // P3: candidates -> block list cl (warp-aggregated compaction)
    uint32_t cmask = 0;  // bit k: record k is a candidate
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const uint32_t mv = lds(xa[k] + d1), av = lds(xa[k] + d2);
      if (ep[k] == cur && mv == st && av == st) cmask |= 1u << k;
    }
    if (wmw) {
      for (int k = 0; k < EPT; ++k)
        if (ep[k] == cur && (meta[k] & 0x1000u) &&
            extra_words(tag_base, d1, d2, src[k * NT + t].x, meta[k] & 0x7FFu, 3, st))
          cmask |= 1u << k;
    }
    if (__any_sync(0xFFFFFFFFu, cmask)) {
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const bool cand = (cmask >> k) & 1u;
        const uint32_t bm = __ballot_sync(0xFFFFFFFFu, cand);
        if (bm) {
          const uint32_t leader = __ffs(bm) - 1u;
          uint32_t base = 0;
          if (lane == leader) base = atomicAdd(clcount, (uint32_t)__popc(bm));
          base = __shfl_sync(0xFFFFFFFFu, base, leader);
          if (cand) cl[base + __popc(bm & ((1u << lane) - 1u))] = (uint16_t)((uint32_t)k * NT + t);
        }
      }
    }
    const bool more = e < n;
    if (more) {  // P1 of the next epoch shares this barrier interval
      cur = acc_epoch(src[e].y);
      st = ++stamp;
      ++sidx;
#pragma unroll
      for (int k = 0; k < EPT; ++k) sts_if(ep[k] == cur, xa[k], meta[k] & 0x7FFu);
      if (wmw) {
        for (int k = 0; k < EPT; ++k)
          if (ep[k] == cur && (meta[k] & 0x1000u))
            extra_words(tag_base, d1, d2, src[k * NT + t].x, meta[k] & 0x7FFu, 1, st);
      }
    }
    fsync();
    if (!more) break;
  }
}

// One CTA = 8 filter warps + 1 exact warp (warp specialised).  Filter warps
// run the epoch filter of block b+1 while the exact warp finishes block b;
// they hand candidate lists over through two mbarrier-guarded buffers.  The
// exact warp also owns the report state and re-issues the TMA load into the
// stage it has just released.
constexpr int NTHREADS = NT + 32;

template <int EPT>
__global__ void __launch_bounds__(NTHREADS, EPT <= 4 ? MCKG_K2_MINB : (EPT <= 8 ? 2 : 1))
    race_detect_kernel(Params P) {
  const Lay L = layout(P.cap, P.wpad);
  const uint32_t t = threadIdx.x, warp = t >> 5, lane = t & 31u;
  uint32_t* misc = s_misc;
  uint64_t* mbar = s_mbar;
  uint4* stage = sp<uint4>(L.stage);
  uint16_t* clbuf = sp<uint16_t>(L.cl);  // 2 x cap
  for (uint32_t i = t; i < HS; i += NTHREADS) s_hset[i] = 0ull;
  for (uint32_t i = t; i < LTN; i += NTHREADS) {
    s_lt_line[i] = INF;
    s_lt_ts[i] = ~0ull;
  }
  for (uint32_t i = t; i < 3 * P.wpad; i += NTHREADS) sp<uint32_t>(L.tag)[i] = 0u;
  if (t < 16) misc[t] = 0u;
  if (t == 0) {
    for (int k = 0; k < NSTAGE; ++k) mbar_init(mbar + k, 1);
    for (int k = 0; k < 2; ++k) {
      mbar_init(s_full_cl + k, 1);
      mbar_init(s_free_cl + k, 1);
    }
    fence_mbar_init();
  }
  __syncthreads();

  const uint32_t G = gridDim.x;
  auto nev = [&](uint32_t b) { return P.bstart[b + 1] - P.bstart[b]; };
  auto issue = [&](uint32_t b, int st) {  // one thread
    const uint64_t n = nev(b);
    if (n == 0 || n > P.cap) return;
    const uint64_t s0 = P.bstart[b];
    const uint32_t bytes = (uint32_t)(n * 16);
    mbar_expect_tx(mbar + st, bytes);
    bulk_g2s(stage + (size_t)st * P.cap, P.ev + s0, bytes, mbar + st);
  };

  if (warp < NT / 32) {
    // ---------------- filter warps ----------------
    uint32_t sphase = 0, stamp = 0;
    int it = 0;
    for (uint32_t b = blockIdx.x; b < P.n_blocks; b += G, ++it) {
      const int st = it % NSTAGE;
      const int p = it & 1;
      const uint32_t u = (uint32_t)(it >> 1);
      mbar_wait(s_free_cl + p, (u & 1u) ^ 1u);  // exact warp done with this buffer
      const uint64_t n_all = nev(b);
      const uint32_t n = n_all <= P.cap ? (uint32_t)n_all : 0u;
      uint32_t* clcount = misc + 8 + p;
      if (n > 0 && (P.debug & 2u)) {
        mbar_wait(mbar + st, (sphase >> st) & 1u);
        sphase ^= 1u << st;
        if (t == 0) *clcount = 0;
        fsync();
      } else if (n > 0) {
        mbar_wait(mbar + st, (sphase >> st) & 1u);
        sphase ^= 1u << st;
        process_block<EPT>(L, P, stage + (size_t)st * P.cap, n, clbuf + (size_t)p * P.cap,
                           clcount, stamp);
      } else {
        if (t == 0) {
          *clcount = 0;
          if (n_all > 0) atomicOr(misc + M_FLAGS, ST_RANGE);  // exceeds the staging capacity
        }
        fsync();
      }
      if (t == 0) {
        s_info[p][0] = n;
        s_info[p][1] = b;
        s_info[p][2] = *clcount;
        mbar_arrive(s_full_cl + p);
      }
    }
  } else {
    // ---------------- exact / report warp ----------------
    if (lane == 0)
      for (int k = 0; k < NSTAGE; ++k) {
        const uint32_t b = blockIdx.x + (uint32_t)k * G;
        if (b < P.n_blocks) issue(b, k);
      }
    unsigned long long bstamp = 0;
    ExactState E{INF, ~0ull, 0u, 0u};
    int it = 0;
    for (uint32_t b = blockIdx.x; b < P.n_blocks; b += G, ++it) {
      const int st = it % NSTAGE;
      const int p = it & 1;
      const uint32_t u = (uint32_t)(it >> 1);
      mbar_wait(s_full_cl + p, u & 1u);
      const uint32_t n = s_info[p][0], m = s_info[p][2];
      ++bstamp;
      if (n > 0 && m > 0 && !(P.debug & 1u))
        exact_block(E, L, P, stage + (size_t)st * P.cap, clbuf + (size_t)p * P.cap, m,
                    P.obj_base + b, P.bid_base + b, bstamp);
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(s_free_cl + p);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t nb = b + (uint32_t)NSTAGE * G;
        if (nb < P.n_blocks) issue(nb, st);
      }
    }
    flush_tbuf(E, P);
    if (E.lc_line != INF) atomicMin(P.line_first + E.lc_line, E.lc_ts);
  }
  __syncthreads();
  if (t == 0 && misc[M_FLAGS]) atomicOr(P.status, misc[M_FLAGS]);
  if (t == 0 && (P.debug & 12u)) {
    atomicAdd(P.status + 1, misc[12]);
    atomicAdd(P.status + 2, misc[13]);
  }
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
  MCKG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, NTHREADS, smem));
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
  {
    const char* dbg = getenv("MCKG_DEBUG");
    P.debug = dbg ? (uint32_t)atoi(dbg) : 0u;
  }
  kern<<<grid, NTHREADS, smem, (cudaStream_t)stream>>>(P);
  MCKG_CUDA_TRY(cudaGetLastError());
  note_launch(1, grid, NTHREADS, (uint32_t)smem);
  return MCKG_OK;
}

extern "C" int mckg_sort_triples(mckg_race_triple* triples, uint64_t n, uint32_t obj_base,
                                 unsigned long long* n_unique, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  keep_pool_memory();
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
