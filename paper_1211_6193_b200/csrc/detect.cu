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
// Two kernels, both streaming many simulated blocks (blocks never interact:
// each owns its shared object, device.cpp:33-38):
//   * fast_kernel (the default path): one warp per block, for trace-mode
//     blocks (1024 records, aligned 4-byte accesses, <= 2 epochs, objects of
//     <= 4 KiB): coalesced 16-byte loads into one packed register per record,
//     the word filter below in the warp's own shared-memory tag arrays with
//     __syncwarp between phases, a match_any exact pass over the candidates.
//     Any other block is handed to
//   * race_detect_kernel (the general path), one CTA per block at a time:
//     1. stage: each block's 16-byte records are pulled into shared memory by
//        the TMA engine (cp.async.bulk + mbarrier, 3 stages);
//     2. filter, on 4-byte words, NSLOT epochs at once in per-slot arrays (a
//        "unit" = block x epoch window): P1 tag[w] = some accessing tid |
//        barrier | P2 stamp the words seen by a second tid / written |
//        barrier | P3 an event is a candidate iff one of its words is both.
//        A byte can race only if its word passes, so the filter has no false
//        negatives;
//     3. exact pass over the (rare) candidates -- the reference predicate
//        verbatim, byte-exact: X races on the bytes it shares with an
//        earlier candidate Y of the same epoch and another thread where X or
//        Y writes;
//     4. report: racing (byte, line) pairs are deduplicated per block through
//        a (word, line) -> byte-mask table, staged and appended to the global
//        triple array; the first racing timestamp per line is min-reduced.
#include <algorithm>
#include <atomic>
#include <vector>
#include <map>
#include <thread>
#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "sort.cuh"

// TMA stages and CTAs/SM of the general kernel
#ifndef MCKG_K2_NSTAGE
#define MCKG_K2_NSTAGE 3
#endif
#ifndef MCKG_K2_MINB
#define MCKG_K2_MINB 3
#endif

namespace mckg {
namespace {

constexpr int NT = 256;
constexpr int NSTAGE_MAX = 3;
constexpr int EPT_MAX = 16;     // records per thread kept in registers (cap <= 4096)
constexpr uint32_t HS = 512;    // (word, line) -> reported byte mask, per block
constexpr uint32_t TBN = 128;   // staged triples per buffer before the global append
constexpr uint32_t LTN = 32;    // line-first local table entries
constexpr uint32_t INF = 0xFFFFFFFFu;
constexpr uint32_t INV = 0xFFFFFFFFu;
constexpr uint32_t ST_OVERFLOW = MCKG_ST_OVERFLOW, ST_RANGE = MCKG_ST_RANGE,
                   ST_ORDER = MCKG_ST_ORDER, ST_DUP = MCKG_ST_DUP;
// NSLOT epochs are filtered at once, each in its own word arrays: tag[slot][w]
// (some accessing tid, u16) and ma[slot][w] = {multi, any-write} 16-bit unit
// stamps.  A stale stamp that wraps to the current one only adds a candidate
// (the exact pass removes it): the filter never misses a race.
constexpr uint32_t NSLOT = 2;

struct Params {
  const mckg_access* ev;
  const uint64_t* bstart;
  uint32_t n_blocks, obj_base, bid_base, shmem_bytes, cap, wpad;
  mckg_race_triple* tri;
  unsigned long long capacity;
  unsigned long long* n_tri;
  unsigned long long* line_first;
  uint32_t* status;
  uint32_t debug;  // experiments only (MCKG_DEBUG): 1 skip the exact pass, 2 TMA stream only
  // the general kernel gated on the fast path's overflow list
  uint32_t gate;       // 1 = only the blocks of olist
  uint32_t skip_big;   // blocks over `cap` records are left to the oversize route (no ST_RANGE)
  uint32_t* ocount;    // [0] blocks in olist
  uint32_t* olist;     // [n_blocks]
};


extern __shared__ __align__(128) uint8_t smem_raw[];
// fixed-size per-CTA state (static shared memory: compile-time addresses)
__shared__ unsigned long long s_hset[HS];
__shared__ unsigned long long s_lt_ts[LTN];
__shared__ mckg_race_triple s_tbuf[2][TBN];
__shared__ uint32_t s_lt_line[LTN];
__shared__ uint32_t s_cnt[4];    // [0..1] candidates per cl buffer, [2..3] staged triples
__shared__ uint32_t s_flags;
__shared__ uint64_t s_mbar[NSTAGE_MAX];
__shared__ uint32_t s_n[NSTAGE_MAX];  // events of the block in each stage (0: none loaded)

// Byte offsets of the size-dependent state in the dynamic shared memory.
struct Lay {
  uint32_t ma, tag, cl, stage, end;
};

__host__ __device__ inline Lay layout(uint32_t cap, uint32_t wpad, uint32_t nstage) {
  Lay L;
  uint32_t p = 0;
  L.ma = p;      p += NSLOT * wpad * 4;
  L.tag = p;     p += NSLOT * wpad * 4;
  L.cl = p;      p += 2 * cap * 2;
  p = (p + 127u) & ~127u;
  L.stage = p;   p += nstage * cap * 16;
  L.end = p;
  return L;
}

template <typename T>
__device__ __forceinline__ T* sp(uint32_t off) {
  return reinterpret_cast<T*>(smem_raw + off);
}

__device__ __forceinline__ uint32_t sw(uint32_t w) { return w ^ ((w >> 5) & 31u); }

// ---- shared-window accessors (plain LDS/STS, predicated stores) ----
__device__ __forceinline__ void sts16_if(bool p, uint32_t a, uint32_t v) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.u16 [%0], %1;\n}" ::"r"(a),
      "h"((uint16_t)v), "r"((uint32_t)p)
      : "memory");
}
__device__ __forceinline__ void sts32_if(bool p, uint32_t a, uint32_t v) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n}" ::"r"(a),
      "r"(v), "r"((uint32_t)p)
      : "memory");
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

// Barrier among the NT threads.
__device__ __forceinline__ void fsync() { asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory"); }
// ... that also returns the OR of p over the threads.
__device__ __forceinline__ bool fsync_or(bool p) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred a, b;\n\tsetp.ne.u32 a, %1, 0;\n\t"
      "barrier.cta.red.or.pred b, 1, %2, a;\n\tselp.u32 %0, 1, 0, b;\n}"
      : "=r"(r)
      : "r"((uint32_t)p), "n"(NT)
      : "memory");
  return r != 0;
}

// Rare path: the 2nd/3rd word of an access spanning several 4-byte words
// (tag_slot / ma_slot: the slot's arrays).
__device__ __noinline__ bool extra_words(uint32_t tag_slot, uint32_t ma_slot, uint32_t w0, uint32_t tid,
                                         int phase, uint32_t st) {
  const uint32_t off = acc_off(w0), len = acc_len(w0);
  const bool wr = acc_write(w0);
  bool cand = false;
  for (uint32_t w = (off >> 2) + 1; w <= (off + len - 1u) >> 2; ++w) {
    const uint32_t a = tag_slot + sw(w) * 4u, m = ma_slot + sw(w) * 4u;
    if (phase == 1) {
      sts32_if(true, a, tid);
    } else if (phase == 2) {
      sts16_if(lds32(a) != tid, m, st);
      sts16_if(wr, m + 2u, st);
    } else {
      cand |= lds32(m) == (st | (st << 16));
    }
  }
  return cand;
}

// First racing timestamp per line: a CTA table, global atomicMin on overflow.
__device__ void line_note(const Params& P, int32_t line, unsigned long long ts) {
  const uint32_t l = (uint32_t)line;
  uint32_t h = l & (LTN - 1);
  for (uint32_t probe = 0; probe < LTN; ++probe) {
    uint32_t v = s_lt_line[h];
    if (v == INF) {
      const uint32_t old = atomicCAS(s_lt_line + h, INF, l);
      v = old == INF ? l : old;
    }
    if (v == l) {
      atomicMin(s_lt_ts + h, ts);
      return;
    }
    h = (h + 1) & (LTN - 1);
  }
  atomicMin(P.line_first + l, ts);
}

// The block's reported set, per (word, line): slot = bstamp:24 | word:18 |
// line:16 | byte mask:4.  Returns the bytes of `mask` not reported before,
// or 0x10 | mask when the probe limit is hit (caller flags ST_DUP).
__device__ uint32_t hset_or(unsigned long long bstamp, uint32_t word, uint32_t line, uint32_t mask) {
  const unsigned long long want = (bstamp << 40) | ((unsigned long long)(word & 0x3FFFFu) << 22) |
                                  ((unsigned long long)(line & 0xFFFFu) << 6);
  uint32_t h = (uint32_t)(((want >> 6) * 0x9E3779B97F4A7C15ull) >> 40) & (HS - 1);
  for (uint32_t probe = 0; probe < 64; ++probe) {
    unsigned long long cur = s_hset[h];
    while ((cur >> 40) != bstamp) {  // stale slot (an earlier block): claim it
      const unsigned long long old = atomicCAS(s_hset + h, cur, want | mask);
      if (old == cur) return mask;
      cur = old;
    }
    if ((cur & ~0x3Full) == want) {
      const unsigned long long old = atomicOr(s_hset + h, (unsigned long long)mask);
      return mask & ~(uint32_t)old & 0xFu;
    }
    h = (h + 1) & (HS - 1);
  }
  return 0x10u | mask;
}

__device__ __forceinline__ unsigned long long shfl64(unsigned long long v, int src) {
  return ((unsigned long long)__shfl_sync(0xFFFFFFFFu, (uint32_t)(v >> 32), src) << 32) |
         __shfl_sync(0xFFFFFFFFu, (uint32_t)v, src);
}

// Exact pass of one block over its m candidates, by all NT threads: group
// of C lanes per candidate X, each lane scanning every C-th candidate Y, the
// lanes' racing bytes OR-reduced.  X races on the bytes it shares with an
// earlier candidate Y of the same epoch and another thread where X or Y
// writes -- the reference predicate (racecheck.cpp:24-32) verbatim.  The
// racing bytes are reported once per (obj, byte, line) and the line's first
// racing timestamp is min-reduced.
__device__ void exact_block(const Params& P, const uint4* src, const uint16_t* cl, uint32_t m, int q,
                            uint32_t obj, uint32_t bid, unsigned long long bstamp) {
  const uint32_t t = threadIdx.x, warp = t >> 5;
  // as few warps as possible (instruction count): W = ceil(m / 32) warps,
  // C lanes per candidate with m * C <= 32 * W
  const uint32_t W = min((m + 31u) >> 5, (uint32_t)NT / 32u);
  uint32_t C = 32;
  while (C > 1 && C * m > 32u * W) C >>= 1;
  const uint32_t groups = 32u * W / C;
  if (warp >= W) return;
  const uint32_t sub = t & (C - 1u);
  for (uint32_t xb = 0; xb < m; xb += groups) {
    const uint32_t i = xb + t / C;
    const bool act = i < m;
    const uint32_t xi = act ? cl[i] : 0u;
    const uint4 X = act ? src[xi] : make_uint4(0, 0, 0, 0);
    const uint32_t xoff = acc_off(X.x), xend = xoff + acc_len(X.x);
    const uint32_t xtid = acc_tid(X.y), xep = acc_epoch(X.y);
    const bool xw = acc_write(X.x);
    uint32_t bits = 0;
    if (act) {
      for (uint32_t j = sub; j < m; j += C) {
        const uint32_t yi = cl[j];
        const uint2 Y = *reinterpret_cast<const uint2*>(src + yi);
        const uint32_t yoff = acc_off(Y.x), yend = yoff + acc_len(Y.x);
        const uint32_t lo = max(xoff, yoff), hi = min(xend, yend);
        const bool hit = yi < xi && acc_epoch(Y.y) == xep && acc_tid(Y.y) != xtid &&
                         (xw || acc_write(Y.x)) && lo < hi;
        if (hit) bits |= ((1u << (hi - lo)) - 1u) << (lo - xoff);
      }
    }
    for (uint32_t d = 1; d < C; d <<= 1) bits |= __shfl_xor_sync(0xFFFFFFFFu, bits, d);
    const bool racing = sub == 0 && bits != 0;
    const uint32_t rm = __ballot_sync(0xFFFFFFFFu, racing);
    if (!rm) continue;
    const uint32_t lane = t & 31u;
    const int32_t line = (int32_t)X.z;
    // first racing timestamp per line: min over the warp's lanes of a line
    const unsigned long long ts = ts_key(X.w, bid, xtid);
    const uint32_t gm = __match_any_sync(0xFFFFFFFFu, racing ? (uint32_t)line : (0x80000000u | lane));
    unsigned long long mn = ts;
    for (uint32_t tmp = rm; tmp; tmp &= tmp - 1u) {
      const int s = __ffs(tmp) - 1;
      const unsigned long long v = shfl64(ts, s);
      if ((gm >> s) & 1u) mn = v < mn ? v : mn;
    }
    if (racing && lane == (uint32_t)(__ffs(gm) - 1)) line_note(P, line, mn);
    // reported set: bytes of (word, line) not reported before in this block
    uint32_t fresh[3] = {0u, 0u, 0u};
    uint32_t k = 0;
    if (racing) {
      const uint64_t ab = (uint64_t)bits << (xoff & 3u);  // bit j = byte (xoff & ~3) + j
      for (uint32_t w = 0; w < 3u && (xoff >> 2) + w <= (xend - 1u) >> 2; ++w) {
        const uint32_t wm = (uint32_t)(ab >> (4u * w)) & 0xFu;
        if (!wm) continue;
        uint32_t f = hset_or(bstamp, (xoff >> 2) + w, (uint32_t)line, wm);
        if (f & 0x10u) {
          atomicOr(&s_flags, ST_DUP);
          f &= 0xFu;
        }
        fresh[w] = f;
        k += __popc(f);
      }
    }
    // one staging-buffer reservation per warp
    uint32_t incl = k;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= (uint32_t)d) incl += v;
    }
    const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
    if (!total) continue;
    uint32_t base = 0;
    if (lane == 31) base = atomicAdd(s_cnt + 2 + q, total);
    base = __shfl_sync(0xFFFFFFFFu, base, 31);
    uint32_t pos = base + incl - k;
    for (uint32_t w = 0; w < 3u; ++w)
      for (uint32_t f = fresh[w]; f; f &= f - 1u, ++pos) {
        const mckg_race_triple tr{obj, ((xoff >> 2) + w) * 4u + (__ffs(f) - 1u), line};
        if (pos < TBN) {
          s_tbuf[q][pos] = tr;
        } else {  // staging buffer full: straight to the global array
          const unsigned long long g = atomicAdd(P.n_tri, 1ull);
          if (g < P.capacity)
            P.tri[g] = tr;
          else
            atomicOr(&s_flags, ST_OVERFLOW);
        }
      }
  }
}

// Appends the staged triples of buffer q to the global array (warp 0).
__device__ void flush_triples(const Params& P, int q) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t n = min(s_cnt[2 + q], TBN);
  if (n == 0) return;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(P.n_tri, (unsigned long long)n);
  base = __shfl_sync(0xFFFFFFFFu, base, 0);
  for (uint32_t i = lane; i < n; i += 32) {
    if (base + i < P.capacity)
      P.tri[base + i] = s_tbuf[q][i];
    else
      atomicOr(&s_flags, ST_OVERFLOW);
  }
}

// One CTA of NT threads streams simulated blocks b = blockIdx.x + k * grid.
// A unit is (block, round): the block's epochs [ws, ws + NSLOT) relative to
// its first epoch (one round unless the block spans more epochs).  Per unit
//   (a) | P2: multi / any-write stamps; exact pass of the previous block
//   (b) | P3: candidates -> cl; P1 (tag <- tid) of the next unit;
//         append the previous block's triples; release its TMA stage
// P3 reads only ma[], P1 writes only tag[]; the exact pass reads the stage
// and cl of the previous block, which nothing else touches until (b).
template <int EPT>
__global__ void __launch_bounds__(NT, EPT <= 4 ? MCKG_K2_MINB : (EPT <= 8 ? 2 : 1))
    race_detect_kernel(Params P) {
  constexpr int NSTAGE = MCKG_K2_NSTAGE;
  // the blocks this launch covers: all, or (gated fused pass) the overflow list
  const uint32_t nblk = P.gate ? *(volatile uint32_t*)P.ocount : P.n_blocks;
  if (nblk == 0) return;
  auto blk = [&](uint32_t j) { return P.gate ? P.olist[j] : j; };
  const Lay L = layout(P.cap, P.wpad, NSTAGE);
  const uint32_t t = threadIdx.x, lane = t & 31u;
  uint64_t* mbar = s_mbar;
  uint4* stage = sp<uint4>(L.stage);
  uint16_t* clbuf = sp<uint16_t>(L.cl);  // 2 x cap
  {
    for (uint32_t i = t; i < HS; i += NT) s_hset[i] = 0ull;
    for (uint32_t i = t; i < LTN; i += NT) {
      s_lt_line[i] = INF;
      s_lt_ts[i] = ~0ull;
    }
  }
  for (uint32_t i = t; i < 2 * NSLOT * P.wpad; i += NT) sp<uint32_t>(L.ma)[i] = 0u;
  if (t < 4) s_cnt[t] = 0u;
  uint32_t flags = 0;
  const uint32_t G = gridDim.x;
  // one thread: stream block b into stage st; s_n[st] = its event count
  // (0 when empty or beyond the staging capacity -- flagged, skipped)
  auto issue = [&](uint32_t j, int st) {  // j: position in the launch's block sequence
    const uint32_t b = blk(j);
    const uint64_t s0 = P.bstart[b], n = P.bstart[b + 1] - s0;
    if (n > P.cap && !P.skip_big) flags |= ST_RANGE;
    const bool go = n > 0 && n <= P.cap;
    s_n[st] = go ? (uint32_t)n : 0u;
    if (!go) return;
    const uint32_t bytes = (uint32_t)(n * 16);
    mbar_expect_tx(mbar + st, bytes);
    bulk_g2s(stage + (size_t)st * P.cap, P.ev + s0, bytes, mbar + st);
  };
  if (t == 0) {
    s_flags = 0;
    for (int k = 0; k < NSTAGE; ++k) mbar_init(mbar + k, 1);
    fence_mbar_init();
    for (int k = 0; k < NSTAGE; ++k) {
      const uint32_t j = blockIdx.x + (uint32_t)k * G;
      if (j < nblk) issue(j, k);
    }
  }
  __syncthreads();

  const uint32_t tag_base = smem_u32(smem_raw) + L.tag;
  const uint32_t ma_delta = L.ma - L.tag;  // ma entry = tag entry + delta (both 4 B per word)
  const uint32_t slotw = P.wpad;
  uint32_t erel[EPT], wsw[EPT], xa[EPT], meta[EPT];
  uint32_t sphase = 0, stamp = 0;
  int it = 0;
  uint32_t j = blockIdx.x, b = j < nblk ? blk(j) : 0u;
  uint32_t n = 0, ws = 0, elast = 0;
  bool wmw = false;
  const uint4* src = stage;
  bool live = j < nblk;
  // the previous block, whose exact pass runs in the next interval
  bool pend = false;
  bool fresh = false;  // the current unit's block was loaded in the last interval
  bool held = false;   // the current block still needs its stage after its first unit
  bool pheld = false;
  int pit = 0;
  uint32_t pb = 0, pj = 0, pn = 0;
  unsigned long long bstamp = 0;

  // P1 of the unit starting at relative epoch `ws` (xa computed for the unit)
  auto p1 = [&](uint32_t st) {
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      const uint32_t slot = erel[k] - ws;
      xa[k] = tag_base + (slot < NSLOT ? (slot * slotw + wsw[k]) << 2 : 0u);  // loads stay in range
      sts32_if(slot < NSLOT, xa[k], meta[k] & 0x7FFu);
    }
    if (wmw) {
      for (int k = 0; k < EPT; ++k) {
        const uint32_t slot = erel[k] - ws;
        if (slot < NSLOT && (meta[k] & 0x1000u))
          extra_words(tag_base + slot * slotw * 4u, tag_base + slot * slotw * 4u + ma_delta,
                      src[k * NT + t].x, meta[k] & 0x7FFu, 1, st);
      }
    }
  };
  auto load_block = [&]() {
    const int sti = it % NSTAGE;
    n = s_n[sti];
    src = stage + (size_t)sti * P.cap;
    if (n > 0) {
      mbar_wait(mbar + sti, (sphase >> sti) & 1u);
      sphase ^= 1u << sti;
    }
    if (P.debug & 2u) n = 0;  // experiment: TMA stream only
    const uint32_t e0 = n > 0 ? acc_epoch(src[0].y) : 0u;
    elast = n > 0 ? acc_epoch(src[n - 1].y) - e0 : 0u;
    ws = 0;
    uint32_t mw = 0;
    // decode; FULL (n == EPT * NT, the common case) drops the bounds predicates
    auto decode = [&](auto full_tag) {
      constexpr bool FULL = decltype(full_tag)::value;
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const uint32_t i = (uint32_t)k * NT + t;
        const bool in = FULL || i < n;
        const uint4 r = in ? src[i] : make_uint4(0, 0, 0, 0);
        const uint32_t e = acc_epoch(r.y);
        uint32_t prev = __shfl_up_sync(0xFFFFFFFFu, e, 1);
        if (lane == 0) prev = i > 0 && in ? acc_epoch(src[i - 1].y) : 0u;
        if (in && e < prev) flags |= ST_ORDER;
        const uint32_t off = acc_off(r.x), len = acc_len(r.x);
        const bool ok = in && (len - 1u) < MCKG_MAX_LEN && off + len <= P.shmem_bytes && (r.z >> 16) == 0u;
        if (in && !ok) flags |= ST_RANGE;
        erel[k] = ok ? e - e0 : INV;  // e < e0 only if unsorted (flagged): out of every window
        wsw[k] = sw(off >> 2);
        const uint32_t spans = ok && ((off & 3u) + len) > 4u;
        meta[k] = (r.y & 0x7FFu) | ((r.x >> 13) & 0x800u) | (spans << 12);
        mw |= spans;
      }
    };
    if (n == (uint32_t)(EPT * NT))
      decode(std::true_type{});
    else
      decode(std::false_type{});
    wmw = __any_sync(0xFFFFFFFFu, mw);
  };

  if (live) {
    load_block();
    p1(++stamp & 0xFFFFu);
    fresh = true;
  }
  while (true) {
    // (a) P1 of this unit and P3 of the previous one are complete
    const bool spans_any = fsync_or(fresh && wmw);
    (void)spans_any;
    if (fresh) {
      held = true;  // the exact pass of this block reads its stage
      fresh = false;
    }
    const bool doexact = pend;
    const int pq = pit & 1;
    pend = false;
    if (doexact) {
      ++bstamp;
      const uint32_t m = pn > 0 ? s_cnt[pq] : 0u;
      if (m > 0 && !(P.debug & 1u)) {
        exact_block(P, stage + (size_t)(pit % NSTAGE) * P.cap, clbuf + (size_t)pq * P.cap, m, pq,
                    P.obj_base + pb, P.bid_base + pb, bstamp);
      }
    }
    const uint32_t st = stamp & 0xFFFFu;
    if (live && !(P.debug & 64u)) {
      // P2: words seen by a second thread; written words
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const bool a = erel[k] - ws < NSLOT;
        const uint32_t tg = lds32(xa[k]);
        const uint32_t mm = xa[k] + ma_delta;
        sts16_if(a && tg != (meta[k] & 0x7FFu), mm, st);
        sts16_if(a && (meta[k] & 0x800u), mm + 2u, st);
      }
      if (wmw) {
        for (int k = 0; k < EPT; ++k) {
          const uint32_t slot = erel[k] - ws;
          if (slot < NSLOT && (meta[k] & 0x1000u))
            extra_words(tag_base + slot * slotw * 4u, tag_base + slot * slotw * 4u + ma_delta,
                        src[k * NT + t].x, meta[k] & 0x7FFu, 2, st);
        }
      }
    }
    fsync();  // (b)
    if (doexact) {
      // the previous block is done: append its triples, free its stage
      if (t < 32) {
        flush_triples(P, pq);
        __syncwarp();
        if (t == 0) s_cnt[2 + pq] = 0;
      }
      if (t == 0) {
        s_cnt[pq] = 0;
        if (pheld) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          const uint32_t nj = pj + (uint32_t)NSTAGE * G;
          if (nj < nblk) issue(nj, pit % NSTAGE);
        }
      }
    }
    if (!live) break;
    // P3: candidates -> the block's list (warp-aggregated compaction)
    const int p = it & 1;
    uint16_t* cl = clbuf + (size_t)p * P.cap;
    uint32_t cmask = 0;
#pragma unroll
    for (int k = 0; k < EPT; ++k) {
      if (P.debug & 64u) break;  // experiment: decode + P1 + barriers only
      const uint32_t v = lds32(xa[k] + ma_delta);
      if (erel[k] - ws < NSLOT && v == (st | (st << 16))) cmask |= 1u << k;
    }
    if (wmw) {
      for (int k = 0; k < EPT; ++k) {
        const uint32_t slot = erel[k] - ws;
        if (slot < NSLOT && (meta[k] & 0x1000u) &&
            extra_words(tag_base + slot * slotw * 4u, tag_base + slot * slotw * 4u + ma_delta,
                        src[k * NT + t].x, meta[k] & 0x7FFu, 3, st))
          cmask |= 1u << k;
      }
    }
    if (__any_sync(0xFFFFFFFFu, cmask)) {
#pragma unroll
      for (int k = 0; k < EPT; ++k) {
        const bool cand = (cmask >> k) & 1u;
        const uint32_t bm = __ballot_sync(0xFFFFFFFFu, cand);
        if (bm) {
          const uint32_t leader = __ffs(bm) - 1u;
          uint32_t base = 0;
          if (lane == leader) base = atomicAdd(s_cnt + p, (uint32_t)__popc(bm));
          base = __shfl_sync(0xFFFFFFFFu, base, leader);
          if (cand) cl[base + __popc(bm & ((1u << lane) - 1u))] = (uint16_t)((uint32_t)k * NT + t);
        }
      }
    }
    // next unit: the next round of this block, or the next block
    if (ws + NSLOT <= elast) {
      // first record past the window (records are in epoch order)
      const uint32_t e0 = acc_epoch(src[0].y), lim = e0 + ws + NSLOT;
      uint32_t lo = 0, hi = n;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (acc_epoch(src[mid].y) < lim) lo = mid + 1; else hi = mid;
      }
      ws = lo < n ? acc_epoch(src[lo].y) - e0 : elast + 1;
      p1(++stamp & 0xFFFFu);
    } else {
      pend = true;
      pheld = held;
      pit = it;
      pb = b;
      pj = j;
      pn = n;
      j += G;
      ++it;
      live = j < nblk;
      if (live) b = blk(j);
      if (live) {
        load_block();
        p1(++stamp & 0xFFFFu);
        fresh = true;
      }
    }
  }
  flags = __reduce_or_sync(0xFFFFFFFFu, flags);
  if (lane == 0 && flags) atomicOr(&s_flags, flags);
  __syncthreads();
  if (t < LTN && s_lt_line[t] != INF) atomicMin(P.line_first + s_lt_line[t], s_lt_ts[t]);
  if (t == 0 && s_flags) atomicOr(P.status, s_flags);
}

// ---------------- per-warp line-first cache (the fast path's report) ----
struct WarpOut {
  uint32_t lc_line;          // lane-owned line cache entry
  unsigned long long lc_ts;
  uint32_t lc_next;          // uniform: next slot to allocate
  uint32_t tbn;              // uniform: staged triples
  uint32_t flags;
};

// one line's first racing timestamp into the lane-owned cache (uniform call)
__device__ __forceinline__ void wo_line1(WarpOut& E, const Params& P, uint32_t L, unsigned long long T) {
  const uint32_t lane = threadIdx.x & 31u;
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

// ---------------- fast_kernel: the default path (one warp per block) ----
// Every warp streams whole simulated blocks on its own -- no CTA barrier on
// the per-event path.  A block's 1024 records are read with coalesced
// 16-byte loads (lane l holds records l, l + 32, ...), validated and packed
// into one register each, and the word filter of the two-pass design runs in
// the warp's own shared-memory tag arrays (one per epoch) with __syncwarp
// between its phases:
//   P1 tag[w] <- some accessing {tid, write} | P2 tid != tag[w] -> multi
//   stamp, write -> write stamp | P3 candidate iff both stamps are current.
// The few candidates (~3 % on C3) go through the exact check: the reference
// predicate (racecheck.cpp:24-32) on same-word groups found with
// __match_any_sync, (word, line) dedup by a second match, and the warp's
// line-first cache.  The fast path takes the shape of trace-mode blocks
// (C3): exactly FMAX records, aligned 4-byte accesses, at most two epochs,
// an object of at most FWORDS words.  Any other block -- or one with more
// than FCMAX candidates -- is appended to the overflow list untouched and
// redone by the general (fused) kernel, which validates every field.
#ifndef MCKG_FK_FW
#define MCKG_FK_FW 16
#endif
#ifndef MCKG_FK_MINB
#define MCKG_FK_MINB 1
#endif
#ifndef MCKG_FK_BR
#define MCKG_FK_BR 2
#endif
constexpr uint32_t FW = MCKG_FK_FW;  // warps per CTA
constexpr uint32_t FRPL = 32;      // records per lane
constexpr uint32_t FMAX = FRPL * 32;
constexpr uint32_t FWORDS = 1024;  // words per epoch (shared objects <= 4 KiB)
constexpr uint32_t FCMAX = 32;     // candidates per block (one per lane in the exact pass)

// per-warp dynamic shared memory: the two epochs' tag arrays, the candidates
constexpr uint32_t FK_TAGS = 0;
constexpr uint32_t FK_CL = FK_TAGS + 2 * FWORDS * 4;
constexpr uint32_t FK_WARP_BYTES = (FK_CL + FCMAX * 2 + 127u) & ~127u;
constexpr uint32_t FK_SMEM = FW * FK_WARP_BYTES;

// Packed record (one register): bits 0..10 tid, 11 write, 14..31 the
// shared-memory byte address of the word's tag entry {u16 tid | write << 11,
// u8 multi stamp, u8 write stamp} in its epoch's array, the word index
// swizzled so that the stride-4-word pattern of per-thread slots (tid * 4 + k)
// is bank-conflict free.  Bits 0..15 are exactly the u16 P1 stores.
__device__ __forceinline__ uint32_t fk_addr(uint32_t x) { return x >> 14; }

// Exact check and report of a block's m <= 32 candidates, one per lane.
// Aligned 4-byte records overlap iff they name the same word, so X races iff
// an earlier candidate Y of the same epoch and word, another thread, and X or
// Y writing exists (racecheck.cpp:24-32); all four bytes of X race then.
// Reported triples: one (obj, byte, line) set per racing (word, line) of the
// block (RaceState::reported, machine.hpp:91), appended with one atomic per
// block; the line's first racing timestamp goes to the warp's line cache.
__device__ __forceinline__ void fk_exact(WarpOut& E, const Params& P, const uint4* src, const uint16_t* cl,
                                         uint32_t m, uint32_t b) {
  const uint32_t lane = threadIdx.x & 31u;
  const bool act = lane < m;
  const uint32_t xi = act ? cl[lane] : 0xFFFFu;
  const uint4 X = act ? __ldg(src + xi) : make_uint4(0, 0, 0, 0);
  const uint32_t key = act ? (X.x & 0xFFFFFu) | ((X.y >> 11) << 20) : 0xFFFFFFFFu - lane;
  uint32_t rest = __match_any_sync(0xFFFFFFFFu, key) & ~(1u << lane);
  bool racing = false;
  while (__any_sync(0xFFFFFFFFu, rest != 0u)) {
    const uint32_t y = rest ? (uint32_t)__ffs(rest) - 1u : lane;
    rest &= rest - 1u;
    const uint32_t yi = __shfl_sync(0xFFFFFFFFu, xi, y), yx = __shfl_sync(0xFFFFFFFFu, X.x, y),
                   yy = __shfl_sync(0xFFFFFFFFu, X.y, y);
    racing |= y != lane && yi < xi && acc_tid(yy) != acc_tid(X.y) && ((X.x | yx) & (1u << 24));
  }
  const uint32_t rm = __ballot_sync(0xFFFFFFFFu, racing);
  if (!rm) return;
  const uint32_t line = X.z;
  // first racing timestamp per line (min over the block's racing lanes)
  const unsigned long long ts = ts_key(X.w, P.bid_base + b, acc_tid(X.y));
  for (uint32_t left = rm; left;) {
    const uint32_t L = __shfl_sync(0xFFFFFFFFu, line, __ffs(left) - 1);
    const bool in = racing && line == L;
    const uint32_t mh = __reduce_min_sync(0xFFFFFFFFu, in ? (uint32_t)(ts >> 32) : ~0u);
    const uint32_t ml = __reduce_min_sync(0xFFFFFFFFu, in && (uint32_t)(ts >> 32) == mh ? (uint32_t)ts : ~0u);
    left &= ~__ballot_sync(0xFFFFFFFFu, in);
    wo_line1(E, P, L, ((unsigned long long)mh << 32) | ml);
  }
  // one reporter per racing (word, line): the lowest racing lane of the group
  const uint32_t grp = __match_any_sync(0xFFFFFFFFu, racing ? ((X.x & 0xFFFFCu) << 12) ^ line : 0xFFFFFFFFu - lane);
  const bool rep = racing && (grp & ((1u << lane) - 1u) & rm) == 0u;
  const uint32_t rb = __ballot_sync(0xFFFFFFFFu, rep);
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(P.n_tri, 4ull * __popc(rb));
  base = __shfl_sync(0xFFFFFFFFu, base, 0);
  if (rep) {
    const unsigned long long at = base + 4ull * __popc(rb & ((1u << lane) - 1u));
    const uint32_t w4 = X.x & 0xFFFFCu;
    for (uint32_t q = 0; q < 4; ++q) {
      if (at + q < P.capacity)
        P.tri[at + q] = mckg_race_triple{P.obj_base + b, w4 + q, (int32_t)line};
      else
        E.flags |= ST_OVERFLOW;
    }
  }
}

__global__ void __launch_bounds__(FW * 32, MCKG_FK_MINB) fast_kernel(Params P) {
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31u;
  uint8_t* wbase = smem_raw + warp * FK_WARP_BYTES;
  uint32_t* tags = reinterpret_cast<uint32_t*>(wbase + FK_TAGS);
  uint16_t* cl = reinterpret_cast<uint16_t*>(wbase + FK_CL);
  for (uint32_t i = lane; i < 2 * FWORDS; i += 32) tags[i] = 0u;
  __syncwarp();
  const uint32_t tagb = smem_u32(tags);
  WarpOut E{INF, ~0ull, 0u, 0u, 0u};
  uint32_t stamp = 0;
  const uint32_t nwarps = gridDim.x * FW;
  const uint32_t shm = P.shmem_bytes;
  for (uint32_t b = blockIdx.x * FW + warp; b < P.n_blocks; b += nwarps) {
    const uint64_t s0 = P.bstart[b], s1 = P.bstart[b + 1];
    if (s1 - s0 != FMAX) {
      if (s1 != s0 && lane == 0) P.olist[atomicAdd(P.ocount, 1u)] = b;
      continue;
    }
    const uint4* src = reinterpret_cast<const uint4*>(P.ev + s0);
    // ---- load, validate, pack (4 rows in flight ahead of the decode) ----
    uint32_t pk[FRPL];
    uint32_t e0 = 0, chk = 0, mo = 0, mz = 0, ms = 0, up = 0;
    constexpr int BR = MCKG_FK_BR;  // rows per batch
    uint4 buf[2][BR];
#pragma unroll
    for (int q = 0; q < BR; ++q) buf[0][q] = __ldg(src + q * 32 + lane);
#pragma unroll
    for (int h = 0; h < (int)FRPL / BR; ++h) {
      if (h + 1 < (int)FRPL / BR) {
#pragma unroll
        for (int q = 0; q < BR; ++q) buf[(h + 1) & 1][q] = __ldg(src + ((h + 1) * BR + q) * 32 + lane);
      }
#pragma unroll
      for (int q = 0; q < BR; ++q) {
        const int j = h * BR + q;
        const uint4 r = buf[h & 1][q];
        const uint32_t ep = acc_epoch(r.y);
        if (j == 0) e0 = __shfl_sync(0xFFFFFFFFu, ep, 0);
        const uint32_t slot = ep - e0;
        const uint32_t off = acc_off(r.x);
        // aligned 4-byte access (len 4, bits 25..31 clear); the object
        // bound, the line and the epoch span are checked on per-lane maxima
        chk |= (r.x & 0xFEF00003u) ^ 0x00400000u;
        mo = max(mo, off);
        mz = max(mz, (uint32_t)r.z);
        ms = max(ms, slot);
        up |= slot << j;  // bit j: record j * 32 + lane is in the second epoch
        const uint32_t a = tagb + ((slot << 12) | (off ^ ((off >> 5) & 0x7Cu)));
        pk[j] = (((r.y & 0x7FFu) | ((r.x >> 13) & 0x800u))) + (a << 14);
      }
    }
    // epochs non-decreasing in record order: every lane's second-epoch rows
    // form a top segment starting at row f_l, with f non-increasing over the
    // lanes and f_0 - f_31 <= 1
    const uint32_t f = up ? (uint32_t)__ffs(up) - 1u : 32u;
    bool bad = chk != 0u || mo + 4u > shm || mz >= 65536u || ms > 1u || (up != 0u && (up | (up - 1u)) != ~0u);
    const uint32_t fn = __shfl_down_sync(0xFFFFFFFFu, f, 1);
    bad |= lane < 31u && fn > f;
    const uint32_t f0 = __shfl_sync(0xFFFFFFFFu, f, 0), f31 = __shfl_sync(0xFFFFFFFFu, f, 31);
    bad |= f0 > f31 + 1u;
    if (__any_sync(0xFFFFFFFFu, bad)) {
      if (lane == 0) P.olist[atomicAdd(P.ocount, 1u)] = b;
      continue;
    }
    stamp = stamp == 255u ? 1u : stamp + 1u;
    const uint32_t pat = (stamp | (stamp << 8)) << 16;
    // P1: the u16 {tid, write} of some accessing record per word
#pragma unroll
    for (int j = 0; j < (int)FRPL; ++j)
      asm volatile("st.shared.u16 [%0], %1;" ::"r"(fk_addr(pk[j])), "h"((uint16_t)pk[j]) : "memory");
    __syncwarp();
    // P2: words seen by a second thread; written words
#pragma unroll
    for (int j = 0; j < (int)FRPL; ++j) {
      const uint32_t x = pk[j], a = fk_addr(x);
      uint16_t tg;
      asm volatile("ld.shared.u16 %0, [%1];" : "=h"(tg) : "r"(a) : "memory");
      if ((((uint32_t)tg ^ x) & 0x7FFu) != 0u)
        asm volatile("st.shared.u8 [%0+2], %1;" ::"r"(a), "h"((uint16_t)stamp) : "memory");
      if (x & 0x800u) asm volatile("st.shared.u8 [%0+3], %1;" ::"r"(a), "h"((uint16_t)stamp) : "memory");
    }
    __syncwarp();
    // P3: candidates -> per-lane row bits
    uint32_t cm = 0;
#pragma unroll
    for (int j = 0; j < (int)FRPL; ++j) {
      uint32_t v;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(fk_addr(pk[j])) : "memory");
      cm |= ((v & 0xFFFF0000u) == pat ? 1u : 0u) << j;
    }
    // compaction (the list order is free: the exact pass compares indices)
    const uint32_t c = __popc(cm);
    uint32_t incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, d);
      if (lane >= (uint32_t)d) incl += t;
    }
    const uint32_t m = __shfl_sync(0xFFFFFFFFu, incl, 31);
    if (m == 0) continue;
    if (m > FCMAX) {
      if (lane == 0) P.olist[atomicAdd(P.ocount, 1u)] = b;
      continue;
    }
    uint32_t pos = incl - c;
    for (uint32_t g = cm; g; g &= g - 1u) cl[pos++] = (uint16_t)((uint32_t)(__ffs(g) - 1) * 32u + lane);
    __syncwarp();
    fk_exact(E, P, src, cl, m, b);
    __syncwarp();
  }
  if (E.lc_line != INF) atomicMin(P.line_first + E.lc_line, E.lc_ts);
  const uint32_t fl = __reduce_or_sync(0xFFFFFFFFu, E.flags);
  if (lane == 0 && fl) atomicOr(P.status, fl);
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



// The overflow list of the default path (two counters, then up to n_blocks
// block indices): one buffer per (device, stream, host thread for the
// special stream handles), grown on demand.
cudaError_t overflow_list(uint32_t n_blocks, cudaStream_t s, uint32_t** out) {
  struct Buf {
    uint32_t* p = nullptr;
    size_t n = 0;
  };
  static std::mutex mu;
  static std::map<std::tuple<int, cudaStream_t, std::thread::id>, Buf> bufs;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const bool special = s == nullptr || s == cudaStreamLegacy || s == cudaStreamPerThread;
  std::lock_guard<std::mutex> lock(mu);
  Buf& b = bufs[{dev, s, special ? std::this_thread::get_id() : std::thread::id()}];
  if (b.n < n_blocks || !b.p) {
    if (b.p) {
      if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
      if ((e = cudaFree(b.p)) != cudaSuccess) return e;
      b.p = nullptr;
    }
    if ((e = cudaMalloc(&b.p, ((size_t)n_blocks + 2) * sizeof(uint32_t))) != cudaSuccess) return e;
    b.n = n_blocks;
  }
  *out = b.p;
  return cudaSuccess;
}

// The >48 KB dynamic shared-memory opt-in is a per-device function
// attribute: remembered per (device, kernel), raised on demand.
cudaError_t ensure_dynamic_smem(void (*k)(Params), size_t bytes) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::map<std::pair<int, void (*)(Params)>, size_t> done;
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[{dev, k}];
  if (bytes <= have) return cudaSuccess;
  e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

// ---- the oversize route: blocks beyond the kernels' staging (more than
// 4096 records) or shared objects beyond the on-chip filter ----
// One block at a time through K6 (mckg_detect_global) with the K2 semantics
// mapped onto it: address = (epoch - first epoch) << 20 | byte offset, so
// records of different epochs never meet; the "block" of a K6 record is the
// thread (races are between threads here); its sweep is the record's index
// in the block, so K6's "earlier" is the replay order of recordAccess
// (racecheck.cpp:24-32).  Racing (address, line) pairs become the block's
// (obj, byte, line) triples; K6's first racing key per line names the
// record, whose real (sweep, bid, tid) key is MIN-ed into line_first.
__global__ void oversize_map_kernel(const mckg_access* ev, uint64_t n, uint32_t shmem, mckg_gaccess* out,
                                    uint32_t* status) {
  const uint32_t e0 = n ? acc_epoch(ev[0].w1) : 0u;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const mckg_access r = ev[i];
    const uint32_t off = acc_off(r.w0), len = acc_len(r.w0), tid = acc_tid(r.w1), ep = acc_epoch(r.w1);
    const uint32_t prev = i ? acc_epoch(ev[i - 1].w1) : ep;
    bool ok = len - 1u < MCKG_MAX_LEN && off + len <= shmem && (uint32_t)r.line < MCKG_MAX_LINES;
    if (ep < prev) atomicOr(status, ST_ORDER);
    const uint32_t rel = ep - e0;
    if (ep < e0 || rel >= (1u << 20)) ok = false;
    if (!ok) atomicOr(status, ST_RANGE);
    // one (byte, line) racing in two epochs is two K6 addresses: the triples
    // may repeat, and the caller's sort restores the set (MCKG_ST_DUP)
    if (__any_sync(__activemask(), rel > 0) && (threadIdx.x & 31u) == (uint32_t)(__ffs(__activemask()) - 1))
      atomicOr(status, ST_DUP);
    const uint32_t ln = (uint32_t)r.line;
    mckg_gaccess g;
    g.a = ((((unsigned long long)rel << 20) | off) & 0xFFFFFFFFFFull) | ((unsigned long long)(ok ? len : 0u) << 40) |
          ((unsigned long long)acc_write(r.w0) << 44) | ((unsigned long long)tid << 45) |
          ((unsigned long long)(ln & 0xFFu) << 56);
    g.sweep = (uint32_t)i;
    g.b = tid | (((ln >> 8) & 0xFFu) << 24);
    out[i] = g;
  }
}

__global__ void oversize_report_kernel(const mckg_grace* races, const unsigned long long* n_races, uint64_t cap_races,
                                       uint32_t obj, mckg_race_triple* tri, unsigned long long capacity,
                                       unsigned long long* n_tri, uint32_t* status) {
  const uint64_t n = *n_races < cap_races ? *n_races : cap_races;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = atomicAdd(n_tri, 1ull);
    if (k < capacity)
      tri[k] = mckg_race_triple{obj, (uint32_t)(races[i].addr & 0xFFFFFu), races[i].line};
    else
      atomicOr(status, ST_OVERFLOW);
  }
}

__global__ void oversize_lines_kernel(const unsigned long long* lf6, const mckg_access* ev, uint32_t bid,
                                      unsigned long long* line_first) {
  const uint32_t l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= MCKG_MAX_LINES || lf6[l] == ~0ull) return;
  const mckg_access r = ev[lf6[l] >> 32];  // the first racing record of the line
  atomicMin(line_first + l, ts_key(r.sweep, bid, acc_tid(r.w1)));
}

int detect_oversize(const mckg_trace* tr, const mckg_race_out* out, cudaStream_t s, const std::vector<uint32_t>& blocks,
                    const std::vector<uint64_t>& hbs) {
  uint64_t maxn = 0;
  for (uint32_t b : blocks) maxn = std::max<uint64_t>(maxn, hbs[b + 1] - hbs[b]);
  if (maxn == 0) return MCKG_OK;
  mckg_gaccess* g = nullptr;
  mckg_grace* races = nullptr;
  unsigned long long* cnt = nullptr;  // [0] races, [1..] K6 line table
  uint32_t* st6 = nullptr;
  const uint64_t rcap = maxn * 8 + 64;
  PoolGuard pg(s);
  MCKG_CUDA_TRY(pg.alloc(&g, maxn * sizeof(mckg_gaccess)));
  MCKG_CUDA_TRY(pg.alloc(&races, rcap * sizeof(mckg_grace)));
  MCKG_CUDA_TRY(pg.alloc(&cnt, (1 + MCKG_MAX_LINES) * sizeof(unsigned long long)));
  MCKG_CUDA_TRY(pg.alloc(&st6, sizeof(uint32_t)));
  for (uint32_t b : blocks) {
    const uint64_t n = hbs[b + 1] - hbs[b];
    if (n == 0) continue;
    const mckg_access* ev = tr->events + hbs[b];
    const uint32_t grid = (uint32_t)std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count() * 8);
    oversize_map_kernel<<<grid, 256, 0, s>>>(ev, n, tr->shmem_bytes, g, out->status);
    MCKG_CUDA_TRY(cudaMemsetAsync(cnt + 1, 0xFF, MCKG_MAX_LINES * sizeof(unsigned long long), s));
    MCKG_CUDA_TRY(cudaMemsetAsync(st6, 0, sizeof(uint32_t), s));
    int rc = mckg_detect_global(g, n, 0, races, rcap, cnt, cnt + 1, st6, s);
    if (rc != MCKG_OK) return rc;
    oversize_report_kernel<<<grid, 256, 0, s>>>(races, cnt, rcap, tr->obj_base + b, out->triples, out->capacity,
                                                out->n_triples, out->status);
    oversize_lines_kernel<<<MCKG_MAX_LINES / 256, 256, 0, s>>>(cnt + 1, ev, tr->bid_base + b, out->line_first);
    MCKG_CUDA_TRY(cudaGetLastError());
  }
  return MCKG_OK;
}

}  // namespace

int detect_config(uint32_t cap, uint32_t shmem_bytes, size_t* smem, uint32_t* wpad) {
  uint32_t words = (shmem_bytes + 3u) / 4u;
  *wpad = (words + 31u) & ~31u;
  if (*wpad == 0) *wpad = 32;
  *smem = layout(cap, *wpad, MCKG_K2_NSTAGE).end;  // the larger (fused) configuration
  return *smem + 11u * 1024u <= 227u * 1024u ? MCKG_OK : MCKG_E_RANGE;
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
  cudaStream_t s = (cudaStream_t)stream;
  size_t smem;
  uint32_t wpad;
  const bool big_blocks = cap > (uint32_t)EPT_MAX * NT;
  const bool big_object = detect_config(std::min<uint32_t>(cap, EPT_MAX * NT), tr->shmem_bytes, &smem, &wpad) != MCKG_OK;
  if (big_blocks || big_object) {
    // blocks past the on-chip staging / filter take the oversize route
    std::vector<uint64_t> hbs((size_t)tr->n_blocks + 1);
    MCKG_CUDA_TRY(cudaMemcpyAsync(hbs.data(), tr->block_start, hbs.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    MCKG_CUDA_TRY(cudaStreamSynchronize(s));
    std::vector<uint32_t> big;
    for (uint32_t b = 0; b < tr->n_blocks; ++b)
      if (big_object || hbs[b + 1] - hbs[b] > (uint64_t)EPT_MAX * NT) big.push_back(b);
    keep_pool_memory();
    const int rc = detect_oversize(tr, out, s, big, hbs);
    if (rc != MCKG_OK || big_object) {
      add_launches((uint32_t)big.size() * 9u);
      return rc;
    }
    cap = EPT_MAX * NT;  // the rest: the kernels below, oversize blocks skipped
  }
  // the general kernel: records staged per block by TMA, EPT per thread
  const int ki = cap <= 4u * NT ? 0 : cap <= 8u * NT ? 1 : 2;
  void (*kf)(Params) = ki == 0 ? race_detect_kernel<4> : ki == 1 ? race_detect_kernel<8> : race_detect_kernel<16>;
  const size_t smem_f = layout(cap, wpad, MCKG_K2_NSTAGE).end;
  MCKG_CUDA_TRY(ensure_dynamic_smem(kf, smem_f));
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kf, NT, smem_f) != cudaSuccess || per_sm < 1) per_sm = 1;
  uint32_t grid_f = (uint32_t)sm_count() * (uint32_t)per_sm;
  if (grid_f > tr->n_blocks) grid_f = tr->n_blocks;
  Params P{};
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
  P.debug = debug_flags();
  P.gate = 0;
  P.skip_big = big_blocks ? 1u : 0u;
  P.ocount = nullptr;
  P.olist = nullptr;
  if ((P.debug & 32u) || tr->shmem_bytes > FWORDS * 4u) {
    // the general kernel alone (MCKG_DEBUG=32: the tests cover both paths;
    // shared objects over 4 KiB: no fast path)
    kf<<<grid_f, NT, smem_f, s>>>(P);
    MCKG_CUDA_TRY(cudaGetLastError());
    note_launch(1, grid_f, NT, (uint32_t)smem_f);
    return MCKG_OK;
  }
  // default path: fast_kernel (one warp per block); the general kernel,
  // gated on the overflow list, redoes the blocks the fast path hands back
  uint32_t* ol = nullptr;
  MCKG_CUDA_TRY(overflow_list(tr->n_blocks, s, &ol));
  P.ocount = ol;
  P.olist = ol + 2;
  MCKG_CUDA_TRY(cudaMemsetAsync(P.ocount, 0, 2 * sizeof(uint32_t), s));
  MCKG_CUDA_TRY(ensure_dynamic_smem(fast_kernel, FK_SMEM));
  int per = 0;
  MCKG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, fast_kernel, FW * 32, FK_SMEM));
  if (per < 1) per = 1;
  uint32_t g = (uint32_t)sm_count() * (uint32_t)per;
  const uint32_t need = (tr->n_blocks + FW - 1) / FW;
  if (g > need) g = need;
  fast_kernel<<<g, FW * 32, FK_SMEM, s>>>(P);
  MCKG_CUDA_TRY(cudaGetLastError());
  P.gate = 1;
  kf<<<grid_f, NT, smem_f, s>>>(P);
  MCKG_CUDA_TRY(cudaGetLastError());
  note_launch(2, g, FW * 32, FK_SMEM);
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
  // (obj - obj_base):22 | byte:20 | line:16 keys, radix-sorted (sort.cu),
  // optionally reduced to the distinct ones, decoded back in place
  unsigned long long *k0 = nullptr, *k1 = nullptr;
  PoolGuard pg(s);
  MCKG_CUDA_TRY(pg.alloc(&k0, n * sizeof(unsigned long long)));
  MCKG_CUDA_TRY(pg.alloc(&k1, n * sizeof(unsigned long long)));
  uint32_t nb = (uint32_t)((n + 255) / 256);
  uint32_t launches = 1;
  encode_triples<<<nb, 256, 0, s>>>(triples, k0, n, obj_base);
  MCKG_CUDA_TRY(radix_sort_u64(k0, k1, n, 58, s, &launches));
  if (n_unique) {
    MCKG_CUDA_TRY(unique_sorted_u64(k0, n, k1, n_unique, s, &launches));
    decode_triples<<<nb, 256, 0, s>>>(k1, triples, n_unique, n, obj_base);
  } else {
    decode_triples<<<nb, 256, 0, s>>>(k0, triples, nullptr, n, obj_base);
  }
  MCKG_CUDA_TRY(cudaGetLastError());
  add_launches(launches + 1);
  return MCKG_OK;
}
