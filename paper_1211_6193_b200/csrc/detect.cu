// detect.cu -- K2: block-local shared-memory race detector (sm_100a).
//
// Replaces Machine::recordAccess / Machine::clearEpoch (racecheck.cpp:9-73)
// for a whole grid at once.  The reference keeps a per-byte shadow list and,
// for every access X of byte b, flags X iff an earlier access to b in the
// same barrier epoch came from another thread and one of the two is a write.
// That predicate only needs, per (epoch, byte):
//     j1 = first access, j2 = first access by a thread other than j1's,
//     w1 = first write,  w2 = first write by a thread other than w1's;
// X (a write) races iff min{other-thread access} = (X.tid != tid(j1) ? j1 : j2) < X,
// X (a read)  races iff (X.tid != tid(w1) ? w1 : w2) < X.
//
// Design (one CTA streams many simulated blocks; blocks never interact
// because every block owns its own shared object, device.cpp:33-38):
//   * the block's records are pulled into shared memory by the TMA engine
//     (cp.async.bulk + mbarrier), double-buffered across blocks;
//   * epoch segments are found with a warp-cooperative 32-ary search (records
//     are in timestamp order, so epochs are non-decreasing);
//   * per epoch a 3-pass shared-memory filter finds the words touched by >= 2
//     threads with >= 1 write (order-free: a byte races at all iff that holds);
//   * only events on such words enter the exact pass (shared atomicMin of
//     (index, tid) keys gives j1/j2/w1/w2);
//   * racing (word, line) pairs are deduplicated per block (the reported set
//     is per object) in a shared hash set, staged in shared memory and
//     appended to the global triple array in chunks; the first racing
//     timestamp per line is min-reduced in shared memory, then globally.
// Words are `g` bytes where g = the largest power of two (<= 8) dividing every
// offset and length of the block, so the per-word state is the per-byte state
// of each of its bytes.
#include <cub/cub.cuh>

#include "common.cuh"

namespace mckg {
namespace {

constexpr int NT = 256;
constexpr int NSTAGE = 2;
constexpr uint32_t HS = 512;    // (word, line) dedup set entries
constexpr uint32_t TBN = 768;   // staged triples before a global flush
constexpr uint32_t LTN = 32;    // line-first local table entries
constexpr uint32_t INF = 0xFFFFFFFFu;
constexpr uint32_t ST_OVERFLOW = 1u, ST_RANGE = 2u, ST_ORDER = 4u;

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

struct Smem {
  mckg_access* stage;
  uint32_t *A, *B, *C, *D;  // tag|A1, multi|W1, anyw|A2, W2
  unsigned long long* hset;
  mckg_race_triple* tbuf;
  uint32_t* lt_line;
  unsigned long long* lt_ts;
  uint8_t* cm;
  uint64_t* mbar;
  uint32_t* misc;  // [0] tbuf fill, [1] OR of off|len, [2] flags, [3] flush base lo, [4] hi
};

__host__ __device__ inline size_t smem_bytes_for(uint32_t cap, uint32_t wpad) {
  size_t b = 0;
  b += (size_t)NSTAGE * cap * sizeof(mckg_access);
  b += 4ull * wpad * sizeof(uint32_t);
  b += HS * sizeof(unsigned long long);
  b += LTN * sizeof(unsigned long long);
  b += TBN * sizeof(mckg_race_triple);
  b += LTN * sizeof(uint32_t);
  b += NSTAGE * sizeof(uint64_t) + 8 * sizeof(uint32_t);
  b += cap;  // cm
  return (b + 127) & ~size_t(127);
}

__device__ __forceinline__ uint32_t sw(uint32_t w) { return w ^ ((w >> 5) & 31u); }

__device__ __forceinline__ void load_ev(const mckg_access* src, uint32_t i, uint32_t& w0,
                                        uint32_t& w1, int32_t& line, uint32_t& sweep) {
  uint4 v = *reinterpret_cast<const uint4*>(src + i);
  w0 = v.x;
  w1 = v.y;
  line = (int32_t)v.z;
  sweep = v.w;
}

__device__ __forceinline__ bool valid_ev(uint32_t w0, int32_t line, uint32_t shm) {
  uint32_t off = acc_off(w0), len = acc_len(w0);
  return len != 0 && len <= MCKG_MAX_LEN && off + len <= shm && (uint32_t)line < MCKG_MAX_LINES;
}

__device__ __forceinline__ uint32_t load_epoch(const mckg_access* src, uint32_t i) {
  return acc_epoch(src[i].w1);
}

// First index in (s, n) whose epoch differs from ep, or n.  Warp-cooperative
// 32-ary search; every warp computes the same (uniform) answer.
__device__ uint32_t seg_end(const mckg_access* src, uint32_t s, uint32_t n, uint32_t ep) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t lo = s, hi = n;  // epoch(lo) == ep; answer in (lo, hi]
  while (hi - lo > 1) {
    uint32_t step = (hi - lo + 31u) / 32u;
    uint32_t p = lo + (lane + 1u) * step;
    bool pred = p < hi && load_epoch(src, p) != ep;
    uint32_t m = __ballot_sync(0xFFFFFFFFu, pred);
    if (m == 0) {
      lo += ((hi - 1u - lo) / step) * step;  // last sampled position below hi
    } else {
      uint32_t f = __ffs(m) - 1u;
      uint32_t pf = lo + (f + 1u) * step;
      lo = f == 0 ? lo : lo + f * step;
      hi = pf;
    }
  }
  return hi;
}

__device__ bool hset_insert(unsigned long long* hs, unsigned long long key, unsigned long long bstamp,
                            bool& overflow) {
  uint32_t h = (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> 40) & (HS - 1);
  for (uint32_t probe = 0; probe < HS; ++probe) {
    unsigned long long cur = hs[h];
    while ((cur >> 36) != bstamp) {  // stale slot: claim it
      unsigned long long old = atomicCAS(hs + h, cur, key);
      if (old == cur) return true;
      cur = old;
    }
    if (cur == key) return false;
    h = (h + 1) & (HS - 1);
  }
  overflow = true;
  return true;  // table full: report (possible duplicate flagged by status)
}

__device__ void line_note(Smem& S, const Params& P, int32_t line, unsigned long long ts) {
  uint32_t l = (uint32_t)line;
  uint32_t h = l & (LTN - 1);
  for (uint32_t probe = 0; probe < LTN; ++probe) {
    uint32_t v = S.lt_line[h];
    if (v == INF) {
      uint32_t old = atomicCAS(S.lt_line + h, INF, l);
      v = old == INF ? l : old;
    }
    if (v == l) {
      atomicMin(S.lt_ts + h, ts);
      return;
    }
    h = (h + 1) & (LTN - 1);
  }
  atomicMin(P.line_first + l, ts);
}

__device__ void emit_word(Smem& S, const Params& P, uint32_t obj, uint32_t w, uint32_t g,
                          int32_t line, unsigned long long bstamp) {
  unsigned long long key =
      (bstamp << 36) | ((unsigned long long)(w & 0xFFFFFu) << 16) | ((uint32_t)line & 0xFFFFu);
  bool ovf = false;
  if (!hset_insert(S.hset, key, bstamp, ovf)) return;
  if (ovf) atomicOr(P.status, ST_OVERFLOW);
  uint32_t pos = atomicAdd(S.misc + 0, g);
  uint32_t inbuf = pos >= TBN ? 0u : (TBN - pos < g ? TBN - pos : g);
  for (uint32_t b = 0; b < inbuf; ++b)
    S.tbuf[pos + b] = mckg_race_triple{obj, w * g + b, line};
  if (inbuf < g) {  // staging buffer full: append the rest directly
    uint32_t rest = g - inbuf;
    unsigned long long gp = atomicAdd(P.n_tri, (unsigned long long)rest);
    for (uint32_t b = 0; b < rest; ++b) {
      if (gp + b < P.capacity)
        P.tri[gp + b] = mckg_race_triple{obj, w * g + inbuf + b, line};
      else
        atomicOr(P.status, ST_OVERFLOW);
    }
  }
}

// Flushes the staged triples (uniform call, all threads).
__device__ void flush_tbuf(Smem& S, const Params& P) {
  __syncthreads();
  uint32_t n = S.misc[0] < TBN ? S.misc[0] : TBN;
  if (n == 0) return;
  if (threadIdx.x == 0) {
    unsigned long long base = atomicAdd(P.n_tri, (unsigned long long)n);
    S.misc[3] = (uint32_t)base;
    S.misc[4] = (uint32_t)(base >> 32);
  }
  __syncthreads();
  unsigned long long base = ((unsigned long long)S.misc[4] << 32) | S.misc[3];
  for (uint32_t i = threadIdx.x; i < n; i += NT) {
    if (base + i < P.capacity)
      P.tri[base + i] = S.tbuf[i];
    else
      atomicOr(P.status, ST_OVERFLOW);
  }
  __syncthreads();
  if (threadIdx.x == 0) S.misc[0] = 0;
}

// One barrier epoch [s, e) of a block.
__device__ void process_epoch(Smem& S, const Params& P, const mckg_access* src, uint32_t s,
                              uint32_t e, uint32_t lg, uint32_t stamp, uint32_t obj, uint32_t bid,
                              unsigned long long bstamp) {
  const uint32_t t = threadIdx.x;
  const uint32_t shm = P.shmem_bytes;
  // P1: tag[w] = some tid that touches w
  for (uint32_t i = s + t; i < e; i += NT) {
    uint32_t w0, w1, sweep;
    int32_t line;
    load_ev(src, i, w0, w1, line, sweep);
    if (!valid_ev(w0, line, shm)) continue;
    uint32_t off = acc_off(w0), len = acc_len(w0);
    uint32_t tid = acc_tid(w1);
    for (uint32_t w = off >> lg; w < (off + len) >> lg; ++w) S.A[sw(w)] = tid;
  }
  __syncthreads();
  // P2: mark words seen by a second thread; mark written words
  for (uint32_t i = s + t; i < e; i += NT) {
    uint32_t w0, w1, sweep;
    int32_t line;
    load_ev(src, i, w0, w1, line, sweep);
    if (!valid_ev(w0, line, shm)) continue;
    uint32_t off = acc_off(w0), len = acc_len(w0);
    uint32_t tid = acc_tid(w1);
    bool wr = acc_write(w0);
    for (uint32_t w = off >> lg; w < (off + len) >> lg; ++w) {
      uint32_t x = sw(w);
      if (S.A[x] != tid) S.B[x] = stamp;
      if (wr) S.C[x] = stamp;
    }
  }
  __syncthreads();
  // P3: candidate words = multi-thread and written
  int cand = 0;
  for (uint32_t i = s + t; i < e; i += NT) {
    uint32_t w0 = src[i].w0;
    uint32_t off = acc_off(w0), len = acc_len(w0);
    uint8_t m = 0;
    if (valid_ev(w0, src[i].line, shm)) {
      uint32_t q = 0;
      for (uint32_t w = off >> lg; w < (off + len) >> lg; ++w, ++q) {
        uint32_t x = sw(w);
        if (S.B[x] == stamp && S.C[x] == stamp) m |= (uint8_t)(1u << q);
      }
    }
    S.cm[i - s] = m;
    cand |= m;
  }
  if (!__syncthreads_or(cand)) return;

  // Exact pass over candidate words only.
  // E1: reset the four key tables for candidate words
  for (uint32_t i = s + t; i < e; i += NT) {
    uint8_t m = S.cm[i - s];
    if (!m) continue;
    uint32_t off = acc_off(src[i].w0);
    for (uint32_t q = 0; m; ++q, m >>= 1)
      if (m & 1) {
        uint32_t x = sw((off >> lg) + q);
        S.A[x] = INF;
        S.B[x] = INF;
        S.C[x] = INF;
        S.D[x] = INF;
      }
  }
  __syncthreads();
  // E2: first access / first write
  for (uint32_t i = s + t; i < e; i += NT) {
    uint8_t m = S.cm[i - s];
    if (!m) continue;
    uint32_t w0 = src[i].w0, w1 = src[i].w1;
    uint32_t key = ((i - s) << 11) | acc_tid(w1);
    bool wr = acc_write(w0);
    uint32_t off = acc_off(w0);
    for (uint32_t q = 0; m; ++q, m >>= 1)
      if (m & 1) {
        uint32_t x = sw((off >> lg) + q);
        atomicMin(S.A + x, key);
        if (wr) atomicMin(S.B + x, key);
      }
  }
  __syncthreads();
  // E3: first access / write by a thread other than the first one's
  for (uint32_t i = s + t; i < e; i += NT) {
    uint8_t m = S.cm[i - s];
    if (!m) continue;
    uint32_t w0 = src[i].w0, w1 = src[i].w1;
    uint32_t tid = acc_tid(w1);
    uint32_t key = ((i - s) << 11) | tid;
    bool wr = acc_write(w0);
    uint32_t off = acc_off(w0);
    for (uint32_t q = 0; m; ++q, m >>= 1)
      if (m & 1) {
        uint32_t x = sw((off >> lg) + q);
        if ((S.A[x] & 0x7FFu) != tid) atomicMin(S.C + x, key);
        if (wr && (S.B[x] & 0x7FFu) != tid) atomicMin(S.D + x, key);
      }
  }
  __syncthreads();
  // E4: decide, dedup, emit
  const uint32_t g = 1u << lg;
  for (uint32_t i = s + t; i < e; i += NT) {
    uint8_t m = S.cm[i - s];
    if (!m) continue;
    uint32_t w0, w1, sweep;
    int32_t line;
    load_ev(src, i, w0, w1, line, sweep);
    uint32_t tid = acc_tid(w1);
    bool wr = acc_write(w0);
    uint32_t off = acc_off(w0);
    uint32_t me = i - s;
    bool raced_any = false;
    for (uint32_t q = 0; m; ++q, m >>= 1)
      if (m & 1) {
        uint32_t w = (off >> lg) + q;
        uint32_t x = sw(w);
        uint32_t other;
        if (wr) {
          uint32_t a1 = S.A[x];
          other = ((a1 & 0x7FFu) != tid ? a1 : S.C[x]) >> 11;
        } else {
          uint32_t f1 = S.B[x];
          other = ((f1 & 0x7FFu) != tid ? f1 : S.D[x]) >> 11;
        }
        if (other < me) {
          raced_any = true;
          emit_word(S, P, obj, w, g, line, bstamp);
        }
      }
    if (raced_any) line_note(S, P, line, ts_key(sweep, bid, tid));
  }
  __syncthreads();
}

__global__ void __launch_bounds__(NT, 2) race_detect_kernel(Params P) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  Smem S;
  {
    uint8_t* p = smem_raw;
    S.stage = reinterpret_cast<mckg_access*>(p);
    p += (size_t)NSTAGE * P.cap * sizeof(mckg_access);
    S.A = reinterpret_cast<uint32_t*>(p);
    S.B = S.A + P.wpad;
    S.C = S.B + P.wpad;
    S.D = S.C + P.wpad;
    p += 4ull * P.wpad * sizeof(uint32_t);
    S.hset = reinterpret_cast<unsigned long long*>(p);
    p += HS * sizeof(unsigned long long);
    S.lt_ts = reinterpret_cast<unsigned long long*>(p);
    p += LTN * sizeof(unsigned long long);
    S.tbuf = reinterpret_cast<mckg_race_triple*>(p);
    p += TBN * sizeof(mckg_race_triple);
    S.lt_line = reinterpret_cast<uint32_t*>(p);
    p += LTN * sizeof(uint32_t);
    S.mbar = reinterpret_cast<uint64_t*>(p);
    p += NSTAGE * sizeof(uint64_t);
    S.misc = reinterpret_cast<uint32_t*>(p);
    p += 8 * sizeof(uint32_t);
    S.cm = p;
  }
  const uint32_t t = threadIdx.x;
  for (uint32_t i = t; i < HS; i += NT) S.hset[i] = 0ull;
  for (uint32_t i = t; i < LTN; i += NT) {
    S.lt_line[i] = INF;
    S.lt_ts[i] = ~0ull;
  }
  for (uint32_t i = t; i < 4 * P.wpad; i += NT) S.A[i] = 0u;
  if (t < 8) S.misc[t] = 0u;
  if (t == 0) {
    for (int k = 0; k < NSTAGE; ++k) mbar_init(S.mbar + k, 1);
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
    uint32_t bytes = (uint32_t)((P.bstart[b + 1] - s0) * sizeof(mckg_access));
    mbar_expect_tx(S.mbar + st, bytes);
    bulk_g2s(S.stage + (size_t)st * P.cap, P.ev + s0, bytes, S.mbar + st);
  };
  if (t == 0) {
    for (int k = 0; k < NSTAGE; ++k) {
      uint32_t b = blockIdx.x + (uint32_t)k * G;
      if (b < P.n_blocks && fits(b)) issue(b, k);
    }
  }
  uint32_t phase = 0;  // bit k = parity of stage k
  uint32_t stamp = 0;
  unsigned long long bstamp = 0;
  int it = 0;
  for (uint32_t b = blockIdx.x; b < P.n_blocks; b += G, ++it) {
    const int st = it % NSTAGE;
    const uint64_t s0 = P.bstart[b];
    const uint64_t n_all = P.bstart[b + 1] - s0;
    const uint32_t n = n_all <= P.cap ? (uint32_t)n_all : 0u;
    const bool staged = n > 0;
    if (t == 0) S.misc[5 + ((it + 1) & 1)] = 0u;  // OR slot of the next block
    const mckg_access* src;
    if (staged) {
      mbar_wait(S.mbar + st, (phase >> st) & 1u);
      phase ^= 1u << st;
      src = S.stage + (size_t)st * P.cap;
    } else {
      src = P.ev + s0;
    }
    ++bstamp;
    const uint32_t obj = P.obj_base + b;
    const uint32_t bid = P.bid_base + b;
    if (staged) {
      // pre-pass: granularity, order and range checks
      uint32_t orb = 0, bad = 0;
      for (uint32_t i = t; i < n; i += NT) {
        uint32_t w0 = src[i].w0;
        uint32_t off = acc_off(w0), len = acc_len(w0);
        orb |= off | len;
        if (len == 0 || len > MCKG_MAX_LEN || off + len > P.shmem_bytes) bad |= ST_RANGE;
        if (i > 0 && load_epoch(src, i) < load_epoch(src, i - 1)) bad |= ST_ORDER;
        if ((uint32_t)src[i].line >= MCKG_MAX_LINES) bad |= ST_RANGE;
      }
      orb = __reduce_or_sync(0xFFFFFFFFu, orb);
      bad = __reduce_or_sync(0xFFFFFFFFu, bad);
      if ((t & 31) == 0) {
        atomicOr(S.misc + 5 + (it & 1), orb & 7u);
        if (bad) atomicOr(S.misc + 2, bad);
      }
      __syncthreads();
      const uint32_t ob = S.misc[5 + (it & 1)];
      const uint32_t lg = (ob & 1u) ? 0u : (ob & 2u) ? 1u : (ob & 4u) ? 2u : 3u;
      uint32_t sgs = 0;
      while (sgs < n) {
        uint32_t ep = load_epoch(src, sgs);
        uint32_t sge = seg_end(src, sgs, n, ep);
        process_epoch(S, P, src, sgs, sge, lg, ++stamp, obj, bid, bstamp);
        sgs = sge;
      }
    } else if (n_all > 0) {
      if (t == 0) atomicOr(S.misc + 2, ST_RANGE);  // block larger than the staging capacity
    }
    __syncthreads();  // stage `st` fully consumed
    if (t == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      uint32_t nb = b + (uint32_t)NSTAGE * G;
      if (nb < P.n_blocks && fits(nb)) issue(nb, st);
    }
    if (S.misc[0] >= TBN / 2) flush_tbuf(S, P);
  }
  flush_tbuf(S, P);
  __syncthreads();
  for (uint32_t i = t; i < LTN; i += NT)
    if (S.lt_line[i] != INF) atomicMin(P.line_first + S.lt_line[i], S.lt_ts[i]);
  if (t == 0 && S.misc[2]) atomicOr(P.status, S.misc[2]);
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

__global__ void decode_triples(const unsigned long long* k, mckg_race_triple* t, uint64_t n,
                               uint32_t obj_base) {
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long v = k[i];
  t[i] = mckg_race_triple{obj_base + (uint32_t)(v >> 36), (uint32_t)((v >> 16) & 0xFFFFFu),
                          (int32_t)(v & 0xFFFFu)};
}

}  // namespace

int detect_config(uint32_t cap, uint32_t shmem_bytes, size_t* smem, uint32_t* wpad) {
  *wpad = (shmem_bytes + 31u) & ~31u;
  if (*wpad == 0) *wpad = 32;
  *smem = smem_bytes_for(cap, *wpad);
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
  if (!tr->events || !tr->block_start) {
    set_error("mckg_detect_shared: null trace");
    return MCKG_E_ARG;
  }
  if (tr->shmem_bytes > MCKG_MAX_OFF || (uint64_t)tr->bid_base + tr->n_blocks > MCKG_MAX_BID) {
    set_error("mckg_detect_shared: shmem_bytes or bid out of range");
    return MCKG_E_RANGE;
  }
  uint32_t cap = tr->max_block_events ? tr->max_block_events : 1024u;
  cap = (cap + 7u) & ~7u;
  size_t smem;
  uint32_t wpad;
  if (detect_config(cap, tr->shmem_bytes, &smem, &wpad) != MCKG_OK) {
    set_error("mckg_detect_shared: block does not fit the shared-memory staging");
    return MCKG_E_RANGE;
  }
  static thread_local size_t configured = 0;
  if (smem > configured) {
    MCKG_CUDA_TRY(cudaFuncSetAttribute(race_detect_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    configured = smem;
  }
  int per_sm = 0;
  MCKG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, race_detect_kernel, NT, smem));
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
  race_detect_kernel<<<grid, NT, smem, (cudaStream_t)stream>>>(P);
  MCKG_CUDA_TRY(cudaGetLastError());
  note_launch(1, grid, NT, (uint32_t)smem);
  return MCKG_OK;
}

extern "C" int mckg_sort_triples(mckg_race_triple* triples, uint64_t n, uint32_t obj_base,
                                 void* stream) {
  if (n == 0) return MCKG_OK;
  if (!triples) return MCKG_E_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long *k0 = nullptr, *k1 = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  MCKG_CUDA_TRY(cudaMallocAsync(&k0, n * sizeof(unsigned long long), s));
  MCKG_CUDA_TRY(cudaMallocAsync(&k1, n * sizeof(unsigned long long), s));
  uint32_t nb = (uint32_t)((n + 255) / 256);
  encode_triples<<<nb, 256, 0, s>>>(triples, k0, n, obj_base);
  cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, k0, k1, (int64_t)n, 0, 58, s);
  MCKG_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, s));
  MCKG_CUDA_TRY(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, k0, k1, (int64_t)n, 0, 58, s));
  decode_triples<<<nb, 256, 0, s>>>(k1, triples, n, obj_base);
  MCKG_CUDA_TRY(cudaGetLastError());
  cudaFreeAsync(tmp, s);
  cudaFreeAsync(k0, s);
  cudaFreeAsync(k1, s);
  add_launches(4);
  return MCKG_OK;
}
