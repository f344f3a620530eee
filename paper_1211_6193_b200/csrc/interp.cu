// interp.cu -- K1: the sm_100a thread-stepping interpreter of a simulated
// CUDA grid, with the shared-memory race detector (K2 contract) and the
// barrier-deadlock classification (K4) fused in.
//
// Mapping: one CTA = one simulated block, one GPU thread = one simulated
// thread (threadIdx.x == tid).  The CTA runs the block in lockstep SWEEPS:
// in sweep s every runnable thread executes exactly one IR instruction (one
// small step of Machine::execThreadStep, /root/reference/proj/src/machine.cpp:
// 493-1178), in the round-robin order of the reference (tid order inside a
// sweep, machine.cpp:411-429).  Barrier rules are not simulated one by one:
// SURVEY Appendix A gives their round-robin timing in closed form -- the
// episode completes in the sweep T of the last arrival (up-sweep chain +
// Turnaround, which clears the epoch, device.cpp:143-200), thread t >= 1 is
// released in sweep T + (L - t) and thread 0 in T + L (L = blockDim - 1), so
// thread t steps again from sweep T + L - t + 1 (t >= 1) / T + L + 1 (t = 0).
//
// Memory order inside a sweep.  Each step performs at most one memory access.
// Accesses to private objects (a thread's locals/params, virtual ids) never
// interact.  Shared/global accesses of one sweep are checked for word-level
// overlap with a write (a CTA-wide hash); without overlap they run in
// parallel, otherwise the memory phase is replayed in tid order (a warp at a
// time, lane by lane), which is exactly the reference's sequential order.
// Cross-block ordering of global accesses inside one sweep is NOT reproduced
// (blocks run independently); it only matters for programs with cross-block
// global races, the extension of SURVEY Appendix E.
//
// Race detection (racecheck.cpp:9-73) is online: a 32-bit shadow word per
// shared byte holds {one accessor tid, multi flag, one writer tid, multi
// flag, epoch stamp}; X races iff (X writes and some OTHER thread accessed
// the byte in this epoch) or (X reads and some other thread wrote it).
// Triples (obj, byte, line) are deduplicated per block and appended; the
// first racing timestamp per line is atomicMin'ed into a line table.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <tuple>
#include <vector>

#include "../host/engine.hpp"
#include "mckg.h"
#include "core.cuh"

namespace mckb {
namespace k1 {

using namespace mck_core;

// ---- per-thread capacity (local memory) ----
// (sized for recursion ~64 deep; local memory is reserved for the resident
// threads only, and only the used top of each array is touched)
#ifndef MCKG_K1_DEEP
#define MCKG_K1_DEEP 1
#endif
constexpr int VS = MCKG_K1_DEEP ? 160 : 48;       // value stack entries
constexpr int SCOPES = MCKG_K1_DEEP ? 160 : 32;
constexpr int OWNED = MCKG_K1_DEEP ? 160 : 48;
constexpr int FRAMES = MCKG_K1_DEEP ? 80 : 16;
constexpr int BINDS = MCKG_K1_DEEP ? 320 : 96;
constexpr int POBJ = MCKG_K1_DEEP ? 160 : 48;
constexpr int PB = MCKG_K1_DEEP ? 2560 : 768;     // private bytes (locals and params of all frames)
constexpr int TEP = TRACE_EPISODES;

constexpr uint32_t PRIV = 0x80000000u;
constexpr uint32_t NONE_TID = 0x7FFu;
constexpr int LINES = 65536;
constexpr int RACE_SET = 1024;  // per-block (byte, line) dedup entries

enum : int { ERR_NONE = 0, ERR_STACK, ERR_PRIV, ERR_SHARED_PTR_ESCAPE, ERR_DIAG_FULL, ERR_TRIPLES_FULL,
             ERR_LINE, ERR_SWEEPS, ERR_OPCODE, ERR_GLOG_FULL };

struct PObj {
  uint16_t off, size, gen;
  uint8_t live, pad;
  int32_t name;
};

struct Frame {
  int32_t retPc, bindBase, fn;
  uint8_t scopeDepth, valueDepth, pad0, pad1;
};

struct TS {
  int pc;
  int nv, nscope, nowned, nframe, npobj, ptop;
  int bb, fn;  // bind base and function of the current frame (cached)
  uint32_t steps, allocs;
  Val vals[VS];
  uint8_t scopeMark[SCOPES];
  uint8_t owned[OWNED];
  Frame frames[FRAMES];
  uint32_t binds[BINDS];
  PObj pobj[POBJ];
  alignas(8) uint8_t pbytes[PB];
  alignas(8) uint8_t pmeta[PB];
};

struct DevDiagRec {
  unsigned long long hkey;  // tuple hash (0 = empty)
  unsigned long long ts;    // min timestamp key
  int32_t code, line, name, pad;
  long long p[4];
};

struct BlockOut {
  unsigned long long sweeps, soloSweeps, cycles, soloCycles;
  unsigned long long steps;
  unsigned long long rules;
  unsigned long long allocs;
  unsigned long long sharedEvents;
  uint32_t lastSweep;
  uint32_t deadlocked;
  uint32_t episodes;  // completed barrier episodes
  uint32_t pad;
};

struct KP {
  const mck_ins* code;
  const mck_fn* fns;
  const mck_local* locals;
  int kernel;
  int nargs;
  const Val* args;
  uint32_t gid, sharedBase, nextId;
  int64_t gridDim, blockDim, shmem;
  int sharedName;
  int64_t warpSize;
  const uint32_t* objIds;     // sorted
  const DevObjInfo* objs;
  int nobjs;
  const uint32_t* globalIds;
  const uint32_t* shRanges;   // (first, count, gid) triples
  int nranges;
  uint8_t* gbytes;
  uint8_t* gmeta;
  int raceCheck;
  int htBits;                 // conflict hash size = 1 << htBits
  uint32_t bidBase;           // first simulated block of this launch (multi-device split)
  uint32_t* tarr;             // trace mode: [block][episode < TEP][tid] arrival sweep + 1
  int markDirty;              // record global writes in META_DIRTY (replicated memory)
  uint32_t maxSweeps;         // < 2^26; each sweep takes >= 1 step (step limit)
  // serial tails: a block whose last unfinished thread runs alone is
  // suspended into a slot and finished by tail_kernel, 32 tails per warp
  struct TailState* tails;    // [tailCap]
  uint8_t* tailSmem;          // [tailCap][tailStride]: bytes, meta, shadow, race set
  uint32_t* tailCount;        // slots taken
  uint32_t* tailBlk;          // [tailCap] the block (launch index) of each slot
  uint32_t tailCap, tailStride;
  // RunOptions::globalRaceCheck: every global access appended here (K6 input)
  mckg_gaccess* glog;
  // per log record (writes only): old bytes, old meta, new bytes, pointer
  // flag -- the grid's write history for mid-flight copies (probe mode)
  uint4* glogv;   // 2 x uint4 per record
  unsigned long long* nglog;
  unsigned long long glogCap;
  int glogStrict;  // a full log is an engine error (globalRaceCheck); else the probe gives up
  // outputs
  unsigned long long* lineFirst;
  int32_t* triples;           // (obj, byte, line) records of 3 x int32
  unsigned long long tripleCap;
  unsigned long long* nTriples;
  DevDiagRec* diags;
  uint32_t diagMask;          // table size - 1
  BlockOut* blocks;
  uint32_t* waitMask;         // gridDim x words
  int* error;
  int* errorInfo;
};

// ---------------- shared-memory layout ----------------
struct SmemLay {
  uint32_t bytes, meta, shadow, htKey, htVal, raceSet, end;
};
__host__ __device__ inline SmemLay smemLayout(int64_t shmem, int raceCheck, int htBits) {
  SmemLay L;
  uint32_t S = (uint32_t)((shmem + 15) & ~15ll);
  uint32_t p = 0;
  L.bytes = p; p += S;
  L.meta = p; p += S;
  L.shadow = p; p += raceCheck ? 4 * S : 0;
  p = (p + 15) & ~15u;
  L.htKey = p; p += 8u << htBits;
  L.htVal = p; p += 4u << htBits;
  L.raceSet = p; p += raceCheck ? 8 * RACE_SET : 0;
  L.end = p;
  return L;
}

extern __shared__ __align__(16) uint8_t smem[];

struct BlockShared {
  int wait[2];      // threads waiting in the open episode (by parity)
  int nz[2];        // nonzero __syncthreads_* operands (by parity)
  int allc[2];      // (operand != 0 || plain) (by parity)
  int fin;          // finished threads
  int conflict;
  unsigned long long steps;
  unsigned long long allocs;
  unsigned long long sharedEvents;
  uint32_t lastSweep;
  uint32_t nextRun[2][32];  // per warp: first sweep a thread of it can step (~0u: none), by sweep parity
  uint32_t soloSweep;  // sweep reached by a solo warp
  int tailSlot;        // >= 0: the block was suspended into this tail slot
};

__device__ __forceinline__ void set_error(const KP& P, int code, int info) {
  if (atomicCAS(P.error, 0, code) == 0) *P.errorInfo = info;
}

// ---------------- diagnostics ----------------
__device__ __forceinline__ unsigned long long mix64(unsigned long long x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33;
  x *= 0xc4ceb9fe1a85ec53ull;
  x ^= x >> 33;
  return x;
}

__host__ __device__ __forceinline__ unsigned long long tskey(uint32_t sweep, uint32_t bid, uint32_t tid, uint32_t sub) {
  return ((unsigned long long)sweep << 38) | ((unsigned long long)(bid & 0x3FFFFFFu) << 12) |
         ((unsigned long long)(tid & 1023u) << 2) | (sub & 3u);
}

struct Ctx {  // per-thread context of the current step
  uint32_t sweep, bid, tid, sub;
};

__device__ void emit_diag(const KP& P, Ctx& c, int code, int line, long long p0 = 0, long long p1 = 0,
                          long long p2 = 0, long long p3 = 0, int name = -1) {
  unsigned long long ts = tskey(c.sweep, c.bid, c.tid, c.sub);
  c.sub = c.sub < 3 ? c.sub + 1 : 3;
  unsigned long long h = mix64((unsigned long long)code * 0x9E3779B97F4A7C15ull ^ (unsigned long long)line);
  h = mix64(h ^ (unsigned long long)p0);
  h = mix64(h ^ (unsigned long long)p1);
  h = mix64(h ^ (unsigned long long)p2);
  h = mix64(h ^ (unsigned long long)p3);
  h = mix64(h ^ (unsigned long long)(unsigned)name);
  if (code == MCK_D_MEMBOUNDARY) h = mix64(h ^ (((unsigned long long)c.bid << 16) | c.tid));
  if (h == 0) h = 1;
  uint32_t slot = (uint32_t)h & P.diagMask;
  for (uint32_t probe = 0; probe <= P.diagMask; ++probe) {
    DevDiagRec* r = P.diags + slot;
    unsigned long long old = atomicCAS(&r->hkey, 0ull, h);
    if (old == 0ull) {
      r->code = code;
      r->line = line;
      r->name = name;
      r->p[0] = p0;
      r->p[1] = p1;
      r->p[2] = p2;
      r->p[3] = p3;
      atomicMin(&r->ts, ts);
      return;
    }
    if (old == h) {
      atomicMin(&r->ts, ts);
      return;
    }
    slot = (slot + 1) & P.diagMask;
  }
  set_error(P, ERR_DIAG_FULL, 0);
}

__device__ __forceinline__ void emit_ops(const KP& P, Ctx& c, const Diags& d, int line) {
  for (int i = 0; i < d.n; ++i) emit_diag(P, c, d.code[i], line);
}

// ---------------- private objects ----------------
__device__ __forceinline__ uint32_t priv_id(int idx, uint16_t gen) {
  return PRIV | ((uint32_t)(gen & 0x7FF) << 20) | (uint32_t)idx;
}

__device__ bool priv_alloc(TS& t, const KP& P, int size, int name, uint32_t& id) {
  const int base = (t.ptop + 7) & ~7;  // 8-byte aligned objects: word-wide scalar access
  if (t.npobj >= POBJ || base + size > PB || size < 0 || t.nowned >= OWNED) {
    set_error(P, ERR_PRIV, size);
    return false;
  }
  int idx = t.npobj++;
  PObj& o = t.pobj[idx];
  o.gen = (uint16_t)(o.gen + 1);
  o.off = (uint16_t)base;
  o.size = (uint16_t)size;
  o.live = 1;
  o.name = name;
  // fresh objects read as zero bytes, undefined (MemObject::bytes.resize, memory.cpp:30)
  for (int i = 0; i < size; i += 8) {
    *reinterpret_cast<uint64_t*>(t.pmeta + base + i) = 0ull;
    *reinterpret_cast<uint64_t*>(t.pbytes + base + i) = 0ull;
  }
  t.ptop = base + size;
  t.owned[t.nowned++] = (uint8_t)idx;
  ++t.allocs;
  id = priv_id(idx, o.gen);
  return true;
}

// scopes die LIFO: release private storage back to the first owned object
__device__ void pop_scopes(TS& t, int depth) {
  while (t.nscope > depth) {
    int m = t.scopeMark[--t.nscope];
    for (int i = m; i < t.nowned; ++i) t.pobj[t.owned[i]].live = 0;
    if (m < t.nowned) {
      int first = t.owned[m];
      t.ptop = t.pobj[first].off;
      t.npobj = first;
    }
    t.nowned = m;
  }
}

// private scalar poke (memory.cpp:184-206)
__device__ void priv_poke(TS& t, const PObj& o, int64_t off, uint8_t ty, const Val& v) {
  int len = (int)t_scalar(ty);
  int base = o.off;
  const int a = base + (int)off;
  if ((len == 4 && (a & 3) == 0) || (len == 8 && (a & 7) == 0)) {
    // aligned scalar: word-wide; pointer slots near it are cleared only if present
    const int lo = base + (off - 7 < 0 ? 0 : (int)off - 7), hi = base + (off + len < o.size ? (int)off + len : o.size);
    uint64_t any = 0;
    for (int wb = lo & ~7; wb < hi; wb += 8) {
      const uint64_t w = *reinterpret_cast<const uint64_t*>(t.pmeta + wb);
      const int s0 = lo - wb > 0 ? lo - wb : 0, s1 = hi - wb < 8 ? hi - wb : 8;
      const uint64_t msk = (s1 >= 8 ? ~0ull : ((1ull << (8 * s1)) - 1)) & ~((1ull << (8 * s0)) - 1);
      any |= w & msk & 0x0202020202020202ull;
    }
    if (any)
      for (int64_t s = off - 7 < 0 ? 0 : off - 7; s < off + len && s < o.size; ++s)
        t.pmeta[base + s] &= (uint8_t)~META_PTR;
    const uint64_t raw = encode_scalar(v, ty);
    const bool ptr = v.kind == MCK_K_PTR && v.obj != 0;
    if (len == 4) {
      *reinterpret_cast<uint32_t*>(t.pbytes + a) = (uint32_t)raw;
      *reinterpret_cast<uint32_t*>(t.pmeta + a) |= 0x01010101u * META_DEF;
    } else {
      *reinterpret_cast<uint64_t*>(t.pbytes + a) = raw;
      *reinterpret_cast<uint64_t*>(t.pmeta + a) |= 0x0101010101010101ull * META_DEF | (ptr ? (uint64_t)META_PTR : 0ull);
    }
    return;
  }
  for (int64_t s = off - 7 < 0 ? 0 : off - 7; s < off + len && s < o.size; ++s)
    if (s + 8 > off) t.pmeta[base + s] &= (uint8_t)~META_PTR;
  uint64_t raw = encode_scalar(v, ty);
  for (int i = 0; i < len; ++i) {
    t.pbytes[base + off + i] = (uint8_t)(raw >> (8 * i));
    t.pmeta[base + off + i] |= META_DEF;
  }
  if (v.kind == MCK_K_PTR && v.obj != 0) t.pmeta[base + off] |= META_PTR;
}

// ---------------- object resolution ----------------
enum : int { R_OK_PRIV, R_OK_SHARED, R_OK_GLOBAL, R_NULL, R_BOUNDARY, R_DEAD, R_OOB };

struct Res {
  int kind;
  int space;       // for R_BOUNDARY: 0 host, 2 shared
  long long target;
  int name;
  int64_t size;
  uint64_t base;   // byte offset (shared: in smem block; global: in arena; private: pbytes)
};

__device__ Res resolve(TS& t, const KP& P, uint32_t bid, uint32_t obj, int64_t off, int len) {
  Res r;
  r.name = -1;
  r.size = 0;
  r.base = 0;
  r.space = 0;
  r.target = 0;
  if (obj == 0) {
    r.kind = R_NULL;
    return r;
  }
  if (obj & PRIV) {
    int idx = (int)(obj & 0xFFFFF);
    uint16_t gen = (uint16_t)((obj >> 20) & 0x7FF);
    if (idx >= POBJ) {
      r.kind = R_NULL;
      return r;
    }
    const PObj& o = t.pobj[idx];
    r.name = o.name;
    r.size = o.size;
    r.base = o.off;
    if (idx >= t.npobj || !o.live || (o.gen & 0x7FF) != gen) {
      r.kind = R_DEAD;
      return r;
    }
    r.kind = (off < 0 || off + len > o.size) ? R_OOB : R_OK_PRIV;
    return r;
  }
  if (obj >= P.sharedBase && (int64_t)(obj - P.sharedBase) < P.gridDim) {
    uint32_t b = obj - P.sharedBase;
    if (b != bid) {
      r.kind = R_BOUNDARY;
      r.space = 2;
      r.target = ((long long)P.gid << 32) | b;
      return r;
    }
    r.name = P.sharedName;
    r.size = P.shmem;
    r.kind = (off < 0 || off + len > P.shmem) ? R_OOB : R_OK_SHARED;
    return r;
  }
  // device-global table (ascending ids)
  int lo = 0, hi = P.nobjs;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (P.objIds[mid] < obj) lo = mid + 1; else hi = mid;
  }
  if (lo < P.nobjs && P.objIds[lo] == obj) {
    const DevObjInfo& o = P.objs[lo];
    r.name = o.name;
    r.size = o.size;
    r.base = o.base;
    if (!o.live) {
      r.kind = R_DEAD;
      return r;
    }
    r.kind = (off < 0 || off + len > o.size) ? R_OOB : R_OK_GLOBAL;
    return r;
  }
  for (int i = 0; i < P.nranges; ++i) {
    uint32_t f = P.shRanges[3 * i], n = P.shRanges[3 * i + 1];
    if (obj >= f && obj - f < n) {
      r.kind = R_BOUNDARY;
      r.space = 2;
      r.target = ((long long)P.shRanges[3 * i + 2] << 32) | (obj - f);
      return r;
    }
  }
  if (obj < P.sharedBase) {  // a host object
    r.kind = R_BOUNDARY;
    r.space = 0;
    return r;
  }
  r.kind = R_NULL;
  return r;
}

// ---------------- raw memory (shared / global) ----------------
__device__ __forceinline__ uint64_t load_raw(const uint8_t* b, int len, bool& undef, const uint8_t* m,
                                             bool& ptrStart) {
  uint64_t raw = 0;
  undef = false;
  for (int i = 0; i < len; ++i) {
    raw |= (uint64_t)b[i] << (8 * i);
    if (!(m[i] & META_DEF)) undef = true;
  }
  ptrStart = (m[0] & META_PTR) != 0;
  return raw;
}

// meta update with word atomics (neighbouring bytes may be written by other
// threads in the same sweep)
__device__ __forceinline__ void meta_and(uint8_t* m, int64_t i, uint8_t mask) {
  uintptr_t a = (uintptr_t)(m + i);
  uint32_t* w = (uint32_t*)(a & ~(uintptr_t)3);
  uint32_t sh = (uint32_t)(a & 3) * 8;
  atomicAnd(w, ~((uint32_t)(uint8_t)~mask << sh));
}
__device__ __forceinline__ void meta_or(uint8_t* m, int64_t i, uint8_t bits) {
  uintptr_t a = (uintptr_t)(m + i);
  uint32_t* w = (uint32_t*)(a & ~(uintptr_t)3);
  uint32_t sh = (uint32_t)(a & 3) * 8;
  atomicOr(w, (uint32_t)bits << sh);
}

__device__ void store_raw(uint8_t* b, uint8_t* m, int64_t objSize, int64_t off, int len, uint64_t raw,
                          bool ptr) {
  // erase pointer slots overlapping [off, off + len) (memory.cpp:89-97)
  for (int64_t s = off - 7 < 0 ? 0 : off - 7; s < off + len && s < objSize; ++s)
    if (s + 8 > off && (m[s] & META_PTR)) meta_and(m, s, (uint8_t)~META_PTR);
  for (int i = 0; i < len; ++i) b[off + i] = (uint8_t)(raw >> (8 * i));
  for (int i = 0; i < len; ++i)
    if ((m[off + i] & META_DEF) == 0) meta_or(m, off + i, META_DEF);
  if (ptr) meta_or(m, off, META_PTR);
}

// ---------------- race shadow (shared memory) ----------------
__device__ __forceinline__ uint32_t shadow_empty(uint32_t stamp) {
  return NONE_TID | (NONE_TID << 12) | (stamp << 24);
}
__device__ __forceinline__ bool other_than(uint32_t tidf, uint32_t multi, uint32_t x) {
  return (tidf != NONE_TID && tidf != x) || multi;
}

struct RaceOut {
  uint32_t bytes;  // bit q: byte off+q raced
};

// Records one access in the shadow; returns the raced byte mask.
__device__ uint32_t shadow_access(uint32_t* sh, int64_t off, int len, uint32_t x, bool w, uint32_t stamp) {
  uint32_t raced = 0;
  for (int q = 0; q < len; ++q) {
    uint32_t* p = sh + off + q;
    uint32_t cur = *p;
    while (true) {
      uint32_t s = (cur >> 24) == stamp ? cur : shadow_empty(stamp);
      uint32_t at = s & 0x7FF, am = (s >> 11) & 1, wt = (s >> 12) & 0x7FF, wm = (s >> 23) & 1;
      bool r = w ? other_than(at, am, x) : other_than(wt, wm, x);
      uint32_t nat = at, nam = am, nwt = wt, nwm = wm;
      if (nat == NONE_TID) nat = x; else if (nat != x) nam = 1;
      if (w) {
        if (nwt == NONE_TID) nwt = x; else if (nwt != x) nwm = 1;
      }
      uint32_t ns = nat | (nam << 11) | (nwt << 12) | (nwm << 23) | (stamp << 24);
      if (ns == cur) {
        if (r) raced |= 1u << q;
        break;
      }
      uint32_t old = atomicCAS(p, cur, ns);
      if (old == cur) {
        if (r) raced |= 1u << q;
        break;
      }
      cur = old;
    }
  }
  return raced;
}

__device__ void report_race(const KP& P, Ctx& c, unsigned long long* set, uint32_t obj, int64_t off,
                            uint32_t raced, int line, uint32_t bstamp) {
  if (!raced) return;
  if (line < 0 || line >= LINES) {
    set_error(P, ERR_LINE, line);
    return;
  }
  unsigned long long ts = tskey(c.sweep, c.bid, c.tid, c.sub);
  atomicMin(P.lineFirst + line, ts);
  for (int q = 0; q < 8; ++q) {
    if (!((raced >> q) & 1u)) continue;
    unsigned long long key = ((unsigned long long)(bstamp & 0xFFFF) << 48) |
                             ((unsigned long long)((off + q) & 0xFFFFFFFF) << 16) | (uint32_t)line;
    key |= 1ull << 63;
    uint32_t h = (uint32_t)(mix64(key) & (RACE_SET - 1));
    bool fresh = true;
    for (int probe = 0; probe < RACE_SET; ++probe) {
      unsigned long long curk = set[h];
      if (curk == key) {
        fresh = false;
        break;
      }
      if (curk == 0) {
        unsigned long long old = atomicCAS(set + h, 0ull, key);
        if (old == 0ull) break;
        if (old == key) {
          fresh = false;
          break;
        }
      }
      h = (h + 1) & (RACE_SET - 1);
    }
    // (a full set appends duplicates; the host dedups the triples)
    if (fresh) {
      unsigned long long i = atomicAdd(P.nTriples, 1ull);
      if (i < P.tripleCap) {
        P.triples[3 * i] = (int32_t)obj;
        P.triples[3 * i + 1] = (int32_t)(off + q);
        P.triples[3 * i + 2] = line;
      } else {
        set_error(P, ERR_TRIPLES_FULL, 0);
      }
    }
  }
  c.sub = c.sub < 3 ? c.sub + 1 : 3;
}

// ---------------- the memory request of one step ----------------
struct Req {
  int kind;     // 0 none, 1 read, 2 write
  int space;    // R_OK_SHARED / R_OK_GLOBAL
  uint8_t ty;
  uint32_t obj;
  int64_t off;
  uint64_t base;
  int64_t size;
  int name;
  uint64_t raw;
  bool ptr;
  int line;
  // results
  bool ok;
  Val val;
};

__device__ __forceinline__ int push(TS& t, const KP& P, const Val& v) {
  if (t.nv >= VS) {
    set_error(P, ERR_STACK, 0);
    return 0;
  }
  t.vals[t.nv++] = v;
  return 1;
}
__device__ __forceinline__ Val pop(TS& t) { return t.vals[--t.nv]; }

// thread states
enum : int { S_READY = 0, S_WAIT = 1, S_FIN = 2 };

struct Thread {
  int state;
  uint32_t readyAt;
  int syncKind;
  long long operand;
  uint32_t E;  // completed episodes (the race epoch)
};

// A suspended block's last thread and the block's counters (tail_kernel).
struct TailState {
  TS t;
  Thread th;
  BlockShared bs;  // step()'s barrier counters
  uint32_t sweep, E, lastStep, tid;
};

// The layout of a suspended block's shared state in global memory.
__host__ __device__ inline SmemLay tailLayout(int64_t shmem, int raceCheck) {
  SmemLay L;
  const uint32_t S = (uint32_t)((shmem + 15) & ~15ll);
  L.bytes = 0;
  L.meta = S;
  L.shadow = 2 * S;
  L.raceSet = (raceCheck ? 6 * S : 2 * S);
  L.htKey = L.htVal = 0;
  L.end = L.raceSet + (raceCheck ? 8 * RACE_SET : 0);
  L.end = (L.end + 15) & ~15u;
  return L;
}

__device__ __forceinline__ const mck_local& local_of(const KP& P, int fn, int slot) {
  return P.locals[P.fns[fn].local_base + slot];
}

__device__ bool enter_fn(TS& t, const KP& P, int fn, int retPc) {
  if (t.nframe >= FRAMES || t.nscope >= SCOPES) {
    set_error(P, ERR_STACK, 1);
    return false;
  }
  Frame f;
  f.retPc = retPc;
  f.bindBase = t.nframe == 0 ? 0 : t.frames[t.nframe - 1].bindBase + P.fns[t.frames[t.nframe - 1].fn].n_slots;
  f.fn = fn;
  f.scopeDepth = (uint8_t)t.nscope;
  f.valueDepth = (uint8_t)t.nv;
  if (f.bindBase + P.fns[fn].n_slots > BINDS) {
    set_error(P, ERR_STACK, 2);
    return false;
  }
  t.frames[t.nframe++] = f;
  t.scopeMark[t.nscope++] = (uint8_t)t.nowned;
  t.bb = f.bindBase;
  t.fn = fn;
  return true;
}

// Leaves the current function; returns false when the thread is finished.
__device__ bool leave_fn(TS& t, const KP& P, Ctx& c, const Val* v, int line, bool conv, Thread& th) {
  Frame f = t.frames[t.nframe - 1];
  pop_scopes(t, f.scopeDepth);
  t.nv = f.valueDepth;
  --t.nframe;
  uint8_t ret = P.fns[f.fn].ret;
  Val out;
  if (conv) {
    Diags d{};
    bool ok = convert(*v, ret, out, d);
    emit_ops(P, c, d, line);
    if (!ok) {
      th.state = S_FIN;
      return false;
    }
  } else {
    out = t_is_void(ret) ? v_void() : v_int(0, ret);
  }
  if (t.nframe == 0) {
    th.state = S_FIN;
    return false;
  }
  push(t, P, out);
  t.pc = f.retPc;
  t.bb = t.frames[t.nframe - 1].bindBase;
  t.fn = t.frames[t.nframe - 1].fn;
  return true;
}

// Read / write through a resolved object for NON-private targets: fills the
// request, the memory phase performs it.  For private targets performs it now.
// Returns: 0 = done (value pushed / halted), 1 = request pending.
__device__ int mem_read(TS& t, const KP& P, Ctx& c, Thread& th, uint32_t obj, int64_t off, uint8_t ty, int line,
                        Req& rq) {
  int len = (int)t_scalar(ty);
  Res r = resolve(t, P, c.bid, obj, off, len);
  switch (r.kind) {
    case R_NULL: emit_diag(P, c, MCK_D_NULL_RW, line, 0); th.state = S_FIN; return 0;
    case R_BOUNDARY: emit_diag(P, c, MCK_D_MEMBOUNDARY, line, 0, r.space, r.target); th.state = S_FIN; return 0;
    case R_DEAD: emit_diag(P, c, MCK_D_DEAD, line, 0, 0, 0, 0, r.name); th.state = S_FIN; return 0;
    case R_OOB: emit_diag(P, c, MCK_D_OOB, line, 0, len, off, r.size, r.name); th.state = S_FIN; return 0;
    default: break;
  }
  if (r.kind == R_OK_PRIV) {
    bool undef, ps;
    uint64_t raw;
    const int64_t a = (int64_t)r.base + off;
    if (len == 4 && (a & 3) == 0) {
      raw = *reinterpret_cast<const uint32_t*>(t.pbytes + a);
      const uint32_t m = *reinterpret_cast<const uint32_t*>(t.pmeta + a);
      undef = (m & 0x01010101u) != 0x01010101u;
      ps = (m & META_PTR) != 0;
    } else if (len == 8 && (a & 7) == 0) {
      raw = *reinterpret_cast<const uint64_t*>(t.pbytes + a);
      const uint64_t m = *reinterpret_cast<const uint64_t*>(t.pmeta + a);
      undef = (m & 0x0101010101010101ull) != 0x0101010101010101ull;
      ps = (m & META_PTR) != 0;
    } else {
      raw = load_raw(t.pbytes + a, len, undef, t.pmeta + a, ps);
    }
    rq.kind = 0;
    rq.ok = true;
    if (MCK_T_PTR(ty) > 0) {
      if (ps) { rq.val = v_ptr((uint32_t)(raw >> 32), (int32_t)(raw & 0xffffffffu), ty); return 0; }
      if (undef) { emit_diag(P, c, MCK_D_UNINIT_PTR, line, 0, 0, 0, 0, r.name); th.state = S_FIN; rq.ok = false; return 0; }
      if (raw == 0) { rq.val = v_ptr(0, 0, ty); return 0; }
      emit_diag(P, c, MCK_D_NONPTR_AS_PTR, line);
      th.state = S_FIN;
      rq.ok = false;
      return 0;
    }
    if (undef) emit_diag(P, c, MCK_D_UNINIT, line, 0, 0, 0, 0, r.name);
    rq.val = decode_scalar(raw, ty);
    return 0;
  }
  rq.kind = 1;
  rq.space = r.kind;
  rq.ty = ty;
  rq.obj = obj;
  rq.off = off;
  rq.base = r.base;
  rq.size = r.size;
  rq.name = r.name;
  rq.line = line;
  return 1;
}

__device__ int mem_write(TS& t, const KP& P, Ctx& c, Thread& th, uint32_t obj, int64_t off, uint8_t ty,
                         const Val& v, int line, Req& rq) {
  int len = (int)t_scalar(ty);
  Res r = resolve(t, P, c.bid, obj, off, len);
  switch (r.kind) {
    case R_NULL: emit_diag(P, c, MCK_D_NULL_RW, line, 1); th.state = S_FIN; return 0;
    case R_BOUNDARY: emit_diag(P, c, MCK_D_MEMBOUNDARY, line, 1, r.space, r.target); th.state = S_FIN; return 0;
    case R_DEAD: emit_diag(P, c, MCK_D_DEAD, line, 1, 0, 0, 0, r.name); th.state = S_FIN; return 0;
    case R_OOB: emit_diag(P, c, MCK_D_OOB, line, 1, len, off, r.size, r.name); th.state = S_FIN; return 0;
    default: break;
  }
  if (r.kind == R_OK_PRIV) {
    priv_poke(t, t.pobj[obj & 0xFFFFF], off, ty, v);
    rq.kind = 0;
    rq.ok = true;
    return 0;
  }
  if (v.kind == MCK_K_PTR && (v.obj & PRIV)) {
    // a private pointer escaping to memory other threads can read: the
    // engine's virtual ids are thread-relative (documented limitation)
    set_error(P, ERR_SHARED_PTR_ESCAPE, line);
    th.state = S_FIN;
    return 0;
  }
  rq.kind = 2;
  rq.space = r.kind;
  rq.ty = ty;
  rq.obj = obj;
  rq.off = off;
  rq.base = r.base;
  rq.size = r.size;
  rq.name = r.name;
  rq.line = line;
  rq.raw = encode_scalar(v, ty);
  rq.ptr = v.kind == MCK_K_PTR && v.obj != 0;
  rq.val = v;
  return 1;
}

// Probe mode: the write history record i -- what this write overwrites
// (bytes, meta), the new bytes, and 'complex' when a pointer slot is stored
// or erased.
__device__ __noinline__ void log_overwrite(const KP& P, unsigned long long i, const Req& rq, const uint8_t* b,
                                           const uint8_t* m, int len) {
  uint32_t ob[2] = {0, 0}, om[2] = {0, 0}, cx = rq.ptr ? 1u : 0u;
  for (int k = 0; k < len; ++k) {
    ob[k >> 2] |= (uint32_t)b[k] << (8 * (k & 3));
    om[k >> 2] |= (uint32_t)m[k] << (8 * (k & 3));
    cx |= (m[k] & META_PTR) ? 1u : 0u;
  }
  for (int64_t k = rq.off - 7 < 0 ? 0 : rq.off - 7; k < rq.off; ++k) cx |= (m[k - rq.off] & META_PTR) ? 1u : 0u;
  P.glogv[2 * i] = make_uint4(ob[0], ob[1], om[0], om[1]);
  P.glogv[2 * i + 1] = make_uint4((uint32_t)rq.raw, (uint32_t)(rq.raw >> 32), cx, 0u);
}

// Performs a pending shared/global request (memory phase).
// HIST: the grid keeps a write history (KP::glogv).  A compile-time switch:
// the history path, even never taken, costs the interpreter ~5% of its step
// rate through register pressure (C2 42.8 -> 45.0 ms measured), so only
// probed grids run the kernel instance that has it.
// sb: the base of the block's shared state laid out by L (the CTA's shared
// memory, or a suspended block's copy in global memory)
template <bool HIST>
__device__ __noinline__ void do_request(const KP& P, Ctx& c, Thread& th, Req& rq, const SmemLay& L, uint32_t stamp,
                                        uint32_t bstamp, unsigned long long& sharedEvents, uint8_t* sb) {
  int len = (int)t_scalar(rq.ty);
  uint8_t *b, *m;
  if (rq.space == R_OK_SHARED) {
    b = sb + L.bytes + rq.off;
    m = sb + L.meta + rq.off;
    if (P.raceCheck) {
      ++sharedEvents;
      uint32_t raced = shadow_access((uint32_t*)(sb + L.shadow), rq.off, len, c.tid, rq.kind == 2, stamp);
      report_race(P, c, (unsigned long long*)(sb + L.raceSet), rq.obj, rq.off, raced, rq.line, bstamp);
    }
  } else {
    b = P.gbytes + rq.base + rq.off;
    m = P.gmeta + rq.base + rq.off;
    if (P.glog) {  // the global-race log: one 16-byte record per access
      const unsigned long long i = atomicAdd(P.nglog, 1ull);
      if (HIST && i < P.glogCap && rq.kind == 2 && P.glogv) log_overwrite(P, i, rq, b, m, len);
      if (i < P.glogCap) {
        mckg_gaccess g;
        const uint64_t addr = rq.base + (uint64_t)rq.off;
        const uint32_t ln = (uint32_t)rq.line;
        g.a = (addr & 0xFFFFFFFFFFull) | ((unsigned long long)(len & 0xF) << 40) |
              ((unsigned long long)(rq.kind == 2 ? 1u : 0u) << 44) | ((unsigned long long)(c.tid & 0x7FFu) << 45) |
              ((unsigned long long)(ln & 0xFFu) << 56);
        g.sweep = c.sweep;
        g.b = (c.bid & 0xFFFFFFu) | (((ln >> 8) & 0xFFu) << 24);
        P.glog[i] = g;
      } else if (P.glogStrict) {
        set_error(P, ERR_GLOG_FULL, 0);
      }
    }
  }
  if (rq.kind == 2) {
    if (rq.space == R_OK_SHARED)
      store_raw(sb + L.bytes, sb + L.meta, rq.size, rq.off, len, rq.raw, rq.ptr);
    else {
      store_raw(P.gbytes + rq.base, P.gmeta + rq.base, rq.size, rq.off, len, rq.raw, rq.ptr);
      if (P.markDirty)
        for (int i = 0; i < len; ++i) meta_or(P.gmeta + rq.base, rq.off + i, META_DIRTY);
    }
    rq.ok = true;
    return;
  }
  bool undef, ps;
  uint64_t raw = load_raw(b, len, undef, m, ps);
  rq.ok = true;
  if (MCK_T_PTR(rq.ty) > 0) {
    if (ps) { rq.val = v_ptr((uint32_t)(raw >> 32), (int32_t)(raw & 0xffffffffu), rq.ty); return; }
    if (undef) { emit_diag(P, c, MCK_D_UNINIT_PTR, rq.line, 0, 0, 0, 0, rq.name); th.state = S_FIN; rq.ok = false; return; }
    if (raw == 0) { rq.val = v_ptr(0, 0, rq.ty); return; }
    emit_diag(P, c, MCK_D_NONPTR_AS_PTR, rq.line);
    th.state = S_FIN;
    rq.ok = false;
    return;
  }
  if (undef) emit_diag(P, c, MCK_D_UNINIT, rq.line, 0, 0, 0, 0, rq.name);
  rq.val = decode_scalar(raw, rq.ty);
}

// After-memory continuation of the instruction that issued a request.
// pendOp: the opcode; for LOADKEEP the LValue is kept in `lv`.
struct Pend {
  int op;
  Val lv;
  Val keep;  // STORE_INC postfix: the old value
  bool postfix;
};

__device__ void finish_request(TS& t, const KP& P, Thread& th, const Req& rq, const Pend& pd) {
  if (th.state == S_FIN || !rq.ok) return;
  switch (pd.op) {
    case OP_LOADRV: push(t, P, rq.val); break;
    case OP_LOADKEEP:
      push(t, P, pd.lv);
      push(t, P, rq.val);
      break;
    default:  // stores push the stored (or old) value
      push(t, P, pd.postfix ? pd.keep : rq.val);
      break;
  }
}

__device__ __forceinline__ mck_ins ldg_ins(const mck_ins* p) {
  const uint4 v = __ldg(reinterpret_cast<const uint4*>(p));
  mck_ins in;
  in.op = (uint8_t)(v.x & 0xFF);
  in.t = (uint8_t)((v.x >> 8) & 0xFF);
  in.f = (uint8_t)((v.x >> 16) & 0xFF);
  in.pad = 0;
  in.a = (int32_t)v.y;
  in.b = (int32_t)v.z;
  in.line = (int32_t)v.w;
  return in;
}

// (barrier.sync, not bar.sync: the parked warps and the solo warp meet at
// different instructions, and a warp need not be converged at its own)
__device__ __forceinline__ void bar_named(uint32_t id, uint32_t nthreads) {
  asm volatile("barrier.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// One small step of thread `t`.  Returns 1 when a shared/global request is
// pending (rq/pd filled), else 0.
__device__ __forceinline__ int step(TS& t, const KP& P, Ctx& c, Thread& th, Req& rq, Pend& pd, BlockShared& bs, uint32_t nthreads) {
  const mck_ins* code = P.code;
  mck_ins in = ldg_ins(code + t.pc);
  while (in.op == OP_JMP) {
    t.pc = in.a;
    in = ldg_ins(code + t.pc);
  }
  ++t.pc;
  ++t.steps;
  const int L = in.line;
  Diags d{};
  rq.kind = 0;
  switch (in.op) {
    case OP_NOP: break;
    case OP_SCOPE_PUSH:
      if (t.nscope >= SCOPES) { set_error(P, ERR_STACK, 3); th.state = S_FIN; break; }
      t.scopeMark[t.nscope++] = (uint8_t)t.nowned;
      break;
    case OP_SCOPE_POP: pop_scopes(t, t.nscope - 1); break;
    case OP_PUSH_INT:
      push(t, P, v_int((int64_t)(((uint64_t)(uint32_t)in.b << 32) | (uint32_t)in.a), in.t));
      break;
    case OP_PUSH_FLT:
      push(t, P, mk(MCK_K_FLOAT, in.t, 0, (int64_t)(((uint64_t)(uint32_t)in.b << 32) | (uint32_t)in.a)));
      break;
    case OP_PUSH_LOCAL: {
      uint32_t o = t.binds[t.bb + in.a];
      if (!o) {
        emit_diag(P, c, MCK_D_FIXED_UB, L, MCK_UB_UNBOUND, 0, 0, 0, in.b);
        th.state = S_FIN;
        break;
      }
      push(t, P, v_lv(o, 0, in.t));
      break;
    }
    case OP_PUSH_GLOBAL: push(t, P, v_lv(P.globalIds[in.a], 0, in.t)); break;
    case OP_PUSH_BUILTIN: {
      int64_t v = 0;
      switch (in.f) {
        case MCK_B_TID: v = in.a == 0 ? c.tid : 0; break;
        case MCK_B_BID: v = in.a == 0 ? c.bid : 0; break;
        case MCK_B_BDIM: v = in.a == 0 ? P.blockDim : 1; break;
        case MCK_B_GDIM: v = in.a == 0 ? P.gridDim : 1; break;
        default: v = P.warpSize; break;
      }
      push(t, P, v_int(v));
      break;
    }
    case OP_UB:
      emit_diag(P, c, MCK_D_FIXED_UB, L, in.a, 0, 0, 0, in.b);
      th.state = S_FIN;
      break;
    case OP_LOADRV: {
      Val lv = pop(t);
      if (MCK_T_ARR(lv.type)) {
        push(t, P, v_ptr(lv.obj, lv.i, t_decay(lv.type)));
        break;
      }
      pd.op = OP_LOADRV;
      pd.postfix = false;
      if (mem_read(t, P, c, th, lv.obj, lv.i, lv.type, L, rq)) return 1;
      if (th.state != S_FIN) push(t, P, rq.val);
      break;
    }
    case OP_LOADKEEP: {
      Val lv = pop(t);
      if (MCK_T_ARR(lv.type)) {
        emit_diag(P, c, MCK_D_MODIFY_ARRAY, L);
        th.state = S_FIN;
        break;
      }
      pd.op = OP_LOADKEEP;
      pd.lv = lv;
      pd.postfix = false;
      if (mem_read(t, P, c, th, lv.obj, lv.i, lv.type, L, rq)) return 1;
      if (th.state != S_FIN) {
        push(t, P, lv);
        push(t, P, rq.val);
      }
      break;
    }
    case OP_STORE:
    case OP_STORE_OP:
    case OP_STORE_INC: {
      Val lv, r, old{};
      bool ok;
      if (in.op == OP_STORE) {
        Val rhs = pop(t);
        lv = pop(t);
        ok = convert(rhs, lv.type, r, d);
      } else if (in.op == OP_STORE_OP) {
        Val rhs = pop(t);
        old = pop(t);
        lv = pop(t);
        Val x;
        ok = binop(in.f, old, rhs, x, d) && convert(x, lv.type, r, d);
      } else {
        old = pop(t);
        lv = pop(t);
        Val x;
        ok = binop(MCK_ADD, old, v_int(in.a), x, d) && convert(x, lv.type, r, d);
      }
      emit_ops(P, c, d, L);
      if (!ok) {
        th.state = S_FIN;
        break;
      }
      pd.op = in.op;
      pd.postfix = in.op == OP_STORE_INC && !in.f;
      pd.keep = old;
      if (mem_write(t, P, c, th, lv.obj, lv.i, lv.type, r, L, rq)) return 1;
      if (th.state != S_FIN) push(t, P, pd.postfix ? old : r);
      break;
    }
    case OP_ADDROF: {
      Val lv = pop(t);
      push(t, P, v_ptr(lv.obj, lv.i, t_addr(lv.type)));
      break;
    }
    case OP_DEREF: {
      Val v = pop(t);
      if (v.kind == MCK_K_INT && v.i == 0) v = v_ptr(0, 0, MCK_T_VOIDP);
      if (v.kind != MCK_K_PTR || MCK_T_PTR(v.type) == 0) {
        emit_diag(P, c, MCK_D_DEREF_NONPTR, L);
        th.state = S_FIN;
        break;
      }
      push(t, P, v_lv(v.obj, v.i, t_elem(v.type)));
      break;
    }
    case OP_INDEX: {
      Val idx = pop(t), base = pop(t);
      if (base.kind != MCK_K_PTR || idx.kind != MCK_K_INT) {
        emit_diag(P, c, MCK_D_SUBSCRIPT, L);
        th.state = S_FIN;
        break;
      }
      uint8_t e = t_elem(base.type);
      push(t, P, v_lv(base.obj, base.i + idx.i * t_scalar(e), e));
      break;
    }
    case OP_UNARY: {
      Val v = pop(t), r;
      bool ok = unop(in.f, v, r, d);
      emit_ops(P, c, d, L);
      if (!ok) { th.state = S_FIN; break; }
      push(t, P, r);
      break;
    }
    case OP_BINARY: {
      Val rr = pop(t), l = pop(t), r;
      bool ok = binop(in.f, l, rr, r, d);
      emit_ops(P, c, d, L);
      if (!ok) { th.state = S_FIN; break; }
      push(t, P, r);
      break;
    }
    case OP_LOGRHS: {
      Val l = pop(t);
      bool isAnd = in.f == 1;
      if (isAnd && !truthy(l)) {
        push(t, P, v_int(0));
        t.pc = in.a;
      } else if (!isAnd && truthy(l)) {
        push(t, P, v_int(1));
        t.pc = in.a;
      }
      break;
    }
    case OP_BOOLIFY: {
      Val v = pop(t);
      push(t, P, v_int(truthy(v) ? 1 : 0));
      break;
    }
    case OP_TERNSEL:
    case OP_IFJUDGE:
    case OP_WHILEJUDGE: {
      Val cv = pop(t);
      if (!truthy(cv)) t.pc = in.a;
      break;
    }
    case OP_CAST: {
      Val v = pop(t), r;
      if (MCK_T_PTR(in.t) > 0 && v.kind == MCK_K_PTR) {
        push(t, P, v_ptr(v.obj, v.i, in.t));
        break;
      }
      bool ok = convert(v, in.t, r, d);
      emit_ops(P, c, d, L);
      if (!ok) { th.state = S_FIN; break; }
      push(t, P, r);
      break;
    }
    case OP_FORJUDGE: {
      bool go = true;
      if (in.f) go = truthy(pop(t));
      if (!go) t.pc = in.a;
      break;
    }
    case OP_POPVALUE: --t.nv; break;
    case OP_RETURN: {
      Val v = in.f ? pop(t) : v_void();
      leave_fn(t, P, c, &v, L, true, th);
      break;
    }
    case OP_FALLOFF: leave_fn(t, P, c, nullptr, L, false, th); break;
    case OP_BREAK:
    case OP_CONTINUE:
      pop_scopes(t, t.nscope - in.b);
      t.pc = in.a;
      break;
    case OP_CALL: {
      const int n = in.b;
      if (t.nv < n) { set_error(P, ERR_STACK, 4); th.state = S_FIN; break; }
      t.nv -= n;
      const int argBase = t.nv;
      // args stay in vals[argBase .. argBase+n) until bound (the frame records nv)
      if (!enter_fn(t, P, in.a, t.pc)) { th.state = S_FIN; break; }
      const int bb = t.bb;
      for (int i = 0; i < n; ++i) {
        const mck_local& pl = local_of(P, in.a, i);
        Val cv;
        Diags dd{};
        bool ok = convert(t.vals[argBase + i], pl.type, cv, dd);
        emit_ops(P, c, dd, L);
        if (!ok) { th.state = S_FIN; break; }
        uint32_t id;
        if (!priv_alloc(t, P, pl.size, pl.name, id)) { th.state = S_FIN; break; }
        priv_poke(t, t.pobj[id & 0xFFFFF], 0, pl.type, cv);
        t.binds[bb + i] = id;
      }
      if (th.state != S_FIN) t.pc = P.fns[in.a].entry;
      break;
    }
    case OP_SYNC: {
      long long operand = 0;
      if (in.f != MCK_SYNC_PLAIN) {
        Val v = pop(t);
        operand = v.i;
      }
      th.state = S_WAIT;
      th.syncKind = in.f;
      th.operand = operand;
      if (P.tarr && th.E < TEP)  // --trace: arrival sweeps give the barrier-rule timeline
        P.tarr[((size_t)(c.bid - P.bidBase) * TEP + th.E) * (size_t)P.blockDim + c.tid] = c.sweep + 1;
      const int p = (th.E + 1) & 1;
      const bool nz = operand != 0;
      atomicAdd(&bs.wait[p], 1);
      if (nz) atomicAdd(&bs.nz[p], 1);
      if (nz || in.f == MCK_SYNC_PLAIN) atomicAdd(&bs.allc[p], 1);
      break;
    }
    case OP_DECL: {
      const int fn = t.fn;
      const int bb = t.bb;
      if (in.f) {  // extern __shared__: bind the block's array
        t.binds[bb + in.a] = P.sharedBase + c.bid;
        break;
      }
      const mck_local& l = local_of(P, fn, in.a);
      uint32_t id;
      if (!priv_alloc(t, P, l.size, l.name, id)) { th.state = S_FIN; break; }
      t.binds[bb + in.a] = id;
      break;
    }
    case OP_INITSTORE: {
      Val v = pop(t), r;
      bool ok = convert(v, in.t, r, d);
      emit_ops(P, c, d, L);
      if (!ok) { th.state = S_FIN; break; }
      const uint32_t o = t.binds[t.bb + in.a];
      pd.op = OP_INITSTORE;
      pd.postfix = false;
      if (mem_write(t, P, c, th, o, 0, in.t, r, L, rq)) {
        rq.kind = 0;  // declared objects are private: never pending
      }
      break;
    }
    default:
      set_error(P, ERR_OPCODE, in.op);
      th.state = S_FIN;
      break;
  }
  return 0;
}

// ---------------- conflict hash ----------------
// Open addressing over (word + 1) keys; every inserter clears its own slots
// after the check, so the table is empty again at the next sweep.
__device__ __forceinline__ int ht_insert(unsigned long long* keys, uint32_t* vals, int bits,
                                         unsigned long long key, uint32_t add) {
  uint32_t mask = (1u << bits) - 1;
  uint32_t h = (uint32_t)mix64(key) & mask;
  for (uint32_t probe = 0; probe <= mask; ++probe) {
    unsigned long long old = atomicCAS(keys + h, 0ull, key);
    if (old == 0ull || old == key) {
      atomicAdd(vals + h, add);
      return (int)h;
    }
    h = (h + 1) & mask;
  }
  return -1;
}


// Copies a block's shared state into its tail slot (threads g < nthr of the
// calling group take part) and the block's last READY thread's state.
// the sub-thread of GPU thread g that is READY (0 when none: suspend_block
// then stores nothing for it)
// A lone thread is suspended once it has run TAIL_MIN sweeps alone: short
// tails (C4's last arrivals) are cheaper finished in place than copied out.
constexpr uint32_t TAIL_MIN = 64;

template <int K>
__device__ __forceinline__ int ready_sub(const Thread* th, uint32_t g, uint32_t CT, uint32_t n) {
  int kk = 0;
#pragma unroll 1
  for (int k = 0; k < K; ++k)
    if ((uint32_t)k * CT + g < n && th[k].state == S_READY) kk = k;
  return kk;
}

// (t/th: this GPU thread's READY sub-thread, simulated tid `tid`, if any)
__device__ void suspend_block(const KP& P, BlockShared& bs, const SmemLay& L, const TS& t, const Thread& th,
                              uint32_t g, uint32_t tid, uint32_t nthr, uint32_t n, uint32_t sweep, uint32_t E,
                              uint32_t lastStep, uint32_t lb) {
  const int sl = *(volatile int*)&bs.tailSlot;
  TailState& TSs = P.tails[sl];
  uint8_t* dst = P.tailSmem + (size_t)sl * P.tailStride;
  const SmemLay TL = tailLayout(P.shmem, P.raceCheck);
  const uint32_t me = g % nthr;
  for (uint32_t i = me; i < (uint32_t)P.shmem; i += nthr) {
    dst[TL.bytes + i] = smem[L.bytes + i];
    dst[TL.meta + i] = smem[L.meta + i];
  }
  if (P.raceCheck) {
    const uint32_t* sh = (const uint32_t*)(smem + L.shadow);
    uint32_t* dsh = (uint32_t*)(dst + TL.shadow);
    for (uint32_t i = me; i < (uint32_t)P.shmem; i += nthr) dsh[i] = sh[i];
    const unsigned long long* rs = (const unsigned long long*)(smem + L.raceSet);
    unsigned long long* drs = (unsigned long long*)(dst + TL.raceSet);
    for (uint32_t i = me; i < RACE_SET; i += nthr) drs[i] = rs[i];
  }
  if (tid < n && th.state == S_READY) {
    TSs.t = t;
    TSs.th = th;
    TSs.sweep = sweep;
    TSs.E = E;
    TSs.lastStep = lastStep;
    TSs.tid = tid;
    P.tailBlk[sl] = lb;
  }
}

// ================= the kernel =================
// K simulated threads per GPU thread: simulated tid = k * CT + threadIdx.x
// (CT = blockDim.x, a multiple of 32).  Smaller CTAs let more simulated
// blocks stay resident, which is what long serial stretches (one live thread
// per block) need; inside a sweep the K sub-threads step in tid order.
template <int K, bool HIST>
#ifndef MCKG_K1_MINB
#define MCKG_K1_MINB 4  // K = 1 serves blocks of <= 256 threads
#endif
__global__ void __launch_bounds__(256, K == 1 ? MCKG_K1_MINB : 4) grid_kernel(KP P) {
  const uint32_t bid = blockIdx.x + P.bidBase;  // simulated block
  const uint32_t lb = blockIdx.x;               // index into this launch's outputs
  const uint32_t g = threadIdx.x;
  const uint32_t CT = blockDim.x;
  const uint32_t SLOTS = CT * K;
  const uint32_t n = (uint32_t)P.blockDim;
  const SmemLay L = smemLayout(P.shmem, P.raceCheck, P.htBits);
  __shared__ BlockShared bs;

  // ---- block init ----
  for (uint32_t i = g; i < (uint32_t)P.shmem; i += CT) {
    smem[L.bytes + i] = 0;
    smem[L.meta + i] = 0;
  }
  if (P.raceCheck) {
    uint32_t* sh = (uint32_t*)(smem + L.shadow);
    for (uint32_t i = g; i < (uint32_t)P.shmem; i += CT) sh[i] = shadow_empty(0);
    unsigned long long* rs = (unsigned long long*)(smem + L.raceSet);
    for (uint32_t i = g; i < RACE_SET; i += CT) rs[i] = 0;
  }
  unsigned long long* hk = (unsigned long long*)(smem + L.htKey);
  uint32_t* hv = (uint32_t*)(smem + L.htVal);
  const uint32_t hmask = (1u << P.htBits) - 1;
  for (uint32_t i = g; i <= hmask; i += CT) {
    hk[i] = 0;
    hv[i] = 0;
  }
  if (g == 0) {
    bs.wait[0] = bs.wait[1] = 0;
    bs.nz[0] = bs.nz[1] = 0;
    bs.allc[0] = bs.allc[1] = 0;
    bs.fin = (int)(SLOTS - n);  // padding sub-threads count as finished
    bs.conflict = 0;
    bs.steps = 0;
    bs.allocs = 0;
    bs.sharedEvents = 0;
    bs.lastSweep = 0;
    for (int w = 0; w < 32; ++w) bs.nextRun[0][w] = bs.nextRun[1][w] = 0u;
    bs.soloSweep = 0;
    bs.tailSlot = -1;
  }
  __syncthreads();

  TS t[K];
  Thread th[K];
  Req rq[K];
  Pend pd[K];
  Ctx c;
  c.bid = bid;
  c.sub = 0;
  c.sweep = 0;
#pragma unroll 1
  for (int k = 0; k < K; ++k) {
    const uint32_t tid = (uint32_t)k * CT + g;
    const bool active = tid < n;
    TS& tk = t[k];
    Thread& hk_ = th[k];
    hk_.state = active ? S_READY : S_FIN;
    hk_.readyAt = 1;
    hk_.E = 0;
    hk_.syncKind = 0;
    hk_.operand = 0;
    tk.pc = 0;
    tk.nv = tk.nscope = tk.nowned = tk.nframe = tk.npobj = tk.ptop = 0;
    tk.steps = tk.allocs = 0;
    for (int i = 0; i < POBJ; ++i) tk.pobj[i].gen = 0;
    for (int i = 0; i < BINDS; ++i) tk.binds[i] = 0;
    if (!active) continue;
    // spawnGrid (device.cpp:40-57): params are objects owned by the spawn
    // scope, the dynamic shared array is bound, k = [CallFrame, body]
    const mck_fn& kf = P.fns[P.kernel];
    tk.frames[0].retPc = -1;
    tk.frames[0].bindBase = 0;
    tk.frames[0].fn = P.kernel;
    tk.frames[0].scopeDepth = 0;
    tk.frames[0].valueDepth = 0;
    tk.nframe = 1;
    tk.scopeMark[0] = 0;
    tk.nscope = 1;
    tk.bb = 0;
    tk.fn = P.kernel;
    for (int i = 0; i < P.nargs; ++i) {
      const mck_local& pl = P.locals[kf.local_base + i];
      uint32_t id;
      if (!priv_alloc(tk, P, pl.size, pl.name, id)) {
        hk_.state = S_FIN;
        break;
      }
      priv_poke(tk, tk.pobj[id & 0xFFFFF], 0, pl.type, P.args[i]);
      tk.binds[i] = id;
    }
    tk.allocs = 0;  // spawn-time params are accounted for by the host
    if (kf.dyn_shared_slot >= 0) tk.binds[kf.dyn_shared_slot] = P.sharedBase + bid;
    tk.pc = kf.entry;
    if (hk_.state == S_FIN) atomicAdd(&bs.fin, 1);
  }
  __syncthreads();

  uint32_t E = 0;  // completed episodes (uniform)
  // barrier counters are cumulative per episode parity: episode j (parity
  // j & 1) completes when wait[j & 1] reaches need[j & 1]
  int need[2] = {(int)n, (int)n};
  int nzPrev[2] = {0, 0}, allcPrev[2] = {0, 0};
  unsigned long long rules = 0;
  uint32_t sweep = 0;
  bool deadlocked = false;
  unsigned long long sharedEvents = 0;
  uint32_t lastStep = 0;
  const uint32_t Lt = n - 1;
  bool justSolo = true;  // the next-run table is valid only after a full sweep
  bool noTail = false;   // a tail slot was refused: no further suspension attempts
  uint32_t aloneFrom = ~0u;  // first block-level sweep with one unfinished thread
  bool released = false;  // an episode completed at the loop top (closed-form release)
  uint32_t relT = 0;
  uint32_t soloH = ~0u;   // solo: the first sweep another warp can step
  unsigned long long soloSweeps = 0;
  long long soloCycles = 0;
  const long long kStart = clock64();
  bool solo = false;  // this warp is running sweeps alone (see below)
  uint32_t soloS0 = 0;
  long long soloC0 = 0;
  const uint32_t myWarp = g >> 5, lane = g & 31;

  auto anyReady = [&]() {
    bool r = false;
#pragma unroll 1
    for (int k = 0; k < K; ++k) r |= th[k].state == S_READY;
    return r;
  };

  while (true) {
    if (!solo) {
      // ---- barrier protocol in closed form (Appendix A); counters cover
      // every step up to and including `sweep` ----
      const int p = (E + 1) & 1;
      const int arrived = bs.wait[p] - (need[p] - (int)n);
      const int nfin = bs.fin;
      const int nzNow = bs.nz[p], allcNow = bs.allc[p];
      // every warp reads the counters before any warp's next step phase can
      // change them (a fast warp would otherwise let a slow one see arrivals
      // of the next sweep)
      __syncthreads();
      if (arrived == (int)n) {
        // episode E+1 completed in sweep T = `sweep` (the last arrival): the
        // up-sweep chain, Turnaround (epoch clear) and Down(L) fire in T, one
        // Down per sweep after that, FinalRelease(0) in T + L
        const uint32_t T = sweep;
        const int nz = nzNow - nzPrev[p], allc = allcNow - allcPrev[p];
        nzPrev[p] += nz;
        allcPrev[p] += allc;
        need[p] += (int)n;  // the next episode of this parity is E + 3
#pragma unroll 1
        for (int k = 0; k < K; ++k) {
          const uint32_t tid = (uint32_t)k * CT + g;
          if (tid >= n) continue;
          Thread& x = th[k];
          x.state = S_READY;
          x.readyAt = tid == 0 ? T + Lt + 1 : T + (Lt - tid) + 1;
          x.E = E + 1;
          Val res;
          switch (x.syncKind) {
            case MCK_SYNC_AND: res = v_int(allc == (int)n ? 1 : 0); break;
            case MCK_SYNC_OR: res = v_int(nz > 0 ? 1 : 0); break;
            case MCK_SYNC_COUNT: res = v_int(nz); break;
            default: res = v_void(); break;
          }
          push(t[k], P, res);
        }
        rules += 2ull * n;
        ++E;
        released = true;  // next-run sweeps follow the closed form below
        relT = T;
        if (P.raceCheck && (E & 0xFF) == 0) {  // stamp wrap: clear the shadow
          uint32_t* sh = (uint32_t*)(smem + L.shadow);
          for (uint32_t i = g; i < (uint32_t)P.shmem; i += CT) sh[i] = shadow_empty(0);
          __syncthreads();
        }
      } else if (nfin == (int)SLOTS) {
        break;  // every thread finished
      } else if (arrived + nfin == (int)SLOTS) {
        // quiescent with waiters: barrier deadlock (deadlock.cpp:15-34)
        deadlocked = true;
        break;
      }
      // ---- the serial tail: one unfinished thread left and it is READY
      // The block is suspended into a tail slot -- its shared
      // state, the thread's interpreter state and the block's counters --
      // and the CTA is freed; tail_kernel finishes it, one lane per block ----
      if (nfin == (int)SLOTS - 1 && aloneFrom == ~0u) aloneFrom = sweep;
      if (P.tailCap && !noTail && nfin == (int)SLOTS - 1 && sweep - aloneFrom >= TAIL_MIN) {
        if (g == 0) {
          const uint32_t sl = atomicAdd(P.tailCount, 1u);
          bs.tailSlot = sl < P.tailCap ? (int)sl : -2;
        }
        __syncthreads();
        if (bs.tailSlot >= 0) {
          const int kk = ready_sub<K>(th, g, CT, n);
          suspend_block(P, bs, L, t[kk], th[kk], g, (uint32_t)kk * CT + g, CT, n, sweep, E, lastStep, lb);
          break;
        }
        __syncthreads();
        if (g == 0) bs.tailSlot = -1;
        noTail = true;  // the slots are taken: this block finishes here
      }
      // ---- solo mode: when a single warp holds every READY thread, no other
      // thread can move until that warp arrives at a barrier or finishes, so
      // it runs sweeps alone with warp-level synchronisation while the other
      // warps park on named barrier 1 ----
      // which warps can step in sweep + 1, and from when the others can
      const uint32_t nw_all = (CT + 31u) >> 5;
      uint32_t nr = ~0u;  // lane w: warp w's first runnable sweep
      if (lane < nw_all) {
        if (released) {
          // closed form: thread t >= 1 runs from T + L - t + 1, thread 0 from T + L + 1
          int64_t maxTid = -1;
          for (int k = K - 1; k >= 0 && maxTid < 0; --k) {
            const int64_t base = (int64_t)k * CT + 32 * (int64_t)lane;
            if (base < (int64_t)n) maxTid = base + 31 < (int64_t)n - 1 ? base + 31 : (int64_t)n - 1;
          }
          if (maxTid >= 0) nr = maxTid == 0 ? relT + Lt + 1 : relT + Lt - (uint32_t)maxTid + 1;
        } else {
          nr = justSolo ? 0u : bs.nextRun[sweep & 1][lane];
        }
      }
      released = false;
      justSolo = false;
      const uint32_t busy = __ballot_sync(0xFFFFFFFFu, nr <= sweep + 1);
      if (busy && (busy & (busy - 1)) == 0) {
        const uint32_t sw = (uint32_t)__ffs(busy) - 1;
        soloH = __reduce_min_sync(0xFFFFFFFFu, lane == sw ? ~0u : nr);
        if (myWarp != sw) {
          const long long c0 = clock64();
          const uint32_t s0 = sweep;
          bar_named(1, CT);  // until the solo warp is done
          soloCycles += clock64() - c0;
          if (*(volatile int*)&bs.tailSlot >= 0) break;  // the block was suspended
          sweep = bs.soloSweep;
          soloSweeps += sweep - s0;
          justSolo = true;
          if (sweep >= P.maxSweeps) break;
          continue;
        }
        solo = true;
        soloS0 = sweep;
        soloC0 = clock64();
      }
    }
    if (solo && (sweep + 1 >= soloH || !__any_sync(0xFFFFFFFFu, anyReady()))) {
      // another warp can step from the next sweep on, or nothing is left to
      // run in this warp: hand back to the block
      if (lane == 0) bs.soloSweep = sweep;
      solo = false;
      soloCycles += clock64() - soloC0;
      soloSweeps += sweep - soloS0;
      bar_named(1, CT);
      justSolo = true;
      continue;
    }
    if (solo && P.tailCap && !noTail && sweep - soloS0 >= TAIL_MIN && *(volatile int*)&bs.fin == (int)SLOTS - 1) {
      // the solo warp's last thread is the block's last: suspend it (the
      // other warps are parked and join the exit below)
      int sl = 0;
      if (lane == 0) {
        const uint32_t x = atomicAdd(P.tailCount, 1u);
        sl = x < P.tailCap ? (int)x : -2;
      }
      sl = __shfl_sync(0xFFFFFFFFu, sl, 0);
      if (sl >= 0) {
        if (lane == 0) bs.tailSlot = sl;
        __syncwarp();
        const int kk = ready_sub<K>(th, g, CT, n);
        suspend_block(P, bs, L, t[kk], th[kk], g, (uint32_t)kk * CT + g, 32u, n, sweep, E, lastStep, lb);
        soloCycles += clock64() - soloC0;
        soloSweeps += sweep - soloS0;
        if (lane == 0) bs.soloSweep = sweep;
        __threadfence_block();
        bar_named(1, CT);  // release the parked warps
        break;
      }
      noTail = true;
    }
    ++sweep;
    if (sweep >= P.maxSweeps) {
      set_error(P, ERR_SWEEPS, 0);
      if (solo) {
        if (lane == 0) bs.soloSweep = sweep;
        bar_named(1, CT);
      }
      break;
    }
    c.sweep = sweep;
    // ---- phase 1: one step per runnable sub-thread (tid order k-major) ----
    uint32_t pendMask = 0, runMask = 0;
    bool anyWrite = false;
#pragma unroll 1
    for (int k = 0; k < K; ++k) {
      const uint32_t tid = (uint32_t)k * CT + g;
      rq[k].kind = 0;
      if (tid < n && th[k].state == S_READY && sweep >= th[k].readyAt) {
        runMask |= 1u << k;
        lastStep = sweep;
        c.tid = tid;
        c.sub = 0;
        const int pending = step(t[k], P, c, th[k], rq[k], pd[k], bs, n);
        if (th[k].state == S_FIN) atomicAdd(&bs.fin, 1);
        if (pending) {
          pendMask |= 1u << k;
          anyWrite |= rq[k].kind == 2;
        }
      }
    }
    bool conflict = false;
    uint32_t ins[3 * K];  // hash slots this thread inserted this sweep (it alone clears them)
    uint32_t nins = 0;
    if (solo) {
      // warp-local memory phase: the other warps are parked
      uint32_t nreq = 0;
#pragma unroll 1
      for (int k = 0; k < K; ++k) nreq += __popc(__ballot_sync(0xFFFFFFFFu, (pendMask >> k) & 1u));
      conflict = nreq > 1 && __any_sync(0xFFFFFFFFu, anyWrite);
    } else {
      // word-level overlap with a write among this sweep's requests (one
      // pass: the later inserter of an overlapping pair sees it)
#pragma unroll 1
      for (int k = 0; k < K; ++k) {
        if (!((pendMask >> k) & 1u)) continue;
        const Req& r = rq[k];
        const int len = (int)t_scalar(r.ty);
        const unsigned long long addr =
            r.space == R_OK_SHARED ? (unsigned long long)r.off : (1ull << 40) | (r.base + (unsigned long long)r.off);
        const bool wr = r.kind == 2;
        for (unsigned long long w = addr >> 2; w <= (addr + len - 1) >> 2; ++w) {
          const unsigned long long key = w + 1;
          uint32_t h = (uint32_t)mix64(key) & hmask;
          int slot = -1;
          for (uint32_t probe = 0; probe <= hmask; ++probe) {
            const unsigned long long old = atomicCAS(hk + h, 0ull, key);
            if (old == 0ull || old == key) {
              slot = (int)h;
              if (old == 0ull) ins[nins++] = h;
              break;
            }
            h = (h + 1) & hmask;
          }
          if (slot < 0) {
            conflict = true;  // table full: replay in order (always correct)
            continue;
          }
          const uint32_t old = atomicAdd(hv + slot, wr ? 0x10001u : 1u);
          if ((old & 0xFFFF) != 0 && (wr || (old >> 16) != 0)) conflict = true;
        }
      }
      {
        uint32_t mine = ~0u;
#pragma unroll 1
        for (int k = 0; k < K; ++k)
          if (th[k].state == S_READY) mine = min(mine, max(th[k].readyAt, sweep + 1));
        mine = __reduce_min_sync(0xFFFFFFFFu, mine);
        if (lane == 0) bs.nextRun[sweep & 1][myWarp] = mine;
      }
      conflict = __syncthreads_or(conflict);
    }
    // ---- memory phase: parallel, or replayed in tid order ----
    if (!conflict) {
#pragma unroll 1
      for (int k = 0; k < K; ++k) {
        if (!((pendMask >> k) & 1u)) continue;
        c.tid = (uint32_t)k * CT + g;
        c.sub = 1;
        do_request<HIST>(P, c, th[k], rq[k], L, E & 0xFF, bid, sharedEvents, smem);
        finish_request(t[k], P, th[k], rq[k], pd[k]);
        if (th[k].state == S_FIN) atomicAdd(&bs.fin, 1);
      }
    } else {
      const uint32_t nw = solo ? 1u : (CT >> 5);
#pragma unroll 1
      for (int k = 0; k < K; ++k) {
        for (uint32_t w = 0; w < nw; ++w) {
          if (solo || myWarp == w) {
            for (uint32_t l = 0; l < 32; ++l) {
              if (lane == l && ((pendMask >> k) & 1u)) {
                c.tid = (uint32_t)k * CT + g;
                c.sub = 1;
                do_request<HIST>(P, c, th[k], rq[k], L, E & 0xFF, bid, sharedEvents, smem);
                finish_request(t[k], P, th[k], rq[k], pd[k]);
                if (th[k].state == S_FIN) atomicAdd(&bs.fin, 1);
              }
              __syncwarp();
            }
          }
          if (!solo) __syncthreads();
        }
      }
    }
    if (solo) {
      __syncwarp();  // this sweep's shared writes before the next sweep's reads (lanes are not lockstep)
      bool arrivedNow = false;
#pragma unroll 1
      for (int k = 0; k < K; ++k) arrivedNow |= ((runMask >> k) & 1u) && th[k].state == S_WAIT;
      bool decide = false;
      if (__any_sync(0xFFFFFFFFu, arrivedNow)) {
        // a lane arrived at a barrier.  Only an arrival that completes the
        // episode or leaves the block quiescent (deadlock) changes what the
        // other warps can do; any other one keeps the warp solo (round 1
        // handed the block back on every arrival: one full-block sweep per
        // thread of a release cascade)
        const int p = (E + 1) & 1;
        const int arrived = *(volatile int*)&bs.wait[p] - (need[p] - (int)n);
        const int nfin = *(volatile int*)&bs.fin;
        decide = arrived == (int)n || arrived + nfin == (int)SLOTS;
      }
      if (decide) {
        // the block decides what happens next
        if (lane == 0) bs.soloSweep = sweep;
        solo = false;
        soloCycles += clock64() - soloC0;
        soloSweeps += sweep - soloS0;
        bar_named(1, CT);
        justSolo = true;
      }
      continue;
    }
    // clear the hash slots of this sweep: each by the thread that inserted
    // its key (no probing, so no thread reads a slot another one clears)
#pragma unroll 1
    for (uint32_t i = 0; i < nins; ++i) {
      hk[ins[i]] = 0ull;
      hv[ins[i]] = 0u;
    }
    __syncthreads();
  }

  if (bs.tailSlot >= 0) {
    // suspended: the counters of every thread but the tail's go to the
    // block's partial outputs; tail_kernel adds the rest
    unsigned long long mySteps = 0, myAllocs = 0;
#pragma unroll 1
    for (int k = 0; k < K; ++k) {
      const uint32_t tid = (uint32_t)k * CT + g;
      if (tid < n && th[k].state == S_READY) continue;  // the tail's own
      mySteps += t[k].steps;
      myAllocs += t[k].allocs;
    }
    atomicAdd(&bs.steps, mySteps);
    atomicAdd(&bs.allocs, myAllocs);
    atomicAdd(&bs.sharedEvents, sharedEvents);
    atomicMax(&bs.lastSweep, lastStep);
    __syncthreads();
    if (g == 0) {
      BlockOut& o = P.blocks[lb];
      o.sweeps = bs.soloSweep > sweep ? bs.soloSweep : sweep;
      o.soloSweeps = soloSweeps;
      o.cycles = (unsigned long long)(clock64() - kStart);
      o.soloCycles = (unsigned long long)soloCycles;
      o.steps = bs.steps;
      o.rules = rules;
      o.allocs = bs.allocs;
      o.sharedEvents = bs.sharedEvents;
      o.lastSweep = bs.lastSweep;
      o.deadlocked = 0;
      o.episodes = E;
    }
    return;
  }
  // ---- block outputs ----
  const uint32_t words = (n + 31) / 32;
  unsigned long long steps = 0, allocs = 0;
#pragma unroll 1
  for (int k = 0; k < K; ++k) {
    steps += t[k].steps;
    allocs += t[k].allocs;
    if (deadlocked) {
      const uint32_t tid = (uint32_t)k * CT + g;
      const bool waiting = tid < n && th[k].state == S_WAIT;
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, waiting);
      const uint32_t word = ((uint32_t)k * CT + (myWarp << 5)) >> 5;
      if (lane == 0 && word < words) P.waitMask[(size_t)lb * words + word] = m;
    }
  }
  atomicAdd(&bs.steps, steps);
  atomicAdd(&bs.allocs, allocs);
  atomicAdd(&bs.sharedEvents, sharedEvents);
  atomicMax(&bs.lastSweep, lastStep);
  __syncthreads();
  if (deadlocked) {
    // up-sweep rules of the stuck episode (device.cpp:111-141): the token ran
    // from tid 0 along the waiting prefix: p - 1 rules, p = first non-waiting tid
    __shared__ uint32_t firstNot;
    if (g == 0) firstNot = n;
    __syncthreads();
#pragma unroll 1
    for (int k = 0; k < K; ++k) {
      const uint32_t tid = (uint32_t)k * CT + g;
      if (tid < n && th[k].state != S_WAIT) atomicMin(&firstNot, tid);
    }
    __syncthreads();
    if (g == 0 && firstNot >= 1) rules += firstNot - 1;
  }
  if (g == 0) {
    BlockOut& o = P.blocks[lb];
    o.sweeps = sweep;
    o.soloSweeps = soloSweeps;
    o.cycles = (unsigned long long)(clock64() - kStart);
    o.soloCycles = (unsigned long long)soloCycles;
    o.steps = bs.steps;
    o.rules = rules;
    o.allocs = bs.allocs;
    o.sharedEvents = bs.sharedEvents;
    o.lastSweep = bs.lastSweep;
    o.deadlocked = deadlocked ? 1 : 0;
    o.episodes = E;
  }
}

// ---- tail_kernel: suspended serial tails, one lane per block ----
// The lane continues its block's last thread exactly where grid_kernel left
// it: one step per sweep from max(sweep + 1, readyAt), memory requests served
// at once against the block's shared state in global memory (a lone thread
// has no conflicts), the same shadow and dedup set.  A barrier completes at
// once for a one-thread block (Turnaround and FinalRelease in the arrival
// sweep, Appendix A); with finished peers it never does: a deadlock whose
// up-sweep stops at the first finished thread.  The tails of C2's blocks run
// the same code, so a warp executes 32 of them in lockstep.
__global__ void __launch_bounds__(32) tail_kernel(KP P) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t cnt = min(*P.tailCount, P.tailCap);
  if (i >= cnt) return;
  TailState& S = P.tails[i];
  const uint32_t lb = P.tailBlk[i];
  const uint32_t bid = lb + P.bidBase;
  const uint32_t n = (uint32_t)P.blockDim;
  uint8_t* sb = P.tailSmem + (size_t)i * P.tailStride;
  const SmemLay TL = tailLayout(P.shmem, P.raceCheck);
  TS t = S.t;  // into local memory (L1-cached), the tail's working copy
  Thread th = S.th;
  uint32_t sweep = S.sweep, lastStep = S.lastStep, E = S.E;
  const uint32_t tid = S.tid, sweep0 = S.sweep;
  unsigned long long sharedEvents = 0, rules = 0;
  const long long c0 = clock64();
  bool deadlocked = false;
  Ctx c;
  c.bid = bid;
  c.tid = tid;
  while (true) {
    if (th.state == S_WAIT) {
      if (n != 1) {
        deadlocked = true;  // every peer has finished: the episode never completes
        break;
      }
      // a one-thread block: the episode completes in the arrival sweep
      Val res;
      switch (th.syncKind) {
        case MCK_SYNC_AND: res = v_int(th.operand != 0 ? 1 : 0); break;
        case MCK_SYNC_OR: res = v_int(th.operand != 0 ? 1 : 0); break;
        case MCK_SYNC_COUNT: res = v_int(th.operand != 0 ? 1 : 0); break;
        default: res = v_void(); break;
      }
      push(t, P, res);
      th.state = S_READY;
      th.readyAt = sweep + 1;
      th.operand = 0;
      ++th.E;
      ++E;
      rules += 2;
      if (P.raceCheck && (E & 0xFF) == 0) {  // stamp wrap: clear the shadow
        uint32_t* sh = (uint32_t*)(sb + TL.shadow);
        for (uint32_t b = 0; b < (uint32_t)P.shmem; ++b) sh[b] = shadow_empty(0);
      }
    }
    if (th.state != S_READY) break;
    sweep = max(sweep + 1, th.readyAt);
    if (sweep >= P.maxSweeps) {
      set_error(P, ERR_SWEEPS, 0);
      break;
    }
    c.sweep = sweep;
    c.sub = 0;
    lastStep = sweep;
    Req rq;
    Pend pd;
    rq.kind = 0;
    if (step(t, P, c, th, rq, pd, S.bs, n) && th.state != S_FIN) {
      c.sub = 1;
      do_request<true>(P, c, th, rq, TL, E & 0xFF, bid, sharedEvents, sb);
      finish_request(t, P, th, rq, pd);
    }
  }
  BlockOut& o = P.blocks[lb];
  o.steps += t.steps;
  o.allocs += t.allocs;
  o.sharedEvents += sharedEvents;
  o.lastSweep = max(o.lastSweep, lastStep);
  o.sweeps = sweep;
  o.soloSweeps += sweep - sweep0;
  o.cycles += (unsigned long long)(clock64() - c0);
  o.rules += rules;
  o.episodes = E;
  if (deadlocked) {
    const uint32_t words = (n + 31) / 32;
    o.deadlocked = 1;
    P.waitMask[(size_t)lb * words + tid / 32] = 1u << (tid % 32);
    // up-sweep rules of the stuck episode: first non-waiting tid - 1
    const uint32_t firstNot = tid == 0 ? 1u : 0u;
    if (firstNot >= 1) o.rules += firstNot - 1;
  }
}

// ======================= GPU exhaustive-interleaving oracle =======================
// oracleRace (oracle.cpp:73-154) on the B200: every interleaving of the
// grid's VISIBLE steps -- device steps whose next Item is a load or store
// (LoadRV, LoadKeepLV, StoreAssign, StoreCompound, StoreIncDec) with a
// DeviceShared lvalue on the operand stack, array decays included
// (oracle.cpp:12-36) -- while every invisible step runs eagerly in the
// canonical order (the lowest (gid, bid, tid) first, barrier rules after
// device steps, oracle.cpp:81-103).  A path is a sequence of choices (the
// index of the chosen visible transition among the enabled ones, in key
// order); one GPU thread explores the subtree below one prefix, depth-first,
// re-simulating the grid from its spawn state for every leaf (replay DFS).
// At a leaf: the ground truth (a conflicting pair on one shared byte with no
// barrier of its block between them, traceHasRace oracle.cpp:47-71) and the
// shadow detector's verdict along the path (racecheck.cpp:24-32).
constexpr int OMAX = 8;      // simulated threads of an explored grid
constexpr int ODEPTH = 128;  // visible steps on one path
constexpr int OTRACE = 192;  // trace entries of one path (accesses + epoch marks)

struct OQ {
  const uint8_t* prefixes;   // [nprefix][ODEPTH] choices
  const uint8_t* plens;      // [nprefix] prefix lengths
  uint32_t nprefix;
  int expand;                // 1: only expand each prefix by one choice point
  uint8_t* outPrefixes;      // expand: children prefixes
  uint8_t* outLens;
  uint32_t* nOut;
  uint32_t outCap;
  uint8_t* arenas;           // [GPU thread][2 * arenaSize]: bytes then meta
  const uint8_t* arenaInit;  // the spawn-time global image (bytes then meta)
  uint64_t arenaSize;
  unsigned long long* leaves;
  uint32_t* flags;           // [0] ground-truth race, [1] detector race, [2] error (1 accesses, 2 depth, 3 trace, 4 leaves)
  uint32_t maxAccesses;      // per thread along one path
  unsigned long long maxLeaves;
  uint32_t S;                // shared bytes per block, rounded to 16
  uint32_t slice;            // shared memory per GPU thread (bytes)
};

struct OEv {  // one trace entry
  uint16_t thread;  // simulated thread index; 0xFFFF = epoch mark of block `obj`
  uint8_t len, write;
  uint32_t obj;
  int64_t off;
};

__device__ __forceinline__ bool o_visible(const TS& t, const KP& P) {
  const mck_ins* code = P.code;
  int pc = t.pc;
  mck_ins in = ldg_ins(code + pc);
  while (in.op == OP_JMP) in = ldg_ins(code + in.a);
  int depth;
  switch (in.op) {
    case OP_LOADRV:
    case OP_LOADKEEP: depth = 0; break;
    case OP_STORE:
    case OP_STORE_INC: depth = 1; break;
    case OP_STORE_OP: depth = 2; break;
    default: return false;
  }
  if (t.nv <= depth) return false;
  const Val& lv = t.vals[t.nv - 1 - depth];
  if (lv.kind != MCK_K_LV) return false;
  const uint32_t obj = lv.obj;
  if (obj >= P.sharedBase && (int64_t)(obj - P.sharedBase) < P.gridDim) return true;
  for (int i = 0; i < P.nranges; ++i)
    if (obj >= P.shRanges[3 * i] && obj - P.shRanges[3 * i] < P.shRanges[3 * i + 1]) return true;
  return false;
}

__global__ void __launch_bounds__(64, 1) oracle_kernel(KP P0, OQ Q) {
  extern __shared__ __align__(16) uint8_t osm[];
  const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x;
  if (gt >= Q.nprefix) return;
  const uint32_t nt = (uint32_t)(P0.gridDim * P0.blockDim);
  const uint32_t nb = (uint32_t)P0.gridDim;
  // this GPU thread's shared-memory slice: per block bytes, meta, shadow (S each x 1, 1, 4)
  uint8_t* mysm = osm + (size_t)threadIdx.x * Q.slice;
  BlockShared& bs = *reinterpret_cast<BlockShared*>(mysm + nb * 6 * Q.S);
  KP P = P0;
  P.raceCheck = 0;  // the oracle runs the shadow itself
  P.tarr = nullptr;
  P.glog = nullptr;
  P.glogv = nullptr;
  P.markDirty = 0;
  uint8_t* arena = Q.arenas + (size_t)gt * 2 * Q.arenaSize;
  P.gbytes = arena;
  P.gmeta = arena + Q.arenaSize;
  TS t[OMAX];
  Thread th[OMAX];
  uint8_t choice[ODEPTH], nopt[ODEPTH];
  const uint8_t* pre = Q.prefixes + (size_t)gt * ODEPTH;
  const uint32_t plen = Q.plens[gt];
  for (uint32_t d = 0; d < plen; ++d) choice[d] = pre[d];
  uint32_t depth = plen;  // levels of choice[] fixed so far (the prefix, then this subtree's path)
  OEv tr[OTRACE];
  unsigned long long leaves = 0;
  bool gtRace = false, detRace = false;
  uint32_t err = 0;
  while (true) {
    // ---- replay from the spawn state, following choice[0 .. ) ----
    for (uint64_t i = 0; i < 2 * Q.arenaSize; ++i) arena[i] = Q.arenaInit[i];
    for (uint32_t i = 0; i < nb * 6 * Q.S; ++i) mysm[i] = 0;
    for (uint32_t b = 0; b < nb; ++b) {
      uint32_t* sh = reinterpret_cast<uint32_t*>(mysm + (size_t)(6 * b + 2) * Q.S);
      for (uint32_t i = 0; i < Q.S; ++i) sh[i] = shadow_empty(0);
    }
    uint32_t epoch[OMAX];
    uint32_t acc[OMAX];
    for (uint32_t i = 0; i < nt; ++i) {
      const uint32_t bid = i / (uint32_t)P.blockDim;
      TS& tk = t[i];
      Thread& hk = th[i];
      hk.state = S_READY;
      hk.readyAt = 0;
      hk.E = 0;
      hk.syncKind = 0;
      hk.operand = 0;
      tk.pc = 0;
      tk.nv = tk.nscope = tk.nowned = tk.nframe = tk.npobj = tk.ptop = 0;
      tk.steps = tk.allocs = 0;
      for (int j = 0; j < POBJ; ++j) tk.pobj[j].gen = 0;
      for (int j = 0; j < BINDS; ++j) tk.binds[j] = 0;
      const mck_fn& kf = P.fns[P.kernel];
      tk.frames[0].retPc = -1;
      tk.frames[0].bindBase = 0;
      tk.frames[0].fn = P.kernel;
      tk.frames[0].scopeDepth = 0;
      tk.frames[0].valueDepth = 0;
      tk.nframe = 1;
      tk.scopeMark[0] = 0;
      tk.nscope = 1;
      tk.bb = 0;
      tk.fn = P.kernel;
      for (int a = 0; a < P.nargs; ++a) {
        const mck_local& pl = P.locals[kf.local_base + a];
        uint32_t id;
        if (!priv_alloc(tk, P, pl.size, pl.name, id)) {
          hk.state = S_FIN;
          break;
        }
        priv_poke(tk, tk.pobj[id & 0xFFFFF], 0, pl.type, P.args[a]);
        tk.binds[a] = id;
      }
      if (kf.dyn_shared_slot >= 0) tk.binds[kf.dyn_shared_slot] = P.sharedBase + bid;
      tk.pc = kf.entry;
      epoch[i] = 0;
      acc[i] = 0;
    }
    uint32_t d = 0, ntr = 0;
    bool detHere = false;
    bool aborted = false;
    // one step of simulated thread i (the memory request served at once)
    auto do_step = [&](uint32_t i) {
      const uint32_t bid = i / (uint32_t)P.blockDim, tid = i % (uint32_t)P.blockDim;
      Ctx c;
      c.bid = bid;
      c.tid = tid;
      c.sub = 0;
      c.sweep = 0;
      Req rq;
      Pend pd;
      rq.kind = 0;
      if (step(t[i], P, c, th[i], rq, pd, bs, (uint32_t)P.blockDim) && th[i].state != S_FIN) {
        SmemLay L;
        L.bytes = (uint32_t)(mysm - osm) + (6 * bid) * Q.S;
        L.meta = L.bytes + Q.S;
        L.shadow = L.bytes + 2 * Q.S;
        L.htKey = L.htVal = L.raceSet = L.end = 0;
        if (rq.space == R_OK_SHARED) {
          const int len = (int)t_scalar(rq.ty);
          // recordAccess (racecheck.cpp:9-52): the shadow detector's verdict
          if (shadow_access(reinterpret_cast<uint32_t*>(osm + L.shadow), rq.off, len, tid, rq.kind == 2,
                            epoch[i] & 0xFFu))
            detHere = true;
          if (ntr < OTRACE)
            tr[ntr++] = OEv{(uint16_t)i, (uint8_t)len, (uint8_t)(rq.kind == 2), rq.obj, rq.off};
          else
            aborted = true, err = err ? err : 3u;
        }
        unsigned long long se = 0;
        do_request<false>(P, c, th[i], rq, L, 0, 0, se, osm);
        finish_request(t[i], P, th[i], rq, pd);
      }
      // barrier: a block whose threads all wait is released (the up /
      // turnaround / down / release rules are invisible, device.cpp:143-200);
      // the turnaround clears the block's race epoch (an epoch mark)
      if (th[i].state == S_WAIT) {
        const uint32_t b0 = bid * (uint32_t)P.blockDim, b1 = b0 + (uint32_t)P.blockDim;
        bool all = true;
        int nz = 0, allc = 0;
        for (uint32_t j = b0; j < b1; ++j) {
          if (th[j].state != S_WAIT) all = false;
          if (th[j].operand != 0) ++nz;
          if (th[j].operand != 0 || th[j].syncKind == MCK_SYNC_PLAIN) ++allc;
        }
        if (all) {
          for (uint32_t j = b0; j < b1; ++j) {
            Val res;
            switch (th[j].syncKind) {
              case MCK_SYNC_AND: res = v_int(allc == (int)P.blockDim ? 1 : 0); break;
              case MCK_SYNC_OR: res = v_int(nz > 0 ? 1 : 0); break;
              case MCK_SYNC_COUNT: res = v_int(nz); break;
              default: res = v_void(); break;
            }
            push(t[j], P, res);
            th[j].state = S_READY;
            th[j].operand = 0;
            ++th[j].E;
            ++epoch[j];
          }
          if (ntr < OTRACE)
            tr[ntr++] = OEv{0xFFFFu, 0, 0, P.sharedBase + bid, 0};
          else
            aborted = true, err = err ? err : 3u;
        }
      }
    };
    bool leaf = false;
    bool branched = false;  // expand mode: the choice point past the prefix was reached
    while (!aborted) {
      // closure: the first READY thread (key order) with an invisible next step
      bool moved = true;
      while (moved && !aborted) {
        moved = false;
        for (uint32_t i = 0; i < nt; ++i)
          if (th[i].state == S_READY && !o_visible(t[i], P)) {
            do_step(i);
            moved = true;
            break;
          }
      }
      if (aborted) break;
      // the choice point: visible transitions in key order
      uint32_t opts[OMAX], no = 0;
      for (uint32_t i = 0; i < nt; ++i)
        if (th[i].state == S_READY) opts[no++] = i;
      if (no == 0) {
        leaf = true;
        break;
      }
      if (d >= ODEPTH) {
        aborted = true;
        err = err ? err : 2u;
        break;
      }
      if (Q.expand && d == plen) {
        // one level down: the children of this prefix
        for (uint32_t k = 0; k < no; ++k) {
          const uint32_t o = atomicAdd(Q.nOut, 1u);
          if (o < Q.outCap) {
            for (uint32_t j = 0; j < plen; ++j) Q.outPrefixes[(size_t)o * ODEPTH + j] = choice[j];
            Q.outPrefixes[(size_t)o * ODEPTH + plen] = (uint8_t)k;
            Q.outLens[o] = (uint8_t)(plen + 1);
          }
        }
        branched = true;
        break;
      }
      if (d >= depth) {  // a new level on this path: take the first option
        choice[d] = 0;
        nopt[d] = (uint8_t)no;
        depth = d + 1;
      }
      const uint32_t i = opts[choice[d] < no ? choice[d] : no - 1];
      if (++acc[i] > Q.maxAccesses) {
        aborted = true;
        err = err ? err : 1u;
        break;
      }
      ++d;
      do_step(i);
    }
    if (aborted) break;
    if (leaf) {
      // the leaf budget: flushed in batches, checked against maxInterleavings
      if (++leaves == 1024) {
        const unsigned long long tot = atomicAdd(Q.leaves, leaves) + leaves;
        leaves = 0;
        if (tot > Q.maxLeaves) {
          err = err ? err : 4u;
          break;
        }
      }
      detRace |= detHere;
      // ground truth (traceHasRace, oracle.cpp:47-71)
      for (uint32_t a = 0; a < ntr && !gtRace; ++a) {
        if (tr[a].thread == 0xFFFFu) continue;
        for (uint32_t b = a + 1; b < ntr; ++b) {
          if (tr[b].thread == 0xFFFFu || tr[a].obj != tr[b].obj || tr[a].thread == tr[b].thread) continue;
          if (!tr[a].write && !tr[b].write) continue;
          if (!(tr[a].off < tr[b].off + tr[b].len && tr[b].off < tr[a].off + tr[a].len)) continue;
          bool sep = false;
          for (uint32_t k = a + 1; k < b; ++k)
            if (tr[k].thread == 0xFFFFu && tr[k].obj == tr[a].obj) {
              sep = true;
              break;
            }
          if (!sep) {
            gtRace = true;
            break;
          }
        }
      }
    }
    if (Q.expand || branched) break;
    // next path below the prefix: the deepest level with an untried option
    int lv = (int)depth - 1;
    while (lv >= (int)plen && choice[lv] + 1u >= nopt[lv]) --lv;
    if (lv < (int)plen) break;
    ++choice[lv];
    depth = (uint32_t)lv + 1;
  }
  if (leaves) atomicAdd(Q.leaves, leaves);
  if (gtRace) atomicOr(Q.flags + 0, 1u);
  if (detRace) atomicOr(Q.flags + 1, 1u);
  if (err) atomicCAS(Q.flags + 2, 0u, err);
}

}  // namespace k1

// ======================= host side of the engine =======================
namespace {

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      err = std::string(#x) + ": " + cudaGetErrorString(e_);                   \
      return false;                                                            \
    }                                                                          \
  } while (0)

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  ~DBuf() {
    if (p) cudaFree(p);
  }
  bool ensure(size_t count, std::string& err) {
    if (count <= n && p) return true;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    size_t want = count ? count : 1;
    cudaError_t e = cudaMalloc(&p, want * sizeof(T));
    if (e != cudaSuccess) {
      err = std::string("cudaMalloc: ") + cudaGetErrorString(e);
      p = nullptr;
      return false;
    }
    n = want;
    return true;
  }
};

// MCKG_K1_K=<1|2|4|8> forces the multiplexing factor (experiments).
static int kForceK = [] {
  const char* e = getenv("MCKG_K1_K");
  return e ? atoi(e) : 0;
}();

__global__ void init_ts_kernel(k1::DevDiagRec* p, uint32_t n) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i].ts = ~0ull;
}

// dst <- src for every byte src wrote in the grid (META_DIRTY)
__global__ void merge_dirty_kernel(uint8_t* db, uint8_t* dm, const uint8_t* sb, const uint8_t* sm, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint8_t m = sm[i];
    if (m & META_DIRTY) {
      db[i] = sb[i];
      dm[i] = m;
    }
  }
}

__global__ void clear_dirty_kernel(uint8_t* m, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    m[i] &= (uint8_t)~META_DIRTY;
}

// [lo, hi) of the bytes written by the grid (lohi = {lo, ~hi}, both atomicMin)
__global__ void dirty_range_kernel(const uint8_t* m, uint64_t n, unsigned long long* lohi) {
  unsigned long long lo = ~0ull, nhi = ~0ull;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    if (m[i] & META_DIRTY) {
      lo = min(lo, (unsigned long long)i);
      nhi = min(nhi, ~(unsigned long long)(i + 1));
    }
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    nhi = min(nhi, __shfl_xor_sync(0xffffffffu, nhi, o));
  }
  if ((threadIdx.x & 31) == 0 && lo != ~0ull) {
    atomicMin(lohi, lo);
    atomicMin(lohi + 1, nhi);
  }
}

// one 32-bit word per byte: written ? (rank+1)<<16 | meta<<8 | byte : 0, so
// an all-reduce MAX picks the highest rank's write (the same rule as the
// local replica merge: a later block range wins)
__global__ void pack_dirty_kernel(const uint8_t* b, const uint8_t* m, uint64_t lo, uint64_t n, uint32_t* w,
                                  uint32_t tag) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint8_t mm = m[lo + i];
    w[i] = (mm & META_DIRTY) ? (tag << 16 | (uint32_t)mm << 8 | b[lo + i]) : 0u;
  }
}

__global__ void unpack_dirty_kernel(uint8_t* b, uint8_t* m, uint64_t lo, uint64_t n, const uint32_t* w) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = w[i];
    if (v) {
      b[lo + i] = (uint8_t)v;
      m[lo + i] = (uint8_t)(v >> 8);
    }
  }
}

// One replica of device-global memory and the per-launch buffers of one
// device.  Several replicas may share a physical device ("virtual devices",
// used to test the multi-device split on one GPU).
struct Replica {
  int dev = 0;
  cudaStream_t stream = nullptr;
  uint8_t* bytes = nullptr;
  uint8_t* meta = nullptr;
  uint64_t cap = 0;
  const Program* prog = nullptr;
  DBuf<mck_ins> code;
  DBuf<mck_fn> fns;
  DBuf<mck_local> locals;
  DBuf<uint32_t> ids, glob, ranges, wait;
  DBuf<DevObjInfo> objs;
  DBuf<mck_core::Val> args;
  DBuf<unsigned long long> line, ntri;
  DBuf<int32_t> tri;
  DBuf<k1::DevDiagRec> diag;
  DBuf<k1::BlockOut> blocks;
  DBuf<uint32_t> tarr;
  DBuf<int> err;
  DBuf<k1::TailState> tails;        // suspended serial tails
  DBuf<uint8_t> tailSmem;
  DBuf<uint32_t> tailCnt, tailBlk;
  uint32_t tailCap = 0;             // tail slots of the current grid (0: none)
  size_t glogCap = 0;               // global-access log records of the current grid
  DBuf<mckg_gaccess> glog;          // RunOptions::globalRaceCheck
  DBuf<uint4> glogv;                // the probe's write history (2 x uint4 per record)
  DBuf<unsigned long long> gcnt;    // [0] log length, [1] K6 races, [2..] K6 line table
  DBuf<uint32_t> gstat;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  uint32_t b0 = 0, nb = 0;
};

class CudaEngine final : public DeviceEngine {
 public:
  CudaEngine(std::vector<int> devs, const EngineComm& comm) : devs_(std::move(devs)), comm_(comm) {}
  ~CudaEngine() override {
    if (nccl_) ncclCommDestroy(nccl_);
    for (auto& r : reps_) {
      cudaSetDevice(r.dev);
      if (r.bytes) cudaFree(r.bytes);
      if (r.meta) cudaFree(r.meta);
      if (r.e0) cudaEventDestroy(r.e0);
      if (r.e1) cudaEventDestroy(r.e1);
      if (r.stream) cudaStreamDestroy(r.stream);
    }
  }
  bool init(std::string& err) {
    reps_.resize(devs_.size());
    for (size_t i = 0; i < devs_.size(); ++i) {
      Replica& r = reps_[i];
      r.dev = devs_[i];
      CK(cudaSetDevice(r.dev));
      CK(cudaStreamCreateWithFlags(&r.stream, cudaStreamNonBlocking));
      CK(cudaEventCreate(&r.e0));
      CK(cudaEventCreate(&r.e1));
      // reserve the interpreter's local memory now (per-thread frames of
      // tens of KB x every resident thread): a lazy reservation at the first
      // grid launch would land inside the grid's timed region
      static bool reserved[64] = {};
      if (r.dev >= 0 && r.dev < 64 && !reserved[r.dev]) {
        cudaFuncAttributes fa;
        size_t frame = 0;
        if (cudaFuncGetAttributes(&fa, k1::grid_kernel<1, false>) == cudaSuccess) frame = std::max(frame, fa.localSizeBytes);
        if (cudaFuncGetAttributes(&fa, k1::grid_kernel<4, false>) == cudaSuccess) frame = std::max(frame, fa.localSizeBytes);
        if (cudaFuncGetAttributes(&fa, k1::grid_kernel<4, true>) == cudaSuccess) frame = std::max(frame, fa.localSizeBytes);
        size_t cur = 0;
        cudaDeviceGetLimit(&cur, cudaLimitStackSize);
        if (frame > cur) CK(cudaDeviceSetLimit(cudaLimitStackSize, frame));
        reserved[r.dev] = true;
      }
    }
    // peer access between distinct physical devices (NVLink / NVSwitch)
    for (size_t i = 0; i < devs_.size(); ++i)
      for (size_t j = 0; j < devs_.size(); ++j) {
        if (devs_[i] == devs_[j]) continue;
        int can = 0;
        cudaDeviceCanAccessPeer(&can, devs_[i], devs_[j]);
        if (!can) {
          err = "devices " + std::to_string(devs_[i]) + " and " + std::to_string(devs_[j]) + " have no peer access";
          return false;
        }
        cudaSetDevice(devs_[i]);
        cudaError_t e = cudaDeviceEnablePeerAccess(devs_[j], 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
          err = std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e);
          return false;
        }
        cudaGetLastError();
      }
    // MCKG_K1_FORCE_EXCHANGE=1: run the rank exchange even for world == 1 (a
    // one-rank NCCL communicator) -- exercises the NCCL path on one GPU
    exch_ = comm_.world > 1 || getenv("MCKG_K1_FORCE_EXCHANGE") != nullptr;
    if (exch_ && !comm_.allgather) {
      if (comm_.rank < 0 || comm_.rank >= comm_.world) {
        err = "rank outside 0..world-1";
        return false;
      }
      ncclUniqueId id;
      static_assert(sizeof(id.internal) == 128, "ncclUniqueId");
      std::memcpy(id.internal, comm_.id.data(), 128);
      if (comm_.world == 1 && ncclGetUniqueId(&id) != ncclSuccess) {
        err = "ncclGetUniqueId failed";
        return false;
      }
      CK(cudaSetDevice(reps_[0].dev));
      ncclResult_t r = ncclCommInitRank(&nccl_, comm_.world, id, comm_.rank);
      if (r != ncclSuccess) {
        err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
        nccl_ = nullptr;
        return false;
      }
    }
    return true;
  }
  bool hasDevice() const override { return true; }

  uint64_t alloc(int64_t size) override {
    uint64_t b = (top_ + 15) & ~15ull;
    uint64_t need = b + (uint64_t)size;
    for (auto& r : reps_)
      if (need > r.cap) grow(r, need);
    top_ = need;
    return b;
  }
  void write(uint64_t base, const uint8_t* b, const uint8_t* m, int64_t n) override {
    for (auto& r : reps_) {
      cudaSetDevice(r.dev);
      cudaMemcpy(r.bytes + base, b, (size_t)n, cudaMemcpyHostToDevice);
      cudaMemcpy(r.meta + base, m, (size_t)n, cudaMemcpyHostToDevice);
    }
  }
  void read(uint64_t base, uint8_t* b, uint8_t* m, int64_t n) override {
    Replica& r = reps_[0];
    cudaSetDevice(r.dev);
    cudaMemcpy(b, r.bytes + base, (size_t)n, cudaMemcpyDeviceToHost);
    cudaMemcpy(m, r.meta + base, (size_t)n, cudaMemcpyDeviceToHost);
  }
  void copy(uint64_t dst, uint64_t src, int64_t n) override {
    for (auto& r : reps_) {
      cudaSetDevice(r.dev);
      cudaMemcpy(r.bytes + dst, r.bytes + src, (size_t)n, cudaMemcpyDeviceToDevice);
      cudaMemcpy(r.meta + dst, r.meta + src, (size_t)n, cudaMemcpyDeviceToDevice);
    }
  }
  void fill(uint64_t base, uint8_t v, uint8_t m, int64_t n) override {
    for (auto& r : reps_) {
      cudaSetDevice(r.dev);
      cudaMemset(r.bytes + base, v, (size_t)n);
      cudaMemset(r.meta + base, m, (size_t)n);
    }
  }
  bool runGrid(const GridSpec& g, GridResult& out) override {
    std::string err;
    bool ok = run(g, out, err);
    if (!ok && out.error.empty()) out.error = err;
    return ok;
  }

  // The exhaustive-interleaving oracle over one grid (k1::oracle_kernel):
  // the frontier of schedule prefixes is expanded level by level until it
  // fills the GPU, then every prefix's subtree is explored by one thread.
  bool exploreGrid(const GridSpec& g, const OracleSpec& o, OracleOut& res) override {
    using namespace k1;
    std::string err;
    auto fail = [&](const std::string& m) {
      res.error = m.empty() ? err : m;
      return false;
    };
    const Program& P = *g.prog;
    const uint64_t nt = (uint64_t)g.gridDim * (uint64_t)g.blockDim;
    if (nt > (uint64_t)OMAX) return fail("the GPU oracle explores grids of at most 8 threads");
    if (reps_.size() != 1 || exch_) return fail("the GPU oracle runs on one device and one rank");
    Replica& R = reps_[0];
    CK(cudaSetDevice(R.dev));
    CK(cudaStreamSynchronize(nullptr));
    if (R.prog != &P) {
      if (!upload(R.code, P.code, err) || !upload(R.fns, P.fns, err) || !upload(R.locals, P.locals, err))
        return fail("");
      R.prog = &P;
    }
    std::vector<uint32_t> ids;
    for (const auto& ob : g.objects) ids.push_back(ob.id);
    std::vector<uint32_t> rng;
    for (const auto& r : g.sharedRanges) rng.insert(rng.end(), r.begin(), r.end());
    if (!upload(R.ids, ids, err) || !upload(R.objs, g.objects, err) || !upload(R.glob, g.globalIds, err) ||
        !upload(R.args, g.args, err) || !upload(R.ranges, rng, err) || !R.diag.ensure(1024, err))
      return fail("");
    CK(cudaMemset(R.diag.p, 0, 1024 * sizeof(DevDiagRec)));
    const mck_fn& kf = P.fns[(size_t)g.kernel];
    KP kp{};
    kp.code = R.code.p;
    kp.fns = R.fns.p;
    kp.locals = R.locals.p;
    kp.kernel = g.kernel;
    kp.nargs = (int)g.args.size();
    kp.args = R.args.p;
    kp.gid = g.gid;
    kp.sharedBase = g.sharedBase;
    kp.nextId = g.nextId;
    kp.gridDim = g.gridDim;
    kp.blockDim = g.blockDim;
    kp.shmem = g.shmemBytes;
    kp.sharedName = kf.dyn_shared_slot >= 0 ? P.locals[(size_t)(kf.local_base + kf.dyn_shared_slot)].name
                                            : P.sharedDefaultName;
    kp.warpSize = g.warpSize;
    kp.objIds = R.ids.p;
    kp.objs = R.objs.p;
    kp.nobjs = (int)g.objects.size();
    kp.globalIds = R.glob.p;
    kp.shRanges = R.ranges.p;
    kp.nranges = (int)g.sharedRanges.size();
    kp.maxSweeps = ~0u;
    kp.diags = R.diag.p;
    kp.diagMask = 1023;
    kp.error = nullptr;
    // per explorer: the spawn-time global image (bytes then meta)
    const uint64_t asz = std::max<uint64_t>(16, top_);
    DBuf<uint8_t> init;
    if (!init.ensure(2 * asz, err)) return fail("");
    if (top_) {
      CK(cudaMemcpy(init.p, R.bytes, top_, cudaMemcpyDeviceToDevice));
      CK(cudaMemcpy(init.p + asz, R.meta, top_, cudaMemcpyDeviceToDevice));
    }
    DBuf<int> errbuf;
    if (!errbuf.ensure(2, err)) return fail("");
    CK(cudaMemset(errbuf.p, 0, 2 * sizeof(int)));
    kp.error = errbuf.p;
    kp.errorInfo = errbuf.p + 1;
    OQ q{};
    q.S = (uint32_t)((g.shmemBytes + 15) & ~15ll);
    q.slice = (uint32_t)(((size_t)g.gridDim * 6 * q.S + sizeof(BlockShared) + 15) & ~(size_t)15);
    q.arenaSize = asz;
    q.arenaInit = init.p;
    q.maxAccesses = (uint32_t)std::min<int64_t>(o.maxAccessesPerThread, ODEPTH);
    q.maxLeaves = o.maxInterleavings;
    const uint32_t TPB = 64;
    const size_t smem = (size_t)TPB * q.slice;
    if (smem > 200 * 1024) return fail("the GPU oracle's per-explorer shared arrays exceed shared memory");
    CK(cudaFuncSetAttribute(oracle_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    DBuf<unsigned long long> leaves;
    DBuf<uint32_t> flags, nout;
    if (!leaves.ensure(1, err) || !flags.ensure(3, err) || !nout.ensure(1, err)) return fail("");
    CK(cudaMemset(leaves.p, 0, sizeof(unsigned long long)));
    CK(cudaMemset(flags.p, 0, 3 * sizeof(uint32_t)));
    // frontier: start from the empty prefix
    const uint32_t kFrontier = 8192;
    DBuf<uint8_t> pa, pb, la, lb, arenas;
    if (!pa.ensure((size_t)kFrontier * 64 * ODEPTH, err) || !pb.ensure((size_t)kFrontier * 64 * ODEPTH, err) ||
        !la.ensure((size_t)kFrontier * 64, err) || !lb.ensure((size_t)kFrontier * 64, err))
      return fail("");
    CK(cudaMemset(pa.p, 0, ODEPTH));
    CK(cudaMemset(la.p, 0, 1));
    uint8_t *curP = pa.p, *nxtP = pb.p, *curL = la.p, *nxtL = lb.p;
    uint32_t n = 1;
    auto launch = [&](const uint8_t* pre, const uint8_t* lens, uint32_t cnt, int expand, uint8_t* op, uint8_t* ol,
                      uint32_t cap) -> bool {
      if (!arenas.ensure((size_t)cnt * 2 * asz, err)) return false;
      q.prefixes = pre;
      q.plens = lens;
      q.nprefix = cnt;
      q.expand = expand;
      q.outPrefixes = op;
      q.outLens = ol;
      q.nOut = nout.p;
      q.outCap = cap;
      q.arenas = arenas.p;
      q.leaves = leaves.p;
      q.flags = flags.p;
      CK(cudaMemset(nout.p, 0, sizeof(uint32_t)));
      oracle_kernel<<<(cnt + TPB - 1) / TPB, TPB, smem>>>(kp, q);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      return true;
    };
    for (int level = 0; level < ODEPTH && n > 0 && n < kFrontier; ++level) {
      if (!launch(curP, curL, n, 1, nxtP, nxtL, kFrontier * 64)) return fail("");
      uint32_t m = 0;
      CK(cudaMemcpy(&m, nout.p, sizeof m, cudaMemcpyDeviceToHost));
      uint32_t fl[3];
      CK(cudaMemcpy(fl, flags.p, sizeof fl, cudaMemcpyDeviceToHost));
      if (fl[2] || m > kFrontier * 64) {
        if (m > kFrontier * 64) return fail("oracle frontier overflow");
        n = 0;
        break;
      }
      std::swap(curP, nxtP);
      std::swap(curL, nxtL);
      n = m;
    }
    if (n > 0 && !launch(curP, curL, n, 0, nullptr, nullptr, 0)) return fail("");
    unsigned long long lv = 0;
    uint32_t fl[3];
    int kerr[2];
    CK(cudaMemcpy(&lv, leaves.p, sizeof lv, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(fl, flags.p, sizeof fl, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(kerr, errbuf.p, sizeof kerr, cudaMemcpyDeviceToHost));
    if (kerr[0]) return fail("B200 engine limitation inside the oracle (code " + std::to_string(kerr[0]) + ")");
    res.interleavings = lv;
    res.oracleRace = fl[0] != 0;
    res.detectorRace = fl[1] != 0;
    switch (fl[2]) {
      case 0: break;
      case 1: res.aborted = true; res.error = "a thread performs more shared accesses than the oracle size bound"; break;
      case 2: res.aborted = true; res.error = "a path exceeds the GPU oracle's depth bound"; break;
      case 3: res.aborted = true; res.error = "a path exceeds the GPU oracle's trace bound"; break;
      default: res.aborted = true; res.error = "interleaving budget exceeded"; break;
    }
    if (lv > o.maxInterleavings) {
      res.aborted = true;
      res.error = "interleaving budget exceeded";
      res.interleavings = o.maxInterleavings + 1;  // the count at which the reference stops
    }
    return true;
  }

 private:
  std::vector<int> devs_;
  EngineComm comm_;
  bool exch_ = false;  // rank exchange after every grid
  ncclComm_t nccl_ = nullptr;
  std::vector<Replica> reps_;
  uint64_t top_ = 0;
  DBuf<unsigned long long> lohi_;
  DBuf<uint32_t> packed_;
  DBuf<uint8_t> blobs_;

  void grow(Replica& r, uint64_t need) {
    cudaSetDevice(r.dev);
    uint64_t nc = std::max<uint64_t>(need, std::max<uint64_t>(r.cap * 2, 1ull << 20));
    uint8_t *nb = nullptr, *nm = nullptr;
    cudaMalloc(&nb, nc);
    cudaMalloc(&nm, nc);
    cudaMemset(nb, 0, nc);
    cudaMemset(nm, 0, nc);
    if (r.bytes) {
      cudaMemcpy(nb, r.bytes, top_, cudaMemcpyDeviceToDevice);
      cudaMemcpy(nm, r.meta, top_, cudaMemcpyDeviceToDevice);
      cudaFree(r.bytes);
      cudaFree(r.meta);
    }
    r.bytes = nb;
    r.meta = nm;
    r.cap = nc;
  }

  template <typename T>
  bool upload(DBuf<T>& d, const std::vector<T>& v, std::string& err) {
    if (!d.ensure(v.size(), err)) return false;
    if (!v.empty()) CK(cudaMemcpy(d.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return true;
  }

  bool runLocal(const GridSpec& g, GridResult& out, std::string& err) {
    using namespace k1;
    const Program& P = *g.prog;
    if (g.blockDim > 1024) {
      out.error = "blockDim > 1024 is not supported by the B200 engine";
      return false;
    }
    if (g.gridDim > (1ll << 26)) {
      out.error = "gridDim > 2^26 is not supported by the B200 engine";
      return false;
    }
    // measured (round 1): C4 1024-thread blocks 33 -> 20 ms with K = 4; the
    // 256-thread C2 blocks are fastest with K = 1 (local-memory bound)
    int K = g.blockDim > 256 ? 4 : 1;
    if (kForceK > 0) K = kForceK;
    if (K > 1 && (g.blockDim + K - 1) / K > 256) K = 4;  // K >= 2 kernels take <= 256 threads
    if (K == 1 && g.blockDim > 256) K = 4;               // so does K = 1
    const int threads = (int)(((g.blockDim + K - 1) / K + 31) / 32 * 32);
    int htBits = 1;
    while ((1 << htBits) < 4 * threads * K) ++htBits;
    const SmemLay L = smemLayout(g.shmemBytes, g.raceCheck ? 1 : 0, htBits);
    if (L.end > 200 * 1024) {
      out.error = "the block's shared array (" + std::to_string(g.shmemBytes) +
                  " bytes) exceeds the engine's on-chip shadow capacity";
      return false;
    }
    const size_t total = (size_t)g.gridDim;
    // the conflict probe needs the same single-device, single-rank log
    const bool glogOn = g.globalRaceCheck || (g.conflictProbe && !exch_ && reps_.size() == 1 && total < MCKG_MAX_BID);
    if (g.globalRaceCheck && (exch_ || reps_.size() > 1 || total >= MCKG_MAX_BID)) {
      out.error = "globalRaceCheck runs a grid of < 2^21 blocks on one device and one rank";
      return false;
    }
    if (g.trace && (exch_ || total * (size_t)TEP * (size_t)g.blockDim > (1ull << 26))) {
      out.error = exch_ ? "--trace is single-rank" : "--trace supports grids up to 2^20 threads";
      return false;
    }
    const size_t D = reps_.size();
    const uint32_t words = (uint32_t)((g.blockDim + 31) / 32);
    const uint32_t diagN = 1u << 18;
    std::vector<uint32_t> ids;
    for (const auto& o : g.objects) ids.push_back(o.id);
    std::vector<uint32_t> rng;
    for (const auto& r : g.sharedRanges) rng.insert(rng.end(), r.begin(), r.end());
    const mck_fn& kf = P.fns[(size_t)g.kernel];
    std::vector<unsigned long long> triCaps(D);
    // host-issued copies/memsets run on the legacy stream, which does not
    // order against the engine's non-blocking streams
    for (const auto& R : reps_) {
      CK(cudaSetDevice(R.dev));
      CK(cudaStreamSynchronize(nullptr));
    }
    // ---- launch every replica's block range ----
    // this rank's block range (one process per GPU under torchrun), split
    // again over the local replicas
    const size_t G0 = total * (size_t)comm_.rank / (size_t)comm_.world;
    const size_t GN = total * (size_t)(comm_.rank + 1) / (size_t)comm_.world - G0;
    for (size_t ri = 0; ri < D; ++ri) {
      Replica& R = reps_[ri];
      R.b0 = (uint32_t)(G0 + GN * ri / D);
      R.nb = (uint32_t)(G0 + GN * (ri + 1) / D) - R.b0;
      if (R.nb == 0) continue;
      CK(cudaSetDevice(R.dev));
      if (R.prog != &P) {
        if (!upload(R.code, P.code, err) || !upload(R.fns, P.fns, err) || !upload(R.locals, P.locals, err))
          return false;
        R.prog = &P;
      }
      if (!upload(R.ids, ids, err) || !upload(R.objs, g.objects, err) || !upload(R.glob, g.globalIds, err) ||
          !upload(R.args, g.args, err) || !upload(R.ranges, rng, err))
        return false;
      const size_t nb = R.nb;
      // racy grids report up to ~shmem bytes x lines per block (C2 racy: 508/block)
      triCaps[ri] = g.raceCheck ? std::min<unsigned long long>(1ull << 28, std::max<unsigned long long>(1ull << 22, nb * 1024ull))
                                : 1;
      if (!R.line.ensure(LINES, err) || !R.ntri.ensure(1, err) || !R.tri.ensure(3 * triCaps[ri], err) ||
          !R.diag.ensure(diagN, err) || !R.blocks.ensure(nb, err) || !R.wait.ensure(nb * words, err) ||
          (g.trace && !R.tarr.ensure(nb * TEP * (size_t)g.blockDim, err)) ||
          !R.err.ensure(2, err))
        return false;
      // the global-race log: up to 64 accesses per simulated thread, within
      // [2^20, 2^27] records; a fuller log is an engine error, never a miss
      const size_t glogCap = glogOn
                                 ? std::min<size_t>(1ull << 27, std::max<size_t>(1ull << 20, 64 * nb * (size_t)g.blockDim))
                                 : 0;
      if (glogOn && (!R.glog.ensure(glogCap, err) || !R.gcnt.ensure(2 + LINES, err) ||
                                !R.gstat.ensure(1, err)))
        return false;
      if (glogOn) CK(cudaMemsetAsync(R.gcnt.p, 0, sizeof(unsigned long long), R.stream));
      const bool histOn = glogOn && g.conflictProbe && g.wantHistory;  // the write history (mid-flight copies)
      if (histOn && !R.glogv.ensure(2 * glogCap, err)) return false;
      CK(cudaMemsetAsync(R.line.p, 0xFF, LINES * sizeof(unsigned long long), R.stream));
      CK(cudaMemsetAsync(R.ntri.p, 0, sizeof(unsigned long long), R.stream));
      CK(cudaMemsetAsync(R.diag.p, 0, diagN * sizeof(DevDiagRec), R.stream));
      CK(cudaMemsetAsync(R.wait.p, 0, nb * words * sizeof(uint32_t), R.stream));
      CK(cudaMemsetAsync(R.err.p, 0, 2 * sizeof(int), R.stream));
      if (g.trace) CK(cudaMemsetAsync(R.tarr.p, 0, nb * TEP * (size_t)g.blockDim * sizeof(uint32_t), R.stream));
      init_ts_kernel<<<(diagN + 255) / 256, 256, 0, R.stream>>>(R.diag.p, diagN);
      KP kp;
      kp.code = R.code.p;
      kp.fns = R.fns.p;
      kp.locals = R.locals.p;
      kp.kernel = g.kernel;
      kp.nargs = (int)g.args.size();
      kp.args = R.args.p;
      kp.gid = g.gid;
      kp.sharedBase = g.sharedBase;
      kp.nextId = g.nextId;
      kp.gridDim = g.gridDim;
      kp.blockDim = g.blockDim;
      kp.shmem = g.shmemBytes;
      kp.sharedName = kf.dyn_shared_slot >= 0 ? P.locals[(size_t)(kf.local_base + kf.dyn_shared_slot)].name
                                              : P.sharedDefaultName;
      kp.warpSize = g.warpSize;
      kp.objIds = R.ids.p;
      kp.objs = R.objs.p;
      kp.nobjs = (int)g.objects.size();
      kp.globalIds = R.glob.p;
      kp.shRanges = R.ranges.p;
      kp.nranges = (int)g.sharedRanges.size();
      kp.gbytes = R.bytes;
      kp.gmeta = R.meta;
      kp.raceCheck = g.raceCheck ? 1 : 0;
      kp.htBits = htBits;
      kp.bidBase = R.b0;
      kp.tarr = g.trace ? R.tarr.p : nullptr;
      kp.markDirty = (D > 1 || exch_) ? 1 : 0;
      kp.maxSweeps = (uint32_t)std::min<uint64_t>((1ull << 26) - 1, g.stepBudget + 2);
      // serial-tail slots (MCKG_K1_TAILS=0 turns the offload off)
      static const bool tailsOn = [] {
        const char* e = getenv("MCKG_K1_TAILS");
        return !(e && e[0] == '0');
      }();
      const uint32_t tailCap = tailsOn ? (uint32_t)std::min<size_t>(nb, 1u << 16) : 0u;
      const SmemLay TL = tailLayout(g.shmemBytes, g.raceCheck ? 1 : 0);
      if (tailCap && (!R.tails.ensure(tailCap, err) || !R.tailSmem.ensure((size_t)tailCap * TL.end, err) ||
                      !R.tailCnt.ensure(1, err) || !R.tailBlk.ensure(tailCap, err)))
        return false;
      if (tailCap) CK(cudaMemsetAsync(R.tailCnt.p, 0, sizeof(uint32_t), R.stream));
      kp.tails = tailCap ? R.tails.p : nullptr;
      kp.tailSmem = tailCap ? R.tailSmem.p : nullptr;
      kp.tailCount = tailCap ? R.tailCnt.p : nullptr;
      kp.tailBlk = tailCap ? R.tailBlk.p : nullptr;
      kp.tailCap = tailCap;
      kp.tailStride = TL.end;
      R.tailCap = tailCap;
      R.glogCap = glogCap;
      kp.glog = glogOn ? R.glog.p : nullptr;
      kp.nglog = glogOn ? R.gcnt.p : nullptr;
      kp.glogCap = glogCap;
      kp.glogStrict = g.globalRaceCheck ? 1 : 0;
      kp.glogv = histOn ? R.glogv.p : nullptr;
      void (*kern)(KP) = histOn ? (K == 1   ? grid_kernel<1, true>
                                   : K == 2 ? grid_kernel<2, true>
                                   : K == 4 ? grid_kernel<4, true>
                                            : grid_kernel<8, true>)
                                : (K == 1   ? grid_kernel<1, false>
                                   : K == 2 ? grid_kernel<2, false>
                                   : K == 4 ? grid_kernel<4, false>
                                            : grid_kernel<8, false>);
      kp.lineFirst = R.line.p;
      kp.triples = R.tri.p;
      kp.tripleCap = triCaps[ri];
      kp.nTriples = R.ntri.p;
      kp.diags = R.diag.p;
      kp.diagMask = diagN - 1;
      kp.blocks = R.blocks.p;
      kp.waitMask = R.wait.p;
      kp.error = R.err.p;
      kp.errorInfo = R.err.p + 1;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.end));
      {
        // shared-memory carveout: experiments (MCKG_K1_CARVEOUT=<percent>)
        static int carve = [] {
          const char* e = getenv("MCKG_K1_CARVEOUT");
          return e ? atoi(e) : -1;
        }();
        if (carve >= 0) CK(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
      }
      cudaEventRecord(R.e0, R.stream);
      kern<<<(unsigned)nb, threads, L.end, R.stream>>>(kp);
      if (tailCap) tail_kernel<<<(tailCap + 31) / 32, 32, 0, R.stream>>>(kp);
      cudaEventRecord(R.e1, R.stream);
      CK(cudaGetLastError());
    }
    // ---- collect ----
    std::vector<unsigned long long> lfAll(LINES, ~0ull);
    std::vector<std::array<int64_t, 3>> tris;
    out.launches = 0;
    for (size_t ri = 0; ri < D; ++ri) {
      Replica& R = reps_[ri];
      if (R.nb == 0) continue;
      CK(cudaSetDevice(R.dev));
      CK(cudaStreamSynchronize(R.stream));
      float ms = 0;
      cudaEventElapsedTime(&ms, R.e0, R.e1);
      out.ms = std::max<double>(out.ms, ms);
      out.launches += R.tailCap ? 3 : 2;
      int herr[2];
      CK(cudaMemcpy(herr, R.err.p, sizeof herr, cudaMemcpyDeviceToHost));
      if (herr[0] == ERR_SWEEPS && g.stepBudget + 2 < (1ull << 26) - 1) {
        // more sweeps than steps left (each sweep takes >= 1 step): the run
        // reaches the step limit inside this grid (machine.cpp:1184-1190)
        out.stepLimitHit = true;
        continue;
      }
      if (herr[0]) {
        static const char* why[] = {"", "thread value/scope/frame stack overflow",
                                    "private memory of a thread exceeds the engine limit",
                                    "a pointer to a thread-private object was stored to shared or global memory",
                                    "too many distinct diagnostics", "too many reported race triples",
                                    "source line outside 0..65535",
                                    "sweep budget exhausted (step limit or 2^26 sweeps)", "bad opcode",
                                    "global-race access log full"};
        out.error = std::string("B200 engine limitation: ") + why[herr[0] < 10 ? herr[0] : 0] + " (info " +
                    std::to_string(herr[1]) + ")";
        return false;
      }
      const size_t nb = R.nb;
      std::vector<BlockOut> bo(nb);
      CK(cudaMemcpy(bo.data(), R.blocks.p, nb * sizeof(BlockOut), cudaMemcpyDeviceToHost));
      if (g.trace) {
        if (out.episodes.empty()) {
          out.episodes.assign(total, 0);
          out.arrivals.assign(total * TEP * (size_t)g.blockDim, 0);
        }
        for (size_t b = 0; b < nb; ++b) out.episodes[R.b0 + b] = bo[b].episodes;
        CK(cudaMemcpy(out.arrivals.data() + (size_t)R.b0 * TEP * (size_t)g.blockDim, R.tarr.p,
                      nb * TEP * (size_t)g.blockDim * sizeof(uint32_t), cudaMemcpyDeviceToHost));
      }
      bool anyDl = false;
      for (const auto& b : bo) {
        out.sweeps += b.sweeps;
        out.soloSweeps += b.soloSweeps;
        out.blockCycles += b.cycles;
        out.soloCycles += b.soloCycles;
        out.deviceSteps += b.steps;
        out.barrierRules += b.rules;
        out.allocs += b.allocs;
        out.sharedEvents += b.sharedEvents;
        out.duration = std::max(out.duration, b.lastSweep);
        if (b.deadlocked) anyDl = true;
      }
      if (anyDl) {
        out.deadlocked = true;
        std::vector<uint32_t> wm(nb * words);
        CK(cudaMemcpy(wm.data(), R.wait.p, wm.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost));
        for (size_t b = 0; b < nb; ++b) {
          if (!bo[b].deadlocked) continue;
          GridResult::Stuck st;
          st.bid = R.b0 + (uint32_t)b;
          for (uint32_t t = 0; t < (uint32_t)g.blockDim; ++t)
            if ((wm[b * words + t / 32] >> (t % 32)) & 1u) st.waiting.push_back((int)t);
          out.stuck.push_back(std::move(st));
        }
      }
      std::vector<DevDiagRec> dr(diagN);
      CK(cudaMemcpy(dr.data(), R.diag.p, diagN * sizeof(DevDiagRec), cudaMemcpyDeviceToHost));
      for (const auto& r : dr)
        if (r.hkey) {
          DevDiag d;
          d.key = r.ts;
          d.code = r.code;
          d.line = r.line;
          for (int i = 0; i < 4; ++i) d.p[i] = r.p[i];
          d.name = r.name;
          out.diags.push_back(d);
        }
      std::vector<unsigned long long> lf(LINES);
      CK(cudaMemcpy(lf.data(), R.line.p, LINES * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
      for (int l = 0; l < LINES; ++l) lfAll[(size_t)l] = std::min(lfAll[(size_t)l], lf[(size_t)l]);
      unsigned long long nlogProbe = 0;
      if (glogOn && !g.globalRaceCheck)
        CK(cudaMemcpy(&nlogProbe, R.gcnt.p, sizeof nlogProbe, cudaMemcpyDeviceToHost));
      if (glogOn && (g.globalRaceCheck || nlogProbe <= R.glogCap)) {
        // cross-block global races of this grid: K6 over the access log
        // (a builder-defined extension, off by default)
        unsigned long long nlog = 0;
        CK(cudaMemcpy(&nlog, R.gcnt.p, sizeof nlog, cudaMemcpyDeviceToHost));
        unsigned long long* glf = R.gcnt.p + 2;
        CK(cudaMemsetAsync(glf, 0xFF, LINES * sizeof(unsigned long long), R.stream));
        CK(cudaMemsetAsync(R.gstat.p, 0, sizeof(uint32_t), R.stream));
        if (mckg_detect_global(R.glog.p, nlog, 0, nullptr, 0, R.gcnt.p + 1, glf, R.gstat.p, R.stream) != MCKG_OK) {
          out.error = std::string("global-race detection failed: ") + mckg_last_error();
          return false;
        }
        std::vector<unsigned long long> gl(LINES);
        CK(cudaMemcpyAsync(gl.data(), glf, LINES * sizeof(unsigned long long), cudaMemcpyDeviceToHost, R.stream));
        CK(cudaStreamSynchronize(R.stream));
        out.launches += 6;
        if (nlog && nlog <= (1ull << 18) && nlog <= R.glogCap) {
          // the grid's global footprint per object (for in-flight overlap checks)
          std::vector<mckg_gaccess> lg(nlog);
          CK(cudaMemcpy(lg.data(), R.glog.p, nlog * sizeof(mckg_gaccess), cudaMemcpyDeviceToHost));
          std::vector<size_t> ord(g.objects.size());
          for (size_t i = 0; i < ord.size(); ++i) ord[i] = i;
          std::sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return g.objects[a].base < g.objects[b].base; });
          std::map<uint32_t, std::array<int64_t, 5>> fp;
          std::vector<uint4> hv;
          if (g.conflictProbe && g.wantHistory && R.glogv.p) {
            hv.resize(2 * nlog);
            CK(cudaMemcpy(hv.data(), R.glogv.p, hv.size() * sizeof(uint4), cudaMemcpyDeviceToHost));
          }
          bool complexAny = false;
          for (size_t li = 0; li < lg.size(); ++li) {
            const mckg_gaccess& x = lg[li];
            const uint64_t a = x.a & 0xFFFFFFFFFFull;
            const int64_t len = (int64_t)((x.a >> 40) & 0xF);
            const bool wr = (x.a >> 44) & 1u;
            auto it = std::upper_bound(ord.begin(), ord.end(), a,
                                       [&](uint64_t v, size_t k) { return v < g.objects[k].base; });
            if (it == ord.begin()) continue;
            const DevObjInfo& o = g.objects[*(it - 1)];
            const int64_t off = (int64_t)(a - o.base);
            if (off >= o.size) continue;
            auto& e = fp.emplace(o.id, std::array<int64_t, 5>{(int64_t)o.id, INT64_MAX, INT64_MIN, INT64_MAX,
                                                              INT64_MIN}).first->second;
            const int k = wr ? 3 : 1;
            e[k] = std::min(e[k], off);
            e[k + 1] = std::max(e[k + 1], off + len);
            if (wr && !hv.empty()) {
              const uint4 v0 = hv[2 * li], v1 = hv[2 * li + 1];
              complexAny |= v1.z != 0u;
              GridResult::Write w;
              w.obj = o.id;
              w.lsweep = x.sweep;
              w.bid = x.b & 0xFFFFFFu;
              w.tid = (uint32_t)((x.a >> 45) & 0x7FFu);
              w.off = off;
              w.len = (uint32_t)len;
              const uint32_t ob[2] = {v0.x, v0.y}, om[2] = {v0.z, v0.w}, nw[2] = {v1.x, v1.y};
              for (int q = 0; q < 8; ++q) {
                w.oldB[q] = (uint8_t)(ob[q >> 2] >> (8 * (q & 3)));
                w.oldM[q] = (uint8_t)(om[q >> 2] >> (8 * (q & 3)));
                w.newB[q] = (uint8_t)(nw[q >> 2] >> (8 * (q & 3)));
              }
              out.writes.push_back(w);
            }
          }
          for (auto& kv : fp) out.footprint.push_back(kv.second);
          if (complexAny) out.writes.clear();
          // global order of the writes: (local sweep, bid, tid)
          std::stable_sort(out.writes.begin(), out.writes.end(), [](const GridResult::Write& p, const GridResult::Write& q) {
            return std::tie(p.lsweep, p.bid, p.tid) < std::tie(q.lsweep, q.bid, q.tid);
          });
        }
        for (int l = 0; l < LINES; ++l)
          if (gl[(size_t)l] != ~0ull) out.globalConflicts = true;
        for (int l = 0; l < LINES && g.globalRaceCheck; ++l)
          if (gl[(size_t)l] != ~0ull) {
            // K6 key sweep:32 | bid:21 | tid:11 -> the device-diagnostic key
            const unsigned long long k = gl[(size_t)l];
            DevDiag d;
            d.key = tskey((uint32_t)(k >> 32), (uint32_t)(k >> 11) & (MCKG_MAX_BID - 1), (uint32_t)k & 0x7FFu, 0);
            d.code = MCK_D_GRACE;
            d.line = l;
            d.p[0] = d.p[1] = d.p[2] = d.p[3] = 0;
            d.name = -1;
            out.diags.push_back(d);
          }
      }
      unsigned long long ntri = 0;
      CK(cudaMemcpy(&ntri, R.ntri.p, sizeof ntri, cudaMemcpyDeviceToHost));
      if (ntri) {
        std::vector<int32_t> tri(3 * std::min<unsigned long long>(ntri, triCaps[ri]));
        CK(cudaMemcpy(tri.data(), R.tri.p, tri.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < tri.size(); i += 3)
          tris.push_back({(int64_t)(uint32_t)tri[i], (int64_t)(uint32_t)tri[i + 1], (int64_t)tri[i + 2]});
      }
    }
    for (int l = 0; l < LINES; ++l)
      if (lfAll[(size_t)l] != ~0ull) {
        DevDiag d;
        d.key = lfAll[(size_t)l];
        d.code = MCK_D_RACE;
        d.line = l;
        d.p[0] = d.p[1] = d.p[2] = d.p[3] = 0;
        d.name = -1;
        out.diags.push_back(d);
      }
    std::sort(tris.begin(), tris.end());
    tris.erase(std::unique(tris.begin(), tris.end()), tris.end());
    out.reported = std::move(tris);
    std::sort(out.stuck.begin(), out.stuck.end(),
              [](const GridResult::Stuck& a, const GridResult::Stuck& b) { return a.bid < b.bid; });
    if (out.stepLimitHit) {
      // the run is abandoned inside this grid: its whole budget is spent and
      // the grid's partial effects are dropped (the host reports the limit)
      out.deviceSteps = std::max<uint64_t>(out.deviceSteps, g.stepBudget);
      out.barrierRules = 0;
      out.diags.clear();
      out.reported.clear();
      out.stuck.clear();
      out.deadlocked = false;
      out.duration = 0;
    }
    return true;
  }

  // ---- replicated global memory: merge every replica's writes into
  // replica 0 in block-range order (a later range wins a cross-block
  // conflict) ----
  bool mergeLocal(GridResult& out, std::string& err) {
    const size_t D = reps_.size();
    if (D == 1 || top_ == 0) return true;
    Replica& R0 = reps_[0];
    CK(cudaSetDevice(R0.dev));
    for (size_t ri = 1; ri < D; ++ri) {
      if (reps_[ri].nb == 0) continue;
      merge_dirty_kernel<<<148u * 8u, 256, 0, R0.stream>>>(R0.bytes, R0.meta, reps_[ri].bytes, reps_[ri].meta, top_);
      ++out.launches;
    }
    CK(cudaStreamSynchronize(R0.stream));
    return true;
  }

  // clear the dirty bits of replica 0, then copy it to the other replicas
  bool finishMemory(GridResult& out, std::string& err) {
    const size_t D = reps_.size();
    if ((D == 1 && !exch_) || top_ == 0) return true;
    Replica& R0 = reps_[0];
    CK(cudaSetDevice(R0.dev));
    clear_dirty_kernel<<<148u * 8u, 256, 0, R0.stream>>>(R0.meta, top_);
    out.launches += 1;
    CK(cudaStreamSynchronize(R0.stream));
    for (size_t ri = 1; ri < D; ++ri) {
      CK(cudaMemcpyPeer(reps_[ri].bytes, reps_[ri].dev, R0.bytes, R0.dev, top_));
      CK(cudaMemcpyPeer(reps_[ri].meta, reps_[ri].dev, R0.meta, R0.dev, top_));
    }
    for (const auto& R : reps_) {
      CK(cudaSetDevice(R.dev));
      CK(cudaDeviceSynchronize());
    }
    return true;
  }

  // ---- ranks: every rank holds the same global image before the grid;
  // the bytes each rank's blocks wrote are combined by one all-reduce(MAX)
  // over the union of the written ranges ----
  // host transport: gather `n` bytes from every rank (rank order)
  bool hostGather(const void* send, size_t n, std::vector<uint8_t>& all, std::string& err) {
    all.assign(n * (size_t)comm_.world, 0);
    if (comm_.allgather(comm_.ctx, send, n, all.data()) != 0) {
      err = "host allgather callback failed";
      return false;
    }
    return true;
  }

  bool exchangeMemoryHost(GridResult& out, std::string& err) {
    Replica& R0 = reps_[0];
    CK(cudaSetDevice(R0.dev));
    if (!lohi_.ensure(2, err)) return false;
    CK(cudaMemsetAsync(lohi_.p, 0xFF, 2 * sizeof(unsigned long long), R0.stream));
    if (top_ > 0) {
      dirty_range_kernel<<<148u * 8u, 256, 0, R0.stream>>>(R0.meta, top_, lohi_.p);
      ++out.launches;
    }
    unsigned long long mine[2];
    CK(cudaMemcpyAsync(mine, lohi_.p, sizeof mine, cudaMemcpyDeviceToHost, R0.stream));
    CK(cudaStreamSynchronize(R0.stream));
    std::vector<uint8_t> all;
    if (!hostGather(mine, sizeof mine, all, err)) return false;
    unsigned long long lo = ~0ull, nhi = ~0ull;
    for (int r = 0; r < comm_.world; ++r) {
      unsigned long long v[2];
      std::memcpy(v, all.data() + r * sizeof v, sizeof v);
      lo = std::min(lo, v[0]);
      nhi = std::min(nhi, v[1]);
    }
    const uint64_t hi = ~nhi;
    if (lo == ~0ull || hi <= lo) return true;
    const uint64_t n = hi - lo;
    if (!packed_.ensure(n, err)) return false;
    pack_dirty_kernel<<<148u * 8u, 256, 0, R0.stream>>>(R0.bytes, R0.meta, lo, n, packed_.p,
                                                        (uint32_t)comm_.rank + 1);
    std::vector<uint32_t> w(n);
    CK(cudaMemcpyAsync(w.data(), packed_.p, n * 4, cudaMemcpyDeviceToHost, R0.stream));
    CK(cudaStreamSynchronize(R0.stream));
    if (!hostGather(w.data(), n * 4, all, err)) return false;
    for (int r = 0; r < comm_.world; ++r) {
      const uint32_t* q = reinterpret_cast<const uint32_t*>(all.data() + (size_t)r * n * 4);
      for (uint64_t i = 0; i < n; ++i) w[i] = std::max(w[i], q[i]);
    }
    CK(cudaMemcpyAsync(packed_.p, w.data(), n * 4, cudaMemcpyHostToDevice, R0.stream));
    unpack_dirty_kernel<<<148u * 8u, 256, 0, R0.stream>>>(R0.bytes, R0.meta, lo, n, packed_.p);
    out.launches += 2;
    CK(cudaStreamSynchronize(R0.stream));
    return true;
  }

  bool exchangeMemory(GridResult& out, std::string& err) {
    if (comm_.allgather) return exchangeMemoryHost(out, err);
    Replica& R0 = reps_[0];
    CK(cudaSetDevice(R0.dev));
    if (!lohi_.ensure(2, err)) return false;
    CK(cudaMemsetAsync(lohi_.p, 0xFF, 2 * sizeof(unsigned long long), R0.stream));
    if (top_ > 0) {
      dirty_range_kernel<<<148u * 8u, 256, 0, R0.stream>>>(R0.meta, top_, lohi_.p);
      ++out.launches;
    }
    if (ncclAllReduce(lohi_.p, lohi_.p, 2, ncclUint64, ncclMin, nccl_, R0.stream) != ncclSuccess) {
      err = "ncclAllReduce (dirty range) failed";
      return false;
    }
    unsigned long long lohi[2];
    CK(cudaMemcpyAsync(lohi, lohi_.p, sizeof lohi, cudaMemcpyDeviceToHost, R0.stream));
    CK(cudaStreamSynchronize(R0.stream));
    const uint64_t lo = lohi[0], hi = ~lohi[1];
    if (lo == ~0ull || hi <= lo) return true;  // nobody wrote device memory
    const uint64_t n = hi - lo;
    if (!packed_.ensure(n, err)) return false;
    pack_dirty_kernel<<<148u * 8u, 256, 0, R0.stream>>>(R0.bytes, R0.meta, lo, n, packed_.p,
                                                        (uint32_t)comm_.rank + 1);
    if (ncclAllReduce(packed_.p, packed_.p, n, ncclUint32, ncclMax, nccl_, R0.stream) != ncclSuccess) {
      err = "ncclAllReduce (written bytes) failed";
      return false;
    }
    unpack_dirty_kernel<<<148u * 8u, 256, 0, R0.stream>>>(R0.bytes, R0.meta, lo, n, packed_.p);
    out.launches += 2;
    CK(cudaStreamSynchronize(R0.stream));
    return true;
  }

  // ---- ranks: gather every rank's partial GridResult (in rank order) ----
  struct BlobHdr {
    uint64_t ok, deviceSteps, barrierRules, allocs, sharedEvents, sweeps, soloSweeps, blockCycles, soloCycles;
    uint64_t duration, deadlocked, nDiag, nStuck, nTids, nTri, errLen, launches;
    double ms;
  };

  static void serialize(const GridResult& r, bool ok, std::vector<uint8_t>& b) {
    BlobHdr h{};
    h.ok = ok;
    h.deviceSteps = r.deviceSteps;
    h.barrierRules = r.barrierRules;
    h.allocs = r.allocs;
    h.sharedEvents = r.sharedEvents;
    h.sweeps = r.sweeps;
    h.soloSweeps = r.soloSweeps;
    h.blockCycles = r.blockCycles;
    h.soloCycles = r.soloCycles;
    h.duration = r.duration;
    h.deadlocked = r.deadlocked;
    h.nDiag = r.diags.size();
    h.nStuck = r.stuck.size();
    for (const auto& s : r.stuck) h.nTids += s.waiting.size();
    h.nTri = r.reported.size();
    h.errLen = r.error.size();
    h.launches = r.launches;
    h.ms = r.ms;
    auto put = [&b](const void* p, size_t n) {
      const uint8_t* c = static_cast<const uint8_t*>(p);
      b.insert(b.end(), c, c + n);
    };
    put(&h, sizeof h);
    if (!r.diags.empty()) put(r.diags.data(), r.diags.size() * sizeof(DevDiag));
    for (const auto& s : r.stuck) {
      uint64_t v[2] = {s.bid, s.waiting.size()};
      put(v, sizeof v);
      if (!s.waiting.empty()) put(s.waiting.data(), s.waiting.size() * sizeof(int));
    }
    if (!r.reported.empty()) put(r.reported.data(), r.reported.size() * sizeof(r.reported[0]));
    put(r.error.data(), r.error.size());
  }

  static void deserializeInto(const uint8_t* p, GridResult& r, bool& ok) {
    BlobHdr h;
    std::memcpy(&h, p, sizeof h);
    p += sizeof h;
    ok = ok && h.ok;
    r.deviceSteps += h.deviceSteps;
    r.barrierRules += h.barrierRules;
    r.allocs += h.allocs;
    r.sharedEvents += h.sharedEvents;
    r.sweeps += h.sweeps;
    r.soloSweeps += h.soloSweeps;
    r.blockCycles += h.blockCycles;
    r.soloCycles += h.soloCycles;
    r.duration = std::max<uint32_t>(r.duration, (uint32_t)h.duration);
    r.deadlocked = r.deadlocked || h.deadlocked;
    r.ms = std::max(r.ms, h.ms);
    for (uint64_t i = 0; i < h.nDiag; ++i, p += sizeof(DevDiag)) {
      DevDiag d;
      std::memcpy(&d, p, sizeof d);
      r.diags.push_back(d);
    }
    for (uint64_t i = 0; i < h.nStuck; ++i) {
      uint64_t v[2];
      std::memcpy(v, p, sizeof v);
      p += sizeof v;
      GridResult::Stuck s;
      s.bid = (uint32_t)v[0];
      s.waiting.resize(v[1]);
      if (v[1]) std::memcpy(s.waiting.data(), p, v[1] * sizeof(int));
      p += v[1] * sizeof(int);
      r.stuck.push_back(std::move(s));
    }
    for (uint64_t i = 0; i < h.nTri; ++i, p += sizeof(std::array<int64_t, 3>)) {
      std::array<int64_t, 3> t;
      std::memcpy(&t, p, sizeof t);
      r.reported.push_back(t);
    }
    if (h.errLen && r.error.empty()) r.error.assign(reinterpret_cast<const char*>(p), h.errLen);
  }

  bool exchangeResults(GridResult& out, bool& ok, std::string& err) {
    Replica& R0 = reps_[0];
    CK(cudaSetDevice(R0.dev));
    std::vector<uint8_t> mine;
    serialize(out, ok, mine);
    const int W = comm_.world;
    std::vector<uint8_t> all;
    size_t slot = 0;
    if (comm_.allgather) {
      unsigned long long sz = mine.size();
      if (!hostGather(&sz, sizeof sz, all, err)) return false;
      unsigned long long mx = 0;
      for (int r = 0; r < W; ++r) {
        unsigned long long v;
        std::memcpy(&v, all.data() + r * sizeof v, sizeof v);
        mx = std::max(mx, v);
      }
      slot = ((size_t)mx + 15) & ~(size_t)15;
      mine.resize(slot, 0);
      if (!hostGather(mine.data(), slot, all, err)) return false;
    } else if (!gatherNccl(mine, all, slot, err)) {
      return false;
    }
    GridResult m;
    bool allOk = true;
    for (int r = 0; r < W; ++r) deserializeInto(all.data() + slot * r, m, allOk);
    std::sort(m.reported.begin(), m.reported.end());
    m.reported.erase(std::unique(m.reported.begin(), m.reported.end()), m.reported.end());
    std::sort(m.stuck.begin(), m.stuck.end(),
              [](const GridResult::Stuck& a, const GridResult::Stuck& b) { return a.bid < b.bid; });
    m.launches = out.launches;
    out = std::move(m);
    ok = allOk;
    if (!ok && out.error.empty()) out.error = "B200 engine: a peer rank failed this grid";
    return true;
  }

  bool gatherNccl(std::vector<uint8_t>& mine, std::vector<uint8_t>& all, size_t& slot, std::string& err) {
    Replica& R0 = reps_[0];
    const int W = comm_.world;
    // sizes
    if (!lohi_.ensure((size_t)W + 1, err)) return false;
    unsigned long long sz = mine.size();
    CK(cudaMemcpyAsync(lohi_.p + W, &sz, sizeof sz, cudaMemcpyHostToDevice, R0.stream));
    if (ncclAllGather(lohi_.p + W, lohi_.p, 1, ncclUint64, nccl_, R0.stream) != ncclSuccess) {
      err = "ncclAllGather (result sizes) failed";
      return false;
    }
    std::vector<unsigned long long> sizes(W);
    CK(cudaMemcpyAsync(sizes.data(), lohi_.p, W * sizeof(unsigned long long), cudaMemcpyDeviceToHost, R0.stream));
    CK(cudaStreamSynchronize(R0.stream));
    const size_t mx = (size_t)*std::max_element(sizes.begin(), sizes.end());
    slot = (mx + 15) & ~(size_t)15;
    if (!blobs_.ensure(slot * (W + 1), err)) return false;
    mine.resize(slot, 0);
    uint8_t* send = blobs_.p + slot * W;
    CK(cudaMemcpyAsync(send, mine.data(), slot, cudaMemcpyHostToDevice, R0.stream));
    if (ncclAllGather(send, blobs_.p, slot, ncclUint8, nccl_, R0.stream) != ncclSuccess) {
      err = "ncclAllGather (results) failed";
      return false;
    }
    all.assign(slot * W, 0);
    CK(cudaMemcpyAsync(all.data(), blobs_.p, all.size(), cudaMemcpyDeviceToHost, R0.stream));
    CK(cudaStreamSynchronize(R0.stream));
    return true;
  }

  bool run(const GridSpec& g, GridResult& out, std::string& err) {
    bool ok = runLocal(g, out, err) && mergeLocal(out, err);
    if (exch_) {
      if (!ok && out.error.empty()) out.error = err.empty() ? "B200 engine error" : err;
      if (!exchangeResults(out, ok, err)) return false;
      if (ok && !exchangeMemory(out, err)) return false;
    }
    if (!finishMemory(out, err)) return false;
    return ok;
  }
};

}  // namespace

std::unique_ptr<DeviceEngine> makeCudaEngine(const std::vector<int>& devices, const EngineComm& comm,
                                             std::string& why) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    why = e != cudaSuccess ? cudaGetErrorString(e) : "no CUDA device";
    cudaGetLastError();
    return nullptr;
  }
  for (int d : devices)
    if (d < 0 || d >= n) {
      why = "no such device " + std::to_string(d);
      return nullptr;
    }
  std::unique_ptr<CudaEngine> eng(new CudaEngine(devices, comm));
  if (!eng->init(why)) return nullptr;
  return std::unique_ptr<DeviceEngine>(eng.release());
}

bool makeCommId(std::array<uint8_t, 128>& id, std::string& why) {
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) {
    why = std::string("ncclGetUniqueId: ") + ncclGetErrorString(r);
    return false;
  }
  std::memcpy(id.data(), u.internal, 128);
  return true;
}

}  // namespace mckb
