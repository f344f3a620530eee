/* global_detector.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * CPU restatement of the cross-block global-memory race extension (BASELINE
 * config 5), the checker of mckg_detect_global.  Parity is
 * UNPINNED: the reference checks DeviceShared objects only
 * (memory.cpp:142-143, 240-241).  The rule is racecheck.cpp:24-32 with
 * "thread" replaced by "block": records are replayed in timestamp order
 * (sweep, bid, tid) over a per-byte shadow {some accessor block + multi flag,
 * some writer block + multi flag}; X races iff (X writes and a block other
 * than X's accessed the byte) or (X reads and a block other than X's wrote
 * it).  Each racing (byte, line) is reported once; line_first keeps the
 * minimum racing timestamp per line.  Also the CPU copy of mckg_gen_c5.
 */
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

static inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void oracle_gen_c5(mckg_gaccess* ev, uint32_t blk0, uint32_t n_blocks, uint32_t n_total, uint64_t seed) {
  const uint64_t per = MCKG_C5_EVENTS_PER_BLOCK;
  for (uint64_t r = 0; r < (uint64_t)n_blocks * per; ++r) {
    uint64_t i = (uint64_t)blk0 * per + r;
    uint32_t b = (uint32_t)(i / per), j = (uint32_t)(i % per);
    uint32_t tid = j % 256u, k = j / 256u;
    uint64_t h = splitmix64(seed + i);
    int write = (int)(h & 1u);
    int redirect = ((h >> 32) % 10000u) < 100u;
    uint32_t tb = redirect ? (b + 1u) % n_total : b;
    uint64_t addr = (uint64_t)tb * MCKG_C5_RANGE + (uint64_t)(tid * 16u + k) * 8u;
    ev[r] = mckg_make_gaccess(addr, 4u, write, tid, b, 200 + (int32_t)(k % 4u), k);
  }
}

typedef struct {
  uint64_t key;  /* byte address + 1 (0 = empty) */
  uint32_t abid, wbid;
  uint8_t amulti, wmulti, has_w, pad;
} slot_t;

typedef struct {
  slot_t* s;
  uint64_t cap, n;
} bmap_t;

static slot_t* bmap_get(bmap_t* m, uint64_t byte) {
  if ((m->n + 1) * 2 > m->cap) {
    uint64_t nc = m->cap ? m->cap * 2 : 1024;
    slot_t* ns = (slot_t*)calloc(nc, sizeof(slot_t));
    for (uint64_t i = 0; i < m->cap; ++i)
      if (m->s[i].key) {
        uint64_t h = (m->s[i].key * 0x9E3779B97F4A7C15ull) & (nc - 1);
        while (ns[h].key) h = (h + 1) & (nc - 1);
        ns[h] = m->s[i];
      }
    free(m->s);
    m->s = ns;
    m->cap = nc;
  }
  uint64_t key = byte + 1, h = (key * 0x9E3779B97F4A7C15ull) & (m->cap - 1);
  while (m->s[h].key && m->s[h].key != key) h = (h + 1) & (m->cap - 1);
  if (!m->s[h].key) {
    m->s[h].key = key;
    m->s[h].abid = 0xFFFFFFFFu;
    m->s[h].wbid = 0xFFFFFFFFu;
    m->n++;
  }
  return &m->s[h];
}

typedef struct {
  const mckg_gaccess* ev;
  uint64_t i;
} ref_t;

static uint64_t tskey(const mckg_gaccess* r) {
  return mckg_ts_key(r->sweep, MCKG_GA_BID(*r), MCKG_GA_TID(*r));
}

static int cmp_ts(const void* a, const void* b) {
  const ref_t* x = (const ref_t*)a;
  const ref_t* y = (const ref_t*)b;
  uint64_t kx = tskey(x->ev + x->i), ky = tskey(y->ev + y->i);
  if (kx != ky) return kx < ky ? -1 : 1;
  return x->i < y->i ? -1 : (x->i > y->i ? 1 : 0);
}

static int cmp_race(const void* a, const void* b) {
  const mckg_grace* x = (const mckg_grace*)a;
  const mckg_grace* y = (const mckg_grace*)b;
  if (x->addr != y->addr) return x->addr < y->addr ? -1 : 1;
  return x->line < y->line ? -1 : (x->line > y->line ? 1 : 0);
}

int oracle_detect_global(const mckg_gaccess* ev, uint64_t n, mckg_grace* races, uint64_t capacity,
                         uint64_t* n_races, uint64_t* line_first) {
  if ((!ev && n) || !n_races || !line_first || (!races && capacity)) return MCKG_E_ARG;
  ref_t* order = (ref_t*)malloc(sizeof(ref_t) * (n ? n : 1));
  for (uint64_t i = 0; i < n; ++i) {
    order[i].ev = ev;
    order[i].i = i;
  }
  qsort(order, n, sizeof(ref_t), cmp_ts);
  bmap_t m = {0, 0, 0};
  mckg_grace* raw = NULL;
  uint64_t nraw = 0, rawcap = 0;
  for (uint64_t q = 0; q < n; ++q) {
    const mckg_gaccess* x = ev + order[q].i;
    uint64_t addr = MCKG_GA_ADDR(*x);
    uint32_t len = MCKG_GA_LEN(*x), bid = MCKG_GA_BID(*x);
    int w = (int)MCKG_GA_WRITE(*x);
    int32_t line = MCKG_GA_LINE(*x);
    int any = 0;
    for (uint64_t byte = addr; byte < addr + len; ++byte) {
      slot_t* s = bmap_get(&m, byte);
      int raced = w ? ((s->abid != 0xFFFFFFFFu && s->abid != bid) || s->amulti)
                    : ((s->wbid != 0xFFFFFFFFu && s->wbid != bid) || s->wmulti);
      if (raced) {
        if (nraw == rawcap) {
          rawcap = rawcap ? rawcap * 2 : 1024;
          raw = (mckg_grace*)realloc(raw, sizeof(mckg_grace) * rawcap);
        }
        raw[nraw].addr = byte;
        raw[nraw].line = line;
        raw[nraw].pad = 0;
        nraw++;
        any = 1;
      }
      if (s->abid == 0xFFFFFFFFu) s->abid = bid; else if (s->abid != bid) s->amulti = 1;
      if (w) {
        if (s->wbid == 0xFFFFFFFFu) s->wbid = bid; else if (s->wbid != bid) s->wmulti = 1;
      }
    }
    if (any && (uint32_t)line < MCKG_MAX_LINES) {
      uint64_t ts = tskey(x);
      if (ts < line_first[line]) line_first[line] = ts;
    }
  }
  qsort(raw, nraw, sizeof(mckg_grace), cmp_race);
  uint64_t u = 0;
  for (uint64_t i = 0; i < nraw; ++i)
    if (u == 0 || raw[i].addr != raw[u - 1].addr || raw[i].line != raw[u - 1].line) raw[u++] = raw[i];
  *n_races = u;
  for (uint64_t i = 0; i < u && i < capacity; ++i) races[i] = raw[i];
  free(raw);
  free(m.s);
  free(order);
  return u > capacity ? MCKG_E_OVERFLOW : MCKG_OK;
}
