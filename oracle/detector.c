/* detector.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain-C restatement of the reference shared-memory race checker over the
 * mckg_access trace format, used as the parity checker for the CUDA detector.
 * It follows the reference line by line, per block:
 *
 *   - racecheck.cpp:24-32  per byte of [off, off+len): raced iff the shadow
 *                          list holds an entry of another thread where either
 *                          side is a write;
 *   - racecheck.cpp:33-41  a raced byte reports (obj, byte, line) once per run
 *                          (RaceState::reported, machine.hpp:91) and adds the
 *                          "Possible race ... <file>:<line>." diagnostic, which
 *                          addDiagnostic (machine.cpp:41-46) dedups by message,
 *                          i.e. per line -> we keep the first racing timestamp
 *                          per line;
 *   - racecheck.cpp:42-50  append (thread, kind) unless already present;
 *   - racecheck.cpp:54-73  clearEpoch erases the block's shadow when the block
 *                          passes a barrier Turnaround (device.cpp:168-178),
 *                          i.e. whenever the epoch field advances.
 *
 * Blocks are independent (shadow keys are per object, objects per block,
 * machine.hpp:86-94), so blocks may be partitioned over pthreads.
 */
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

typedef struct {
  uint16_t tid;
  uint8_t write;
} entry_t;

typedef struct {
  entry_t* e;
  uint32_t n, cap;
} elist_t;

typedef struct { /* (byte, line) set of one block, open addressing */
  uint64_t* keys;
  uint32_t cap, n;
} kset_t;

static int kset_insert(kset_t* s, uint64_t key) { /* 1 if new */
  if ((s->n + 1) * 2 > s->cap) {
    uint32_t ncap = s->cap ? s->cap * 2 : 64;
    uint64_t* nk = (uint64_t*)malloc(sizeof(uint64_t) * ncap);
    for (uint32_t i = 0; i < ncap; ++i) nk[i] = UINT64_MAX;
    for (uint32_t i = 0; i < s->cap; ++i)
      if (s->keys[i] != UINT64_MAX) {
        uint32_t h = (uint32_t)((s->keys[i] * 0x9E3779B97F4A7C15ull) >> 40) & (ncap - 1);
        while (nk[h] != UINT64_MAX) h = (h + 1) & (ncap - 1);
        nk[h] = s->keys[i];
      }
    free(s->keys);
    s->keys = nk;
    s->cap = ncap;
  }
  uint32_t h = (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> 40) & (s->cap - 1);
  while (s->keys[h] != UINT64_MAX) {
    if (s->keys[h] == key) return 0;
    h = (h + 1) & (s->cap - 1);
  }
  s->keys[h] = key;
  s->n++;
  return 1;
}

typedef struct {
  const mckg_trace* t;
  uint32_t b0, b1;
  mckg_race_triple* out;
  uint64_t n, cap;
  uint64_t* line_first;
  int err;
} job_t;

static void emit(job_t* j, uint32_t obj, uint32_t byte, int32_t line) {
  if (j->n == j->cap) {
    j->cap = j->cap ? j->cap * 2 : 1024;
    j->out = (mckg_race_triple*)realloc(j->out, sizeof(mckg_race_triple) * j->cap);
  }
  j->out[j->n].obj = obj;
  j->out[j->n].byte = byte;
  j->out[j->n].line = line;
  j->n++;
}

static void* run_job(void* arg) {
  job_t* j = (job_t*)arg;
  const mckg_trace* t = j->t;
  uint32_t sb = t->shmem_bytes;
  elist_t* shadow = (elist_t*)calloc(sb ? sb : 1, sizeof(elist_t));
  uint32_t* touched = (uint32_t*)malloc(sizeof(uint32_t) * (sb ? sb : 1));
  uint32_t ntouched = 0;
  kset_t rep = {0, 0, 0};
  for (uint32_t b = j->b0; b < j->b1 && !j->err; ++b) {
    uint32_t obj = t->obj_base + b;
    uint32_t bid = t->bid_base + b;
    uint64_t s = t->block_start[b], e = t->block_start[b + 1];
    uint32_t cur_epoch = 0;
    int have_epoch = 0;
    for (uint64_t i = s; i < e; ++i) {
      mckg_access a = t->events[i];
      uint32_t off = MCKG_ACC_OFF(a), len = MCKG_ACC_LEN(a), ep = MCKG_ACC_EPOCH(a);
      uint32_t tid = MCKG_ACC_TID(a);
      int w = (int)MCKG_ACC_WRITE(a);
      if (len == 0 || len > MCKG_MAX_LEN || off + len > sb) { j->err = MCKG_E_RANGE; break; }
      if (a.line < 0 || (uint32_t)a.line >= MCKG_MAX_LINES) { j->err = MCKG_E_RANGE; break; }
      if (!have_epoch || ep != cur_epoch) {
        if (have_epoch && ep < cur_epoch) { j->err = MCKG_E_ORDER; break; }
        /* clearEpoch (racecheck.cpp:54-73) */
        for (uint32_t q = 0; q < ntouched; ++q) shadow[touched[q]].n = 0;
        ntouched = 0;
        cur_epoch = ep;
        have_epoch = 1;
      }
      for (uint32_t by = off; by < off + len; ++by) {
        elist_t* L = &shadow[by];
        int raced = 0;
        for (uint32_t q = 0; q < L->n; ++q)
          if (L->e[q].tid != tid && (L->e[q].write || w)) { raced = 1; break; }
        if (raced) {
          uint64_t key = ((uint64_t)by << 32) | (uint32_t)a.line;
          if (kset_insert(&rep, key)) {
            emit(j, obj, by, a.line);
            uint64_t ts = mckg_ts_key(a.sweep, bid, tid);
            if (ts < j->line_first[a.line]) j->line_first[a.line] = ts;
          }
        }
        int present = 0;
        for (uint32_t q = 0; q < L->n; ++q)
          if (L->e[q].tid == tid && L->e[q].write == w) { present = 1; break; }
        if (!present) {
          if (L->n == 0) touched[ntouched++] = by;
          if (L->n == L->cap) {
            L->cap = L->cap ? L->cap * 2 : 4;
            L->e = (entry_t*)realloc(L->e, sizeof(entry_t) * L->cap);
          }
          L->e[L->n].tid = (uint16_t)tid;
          L->e[L->n].write = (uint8_t)w;
          L->n++;
        }
      }
    }
    /* block done: its shared object dies (device.cpp:204-216) */
    for (uint32_t q = 0; q < ntouched; ++q) shadow[touched[q]].n = 0;
    ntouched = 0;
    if (rep.cap) {
      for (uint32_t q = 0; q < rep.cap; ++q) rep.keys[q] = UINT64_MAX;
      rep.n = 0;
    }
  }
  for (uint32_t q = 0; q < sb; ++q) free(shadow[q].e);
  free(shadow);
  free(touched);
  free(rep.keys);
  return NULL;
}

int oracle_detect_shared(const mckg_trace* t, mckg_race_triple* triples, uint64_t capacity,
                         uint64_t* n_triples, uint64_t* line_first, int nthreads) {
  if (!t || !n_triples || !line_first || (!triples && capacity)) return MCKG_E_ARG;
  if (t->shmem_bytes > MCKG_MAX_OFF) return MCKG_E_RANGE;
  if (nthreads < 1) nthreads = 1;
  if ((uint32_t)nthreads > t->n_blocks) nthreads = t->n_blocks ? (int)t->n_blocks : 1;
  job_t* jobs = (job_t*)calloc((size_t)nthreads, sizeof(job_t));
  pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
  for (int k = 0; k < nthreads; ++k) {
    jobs[k].t = t;
    jobs[k].b0 = (uint32_t)((uint64_t)t->n_blocks * k / nthreads);
    jobs[k].b1 = (uint32_t)((uint64_t)t->n_blocks * (k + 1) / nthreads);
    jobs[k].line_first = (uint64_t*)malloc(sizeof(uint64_t) * MCKG_MAX_LINES);
    for (uint32_t l = 0; l < MCKG_MAX_LINES; ++l) jobs[k].line_first[l] = MCKG_TS_NONE;
  }
  if (nthreads == 1) {
    run_job(&jobs[0]);
  } else {
    for (int k = 0; k < nthreads; ++k) pthread_create(&th[k], NULL, run_job, &jobs[k]);
    for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
  }
  int err = MCKG_OK;
  uint64_t n = 0;
  for (int k = 0; k < nthreads; ++k) {
    if (jobs[k].err && !err) err = jobs[k].err;
    for (uint64_t q = 0; q < jobs[k].n; ++q, ++n)
      if (n < capacity) triples[n] = jobs[k].out[q];
    for (uint32_t l = 0; l < MCKG_MAX_LINES; ++l)
      if (jobs[k].line_first[l] < line_first[l]) line_first[l] = jobs[k].line_first[l];
    free(jobs[k].out);
    free(jobs[k].line_first);
  }
  *n_triples = n;
  free(jobs);
  free(th);
  if (!err && n > capacity) err = MCKG_E_OVERFLOW;
  return err;
}
