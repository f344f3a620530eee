/* tracegen.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * CPU copy of the synthetic BASELINE config-3 trace (mckg_gen_c3 in
 * paper_1211_6193_b200/csrc/gen.cu).  The recipe follows SURVEY §8(d) C3 /
 * Appendix D probe6: per block, per epoch, per k, per tid, one 4-byte access
 * at slot tid*4+k of a 4 KiB shared object, line 100+k; 1% of accesses are
 * redirected to the slot of thread (tid+1)%256 (same epoch, same k); write
 * with p = 1/2.  A counter-based generator (splitmix64 of seed+index) replaces
 * the survey's sequential mt19937_64 so that every event can be generated
 * independently on the GPU.
 */
#include "oracle.h"

static inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void oracle_gen_c3(mckg_access* events, uint64_t* block_start, uint32_t blk0, uint32_t n_blocks,
                   uint64_t seed) {
  const uint64_t per = MCKG_C3_EVENTS_PER_BLOCK;
  for (uint32_t b = 0; b <= n_blocks; ++b) block_start[b] = (uint64_t)b * per;
  for (uint64_t r = 0; r < (uint64_t)n_blocks * per; ++r) {
    uint64_t i = (uint64_t)blk0 * per + r;  /* global event index */
    uint32_t j = (uint32_t)(i % per);
    uint32_t e = j / (MCKG_C3_THREADS * MCKG_C3_K);
    uint32_t k = (j / MCKG_C3_THREADS) % MCKG_C3_K;
    uint32_t tid = j % MCKG_C3_THREADS;
    uint64_t h = splitmix64(seed + i);
    int write = (int)(h & 1u);
    int redirect = ((h >> 32) % 10000u) < 100u;
    uint32_t t2 = redirect ? (tid + 1u) % MCKG_C3_THREADS : tid;
    uint32_t off = (t2 * 4u + k) * 4u;
    events[r] = mckg_make_access(off, 4u, write, tid, e, (int32_t)(100 + k), (uint32_t)i);
  }
}
