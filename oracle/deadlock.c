/* deadlock.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Restatement of the BarrierDeadlock classification of Machine::scanStuck
 * (deadlock.cpp:12-34) from per-thread barrier arrival counts at quiescence.
 * In the reference a thread waiting at a barrier keeps `barrier.waiting`;
 * finished or halted threads are erased from cfg_.device (machine.cpp:460-463)
 * so the token (device.cpp:111-141) can never pass them.  At quiescence the
 * block's completed episodes are m = min_t c_t; a thread waits iff c_t > m,
 * and the report lists waiting tids ascending and the complement in
 * 0..blockDim-1 as finished-or-absent (deadlock.cpp:19-33).  Blocks are
 * reported in ascending (gid, bid) order (the std::map walk at deadlock.cpp:15-18).
 */
#include <string.h>
#include "oracle.h"

int oracle_scan_stuck(const uint32_t* arrivals, uint32_t n_blocks, uint32_t block_dim,
                      uint32_t bid_base, uint32_t* waiting_mask, uint32_t* dl_bids,
                      uint32_t* n_dl) {
  if (!arrivals || !waiting_mask || !dl_bids || !n_dl || block_dim == 0) return MCKG_E_ARG;
  uint32_t words = (block_dim + 31) / 32;
  uint32_t nd = 0;
  for (uint32_t b = 0; b < n_blocks; ++b) {
    const uint32_t* c = arrivals + (uint64_t)b * block_dim;
    uint32_t m = c[0];
    for (uint32_t t = 1; t < block_dim; ++t)
      if (c[t] < m) m = c[t];
    uint32_t* wm = waiting_mask + (uint64_t)b * words;
    memset(wm, 0, sizeof(uint32_t) * words);
    int any = 0;
    for (uint32_t t = 0; t < block_dim; ++t)
      if (c[t] > m) {
        wm[t / 32] |= 1u << (t % 32);
        any = 1;
      }
    if (any) dl_bids[nd++] = bid_base + b;
  }
  *n_dl = nd;
  return MCKG_OK;
}
