/* oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement ("port") of the reference checker's hot path, used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * checker of the CUDA path.  Never linked or called by the product
 * (paper_1211_6193_b200/).  Parity of this restatement is pinned against the
 * reference itself (oracle/_ref/libmckref.so, built from /root/reference by
 * oracle/Makefile) and the committed fixtures in tests/golden/.
 */
#ifndef MCK_ORACLE_H
#define MCK_ORACLE_H
#include <stdint.h>
#include "mckg.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Shared-memory race detection over a block-segmented trace, following
 * Machine::recordAccess / clearEpoch (racecheck.cpp:9-73) block by block.
 * Host pointers.  triples: capacity entries, filled in discovery order.
 * line_first: MCKG_MAX_LINES entries, set to the min timestamp key per raced
 * line (caller initialises to MCKG_TS_NONE).  nthreads > 1 partitions blocks.
 * Returns MCKG_OK or an MCKG_E_* code. */
int oracle_detect_shared(const mckg_trace* t, mckg_race_triple* triples, uint64_t capacity,
                         uint64_t* n_triples, uint64_t* line_first, int nthreads);

/* Deadlock classification (deadlock.cpp:12-34) from per-thread arrival counts.
 * waiting_mask: n_blocks*ceil(block_dim/32) words; dl_bids ascending. */
int oracle_scan_stuck(const uint32_t* arrivals, uint32_t n_blocks, uint32_t block_dim,
                      uint32_t bid_base, uint32_t* waiting_mask, uint32_t* dl_bids,
                      uint32_t* n_dl);

/* CPU copy of mckg_gen_c3 (record-for-record identical). */
void oracle_gen_c3(mckg_access* events, uint64_t* block_start, uint32_t blk0, uint32_t n_blocks,
                   uint64_t seed);

/* Cross-block global races (parity unpinned): see
 * oracle/global_detector.c.  races sorted by (addr, line). */
int oracle_detect_global(const mckg_gaccess* ev, uint64_t n, mckg_grace* races, uint64_t capacity,
                         uint64_t* n_races, uint64_t* line_first);
void oracle_gen_c5(mckg_gaccess* ev, uint32_t blk0, uint32_t n_blocks, uint32_t n_total, uint64_t seed);

#ifdef __cplusplus
}
#endif
#endif
