/*
 * mckg.h -- C ABI of the B200-native checker core (paper_1211_6193_b200).
 *
 * This is the drop-in boundary between host C++ (the mck:: API that mirrors
 * /root/reference/proj/include/minicudak/ headers) and the hand-written sm_100a
 * kernels in paper_1211_6193_b200/csrc/.  Plain pointers and sizes only; every
 * entry point returns an int status (0 = MCKG_OK) and never throws.
 *
 * Reference interfaces each entry point replaces (file:line in
 * /root/reference/proj):
 *
 *   mckg_detect_shared      Machine::recordAccess + Machine::clearEpoch
 *                           (src/racecheck.cpp:9-73, include/minicudak/machine.hpp:407-409),
 *                           batched over a per-block access trace; the
 *                           RaceState::reported set (machine.hpp:86-94) and the
 *                           first-detection order of the Race diagnostics
 *                           (addDiagnostic, src/machine.cpp:41-46).
 *   mckg_detect_shared_host the same, from HOST buffers (copies pipelined with
 *                           detection); the call a CPU-side user makes.
 *   mckg_sort_triples       iteration order of std::set<tuple<ObjectId,int64_t,int>>
 *                           RaceState::reported (machine.hpp:91).
 *   mckg_scan_stuck         the BarrierDeadlock part of Machine::scanStuck
 *                           (src/deadlock.cpp:12-34): per-block waiting /
 *                           finished-or-absent thread sets at quiescence.
 *   mckg_gen_c3             synthetic workload generator (BASELINE config 3);
 *                           not a reference interface.
 *   mck_run_source          mck::runFile / Machine::run end to end
 *                           (include/minicudak/driver.hpp:25-36,
 *                           machine.hpp:359-375): compile a CUDA-C program,
 *                           interpret the host thread, run every grid on the
 *                           B200 (K1 + fused race detector + K4), return the
 *                           RunResult as JSON.
 *   mck_disassemble         the step-exact IR of a program (debugging aid).
 *
 * Device pointers are CUDA device pointers on the current device; `stream` is
 * a cudaStream_t (NULL = legacy default stream).  All launches are
 * asynchronous on `stream` unless stated otherwise.
 */
#ifndef MCKG_H
#define MCKG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCKG_ABI_VERSION 1

/* ---- status codes ---- */
#define MCKG_OK 0
#define MCKG_E_ARG 1       /* invalid argument (null pointer, bad size)            */
#define MCKG_E_RANGE 2     /* a field exceeds the packed-record limits below       */
#define MCKG_E_CUDA 3      /* a CUDA runtime call failed (see mckg_last_error)     */
#define MCKG_E_OVERFLOW 4  /* output capacity exceeded; counts are still complete  */
#define MCKG_E_ORDER 5     /* trace not in per-block timestamp order (epoch went back) */

/* ---- limits of the packed 16-byte access record ---- */
#define MCKG_MAX_OFF (1u << 20)   /* byte offset inside a block's shared object  */
#define MCKG_MAX_LEN 8u           /* scalar access length (char/int/long/ptr)     */
#define MCKG_MAX_TID (1u << 11)   /* blockDim <= 2048 (reference default 1024)    */
#define MCKG_MAX_EPOCH (1u << 21) /* barrier episodes per thread                  */
#define MCKG_MAX_LINES 65536u     /* source lines 0..65535 (line-first table)     */
#define MCKG_MAX_BID (1u << 21)   /* global block index inside a timestamp key    */

/*
 * One shared-memory access event, exactly what Machine::recordAccess receives
 * (racecheck.cpp:9: object, offset, len, ThreadKey, AccessKind, SourceLoc),
 * with the object and block implied by the trace segment it sits in.
 *
 *   w0  bits  0..19  byte offset inside the block's shared object
 *       bits 20..23  length in bytes (1..8)
 *       bit  24      1 = write, 0 = read
 *   w1  bits  0..10  tid (threadIdx.x)
 *       bits 11..31  epoch = barrier episodes the accessing thread has passed
 *   line            SourceLoc::line of the access (the reported line)
 *   sweep           round-robin sweep of the access; the global timestamp of
 *                   an access is (sweep, gid, bid, tid)
 *
 * Within one block segment records are in timestamp order, so epochs are
 * non-decreasing (every epoch-e access precedes the Turnaround that clears
 * epoch e, device.cpp:168-178).
 */
typedef struct mckg_access {
  uint32_t w0;
  uint32_t w1;
  int32_t line;
  uint32_t sweep;
} mckg_access;

#define MCKG_ACC_OFF(a) ((a).w0 & 0xFFFFFu)
#define MCKG_ACC_LEN(a) (((a).w0 >> 20) & 0xFu)
#define MCKG_ACC_WRITE(a) (((a).w0 >> 24) & 1u)
#define MCKG_ACC_TID(a) ((a).w1 & 0x7FFu)
#define MCKG_ACC_EPOCH(a) ((a).w1 >> 11)

static inline mckg_access mckg_make_access(uint32_t off, uint32_t len, int write, uint32_t tid,
                                           uint32_t epoch, int32_t line, uint32_t sweep) {
  mckg_access a;
  a.w0 = (off & 0xFFFFFu) | ((len & 0xFu) << 20) | ((uint32_t)(write ? 1 : 0) << 24);
  a.w1 = (tid & 0x7FFu) | (epoch << 11);
  a.line = line;
  a.sweep = sweep;
  return a;
}

/* Timestamp key of an access: (sweep, bid, tid) packed so that unsigned
 * comparison is the reference's first-detection order within one grid. */
static inline uint64_t mckg_ts_key(uint32_t sweep, uint32_t bid, uint32_t tid) {
  return ((uint64_t)sweep << 32) | ((uint64_t)(bid & (MCKG_MAX_BID - 1)) << 11) | (tid & (MCKG_MAX_TID - 1));
}
#define MCKG_TS_NONE UINT64_MAX

/*
 * A block-segmented access trace: the events of simulated block b are
 * events[block_start[b] .. block_start[b+1]).  Block b owns the shared object
 * obj_base + b (spawnGrid allocates one DeviceShared object per block in bid
 * order, device.cpp:33-38) of shmem_bytes bytes.
 */
typedef struct mckg_trace {
  const mckg_access* events;
  const uint64_t* block_start; /* n_blocks + 1 entries, block_start[0] == 0 */
  uint64_t n_events;
  uint32_t n_blocks;
  uint32_t max_block_events;   /* upper bound on any block's event count (staging size) */
  uint32_t obj_base;
  uint32_t bid_base;           /* global bid of block 0 (shards of a grid) */
  uint32_t shmem_bytes;
  uint32_t gid;
} mckg_trace;

/* One element of RaceState::reported (machine.hpp:91). */
typedef struct mckg_race_triple {
  uint32_t obj;
  uint32_t byte;
  int32_t line;
} mckg_race_triple;

/*
 * Detector outputs (device memory, caller-owned).  `triples` receives each
 * reported (obj, byte, line) exactly once, grouped by block in no particular
 * block order (mckg_sort_triples orders them).  `line_first[l]` receives the
 * minimum timestamp key at which line l raced (MCKG_TS_NONE if never): the
 * Race diagnostics are the lines with a key, in increasing key order.
 * mckg_race_out_reset() initialises counters and the line table.
 */
typedef struct mckg_race_out {
  mckg_race_triple* triples;
  uint64_t capacity;
  unsigned long long* n_triples; /* device counter: total reported triples   */
  unsigned long long* line_first;/* device, MCKG_MAX_LINES entries            */
  uint32_t* status;              /* device: MCKG_ST_* bits                     */
} mckg_race_out;

/* status bits written by the detector */
#define MCKG_ST_OVERFLOW 1u  /* triples exceeded `capacity` (n_triples is still the full count) */
#define MCKG_ST_RANGE 2u     /* an event or block exceeded the record / staging limits; skipped */
#define MCKG_ST_ORDER 4u     /* a block's epochs decreased (trace not in timestamp order)       */
#define MCKG_ST_DUP 8u       /* the per-block dedup set overflowed: triples may repeat, run
                                mckg_sort_triples with n_unique to restore the exact set     */

/* Stats of the last launch made through this library on the calling thread. */
typedef struct mckg_launch_stats {
  uint32_t kernels;      /* kernels launched by the last entry point call */
  uint32_t grid;         /* CTAs of the main detector kernel              */
  uint32_t block;        /* threads per CTA                               */
  uint32_t smem_bytes;   /* dynamic shared memory per CTA                 */
} mckg_launch_stats;

int mckg_abi_version(void);
const char* mckg_last_error(void);
int mckg_device_count(int* n);
int mckg_get_launch_stats(mckg_launch_stats* out);
/* Test switches that force one route of a detector, so the tests cover every
 * route at small sizes (initial value: the MCKG_DEBUG environment variable,
 * read once at load).  Bits: 32 = K2's general (TMA) kernel for every block
 * instead of the warp-per-block fast path; 128 = K6's bucket pipeline in
 * sparse (hashed) mode; 256 = K6 never takes the tile path; 512 = K6 takes
 * the tile path at any size (default: from 2^20 records); 1024 = the tile
 * path's pass 1 re-reads every tile (default: only tiles whose in-window
 * records come from two or more blocks; the others from pass 0's codes). */
void mckg_set_debug(uint32_t flags);

int mckg_race_out_reset(const mckg_race_out* out, void* stream);
int mckg_detect_shared(const mckg_trace* trace, const mckg_race_out* out, void* stream);

/* Host-buffer entry point: trace->events and trace->block_start are HOST
 * pointers (pinned or pageable); the events are streamed to the device in
 * chunks overlapped with detection.  Results are copied back to host:
 * triples_host (capacity entries; may be NULL when capacity == 0),
 * *n_triples_host, line_first_host (MCKG_MAX_LINES entries), *status_host.
 * Synchronous. */
int mckg_detect_shared_host(const mckg_trace* trace, mckg_race_triple* triples_host,
                            uint64_t capacity, uint64_t* n_triples_host,
                            uint64_t* line_first_host, uint32_t* status_host);

/* Sort n device triples into std::set order (obj, byte, line); in place.
 * obj must lie in [obj_base, obj_base + 2^22).  When n_unique (a device
 * counter) is non-NULL, duplicates are removed and the unique count written
 * there (needed only after MCKG_ST_DUP). */
int mckg_sort_triples(mckg_race_triple* triples, uint64_t n, uint32_t obj_base,
                      unsigned long long* n_unique, void* stream);

/*
 * Deadlock classification at quiescence (deadlock.cpp:12-34).  arrivals[b *
 * block_dim + t] = number of __syncthreads*() arrivals of thread t of block b
 * when nothing can move (finished / halted threads keep their final count, a
 * thread blocked at a barrier counts the barrier it waits at).  A block is
 * deadlocked iff its counts differ; its waiting threads are those above the
 * block minimum (the token protocol of device.cpp:111-200 can
 * never pass a finished thread).  Outputs (device):
 *   waiting_mask  n_blocks * ceil(block_dim/32) words, bit t = thread t waits
 *   dl_bids       ascending bids (bid_base + b) of deadlocked blocks
 *   n_dl          device counter of deadlocked blocks
 */
int mckg_scan_stuck(const uint32_t* arrivals, uint32_t n_blocks, uint32_t block_dim,
                    uint32_t bid_base, uint32_t* waiting_mask, uint32_t* dl_bids,
                    uint32_t* n_dl, void* stream);

/*
 * Synthetic BASELINE config-3 trace, generated on the device: blocks
 * [blk0, blk0 + n_blocks) of the 2^20-block, 1024-event-per-block layout
 * (256 threads x 2 epochs x 2 accesses of 4 bytes at slot tid*4+k; 1% of the
 * accesses redirected to thread (tid+1)%256's slot; write with p = 1/2;
 * line 100+k; sweep = global event index).  Identical, record for record, to
 * oracle/tracegen.c (the CPU copy used by the tests).  events must hold
 * n_blocks*1024 records; block_start n_blocks+1 entries (relative to events).
 */
int mckg_gen_c3(mckg_access* events, uint64_t* block_start, uint32_t blk0, uint32_t n_blocks,
                uint64_t seed, void* stream);

/* ---- cross-block global-memory races (BASELINE config 5) ----
 *
 * NOT a reference interface: the reference checks DeviceShared objects only
 * (memory.cpp:142-143, 240-241).  The extension applies the racecheck.cpp:24-32
 * rule to global memory with "thread" replaced by "block": within one grid
 * (the kernel-end barrier separates grids) an access X to byte b races iff an
 * EARLIER access to b, in (sweep, bid, tid) order, came from another BLOCK and
 * X or it writes.  Reported once per (byte, line); the "Possible race on
 * global device memory detected at <file>:<line>." diagnostic of a line sits
 * at its first racing access.  Parity is unpinned (no reference semantics);
 * the checker is oracle/global_detector.c.
 *
 *   a     = addr:40 | len:4 | write:1 | tid:11 | line & 0xFF
 *   sweep = round-robin sweep of the access
 *   b     = bid:24 | line >> 8
 */
typedef struct mckg_gaccess {
  uint64_t a;
  uint32_t sweep;
  uint32_t b;
} mckg_gaccess;

#define MCKG_GA_ADDR(r) ((r).a & 0xFFFFFFFFFFull)
#define MCKG_GA_LEN(r) ((uint32_t)(((r).a >> 40) & 0xFu))
#define MCKG_GA_WRITE(r) ((uint32_t)(((r).a >> 44) & 1u))
#define MCKG_GA_TID(r) ((uint32_t)(((r).a >> 45) & 0x7FFu))
#define MCKG_GA_LINE(r) ((int32_t)((((r).b >> 24) << 8) | (uint32_t)(((r).a >> 56) & 0xFFu)))
#define MCKG_GA_BID(r) ((r).b & 0xFFFFFFu)

static inline mckg_gaccess mckg_make_gaccess(uint64_t addr, uint32_t len, int write, uint32_t tid,
                                             uint32_t bid, int32_t line, uint32_t sweep) {
  mckg_gaccess g;
  g.a = (addr & 0xFFFFFFFFFFull) | ((uint64_t)(len & 0xFu) << 40) | ((uint64_t)(write ? 1 : 0) << 44) |
        ((uint64_t)(tid & 0x7FFu) << 45) | ((uint64_t)((uint32_t)line & 0xFFu) << 56);
  g.sweep = sweep;
  g.b = (bid & 0xFFFFFFu) | ((((uint32_t)line >> 8) & 0xFFu) << 24);
  return g;
}

/* Timestamp key of a global access: sweep:32 | bid:21 | tid:11 (as mckg_ts_key);
 * a global trace's bids must stay below MCKG_MAX_BID. */

/* One reported (byte address, line) pair. */
typedef struct mckg_grace {
  uint64_t addr;
  int32_t line;
  int32_t pad;
} mckg_grace;

/* Synthetic BASELINE config-5 records of blocks [blk0, blk0 + n_blocks) of an
 * n_total-block grid: MCKG_C5_EVENTS_PER_BLOCK 4-byte accesses per block at
 * 8-byte-aligned addresses of the block's own 64 KiB range (slot tid*16 + k);
 * 1% go to the same slot of block (b + 1) % n_total; write with p = 1/2; line
 * 200 + k % 4; sweep = k.  Identical to oracle_gen_c5. */
int mckg_gen_c5(mckg_gaccess* events, uint32_t blk0, uint32_t n_blocks, uint32_t n_total, uint64_t seed,
                void* stream);

/* Stable partition of n records by owner rank (owner = addr * n_ranks / addr_space,
 * address-range partition): out[] holds the records grouped by rank, counts[r]
 * (device, n_ranks entries) the group sizes. */
int mckg_partition_global(const mckg_gaccess* events, uint64_t n, uint32_t n_ranks, uint64_t addr_space,
                          mckg_gaccess* out, uint64_t* counts, void* stream);

/* Detects cross-block races among n records whose addresses lie in
 * [addr_lo, addr_lo + 2^35).  Outputs (device, caller-owned): races[capacity]
 * (unordered, unique per (byte, line)), *n_races (device counter; reset by the
 * call), line_first[MCKG_MAX_LINES] (min timestamp key per line; reset by the
 * caller with mckg_race_out_reset semantics), *status.  Scratch is allocated
 * on `stream`. */
int mckg_detect_global(const mckg_gaccess* events, uint64_t n, uint64_t addr_lo, mckg_grace* races,
                       uint64_t capacity, unsigned long long* n_races, unsigned long long* line_first,
                       uint32_t* status, void* stream);

/* ---- multi-GPU (one process per GPU) ----
 * An NCCL communicator owned by the library: `id` from mckg_comm_id() on
 * rank 0, broadcast by the launcher; `device` the CUDA ordinal of this rank. */
typedef struct mckg_comm mckg_comm;
int mckg_comm_init(const uint8_t id[128], int rank, int world, int device, mckg_comm** out);
void mckg_comm_destroy(mckg_comm* comm);

/* C3 sharded by blocks: mckg_detect_shared on this rank's shard, then an
 * all-reduce(MIN) of out->line_first, so every rank holds the Race diagnostic
 * order of the whole grid.  Triples stay with the rank that found them (the
 * shards own disjoint shared objects). */
int mckg_detect_shared_mgpu(mckg_comm* comm, const mckg_trace* shard, const mckg_race_out* out, void* stream);

/* C5: the global-race exchange in the library -- partition this rank's
 * records by owner (rank r owns addresses [r*A/P, (r+1)*A/P), A = addr_space),
 * count all-gather, grouped ncclSend/ncclRecv of the records, then
 * mckg_detect_global on the owned range and an all-reduce(MIN) of line_first
 * (reset by the caller beforehand).  races / n_races: this rank's (byte,
 * line) pairs, disjoint across ranks. */
int mckg_detect_global_mgpu(mckg_comm* comm, const mckg_gaccess* events, uint64_t n, uint64_t addr_space,
                            mckg_grace* races, uint64_t capacity, unsigned long long* n_races,
                            unsigned long long* line_first, uint32_t* status, void* stream);

#define MCKG_C5_EVENTS_PER_BLOCK 4096u
#define MCKG_C5_RANGE 65536u
#define MCKG_C5_SEED 0x12116193ull

/* ---- whole-program checking (host + B200 grid engine) ---- */
typedef struct mck_run_opts {
  uint64_t step_limit;        /* 0 = reference default 50,000,000 (machine.hpp:313) */
  uint64_t seed;              /* RunOptions::seed                                     */
  int32_t race_check;         /* RunOptions::raceCheck                                 */
  int32_t round_robin;        /* 1 = SchedulePolicy::RoundRobin (the engine's schedule) */
  int32_t device;             /* CUDA device ordinal                                    */
  int32_t max_threads_per_block; /* ArchParams::maxThreadsPerBlock, 0 = 1024           */
  int32_t n_devices;          /* > 0: split every grid over devices[0 .. n_devices)    */
  int32_t devices[8];         /* CUDA ordinals; repeating one = virtual devices (tests) */
  int32_t rank;               /* world > 1: one process per GPU; this rank runs blocks  */
  int32_t world;              /*   [gridDim*rank/world, gridDim*(rank+1)/world)          */
  uint8_t comm_id[128];       /* from mckg_comm_id() on rank 0, broadcast by the caller  */
  /* optional host transport instead of NCCL (ranks sharing a GPU, tests):
   * gather n bytes from every rank into recv[world*n] in rank order, 0 = ok */
  int (*allgather)(void* ctx, const void* send, uint64_t n, void* recv);
  void* allgather_ctx;
  int32_t trace;              /* RunOptions::trace: JSON "trace" = the --trace lines  */
  int32_t global_race_check;  /* RunOptions::globalRaceCheck       */
} mck_run_opts;

/* A fresh NCCL communicator id for mck_run_opts.comm_id. */
int mckg_comm_id(uint8_t out[128]);

/* JSON keys: exit, output, steps, stuck, main_return, diags[{cat,sev,msg,line}],
 * stuck_reports[{kind,gid,bid,waiting,missing,reason}], report_text,
 * reported[[obj,byte,line]], stats{...}, engine_error; or frontend_error.
 * *json is malloc'ed: release with mck_free. */
int mck_run_source(const char* src, const char* filename, const mck_run_opts* opts, char** json);

/* ---- whole-program checking, result records (no JSON) ----
 * mck_run: compileSource + Machine(prog, opts).run() (program.hpp:59-60,
 * machine.hpp:359/375; the reference driver's path, driver.cpp:87-161).  The
 * RunResult stays in an opaque handle; strings and arrays handed out by the
 * accessors live until mck_result_free.  A frontend failure (LexError /
 * ParseError / SemanticError, diagnostics.hpp:35-56) is not an ABI error: the
 * handle reports it in the summary (frontend_stage non-empty, exit_code 2). */
typedef struct mck_result mck_result;

typedef struct mck_summary {
  int32_t exit_code;          /* RunResult::exitCode (2 = frontend error)          */
  int32_t stuck;              /* RunResult::stuck                                   */
  int32_t has_main_return;    /* RunResult::mainReturn engaged                      */
  int32_t frontend_line;      /* frontend failure: its line                         */
  int64_t main_return;
  uint64_t steps;             /* RunResult::steps                                   */
  uint64_t n_diags;           /* RunResult::diagnostics, report order               */
  uint64_t n_stuck;           /* RunResult::stuckReports                            */
  uint64_t n_reported;        /* RaceState::reported triples, std::set order        */
  uint64_t n_trace;           /* --trace lines                                      */
  uint64_t output_bytes;
  const char* output;         /* RunResult::output (NUL-terminated)                 */
  const char* engine_error;   /* "" unless the engine abandoned the run             */
  const char* frontend_stage; /* "" or "lex" / "parse" / "semantic"                 */
  const char* frontend_message;
  const char* report_text;    /* formatStuckReports(stuckReports) (machine.hpp:449) */
  const char* engine_note;    /* RunResult::engineNote: "" unless the run departs from the
                                 reference (a non-round-robin schedule requested; a grid with
                                 cross-block global conflicts, whose values follow block order) */
} mck_summary;

typedef struct mck_diag_rec {
  int32_t category;           /* DiagCategory: 0 race, 1 deadlock, 2 memBoundary,
                                 3 undefinedBehavior, 4 apiError                     */
  int32_t severity;           /* 0 error, 1 warning                                 */
  int32_t line;               /* Diagnostic::loc.line                               */
  int32_t pad;
  uint64_t sweep;             /* round-robin sweep of the first occurrence          */
  const char* message;        /* Diagnostic::message                                */
} mck_diag_rec;

typedef struct mck_stuck_rec {
  int32_t kind;               /* 0 BarrierDeadlock, 1 HostHang, 2 StreamStall       */
  uint32_t gid;
  int32_t bid;
  uint32_t sid;
  uint64_t n_waiting, n_missing;
  const int32_t* waiting;     /* waitingTids, ascending                             */
  const int32_t* missing;     /* missingTids, ascending                             */
  const char* reason;
  const char* item;
} mck_stuck_rec;

int mck_run(const char* src, const char* filename, const mck_run_opts* opts, mck_result** out);
int mck_result_summary(const mck_result* r, mck_summary* out);
int mck_result_diag(const mck_result* r, uint64_t i, mck_diag_rec* out);
int mck_result_stuck(const mck_result* r, uint64_t i, mck_stuck_rec* out);
/* triples [first, first + count) of RaceState::reported (machine.hpp:91) */
int mck_result_reported(const mck_result* r, uint64_t first, uint64_t count, mckg_race_triple* out);
const char* mck_result_trace(const mck_result* r, uint64_t i);
/* the engine's counters of the run (mck::EngineStats; not a reference
 * interface: what bench.py and the tests read instead of parsing JSON) */
typedef struct mck_run_stats {
  uint64_t host_steps, device_steps, barrier_rules, dispatches, shared_events, grids, sweeps;
  double grid_ms;             /* device time of the grid kernels (CUDA events)      */
  uint32_t kernel_launches, pad;
  uint64_t block_sweeps, solo_sweeps, block_cycles, solo_cycles;
} mck_run_stats;
int mck_result_stats(const mck_result* r, mck_run_stats* out);
void mck_result_free(mck_result* r);
/* oracleRace (oracle.hpp:34): every interleaving of the shared accesses of a
 * small program's grid, explored on the GPU. */
typedef struct mck_oracle_result {
  int32_t oracle_race;     /* ground truth: a conflicting pair with no barrier between */
  int32_t detector_race;   /* the shadow detector reported on some schedule            */
  int32_t aborted;         /* a bound was hit (error says which)                         */
  int32_t frontend_error;  /* the program did not compile (error holds the message)      */
  uint64_t interleavings;
  char error[256];
} mck_oracle_result;
int mck_oracle(const char* src, const char* filename, uint64_t max_interleavings, int32_t max_threads,
               int32_t max_accesses_per_thread, mck_oracle_result* out);
int mck_disassemble(const char* src, const char* filename, char** text);
void mck_free(char* p);

#define MCKG_C3_THREADS 256u
#define MCKG_C3_EPOCHS 2u
#define MCKG_C3_K 2u
#define MCKG_C3_EVENTS_PER_BLOCK (MCKG_C3_THREADS * MCKG_C3_EPOCHS * MCKG_C3_K)
#define MCKG_C3_SHMEM 4096u
#define MCKG_C3_SEED 0x12116193ull

#ifdef __cplusplus
}
#endif
#endif /* MCKG_H */
