// engine.hpp -- interface between the host machine (host/machine.cpp) and the
// device grid engine (csrc/interp.cu, the K1 thread-stepping interpreter with
// the fused shared-memory race detector and the K4 barrier-deadlock scan).
//
// The host dispatches a whole grid at the reference's StreamDispatch point
// (streams.cpp:42-45 -> spawnGrid, device.cpp:19-66); the engine runs every
// simulated block to completion or deadlock under the round-robin schedule
// and returns step counts, the block outcomes, timestamped diagnostics and
// the reported race triples.
#pragma once
#include <array>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../csrc/core.cuh"
#include "program.hpp"

namespace mckb {

// Per-byte metadata of every memory object (host and device):
constexpr uint8_t META_DEF = 1;  // byte defined (MemByte::defined, machine.hpp:33-37)
constexpr uint8_t META_PTR = 2;  // a pointer slot starts here (MemObject::ptrs, machine.hpp:45)
constexpr uint8_t META_DIRTY = 4;
constexpr int TRACE_EPISODES = 64;  // --trace: barrier episodes recorded per block  // written by the running grid (replica merge; cleared after)

// A device-global object as the engine sees it.
struct DevObjInfo {
  uint32_t id;
  int64_t size;
  uint64_t base;  // byte offset in the device arena
  bool live;
  int name;       // diagnostic name handle echoed back in DevDiag::name
};

struct GridSpec {
  const Program* prog = nullptr;
  int kernel = -1;
  int64_t gridDim = 1, blockDim = 1, shmemBytes = 0;
  uint32_t gid = 0;
  std::vector<mck_core::Val> args;  // converted to the parameter types
  uint64_t spawnSweep = 0;          // sweep of the dispatch; first steps at +1
  uint32_t sharedBase = 0;          // object id of block 0's shared array
  uint32_t nextId = 0;              // ids >= nextId (and not private) are invalid
  bool raceCheck = true;
  int64_t warpSize = 32;
  uint64_t stepBudget = ~0ull;      // steps left before the run's step limit
  std::vector<DevObjInfo> objects;  // every device-global object, ascending id
  std::vector<uint32_t> globalIds;  // object id of every TU global (host or device)
  // shared arrays of earlier grids (for memBoundary messages): (first id, count, gid)
  std::vector<std::array<uint32_t, 3>> sharedRanges;
  bool trace = false;               // record barrier arrivals (GridResult::arrivals)
  bool globalRaceCheck = false;     // log global accesses, run K6 on them after the grid
  // without globalRaceCheck: the same log and K6 pass, reporting only whether
  // the grid had cross-block global conflicts (GridResult::globalConflicts)
  bool conflictProbe = false;
  // ... and keep the grid's write history (another stream exists, so a
  // copy may read the grid's bytes while it is in flight)
  bool wantHistory = false;
};

struct DevDiag {
  uint64_t key;      // (local sweep:26 | bid:26 | tid:10 | sub:2)
  int code;          // MCK_D_*
  int line;
  int64_t p[4];
  int name;          // string id or -1
};

struct GridResult {
  uint64_t deviceSteps = 0;
  uint64_t barrierRules = 0;
  uint64_t allocs = 0;          // device-side object allocations (locals + call params)
  uint64_t sharedEvents = 0;
  uint64_t sweeps = 0, soloSweeps = 0;  // block-sweeps executed (diagnostics)
  uint64_t blockCycles = 0, soloCycles = 0;
  uint32_t duration = 0;        // local sweep of the last device step (complete grids)
  bool deadlocked = false;
  struct Stuck {
    uint32_t bid;
    std::vector<int> waiting;
  };
  std::vector<Stuck> stuck;     // ascending bid
  std::vector<DevDiag> diags;
  std::vector<std::array<int64_t, 3>> reported;  // (obj, byte, line)
  double ms = 0;
  uint32_t launches = 0;
  std::string error;            // engine limitation hit: run abandoned
  bool stepLimitHit = false;    // the grid ran out of the run's step budget
  bool globalConflicts = false; // conflictProbe: blocks touched a global byte, one of them writing
  // conflictProbe / globalRaceCheck: per device-global object the grid touched,
  // {object id, read lo, read hi, write lo, write hi} (byte offsets, hi
  // exclusive; lo > hi: none) -- the host checks stream operations issued
  // while the grid is in flight against it
  std::vector<std::array<int64_t, 5>> footprint;
  // ... and every global write of the grid with what it overwrote, so that a
  // copy on another stream reading the grid's bytes mid-flight sees them as
  // of its sweep (empty when any write stored or erased a pointer slot)
  struct Write {
    uint32_t obj;
    uint32_t lsweep, bid, tid;  // local sweep (global = dispatch sweep + lsweep)
    int64_t off;
    uint32_t len;
    uint8_t oldB[8], oldM[8], newB[8];
  };
  std::vector<Write> writes;
  // trace mode: per block, completed barrier episodes, and the local arrival
  // sweep + 1 of every thread in its first TRACE_EPISODES episodes (0 = none)
  std::vector<uint32_t> episodes;   // [gridDim]
  std::vector<uint32_t> arrivals;   // [gridDim][TRACE_EPISODES][blockDim]
};

// The exhaustive-interleaving oracle over one grid (oracle.hpp:10-34).
struct OracleSpec {
  uint64_t maxInterleavings = 1'000'000;
  int maxAccessesPerThread = 8;
};
struct OracleOut {
  bool oracleRace = false, detectorRace = false, aborted = false;
  uint64_t interleavings = 0;
  std::string error;
};

class DeviceEngine {
 public:
  virtual ~DeviceEngine() = default;
  virtual bool hasDevice() const = 0;
  virtual uint64_t alloc(int64_t size) = 0;
  virtual void write(uint64_t base, const uint8_t* bytes, const uint8_t* meta, int64_t n) = 0;
  virtual void read(uint64_t base, uint8_t* bytes, uint8_t* meta, int64_t n) = 0;
  virtual void copy(uint64_t dst, uint64_t src, int64_t n) = 0;
  virtual void fill(uint64_t base, uint8_t v, uint8_t meta, int64_t n) = 0;
  virtual bool runGrid(const GridSpec& spec, GridResult& out) = 0;
  // explores every interleaving of the grid's visible steps; false: error set
  virtual bool exploreGrid(const GridSpec& spec, const OracleSpec& o, OracleOut& out) {
    (void)spec;
    (void)o;
    out.error = "no CUDA device: the oracle explores on the GPU";
    return false;
  }
};

// Rank sharding (one process per GPU): rank r runs blocks
// [gridDim*r/world, gridDim*(r+1)/world) of every grid; the written global
// bytes and the partial results are combined over NCCL after each grid.
struct EngineComm {
  int rank = 0, world = 1;
  std::array<uint8_t, 128> id{};  // ncclUniqueId made by rank 0
  // host transport instead of NCCL (ranks sharing one GPU, gloo tests):
  // gather n bytes from every rank into recv[world * n], rank order; 0 = ok
  int (*allgather)(void* ctx, const void* send, uint64_t n, void* recv) = nullptr;
  void* ctx = nullptr;
};

// The B200 engine over one or more devices (a grid's blocks are split into
// contiguous ranges, one per device; device-global memory is replicated and
// merged after each grid).  A device may be listed twice ("virtual devices").
// Returns nullptr (with `why`) when no CUDA device is usable.
std::unique_ptr<DeviceEngine> makeCudaEngine(const std::vector<int>& devices, const EngineComm& comm,
                                             std::string& why);
// a fresh ncclUniqueId (rank 0 makes it; the launcher broadcasts it)
bool makeCommId(std::array<uint8_t, 128>& id, std::string& why);
// Storage-only stand-in used when no GPU is present: device allocations and
// copies work, launching a grid fails loudly (there is no CPU execution path).
std::unique_ptr<DeviceEngine> makeStorageOnlyEngine(const std::string& why);

}  // namespace mckb
