// mck/checker.hpp -- public C++ API of the B200 checker, source-compatible
// with the reference's proj/include/minicudak headers for the program-load /
// launch-configuration / check / report path:
//
//   compileSource(src, file)        program.hpp:59-60  (throws LexError /
//                                   ParseError / SemanticError)
//   RunOptions / ArchParams         machine.hpp:300-316
//   Machine(prog, opts).run()       machine.hpp:357-375
//   scanStuck, hooks                machine.hpp:378, 384-388
//   recordAccess / clearEpoch       machine.hpp:407-409 (batched on the K2 kernel)
//   oracleRace                      oracle.hpp:34 (explored on the GPU)
//   RunResult / StuckReport         machine.hpp:318-338
//   Diagnostic / DiagCategory       diagnostics.hpp:10-31
//   formatStuckReports              machine.hpp:449
//   runFile(CliOptions)             driver.hpp:13-36
//
// Device grids run on the B200 (K1 thread-stepping interpreter, csrc/interp.cu)
// under the round-robin schedule; the host thread is interpreted on the CPU
// with the same step-exact IR.  There is no CPU execution path for device
// code: a launch without a CUDA device is an error.
#pragma once
#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <string>
#include <vector>

namespace mckb {
struct Program;
}

namespace mck {

struct SourceLoc {
  int line = 0;
  int col = 0;
  bool valid() const { return line > 0; }
  bool operator==(const SourceLoc& o) const { return line == o.line && col == o.col; }
};

enum class Severity { Error, Warning };
enum class DiagCategory { Race, Deadlock, MemBoundary, UndefinedBehavior, ApiError };
const char* categoryName(DiagCategory c);

struct Diagnostic {
  Severity severity = Severity::Error;
  DiagCategory category = DiagCategory::UndefinedBehavior;
  std::string message;
  SourceLoc loc;
  uint64_t sweep = 0;  // B200 extension: round-robin sweep of the first occurrence
};

struct FrontendError {
  std::string stage;  // "lex", "parse", "semantic"
  SourceLoc loc;
  std::string message;
};

// The typed frontend failures compileSource throws (diagnostics.hpp:41-56).
struct LexError : FrontendError {
  LexError(SourceLoc l, std::string m) : FrontendError{"lex", l, std::move(m)} {}
};

struct ParseError : FrontendError {
  ParseError(SourceLoc l, std::string expected, std::string found)
      : FrontendError{"parse", l, "expected " + expected + ", found " + found},
        expected(std::move(expected)),
        found(std::move(found)) {}
  std::string expected;
  std::string found;
};

struct SemanticError : FrontendError {
  SemanticError(SourceLoc l, std::string m) : FrontendError{"semantic", l, std::move(m)} {}
};

// ----- identities and memory (machine.hpp:19-75, value.hpp:10-20) -----
using ObjectId = uint32_t;
using GridId = uint32_t;
using StreamId = uint32_t;
using EventId = uint32_t;

struct ThreadKey {
  GridId gid = 0;  // 0 = host
  int bid = 0;
  int tid = 0;
  bool isHost() const { return gid == 0; }
  bool operator==(const ThreadKey& o) const { return gid == o.gid && bid == o.bid && tid == o.tid; }
  bool operator!=(const ThreadKey& o) const { return !(*this == o); }
  bool operator<(const ThreadKey& o) const {
    if (gid != o.gid) return gid < o.gid;
    if (bid != o.bid) return bid < o.bid;
    return tid < o.tid;
  }
};

enum class AccessKind { Read, Write };
enum class SpaceKind { Host, DeviceGlobal, DeviceShared, Local };

struct MemSpace {
  SpaceKind kind = SpaceKind::Host;
  GridId gid = 0;  // DeviceShared only
  int bid = 0;
  static MemSpace host() { return {SpaceKind::Host, 0, 0}; }
  static MemSpace deviceGlobal() { return {SpaceKind::DeviceGlobal, 0, 0}; }
  static MemSpace deviceShared(GridId g, int b) { return {SpaceKind::DeviceShared, g, b}; }
  bool operator==(const MemSpace& o) const { return kind == o.kind && gid == o.gid && bid == o.bid; }
};

struct Location {
  ObjectId object = 0;
  int64_t offset = 0;
};

// The part of MemObject (machine.hpp:39-55) the race checker reads.
struct MemObject {
  ObjectId id = 0;
  MemSpace space;
  int64_t size = 0;
  std::string name;
  bool live = true;
};

// Runtime-API ids (program.hpp:14-37), the onApiCall argument.
enum class ApiId {
  Malloc, Free, Memcpy, MemcpyAsync, Memset, DeviceSynchronize, StreamCreate, StreamDestroy,
  StreamSynchronize, StreamQuery, StreamWaitEvent, EventCreate, EventDestroy, EventRecord,
  EventSynchronize, EventQuery, EventElapsedTime, GetLastError, GetErrorString, DeviceGetAttribute,
  DriverGetVersion, RuntimeGetVersion,
};
const char* apiName(ApiId id);

// Observer record of the memory-access hook (machine.hpp:340-350).
struct MemAccessInfo {
  ThreadKey accessor;
  AccessKind kind = AccessKind::Read;
  ObjectId object = 0;
  MemSpace space;
  int64_t offset = 0;
  int64_t len = 0;
  bool allowed = true;
  SourceLoc loc;
};

// The lowered program (opaque; shared, immutable).
using Program = mckb::Program;
std::shared_ptr<const Program> compileSource(const std::string& source, const std::string& filename);

enum class SchedulePolicy { SeededRandom, RoundRobin, Exhaustive };

struct ArchParams {
  int64_t warpSize = 32;
  int64_t computeCapabilityMajor = 2;
  int64_t computeCapabilityMinor = 0;
  int64_t maxThreadsPerBlock = 1024;
  int64_t driverVersion = 4000;
  int64_t runtimeVersion = 4000;
};

struct RunOptions {
  // The device engine reproduces the round-robin schedule exactly
  // (SURVEY F2/F4).  SeededRandom with a nonzero seed (and Exhaustive) run
  // as round-robin and say so in RunResult::engineNote.
  SchedulePolicy policy = SchedulePolicy::SeededRandom;
  uint64_t seed = 0;
  bool raceCheck = true;
  uint64_t stepLimit = 50'000'000;
  bool trace = false;
  ArchParams arch;
  // B200 extensions (not in the reference):
  int device = 0;             // CUDA device ordinal of the grid engine
  std::vector<int> devices;   // several devices: each grid's blocks are split across them
  int rank = 0, world = 1;    // one process per GPU: this rank runs its share of every grid's
  std::vector<uint8_t> commId;  // blocks; 128-byte NCCL id from mck::makeCommId on rank 0
  // host transport instead of NCCL (gather n bytes per rank, rank order; 0 = ok)
  int (*allgather)(void* ctx, const void* send, uint64_t n, void* recv) = nullptr;
  void* allgatherCtx = nullptr;
  // SURVEY Appendix E (builder-defined; off: reference-identical output):
  // cross-block races on global memory within one grid, reported as
  // "Possible race on global device memory detected at <file>:<line>."
  // (one device, one rank)
  bool globalRaceCheck = false;
};

struct StuckReport {
  enum class Kind { BarrierDeadlock, HostHang, StreamStall };
  Kind kind = Kind::BarrierDeadlock;
  uint32_t gid = 0;
  int bid = 0;
  std::vector<int> waitingTids;
  std::vector<int> missingTids;
  std::string reason;
  uint32_t sid = 0;
  std::string item;
};

// Per-run engine statistics (B200 extension).
struct EngineStats {
  uint64_t hostSteps = 0, deviceSteps = 0, barrierRules = 0, dispatches = 0;
  uint64_t sharedEvents = 0;     // race-checked shared accesses
  uint64_t grids = 0;
  uint64_t sweeps = 0;           // global round-robin sweeps
  double gridMs = 0;             // device time of the grid kernels (CUDA events)
  uint32_t kernelLaunches = 0;   // sm_100a kernels launched
  uint64_t blockSweeps = 0;      // K1: sweeps executed, summed over blocks
  uint64_t soloSweeps = 0;       // K1: of which in single-warp mode
  uint64_t blockCycles = 0, soloCycles = 0;  // K1: SM cycles per block, summed
};

struct RaceTriple {
  uint32_t object = 0;
  int64_t byte = 0;
  int line = 0;
  bool operator<(const RaceTriple& o) const {
    if (object != o.object) return object < o.object;
    if (byte != o.byte) return byte < o.byte;
    return line < o.line;
  }
  bool operator==(const RaceTriple& o) const {
    return object == o.object && byte == o.byte && line == o.line;
  }
};

struct RunResult {
  int exitCode = 0;
  std::string output;
  std::vector<Diagnostic> diagnostics;
  bool stuck = false;
  std::vector<StuckReport> stuckReports;
  uint64_t steps = 0;
  std::optional<int64_t> mainReturn;
  // B200 extensions
  std::vector<RaceTriple> reported;  // RaceState::reported, std::set order
  EngineStats stats;
  std::string engineError;           // non-empty: the run was abandoned by the engine
  std::string engineNote;            // non-empty: how the run departs from the requested options
  std::vector<std::string> trace;    // RunOptions::trace: the Machine::trace lines, in order
};

class MachineImpl;

class Machine {
 public:
  Machine(std::shared_ptr<const Program> prog, RunOptions opts);
  ~Machine();
  Machine(const Machine&) = delete;
  Machine& operator=(const Machine&) = delete;

  const Program& program() const { return *prog_; }
  const RunOptions& options() const { return opts_; }

  // Runs to completion (or stuck / step limit) and computes the exit code
  // (machine.cpp:1180-1227).  Device grids run on the B200 at dispatch.
  RunResult run();

  // Stuck-state classification of the final (frozen) configuration of the
  // last run() (deadlock.cpp:12-71): empty before run() and after a run
  // that terminated normally.
  std::vector<StuckReport> scanStuck() const;

  // Hooks, called synchronously on the calling thread (machine.hpp:384-388):
  //  * onOutput: every printf of the host thread, as it happens;
  //  * onApiCall: every runtime-API call of the host thread with its result
  //    code (blocking calls report success when they block, as the reference);
  //  * onMemAccess: every host-thread memory access.  Device accesses happen
  //    inside the B200 grid kernel and are not observable one by one: a grid
  //    launched while onMemAccess is set abandons the run with an engine
  //    error instead of silently skipping them;
  //  * onTrace: the --trace lines (RunOptions::trace), in the reference's
  //    order, once the run's timeline is complete.
  std::function<void(const MemAccessInfo&)> onMemAccess;
  std::function<void(ApiId, int)> onApiCall;
  std::function<void(const std::string&)> onTrace;
  std::function<void(const std::string&)> onOutput;

  // ---- the race checker as a library (racecheck.cpp:9-73), batched on K2 ----
  // allocObject mints an object id from the machine's counter (memory.cpp:
  // 12-31); object() returns the checker's view of it.
  Location allocObject(MemSpace space, int64_t size, const std::string& name);
  const MemObject& object(ObjectId id) const;
  // recordAccess / clearEpoch keep the reference's signatures.  Accesses are
  // buffered per shared object (in call order) and checked by the K2 kernel
  // on the GPU when flushRaces() (or raceReport()) runs; the reported set and
  // the Race diagnostics (first-detection order, addDiagnostic dedup) are
  // exactly the reference's, only deferred to the flush.  Accesses to
  // non-shared objects are ignored, as the reference only checks
  // DeviceShared memory (memory.cpp:142-143, 240-241).
  void recordAccess(const MemObject& obj, int64_t off, int64_t len, ThreadKey thread, AccessKind kind,
                    SourceLoc loc);
  void clearEpoch(GridId gid, int bid);
  void flushRaces();
  // RaceState::reported (std::set order) and the Race diagnostics so far
  // (flushes first).
  const std::vector<RaceTriple>& raceReport();
  const std::vector<Diagnostic>& raceDiagnostics();

 private:
  std::shared_ptr<const Program> prog_;
  RunOptions opts_;
  std::unique_ptr<MachineImpl> impl_;
};

// ---- the exhaustive-interleaving oracle (oracle.hpp:10-34) ----
// Explores every interleaving of the shared-memory accesses of a small
// program's grid on the GPU (one explorer thread per schedule prefix, replay
// DFS); invisible steps run eagerly in the canonical order.  The ground truth
// looks for a conflicting pair on one byte with no barrier of its block in
// between; detectorRace is the shadow detector's verdict on any schedule.
// B200 bounds: grids of <= 8 threads, one kernel launch per program.
struct OracleOptions {
  uint64_t maxInterleavings = 1'000'000;
  int maxThreads = 3;
  int maxAccessesPerThread = 8;
  ArchParams arch;
};

struct OracleResult {
  bool oracleRace = false;    // ground truth from exhaustive trace analysis
  bool detectorRace = false;  // any explored schedule where the shadow detector reports
  uint64_t interleavings = 0;
  bool aborted = false;       // a limit was exceeded
  std::string error;
};

OracleResult oracleRace(std::shared_ptr<const Program> prog, OracleOptions opts = {});

// A fresh 128-byte communicator id for RunOptions::commId (rank 0 makes it,
// the launcher broadcasts it).  Empty on failure.
std::vector<uint8_t> makeCommId();

std::string formatStuckReports(const std::vector<StuckReport>& reports);

struct CliOptions {
  std::string inputPath;
  bool raceCheck = true;
  uint64_t seed = 0;
  SchedulePolicy schedule = SchedulePolicy::SeededRandom;
  bool trace = false;
  uint64_t stepLimit = 50'000'000;
  std::string archFile;
  std::string reportPath;
  ArchParams arch;
};

struct FileRunOutcome {
  int exitCode = 0;
  std::string stdoutText;
  std::string stderrText;
  bool frontendError = false;
  RunResult run;
};

FileRunOutcome runFile(const CliOptions& opts, bool live = false);
FileRunOutcome runSourceText(const std::string& source, const std::string& filename, const CliOptions& opts);

// Architecture-parameter file, one `key = integer` per line (driver.hpp:37-41);
// throws std::runtime_error with file:line on malformed input.
ArchParams loadArchFile(const std::string& path);

struct CorpusOutcome {
  int passed = 0;
  int failed = 0;
  std::string table;  // one PASS/FAIL line per fixture
};
// Every .cu file of a directory against its .expect sidecar (driver.hpp:43-57).
CorpusOutcome runCorpus(const std::string& directory);

}  // namespace mck
