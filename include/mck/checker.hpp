// mck/checker.hpp -- public C++ API of the B200 checker, source-compatible
// with the reference's proj/include/minicudak headers for the program-load /
// launch-configuration / check / report path:
//
//   compileSource(src, file)        program.hpp:59-60  (throws FrontendError)
//   RunOptions / ArchParams         machine.hpp:300-316
//   Machine(prog, opts).run()       machine.hpp:357-375
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
  // (SURVEY F2/F4); SeededRandom is accepted and run as round-robin.
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
  bool globalRaceCheck = false;  // SURVEY Appendix E (off: reference-identical output)
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
  std::vector<std::string> trace;    // RunOptions::trace: the Machine::trace lines, in order
};

class MachineImpl;

class Machine {
 public:
  Machine(std::shared_ptr<const Program> prog, RunOptions opts);
  ~Machine();
  Machine(const Machine&) = delete;
  Machine& operator=(const Machine&) = delete;
  RunResult run();
  const RunOptions& options() const { return opts_; }

 private:
  std::shared_ptr<const Program> prog_;
  RunOptions opts_;
  std::unique_ptr<MachineImpl> impl_;
};

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
