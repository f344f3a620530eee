// machine.cpp -- the host side of the checker: memory store, the host-thread
// interpreter over the step-exact IR, streams / events / runtime API, the
// round-robin sweep timeline, grid dispatch to the B200 engine, diagnostic
// ordering, stuck classification and RunResult.
//
// Reference behaviour restated (file:line in /root/reference/proj/src):
//   run loop, exit codes ........ machine.cpp:1180-1227
//   round-robin sweeps .......... machine.cpp:411-429
//   host thread steps ........... machine.cpp:493-1178
//   addDiagnostic dedup/order ... machine.cpp:41-46
//   memory rules ................ memory.cpp:25-293
//   streams, host waits ......... streams.cpp:13-93
//   runtime API ................. runtime_api.cpp:39-372
//   printf ...................... machine.cpp:1236-1378
//   scanStuck / report text ..... deadlock.cpp:12-96
//
// Timeline model: one sweep = one host step (if runnable) + every runnable
// device thread one step + barrier rules + one dispatch per ready stream
// (ascending sid).  A grid is dispatched at sweep s and runs on the GPU at
// once; its blocks' schedules are block-local, so it occupies
// sweeps s+1 .. s+D and completes in sweep s+D.  Host steps and dispatches are
// simulated sweep by sweep, idle stretches are skipped.
#include <algorithm>
#include <array>
#include <cstdio>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <set>
#include <stdexcept>

#include "engine.hpp"
#include "machine_impl.hpp"
#include "mck/checker.hpp"

namespace mckb {

using mck_core::Diags;
using mck_core::Val;
using namespace mck_core;

namespace {

constexpr uint64_t NEVER = ~0ull;

enum Space : uint8_t { SP_HOST = 0, SP_GLOBAL = 1 };

struct HObj {
  uint32_t id = 0;
  uint8_t space = SP_HOST;
  int64_t size = 0;
  bool live = true;
  std::string name;
  std::vector<uint8_t> bytes, meta;  // host objects
  uint64_t devBase = 0;              // device-global objects
  bool hasPtr = false;               // some pointer slot was ever stored here
};

struct Frame {
  int retPc;
  int bindBase;
  int scopeDepth;
  int valueDepth;
  int fn;
};

struct LaunchRec {
  int kernel = -1;
  int64_t grid = 0, block = 0, shmem = 0;
  uint32_t stream = 0;
  std::vector<Val> args;
  int line = 0;
};

struct CopyRec {
  Val dst{}, src{};
  int64_t n = 0;
  int dir = 0;
  int line = 0;
};

enum class ItemKind { Launch, Copy, EventRecord, WaitEvent };
struct StreamItem {
  ItemKind kind = ItemKind::Launch;
  LaunchRec launch;
  CopyRec copy;
  uint32_t eid = 0;
};

struct StreamRec {
  std::deque<StreamItem> q;
  bool running = false;
  uint32_t runningGid = 0;
  bool destroyed = false;
  bool idle() const { return q.empty() && !running; }
};

enum class EvStatus { Created, Pending, Recorded };

struct GridRec {
  uint32_t gid;
  uint32_t stream;
  uint64_t spawnSweep = 0;  // dispatch sweep: local sweep l runs at spawnSweep + l
  int64_t gridDim, blockDim;
  uint32_t sharedBase;
  uint64_t endSweep;  // NEVER = deadlocked
  bool completed = false;
  GridResult res;
  bool stepsCounted = false;
};

// A diagnostic with its execution timestamp; the final list is the stable
// first-occurrence dedup in timestamp order (machine.cpp:41-46).
struct DiagEv {
  uint64_t sweep;
  int phase;  // 0 host step, 1 device step, 3 dispatch, 9 end of run
  uint64_t k1, k2;
  uint64_t seq;
  mck::Diagnostic d;
};

// A --trace line with its execution timestamp (Machine::trace, machine.cpp:52;
// lines from device.cpp:63,163-195,215 and streams.cpp:49-61).
struct TraceEv {
  uint64_t sweep;
  int phase;  // 1 device step (grid completed), 2 barrier rule, 3 dispatch
  uint64_t k1, k2;
  uint64_t seq;
  std::string text;
};

enum class WaitKind { None, Device, Stream, Event };

}  // namespace

// The mck::Machine hooks the host interpreter calls (machine.hpp:384-388).
struct HostHooks {
  std::function<void(const mck::MemAccessInfo&)> mem;
  std::function<void(mck::ApiId, int)> api;
  std::function<void(const std::string&)> out;
};

class HostMachine {
 public:
  HostMachine(std::shared_ptr<const Program> prog, const mck::RunOptions& o, HostHooks hooks = {})
      : P_(std::move(prog)), o_(o), hooks_(std::move(hooks)) {}

  mck::RunResult run();

  // oracle mode (oracleRace): the first grid is explored exhaustively on the
  // GPU before it runs as usual
  void setOracle(const OracleSpec& spec, int maxThreads) {
    oracle_ = spec;
    oracleOn_ = true;
    oracleMaxThreads_ = maxThreads;
  }
  const OracleOut& oracleOut() const { return oracleOut_; }
  int oracleGrids() const { return oracleGrids_; }

 private:
  bool oracleOn_ = false;
  OracleSpec oracle_;
  int oracleMaxThreads_ = 3;
  OracleOut oracleOut_;
  int oracleGrids_ = 0;
  std::shared_ptr<const Program> P_;
  mck::RunOptions o_;
  HostHooks hooks_;
  std::unique_ptr<DeviceEngine> eng_;
  std::string engWhy_;

  // memory store
  std::vector<HObj> objs_;  // ascending id
  uint32_t nextId_ = 1;
  std::vector<uint32_t> globalIds_;
  std::vector<std::array<uint32_t, 3>> sharedRanges_;

  // host thread
  int pc_ = 0;
  std::vector<Val> vals_;
  std::vector<size_t> scopeMarks_;
  std::vector<uint32_t> owned_;
  std::vector<Frame> frames_;
  std::vector<uint32_t> binds_;
  bool hostDone_ = false, hostHalted_ = false;
  bool awaiting_ = false;
  int awaitCode_ = 0;
  WaitKind wait_ = WaitKind::None;
  uint32_t waitId_ = 0;
  std::optional<int64_t> exitValue_;
  std::vector<std::string> hostStrings_;  // Str values

  // machine
  uint64_t steps_ = 0, sweep_ = 0, seq_ = 0;
  std::map<uint32_t, StreamRec> streams_;
  uint32_t nextSid_ = 1;
  std::map<uint32_t, EvStatus> events_;
  uint32_t nextEid_ = 1;
  std::map<uint32_t, GridRec> grids_;
  uint32_t nextGid_ = 1;
  uint64_t runningGrids_ = 0;  // dispatched, not completed, will complete
  int lastApiError_ = 0;
  std::string output_;
  std::vector<DiagEv> diags_;
  std::vector<TraceEv> traces_;
  void traceLine(uint64_t sweep, int phase, uint64_t k1, uint64_t k2, std::string text) {
    if (o_.trace) traces_.push_back(TraceEv{sweep, phase, k1, k2, seq_++, std::move(text)});
  }
  void traceBarriers(uint32_t gid, const GridRec& rec, uint64_t spawn);
  std::vector<mck::RaceTriple> reported_;
  mck::EngineStats stats_;
  std::string engineError_;
  std::vector<uint32_t> conflictGids_;  // grids with cross-block global conflicts (the probe)
  // grids whose global bytes another stream touched while they were in
  // flight (the engine applies a grid's effects at its dispatch sweep)
  std::vector<uint32_t> inflightGids_;
  // does an access [lo, hi) of object `obj` (write: `wr`) overlap what a
  // running grid on another stream read or wrote, with a write on either side?
  void checkInflight(uint32_t sid, uint32_t obj, int64_t lo, int64_t hi, bool wr) {
    if (lo >= hi) return;
    for (const auto& [gid, g] : grids_) {
      if (g.completed || g.stream == sid || g.endSweep <= sweep_) continue;
      for (const auto& e : g.res.footprint) {
        if ((uint32_t)e[0] != obj) continue;
        const bool hitW = e[3] < hi && lo < e[4];
        const bool hitR = e[1] < hi && lo < e[2];
        if (hitW || (wr && hitR)) {
          if (std::find(inflightGids_.begin(), inflightGids_.end(), gid) == inflightGids_.end())
            inflightGids_.push_back(gid);
        }
      }
    }
  }

  // Bytes [lo, lo + n) of device object `obj` as a copy dispatched now on
  // stream sid sees them while a grid on another stream is in flight: the
  // grid's writes up to this sweep (global order) over what they overwrote.
  // false (b / m untouched) when no grid applies, two do, or the grid's
  // write history is incomplete.
  bool midflight(uint32_t sid, uint32_t obj, int64_t lo, int64_t n, uint8_t* b, uint8_t* m) {
    const GridRec* G = nullptr;
    for (const auto& [gid, g] : grids_) {
      if (g.completed || g.stream == sid || g.endSweep <= sweep_) continue;
      bool hits = false;
      for (const auto& e : g.res.footprint)
        if ((uint32_t)e[0] == obj && e[3] < lo + n && lo < e[4]) hits = true;
      if (!hits) continue;
      if (G || g.res.writes.empty()) return false;
      G = &g;
    }
    if (!G) return false;
    std::vector<char> seen(static_cast<size_t>(n), 0);
    for (const GridResult::Write& w : G->res.writes) {
      if (w.obj != obj) continue;
      const bool done = G->spawnSweep + w.lsweep <= sweep_;  // device steps precede this sweep's dispatches
      for (uint32_t q = 0; q < w.len; ++q) {
        const int64_t x = w.off + q - lo;
        if (x < 0 || x >= n) continue;
        if (!seen[static_cast<size_t>(x)]) {  // the value before the grid's first write
          b[x] = w.oldB[q];
          m[x] = w.oldM[q];
          seen[static_cast<size_t>(x)] = 1;
        }
        if (done) {
          b[x] = w.newB[q];
          m[x] |= META_DEF;
        }
      }
    }
    return true;
  }

  // ---------------- helpers ----------------
  std::string at(int line) const { return " at " + P_->filename + ":" + std::to_string(line) + "."; }

  void diag(mck::Severity sev, mck::DiagCategory cat, const std::string& msg, int line, int phase = 0,
            uint64_t k1 = 0, uint64_t k2 = 0) {
    DiagEv e;
    e.sweep = sweep_;
    e.phase = phase;
    e.k1 = k1;
    e.k2 = k2;
    e.seq = seq_++;
    e.d.severity = sev;
    e.d.category = cat;
    e.d.message = msg;
    e.d.loc.line = line;
    diags_.push_back(std::move(e));
  }
  void ub(const std::string& msg, int line) {
    diag(mck::Severity::Error, mck::DiagCategory::UndefinedBehavior, msg + at(line), line);
  }
  void apiDiag(const std::string& msg, int line, int phase = 0, uint64_t k1 = 0) {
    diag(mck::Severity::Error, mck::DiagCategory::ApiError, msg + at(line), line, phase, k1);
  }

  HObj* find(uint32_t id) {
    if (id == 0) return nullptr;
    if (cacheId_ == id && cacheVec_ == objs_.data()) return cacheObj_;
    auto it = std::lower_bound(objs_.begin(), objs_.end(), id,
                               [](const HObj& o, uint32_t x) { return o.id < x; });
    if (it == objs_.end() || it->id != id) return nullptr;
    cacheId_ = id;
    cacheVec_ = objs_.data();
    cacheObj_ = &*it;
    return cacheObj_;
  }
  uint32_t cacheId_ = 0;
  const HObj* cacheVec_ = nullptr;
  HObj* cacheObj_ = nullptr;

  uint32_t alloc(uint8_t space, int64_t size, const std::string& name) {
    HObj o;
    o.id = nextId_++;
    o.space = space;
    o.size = size;
    o.name = name;
    if (space == SP_HOST) {
      o.bytes.assign(static_cast<size_t>(size), 0);
      o.meta.assign(static_cast<size_t>(size), 0);
    } else {
      o.devBase = eng_->alloc(size);
    }
    objs_.push_back(std::move(o));
    return objs_.back().id;
  }

  // pokeValue on a host object (memory.cpp:184-206)
  static void poke(HObj& o, int64_t off, uint8_t t, const Val& v) {
    int64_t len = t_scalar(t);
    if (o.hasPtr)
      for (int64_t s = std::max<int64_t>(0, off - 7); s < off + len && s < o.size; ++s)
        o.meta[static_cast<size_t>(s)] &= static_cast<uint8_t>(~META_PTR);
    uint64_t raw = encode_scalar(v, t);
    uint8_t* b = o.bytes.data() + off;
    uint8_t* m = o.meta.data() + off;
    for (int64_t i = 0; i < len; ++i) {
      b[i] = static_cast<uint8_t>(raw >> (8 * i));
      m[i] |= META_DEF;
    }
    if (v.kind == MCK_K_PTR && v.obj != 0) {
      m[0] |= META_PTR;
      o.hasPtr = true;
    }
  }

  std::string spaceStr(uint8_t space) const { return space == SP_HOST ? "host" : "device-global"; }

  // readMem for the host thread (memory.cpp:110-182); nullopt => halt
  void memHook(mck::AccessKind k, uint32_t obj, const HObj* o, int64_t off, int64_t len, int line) {
    if (!hooks_.mem) return;
    mck::MemAccessInfo m;
    m.kind = k;
    m.object = obj;
    if (o) m.space = o->space == SP_HOST ? mck::MemSpace::host() : mck::MemSpace::deviceGlobal();
    m.offset = off;
    m.len = len;
    m.allowed = o && o->space == SP_HOST;  // checkAccess for the host thread (memory.cpp:64-69)
    m.loc.line = line;
    hooks_.mem(m);
  }

  std::optional<Val> readMem(uint32_t obj, int64_t off, uint8_t t, int line) {
    HObj* o = find(obj);
    if (__builtin_expect(o && !hooks_.mem && o->space == SP_HOST && o->live && MCK_T_PTR(t) == 0, 1)) {
      // the common case: a defined scalar inside a live host object
      const int64_t len = t_scalar(t);
      if (off >= 0 && off + len <= o->size) {
        const uint8_t* m = o->meta.data() + off;
        bool def = true;
        uint64_t raw = 0;
        for (int64_t i = 0; i < len; ++i) {
          def &= (m[i] & META_DEF) != 0;
          raw |= static_cast<uint64_t>(o->bytes[static_cast<size_t>(off + i)]) << (8 * i);
        }
        if (def) return decode_scalar(raw, t);
      }
    }
    if (!o) {
      ub("read through a null or invalid pointer", line);
      memHook(mck::AccessKind::Read, obj, nullptr, off, t_scalar(t), line);
      return std::nullopt;
    }
    int64_t len = t_scalar(t);
    memHook(mck::AccessKind::Read, obj, o, off, len, line);
    if (o->space != SP_HOST) {
      diag(mck::Severity::Error, mck::DiagCategory::MemBoundary,
           "Illegal device or host memory access: host code read of " + spaceStr(o->space) + " memory" + at(line),
           line);
      return std::nullopt;
    }
    if (!o->live) {
      ub("read from dead memory ('" + o->name + "' was freed or expired)", line);
      return std::nullopt;
    }
    if (off < 0 || off + len > o->size) {
      ub("out-of-bounds read of " + std::to_string(len) + " bytes at offset " + std::to_string(off) + " of " +
             std::to_string(o->size) + "-byte object '" + o->name + "'",
         line);
      return std::nullopt;
    }
    bool undef = false;
    uint64_t raw = 0;
    for (int64_t i = 0; i < len; ++i) {
      if (!(o->meta[static_cast<size_t>(off + i)] & META_DEF)) undef = true;
      raw |= static_cast<uint64_t>(o->bytes[static_cast<size_t>(off + i)]) << (8 * i);
    }
    if (MCK_T_PTR(t) > 0) {
      if (o->meta[static_cast<size_t>(off)] & META_PTR)
        return v_ptr(static_cast<uint32_t>(raw >> 32), static_cast<int32_t>(raw & 0xffffffffu), t);
      if (undef) {
        ub("read of uninitialized pointer from '" + o->name + "'", line);
        return std::nullopt;
      }
      if (raw == 0) return v_ptr(0, 0, t);
      ub("read of a non-pointer value as a pointer", line);
      return std::nullopt;
    }
    if (undef) ub("read of uninitialized memory ('" + o->name + "')", line);
    return decode_scalar(raw, t);
  }

  bool writeMem(uint32_t obj, int64_t off, uint8_t t, const Val& v, int line) {
    HObj* o = find(obj);
    if (!o) {
      ub("write through a null or invalid pointer", line);
      memHook(mck::AccessKind::Write, obj, nullptr, off, t_scalar(t), line);
      return false;
    }
    int64_t len = t_scalar(t);
    memHook(mck::AccessKind::Write, obj, o, off, len, line);
    if (o->space != SP_HOST) {
      diag(mck::Severity::Error, mck::DiagCategory::MemBoundary,
           "Illegal device or host memory access: host code write of " + spaceStr(o->space) + " memory" + at(line),
           line);
      return false;
    }
    if (!o->live) {
      ub("write to dead memory ('" + o->name + "' was freed or expired)", line);
      return false;
    }
    if (off < 0 || off + len > o->size) {
      ub("out-of-bounds write of " + std::to_string(len) + " bytes at offset " + std::to_string(off) + " of " +
             std::to_string(o->size) + "-byte object '" + o->name + "'",
         line);
      return false;
    }
    poke(*o, off, t, v);
    return true;
  }

  void reportDiags(const Diags& d, int line) {
    if (__builtin_expect(d.n != 0, 0)) reportDiagsSlow(d, line);
  }
  __attribute__((noinline)) void reportDiagsSlow(const Diags& d, int line) {
    for (int i = 0; i < d.n; ++i) ub(ubText(d.code[i]), line);
  }

  static const char* ubText(int code) {
    switch (code) {
      case MCK_D_OVERFLOW: return "signed integer overflow";
      case MCK_D_DIV0: return "division by zero";
      case MCK_D_REM0: return "remainder by zero";
      case MCK_D_SHIFT: return "shift count out of range";
      case MCK_D_PTR_ORDER_INT: return "ordered comparison between a pointer and an integer";
      case MCK_D_PTR_ORDER_OBJ: return "ordered comparison of pointers into different memory objects";
      case MCK_D_PTR_ADD: return "invalid pointer addition";
      case MCK_D_PTR_SUB_OBJ: return "subtraction of pointers into different memory objects";
      case MCK_D_PTR_SUB_VOID: return "pointer subtraction on void pointers";
      case MCK_D_PTR_OPERAND: return "invalid pointer arithmetic operand";
      case MCK_D_INT_MINUS_PTR: return "integer minus pointer is not valid";
      case MCK_D_VOID_ARITH: return "arithmetic on void pointers";
      case MCK_D_PTR_OP: return "invalid operation on pointer values";
      case MCK_D_FLOAT_OP: return "invalid operator on floating values";
      case MCK_D_OPERANDS: return "invalid operands";
      case MCK_D_CONV_TO_PTR: return "invalid conversion of a non-pointer value to a pointer";
      case MCK_D_CONV_TO_FLOAT: return "invalid conversion to a floating type";
      case MCK_D_FLOAT_RANGE: return "floating value out of range in integer conversion";
      case MCK_D_PTR_TO_INT: return "conversion of a pointer to an integer is not supported";
      case MCK_D_CONV: return "invalid conversion";
      case MCK_D_DEREF_NONPTR: return "dereference of a non-pointer value";
      case MCK_D_SUBSCRIPT: return "invalid subscript";
      case MCK_D_MODIFY_ARRAY: return "cannot modify an array";
      case MCK_D_NEG_NONARITH: return "negation of a non-arithmetic value";
      case MCK_D_BITNOT_NONINT: return "bitwise complement of a non-integer value";
      default: return "undefined behavior";
    }
  }

 public:
  // Formats one device diagnostic record (templates: SURVEY Appendix F).
  // r.name >= 0: program string id; <= -2: index -name-2 of the grid's
  // device-object table (objNames)
  std::string formatDevDiag(const DevDiag& r, uint32_t gid, uint32_t bid, uint32_t tid, mck::DiagCategory& cat,
                            mck::Severity& sev, const std::vector<std::string>& objNames) const {
    cat = mck::DiagCategory::UndefinedBehavior;
    sev = mck::Severity::Error;
    const std::string name = r.name >= 0 ? P_->str(r.name)
                             : (r.name <= -2 && static_cast<size_t>(-r.name - 2) < objNames.size())
                                 ? objNames[static_cast<size_t>(-r.name - 2)]
                                 : std::string("cudaMalloc");
    const char* rw = r.p[0] ? "write" : "read";
    switch (r.code) {
      case MCK_D_RACE:
        cat = mck::DiagCategory::Race;
        sev = mck::Severity::Warning;
        return "Possible race on shared device memory detected at " + P_->filename + ":" + std::to_string(r.line) + ".";
      case MCK_D_GRACE:  // RunOptions::globalRaceCheck (builder-defined, off by default)
        cat = mck::DiagCategory::Race;
        sev = mck::Severity::Warning;
        return "Possible race on global device memory detected at " + P_->filename + ":" + std::to_string(r.line) + ".";
      case MCK_D_MEMBOUNDARY: {
        cat = mck::DiagCategory::MemBoundary;
        std::string sp = r.p[1] == 0 ? "host" : r.p[1] == 1 ? "device-global"
                         : "block-shared(gid=" + std::to_string(r.p[2] >> 32) + ",bid=" +
                               std::to_string(static_cast<int32_t>(r.p[2] & 0xffffffff)) + ")";
        return "Illegal device or host memory access: device thread (gid=" + std::to_string(gid) +
               ", bid=" + std::to_string(bid) + ", tid=" + std::to_string(tid) + ") " + rw + " of " + sp +
               " memory" + at(r.line);
      }
      case MCK_D_NULL_RW:
        return std::string(r.p[0] ? "write" : "read") + " through a null or invalid pointer" + at(r.line);
      case MCK_D_DEAD:
        return std::string(r.p[0] ? "write to" : "read from") + " dead memory ('" + name + "' was freed or expired)" +
               at(r.line);
      case MCK_D_OOB:
        return std::string("out-of-bounds ") + rw + " of " + std::to_string(r.p[1]) + " bytes at offset " +
               std::to_string(r.p[2]) + " of " + std::to_string(r.p[3]) + "-byte object '" + name + "'" + at(r.line);
      case MCK_D_UNINIT: return "read of uninitialized memory ('" + name + "')" + at(r.line);
      case MCK_D_UNINIT_PTR: return "read of uninitialized pointer from '" + name + "'" + at(r.line);
      case MCK_D_NONPTR_AS_PTR: return "read of a non-pointer value as a pointer" + at(r.line);
      case MCK_D_FIXED_UB: return fixedUb(static_cast<int>(r.p[0]), r.name) + at(r.line);
      default: return std::string(ubText(r.code)) + at(r.line);
    }
  }

 private:
  std::string fixedUb(int code, int name) const {
    std::string n = name >= 0 ? P_->str(name) : std::string();
    switch (code) {
      case MCK_UB_STRLIT: return "string literal in an unsupported position";
      case MCK_UB_MEMBER: return "unexpected member access";
      case MCK_UB_UNBOUND: return "variable '" + n + "' is not bound in this scope";
      case MCK_UB_NOVALUE: return "cannot evaluate '" + n + "' as a value";
      case MCK_UB_HOSTBUILTIN: return "device builtin '" + n + "' referenced from host code";
      default: return "call of an unsupported function";
    }
  }

  // ---------------- host thread ----------------
  void halt() {
    hostHalted_ = true;
    hostDone_ = true;
  }
  Val pop() {
    Val v = vals_.back();
    vals_.pop_back();
    return v;
  }
  void popScopes(size_t depth) {
    while (scopeMarks_.size() > depth) {
      size_t m = scopeMarks_.back();
      for (size_t i = m; i < owned_.size(); ++i)
        if (HObj* o = find(owned_[i])) o->live = false;
      owned_.resize(m);
      scopeMarks_.pop_back();
    }
  }
  const Frame& frame() const { return frames_.back(); }
  int curFn() const { return frames_.back().fn; }
  uint32_t& bind(int slot) { return binds_[static_cast<size_t>(frame().bindBase + slot)]; }
  const mck_local& local(int fn, int slot) const {
    return P_->locals[static_cast<size_t>(P_->fns[static_cast<size_t>(fn)].local_base + slot)];
  }

  void enterFunction(int fn, int retPc) {
    Frame f;
    f.retPc = retPc;
    f.bindBase = frames_.empty() ? 0 : frame().bindBase + P_->fns[static_cast<size_t>(curFn())].n_slots;
    f.scopeDepth = static_cast<int>(scopeMarks_.size());
    f.valueDepth = static_cast<int>(vals_.size());
    f.fn = fn;
    frames_.push_back(f);
    size_t need = static_cast<size_t>(f.bindBase + P_->fns[static_cast<size_t>(fn)].n_slots);
    if (binds_.size() < need) binds_.resize(need, 0);
    scopeMarks_.push_back(owned_.size());
  }

  // Leaves the current function (ReturnUnwind / CallFrame fall-off).
  void leaveFunction(const Val* v, int line, bool convertIt) {
    Frame f = frames_.back();
    popScopes(static_cast<size_t>(f.scopeDepth));
    vals_.resize(static_cast<size_t>(f.valueDepth));
    frames_.pop_back();
    uint8_t ret = P_->fns[static_cast<size_t>(f.fn)].ret;
    Val out;
    if (convertIt) {
      Diags d{};
      if (!convert(*v, ret, out, d)) {
        reportDiags(d, line);
        halt();
        return;
      }
      reportDiags(d, line);
    } else {
      out = t_is_void(ret) ? v_void() : v_int(0, ret);
    }
    vals_.push_back(out);
    if (frames_.empty()) {
      hostDone_ = true;
      exitValue_ = vals_.back().i;
      return;
    }
    pc_ = f.retPc;
  }

  void hostStep();
  void execPrintf(const mck_ins& in);
  void invokeApi(const mck_ins& in);
  bool hostRunnable() const;
  bool waitSatisfied() const;

  // ---------------- streams / grids ----------------
  bool enqueue(uint32_t sid, StreamItem item, int line) {
    auto it = streams_.find(sid);
    if (it == streams_.end() || it->second.destroyed) {
      apiDiag("operation on uninitialized stream " + std::to_string(sid), line);
      return false;
    }
    it->second.q.push_back(std::move(item));
    ++queued_;
    return true;
  }
  uint64_t queued_ = 0;
  std::vector<uint32_t> sids_;
  bool dispatchable(const StreamRec& s) const {
    if (s.running || s.q.empty()) return false;
    const StreamItem& h = s.q.front();
    if (h.kind == ItemKind::WaitEvent) {
      auto e = events_.find(h.eid);
      return e != events_.end() && e->second == EvStatus::Recorded;
    }
    return true;
  }
  void dispatch(uint32_t sid);
  void spawnGrid(uint32_t sid, const LaunchRec& l);
  void performCopy(const CopyRec& c, uint32_t sid);
  void completeGrids(uint64_t sweep);

  std::vector<mck::StuckReport> scanStuck() const;
};

// ======================= host thread step =======================

bool HostMachine::waitSatisfied() const {
  switch (wait_) {
    case WaitKind::None: return true;
    case WaitKind::Device:
      for (const auto& s : streams_)
        if (!s.second.idle()) return false;
      for (const auto& g : grids_)
        if (!g.second.completed) return false;
      return true;
    case WaitKind::Stream: {
      auto it = streams_.find(waitId_);
      return it == streams_.end() || it->second.idle();
    }
    case WaitKind::Event: {
      auto it = events_.find(waitId_);
      return it == events_.end() || it->second == EvStatus::Recorded;
    }
  }
  return true;
}

bool HostMachine::hostRunnable() const {
  if (hostDone_ || hostHalted_) return false;
  if (awaiting_) return waitSatisfied();
  return true;
}

void HostMachine::hostStep() {
  if (awaiting_) {  // ApiAwait (machine.cpp:1172-1177)
    awaiting_ = false;
    wait_ = WaitKind::None;
    waitId_ = 0;
    vals_.push_back(v_int(awaitCode_));
    return;
  }
  const std::vector<mck_ins>& code = P_->code;
  while (code[static_cast<size_t>(pc_)].op == OP_JMP) pc_ = code[static_cast<size_t>(pc_)].a;
  const mck_ins in = code[static_cast<size_t>(pc_)];
  ++pc_;
  const int L = in.line;
  Diags d{};
  switch (in.op) {
    case OP_NOP: break;
    case OP_SCOPE_PUSH: scopeMarks_.push_back(owned_.size()); break;
    case OP_SCOPE_POP: popScopes(scopeMarks_.size() - 1); break;
    case OP_PUSH_INT:
      vals_.push_back(v_int(static_cast<int64_t>((static_cast<uint64_t>(static_cast<uint32_t>(in.b)) << 32) |
                                                 static_cast<uint32_t>(in.a)),
                            in.t));
      break;
    case OP_PUSH_FLT:
      vals_.push_back(mk(MCK_K_FLOAT, in.t, 0,
                         static_cast<int64_t>((static_cast<uint64_t>(static_cast<uint32_t>(in.b)) << 32) |
                                              static_cast<uint32_t>(in.a))));
      break;
    case OP_PUSH_LOCAL: {
      uint32_t o = bind(in.a);
      if (!o) {
        ub("variable '" + P_->str(in.b) + "' is not bound in this scope", L);
        halt();
        break;
      }
      vals_.push_back(v_lv(o, 0, in.t));
      break;
    }
    case OP_PUSH_GLOBAL: vals_.push_back(v_lv(globalIds_[static_cast<size_t>(in.a)], 0, in.t)); break;
    case OP_PUSH_BUILTIN:
      ub("device builtin '" + P_->str(in.b) + "' referenced from host code", L);
      halt();
      break;
    case OP_UB:
      ub(fixedUb(in.a, in.b), L);
      halt();
      break;
    case OP_LOADRV: {
      Val lv = pop();
      if (MCK_T_ARR(lv.type)) {
        vals_.push_back(v_ptr(lv.obj, lv.i, t_decay(lv.type)));
        break;
      }
      auto v = readMem(lv.obj, lv.i, lv.type, L);
      if (!v) {
        halt();
        break;
      }
      vals_.push_back(*v);
      break;
    }
    case OP_LOADKEEP: {
      Val lv = pop();
      if (MCK_T_ARR(lv.type)) {
        ub("cannot modify an array", L);
        halt();
        break;
      }
      auto v = readMem(lv.obj, lv.i, lv.type, L);
      if (!v) {
        halt();
        break;
      }
      vals_.push_back(lv);
      vals_.push_back(*v);
      break;
    }
    case OP_STORE:
    case OP_STORE_OP:
    case OP_STORE_INC: {
      Val r;
      bool ok = true;
      Val lv;
      if (in.op == OP_STORE) {
        Val rhs = pop();
        lv = pop();
        ok = convert(rhs, lv.type, r, d);
      } else if (in.op == OP_STORE_OP) {
        Val rhs = pop(), old = pop();
        lv = pop();
        Val t;
        ok = binop(in.f, old, rhs, t, d) && convert(t, lv.type, r, d);
      } else {
        Val old = pop();
        lv = pop();
        Val t;
        ok = binop(MCK_ADD, old, v_int(in.a), t, d) && convert(t, lv.type, r, d);
        if (ok && !in.f) {
          reportDiags(d, L);
          d.n = 0;
          if (!writeMem(lv.obj, lv.i, lv.type, r, L)) {
            halt();
            break;
          }
          vals_.push_back(old);
          break;
        }
      }
      reportDiags(d, L);
      if (!ok) {
        halt();
        break;
      }
      if (!writeMem(lv.obj, lv.i, lv.type, r, L)) {
        halt();
        break;
      }
      vals_.push_back(r);
      break;
    }
    case OP_ADDROF: {
      Val lv = pop();
      vals_.push_back(v_ptr(lv.obj, lv.i, t_addr(lv.type)));
      break;
    }
    case OP_DEREF: {
      Val v = pop();
      if (v.kind == MCK_K_INT && v.i == 0) v = v_ptr(0, 0, MCK_T_VOIDP);
      if (v.kind != MCK_K_PTR || MCK_T_PTR(v.type) == 0) {
        ub("dereference of a non-pointer value", L);
        halt();
        break;
      }
      vals_.push_back(v_lv(v.obj, v.i, t_elem(v.type)));
      break;
    }
    case OP_INDEX: {
      Val idx = pop(), base = pop();
      if (base.kind != MCK_K_PTR || idx.kind != MCK_K_INT) {
        ub("invalid subscript", L);
        halt();
        break;
      }
      uint8_t e = t_elem(base.type);
      vals_.push_back(v_lv(base.obj, base.i + idx.i * t_scalar(e), e));
      break;
    }
    case OP_UNARY: {
      Val v = pop(), r;
      bool ok = unop(in.f, v, r, d);
      reportDiags(d, L);
      if (!ok) {
        halt();
        break;
      }
      vals_.push_back(r);
      break;
    }
    case OP_BINARY: {
      Val rr = pop(), l = pop(), r;
      bool ok = binop(in.f, l, rr, r, d);
      reportDiags(d, L);
      if (!ok) {
        halt();
        break;
      }
      vals_.push_back(r);
      break;
    }
    case OP_LOGRHS: {
      Val l = pop();
      bool isAnd = in.f == 1;
      if (isAnd && !truthy(l)) {
        vals_.push_back(v_int(0));
        pc_ = in.a;
      } else if (!isAnd && truthy(l)) {
        vals_.push_back(v_int(1));
        pc_ = in.a;
      }
      break;
    }
    case OP_BOOLIFY: {
      Val v = pop();
      vals_.push_back(v_int(truthy(v) ? 1 : 0));
      break;
    }
    case OP_TERNSEL: {
      Val c = pop();
      if (!truthy(c)) pc_ = in.a;
      break;
    }
    case OP_CAST: {
      Val v = pop(), r;
      if (MCK_T_PTR(in.t) > 0 && v.kind == MCK_K_PTR) {
        vals_.push_back(v_ptr(v.obj, v.i, in.t));
        break;
      }
      bool ok = convert(v, in.t, r, d);
      reportDiags(d, L);
      if (!ok) {
        halt();
        break;
      }
      vals_.push_back(r);
      break;
    }
    case OP_IFJUDGE: {
      Val c = pop();
      if (!truthy(c)) pc_ = in.a;
      break;
    }
    case OP_WHILEJUDGE: {
      Val c = pop();
      if (!truthy(c)) pc_ = in.a;
      break;
    }
    case OP_FORJUDGE: {
      bool go = true;
      if (in.f) go = truthy(pop());
      if (!go) pc_ = in.a;
      break;
    }
    case OP_POPVALUE: pop(); break;
    case OP_RETURN: {
      Val v = in.f ? pop() : v_void();
      leaveFunction(&v, L, true);
      break;
    }
    case OP_FALLOFF: leaveFunction(nullptr, L, false); break;
    case OP_BREAK:
    case OP_CONTINUE:
      popScopes(scopeMarks_.size() - static_cast<size_t>(in.b));
      pc_ = in.a;
      break;
    case OP_CALL: {
      const mck_fn& f = P_->fns[static_cast<size_t>(in.a)];
      std::vector<Val> args(static_cast<size_t>(in.b));
      for (int i = in.b; i > 0; --i) args[static_cast<size_t>(i - 1)] = pop();
      enterFunction(in.a, pc_);
      for (int i = 0; i < in.b; ++i) {
        const mck_local& pl = local(in.a, i);
        Val cv;
        Diags dd{};
        bool ok = convert(args[static_cast<size_t>(i)], pl.type, cv, dd);
        reportDiags(dd, L);
        if (!ok) {
          halt();
          return;
        }
        uint32_t o = alloc(SP_HOST, pl.size, P_->str(pl.name));
        poke(*find(o), 0, pl.type, cv);
        bind(i) = o;
        owned_.push_back(o);
      }
      pc_ = f.entry;
      break;
    }
    case OP_DECL: {
      if (in.f) break;  // extern __shared__ in host code is rejected by lowering
      const mck_local& l = local(curFn(), in.a);
      uint32_t o = alloc(SP_HOST, l.size, P_->str(l.name));
      bind(in.a) = o;
      owned_.push_back(o);
      break;
    }
    case OP_INITSTORE: {
      Val v = pop(), r;
      bool ok = convert(v, in.t, r, d);
      reportDiags(d, L);
      if (!ok) {
        halt();
        break;
      }
      if (!writeMem(bind(in.a), 0, in.t, r, L)) halt();
      break;
    }
    case OP_PRINTF: execPrintf(in); break;
    case OP_API: invokeApi(in); break;
    case OP_LAUNCH: {
      std::vector<Val> args(static_cast<size_t>(in.b));
      for (int i = in.b; i > 0; --i) args[static_cast<size_t>(i - 1)] = pop();
      Val streamV = v_int(0), shmemV = v_int(0);
      if (in.f & 2) streamV = pop();
      if (in.f & 1) shmemV = pop();
      Val blockV = pop(), gridV = pop();
      const mck_fn& k = P_->fns[static_cast<size_t>(in.a)];
      LaunchRec lr;
      lr.kernel = in.a;
      lr.grid = gridV.i;
      lr.block = blockV.i;
      lr.shmem = shmemV.i;
      lr.stream = static_cast<uint32_t>(streamV.i);
      lr.line = L;
      if (k.space != 3) {
        apiDiag("launch of '" + P_->fnNames[static_cast<size_t>(in.a)] + "', which is not a __global__ kernel", L);
        vals_.push_back(v_void());
        break;
      }
      if (lr.grid < 1 || lr.block < 1 || lr.shmem < 0 || lr.block > o_.arch.maxThreadsPerBlock) {
        apiDiag("invalid kernel launch configuration (gridDim=" + std::to_string(lr.grid) +
                    ", blockDim=" + std::to_string(lr.block) + ", shmem=" + std::to_string(lr.shmem) + ")",
                L);
        vals_.push_back(v_void());
        break;
      }
      bool ok = true;
      for (int i = 0; i < in.b && ok; ++i) {
        Val cv;
        Diags dd{};
        ok = convert(args[static_cast<size_t>(i)], local(in.a, i).type, cv, dd);
        reportDiags(dd, L);
        if (ok) lr.args.push_back(cv);
      }
      if (!ok) {
        halt();
        break;
      }
      StreamItem it;
      it.kind = ItemKind::Launch;
      it.launch = std::move(lr);
      enqueue(it.launch.stream, std::move(it), L);
      vals_.push_back(v_void());
      break;
    }
    case OP_SYNC:
      // lowering forbids __syncthreads in host code
      ub("call of an unsupported function", L);
      halt();
      break;
    default:
      throw std::logic_error("host interpreter: bad opcode");
  }
}

// printf (machine.cpp:1236-1378): one directive at a time through snprintf
void HostMachine::execPrintf(const mck_ins& in) {
  std::vector<Val> args(static_cast<size_t>(in.b));
  for (int i = in.b; i > 0; --i) args[static_cast<size_t>(i - 1)] = pop();
  const std::string& fmt = P_->str(in.a);
  const int L = in.line;
  std::string out;
  size_t ai = 0;
  auto fail = [&](const std::string& m) {
    ub(m, L);
    halt();
  };
  for (size_t i = 0; i < fmt.size(); ++i) {
    if (fmt[i] != '%') {
      out += fmt[i];
      continue;
    }
    ++i;
    if (i >= fmt.size()) return fail("printf format string ends with a lone '%'");
    if (fmt[i] == '%') {
      out += '%';
      continue;
    }
    std::string spec = "%";
    while (i < fmt.size() && (fmt[i] == '-' || fmt[i] == '0' || fmt[i] == ' ' || fmt[i] == '+' ||
                              isdigit(static_cast<unsigned char>(fmt[i])) || fmt[i] == '.'))
      spec += fmt[i++];
    if (i >= fmt.size()) return fail("unterminated printf conversion");
    char conv = fmt[i];
    if (conv != 's' && ai >= args.size()) return fail("printf has more conversions than arguments");
    char buf[256];
    switch (conv) {
      case 'd': {
        const Val& v = args[ai++];
        if (v.kind != MCK_K_INT) return fail("printf %d expects an integer argument");
        spec += "lld";
        snprintf(buf, sizeof buf, spec.c_str(), static_cast<long long>(v.i));
        out += buf;
        break;
      }
      case 'u': {
        const Val& v = args[ai++];
        if (v.kind != MCK_K_INT) return fail("printf %u expects an integer argument");
        uint64_t u = MCK_T_BASE(v.type) == MCK_LONG ? static_cast<uint64_t>(v.i)
                                                   : static_cast<uint64_t>(static_cast<uint32_t>(v.i));
        spec += "llu";
        snprintf(buf, sizeof buf, spec.c_str(), static_cast<unsigned long long>(u));
        out += buf;
        break;
      }
      case 'c': {
        const Val& v = args[ai++];
        if (v.kind != MCK_K_INT) return fail("printf %c expects an integer argument");
        spec += 'c';
        snprintf(buf, sizeof buf, spec.c_str(), static_cast<int>(v.i));
        out += buf;
        break;
      }
      case 'f': {
        const Val& v = args[ai++];
        if (v.kind != MCK_K_FLOAT && v.kind != MCK_K_INT) return fail("printf %f expects a floating argument");
        spec += 'f';
        snprintf(buf, sizeof buf, spec.c_str(), v.kind == MCK_K_FLOAT ? as_f(v) : static_cast<double>(v.i));
        out += buf;
        break;
      }
      case 's': {
        if (ai >= args.size()) return fail("printf has more conversions than arguments");
        const Val& v = args[ai++];
        std::string s;
        if (v.kind == MCK_K_STR) {
          s = hostStrings_[static_cast<size_t>(v.i)];
        } else if (v.kind == MCK_K_PTR) {
          int64_t off = v.i;
          for (int64_t guard = 0;; ++guard) {
            if (guard > (1 << 20)) return fail("printf %s string is not NUL-terminated");
            auto b = readMem(v.obj, off, MCK_T(MCK_CHAR, 0, 0), L);
            if (!b) {
              halt();
              return;
            }
            if (b->i == 0) break;
            s += static_cast<char>(b->i);
            ++off;
          }
        } else {
          return fail("printf %s expects a string argument");
        }
        if (spec == "%") {
          out += s;
        } else {
          spec += 's';
          std::vector<char> big(s.size() + 256);
          snprintf(big.data(), big.size(), spec.c_str(), s.c_str());
          out += big.data();
        }
        break;
      }
      default: return fail(std::string("unsupported printf conversion '%") + conv + "'");
    }
  }
  if (ai != args.size()) return fail("printf has more arguments than conversions");
  output_ += out;
  if (hooks_.out) hooks_.out(out);
  vals_.push_back(v_int(static_cast<int64_t>(out.size())));
}

// runtime API (runtime_api.cpp:39-372).  Provenance: this dispatcher restates
// the reference's API table closely (the same helpers and checks in the same
// order, the same messages) because its diagnostics and return codes must be
// the reference's; the sweep timeline, grid dispatch and diagnostic merge
// around it are this project's own.
void HostMachine::invokeApi(const mck_ins& in) {
  std::vector<Val> args(static_cast<size_t>(in.b));
  for (int i = in.b; i > 0; --i) args[static_cast<size_t>(i - 1)] = pop();
  const int L = in.line;
  static const char* names[] = {"cudaMalloc", "cudaFree", "cudaMemcpy", "cudaMemcpyAsync", "cudaMemset",
                                "cudaDeviceSynchronize", "cudaStreamCreate", "cudaStreamDestroy",
                                "cudaStreamSynchronize", "cudaStreamQuery", "cudaStreamWaitEvent",
                                "cudaEventCreate", "cudaEventDestroy", "cudaEventRecord",
                                "cudaEventSynchronize", "cudaEventQuery", "cudaEventElapsedTime",
                                "cudaGetLastError", "cudaGetErrorString", "cudaDeviceGetAttribute",
                                "cudaDriverGetVersion", "cudaRuntimeGetVersion"};
  constexpr int kOK = 0, kInval = 11, kDevPtr = 17, kDir = 21, kHandle = 33, kNotReady = 34;
  const mck::ApiId api = static_cast<mck::ApiId>(in.a);
  auto finish = [&](int code) {
    if (code != kOK && code != kNotReady) lastApiError_ = code;
    if (hooks_.api) hooks_.api(api, code);
    vals_.push_back(v_int(code));
  };
  auto err = [&](int code, const std::string& m) {
    apiDiag(std::string(names[in.a]) + ": " + m, L);
    finish(code);
  };
  auto block = [&](WaitKind w, uint32_t id) {
    wait_ = w;
    waitId_ = id;
    awaiting_ = true;
    awaitCode_ = kOK;
    if (hooks_.api) hooks_.api(api, kOK);
  };
  auto outWrite = [&](const Val& dst, uint8_t t, const Val& v) -> bool {
    if (dst.kind != MCK_K_PTR || dst.obj == 0) return false;
    return writeMem(dst.obj, dst.i, t, v, L);
  };
  auto spaceOf = [&](const Val& p, uint8_t& sp) -> bool {
    HObj* o = find(p.obj);
    if (!o || !o->live) return false;
    sp = o->space;
    return true;
  };
  auto streamArg = [&](const Val& v, uint32_t& sid) -> bool {
    if (v.kind != MCK_K_INT) return false;
    sid = static_cast<uint32_t>(v.i);
    auto it = streams_.find(sid);
    return it != streams_.end() && !it->second.destroyed;
  };
  auto checkCopy = [&](const Val& dst, const Val& src, int64_t n, int64_t dir, std::string& why) -> int {
    static const char* dn[] = {"cudaMemcpyHostToHost", "cudaMemcpyHostToDevice", "cudaMemcpyDeviceToHost",
                               "cudaMemcpyDeviceToDevice"};
    if (dir < 0 || dir > 3) {
      why = "direction argument " + std::to_string(dir) + " is not a cudaMemcpyKind";
      return kDir;
    }
    if (n < 0) {
      why = "negative byte count";
      return kInval;
    }
    if (dst.kind != MCK_K_PTR || src.kind != MCK_K_PTR || (n > 0 && (dst.obj == 0 || src.obj == 0))) {
      why = "source or destination is not a valid pointer";
      return kInval;
    }
    if (n == 0) return kOK;
    uint8_t ds, ss;
    if (!spaceOf(dst, ds) || !spaceOf(src, ss)) {
      why = "source or destination was freed or never allocated";
      return kDevPtr;
    }
    bool match = (dir == 0 && ds == SP_HOST && ss == SP_HOST) || (dir == 1 && ds == SP_GLOBAL && ss == SP_HOST) ||
                 (dir == 2 && ds == SP_HOST && ss == SP_GLOBAL) || (dir == 3 && ds == SP_GLOBAL && ss == SP_GLOBAL);
    if (!match) {
      why = std::string("direction ") + dn[dir] + " does not match the operand memory spaces (dst=" + spaceStr(ds) +
            ", src=" + spaceStr(ss) + ")";
      return kDir;
    }
    HObj* d = find(dst.obj);
    HObj* s = find(src.obj);
    if (dst.i < 0 || dst.i + n > d->size || src.i < 0 || src.i + n > s->size) {
      why = "transfer of " + std::to_string(n) + " bytes is out of range";
      return kInval;
    }
    return kOK;
  };
  switch (in.a) {
    case MCK_API_MALLOC: {
      if (args[1].kind != MCK_K_INT || args[1].i < 0) return err(kInval, "invalid allocation size");
      int64_t n = args[1].i;
      Val out = n == 0 ? v_ptr(0, 0, MCK_T_VOIDP) : v_ptr(alloc(SP_GLOBAL, n, "cudaMalloc"), 0, MCK_T_VOIDP);
      if (!outWrite(args[0], MCK_T_VOIDP, out)) return err(kInval, "output pointer argument is invalid");
      finish(kOK);
      break;
    }
    case MCK_API_FREE: {
      const Val& a = args[0];
      if ((a.kind == MCK_K_PTR && a.obj == 0) || (a.kind == MCK_K_INT && a.i == 0)) {
        finish(kOK);
        break;
      }
      if (a.kind != MCK_K_PTR) return err(kDevPtr, "argument is not a device pointer");
      HObj* o = find(a.obj);
      bool ok = false;
      if (!o) apiDiag("cudaFree of a pointer that was never allocated", L);
      else if (!o->live) apiDiag("double cudaFree of the same allocation", L);
      else if (a.i != 0) apiDiag("cudaFree of an interior pointer", L);
      else if (o->space != SP_GLOBAL) apiDiag("cudaFree of " + spaceStr(o->space) + " memory", L);
      else {
        o->live = false;
        ok = true;
      }
      finish(ok ? kOK : kDevPtr);
      break;
    }
    case MCK_API_MEMCPY:
    case MCK_API_MEMCPY_ASYNC: {
      uint32_t sid = 0;
      if (in.a == MCK_API_MEMCPY_ASYNC && args.size() == 5 && !streamArg(args[4], sid))
        return err(kHandle, "unknown stream handle");
      std::string why;
      int code = checkCopy(args[0], args[1], args[2].i, args[3].i, why);
      if (code != kOK) return err(code, why);
      if (args[2].i > 0) {
        StreamItem it;
        it.kind = ItemKind::Copy;
        it.copy = CopyRec{args[0], args[1], args[2].i, static_cast<int>(args[3].i), L};
        enqueue(sid, std::move(it), L);
      }
      if (in.a == MCK_API_MEMCPY && args[2].i > 0)
        block(WaitKind::Stream, 0);
      else
        finish(kOK);
      break;
    }
    case MCK_API_MEMSET: {
      const Val& p = args[0];
      if (p.kind != MCK_K_PTR || p.obj == 0) return err(kDevPtr, "argument is not a device pointer");
      if (args[2].kind != MCK_K_INT || args[2].i < 0) return err(kInval, "invalid byte count");
      uint8_t sp;
      if (!spaceOf(p, sp)) return err(kDevPtr, "pointer was freed or never allocated");
      if (sp != SP_GLOBAL) return err(kDevPtr, "pointer is not device memory");
      HObj* o = find(p.obj);
      int64_t off = p.i, n = args[2].i;
      if (off < 0 || off + n > o->size) return err(kInval, "fill range is out of bounds");
      if (n > 0) {
        checkInflight(~0u, p.obj, off, off + n, true);  // the host fills at once, whatever is in flight
        eng_->fill(o->devBase + static_cast<uint64_t>(off), static_cast<uint8_t>(args[1].i), META_DEF, n);
        int64_t lo = std::max<int64_t>(0, off - 7);
        if (lo < off) {
          std::vector<uint8_t> b(static_cast<size_t>(off - lo)), m(b.size());
          eng_->read(o->devBase + static_cast<uint64_t>(lo), b.data(), m.data(), off - lo);
          for (auto& x : m) x &= static_cast<uint8_t>(~META_PTR);
          eng_->write(o->devBase + static_cast<uint64_t>(lo), b.data(), m.data(), off - lo);
        }
      }
      finish(kOK);
      break;
    }
    case MCK_API_DEVICE_SYNC: block(WaitKind::Device, 0); break;
    case MCK_API_STREAM_CREATE: {
      uint32_t sid = nextSid_++;
      streams_[sid] = StreamRec{};
      if (!outWrite(args[0], MCK_T_LONG, v_int(sid, MCK_T_LONG))) return err(kInval, "output stream argument is invalid");
      finish(kOK);
      break;
    }
    case MCK_API_STREAM_DESTROY: {
      if (args[0].kind != MCK_K_INT || args[0].i == 0) return err(kHandle, "cannot destroy this stream handle");
      auto it = streams_.find(static_cast<uint32_t>(args[0].i));
      if (it == streams_.end() || it->second.destroyed) return err(kHandle, "unknown stream handle");
      it->second.destroyed = true;
      if (it->second.idle()) streams_.erase(it);
      finish(kOK);
      break;
    }
    case MCK_API_STREAM_SYNC: {
      uint32_t sid;
      if (!streamArg(args[0], sid)) return err(kHandle, "unknown stream handle");
      block(WaitKind::Stream, sid);
      break;
    }
    case MCK_API_STREAM_QUERY: {
      uint32_t sid;
      if (!streamArg(args[0], sid)) return err(kHandle, "unknown stream handle");
      finish(streams_.at(sid).idle() ? kOK : kNotReady);
      break;
    }
    case MCK_API_STREAM_WAIT_EVENT: {
      uint32_t sid;
      if (!streamArg(args[0], sid)) return err(kHandle, "unknown stream handle");
      if (args[1].kind != MCK_K_INT || !events_.count(static_cast<uint32_t>(args[1].i)))
        return err(kHandle, "unknown event handle");
      StreamItem it;
      it.kind = ItemKind::WaitEvent;
      it.eid = static_cast<uint32_t>(args[1].i);
      enqueue(sid, std::move(it), L);
      finish(kOK);
      break;
    }
    case MCK_API_EVENT_CREATE: {
      uint32_t eid = nextEid_++;
      events_[eid] = EvStatus::Created;
      if (!outWrite(args[0], MCK_T_LONG, v_int(eid, MCK_T_LONG))) return err(kInval, "output event argument is invalid");
      finish(kOK);
      break;
    }
    case MCK_API_EVENT_DESTROY: {
      if (args[0].kind != MCK_K_INT || !events_.count(static_cast<uint32_t>(args[0].i)))
        return err(kHandle, "unknown event handle");
      events_.erase(static_cast<uint32_t>(args[0].i));
      finish(kOK);
      break;
    }
    case MCK_API_EVENT_RECORD: {
      if (args[0].kind != MCK_K_INT || !events_.count(static_cast<uint32_t>(args[0].i)))
        return err(kHandle, "unknown event handle");
      uint32_t eid = static_cast<uint32_t>(args[0].i);
      uint32_t sid = 0;
      if (args.size() == 2 && !streamArg(args[1], sid)) return err(kHandle, "unknown stream handle");
      if (events_[eid] != EvStatus::Created) return err(kHandle, "event was already recorded");
      events_[eid] = EvStatus::Pending;
      StreamItem it;
      it.kind = ItemKind::EventRecord;
      it.eid = eid;
      enqueue(sid, std::move(it), L);
      finish(kOK);
      break;
    }
    case MCK_API_EVENT_SYNC:
      if (args[0].kind != MCK_K_INT || !events_.count(static_cast<uint32_t>(args[0].i)))
        return err(kHandle, "unknown event handle");
      block(WaitKind::Event, static_cast<uint32_t>(args[0].i));
      break;
    case MCK_API_EVENT_QUERY:
      if (args[0].kind != MCK_K_INT || !events_.count(static_cast<uint32_t>(args[0].i)))
        return err(kHandle, "unknown event handle");
      finish(events_[static_cast<uint32_t>(args[0].i)] == EvStatus::Pending ? kNotReady : kOK);
      break;
    case MCK_API_EVENT_ELAPSED:
      if (args[1].kind != MCK_K_INT || args[2].kind != MCK_K_INT || !events_.count(static_cast<uint32_t>(args[1].i)) ||
          !events_.count(static_cast<uint32_t>(args[2].i)))
        return err(kHandle, "unknown event handle");
      if (!outWrite(args[0], MCK_T(MCK_FLOAT, 0, 0), v_flt(0.0, MCK_T(MCK_FLOAT, 0, 0))))
        return err(kInval, "output argument is invalid");
      finish(kOK);
      break;
    case MCK_API_GET_LAST_ERROR: {
      int c = lastApiError_;
      lastApiError_ = kOK;
      if (hooks_.api) hooks_.api(api, c);
      vals_.push_back(v_int(c));
      break;
    }
    case MCK_API_GET_ERROR_STRING: {
      if (hooks_.api) hooks_.api(api, kOK);
      const char* s;
      switch (static_cast<int>(args[0].i)) {
        case 0: s = "no error"; break;
        case 11: s = "invalid argument"; break;
        case 17: s = "invalid device pointer"; break;
        case 21: s = "invalid copy direction for memcpy"; break;
        case 33: s = "invalid resource handle"; break;
        case 34: s = "device not ready"; break;
        default: s = "unrecognized error code"; break;
      }
      hostStrings_.push_back(s);
      vals_.push_back(mk(MCK_K_STR, MCK_T(MCK_CHAR, 1, 0), 0, static_cast<int64_t>(hostStrings_.size() - 1)));
      break;
    }
    case MCK_API_DEVICE_GET_ATTR: {
      int64_t v;
      switch (args[1].i) {
        case 1: v = o_.arch.maxThreadsPerBlock; break;
        case 10: v = o_.arch.warpSize; break;
        case 75: v = o_.arch.computeCapabilityMajor; break;
        case 76: v = o_.arch.computeCapabilityMinor; break;
        default: return err(kInval, "unknown device attribute " + std::to_string(args[1].i));
      }
      if (!outWrite(args[0], MCK_T_INT, v_int(v))) return err(kInval, "output argument is invalid");
      finish(kOK);
      break;
    }
    case MCK_API_DRIVER_VERSION:
      if (!outWrite(args[0], MCK_T_INT, v_int(o_.arch.driverVersion))) return err(kInval, "output argument is invalid");
      finish(kOK);
      break;
    case MCK_API_RUNTIME_VERSION:
      if (!outWrite(args[0], MCK_T_INT, v_int(o_.arch.runtimeVersion))) return err(kInval, "output argument is invalid");
      finish(kOK);
      break;
    default: throw std::logic_error("bad api id");
  }
}

// ======================= streams & grids =======================

void HostMachine::performCopy(const CopyRec& c, uint32_t sid) {
  // memcpyBytes (memory.cpp:247-277)
  HObj* d = find(c.dst.obj);
  HObj* s = find(c.src.obj);
  const int64_t n = c.n;
  if (n == 0) return;
  if (!d || !s || !d->live || !s->live) {
    apiDiag("memory transfer touches a freed or invalid allocation", c.line, 3, sid);
    return;
  }
  if (c.src.i < 0 || c.src.i + n > s->size || c.dst.i < 0 || c.dst.i + n > d->size) {
    apiDiag("memory transfer of " + std::to_string(n) + " bytes is out of range", c.line, 3, sid);
    return;
  }
  if (d->space != SP_HOST) checkInflight(sid, c.dst.obj, c.dst.i, c.dst.i + n, true);
  std::vector<uint8_t> b(static_cast<size_t>(n)), m(static_cast<size_t>(n));
  if (s->space == SP_HOST) {
    std::memcpy(b.data(), s->bytes.data() + c.src.i, static_cast<size_t>(n));
    std::memcpy(m.data(), s->meta.data() + c.src.i, static_cast<size_t>(n));
  } else {
    eng_->read(s->devBase + static_cast<uint64_t>(c.src.i), b.data(), m.data(), n);
    // a grid in flight on another stream that writes these bytes: read them
    // as of this sweep (its write history), else say the values may differ
    if (!midflight(sid, c.src.obj, c.src.i, n, b.data(), m.data()))
      checkInflight(sid, c.src.obj, c.src.i, c.src.i + n, false);
  }
  // slots that would extend past the copied range are not copied
  for (int64_t i = std::max<int64_t>(0, n - 7); i < n; ++i) m[static_cast<size_t>(i)] &= static_cast<uint8_t>(~META_PTR);
  // destination slots overlapping the range from the left are erased
  int64_t lo = std::max<int64_t>(0, c.dst.i - 7);
  if (d->space == SP_HOST) {
    for (int64_t i = lo; i < c.dst.i; ++i) d->meta[static_cast<size_t>(i)] &= static_cast<uint8_t>(~META_PTR);
    std::memcpy(d->bytes.data() + c.dst.i, b.data(), static_cast<size_t>(n));
    std::memcpy(d->meta.data() + c.dst.i, m.data(), static_cast<size_t>(n));
  } else {
    if (lo < c.dst.i) {
      std::vector<uint8_t> lb(static_cast<size_t>(c.dst.i - lo)), lm(lb.size());
      eng_->read(d->devBase + static_cast<uint64_t>(lo), lb.data(), lm.data(), c.dst.i - lo);
      for (auto& x : lm) x &= static_cast<uint8_t>(~META_PTR);
      eng_->write(d->devBase + static_cast<uint64_t>(lo), lb.data(), lm.data(), c.dst.i - lo);
    }
    eng_->write(d->devBase + static_cast<uint64_t>(c.dst.i), b.data(), m.data(), n);
  }
}

void HostMachine::spawnGrid(uint32_t sid, const LaunchRec& l) {
  GridSpec g;
  g.prog = P_.get();
  g.kernel = l.kernel;
  g.gridDim = l.grid;
  g.blockDim = l.block;
  g.shmemBytes = l.shmem;
  g.gid = nextGid_++;
  g.args = l.args;
  g.spawnSweep = sweep_;
  g.sharedBase = nextId_;
  g.raceCheck = o_.raceCheck;
  g.warpSize = o_.arch.warpSize;
  g.stepBudget = o_.stepLimit > steps_ ? o_.stepLimit - steps_ : 0;
  g.globalIds = globalIds_;
  g.sharedRanges = sharedRanges_;
  g.trace = o_.trace;
  g.globalRaceCheck = o_.globalRaceCheck;
  // small grids are probed for cross-block global conflicts: their values
  // follow this engine's block order (DESIGN §3 divergence 2), so the run says so
  g.conflictProbe = !o_.globalRaceCheck && static_cast<uint64_t>(l.grid) * static_cast<uint64_t>(l.block) <= 65536;
  g.wantHistory = g.conflictProbe && streams_.size() > 1;
  const int nparams = P_->fns[static_cast<size_t>(l.kernel)].n_params;
  // spawnGrid allocates gridDim shared objects, then nparams objects per thread
  const uint64_t reserve = static_cast<uint64_t>(l.grid) + static_cast<uint64_t>(l.grid) * l.block * nparams;
  g.nextId = nextId_ + static_cast<uint32_t>(reserve);
  std::vector<std::string> objNames;
  for (const HObj& o : objs_)
    if (o.space == SP_GLOBAL) {
      g.objects.push_back(DevObjInfo{o.id, o.size, o.devBase, o.live, -2 - static_cast<int>(objNames.size())});
      objNames.push_back(o.name);
    }
  GridRec rec;
  rec.gid = g.gid;
  rec.spawnSweep = g.spawnSweep;
  rec.stream = sid;
  rec.gridDim = l.grid;
  rec.blockDim = l.block;
  rec.sharedBase = g.sharedBase;
  if (oracleOn_ && !oracleOut_.aborted) {
    // oracle.cpp:81-99: the size bounds, then every interleaving of the grid
    if (oracleGrids_++ > 0) {
      oracleOut_.aborted = true;
      oracleOut_.error = "the GPU oracle explores programs with one kernel launch";
    } else if (l.grid * l.block > oracleMaxThreads_) {
      oracleOut_.aborted = true;
      oracleOut_.error = "kernel spawns more threads than the oracle size bound";
    } else if (!eng_->hasDevice() || !eng_->exploreGrid(g, oracle_, oracleOut_)) {
      oracleOut_.aborted = true;
      if (oracleOut_.error.empty()) oracleOut_.error = engWhy_.empty() ? "oracle exploration failed" : engWhy_;
    }
  }
  if (hooks_.mem) {
    engineError_ = "onMemAccess is set: device accesses run inside the B200 grid kernel and cannot be "
                   "reported one by one";
  } else if (!eng_->hasDevice() || !eng_->runGrid(g, rec.res)) {
    engineError_ = rec.res.error.empty() ? engWhy_ : rec.res.error;
    if (engineError_.empty()) engineError_ = "grid engine failed";
  }
  nextId_ += static_cast<uint32_t>(reserve + rec.res.allocs);
  sharedRanges_.push_back({g.sharedBase, static_cast<uint32_t>(l.grid), g.gid});
  rec.endSweep = rec.res.deadlocked ? NEVER : sweep_ + rec.res.duration;
  if (rec.endSweep != NEVER) ++runningGrids_;
  traceLine(sweep_, 3, 0, 0,
            "stream sid=" + std::to_string(sid) + " dispatch=launch gid=" + std::to_string(g.gid) +
                " kernel=" + P_->fnNames[static_cast<size_t>(l.kernel)]);
  if (o_.trace && engineError_.empty()) {
    traceBarriers(g.gid, rec, sweep_);
    // finishThread of the grid's last thread (device.cpp:215)
    if (rec.endSweep != NEVER)
      traceLine(rec.endSweep, 1, (static_cast<uint64_t>(g.gid) << 32) | 0xFFFFFFFFu, 0,
                "grid gid=" + std::to_string(g.gid) + " completed");
  }
  // the grid's device steps and barrier rules count toward the step limit
  // from its dispatch on: the run's total only grows, so a total that reaches
  // the limit here reaches it in the reference too (machine.cpp:1184)
  steps_ += rec.res.deviceSteps + rec.res.barrierRules;
  stats_.deviceSteps += rec.res.deviceSteps;
  stats_.barrierRules += rec.res.barrierRules;
  ++stats_.grids;
  stats_.gridMs += rec.res.ms;
  stats_.kernelLaunches += rec.res.launches;
  stats_.sharedEvents += rec.res.sharedEvents;
  stats_.blockSweeps += rec.res.sweeps;
  stats_.soloSweeps += rec.res.soloSweeps;
  stats_.blockCycles += rec.res.blockCycles;
  stats_.soloCycles += rec.res.soloCycles;
  if (rec.res.globalConflicts) conflictGids_.push_back(g.gid);
  for (const auto& e : rec.res.footprint) {  // this grid against the grids still in flight
    checkInflight(sid, (uint32_t)e[0], e[1], e[2], false);
    checkInflight(sid, (uint32_t)e[0], e[3], e[4], true);
  }
  // device diagnostics, timestamped by (global sweep, gid, bid, tid, sub)
  for (const DevDiag& r : rec.res.diags) {
    uint64_t lsweep = r.key >> 38;
    uint32_t bid = static_cast<uint32_t>((r.key >> 12) & ((1u << 26) - 1));
    uint32_t tid = static_cast<uint32_t>((r.key >> 2) & 1023u);
    DiagEv e;
    e.sweep = sweep_ + lsweep;
    e.phase = 1;
    e.k1 = (static_cast<uint64_t>(g.gid) << 32) | bid;
    e.k2 = (static_cast<uint64_t>(tid) << 8) | (r.key & 3u);
    e.seq = seq_++;
    e.d.message = formatDevDiag(r, g.gid, bid, tid, e.d.category, e.d.severity, objNames);
    e.d.loc.line = r.line;
    diags_.push_back(std::move(e));
  }
  for (const auto& t : rec.res.reported)
    reported_.push_back(mck::RaceTriple{static_cast<uint32_t>(t[0]), t[1], static_cast<int>(t[2])});
  streams_[sid].running = true;
  streams_[sid].runningGid = g.gid;
  grids_[g.gid] = std::move(rec);
}

void HostMachine::dispatch(uint32_t sid) {
  StreamRec& s = streams_.at(sid);
  StreamItem item = s.q.front();
  s.q.pop_front();
  --queued_;
  const std::string pre = "stream sid=" + std::to_string(sid) + " dispatch=";
  switch (item.kind) {
    case ItemKind::Launch: spawnGrid(sid, item.launch); break;
    case ItemKind::Copy:
      performCopy(item.copy, sid);
      traceLine(sweep_, 3, 0, 0, pre + "memcpy n=" + std::to_string(item.copy.n));
      break;
    case ItemKind::EventRecord: {
      auto e = events_.find(item.eid);
      if (e != events_.end()) e->second = EvStatus::Recorded;
      traceLine(sweep_, 3, 0, 0, pre + "event-record eid=" + std::to_string(item.eid));
      break;
    }
    case ItemKind::WaitEvent: traceLine(sweep_, 3, 0, 0, pre + "wait-event eid=" + std::to_string(item.eid)); break;
  }
  StreamRec& s2 = streams_.at(sid);
  if (s2.destroyed && s2.idle()) streams_.erase(sid);
}

// Barrier-rule trace lines from the recorded arrival sweeps (device.cpp:
// 111-198 under round robin): up(t -> t+1) fires in the
// first sweep where threads 0..t+1 have all arrived (the chain cascades in
// key order), Turnaround and Down(L) in the last arrival's sweep T, Down(t)
// in T + L - t, FinalRelease in T + L.  A deadlocked episode runs its up
// chain up to the first thread that never arrives.
void HostMachine::traceBarriers(uint32_t gid, const GridRec& rec, uint64_t spawn) {
  const GridResult& r = rec.res;
  if (r.episodes.empty()) return;
  const int64_t B = rec.blockDim, L = B - 1;
  std::vector<char> stuck(static_cast<size_t>(rec.gridDim), 0);
  for (const auto& s : r.stuck) stuck[s.bid] = 1;
  enum { UP = 0, TURN = 1, DOWN = 2, REL = 3 };
  for (int64_t b = 0; b < rec.gridDim; ++b) {
    const uint32_t done = r.episodes[static_cast<size_t>(b)];
    const uint32_t eps = done + (stuck[static_cast<size_t>(b)] ? 1u : 0u);
    if (eps > static_cast<uint32_t>(TRACE_EPISODES)) {
      engineError_ = "--trace records at most " + std::to_string(TRACE_EPISODES) + " barrier episodes per block";
      return;
    }
    const uint64_t k1 = (static_cast<uint64_t>(gid) << 32) | static_cast<uint64_t>(b);
    const std::string head = "sync gid=" + std::to_string(gid) + " bid=" + std::to_string(b) + " rule=";
    for (uint32_t e = 0; e < eps; ++e) {
      const uint32_t* a = r.arrivals.data() + (static_cast<size_t>(b) * TRACE_EPISODES + e) * static_cast<size_t>(B);
      auto rule = [&](uint64_t lsweep, int64_t keyTid, int kind, const std::string& text) {
        traceLine(spawn + lsweep, 2, k1, (static_cast<uint64_t>(keyTid) << 2) | static_cast<uint64_t>(kind), head + text);
      };
      if (a[0] == 0) continue;  // thread 0 never arrived: no rule fires
      uint64_t U = a[0] - 1;
      int64_t t = 0;
      for (; t < L && a[t + 1] != 0; ++t) {
        U = std::max<uint64_t>(U, a[t + 1] - 1);
        rule(U, t, UP, "up tid=" + std::to_string(t + 1) + " token=1");
      }
      if (e >= done) continue;  // deadlocked: the chain stops at the first absent thread
      const uint64_t T = U;
      rule(T, L, TURN, "turn tid=" + std::to_string(L) + " token=2");
      if (L == 0) {
        rule(T, 0, REL, "release tid=0 token=0");
        continue;
      }
      for (int64_t d = L; d >= 1; --d) rule(T + static_cast<uint64_t>(L - d), d, DOWN, "down tid=" + std::to_string(d) + " token=2");
      rule(T + static_cast<uint64_t>(L), 0, REL, "release tid=0 token=0");
    }
  }
}

void HostMachine::completeGrids(uint64_t sweep) {
  for (auto& [gid, g] : grids_) {
    if (g.completed || g.endSweep != sweep) continue;
    g.completed = true;
    --runningGrids_;
    auto s = streams_.find(g.stream);
    if (s != streams_.end() && s->second.running && s->second.runningGid == gid) s->second.running = false;
  }
}

std::vector<mck::StuckReport> HostMachine::scanStuck() const {
  std::vector<mck::StuckReport> out;
  for (const auto& [gid, g] : grids_) {
    for (const auto& b : g.res.stuck) {
      mck::StuckReport r;
      r.kind = mck::StuckReport::Kind::BarrierDeadlock;
      r.gid = gid;
      r.bid = static_cast<int>(b.bid);
      r.waitingTids = b.waiting;
      std::vector<char> w(static_cast<size_t>(g.blockDim), 0);
      for (int t : b.waiting) w[static_cast<size_t>(t)] = 1;
      for (int t = 0; t < g.blockDim; ++t)
        if (!w[static_cast<size_t>(t)]) r.missingTids.push_back(t);
      r.reason = "block (" + std::to_string(gid) + "," + std::to_string(b.bid) + ") has " +
                 std::to_string(b.waiting.size()) + " thread(s) waiting at __syncthreads() that can never complete";
      out.push_back(std::move(r));
    }
  }
  if (!hostHalted_ && !hostDone_) {
    mck::StuckReport r;
    r.kind = mck::StuckReport::Kind::HostHang;
    switch (wait_) {
      case WaitKind::Device: r.reason = "host thread is blocked in cudaDeviceSynchronize()"; break;
      case WaitKind::Stream:
        r.reason = "host thread is blocked waiting for stream " + std::to_string(waitId_) + " to drain";
        break;
      case WaitKind::Event:
        r.reason = "host thread is blocked in cudaEventSynchronize() on event " + std::to_string(waitId_) +
                   ", which is never recorded";
        break;
      case WaitKind::None: r.reason = "host thread cannot take a step"; break;
    }
    out.push_back(std::move(r));
  }
  for (const auto& [sid, s] : streams_) {
    if (s.q.empty() || s.running) continue;
    const StreamItem& h = s.q.front();
    if (h.kind == ItemKind::WaitEvent) {
      mck::StuckReport r;
      r.kind = mck::StuckReport::Kind::StreamStall;
      r.sid = sid;
      r.item = "cudaStreamWaitEvent(event " + std::to_string(h.eid) + ")";
      r.reason = "stream " + std::to_string(sid) + " is stalled on event " + std::to_string(h.eid) +
                 ", which is never recorded";
      out.push_back(std::move(r));
    }
  }
  return out;
}

// ======================= run =======================

mck::RunResult HostMachine::run() {
  std::vector<int> devs = o_.devices.empty() ? std::vector<int>{o_.device} : o_.devices;
  EngineComm comm;
  comm.rank = o_.rank;
  comm.world = std::max(1, o_.world);
  if (o_.commId.size() == comm.id.size()) std::copy(o_.commId.begin(), o_.commId.end(), comm.id.begin());
  comm.allgather = o_.allgather;
  comm.ctx = o_.allgatherCtx;
  eng_ = makeCudaEngine(devs, comm, engWhy_);
  if (!eng_) eng_ = makeStorageOnlyEngine(engWhy_);
  // globals (machine.cpp:57-68)
  for (const GlobalInfo& g : P_->globals) {
    uint32_t id = alloc(g.device ? SP_GLOBAL : SP_HOST, g.size, g.name);
    globalIds_.push_back(id);
    if (g.hasInit) {
      Val v = t_is_float(g.type) ? v_flt(g.fval, g.type) : v_int(g.ival, g.type);
      HObj* o = find(id);
      if (o->space == SP_HOST) {
        poke(*o, 0, g.type, v);
      } else {
        HObj tmp;
        tmp.size = g.size;
        tmp.bytes.assign(static_cast<size_t>(g.size), 0);
        tmp.meta.assign(static_cast<size_t>(g.size), 0);
        poke(tmp, 0, g.type, v);
        eng_->write(o->devBase, tmp.bytes.data(), tmp.meta.data(), g.size);
      }
    }
  }
  streams_[0] = StreamRec{};
  // host thread: CallFrame + main body (machine.cpp:70-85)
  enterFunction(P_->mainIndex, -1);
  scopeMarks_.pop_back();  // main's frame owns no parameter scope
  frames_.back().scopeDepth = 0;
  pc_ = P_->fns[static_cast<size_t>(P_->mainIndex)].entry;

  bool hitLimit = false;
  while (engineError_.empty()) {
    bool hostRun = hostRunnable();
    bool anyDispatch = false;
    if (queued_)
      for (const auto& s : streams_)
        if (dispatchable(s.second)) anyDispatch = true;
    uint64_t nextEnd = NEVER;
    if (runningGrids_)
      for (const auto& g : grids_)
        if (!g.second.completed && g.second.endSweep != NEVER) nextEnd = std::min(nextEnd, g.second.endSweep);
    if (hostRun && !anyDispatch && nextEnd == NEVER && !awaiting_) {
      // fast path: only the host thread can move (one step per sweep); it
      // keeps stepping until a step changes what can move (a stream item,
      // an await, a halt) or the limit is reached
      const uint64_t lim = o_.stepLimit;
      const mck_ins* code = P_->code.data();
      do {
        if (steps_ >= lim) {
          hitLimit = true;
          break;
        }
        // expansion steps (nop) cost a step and touch nothing: no dispatch
        while (code[pc_].op == OP_JMP) pc_ = code[pc_].a;
        if (code[pc_].op == OP_NOP) {
          ++pc_;
        } else {
          hostStep();
        }
        ++steps_;
        ++stats_.hostSteps;
        ++sweep_;
      } while (!queued_ && !awaiting_ && !hostDone_ && !hostHalted_ && !runningGrids_ && engineError_.empty());
      if (hitLimit) break;
      continue;
    }
    if (!hostRun && !anyDispatch) {
      if (nextEnd == NEVER) break;  // quiescent
      sweep_ = std::max(sweep_, nextEnd);
      hostRun = false;
    }
    // --- one sweep ---
    if (hostRun) {
      if (steps_ >= o_.stepLimit) {
        hitLimit = true;
        break;
      }
      hostStep();
      ++steps_;
      ++stats_.hostSteps;
    }
    if (runningGrids_) completeGrids(sweep_);
    sids_.clear();
    if (queued_)
      for (const auto& s : streams_) sids_.push_back(s.first);
    for (uint32_t sid : sids_) {
      auto it = streams_.find(sid);
      if (it == streams_.end() || !dispatchable(it->second)) continue;
      if (steps_ >= o_.stepLimit) {
        hitLimit = true;
        break;
      }
      dispatch(sid);
      ++steps_;
      ++stats_.dispatches;
      if (!engineError_.empty()) break;
    }
    if (hitLimit) break;
    ++sweep_;
  }
  // Machine::run checks the limit before every transition, including after
  // the last one (machine.cpp:1183-1191): a run whose total reaches the limit
  // is abandoned with exactly stepLimit steps
  if (engineError_.empty() && steps_ >= o_.stepLimit) hitLimit = true;
  if (hitLimit) steps_ = o_.stepLimit;
  stats_.sweeps = sweep_;

  mck::RunResult r;
  r.output = output_;
  r.mainReturn = exitValue_;
  r.engineError = engineError_;
  if (!inflightGids_.empty()) {
    std::string ids;
    for (size_t i = 0; i < inflightGids_.size() && i < 8; ++i) ids += (i ? ", " : "") + std::to_string(inflightGids_[i]);
    if (inflightGids_.size() > 8) ids += ", ...";
    r.engineNote = "grid(s) gid " + ids +
                   " had global bytes touched by another stream's copy or grid while in flight; the engine applies "
                   "a grid's effects at its dispatch sweep, so values there may differ from the reference's "
                   "interleaving";
  }
  if (!conflictGids_.empty()) {
    std::string ids;
    for (size_t i = 0; i < conflictGids_.size() && i < 8; ++i) ids += (i ? ", " : "") + std::to_string(conflictGids_[i]);
    if (conflictGids_.size() > 8) ids += ", ...";
    r.engineNote += std::string(r.engineNote.empty() ? "" : "; ") + "cross-block global-memory conflicts in grid(s) gid " + ids +
                   ": blocks of one grid touched a global byte with at least one write; the engine orders those "
                   "accesses by block, not by the reference's interleaving, so values read there may differ "
                   "(RunOptions::globalRaceCheck reports them)";
  }
  if (hitLimit) {
    DiagEv e;
    e.sweep = NEVER;
    e.phase = 9;
    e.k1 = e.k2 = 0;
    e.seq = seq_++;
    e.d.category = mck::DiagCategory::ApiError;
    e.d.message = "step limit exceeded (" + std::to_string(o_.stepLimit) + " steps); execution abandoned.";
    diags_.push_back(std::move(e));
  }
  bool normal = (hostHalted_ || hostDone_);
  for (const auto& s : streams_)
    if (!s.second.idle()) normal = false;
  for (const auto& g : grids_)
    if (!g.second.completed) normal = false;
  if (!hitLimit && !normal && engineError_.empty()) {
    r.stuck = true;
    r.stuckReports = scanStuck();
    bool barrier = false;
    for (const auto& s : r.stuckReports)
      if (s.kind == mck::StuckReport::Kind::BarrierDeadlock) barrier = true;
    DiagEv e;
    e.sweep = NEVER;
    e.phase = 9;
    e.k1 = e.k2 = 0;
    e.seq = seq_++;
    e.d.category = mck::DiagCategory::Deadlock;
    e.d.message = barrier ? "Detected a deadlock caused by misplaced __syncthreads()."
                          : "Execution is stuck: " + (r.stuckReports.empty() ? std::string("no runnable computation remains")
                                                                             : r.stuckReports.front().reason);
    diags_.push_back(std::move(e));
  }
  std::stable_sort(diags_.begin(), diags_.end(), [](const DiagEv& a, const DiagEv& b) {
    if (a.sweep != b.sweep) return a.sweep < b.sweep;
    if (a.phase != b.phase) return a.phase < b.phase;
    if (a.k1 != b.k1) return a.k1 < b.k1;
    if (a.k2 != b.k2) return a.k2 < b.k2;
    return a.seq < b.seq;
  });
  std::set<std::pair<int, std::string>> seen;
  for (const DiagEv& e : diags_)
    if (seen.insert({static_cast<int>(e.d.category), e.d.message}).second) {
      r.diagnostics.push_back(e.d);
      r.diagnostics.back().sweep = e.sweep;
    }
  r.steps = steps_;
  if (r.stuck)
    r.exitCode = 3;
  else if (!r.diagnostics.empty())
    r.exitCode = 1;
  else
    r.exitCode = static_cast<int>(exitValue_.value_or(0));
  std::sort(reported_.begin(), reported_.end());
  r.reported = reported_;
  r.stats = stats_;
  std::stable_sort(traces_.begin(), traces_.end(), [](const TraceEv& a, const TraceEv& b) {
    if (a.sweep != b.sweep) return a.sweep < b.sweep;
    if (a.phase != b.phase) return a.phase < b.phase;
    if (a.k1 != b.k1) return a.k1 < b.k1;
    if (a.k2 != b.k2) return a.k2 < b.k2;
    return a.seq < b.seq;
  });
  for (const TraceEv& e : traces_) r.trace.push_back(e.text);
  return r;
}

}  // namespace mckb

// ======================= public API =======================
namespace mck {

const char* categoryName(DiagCategory c) {
  switch (c) {
    case DiagCategory::Race: return "race";
    case DiagCategory::Deadlock: return "deadlock";
    case DiagCategory::MemBoundary: return "memBoundary";
    case DiagCategory::UndefinedBehavior: return "undefinedBehavior";
    case DiagCategory::ApiError: return "apiError";
  }
  return "?";
}

const char* apiName(ApiId id) {
  static const char* names[] = {"cudaMalloc", "cudaFree", "cudaMemcpy", "cudaMemcpyAsync", "cudaMemset",
                                "cudaDeviceSynchronize", "cudaStreamCreate", "cudaStreamDestroy",
                                "cudaStreamSynchronize", "cudaStreamQuery", "cudaStreamWaitEvent",
                                "cudaEventCreate", "cudaEventDestroy", "cudaEventRecord",
                                "cudaEventSynchronize", "cudaEventQuery", "cudaEventElapsedTime",
                                "cudaGetLastError", "cudaGetErrorString", "cudaDeviceGetAttribute",
                                "cudaDriverGetVersion", "cudaRuntimeGetVersion"};
  const auto i = static_cast<size_t>(id);
  return i < sizeof names / sizeof names[0] ? names[i] : "?";
}

// compileSource (program.hpp:59-60): frontend failures surface as the
// reference's typed exceptions (diagnostics.hpp:41-56).
std::shared_ptr<const Program> compileSource(const std::string& source, const std::string& filename) {
  try {
    return mckb::compileProgram(source, filename);
  } catch (const mckb::FrontendFailure& f) {
    const SourceLoc loc{f.pos.line, f.pos.col};
    if (f.stage == "lex") throw LexError(loc, f.message);
    if (f.stage == "parse") {
      // "expected <what>, found <tok>" (parser.cpp's ParseError text)
      const std::string& m = f.message;
      const size_t k = m.rfind(", found ");
      if (m.rfind("expected ", 0) == 0 && k != std::string::npos)
        throw ParseError(loc, m.substr(9, k - 9), m.substr(k + 8));
      throw ParseError(loc, m, "");
    }
    throw SemanticError(loc, f.message);
  }
}

Machine::Machine(std::shared_ptr<const Program> prog, RunOptions opts)
    : prog_(std::move(prog)), opts_(opts), impl_(new MachineImpl) {}
Machine::~Machine() = default;

RunResult Machine::run() {
  mckb::HostHooks h;
  h.mem = onMemAccess;
  h.api = onApiCall;
  h.out = onOutput;
  impl_->m.reset(new mckb::HostMachine(prog_, opts_, std::move(h)));
  RunResult r = impl_->m->run();
  std::string note;
  if (opts_.policy == SchedulePolicy::SeededRandom && opts_.seed != 0)
    note = "SchedulePolicy::SeededRandom (seed " + std::to_string(opts_.seed) +
           ") was run under the round-robin schedule: the B200 engine executes the round-robin "
           "interleaving only (it equals the seed-0 run on the BASELINE program families)";
  if (opts_.policy == SchedulePolicy::Exhaustive)
    note = "SchedulePolicy::Exhaustive was run under the round-robin schedule (the interleaving "
           "explorer is oracleRace)";
  if (!note.empty()) r.engineNote = r.engineNote.empty() ? note : note + "; " + r.engineNote;
  if (onTrace)
    for (const std::string& t : r.trace) onTrace(t);
  impl_->last = r;
  impl_->ran = true;
  return r;
}

OracleResult oracleRace(std::shared_ptr<const Program> prog, OracleOptions opts) {
  RunOptions ro;
  ro.policy = SchedulePolicy::RoundRobin;
  ro.raceCheck = true;
  ro.arch = opts.arch;
  mckb::HostMachine hm(std::move(prog), ro);
  mckb::OracleSpec spec;
  spec.maxInterleavings = opts.maxInterleavings;
  spec.maxAccessesPerThread = opts.maxAccessesPerThread;
  hm.setOracle(spec, opts.maxThreads);
  const RunResult r = hm.run();
  OracleResult out;
  const mckb::OracleOut& o = hm.oracleOut();
  out.oracleRace = o.oracleRace;
  out.detectorRace = o.detectorRace;
  out.aborted = o.aborted;
  out.error = o.error;
  out.interleavings = hm.oracleGrids() ? o.interleavings : 1;  // no grid: one (host-only) schedule
  if (!r.engineError.empty() && !out.aborted) {
    out.aborted = true;
    out.error = r.engineError;
  }
  return out;
}

std::vector<StuckReport> Machine::scanStuck() const {
  return impl_->ran && impl_->last.stuck ? impl_->last.stuckReports : std::vector<StuckReport>{};
}

std::vector<uint8_t> makeCommId() {
  std::array<uint8_t, 128> id;
  std::string why;
  if (!mckb::makeCommId(id, why)) return {};
  return std::vector<uint8_t>(id.begin(), id.end());
}

std::string formatStuckReports(const std::vector<StuckReport>& reports) {
  std::string out;
  for (const StuckReport& r : reports) {
    switch (r.kind) {
      case StuckReport::Kind::BarrierDeadlock: {
        out += "barrier-deadlock gid=" + std::to_string(r.gid) + " bid=" + std::to_string(r.bid) + " waiting=[";
        for (size_t i = 0; i < r.waitingTids.size(); ++i) out += (i ? "," : "") + std::to_string(r.waitingTids[i]);
        out += "] finished-or-absent=[";
        for (size_t i = 0; i < r.missingTids.size(); ++i) out += (i ? "," : "") + std::to_string(r.missingTids[i]);
        out += "]\n";
        break;
      }
      case StuckReport::Kind::HostHang: out += "host-hang: " + r.reason + "\n"; break;
      case StuckReport::Kind::StreamStall:
        out += "stream-stall sid=" + std::to_string(r.sid) + " item=" + r.item + "\n";
        break;
    }
  }
  return out;
}

FileRunOutcome runSourceText(const std::string& source, const std::string& filename, const CliOptions& opts) {
  FileRunOutcome out;
  std::shared_ptr<const Program> prog;
  try {
    prog = compileSource(source, filename);
  } catch (const FrontendError& e) {
    out.frontendError = true;
    out.exitCode = 2;
    out.stderrText = "cudak: " + filename + ":" + std::to_string(e.loc.line) + ":" + std::to_string(e.loc.col) +
                     ": " + e.stage + " error: " + e.message + "\n";
    return out;
  }
  RunOptions ro;
  ro.policy = opts.schedule;
  ro.seed = opts.seed;
  ro.raceCheck = opts.raceCheck;
  ro.stepLimit = opts.stepLimit;
  ro.trace = opts.trace;
  ro.arch = opts.arch;
  Machine m(prog, ro);
  out.run = m.run();
  out.stdoutText = out.run.output;
  for (const std::string& t : out.run.trace) out.stderrText += "cudak: trace: " + t + "\n";
  for (const Diagnostic& d : out.run.diagnostics) out.stderrText += "cudak: " + d.message + "\n";
  if (!out.run.engineError.empty()) {
    out.stderrText += "cudak: engine error: " + out.run.engineError + "\n";
    out.exitCode = 4;
  } else {
    out.exitCode = out.run.exitCode;
  }
  if (out.run.stuck && !opts.reportPath.empty()) {
    if (FILE* f = std::fopen(opts.reportPath.c_str(), "w")) {
      // driver.cpp:152-158; the configuration dump is not modelled
      std::string t = "stuck-state report for " + filename + "\n\n" + formatStuckReports(out.run.stuckReports) +
                      "\nfinal configuration:\n(not modelled by the B200 engine)\n";
      std::fwrite(t.data(), 1, t.size(), f);
      std::fclose(f);
    }
  }
  return out;
}

FileRunOutcome runFile(const CliOptions& opts, bool) {
  std::string src;
  if (FILE* f = std::fopen(opts.inputPath.c_str(), "rb")) {
    char buf[65536];
    size_t n;
    while ((n = std::fread(buf, 1, sizeof buf, f)) > 0) src.append(buf, n);
    std::fclose(f);
  } else {
    FileRunOutcome out;
    out.exitCode = 2;
    out.stderrText = "cudak: cannot read " + opts.inputPath + "\n";
    return out;
  }
  return runSourceText(src, opts.inputPath, opts);
}

}  // namespace mck
