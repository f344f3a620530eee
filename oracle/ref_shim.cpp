// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY (see oracle/oracle.h).
//
// extern "C" shim over the UNMODIFIED reference library, compiled by
// oracle/Makefile from /root/reference/proj/src/*.cpp into
// oracle/_ref/libmckref.so.  It exposes
//   * mckref_replay_shared: the reference's own Machine::recordAccess /
//     Machine::clearEpoch (racecheck.cpp:9-73) driven over an mckg_access
//     trace (SURVEY Appendix D probe6), block-partitioned over pthreads;
//   * mckref_run: Machine::run (machine.cpp:1180-1227) on a source program,
//     returning RunResult, RaceState::reported and the shared-access trace the
//     detector saw (filtered exactly as memory.cpp:110-245 calls recordAccess,
//     timestamped with the round-robin sweep, epoch = per-thread releases),
//     as JSON.
// Nothing in the product links this library.
#include <pthread.h>

#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "minicudak/machine.hpp"
#include "minicudak/oracle.hpp"
#include "minicudak/program.hpp"

extern "C" {
#include "mckg.h"
}

using namespace mck;

namespace {

struct Job {
    const mckg_trace* t;
    uint32_t b0, b1;
    std::vector<mckg_race_triple> out;
    std::vector<uint64_t> lineFirst;
    int err = 0;
};

void* replayJob(void* arg) {
    Job* j = static_cast<Job*>(arg);
    const mckg_trace* t = j->t;
    j->lineFirst.assign(MCKG_MAX_LINES, MCKG_TS_NONE);
    auto prog = compileSource("int main(void) { return 0; }\n", "trace.cu");
    Machine m(prog, RunOptions{});
    GridId gid = t->gid ? t->gid : 1;
    for (uint32_t b = j->b0; b < j->b1; ++b) {
        int bid = static_cast<int>(t->bid_base + b);
        Configuration& cfg = m.config();
        cfg.memory.next = t->obj_base + b;
        Location l = m.allocObject(MemSpace::deviceShared(gid, bid), t->shmem_bytes, "shared");
        const MemObject& obj = cfg.memory.objects.at(l.object);
        bool have = false;
        uint32_t epoch = 0;
        for (uint64_t i = t->block_start[b]; i < t->block_start[b + 1]; ++i) {
            const mckg_access& a = t->events[i];
            uint32_t ep = MCKG_ACC_EPOCH(a);
            if (!have || ep != epoch) {
                if (have) m.clearEpoch(gid, bid);
                epoch = ep;
                have = true;
            }
            size_t before = cfg.race.reported.size();
            ThreadKey who{gid, bid, static_cast<int>(MCKG_ACC_TID(a))};
            m.recordAccess(obj, MCKG_ACC_OFF(a), MCKG_ACC_LEN(a), who,
                           MCKG_ACC_WRITE(a) ? AccessKind::Write : AccessKind::Read,
                           SourceLoc{a.line, 1});
            if (cfg.race.reported.size() != before && a.line >= 0 &&
                static_cast<uint32_t>(a.line) < MCKG_MAX_LINES) {
                uint64_t ts = mckg_ts_key(a.sweep, static_cast<uint32_t>(bid), MCKG_ACC_TID(a));
                if (ts < j->lineFirst[a.line]) j->lineFirst[a.line] = ts;
            }
        }
        m.clearEpoch(gid, bid);
        for (const auto& [o, byte, line] : cfg.race.reported)
            j->out.push_back(mckg_race_triple{o, static_cast<uint32_t>(byte), line});
        cfg.race.reported.clear();
        cfg.memory.objects.erase(l.object);
    }
    return nullptr;
}

std::string jsonStr(const std::string& s) {
    std::string o = "\"";
    for (unsigned char c : s) {
        if (c == '"' || c == '\\') {
            o += '\\';
            o += static_cast<char>(c);
        } else if (c < 0x20) {
            char buf[8];
            std::snprintf(buf, sizeof buf, "\\u%04x", c);
            o += buf;
        } else {
            o += static_cast<char>(c);
        }
    }
    return o + "\"";
}

struct CapEvent {
    uint32_t gid, bid, tid, obj, off, len, write, epoch, sweep;
    int line;
    uint64_t step;
};

}  // namespace

extern "C" {

int mckref_replay_shared(const mckg_trace* t, mckg_race_triple* triples, uint64_t capacity,
                         uint64_t* n_triples, uint64_t* line_first, int nthreads) {
    if (!t || !n_triples || !line_first) return MCKG_E_ARG;
    if (nthreads < 1) nthreads = 1;
    if (static_cast<uint32_t>(nthreads) > t->n_blocks) nthreads = t->n_blocks ? t->n_blocks : 1;
    std::vector<Job> jobs(nthreads);
    std::vector<pthread_t> th(nthreads);
    for (int k = 0; k < nthreads; ++k) {
        jobs[k].t = t;
        jobs[k].b0 = static_cast<uint32_t>(uint64_t(t->n_blocks) * k / nthreads);
        jobs[k].b1 = static_cast<uint32_t>(uint64_t(t->n_blocks) * (k + 1) / nthreads);
    }
    if (nthreads == 1) {
        replayJob(&jobs[0]);
    } else {
        for (int k = 0; k < nthreads; ++k) pthread_create(&th[k], nullptr, replayJob, &jobs[k]);
        for (int k = 0; k < nthreads; ++k) pthread_join(th[k], nullptr);
    }
    uint64_t n = 0;
    for (auto& j : jobs) {
        for (auto& tr : j.out) {
            if (n < capacity) triples[n] = tr;
            ++n;
        }
        for (uint32_t l = 0; l < MCKG_MAX_LINES; ++l)
            if (j.lineFirst[l] < line_first[l]) line_first[l] = j.lineFirst[l];
    }
    *n_triples = n;
    return n > capacity ? MCKG_E_OVERFLOW : MCKG_OK;
}

// policy: 0 = seeded random, 1 = round robin.  Writes NUL-terminated JSON into
// a malloc'ed buffer returned through *json (free with mckref_free).
int mckref_run(const char* src, const char* filename, int policy, uint64_t seed,
               uint64_t step_limit, int race_check, int capture, char** json) {
    std::ostringstream o;
    std::shared_ptr<const Program> prog;
    try {
        prog = compileSource(src, filename);
    } catch (const FrontendError& e) {
        o << "{\"frontend_error\":" << jsonStr(e.stage + ": " + e.message)
          << ",\"line\":" << e.loc.line << ",\"exit\":2}";
        *json = strdup(o.str().c_str());
        return 0;
    }
    RunOptions ro;
    ro.policy = policy == 1 ? SchedulePolicy::RoundRobin : SchedulePolicy::SeededRandom;
    ro.seed = seed;
    ro.stepLimit = step_limit;
    ro.raceCheck = race_check != 0;
    ro.trace = (capture & 2) != 0;  // bit 1: the --trace lines
    Machine m(prog, ro);
    std::vector<std::string> traceLines;
    m.onTrace = [&](const std::string& line) { traceLines.push_back(line); };

    std::vector<CapEvent> ev;
    std::map<ThreadKey, uint32_t> epochOf;
    uint32_t sweep = 0;
    bool havePrev = false;
    Transition prev{};
    size_t stepMark = 0;
    uint64_t devSteps = 0, barrierRules = 0, hostSteps = 0, dispatches = 0;
    m.onMemAccess = [&](const MemAccessInfo& a) {
        if (!(capture & 1) || !a.allowed || a.space.kind != SpaceKind::DeviceShared) return;
        const Configuration& cfg = m.config();
        if (!cfg.race.enabled) return;
        auto it = cfg.memory.objects.find(a.object);
        if (it == cfg.memory.objects.end() || !it->second.live) return;
        if (a.offset < 0 || a.offset + a.len > it->second.size) return;
        CapEvent e{};
        e.gid = a.accessor.gid;
        e.bid = static_cast<uint32_t>(a.accessor.bid);
        e.tid = static_cast<uint32_t>(a.accessor.tid);
        e.obj = a.object;
        e.off = static_cast<uint32_t>(a.offset);
        e.len = static_cast<uint32_t>(a.len);
        e.write = a.kind == AccessKind::Write;
        e.epoch = epochOf[a.accessor];
        e.sweep = sweep;  // fixed up in onStep if this transition wraps
        e.line = a.loc.line;
        e.step = cfg.steps;  // already incremented for this transition
        ev.push_back(e);
    };
    m.onStep = [&](Machine&, const Transition& t) {
        if (havePrev && !(prev < t)) {
            ++sweep;
            for (size_t i = stepMark; i < ev.size(); ++i) ev[i].sweep = sweep;
        }
        havePrev = true;
        prev = t;
        stepMark = ev.size();
        switch (t.kind) {
            case TransitionKind::HostStep: ++hostSteps; break;
            case TransitionKind::DeviceStep: ++devSteps; break;
            case TransitionKind::StreamDispatch: ++dispatches; break;
            case TransitionKind::BarrierRule:
                ++barrierRules;
                if (t.rule == BarrierRuleKind::DownSweep || t.rule == BarrierRuleKind::FinalRelease)
                    ++epochOf[t.thread];
                break;
        }
    };
    RunResult r = m.run();

    o << "{\"exit\":" << r.exitCode << ",\"output\":" << jsonStr(r.output)
      << ",\"steps\":" << r.steps << ",\"device_steps\":" << devSteps
      << ",\"barrier_rules\":" << barrierRules << ",\"host_steps\":" << hostSteps
      << ",\"dispatches\":" << dispatches << ",\"sweeps\":" << (havePrev ? sweep + 1 : 0)
      << ",\"stuck\":" << (r.stuck ? "true" : "false") << ",\"main_return\":"
      << (r.mainReturn ? std::to_string(*r.mainReturn) : std::string("null"));
    o << ",\"diags\":[";
    for (size_t i = 0; i < r.diagnostics.size(); ++i) {
        const Diagnostic& d = r.diagnostics[i];
        o << (i ? "," : "") << "{\"cat\":" << jsonStr(categoryName(d.category))
          << ",\"sev\":" << (d.severity == Severity::Error ? "\"error\"" : "\"warning\"")
          << ",\"msg\":" << jsonStr(d.message) << ",\"line\":" << d.loc.line << "}";
    }
    o << "],\"stuck_reports\":[";
    for (size_t i = 0; i < r.stuckReports.size(); ++i) {
        const StuckReport& s = r.stuckReports[i];
        const char* kind = s.kind == StuckReport::Kind::BarrierDeadlock ? "barrier"
                           : s.kind == StuckReport::Kind::HostHang      ? "host"
                                                                        : "stream";
        o << (i ? "," : "") << "{\"kind\":\"" << kind << "\",\"gid\":" << s.gid
          << ",\"bid\":" << s.bid << ",\"waiting\":[";
        for (size_t k = 0; k < s.waitingTids.size(); ++k) o << (k ? "," : "") << s.waitingTids[k];
        o << "],\"missing\":[";
        for (size_t k = 0; k < s.missingTids.size(); ++k) o << (k ? "," : "") << s.missingTids[k];
        o << "],\"reason\":" << jsonStr(s.reason) << "}";
    }
    o << "],\"report_text\":" << jsonStr(formatStuckReports(r.stuckReports));
    o << ",\"reported\":[";
    bool first = true;
    for (const auto& [obj, byte, line] : m.config().race.reported) {
        o << (first ? "" : ",") << "[" << obj << "," << byte << "," << line << "]";
        first = false;
    }
    o << "],\"arrivals\":{";
    // per grid, per block: __syncthreads arrivals of every thread at the end
    // of the run (releases + 1 if still waiting), the input of the K4 check
    {
        bool firstG = true;
        for (const auto& [gid, g] : m.config().grids) {
            if (g.gridDim * g.blockDim > (1 << 16)) continue;
            o << (firstG ? "" : ",") << "\"" << gid << "\":[";
            firstG = false;
            for (int64_t b = 0; b < g.gridDim; ++b) {
                o << (b ? "," : "") << "[";
                for (int64_t t = 0; t < g.blockDim; ++t) {
                    ThreadKey k{gid, static_cast<int>(b), static_cast<int>(t)};
                    uint32_t c = 0;
                    auto e = epochOf.find(k);
                    if (e != epochOf.end()) c = e->second;
                    auto d = m.config().device.find(k);
                    if (d != m.config().device.end() && d->second.barrier.waiting) ++c;
                    o << (t ? "," : "") << c;
                }
                o << "]";
            }
            o << "]";
        }
    }
    o << "},\"trace\":[";
    for (size_t i = 0; i < traceLines.size(); ++i) o << (i ? "," : "") << jsonStr(traceLines[i]);
    o << "],\"events\":[";
    for (size_t i = 0; i < ev.size(); ++i) {
        const CapEvent& e = ev[i];
        o << (i ? "," : "") << "[" << e.gid << "," << e.bid << "," << e.tid << "," << e.obj << ","
          << e.off << "," << e.len << "," << e.write << "," << e.epoch << "," << e.line << ","
          << e.sweep << "," << e.step << "]";
    }
    o << "]}";
    *json = strdup(o.str().c_str());
    return 0;
}

// oracleRace (oracle.cpp:140-152): the reference's exhaustive interleaving
// explorer on a source program; JSON {oracle_race, detector_race,
// interleavings, aborted, error} or {frontend_error}.
int mckref_oracle(const char* src, const char* filename, uint64_t max_interleavings, int max_threads,
                  int max_accesses, char** json) {
    std::ostringstream o;
    try {
        auto prog = compileSource(src, filename);
        OracleOptions opts;
        opts.maxInterleavings = max_interleavings;
        opts.maxThreads = max_threads;
        opts.maxAccessesPerThread = max_accesses;
        OracleResult r = oracleRace(prog, opts);
        o << "{\"oracle_race\":" << (r.oracleRace ? "true" : "false")
          << ",\"detector_race\":" << (r.detectorRace ? "true" : "false")
          << ",\"interleavings\":" << r.interleavings << ",\"aborted\":" << (r.aborted ? "true" : "false")
          << ",\"error\":" << jsonStr(r.error) << "}";
    } catch (const FrontendError& e) {
        o << "{\"frontend_error\":" << jsonStr(e.stage + ": " + e.message) << "}";
    } catch (const std::exception& e) {
        o << "{\"internal_error\":" << jsonStr(e.what()) << "}";
    }
    *json = strdup(o.str().c_str());
    return 0;
}

void mckref_free(char* p) { free(p); }

}  // extern "C"
