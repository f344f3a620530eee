// capi.cpp -- C ABI over the mck:: C++ API (declared in include/mckg.h):
// run a CUDA-C program end to end and return the RunResult as JSON, the
// boundary the Python tests and bench.py call through ctypes.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime_api.h>

#include "mck/checker.hpp"
#include "mckg.h"
#include "program.hpp"

namespace mckg {
void set_error(const char* what, cudaError_t e);  // csrc/abi.cu: mckg_last_error()
}

namespace {

std::string js(const std::string& s) {
  std::string o = "\"";
  for (unsigned char c : s) {
    if (c == '"' || c == '\\') {
      o += '\\';
      o += static_cast<char>(c);
    } else if (c < 0x20) {
      char b[8];
      std::snprintf(b, sizeof b, "\\u%04x", c);
      o += b;
    } else {
      o += static_cast<char>(c);
    }
  }
  return o + "\"";
}

mck::RunOptions toOptions(const mck_run_opts* opts) {
  mck::RunOptions ro;
  if (opts) {
    ro.stepLimit = opts->step_limit ? opts->step_limit : ro.stepLimit;
    ro.raceCheck = opts->race_check != 0;
    ro.device = opts->device;
    ro.policy = opts->round_robin ? mck::SchedulePolicy::RoundRobin : mck::SchedulePolicy::SeededRandom;
    ro.seed = opts->seed;
    if (opts->max_threads_per_block > 0) ro.arch.maxThreadsPerBlock = opts->max_threads_per_block;
    for (int i = 0; i < opts->n_devices && i < 8; ++i) ro.devices.push_back(opts->devices[i]);
    ro.trace = opts->trace != 0;
    ro.globalRaceCheck = opts->global_race_check != 0;
    if (opts->world > 1) {
      ro.rank = opts->rank;
      ro.world = opts->world;
      ro.commId.assign(opts->comm_id, opts->comm_id + 128);
      ro.allgather = opts->allgather;
      ro.allgatherCtx = opts->allgather_ctx;
    }
  }
  return ro;
}

}  // namespace

extern "C" int mck_run_source(const char* src, const char* filename, const mck_run_opts* opts, char** json) {
  if (!src || !filename || !json) return MCKG_E_ARG;
  const mck::RunOptions ro = toOptions(opts);
  std::string o;
  try {
    auto prog = mck::compileSource(src, filename);
    mck::Machine m(prog, ro);
    mck::RunResult r = m.run();
    o = "{\"exit\":" + std::to_string(r.exitCode) + ",\"output\":" + js(r.output) +
        ",\"steps\":" + std::to_string(r.steps) + ",\"stuck\":" + (r.stuck ? "true" : "false") +
        ",\"main_return\":" + (r.mainReturn ? std::to_string(*r.mainReturn) : std::string("null")) +
        ",\"engine_error\":" + js(r.engineError) + ",\"engine_note\":" + js(r.engineNote) + ",\"diags\":[";
    for (size_t i = 0; i < r.diagnostics.size(); ++i) {
      const auto& d = r.diagnostics[i];
      o += std::string(i ? "," : "") + "{\"cat\":" + js(mck::categoryName(d.category)) + ",\"sev\":" +
           (d.severity == mck::Severity::Error ? "\"error\"" : "\"warning\"") + ",\"msg\":" + js(d.message) +
           ",\"line\":" + std::to_string(d.loc.line) +
           (getenv("MCK_DIAG_SWEEP") ? ",\"sweep\":" + std::to_string(d.sweep) : std::string()) + "}";
    }
    o += "],\"stuck_reports\":[";
    for (size_t i = 0; i < r.stuckReports.size(); ++i) {
      const auto& s = r.stuckReports[i];
      const char* kind = s.kind == mck::StuckReport::Kind::BarrierDeadlock ? "barrier"
                         : s.kind == mck::StuckReport::Kind::HostHang      ? "host"
                                                                          : "stream";
      o += std::string(i ? "," : "") + "{\"kind\":\"" + kind + "\",\"gid\":" + std::to_string(s.gid) +
           ",\"bid\":" + std::to_string(s.bid) + ",\"waiting\":[";
      for (size_t k = 0; k < s.waitingTids.size(); ++k) o += (k ? "," : "") + std::to_string(s.waitingTids[k]);
      o += "],\"missing\":[";
      for (size_t k = 0; k < s.missingTids.size(); ++k) o += (k ? "," : "") + std::to_string(s.missingTids[k]);
      o += "],\"reason\":" + js(s.reason) + "}";
    }
    o += "],\"report_text\":" + js(mck::formatStuckReports(r.stuckReports)) + ",\"reported\":[";
    for (size_t i = 0; i < r.reported.size(); ++i)
      o += std::string(i ? "," : "") + "[" + std::to_string(r.reported[i].object) + "," +
           std::to_string(r.reported[i].byte) + "," + std::to_string(r.reported[i].line) + "]";
    o += "],\"trace\":[";
    for (size_t i = 0; i < r.trace.size(); ++i) o += std::string(i ? "," : "") + js(r.trace[i]);
    const auto& st = r.stats;
    o += "],\"stats\":{\"host_steps\":" + std::to_string(st.hostSteps) + ",\"device_steps\":" +
         std::to_string(st.deviceSteps) + ",\"barrier_rules\":" + std::to_string(st.barrierRules) +
         ",\"dispatches\":" + std::to_string(st.dispatches) + ",\"shared_events\":" +
         std::to_string(st.sharedEvents) + ",\"grids\":" + std::to_string(st.grids) + ",\"sweeps\":" +
         std::to_string(st.sweeps) + ",\"grid_ms\":" + std::to_string(st.gridMs) + ",\"kernel_launches\":" +
         std::to_string(st.kernelLaunches) + ",\"block_sweeps\":" + std::to_string(st.blockSweeps) +
         ",\"solo_sweeps\":" + std::to_string(st.soloSweeps) + ",\"block_cycles\":" +
         std::to_string(st.blockCycles) + ",\"solo_cycles\":" + std::to_string(st.soloCycles) + "}}";
  } catch (const mck::FrontendError& e) {
    o = "{\"frontend_error\":" + js(e.stage + ": " + e.message) + ",\"line\":" + std::to_string(e.loc.line) +
        ",\"exit\":2}";
  } catch (const std::exception& e) {
    o = "{\"internal_error\":" + js(e.what()) + ",\"exit\":5}";
  }
  *json = strdup(o.c_str());
  return MCKG_OK;
}

extern "C" int mck_disassemble(const char* src, const char* filename, char** text) {
  if (!src || !filename || !text) return MCKG_E_ARG;
  try {
    auto p = mckb::compileProgram(src, filename);
    *text = strdup(p->disassemble().c_str());
  } catch (const mckb::FrontendFailure& f) {
    *text = strdup((f.stage + ": " + f.message).c_str());
    return MCKG_E_ARG;
  }
  return MCKG_OK;
}

extern "C" void mck_free(char* p) { std::free(p); }

extern "C" int mckg_comm_id(uint8_t out[128]) {
  std::vector<uint8_t> id = mck::makeCommId();
  if (id.size() != 128) return MCKG_E_CUDA;
  std::memcpy(out, id.data(), 128);
  return MCKG_OK;
}

// ---- result records ----
struct mck_result {
  mck::RunResult run;
  std::string frontendStage, frontendMessage;
  int frontendLine = 0;
  std::string reportText;
  std::vector<std::vector<int32_t>> waiting, missing;
};

extern "C" int mck_run(const char* src, const char* filename, const mck_run_opts* opts, mck_result** out) {
  if (!src || !filename || !out) return MCKG_E_ARG;
  *out = nullptr;
  auto r = std::make_unique<mck_result>();
  try {
    auto prog = mck::compileSource(src, filename);
    mck::Machine m(prog, toOptions(opts));
    r->run = m.run();
  } catch (const mck::FrontendError& e) {
    r->frontendStage = e.stage;
    r->frontendMessage = e.message;
    r->frontendLine = e.loc.line;
    r->run.exitCode = 2;
  } catch (const std::exception& e) {
    mckg::set_error((std::string("mck_run: ") + e.what()).c_str(), cudaSuccess);
    return MCKG_E_CUDA;
  }
  r->reportText = mck::formatStuckReports(r->run.stuckReports);
  for (const auto& sr : r->run.stuckReports) {
    r->waiting.emplace_back(sr.waitingTids.begin(), sr.waitingTids.end());
    r->missing.emplace_back(sr.missingTids.begin(), sr.missingTids.end());
  }
  *out = r.release();
  return MCKG_OK;
}

extern "C" int mck_result_summary(const mck_result* r, mck_summary* out) {
  if (!r || !out) return MCKG_E_ARG;
  const mck::RunResult& x = r->run;
  *out = mck_summary{};
  out->exit_code = x.exitCode;
  out->stuck = x.stuck ? 1 : 0;
  out->has_main_return = x.mainReturn ? 1 : 0;
  out->main_return = x.mainReturn ? *x.mainReturn : 0;
  out->frontend_line = r->frontendLine;
  out->steps = x.steps;
  out->n_diags = x.diagnostics.size();
  out->n_stuck = x.stuckReports.size();
  out->n_reported = x.reported.size();
  out->n_trace = x.trace.size();
  out->output_bytes = x.output.size();
  out->output = x.output.c_str();
  out->engine_error = x.engineError.c_str();
  out->engine_note = x.engineNote.c_str();
  out->frontend_stage = r->frontendStage.c_str();
  out->frontend_message = r->frontendMessage.c_str();
  out->report_text = r->reportText.c_str();
  return MCKG_OK;
}

extern "C" int mck_result_diag(const mck_result* r, uint64_t i, mck_diag_rec* out) {
  if (!r || !out || i >= r->run.diagnostics.size()) return MCKG_E_ARG;
  const mck::Diagnostic& d = r->run.diagnostics[i];
  out->category = static_cast<int32_t>(d.category);
  out->severity = d.severity == mck::Severity::Error ? 0 : 1;
  out->line = d.loc.line;
  out->pad = 0;
  out->sweep = d.sweep;
  out->message = d.message.c_str();
  return MCKG_OK;
}

extern "C" int mck_result_stuck(const mck_result* r, uint64_t i, mck_stuck_rec* out) {
  if (!r || !out || i >= r->run.stuckReports.size()) return MCKG_E_ARG;
  const mck::StuckReport& s = r->run.stuckReports[i];
  out->kind = static_cast<int32_t>(s.kind);
  out->gid = s.gid;
  out->bid = s.bid;
  out->sid = s.sid;
  out->n_waiting = r->waiting[i].size();
  out->n_missing = r->missing[i].size();
  out->waiting = r->waiting[i].data();
  out->missing = r->missing[i].data();
  out->reason = s.reason.c_str();
  out->item = s.item.c_str();
  return MCKG_OK;
}

extern "C" int mck_result_stats(const mck_result* r, mck_run_stats* out) {
  if (!r || !out) return MCKG_E_ARG;
  const mck::EngineStats& st = r->run.stats;
  *out = mck_run_stats{};
  out->host_steps = st.hostSteps;
  out->device_steps = st.deviceSteps;
  out->barrier_rules = st.barrierRules;
  out->dispatches = st.dispatches;
  out->shared_events = st.sharedEvents;
  out->grids = st.grids;
  out->sweeps = st.sweeps;
  out->grid_ms = st.gridMs;
  out->kernel_launches = st.kernelLaunches;
  out->block_sweeps = st.blockSweeps;
  out->solo_sweeps = st.soloSweeps;
  out->block_cycles = st.blockCycles;
  out->solo_cycles = st.soloCycles;
  return MCKG_OK;
}

extern "C" int mck_result_reported(const mck_result* r, uint64_t first, uint64_t count, mckg_race_triple* out) {
  if (!r || (!out && count)) return MCKG_E_ARG;
  const auto& rep = r->run.reported;
  if (first > rep.size() || count > rep.size() - first) return MCKG_E_RANGE;
  for (uint64_t k = 0; k < count; ++k) {
    const mck::RaceTriple& t = rep[first + k];
    out[k] = mckg_race_triple{t.object, static_cast<uint32_t>(t.byte), t.line};
  }
  return MCKG_OK;
}

extern "C" const char* mck_result_trace(const mck_result* r, uint64_t i) {
  if (!r || i >= r->run.trace.size()) return nullptr;
  return r->run.trace[i].c_str();
}

extern "C" void mck_result_free(mck_result* r) { delete r; }

extern "C" int mck_oracle(const char* src, const char* filename, uint64_t max_interleavings, int32_t max_threads,
                          int32_t max_accesses_per_thread, mck_oracle_result* out) {
  if (!src || !filename || !out) return MCKG_E_ARG;
  *out = mck_oracle_result{};
  std::string err;
  try {
    auto prog = mck::compileSource(src, filename);
    mck::OracleOptions o;
    o.maxInterleavings = max_interleavings;
    o.maxThreads = max_threads;
    o.maxAccessesPerThread = max_accesses_per_thread;
    const mck::OracleResult r = mck::oracleRace(prog, o);
    out->oracle_race = r.oracleRace;
    out->detector_race = r.detectorRace;
    out->aborted = r.aborted;
    out->interleavings = r.interleavings;
    err = r.error;
  } catch (const mck::FrontendError& e) {
    out->frontend_error = 1;
    err = e.stage + ": " + e.message;
  }
  std::snprintf(out->error, sizeof out->error, "%s", err.c_str());
  return MCKG_OK;
}
