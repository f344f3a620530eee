// mckb -- command-line driver over the public C++ API (include/mck/checker.hpp),
// the drop-in for the reference CLI's checking path (tools/minicudak.cpp:14-96,
// driver.cpp:87-161): program output on stdout, one "cudak: <message>" line
// per diagnostic on stderr, the stuck-report file on deadlock, and the
// reference exit codes (0 clean, 1 diagnostics, 2 frontend error, 3 stuck).
//
//   mckb [--no-race-check] [--schedule roundrobin|random] [--seed N]
//        [--step-limit N] [--report FILE] [--trace] [--arch FILE] [--stats] file.cu
//   mckb --run-corpus DIR        (every DIR/*.cu against its .expect sidecar)
//
// On a stuck run the report file (default: <file>.cudak-report.txt, as the
// reference CLI) receives the stuck reports.
//
// Device grids run on the B200 engine; the schedule is round-robin (the
// engine's exact schedule; --schedule random is accepted and noted).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <string>

#include "mck/checker.hpp"

int main(int argc, char** argv) {
  mck::CliOptions o;
  bool stats = false;
  bool reportSet = false;
  std::string corpusDir;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) {
        std::fprintf(stderr, "mckb: %s needs a value\n", a.c_str());
        std::exit(2);
      }
      return argv[++i];
    };
    if (a == "--no-race-check") o.raceCheck = false;
    else if (a == "--schedule") {
      std::string v = next();
      o.schedule = v == "roundrobin" ? mck::SchedulePolicy::RoundRobin : mck::SchedulePolicy::SeededRandom;
    } else if (a == "--seed") o.seed = std::strtoull(next().c_str(), nullptr, 10);
    else if (a == "--step-limit") o.stepLimit = std::strtoull(next().c_str(), nullptr, 10);
    else if (a == "--report") {
      o.reportPath = next();
      reportSet = true;
    } else if (a == "--arch") o.archFile = next();
    else if (a == "--run-corpus") corpusDir = next();
    else if (a == "--trace") o.trace = true;
    else if (a == "--stats") stats = true;
    else if (a == "-h" || a == "--help") {
      std::printf("usage: mckb [--no-race-check] [--schedule roundrobin|random] [--seed N] "
                  "[--step-limit N] [--report FILE] [--trace] [--arch FILE] [--stats] file.cu\n"
                  "       mckb --run-corpus DIR\n");
      return 0;
    } else if (!a.empty() && a[0] == '-') {
      std::fprintf(stderr, "mckb: unknown option %s\n", a.c_str());
      return 2;
    } else {
      o.inputPath = a;
    }
  }
  if (!corpusDir.empty()) {
    const mck::CorpusOutcome c = mck::runCorpus(corpusDir);
    std::printf("%s%d passed, %d failed\n", c.table.c_str(), c.passed, c.failed);
    return c.failed == 0 ? 0 : 1;
  }
  if (o.inputPath.empty()) {
    std::fprintf(stderr, "mckb: no input file\n");
    return 2;
  }
  if (!reportSet) o.reportPath = o.inputPath + ".cudak-report.txt";
  if (!o.archFile.empty()) {
    try {
      o.arch = mck::loadArchFile(o.archFile);
    } catch (const std::exception& e) {
      std::fprintf(stderr, "cudak: %s\n", e.what());
      return 2;
    }
  }
  mck::FileRunOutcome out = mck::runFile(o);
  std::fwrite(out.stdoutText.data(), 1, out.stdoutText.size(), stdout);
  std::fflush(stdout);
  std::fwrite(out.stderrText.data(), 1, out.stderrText.size(), stderr);
  if (stats) {
    const mck::EngineStats& s = out.run.stats;
    std::fprintf(stderr,
                 "mckb: stats steps=%llu host=%llu device=%llu barrier=%llu dispatch=%llu grids=%llu "
                 "grid_ms=%.3f shared_events=%llu\n",
                 (unsigned long long)out.run.steps, (unsigned long long)s.hostSteps,
                 (unsigned long long)s.deviceSteps, (unsigned long long)s.barrierRules,
                 (unsigned long long)s.dispatches, (unsigned long long)s.grids, s.gridMs,
                 (unsigned long long)s.sharedEvents);
  }
  return out.exitCode;
}
