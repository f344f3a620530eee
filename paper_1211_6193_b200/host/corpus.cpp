// corpus.cpp -- the reference driver's file utilities on the report path
// (driver.hpp:37-57): architecture-parameter files and the corpus runner
// (.cu fixtures checked against .expect sidecars).  Host-only C++; every run
// goes through mck::runFile, i.e. the B200 engine.
#include <algorithm>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <regex>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "mck/checker.hpp"

namespace mck {

namespace {

std::string trimmed(const std::string& s) {
  const char* ws = " \t\r";
  const size_t a = s.find_first_not_of(ws);
  if (a == std::string::npos) return {};
  return s.substr(a, s.find_last_not_of(ws) - a + 1);
}

// A parsed .expect sidecar (format: driver.hpp:49-56).
struct Sidecar {
  int exitCode = 0;
  std::vector<std::string> args;
  std::vector<std::string> stderrPatterns;
  std::string stdoutText;
  std::string error;  // non-empty: the sidecar itself is malformed / missing
};

Sidecar readSidecar(const std::filesystem::path& p) {
  Sidecar sc;
  std::ifstream in(p, std::ios::binary);
  if (!in) {
    sc.error = "missing sidecar " + p.string();
    return sc;
  }
  bool collecting = false;
  for (std::string line; std::getline(in, line);) {
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (collecting) {
      if (line == "EOF")
        collecting = false;
      else
        sc.stdoutText += line + '\n';
      continue;
    }
    if (line.empty() || line.front() == '#') continue;
    auto starts = [&](const char* k) { return line.compare(0, std::char_traits<char>::length(k), k) == 0; };
    if (line == "stdout<<EOF") {
      collecting = true;
    } else if (starts("exit ")) {
      sc.exitCode = std::atoi(line.c_str() + 5);
    } else if (starts("args ")) {
      std::istringstream words(line.substr(5));
      for (std::string w; words >> w;) sc.args.push_back(w);
    } else if (starts("stderr-re ")) {
      sc.stderrPatterns.push_back(line.substr(10));
    } else {
      sc.error = "unrecognized sidecar line: " + line;
      return sc;
    }
  }
  if (collecting) sc.error = "unterminated stdout<<EOF block";
  return sc;
}

// The subset of command-line options a sidecar's `args` line may carry.
std::string applyArgs(CliOptions& o, const std::vector<std::string>& args) {
  for (size_t i = 0; i < args.size(); ++i) {
    const std::string& a = args[i];
    const bool hasValue = i + 1 < args.size();
    if (a == "--no-race-check") {
      o.raceCheck = false;
    } else if (a == "--trace") {
      o.trace = true;
    } else if (a == "--seed" || a == "--step-limit") {
      if (!hasValue) return a + " needs a value";
      (a == "--seed" ? o.seed : o.stepLimit) = std::strtoull(args[++i].c_str(), nullptr, 10);
    } else if (a == "--schedule") {
      if (!hasValue) return "--schedule needs a value";
      const std::string& v = args[++i];
      if (v == "random")
        o.schedule = SchedulePolicy::SeededRandom;
      else if (v == "roundrobin")
        o.schedule = SchedulePolicy::RoundRobin;
      else
        return "unknown schedule '" + v + "'";
    } else {
      return "unknown option '" + a + "' in sidecar args";
    }
  }
  return {};
}

std::vector<std::string> lines(const std::string& text) {
  std::vector<std::string> out;
  std::istringstream in(text);
  for (std::string l; std::getline(in, l);) out.push_back(l);
  return out;
}

}  // namespace

ArchParams loadArchFile(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open architecture file '" + path + "'");
  ArchParams arch;
  const std::pair<const char*, int64_t ArchParams::*> keys[] = {
      {"warpSize", &ArchParams::warpSize},
      {"computeCapabilityMajor", &ArchParams::computeCapabilityMajor},
      {"computeCapabilityMinor", &ArchParams::computeCapabilityMinor},
      {"maxThreadsPerBlock", &ArchParams::maxThreadsPerBlock},
      {"driverVersion", &ArchParams::driverVersion},
      {"runtimeVersion", &ArchParams::runtimeVersion},
  };
  int lineNo = 0;
  for (std::string line; std::getline(in, line);) {
    ++lineNo;
    const std::string where = path + ":" + std::to_string(lineNo) + ": ";
    line = trimmed(line.substr(0, line.find('#')));
    if (line.empty()) continue;
    const size_t eq = line.find('=');
    if (eq == std::string::npos) throw std::runtime_error(where + "expected 'key = integer'");
    const std::string key = trimmed(line.substr(0, eq)), val = trimmed(line.substr(eq + 1));
    int64_t v = 0;
    try {
      v = std::stoll(val);
    } catch (...) {
      throw std::runtime_error(where + "'" + val + "' is not an integer");
    }
    auto k = std::find_if(std::begin(keys), std::end(keys), [&](const auto& e) { return key == e.first; });
    if (k == std::end(keys)) throw std::runtime_error(where + "unknown architecture key '" + key + "'");
    arch.*(k->second) = v;
  }
  return arch;
}

CorpusOutcome runCorpus(const std::string& directory) {
  namespace fs = std::filesystem;
  CorpusOutcome out;
  std::vector<fs::path> fixtures;
  std::error_code ec;
  for (const auto& e : fs::directory_iterator(directory, ec))
    if (e.path().extension() == ".cu") fixtures.push_back(e.path());
  std::sort(fixtures.begin(), fixtures.end());
  for (const fs::path& f : fixtures) {
    const std::string name = f.filename().string();
    const std::string why = [&]() -> std::string {
      const Sidecar sc = readSidecar(fs::path(f).replace_extension(".expect"));
      if (!sc.error.empty()) return sc.error;
      CliOptions o;
      o.inputPath = f.string();
      if (std::string bad = applyArgs(o, sc.args); !bad.empty()) return bad;
      const FileRunOutcome r = runFile(o);
      if (r.exitCode != sc.exitCode)
        return "exit code " + std::to_string(r.exitCode) + ", expected " + std::to_string(sc.exitCode);
      if (r.stdoutText != sc.stdoutText) return "stdout mismatch";
      const std::vector<std::string> err = lines(r.stderrText);
      if (err.size() != sc.stderrPatterns.size())
        return "stderr has " + std::to_string(err.size()) + " line(s), expected " +
               std::to_string(sc.stderrPatterns.size());
      for (size_t i = 0; i < err.size(); ++i)
        if (!std::regex_match(err[i], std::regex(sc.stderrPatterns[i])))
          return "stderr line " + std::to_string(i + 1) + " does not match /" + sc.stderrPatterns[i] + "/";
      return {};
    }();
    if (why.empty()) {
      ++out.passed;
      out.table += "PASS " + name + "\n";
    } else {
      ++out.failed;
      out.table += "FAIL " + name + " (" + why + ")\n";
    }
  }
  return out;
}

}  // namespace mck
