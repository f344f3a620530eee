// A reference-style client of the B200 checker, written against
// include/mck/checker.hpp exactly as a user of the reference's
// proj/include/minicudak headers would write it: a subset of the reference's
// own unit tests (tests/unit/test_machine.cpp, test_device.cpp,
// test_frontend.cpp) plus the hooks, scanStuck and the batched
// recordAccess/clearEpoch front-end.  Built and run by tests/test_cpp_client.py;
// the cases that launch grids need a CUDA device and are skipped without one
// (argv[1] == "--no-gpu").
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "mck/checker.hpp"

using namespace mck;

namespace {

int g_failed = 0, g_checks = 0;
bool g_gpu = true;
const char* g_case = "";

#define CHECK(cond)                                                                       \
  do {                                                                                    \
    ++g_checks;                                                                           \
    if (!(cond)) {                                                                        \
      ++g_failed;                                                                         \
      std::fprintf(stderr, "FAIL [%s] %s:%d: %s\n", g_case, __FILE__, __LINE__, #cond);  \
    }                                                                                     \
  } while (0)

template <typename E, typename F>
bool throwsAs(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

std::shared_ptr<const Program> compile(const std::string& src, const std::string& name = "test.cu") {
  return compileSource(src, name);
}

RunResult runSource(const std::string& src, RunOptions opts = {}, const std::string& name = "test.cu") {
  opts.policy = SchedulePolicy::RoundRobin;
  Machine m(compile(src, name), opts);
  return m.run();
}

bool hasCategory(const RunResult& r, DiagCategory cat) {
  for (const auto& d : r.diagnostics)
    if (d.category == cat) return true;
  return false;
}

struct Case {
  const char* name;
  bool gpu;
  std::function<void()> body;
};

// The reference corpus file (tests/golden/sum.cu = proj/tests/corpus/sum.cu),
// read from $MCK_CORPUS_DIR as the reference tests' corpusPath() does.
std::string slurp(const std::string& path) {
  std::string s;
  if (FILE* f = std::fopen(path.c_str(), "rb")) {
    char buf[4096];
    size_t n;
    while ((n = std::fread(buf, 1, sizeof buf, f)) > 0) s.append(buf, n);
    std::fclose(f);
  }
  return s;
}

std::string corpusPath(const std::string& name) {
  const char* d = std::getenv("MCK_CORPUS_DIR");
  return std::string(d ? d : ".") + "/" + name;
}

// line k (1-based) of src replaced by `text`
std::string withLine(const std::string& src, int k, const std::string& text) {
  std::string out;
  size_t pos = 0;
  for (int line = 1; pos <= src.size(); ++line) {
    size_t e = src.find('\n', pos);
    if (e == std::string::npos) e = src.size();
    out += (line == k ? text : src.substr(pos, e - pos));
    if (e < src.size()) out += '\n';
    pos = e + 1;
  }
  return out;
}

std::vector<Case> cases() {
  std::vector<Case> c;
  // ---- test_machine.cpp ----
  c.push_back({"main's return value becomes the exit code", false, [] {
                 CHECK(runSource("int main(void){return 7;}").exitCode == 7);
                 CHECK(runSource("int main(void){return 0;}").exitCode == 0);
                 CHECK(runSource("int main(void){}").exitCode == 0);
                 CHECK(runSource("int main(void){return 7;}").output.empty());
               }});
  c.push_back({"identical options and seed give identical results", false, [] {
                 const char* src = "int main(void){ int i, s = 0; for (i = 0; i != 40; ++i) s += i * i;\n"
                                   "  printf(\"%d\\n\", s); return 0; }\n";
                 for (uint64_t seed : {0ull, 1ull, 42ull}) {
                   RunOptions o;
                   o.seed = seed;
                   auto a = runSource(src, o);
                   auto b = runSource(src, o);
                   CHECK(a.output == b.output);
                   CHECK(a.exitCode == b.exitCode);
                   CHECK(a.steps == b.steps);
                   CHECK(a.diagnostics.size() == b.diagnostics.size());
                 }
               }});
  c.push_back({"the step limit aborts runaway programs with a diagnostic", false, [] {
                 RunOptions o;
                 o.stepLimit = 500;
                 auto r = runSource("int main(void){ while (1) {} return 0; }", o);
                 CHECK(r.exitCode == 1);
                 CHECK(r.steps == 500);
                 CHECK(r.diagnostics.size() == 1);
                 CHECK(!r.diagnostics.empty() &&
                       r.diagnostics[0].message.find("step limit exceeded") != std::string::npos);
               }});
  c.push_back({"a stuck configuration has no transitions and triggers the scanner", true, [] {
                 Machine m(compile("__global__ void k(void) { if (threadIdx.x == 0) { __syncthreads(); } }\n"
                                   "int main(void) { k<<<1, 2>>>(); cudaDeviceSynchronize(); return 0; }\n"),
                           RunOptions{});
                 CHECK(m.scanStuck().empty());  // nothing ran yet
                 auto r = m.run();
                 CHECK(r.stuck);
                 CHECK(r.exitCode == 3);
                 CHECK(!r.stuckReports.empty() && r.stuckReports[0].kind == StuckReport::Kind::BarrierDeadlock);
                 auto s = m.scanStuck();
                 CHECK(s.size() == r.stuckReports.size());
                 CHECK(!s.empty() && s[0].waitingTids == std::vector<int>{0} && s[0].missingTids == std::vector<int>{1});
               }});
  // ---- test_device.cpp ----
  c.push_back({"syncthreads_count broadcasts the number of true predicates", true, [] {
                 auto r = runSource(
                     "__global__ void k(int* g) { g[threadIdx.x] = __syncthreads_count(threadIdx.x == 0); }\n"
                     "int main(void) { int i, *g, h[2]; cudaMalloc(&g, 8);\n"
                     "  k<<<1, 2>>>(g);\n"
                     "  cudaMemcpy(h, g, 8, cudaMemcpyDeviceToHost);\n"
                     "  printf(\"%d %d\\n\", h[0], h[1]);\n"
                     "  cudaFree(g); return 0; }\n");
                 CHECK(r.exitCode == 0);
                 CHECK(r.output == "1 1\n");
               }});
  c.push_back({"a barrier missed by one thread leaves the protocol unmatched", true, [] {
                 auto r = runSource(
                     "__global__ void k(int* g) {\n  if (threadIdx.x != 3) { __syncthreads(); }\n"
                     "  g[threadIdx.x] = 1;\n}\n"
                     "int main(void) { int* g; cudaMalloc(&g, 9 * sizeof(int)); k<<<1, 9>>>(g);\n"
                     "  cudaDeviceSynchronize(); return 0; }\n");
                 CHECK(r.stuck);
                 CHECK(r.exitCode == 3);
                 bool saw = false;
                 for (const auto& d : r.diagnostics)
                   if (d.message == "Detected a deadlock caused by misplaced __syncthreads().") saw = true;
                 CHECK(saw);
               }});
  c.push_back({"a degenerate launch of one thread and zero shared bytes works", true, [] {
                 auto r = runSource(
                     "__global__ void k(int* g) { extern __shared__ int s[]; g[0] = 5; }\n"
                     "int main(void) { int *g, h; cudaMalloc(&g, 4); k<<<1, 1>>>(g);\n"
                     "  cudaMemcpy(&h, g, 4, cudaMemcpyDeviceToHost); printf(\"%d\\n\", h);\n"
                     "  return 0; }\n");
                 CHECK(r.exitCode == 0);
                 CHECK(r.output == "5\n");
               }});
  c.push_back({"any access to a zero-byte shared array is out of bounds", true, [] {
                 auto r = runSource(
                     "__global__ void k(void) { extern __shared__ int s[]; s[0] = 1; }\n"
                     "int main(void) { k<<<1, 1>>>(); cudaDeviceSynchronize(); return 0; }\n");
                 CHECK(r.exitCode == 1);
                 CHECK(!r.diagnostics.empty() && r.diagnostics[0].message.find("out-of-bounds") != std::string::npos);
               }});
  c.push_back({"launch configurations are validated", false, [] {
                 auto r = runSource(
                     "__global__ void k(void) {}\n"
                     "int main(void) { k<<<0, 1>>>(); cudaDeviceSynchronize(); return 0; }\n");
                 CHECK(r.exitCode == 1);
                 CHECK(hasCategory(r, DiagCategory::ApiError));
               }});
  c.push_back({"the figure program computes its sum and the mutants are diagnosed", true, [] {
                 const std::string fig1 = slurp(corpusPath("sum.cu"));
                 CHECK(!fig1.empty());
                 auto r = runSource(fig1, {}, "sum.cu");
                 CHECK(r.exitCode == 0);
                 CHECK(r.output.find("OUTPUT: 767\n") != std::string::npos);
                 CHECK(r.steps == 3114);  // the reference's count
                 auto rr = runSource(withLine(fig1, 14, ""), {}, "sum.cu");  // the race mutant
                 CHECK(rr.exitCode == 1);
                 CHECK(rr.steps == 2994);
                 CHECK(!rr.diagnostics.empty() &&
                       rr.diagnostics[0].message == "Possible race on shared device memory detected at sum.cu:17.");
                 auto rd = runSource(withLine(fig1, 12, "    shared[tid] += shared[bdim/2 + tid]; __syncthreads();"),
                                     {}, "sum.cu");  // the deadlock mutant
                 CHECK(rd.exitCode == 3);
                 CHECK(rd.steps == 2408);
                 CHECK(rd.stuckReports.size() == 3);
                 CHECK(formatStuckReports(rd.stuckReports) ==
                       "barrier-deadlock gid=1 bid=0 waiting=[0,1,2,3] finished-or-absent=[4,5,6,7,8]\n"
                       "barrier-deadlock gid=1 bid=1 waiting=[0,1,2,3] finished-or-absent=[4,5,6,7,8]\n"
                       "host-hang: host thread is blocked waiting for stream 0 to drain\n");
               }});
  // ---- test_frontend.cpp ----
  c.push_back({"frontend failures are the reference's typed exceptions", false, [] {
                 try {
                   compile("int main(void) { return 0 }", "x.cu");
                   CHECK(false);
                 } catch (const ParseError& e) {
                   CHECK(e.expected == "';'");
                   CHECK(e.loc.line == 1);
                   CHECK(e.stage == "parse");
                 }
                 CHECK(throwsAs<ParseError>([] { compile("int f(int a[2][2]) { return 0; }", "x.cu"); }));
                 CHECK(throwsAs<LexError>([] { compile("#define F(x) x\n", "x.cu"); }));
                 CHECK(throwsAs<LexError>([] { compile("int $;", "x.cu"); }));
                 CHECK(throwsAs<LexError>([] { compile("/* no end", "x.cu"); }));
                 CHECK(throwsAs<SemanticError>([] { compile("int main(void){ __syncthreads(); return 0; }"); }));
                 CHECK(throwsAs<SemanticError>([] {
                   compile("__global__ int f(void) { return 1; }\nint main(void){return 0;}");
                 }));
                 CHECK(throwsAs<SemanticError>([] { compile("int main(void){ return nope; }"); }));
                 CHECK(throwsAs<SemanticError>([] {
                   compile("__global__ void k(void){}\nint main(void){ k(); return 0; }");
                 }));
                 CHECK(throwsAs<FrontendError>([] { compile("int main(void){ return nope; }"); }));
               }});
  // ---- hooks (machine.hpp:384-388) ----
  c.push_back({"onOutput, onApiCall and onMemAccess observe the host thread", false, [] {
                 Machine m(compile("int main(void) { int x = 3; int* g; cudaMalloc(&g, 8);\n"
                                   "  printf(\"a%d\\n\", x); printf(\"b\\n\"); cudaFree(g); return 0; }\n"),
                           RunOptions{});
                 std::string out;
                 std::vector<std::pair<ApiId, int>> api;
                 int reads = 0, writes = 0;
                 m.onOutput = [&](const std::string& s) { out += s; };
                 m.onApiCall = [&](ApiId id, int code) { api.push_back({id, code}); };
                 m.onMemAccess = [&](const MemAccessInfo& a) {
                   (a.kind == AccessKind::Read ? reads : writes) += 1;
                   CHECK(a.accessor.isHost());
                 };
                 auto r = m.run();
                 CHECK(r.exitCode == 0);
                 CHECK(out == r.output);
                 CHECK(out == "a3\nb\n");
                 CHECK(api.size() == 2);
                 CHECK(api.size() == 2 && api[0].first == ApiId::Malloc && api[0].second == 0);
                 CHECK(api.size() == 2 && api[1].first == ApiId::Free);
                 CHECK(std::string(apiName(ApiId::Malloc)) == "cudaMalloc");
                 CHECK(reads > 0 && writes > 0);
               }});
  c.push_back({"onTrace receives the --trace lines in order", true, [] {
                 RunOptions o;
                 o.trace = true;
                 Machine m(compile(slurp(corpusPath("sum.cu")), "sum.cu"), o);
                 std::vector<std::string> lines;
                 m.onTrace = [&](const std::string& s) { lines.push_back(s); };
                 auto r = m.run();
                 CHECK(!lines.empty());
                 CHECK(lines == r.trace);
               }});
  c.push_back({"a non-round-robin schedule is flagged, not silent", false, [] {
                 RunOptions o;
                 o.policy = SchedulePolicy::SeededRandom;
                 o.seed = 7;
                 Machine m(compile("int main(void){return 0;}"), o);
                 CHECK(!m.run().engineNote.empty());
                 RunOptions z;
                 Machine m0(compile("int main(void){return 0;}"), z);
                 CHECK(m0.run().engineNote.empty());
               }});
  // ---- the race checker as a library (racecheck.cpp:9-73) ----
  c.push_back({"recordAccess / clearEpoch report the reference's races", true, [] {
                 Machine m(compile("int main(void){return 0;}", "trace.cu"), RunOptions{});
                 Location l = m.allocObject(MemSpace::deviceShared(1, 0), 64, "shared");
                 const MemObject& obj = m.object(l.object);
                 ThreadKey t0{1, 0, 0}, t1{1, 0, 1};
                 m.recordAccess(obj, 0, 4, t0, AccessKind::Write, SourceLoc{10, 1});
                 m.recordAccess(obj, 2, 4, t1, AccessKind::Read, SourceLoc{11, 1});   // bytes 2,3 race
                 m.recordAccess(obj, 8, 4, t1, AccessKind::Read, SourceLoc{12, 1});   // alone
                 m.flushRaces();
                 m.recordAccess(obj, 8, 4, t0, AccessKind::Write, SourceLoc{13, 1});  // sees the kept read
                 m.clearEpoch(1, 0);
                 m.recordAccess(obj, 16, 4, t0, AccessKind::Write, SourceLoc{14, 1});
                 m.recordAccess(obj, 16, 4, t0, AccessKind::Write, SourceLoc{15, 1});  // same thread: no race
                 m.recordAccess(obj, 0, 4, t1, AccessKind::Write, SourceLoc{16, 1});   // new epoch: no race
                 const auto& rep = m.raceReport();
                 std::vector<RaceTriple> want = {{l.object, 2, 11}, {l.object, 3, 11}, {l.object, 8, 13},
                                                 {l.object, 9, 13}, {l.object, 10, 13}, {l.object, 11, 13}};
                 CHECK(rep == want);
                 const auto& d = m.raceDiagnostics();
                 CHECK(d.size() == 2);
                 CHECK(d.size() == 2 && d[0].message == "Possible race on shared device memory detected at trace.cu:11.");
                 CHECK(d.size() == 2 && d[1].message == "Possible race on shared device memory detected at trace.cu:13.");
                 CHECK(d.size() == 2 && d[0].category == DiagCategory::Race && d[0].severity == Severity::Warning);
               }});
  return c;
}

}  // namespace

int main(int argc, char** argv) {
  for (int i = 1; i < argc; ++i)
    if (!std::strcmp(argv[i], "--no-gpu")) g_gpu = false;
  int ran = 0, skipped = 0;
  for (const Case& k : cases()) {
    if (k.gpu && !g_gpu) {
      ++skipped;
      continue;
    }
    g_case = k.name;
    try {
      k.body();
    } catch (const std::exception& e) {
      ++g_failed;
      std::fprintf(stderr, "FAIL [%s] exception: %s\n", k.name, e.what());
    }
    ++ran;
  }
  std::printf("%d cases run, %d skipped, %d checks, %d failed\n", ran, skipped, g_checks, g_failed);
  return g_failed ? 1 : 0;
}
