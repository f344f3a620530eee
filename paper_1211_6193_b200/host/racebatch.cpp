// racebatch.cpp -- Machine::recordAccess / Machine::clearEpoch as a library,
// batched on the K2 kernel (include/mck/checker.hpp; reference:
// racecheck.cpp:9-73, machine.hpp:407-409).
//
// The reference checks one access at a time against a per-byte shadow map.
// Here each call appends a 16-byte mckg_access record to its object's segment
// (timestamp = call sequence number, epoch = the clearEpoch count of the
// object's block), and flushRaces() hands every segment to K2 through
// mckg_detect_shared_host.  Objects never interact (the shadow is keyed by
// object), so the K2 trace holds one segment per object.  The reported set
// and the first-detection order of the Race diagnostics are the reference's
// (K2's parity contract); a flush only defers them.  The records
// of each segment's open epoch stay in the batch, so accesses after a flush
// still see them; the races they already produced are deduplicated by the
// reported set and by the diagnostic messages, as addDiagnostic does.
#include <algorithm>
#include <stdexcept>
#include <string>

#include "machine_impl.hpp"
#include "program.hpp"

namespace mck {

Location Machine::allocObject(MemSpace space, int64_t size, const std::string& name) {
  if (size < 0) throw std::invalid_argument("allocObject: negative size");
  MemObject o;
  o.id = impl_->nextObject++;
  o.space = space;
  o.size = size;
  o.name = name;
  impl_->objects[o.id] = o;
  return Location{o.id, 0};
}

const MemObject& Machine::object(ObjectId id) const {
  auto it = impl_->objects.find(id);
  if (it == impl_->objects.end()) throw std::out_of_range("object: unknown object id " + std::to_string(id));
  return it->second;
}

void Machine::recordAccess(const MemObject& obj, int64_t off, int64_t len, ThreadKey thread, AccessKind kind,
                           SourceLoc loc) {
  if (!opts_.raceCheck) return;  // RaceState::enabled (racecheck.cpp:11)
  if (len <= 0) return;
  if (off < 0 || off + len > static_cast<int64_t>(MCKG_MAX_OFF))
    throw std::out_of_range("recordAccess: byte offset beyond the packed record's 2^20");
  if (loc.line < 0 || loc.line >= static_cast<int>(MCKG_MAX_LINES))
    throw std::out_of_range("recordAccess: source line outside 0..65535");
  RaceBatch& B = impl_->race;
  RaceBatch::Segment& seg = B.segments[obj.id];
  seg.object = obj.id;
  seg.space = obj.space;
  // clearEpoch(gid, bid) erases the shadow of DeviceShared(gid, bid) objects
  // only (racecheck.cpp:54-73): any other object stays in epoch 0
  const uint32_t epoch = obj.space.kind == SpaceKind::DeviceShared ? B.epochOf[{obj.space.gid, obj.space.bid}] : 0u;
  if (epoch >= MCKG_MAX_EPOCH) throw std::length_error("recordAccess: more than 2^21 epochs of one block");
  auto t = seg.tids.find(thread);
  if (t == seg.tids.end()) {
    if (seg.tids.size() >= MCKG_MAX_TID)
      throw std::length_error("recordAccess: more than 2048 threads access one object");
    t = seg.tids.emplace(thread, static_cast<uint32_t>(seg.tids.size())).first;
  }
  // an access longer than a scalar is split into <= 8-byte pieces: the check
  // is per byte (racecheck.cpp:24), and the pieces cover disjoint bytes
  for (int64_t p = off; p < off + len; p += MCKG_MAX_LEN) {
    if (B.seq >= 0xFFFFFFFFull) flushRaces();
    if (B.seq >= 0xFFFFFFFFull) throw std::length_error("recordAccess: more than 2^32 accesses in one epoch");
    const uint32_t piece = static_cast<uint32_t>(std::min<int64_t>(MCKG_MAX_LEN, off + len - p));
    seg.events.push_back(mckg_make_access(static_cast<uint32_t>(p), piece, kind == AccessKind::Write, t->second,
                                          epoch, loc.line, static_cast<uint32_t>(B.seq++)));
  }
  seg.lastEpoch = epoch;
}

void Machine::clearEpoch(GridId gid, int bid) { ++impl_->race.epochOf[{gid, bid}]; }

void Machine::flushRaces() {
  RaceBatch& B = impl_->race;
  std::vector<mckg_access> ev;
  std::vector<uint64_t> starts{0};
  std::vector<ObjectId> objs;
  uint32_t maxBlock = 0, extent = 4;
  uint64_t bytes = 0;
  for (auto& [id, seg] : B.segments) {
    if (seg.fresh == seg.events.size()) continue;  // nothing new: its races are known
    ev.insert(ev.end(), seg.events.begin(), seg.events.end());
    starts.push_back(ev.size());
    objs.push_back(id);
    maxBlock = std::max<uint32_t>(maxBlock, static_cast<uint32_t>(seg.events.size()));
    for (const mckg_access& a : seg.events) {
      bytes += MCKG_ACC_LEN(a);
      extent = std::max<uint32_t>(extent, MCKG_ACC_OFF(a) + MCKG_ACC_LEN(a));
    }
  }
  if (!objs.empty()) {
    if (objs.size() >= MCKG_MAX_BID) throw std::length_error("flushRaces: more than 2^21 objects in one flush");
    mckg_trace tr{};
    tr.events = ev.data();
    tr.block_start = starts.data();
    tr.n_events = ev.size();
    tr.n_blocks = static_cast<uint32_t>(objs.size());
    tr.max_block_events = maxBlock;
    tr.obj_base = 0;  // K2 reports the segment index; mapped back to the object below
    tr.bid_base = 0;
    tr.shmem_bytes = extent;  // the largest object extent touched
    tr.gid = 1;
    std::vector<mckg_race_triple> tri(std::max<uint64_t>(1, bytes));
    std::vector<uint64_t> lineFirst(MCKG_MAX_LINES, MCKG_TS_NONE);
    uint64_t n = 0;
    uint32_t status = 0;
    const int rc = mckg_detect_shared_host(&tr, tri.data(), tri.size(), &n, lineFirst.data(), &status);
    if (rc != MCKG_OK) throw std::runtime_error(std::string("flushRaces: K2 failed: ") + mckg_last_error());
    if (status & (MCKG_ST_RANGE | MCKG_ST_ORDER | MCKG_ST_OVERFLOW))
      throw std::runtime_error("flushRaces: K2 status " + std::to_string(status));
    for (uint64_t i = 0; i < std::min<uint64_t>(n, tri.size()); ++i)
      B.reportedSet.insert(RaceTriple{objs[tri[i].obj], tri[i].byte, tri[i].line});
    // Race diagnostics of this flush in first-detection order (addDiagnostic
    // dedups by message, machine.cpp:41-46)
    std::vector<std::pair<uint64_t, uint32_t>> lines;
    for (uint32_t l = 0; l < MCKG_MAX_LINES; ++l)
      if (lineFirst[l] != MCKG_TS_NONE) lines.push_back({lineFirst[l], l});
    std::sort(lines.begin(), lines.end());
    for (const auto& [ts, l] : lines) {
      (void)ts;
      Diagnostic d;
      d.severity = Severity::Warning;
      d.category = DiagCategory::Race;
      d.message = "Possible race on shared device memory detected at " + program().filename + ":" +
                  std::to_string(l) + ".";
      d.loc.line = static_cast<int>(l);
      if (B.messages.insert(d.message).second) B.diagnostics.push_back(std::move(d));
    }
  }
  B.reported.assign(B.reportedSet.begin(), B.reportedSet.end());
  // keep each segment's open epoch only (later accesses of that epoch must
  // still see it); an object whose block moved on keeps nothing
  for (auto& [id, seg] : B.segments) {
    const uint32_t cur =
        seg.space.kind == SpaceKind::DeviceShared ? B.epochOf[{seg.space.gid, seg.space.bid}] : seg.lastEpoch;
    auto first = std::find_if(seg.events.begin(), seg.events.end(),
                              [&](const mckg_access& a) { return MCKG_ACC_EPOCH(a) == cur; });
    seg.events.erase(seg.events.begin(), first);
    seg.fresh = seg.events.size();
  }
}

const std::vector<RaceTriple>& Machine::raceReport() {
  flushRaces();
  return impl_->race.reported;
}

const std::vector<Diagnostic>& Machine::raceDiagnostics() {
  flushRaces();
  return impl_->race.diagnostics;
}

}  // namespace mck
