// machine_impl.hpp -- the state behind mck::Machine (include/mck/checker.hpp):
// the last run's host interpreter and result, the object table of the
// library-level race checker, and the batch of shared accesses waiting for
// the K2 kernel (host/racebatch.cpp).
#pragma once
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "mck/checker.hpp"
#include "mckg.h"

namespace mckb {
class HostMachine;
}

namespace mck {

// Accesses recorded through Machine::recordAccess, grouped per object (one
// K2 trace segment each) in call order; timestamps are the call sequence.
struct RaceBatch {
  struct Segment {
    ObjectId object = 0;
    MemSpace space;
    std::vector<mckg_access> events;     // the open epoch first (kept across flushes), then new ones
    size_t fresh = 0;                    // events[fresh..] arrived since the last flush
    std::map<ThreadKey, uint32_t> tids;  // accessing threads -> dense K2 tids
    uint32_t lastEpoch = 0;
  };
  std::map<ObjectId, Segment> segments;
  std::map<std::pair<GridId, int>, uint32_t> epochOf;  // clearEpoch count per block
  uint64_t seq = 0;
  std::set<RaceTriple> reportedSet;
  std::vector<RaceTriple> reported;  // std::set order, refreshed by each flush
  std::set<std::string> messages;
  std::vector<Diagnostic> diagnostics;
};

class MachineImpl {
 public:
  std::unique_ptr<mckb::HostMachine> m;
  RunResult last;
  bool ran = false;
  std::map<ObjectId, MemObject> objects;
  ObjectId nextObject = 1;
  RaceBatch race;
};

}  // namespace mck
