// mgpu.cu -- the multi-GPU entry points of the C ABI (include/mckg.h): one
// process per GPU, an NCCL communicator owned by the library, the exchange
// steps of SURVEY §8(e) done in C++ rather than by the caller.
//
//   mckg_detect_shared_mgpu  C3 sharded by blocks: K2 on this rank's blocks,
//                            then one all-reduce(MIN) of the per-line first
//                            racing keys, so every rank holds the report
//                            order (the triples stay per rank, disjoint).
//   mckg_detect_global_mgpu  C5: K3 partition by owner (address range),
//                            count all-gather, grouped ncclSend/ncclRecv of
//                            the 16-byte records (all-to-all over NVLink),
//                            K6 on the records this rank owns, all-reduce(MIN)
//                            of the line table.  The (byte, line) sets are
//                            disjoint across ranks by construction.
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

struct mckg_comm {
  ncclComm_t nccl = nullptr;
  int rank = 0, world = 1, device = 0;
  uint64_t* counts = nullptr;  // device: [world] send counts, [world * world] gathered
};

namespace mckg {
namespace {

int nccl_err(const char* what, ncclResult_t r) {
  std::string m = std::string(what) + ": " + ncclGetErrorString(r);
  set_error(m.c_str());
  return MCKG_E_CUDA;
}

}  // namespace
}  // namespace mckg

using namespace mckg;

#define MCKG_NCCL_TRY(expr)                            \
  do {                                                 \
    ncclResult_t _r = (expr);                          \
    if (_r != ncclSuccess) return nccl_err(#expr, _r); \
  } while (0)

extern "C" int mckg_comm_init(const uint8_t id[128], int rank, int world, int device, mckg_comm** out) {
  if (!id || !out || world < 1 || rank < 0 || rank >= world || world > 64) {
    set_error("mckg_comm_init: bad argument");
    return MCKG_E_ARG;
  }
  *out = nullptr;
  MCKG_CUDA_TRY(cudaSetDevice(device));
  ncclUniqueId u;
  static_assert(sizeof(u.internal) == 128, "ncclUniqueId");
  std::memcpy(u.internal, id, 128);
  auto* c = new mckg_comm;
  c->rank = rank;
  c->world = world;
  c->device = device;
  ncclResult_t r = ncclCommInitRank(&c->nccl, world, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_err("ncclCommInitRank", r);
  }
  if (cudaMalloc(&c->counts, (size_t)(world + world * world) * sizeof(uint64_t)) != cudaSuccess) {
    ncclCommDestroy(c->nccl);
    delete c;
    set_error("mckg_comm_init: cudaMalloc");
    return MCKG_E_CUDA;
  }
  *out = c;
  return MCKG_OK;
}

extern "C" void mckg_comm_destroy(mckg_comm* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->nccl) ncclCommDestroy(c->nccl);
  if (c->counts) cudaFree(c->counts);
  delete c;
}

extern "C" int mckg_detect_shared_mgpu(mckg_comm* c, const mckg_trace* shard, const mckg_race_out* out,
                                       void* stream) {
  if (!c || !out || !out->line_first) {
    set_error("mckg_detect_shared_mgpu: null argument");
    return MCKG_E_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  int rc = mckg_detect_shared(shard, out, stream);
  if (rc != MCKG_OK) return rc;
  // unsigned 64-bit MIN: the earliest racing key of every line over all ranks
  MCKG_NCCL_TRY(ncclAllReduce(out->line_first, out->line_first, MCKG_MAX_LINES, ncclUint64, ncclMin, c->nccl, s));
  add_launches(3);
  return MCKG_OK;
}

extern "C" int mckg_detect_global_mgpu(mckg_comm* c, const mckg_gaccess* events, uint64_t n, uint64_t addr_space,
                                       mckg_grace* races, uint64_t capacity, unsigned long long* n_races,
                                       unsigned long long* line_first, uint32_t* status, void* stream) {
  if (!c || (!events && n) || !n_races || !line_first || !status || addr_space == 0) {
    set_error("mckg_detect_global_mgpu: bad argument");
    return MCKG_E_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  keep_pool_memory();
  const int P = c->world;
  const uint64_t lo = ((uint64_t)c->rank * addr_space + P - 1) / P;  // first address this rank owns
  if (P == 1) {
    int rc = mckg_detect_global(events, n, lo, races, capacity, n_races, line_first, status, stream);
    if (rc != MCKG_OK) return rc;
    MCKG_NCCL_TRY(ncclAllReduce(line_first, line_first, MCKG_MAX_LINES, ncclUint64, ncclMin, c->nccl, s));
    return MCKG_OK;
  }
  // 1. K3: records grouped by owner, per-owner counts
  PoolGuard pg(s);
  mckg_gaccess* grouped = nullptr;
  MCKG_CUDA_TRY(pg.alloc(&grouped, (n ? n : 1) * sizeof(mckg_gaccess)));
  int rc = mckg_partition_global(events, n, (uint32_t)P, addr_space, grouped, c->counts, stream);
  if (rc != MCKG_OK) return rc;
  // 2. every rank's counts to every rank
  uint64_t* all = c->counts + P;
  MCKG_NCCL_TRY(ncclAllGather(c->counts, all, (size_t)P, ncclUint64, c->nccl, s));
  std::vector<uint64_t> h((size_t)P * P);
  MCKG_CUDA_TRY(cudaMemcpyAsync(h.data(), all, h.size() * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  MCKG_CUDA_TRY(cudaStreamSynchronize(s));
  std::vector<uint64_t> sendOff(P + 1, 0), recvOff(P + 1, 0);
  for (int r = 0; r < P; ++r) {
    sendOff[r + 1] = sendOff[r] + h[(size_t)c->rank * P + r];  // what this rank sends to r
    recvOff[r + 1] = recvOff[r] + h[(size_t)r * P + c->rank];  // what r sends to this rank
  }
  const uint64_t nrecv = recvOff[P];
  mckg_gaccess* mine = nullptr;
  MCKG_CUDA_TRY(pg.alloc(&mine, (nrecv ? nrecv : 1) * sizeof(mckg_gaccess)));
  // 3. the all-to-all of the records (NVLink peer to peer)
  MCKG_NCCL_TRY(ncclGroupStart());
  for (int r = 0; r < P; ++r) {
    const size_t sb = (size_t)(sendOff[r + 1] - sendOff[r]) * sizeof(mckg_gaccess);
    const size_t rb = (size_t)(recvOff[r + 1] - recvOff[r]) * sizeof(mckg_gaccess);
    if (sb) MCKG_NCCL_TRY(ncclSend(grouped + sendOff[r], sb, ncclUint8, r, c->nccl, s));
    if (rb) MCKG_NCCL_TRY(ncclRecv(mine + recvOff[r], rb, ncclUint8, r, c->nccl, s));
  }
  MCKG_NCCL_TRY(ncclGroupEnd());
  // 4. K6 on the owned range, 5. the report order over all ranks
  rc = mckg_detect_global(mine, nrecv, lo, races, capacity, n_races, line_first, status, stream);
  if (rc != MCKG_OK) return rc;
  MCKG_NCCL_TRY(ncclAllReduce(line_first, line_first, MCKG_MAX_LINES, ncclUint64, ncclMin, c->nccl, s));
  return MCKG_OK;
}
