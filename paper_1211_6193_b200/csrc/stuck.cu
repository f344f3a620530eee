// stuck.cu -- K4: barrier-deadlock classification at quiescence (sm_100a).
//
// Replaces the BarrierDeadlock part of Machine::scanStuck (deadlock.cpp:12-34).
// Input: per-thread __syncthreads arrival counts when nothing can move.  The
// token protocol (device.cpp:111-200) can only complete an episode once every
// thread of the block has arrived, and finished/halted threads leave
// cfg_.device (machine.cpp:460-463), so at quiescence the completed episodes
// are m = min_t c_t and exactly the threads with c_t > m wait.  One CTA per
// simulated block: a warp-shuffle min reduction, then one __ballot_sync per
// 32 tids builds the waiting mask (the report's waitingTids; its complement
// is missingTids), and __syncthreads_or flags the block.  Deadlocked bids are
// stream-compacted in ascending order (the std::map walk of deadlock.cpp:15).

#include "common.cuh"
#include "sort.cuh"

namespace mckg {
namespace {

constexpr int NT = 256;

__global__ void __launch_bounds__(NT) stuck_kernel(const uint32_t* __restrict__ arr,
                                                   uint32_t n_blocks, uint32_t block_dim,
                                                   uint32_t words, uint32_t* __restrict__ wmask,
                                                   uint8_t* __restrict__ flags) {
  __shared__ uint32_t wmin[NT / 32];
  const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
  for (uint32_t b = blockIdx.x; b < n_blocks; b += gridDim.x) {
    const uint32_t* base = arr + (size_t)b * block_dim;
    uint32_t m = 0xFFFFFFFFu;
    for (uint32_t i = t; i < block_dim; i += NT) m = min(m, __ldg(base + i));
    m = __reduce_min_sync(0xFFFFFFFFu, m);
    if (lane == 0) wmin[warp] = m;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NT / 32; ++k) m = min(m, wmin[k]);
    uint32_t any = 0;
    for (uint32_t j = warp; j < words; j += NT / 32) {
      uint32_t tid = j * 32u + lane;
      uint32_t c = tid < block_dim ? __ldg(base + tid) : m;
      uint32_t bits = __ballot_sync(0xFFFFFFFFu, c > m);
      if (lane == 0) wmask[(size_t)b * words + j] = bits;
      any |= bits;
    }
    int dl = __syncthreads_or(any != 0);
    if (t == 0) flags[b] = dl ? 1 : 0;
  }
}

}  // namespace
}  // namespace mckg

using namespace mckg;

extern "C" int mckg_scan_stuck(const uint32_t* arrivals, uint32_t n_blocks, uint32_t block_dim,
                               uint32_t bid_base, uint32_t* waiting_mask, uint32_t* dl_bids,
                               uint32_t* n_dl, void* stream) {
  if (!arrivals || !waiting_mask || !dl_bids || !n_dl || block_dim == 0) {
    set_error("mckg_scan_stuck: null argument");
    return MCKG_E_ARG;
  }
  cudaStream_t s = (cudaStream_t)stream;
  keep_pool_memory();
  if (n_blocks == 0) {
    MCKG_CUDA_TRY(cudaMemsetAsync(n_dl, 0, sizeof(uint32_t), s));
    return MCKG_OK;
  }
  const uint32_t words = (block_dim + 31u) / 32u;
  PoolGuard pg(s);
  uint8_t* flags = nullptr;
  MCKG_CUDA_TRY(pg.alloc(&flags, n_blocks));
  uint32_t grid = n_blocks < (uint32_t)sm_count() * 8u ? n_blocks : (uint32_t)sm_count() * 8u;
  stuck_kernel<<<grid, NT, 0, s>>>(arrivals, n_blocks, block_dim, words, waiting_mask, flags);
  MCKG_CUDA_TRY(cudaGetLastError());
  // the deadlocked bids in ascending order (hand-written compaction, sort.cu)
  uint32_t launches = 1;
  MCKG_CUDA_TRY(select_flagged_index(flags, n_blocks, bid_base, dl_bids, n_dl, s, &launches));
  note_launch(launches, grid, NT, 0);
  return MCKG_OK;
}
