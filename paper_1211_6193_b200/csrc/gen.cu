// gen.cu -- on-device generator of the synthetic BASELINE config-3 trace.
// Record-for-record identical to oracle/tracegen.c (see the recipe in
// include/mckg.h, mckg_gen_c3).  Not a reference interface: it fills HBM with
// the benchmark input so the timed region starts with inputs resident.
#include "common.cuh"

namespace mckg {
namespace {

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void gen_c3_kernel(uint4* ev, unsigned long long* bs, uint32_t blk0, uint32_t n_blocks,
                              unsigned long long seed) {
  const unsigned long long per = MCKG_C3_EVENTS_PER_BLOCK;
  const unsigned long long total = (unsigned long long)n_blocks * per;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  for (unsigned long long r = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; r < total;
       r += stride) {
    unsigned long long i = (unsigned long long)blk0 * per + r;
    uint32_t j = (uint32_t)(i % per);
    uint32_t e = j / (MCKG_C3_THREADS * MCKG_C3_K);
    uint32_t k = (j / MCKG_C3_THREADS) % MCKG_C3_K;
    uint32_t tid = j % MCKG_C3_THREADS;
    unsigned long long h = splitmix64(seed + i);
    uint32_t write = (uint32_t)(h & 1u);
    bool redirect = ((h >> 32) % 10000u) < 100u;
    uint32_t t2 = redirect ? (tid + 1u) % MCKG_C3_THREADS : tid;
    uint32_t off = (t2 * 4u + k) * 4u;
    uint4 v;
    v.x = (off & 0xFFFFFu) | (4u << 20) | (write << 24);
    v.y = (tid & 0x7FFu) | (e << 11);
    v.z = 100u + k;
    v.w = (uint32_t)i;
    ev[r] = v;
  }
  for (unsigned long long b = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
       b <= n_blocks; b += stride)
    bs[b] = b * per;
}

}  // namespace
}  // namespace mckg

using namespace mckg;

extern "C" int mckg_gen_c3(mckg_access* events, uint64_t* block_start, uint32_t blk0,
                           uint32_t n_blocks, uint64_t seed, void* stream) {
  if (!events || !block_start) {
    set_error("mckg_gen_c3: null buffer");
    return MCKG_E_ARG;
  }
  uint32_t grid = (uint32_t)sm_count() * 8u;
  gen_c3_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<uint4*>(events), reinterpret_cast<unsigned long long*>(block_start), blk0,
      n_blocks, seed);
  MCKG_CUDA_TRY(cudaGetLastError());
  note_launch(1, grid, 256, 0);
  return MCKG_OK;
}
