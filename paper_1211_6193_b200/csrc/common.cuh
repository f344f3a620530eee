// common.cuh -- shared helpers of the sm_100a kernels behind include/mckg.h.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "mckg.h"

namespace mckg {

// Records the last CUDA/argument error of this thread for mckg_last_error().
void set_error(const char* what, cudaError_t e = cudaSuccess);
void note_launch(uint32_t kernels, uint32_t grid, uint32_t block, uint32_t smem);
void add_launches(uint32_t kernels);
// MCKG_DEBUG / mckg_set_debug switches (experiments, and the tests that
// exercise the general paths)
uint32_t debug_flags();
int sm_count();
// Keeps freed stream-ordered allocations in the device's default memory pool
// (release threshold = max): the detectors allocate multi-GB scratch per call.
void keep_pool_memory();

#define MCKG_CUDA_TRY(expr)                                  \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) {                                 \
      ::mckg::set_error(#expr, _e);                          \
      return MCKG_E_CUDA;                                    \
    }                                                        \
  } while (0)

// ---- record field access (mirrors the MCKG_ACC_* macros) ----
__device__ __forceinline__ uint32_t acc_off(uint32_t w0) { return w0 & 0xFFFFFu; }
__device__ __forceinline__ uint32_t acc_len(uint32_t w0) { return (w0 >> 20) & 0xFu; }
__device__ __forceinline__ uint32_t acc_write(uint32_t w0) { return (w0 >> 24) & 1u; }
__device__ __forceinline__ uint32_t acc_tid(uint32_t w1) { return w1 & 0x7FFu; }
__device__ __forceinline__ uint32_t acc_epoch(uint32_t w1) { return w1 >> 11; }

__device__ __forceinline__ unsigned long long ts_key(uint32_t sweep, uint32_t bid, uint32_t tid) {
  return ((unsigned long long)sweep << 32) |
         ((unsigned long long)(bid & (MCKG_MAX_BID - 1)) << 11) | (tid & (MCKG_MAX_TID - 1));
}

// ---- mbarrier + 1-D bulk copy (TMA engine, cp.async.bulk) ----
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Frees the stream-ordered allocations of a host routine when it returns,
// the early error returns of MCKG_CUDA_TRY included.
struct PoolGuard {
  cudaStream_t s;
  std::vector<void*> p;
  explicit PoolGuard(cudaStream_t st) : s(st) {}
  PoolGuard(const PoolGuard&) = delete;
  PoolGuard& operator=(const PoolGuard&) = delete;
  template <typename T>
  cudaError_t alloc(T** out, size_t bytes) {
    const cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(out), bytes, s);
    if (e == cudaSuccess) p.push_back(*out);
    return e;
  }
  ~PoolGuard() {
    for (void* x : p) cudaFreeAsync(x, s);
  }
};

}  // namespace mckg
