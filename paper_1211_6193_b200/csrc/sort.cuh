// sort.cuh -- the hand-written device primitives of sort.cu (stream-ordered
// on `s`; scratch from the stream-ordered pool; `launches` counts kernels).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace mckg {

// out[i] = in[0] + ... + in[i-1] for i <= n (out has n + 1 entries)
cudaError_t exclusive_scan_u32(const uint32_t* in, uint64_t n, uint64_t* out, cudaStream_t s, uint32_t* launches);
// stable LSD radix sort of the low `bits` bits of n keys; tmp: n keys of scratch
cudaError_t radix_sort_u64(unsigned long long* keys, unsigned long long* tmp, uint64_t n, uint32_t bits,
                           cudaStream_t s, uint32_t* launches);
// distinct keys of a sorted array (out may not alias), *n_out their count (device)
cudaError_t unique_sorted_u64(const unsigned long long* sorted, uint64_t n, unsigned long long* out,
                              unsigned long long* n_out, cudaStream_t s, uint32_t* launches);
// out = { first + i : flags[i] != 0 } ascending, *n_out their count (device)
cudaError_t select_flagged_index(const uint8_t* flags, uint64_t n, uint32_t first, uint32_t* out, uint32_t* n_out,
                                 cudaStream_t s, uint32_t* launches);

}  // namespace mckg
