// radix_sort.cuh — stable LSD radix sort of (u64 key, u32 value) pairs.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tio {

// Sorts the low `bits` bits of keys (stable).  hist needs radix_hist_elems(n)
// uint32.  On return *result_in_tmp says whether the sorted data is in the
// *_tmp buffers (odd number of passes).
int radix_sort_pairs(uint64_t *keys, uint32_t *vals, uint64_t *keys_tmp, uint32_t *vals_tmp,
                     int64_t *hist, int64_t n, int bits, cudaStream_t stream, bool *result_in_tmp);
int64_t radix_hist_elems(int64_t n);

}  // namespace tio
