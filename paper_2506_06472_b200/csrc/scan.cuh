// scan.cuh — device-wide int64 exclusive scan.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tio {
int64_t scan_tmp_elems(int64_t n);
// out = exclusive prefix of in (may alias); *grand = total (device pointer, may be null)
int exclusive_scan(const int64_t *in, int64_t *out, int64_t n, int64_t *tmp, int64_t *grand,
                   cudaStream_t stream);
}  // namespace tio
