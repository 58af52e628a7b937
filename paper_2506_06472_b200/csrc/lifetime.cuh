// lifetime.cuh — lifetime-stage kernel interface.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tio {

#ifndef TIO_LT_THREADS
#define TIO_LT_THREADS 256
#endif
constexpr int LIFETIME_THREADS = TIO_LT_THREADS;   // event-tile block size (build knob)

// scalars[] slots shared by the lifetime and planner kernels
enum { SC_GLOBAL_BYTES = 0, SC_NUM_PERIODS = 1, SC_FLAGS = 2, SC_IDS_UNSORTED = 3, SC_COUNT = 8 };

struct LifetimeArgs {
    int64_t N, T, E;
    const int64_t *dur;
    const int64_t *tid;
    const int64_t *size;
    const int8_t *kind;
    const int64_t *ptr;
    const int32_t *acc;
    int64_t *starts;       // [N+1]
    int64_t *timeline;     // [N]
    int64_t *active;       // [N]   zeroed by the caller
    int64_t *diff;         // [N+1] zeroed by the caller
    int64_t *p_tensor;     // [E]   capacity (P <= E)
    int32_t *p_start;
    int32_t *p_end;
    int8_t *p_wraps;
    int64_t *tensor_pptr;  // [T+1]
    int64_t *work;         // [lifetime_workspace_elems(N, E)] tile counters, owners, look-back status
    int64_t *scalars;      // [SC_COUNT] zeroed by the caller
};

__host__ __device__ int64_t lifetime_event_tiles(int64_t E);
__host__ __device__ int64_t lifetime_kernel_tiles(int64_t N);
int64_t lifetime_workspace_elems(int64_t N, int64_t E);
// enqueues the lifetime stage (memsets of its look-back state + 3 kernels)
int launch_lifetime(const LifetimeArgs &args, cudaStream_t stream);

}  // namespace tio
