// red_floor.cu — the floor of the lifetime stage's scattered 64-bit RED
// atomics: per_kernel_active_bytes is one
// `active[kernel] += size` per access event (reference analysis.py:111-117)
// and the timeline difference array two more per intermediate tensor
// (:97-108).  These kernels issue exactly those REDs over a real trace's
// access column and nothing else, so their time bounds k_events from below.
//
//   mode 0  stream the access column only (int4 loads), no atomics
//   mode 1  one RED.64 per event to active[acc[e]]              (10M at C3)
//   mode 2  mode 1 + the difference-array REDs (first / last+1 of every
//           intermediate tensor), i.e. k_events' full atomic traffic
//   mode 3  mode 1 with 32-bit REDs (half the L2 payload, same op count)
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC
//      tools/micro/red_floor.cu -o tools/micro/libred_floor.so
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_stream(const int4 *acc4, int64_t n4, unsigned long long *sink) {
    int s = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const int4 v = __ldg(acc4 + i);
        s ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (s == 0x7fffffff) atomicAdd(sink, 1ull);
}

__global__ void k_red_events(const int *acc, int64_t E, unsigned long long *active) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(active + __ldg(acc + e), 3ull);
}

__global__ void k_red_events32(const int *acc, int64_t E, unsigned *active) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(active + __ldg(acc + e), 3u);
}

// diff REDs: one thread per tensor, intermediates only
__global__ void k_red_diff(const int *acc, const int64_t *ptr, const int8_t *kind, int64_t T,
                           unsigned long long *diff) {
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
        if (__ldg(kind + t) == 1) continue;
        const int64_t b = __ldg(ptr + t), e = __ldg(ptr + t + 1);
        atomicAdd(diff + __ldg(acc + b), 5ull);
        atomicAdd(diff + __ldg(acc + e - 1) + 1, (unsigned long long)-5ll);
    }
}

extern "C" int red_floor(const int *acc, const int64_t *ptr, const int8_t *kind, int64_t E, int64_t T, int64_t N,
                         void *active, void *diff, int mode, int reps, float *ms_best) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    void *flush = nullptr;
    const size_t FL = 256u << 20;
    if (cudaMalloc(&flush, FL) != cudaSuccess) return 1;
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) {
        cudaMemsetAsync(flush, r & 0xff, FL);           // L2 flush
        cudaMemsetAsync(active, 0, 8 * (N + 1));
        cudaMemsetAsync(diff, 0, 8 * (N + 1));
        cudaEventRecord(a);
        const int G = sms * 8, B = 256;
        if (mode == 0) k_stream<<<G, B>>>(reinterpret_cast<const int4 *>(acc), E / 4,
                                          static_cast<unsigned long long *>(diff));
        if (mode == 1 || mode == 2)
            k_red_events<<<G, B>>>(acc, E, static_cast<unsigned long long *>(active));
        if (mode == 2) k_red_diff<<<G, B>>>(acc, ptr, kind, T, static_cast<unsigned long long *>(diff));
        if (mode == 3) k_red_events32<<<G, B>>>(acc, E, static_cast<unsigned *>(active));
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    *ms_best = best;
    cudaFree(flush);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
