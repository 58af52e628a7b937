// block_scan.cuh — warp-shuffle block-wide scans/reductions (hand-written).
#pragma once
#include <cstdint>

namespace tio {

template <typename T>
__device__ __forceinline__ T warp_inclusive_sum(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Exclusive block scan; returns this thread's exclusive prefix and writes the
// block total to *total.  `sm` must hold >= 33 T and be private to the call.
// Contains __syncthreads: call from all threads of the block.
template <typename T>
__device__ __forceinline__ T block_exclusive_sum(T v, T *sm, T *total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = (blockDim.x + 31) >> 5;
    T inc = warp_inclusive_sum(v);
    if (lane == 31) sm[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T w = lane < nwarps ? sm[lane] : T(0);
        T wi = warp_inclusive_sum(w);
        if (lane < nwarps) sm[lane] = wi - w;
        if (lane == nwarps - 1) sm[32] = wi;
    }
    __syncthreads();
    T res = sm[warp] + inc - v;
    *total = sm[32];
    __syncthreads();
    return res;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T *sm) {
    T total;
    block_exclusive_sum(v, sm, &total);
    return total;
}

}  // namespace tio
