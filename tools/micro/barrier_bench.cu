// Micro-benchmark: grid-barrier latency of a co-resident grid (296 blocks x
// 256 threads = the planner's grid) for the flat barrier used by the planner
// and a two-level variant.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void flat_barrier(unsigned *bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            unsigned ns = 32;
            while (*gen == g) { __nanosleep(ns); if (ns < 256) ns <<= 1; }
        }
        __threadfence();
    }
    __syncthreads();
}

__device__ __forceinline__ void flat_barrier_spin(unsigned *bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) { }
        }
        __threadfence();
    }
    __syncthreads();
}

// two-level: groups of GS blocks; the group's last arriver joins the top
// counter; release through one generation word
template <int GS>
__device__ __forceinline__ void tree_barrier(unsigned *bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *gen = bar + 1;
        const unsigned g = *gen;
        const int grp = blockIdx.x / GS;
        const int ngrp = (gridDim.x + GS - 1) / GS;
        const unsigned gsize = (grp == ngrp - 1) ? gridDim.x - grp * GS : GS;
        unsigned *gc = bar + 64 + 32 * grp;    // one 128-byte line per group
        __threadfence();
        bool released = false;
        if (atomicAdd(gc, 1u) == gsize - 1) {
            atomicExch(gc, 0u);
            if (atomicAdd(bar, 1u) == (unsigned)ngrp - 1) {
                atomicExch(bar, 0u);
                __threadfence();
                atomicAdd(bar + 1, 1u);
                released = true;
            }
        }
        if (!released) while (*gen == g) { }
        __threadfence();
    }
    __syncthreads();
}

// monotone counter: every block adds 1 with release semantics, then waits
// (acquire loads) until the counter reaches the next multiple of gridDim.x
__device__ __forceinline__ void count_barrier(unsigned long long *ctr, unsigned long long &target) {
    __syncthreads();
    target += gridDim.x;
    if (threadIdx.x == 0) {
        unsigned long long v;
        asm volatile("atom.add.release.gpu.u64 %0, [%1], 1;" : "=l"(v) : "l"(ctr) : "memory");
        while (v < target) {
            asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        }
    }
    __syncthreads();
}

template <int MODE>
__global__ void k(unsigned *bar, int iters, long long *out) {
    long long t0 = clock64();
    unsigned long long target = 0;
    for (int i = 0; i < iters; ++i) {
        if (MODE == 3) count_barrier(reinterpret_cast<unsigned long long *>(bar + 2048), target);
        else if (MODE == 0) flat_barrier(bar);
        else if (MODE == 1) flat_barrier_spin(bar);
        else tree_barrier<16>(bar);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = clock64() - t0;
}

int main() {
    unsigned *bar; long long *out;
    cudaMalloc(&bar, 64 * 1024);
    cudaMalloc(&out, 8);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 20000;
    for (int grid : {sms, 2 * sms}) {
        for (int mode = 0; mode < 4; ++mode) {
            cudaMemset(bar, 0, 64 * 1024);
            cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
            void *args[] = {&bar, (void *)&iters, &out};
            const void *f = mode == 0 ? (const void *)k<0> : mode == 1 ? (const void *)k<1> : mode == 2 ? (const void *)k<2> : (const void *)k<3>;
            cudaLaunchCooperativeKernel(f, grid, 256, args, 0, 0);   // warm
            cudaMemset(bar, 0, 64 * 1024);
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel(f, grid, 256, args, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("grid %d mode %s: %.3f us per barrier (%s)\n", grid, mode == 0 ? "flat+nanosleep" : mode == 1 ? "flat spin" : mode == 2 ? "tree16 spin" : "counter acq/rel",
                   ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
