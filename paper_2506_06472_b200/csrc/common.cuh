// common.cuh — shared helpers for libtio (sm_100a).
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>

#include "../../include/tio.h"

namespace tio {

typedef unsigned __int128 u128;

// ---- error plumbing --------------------------------------------------------
void set_error(const char *fmt, ...);
int fail(int code, const char *fmt, ...);
// process-wide count of libtio kernel launches (tio_kernel_launches)
void count_launch(int n = 1);

#define TIO_CUDA(expr)                                                                      \
    do {                                                                                    \
        cudaError_t _e = (expr);                                                            \
        if (_e != cudaSuccess)                                                              \
            return ::tio::fail(TIO_ERR_CUDA, "%s failed: %s (%s:%d)", #expr,                 \
                               cudaGetErrorString(_e), __FILE__, __LINE__);                 \
    } while (0)

#define TIO_TRY(expr)                                                                       \
    do {                                                                                    \
        int _rc = (expr);                                                                   \
        if (_rc != TIO_OK) return _rc;                                                      \
    } while (0)

// ---- device helpers ----------------------------------------------------------

// Loads that bypass L1: every mutable array of the persistent planner is read
// with these so a CTA never sees a stale line written by another SM.
__device__ __forceinline__ int64_t ld_cg(const int64_t *p) { return __ldcg(reinterpret_cast<const long long *>(p)); }
__device__ __forceinline__ int32_t ld_cg(const int32_t *p) { return __ldcg(p); }
__device__ __forceinline__ uint64_t ld_cg(const uint64_t *p) { return __ldcg(reinterpret_cast<const unsigned long long *>(p)); }
__device__ __forceinline__ int8_t ld_cg(const int8_t *p) { return (int8_t)__ldcg(reinterpret_cast<const signed char *>(p)); }
__device__ __forceinline__ uint8_t ld_cg(const uint8_t *p) { return (uint8_t)__ldcg(reinterpret_cast<const unsigned char *>(p)); }

// Grid-wide barrier for a co-resident (cooperatively launched) grid: one
// monotone 64-bit arrival counter.  Thread 0 of every block adds 1 with
// release semantics (gpu scope; cumulative over the block's writes ordered by
// the preceding __syncthreads) and polls with acquire loads until the counter
// reaches the next multiple of gridDim.x: the value it added to tells the
// barrier's phase, so no reset or generation word is needed.  Measured on
// the B200: 1.18 us per barrier at 296 blocks (a counter + generation
// barrier with __threadfence: 2.44 us; tools/micro/barrier_bench.cu).
// bar[0..1] = the counter (zeroed before the launch).
// G: the blocks taking part (gridDim.x, or one rank's share of a grid that
// runs several planner instances).
__device__ __forceinline__ void grid_barrier(unsigned *bar, unsigned G) {
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long *ctr = reinterpret_cast<unsigned long long *>(bar);
        unsigned long long v;
        asm volatile("atom.add.release.gpu.u64 %0, [%1], 1;" : "=l"(v) : "l"(ctr) : "memory");
        const unsigned long long target = (v / G + 1) * G;
        while (v < target) {
            asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
        }
    }
    __syncthreads();
}
__device__ __forceinline__ void grid_barrier(unsigned *bar) { grid_barrier(bar, gridDim.x); }

__device__ __forceinline__ void atomic_add_i64(int64_t *p, int64_t v) {
    atomicAdd(reinterpret_cast<unsigned long long *>(p), (unsigned long long)v);
}

// a/b > c/d exactly for a,c < 2^128 and b,d < 2^63 (192-bit cross products).
__host__ __device__ __forceinline__ bool ratio_gt(u128 a, int64_t b, u128 c, int64_t d) {
    uint64_t a0 = (uint64_t)a, a1 = (uint64_t)(a >> 64);
    uint64_t c0 = (uint64_t)c, c1 = (uint64_t)(c >> 64);
    u128 lo1 = (u128)a0 * (uint64_t)d, hi1 = (u128)a1 * (uint64_t)d;
    u128 lo2 = (u128)c0 * (uint64_t)b, hi2 = (u128)c1 * (uint64_t)b;
    u128 top1 = hi1 + (lo1 >> 64), top2 = hi2 + (lo2 >> 64);
    if (top1 != top2) return top1 > top2;
    return (uint64_t)lo1 > (uint64_t)lo2;
}

// Exact transfer duration of bandwidth.py:75-84 given a pre-decoded rate.
// Integral rate r: ceil(n / r).  Fractional rate m / 2^k (the exact value of
// the double): ceil(n * 2^k / m).
struct RateCode {
    int64_t num;    // integral rate, or mantissa m
    int32_t shift;  // 0 for integral, k for fractional
    int32_t huge;   // integral rate >= 2^63: every non-empty transfer takes 1 us
};

// Decode a rate (bytes/us, a double) into RateCode; TIO_ERR_CHANNEL_CONFIG if <= 0.
int decode_rate(double rate, RateCode *rc);

__host__ __device__ __forceinline__ int64_t duration_of(const RateCode &r, int64_t nbytes) {
    if (nbytes <= 0) return 0;
    if (r.huge) return 1;
    if (r.shift == 0) return nbytes / r.num + (nbytes % r.num != 0);
    if (r.shift > 64) {
        // ceil(nbytes * 2^shift / num) by long division, 8 bits at a time
        // (num < 2^53, so the shifted remainder stays below 2^61); only very
        // small fractional rates (< ~5e-4 B/us) take this path
        const uint64_t m = (uint64_t)r.num;
        uint64_t q = (uint64_t)nbytes / m, rem = (uint64_t)nbytes % m;
        for (int left = r.shift; left > 0;) {
            const int c = left < 8 ? left : 8;
            if (q >> (63 - c)) return INT64_MAX;   // saturates: > any iteration
            rem <<= c;
            q = (q << c) | (rem / m);
            rem %= m;
            left -= c;
        }
        q += rem != 0;
        return q > (uint64_t)INT64_MAX ? INT64_MAX : (int64_t)q;
    }
    u128 num = ((u128)(uint64_t)nbytes) << r.shift;
    u128 m = (u128)(uint64_t)r.num;
    u128 q = num / m + (num % m != 0);
    if (q > (u128)INT64_MAX) return INT64_MAX;  // flagged on the host side (>iteration anyway)
    return (int64_t)q;
}

// grid size used by all persistent / cooperative kernels
struct Launch {
    int sms = 148;
    int blocks = 296;
};

// Programmatic dependent launch: the kernel may become resident while the
// previous kernel on the stream drains; it must execute pdl_wait() before
// touching anything (every kernel launched this way does so first).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args... args) {
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

}  // namespace tio
