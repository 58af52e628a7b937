// lifetime.cu — the lifetime stage on sm_100a.
//
// One cooperative (persistent) kernel, three phases separated by grid
// barriers, replacing reference analysis.py:58-117 and trace.py:97-107:
//
//   phase A  events (tensor-major CSR, each thread a contiguous strip):
//              active[k] += size        (per_kernel_active_bytes, :111-117)
//              diff[first] += size, diff[last+1] -= size for intermediates,
//              global bytes summed      (compute_memory_timeline, :97-108)
//              per-thread count of inactive periods (gaps b-a>1, wrap of
//              globals when (n-1-last)+first > 0)   (compute_inactive_periods)
//              validation flags for the invariants the kernels rely on
//            kernels: per-block duration sums (start-time scan)
//   phase B  period records written at their scanned offsets, in reference
//            order (tensor order, gaps ascending, wrap last), plus the
//            per-tensor period offsets; kernel start times; diff block sums
//   phase C  timeline = globals + inclusive scan of diff
//
// Roofline: HBM-bound integer work; algorithmic bytes per trace
//   B_L = 8E (event read, +4E for the second pass, L2-resident) ... see DESIGN.md.
#include "common.cuh"
#include "block_scan.cuh"
#include "lifetime.cuh"

namespace cg = cooperative_groups;

namespace tio {

// error flag bits (scalars[2])
enum : unsigned long long {
    LF_BAD_DURATION = 1, LF_BAD_SIZE = 2, LF_BAD_PTR = 4, LF_ACCESS_RANGE = 8,
    LF_NOT_INCREASING = 16, LF_BAD_KIND = 32
};

// largest i in [0, T) with ptr[i] <= e  (ptr strictly increasing for valid traces)
__device__ __forceinline__ int64_t owner_of(const int64_t *ptr, int64_t T, int64_t e) {
    int64_t lo = 0, hi = T;  // answer in [lo, hi)
    while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if (ptr[mid] <= e) lo = mid; else hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(LIFETIME_THREADS)
lifetime_kernel(LifetimeArgs a) {
    cg::grid_group grid = cg::this_grid();
    __shared__ int64_t sm[40];
    __shared__ int64_t s_off;

    const int64_t N = a.N, T = a.T, E = a.E;
    const int64_t nthreads = (int64_t)gridDim.x * blockDim.x;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t strip = (E + nthreads - 1) / nthreads;
    const int64_t e0 = gtid * strip < E ? gtid * strip : E;
    const int64_t e1 = e0 + strip < E ? e0 + strip : E;
    const int64_t kchunk = (N + gridDim.x - 1) / gridDim.x;
    const int64_t k0 = (int64_t)blockIdx.x * kchunk < N ? (int64_t)blockIdx.x * kchunk : N;
    const int64_t k1 = k0 + kchunk < N ? k0 + kchunk : N;

    // ------------------------------------------------------------ phase 0
    // CSR shape first: every later phase indexes through access_ptr.
    {
        unsigned long long f0 = 0;
        for (int64_t i = gtid; i < T; i += nthreads)
            if (a.ptr[i + 1] <= a.ptr[i]) f0 |= LF_BAD_PTR;
        if (gtid == 0 && (a.ptr[0] != 0 || a.ptr[T] != E)) f0 |= LF_BAD_PTR;
        if (f0) atomicOr(reinterpret_cast<unsigned long long *>(&a.scalars[SC_FLAGS]), f0);
    }
    grid.sync();
    if (__ldcg(reinterpret_cast<const long long *>(&a.scalars[SC_FLAGS])) != 0) return;

    // ------------------------------------------------------------ phase A
    unsigned long long flags = 0;
    int64_t glob = 0;
    int64_t my_periods = 0;
    // tensor-level checks
    for (int64_t i = gtid; i < T; i += nthreads) {
        if (a.size[i] <= 0) flags |= LF_BAD_SIZE;
        int8_t kd = a.kind[i];
        if (kd != 0 && kd != 1) flags |= LF_BAD_KIND;
        if (kd == 1) glob += a.size[i];
        if (i + 1 < T && !(a.tid[i] < a.tid[i + 1])) a.scalars[SC_IDS_UNSORTED] = 1;
    }
    if (e0 < e1) {
        int64_t own = owner_of(a.ptr, T, e0);
        int64_t beg = a.ptr[own], nxt = a.ptr[own + 1];
        int64_t size = a.size[own];
        int8_t kd = a.kind[own];
        for (int64_t e = e0; e < e1; ++e) {
            while (e >= nxt) {
                ++own; beg = nxt; nxt = a.ptr[own + 1];
                size = a.size[own]; kd = a.kind[own];
            }
            const int64_t k = a.acc[e];
            if (k < 0 || k >= N) { flags |= LF_ACCESS_RANGE; continue; }
            atomic_add_i64(&a.active[k], size);
            const bool last = (e == nxt - 1);
            if (!last) {
                const int64_t k2 = a.acc[e + 1];
                if (k2 <= k) flags |= LF_NOT_INCREASING;
                else if (k2 - k > 1) ++my_periods;
            } else if (kd == 1) {
                const int64_t first = a.acc[beg];
                if ((N - 1 - k) + first > 0) ++my_periods;
            }
            if (kd == 0) {
                if (e == beg) atomic_add_i64(&a.diff[k], size);
                if (last) atomic_add_i64(&a.diff[k + 1], -size);
            }
        }
    }
    // kernel chunk: duration sum + validation
    int64_t dsum = 0;
    for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
        int64_t d = a.dur[k];
        if (d <= 0) flags |= LF_BAD_DURATION;
        dsum += d;
    }
    {
        int64_t tot;
        block_exclusive_sum<int64_t>(my_periods, sm, &tot);
        if (threadIdx.x == 0) a.blk_periods[blockIdx.x] = tot;
        int64_t dtot = block_sum<int64_t>(dsum, sm);
        if (threadIdx.x == 0) a.blk_dur[blockIdx.x] = dtot;
        int64_t gtot = block_sum<int64_t>(glob, sm);
        if (threadIdx.x == 0 && gtot) atomic_add_i64(&a.scalars[SC_GLOBAL_BYTES], gtot);
    }
    if (flags) atomicOr(reinterpret_cast<unsigned long long *>(&a.scalars[SC_FLAGS]), flags);
    grid.sync();

    // ------------------------------------------------------------ phase B
    // block offsets (redundant per block; gridDim <= 1024)
    {
        int64_t v = 0, w = 0;
        for (int j = threadIdx.x; j < (int)blockIdx.x; j += blockDim.x) {
            v += __ldcg(reinterpret_cast<const long long *>(&a.blk_periods[j]));
            w += __ldcg(reinterpret_cast<const long long *>(&a.blk_dur[j]));
        }
        int64_t pv = block_sum<int64_t>(v, sm);
        int64_t pw = block_sum<int64_t>(w, sm);
        if (threadIdx.x == 0) { s_off = pv; sm[36] = pw; }
        __syncthreads();
    }
    const int64_t period_base = s_off;
    const int64_t dur_base = sm[36];
    __syncthreads();
    const bool valid = __ldcg(reinterpret_cast<const long long *>(&a.scalars[SC_FLAGS])) == 0;
    {
        int64_t tot;
        int64_t my_off = block_exclusive_sum<int64_t>(my_periods, sm, &tot) + period_base;
        if (valid && e0 < e1) {
            int64_t own = owner_of(a.ptr, T, e0);
            int64_t beg = a.ptr[own], nxt = a.ptr[own + 1];
            int8_t kd = a.kind[own];
            int64_t out = my_off;
            for (int64_t e = e0; e < e1; ++e) {
                while (e >= nxt) { ++own; beg = nxt; nxt = a.ptr[own + 1]; kd = a.kind[own]; }
                if (e == beg) a.tensor_pptr[own] = out;
                const int64_t k = a.acc[e];
                if (e != nxt - 1) {
                    const int64_t k2 = a.acc[e + 1];
                    if (k2 - k > 1) {
                        a.p_tensor[out] = own; a.p_start[out] = (int32_t)(k + 1);
                        a.p_end[out] = (int32_t)(k2 - 1); a.p_wraps[out] = 0; ++out;
                    }
                } else if (kd == 1) {
                    const int64_t first = a.acc[beg];
                    if ((N - 1 - k) + first > 0) {
                        a.p_tensor[out] = own; a.p_start[out] = (int32_t)((k + 1) % N);
                        a.p_end[out] = (int32_t)(((first - 1) % N + N) % N);
                        a.p_wraps[out] = 1; ++out;
                    }
                }
            }
        }
        if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
            int64_t total = period_base + tot;
            a.tensor_pptr[T] = total;
            a.scalars[SC_NUM_PERIODS] = total;
        }
    }
    // kernel start times for this block's chunk
    {
        int64_t run = dur_base;
        for (int64_t base = k0; base < k1; base += blockDim.x) {
            int64_t k = base + threadIdx.x;
            int64_t d = k < k1 ? a.dur[k] : 0;
            int64_t tot;
            int64_t ex = block_exclusive_sum<int64_t>(d, sm, &tot);
            if (k < k1) a.starts[k] = run + ex;
            run += tot;
        }
        if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) a.starts[N] = run;
    }
    // diff block sums (atomics of phase A are complete after grid.sync)
    {
        int64_t v = 0;
        for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x)
            v += __ldcg(reinterpret_cast<const long long *>(&a.diff[k]));
        int64_t tot = block_sum<int64_t>(v, sm);
        if (threadIdx.x == 0) a.blk_diff[blockIdx.x] = tot;
    }
    grid.sync();

    // ------------------------------------------------------------ phase C
    {
        int64_t v = 0;
        for (int j = threadIdx.x; j < (int)blockIdx.x; j += blockDim.x)
            v += __ldcg(reinterpret_cast<const long long *>(&a.blk_diff[j]));
        int64_t pv = block_sum<int64_t>(v, sm);
        int64_t run = pv + __ldcg(reinterpret_cast<const long long *>(&a.scalars[SC_GLOBAL_BYTES]));
        for (int64_t base = k0; base < k1; base += blockDim.x) {
            int64_t k = base + threadIdx.x;
            int64_t d = k < k1 ? __ldcg(reinterpret_cast<const long long *>(&a.diff[k])) : 0;
            int64_t tot;
            int64_t ex = block_exclusive_sum<int64_t>(d, sm, &tot);
            if (k < k1) a.timeline[k] = run + ex + d;
            run += tot;
        }
    }
}

int lifetime_grid(int *blocks) {
    static int cached = 0;
    if (!cached) {
        int dev = 0, sms = 0, per_sm = 0;
        TIO_CUDA(cudaGetDevice(&dev));
        TIO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        TIO_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lifetime_kernel,
                                                               LIFETIME_THREADS, 0));
        if (per_sm < 1) return fail(TIO_ERR_CUDA, "lifetime kernel cannot be resident");
        cached = sms * (per_sm < 4 ? per_sm : 4);
        if (cached > 1024) cached = 1024;
    }
    *blocks = cached;
    return TIO_OK;
}

int launch_lifetime(const LifetimeArgs &args, int blocks, cudaStream_t stream) {
    void *params[] = {const_cast<LifetimeArgs *>(&args)};
    TIO_CUDA(cudaLaunchCooperativeKernel((const void *)lifetime_kernel, dim3(blocks),
                                         dim3(LIFETIME_THREADS), params, 0, stream));
    count_launch();
    return TIO_OK;
}

}  // namespace tio
