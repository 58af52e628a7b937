// lifetime.cu — the lifetime stage on sm_100a.
//
// One cooperative (persistent) kernel, three phases separated by two grid
// barriers, replacing reference analysis.py:58-117 and trace.py:97-107:
//
//   phase A  event tiles (TILE_E consecutive access events of the
//            tensor-major CSR): the tile's accesses, CSR offsets and tensor
//            sizes/kinds are staged in shared memory with coalesced loads;
//            each thread walks a contiguous run of events and
//              active[k] += size                (per_kernel_active_bytes, :111-117)
//              diff[first] += size, diff[last+1] -= size for intermediates
//                                               (compute_memory_timeline, :97-108)
//              counts inactive periods: gaps b-a>1, and the wrap of a global
//              when (n-1-last)+first > 0        (compute_inactive_periods, :58-83)
//              and validates the CSR invariants the kernels rely on;
//            tensor chunks: sizes/kinds/ids checks, global bytes;
//            kernel chunks: duration sums (start-time scan).
//   phase B  period records written at their scanned offsets in reference
//            order (tensor order, gaps ascending, wrap last) with per-tensor
//            period offsets; kernel start times; per-chunk diff sums.
//   phase C  timeline = global bytes + inclusive scan of diff (diff is
//            re-zeroed behind the scan for the next call).
//
// Invalid input never faults (every index is range-checked); it raises a flag
// the host turns into TIO_ERR_INVALID.
// Roofline: HBM-bound integer work, algorithmic bytes per trace
//   B_L = 8E + 16T + 8N + 24P + 24N; DESIGN.md §4.
#include "common.cuh"
#include "block_scan.cuh"
#include "lifetime.cuh"
#include "warp_search.cuh"

namespace cg = cooperative_groups;

namespace tio {

enum : unsigned long long {
    LF_BAD_DURATION = 1, LF_BAD_SIZE = 2, LF_BAD_PTR = 4, LF_ACCESS_RANGE = 8,
    LF_NOT_INCREASING = 16, LF_BAD_KIND = 32
};

constexpr int EV_PER_THREAD = 8;
constexpr int TILE_E = LIFETIME_THREADS * EV_PER_THREAD;    // events per tile

// largest i in [0, T) with ptr[i] <= e (ptr non-decreasing for valid traces)
__device__ __forceinline__ int64_t owner_global(const int64_t *ptr, int64_t T, int64_t e) {
    int64_t lo = 0, hi = T;
    while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if (ptr[mid] <= e) lo = mid; else hi = mid;
    }
    return lo;
}

// A staged tile: events [e0, e1), tensors [o0, o0 + no) with their CSR
// offsets ptr[o0 .. o0 + no], sizes and kinds; accesses acc[e0 .. e1] (+1
// for the next-access look-ahead).  Reads outside the staged ranges fall
// back to global memory (only reachable with invalid input).
struct Tile {
    int64_t e0, e1, o0, no;
    int64_t *ptr;      // [TILE_E + 2]
    int64_t *size;     // [TILE_E + 1]
    int8_t *kind;      // [TILE_E + 1]
    int32_t *acc;      // [TILE_E + 1]
};

struct TileSmem {
    int64_t ptr[TILE_E + 2];
    int64_t size[TILE_E + 1];
    int32_t acc[TILE_E + 1];
    int8_t kind[TILE_E + 1];
    int64_t o[2];
};

__device__ void stage_tile(const LifetimeArgs &a, int64_t tile, TileSmem &sm, Tile &t) {
    const int64_t E = a.E, T = a.T;
    const int64_t e0 = tile * TILE_E, e1 = (e0 + TILE_E < E) ? e0 + TILE_E : E;
    const int warp = threadIdx.x >> 5;
    // owners of the first and last event: 32-ary warp searches (largest i with ptr[i] <= e)
    if (warp < 2) {
        const int64_t e = warp == 0 ? e0 : e1 - 1;
        int64_t o = warp_lower_bound(0, T, [&](int64_t j) { return __ldg(a.ptr + j) > e; }) - 1;
        if (o < 0) o = 0;
        if ((threadIdx.x & 31) == 0) sm.o[warp] = o;
    }
    __syncthreads();
    int64_t o0 = sm.o[0], o1 = sm.o[1];
    if (o1 < o0) o1 = o0;
    int64_t no = o1 - o0 + 1;
    if (no > TILE_E + 1) no = TILE_E + 1;
    for (int64_t i = threadIdx.x; i <= no; i += blockDim.x) sm.ptr[i] = (o0 + i <= T) ? a.ptr[o0 + i] : E;
    for (int64_t i = threadIdx.x; i < no; i += blockDim.x) {
        sm.size[i] = a.size[o0 + i];
        sm.kind[i] = a.kind[o0 + i];
    }
    for (int64_t i = threadIdx.x; i <= e1 - e0; i += blockDim.x)
        sm.acc[i] = (e0 + i < E) ? a.acc[e0 + i] : 0;
    __syncthreads();
    t.e0 = e0; t.e1 = e1; t.o0 = o0; t.no = no;
    t.ptr = sm.ptr; t.size = sm.size; t.kind = sm.kind; t.acc = sm.acc;
}

// staged accessors with global fallback
__device__ __forceinline__ int64_t t_ptr(const LifetimeArgs &a, const Tile &t, int64_t i) {
    return (i >= t.o0 && i <= t.o0 + t.no) ? t.ptr[i - t.o0] : (i <= a.T ? a.ptr[i] : a.E);
}
__device__ __forceinline__ int64_t t_size(const LifetimeArgs &a, const Tile &t, int64_t i) {
    return (i >= t.o0 && i < t.o0 + t.no) ? t.size[i - t.o0] : a.size[i];
}
__device__ __forceinline__ int8_t t_kind(const LifetimeArgs &a, const Tile &t, int64_t i) {
    return (i >= t.o0 && i < t.o0 + t.no) ? t.kind[i - t.o0] : a.kind[i];
}
__device__ __forceinline__ int64_t t_acc(const LifetimeArgs &a, const Tile &t, int64_t e) {
    return (e >= t.e0 && e <= t.e1) ? t.acc[e - t.e0] : (e < a.E ? a.acc[e] : 0);
}

// owner of event e inside the staged tensor range: largest i with ptr[i] <= e
__device__ __forceinline__ int64_t t_owner(const LifetimeArgs &a, const Tile &t, int64_t e) {
    int64_t lo = 0, hi = t.no;           // staged ptr[0 .. no]
    if (t.no <= 0 || t.ptr[0] > e) return owner_global(a.ptr, a.T, e);
    while (hi - lo > 1) {
        int64_t mid = (lo + hi) >> 1;
        if (t.ptr[mid] <= e) lo = mid; else hi = mid;
    }
    int64_t own = t.o0 + lo;
    if (own >= a.T) own = a.T - 1;
    return own;
}

__global__ void __launch_bounds__(LIFETIME_THREADS)
lifetime_kernel(LifetimeArgs a) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) unsigned char smraw[];
    TileSmem &tsm = *reinterpret_cast<TileSmem *>(smraw);
    __shared__ int64_t sm[40];
    __shared__ int64_t s_pre[64];            // prefixes of this block's tiles / chunks

    const int64_t N = a.N, T = a.T, E = a.E;
    const int G = gridDim.x, b = blockIdx.x;
    const int64_t NT = (E + TILE_E - 1) / TILE_E;                 // event tiles
    const int64_t gtid = (int64_t)b * blockDim.x + threadIdx.x;
    const int64_t nthreads = (int64_t)G * blockDim.x;
    const int64_t kchunk = (N + G - 1) / G;                       // kernel chunk per block
    const int64_t k0 = (int64_t)b * kchunk < N ? (int64_t)b * kchunk : N;
    const int64_t k1 = k0 + kchunk < N ? k0 + kchunk : N;
    unsigned long long flags = 0;

    // ------------------------------------------------------------ phase A
    // tensor-level checks and global bytes
    int64_t glob = 0;
    for (int64_t i = gtid; i < T; i += nthreads) {
        const int64_t p0 = a.ptr[i], p1 = a.ptr[i + 1];
        if (p1 <= p0) flags |= LF_BAD_PTR;
        if (a.size[i] <= 0) flags |= LF_BAD_SIZE;
        const int8_t kd = a.kind[i];
        if (kd != 0 && kd != 1) flags |= LF_BAD_KIND;
        if (kd == 1) glob += a.size[i];
        if (i + 1 < T && !(a.tid[i] < a.tid[i + 1])) a.scalars[SC_IDS_UNSORTED] = 1;
    }
    if (gtid == 0 && (a.ptr[0] != 0 || a.ptr[T] != E)) flags |= LF_BAD_PTR;
    // event tiles: atomics and period counts
    const bool single_tile = NT > b && NT - b <= G;    // this block owns exactly one tile
    Tile kept{};
    for (int64_t tile = b; tile < NT; tile += G) {
        Tile t;
        stage_tile(a, tile, tsm, t);
        kept = t;
        const int64_t r0 = t.e0 + (int64_t)threadIdx.x * EV_PER_THREAD;
        const int64_t r1 = r0 + EV_PER_THREAD < t.e1 ? r0 + EV_PER_THREAD : t.e1;
        int64_t cnt = 0;
        if (r0 < r1) {
            int64_t own = t_owner(a, t, r0);
            int64_t beg = t_ptr(a, t, own), nxt = t_ptr(a, t, own + 1);
            for (int64_t e = r0; e < r1; ++e) {
                while (e >= nxt && own + 1 < T) { ++own; beg = nxt; nxt = t_ptr(a, t, own + 1); }
                const int64_t k = t_acc(a, t, e);
                if (k < 0 || k >= N) { flags |= LF_ACCESS_RANGE; continue; }
                const int64_t size = t_size(a, t, own);
                const int8_t kd = t_kind(a, t, own);
                atomic_add_i64(&a.active[k], size);
                const bool last = (e == nxt - 1);
                if (!last) {
                    const int64_t k2 = t_acc(a, t, e + 1);
                    if (k2 <= k) flags |= LF_NOT_INCREASING;
                    else if (k2 - k > 1) ++cnt;
                } else if (kd == 1) {
                    const int64_t first = t_acc(a, t, beg);
                    if ((N - 1 - k) + first > 0) ++cnt;
                }
                if (kd == 0) {
                    if (e == beg) atomic_add_i64(&a.diff[k], size);
                    if (last) atomic_add_i64(&a.diff[k + 1], -size);
                }
            }
        }
        const int64_t tot = block_sum<int64_t>(cnt, sm);
        if (threadIdx.x == 0) a.blk_periods[tile] = tot;
    }
    // kernel chunk: duration sum + validation
    {
        int64_t dsum = 0;
        for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) {
            const int64_t d = a.dur[k];
            if (d <= 0) flags |= LF_BAD_DURATION;
            dsum += d;
        }
        const int64_t dtot = block_sum<int64_t>(dsum, sm);
        if (threadIdx.x == 0) a.blk_dur[b] = dtot;
        const int64_t gtot = block_sum<int64_t>(glob, sm);
        if (threadIdx.x == 0 && gtot) atomic_add_i64(&a.scalars[SC_GLOBAL_BYTES], gtot);
    }
    if (flags) atomicOr(reinterpret_cast<unsigned long long *>(&a.scalars[SC_FLAGS]), flags);
    grid.sync();

    // ------------------------------------------------------------ phase B
    // exclusive prefixes of the tile period counts for this block's tiles
    // (scanned redundantly per block; tiles b, b + G, ... take slots 0, 1, ...)
    auto prefix_for_mine = [&](const int64_t *vals, int64_t n, int64_t *out_slots, int64_t *grand) {
        int64_t run = 0;
        for (int64_t base = 0; base < n; base += blockDim.x) {
            const int64_t j = base + threadIdx.x;
            const int64_t v = j < n ? __ldcg(reinterpret_cast<const long long *>(vals + j)) : 0;
            int64_t tot;
            const int64_t ex = block_exclusive_sum<int64_t>(v, sm, &tot);
            if (j < n && j % G == b && j / G < 64) out_slots[j / G] = run + ex;
            run += tot;
        }
        if (grand) *grand = run;
    };
    const bool valid = __ldcg(reinterpret_cast<const long long *>(&a.scalars[SC_FLAGS])) == 0;
    int64_t total_periods = 0;
    prefix_for_mine(a.blk_periods, NT, s_pre, &total_periods);
    __syncthreads();
    int64_t slot = 0;
    for (int64_t tile = b; tile < NT; tile += G, ++slot) {
        // more than 64 tiles per block: recompute the prefix directly
        int64_t base_off;
        if (slot < 64) base_off = s_pre[slot];
        else {
            int64_t v = 0;
            for (int64_t j = threadIdx.x; j < tile; j += blockDim.x)
                v += __ldcg(reinterpret_cast<const long long *>(a.blk_periods + j));
            base_off = block_sum<int64_t>(v, sm);
        }
        Tile t;
        if (single_tile) t = kept;              // still staged in shared memory
        else stage_tile(a, tile, tsm, t);
        const int64_t r0 = t.e0 + (int64_t)threadIdx.x * EV_PER_THREAD;
        const int64_t r1 = r0 + EV_PER_THREAD < t.e1 ? r0 + EV_PER_THREAD : t.e1;
        // count again (cheap, staged) to place this thread's periods
        int64_t cnt = 0;
        int64_t own = 0, beg = 0, nxt = 0;
        if (valid && r0 < r1) {
            own = t_owner(a, t, r0);
            beg = t_ptr(a, t, own); nxt = t_ptr(a, t, own + 1);
            int64_t o = own, bg = beg, nx = nxt;
            for (int64_t e = r0; e < r1; ++e) {
                while (e >= nx && o + 1 < T) { ++o; bg = nx; nx = t_ptr(a, t, o + 1); }
                const int64_t k = t_acc(a, t, e);
                if (e != nx - 1) { if (t_acc(a, t, e + 1) - k > 1) ++cnt; }
                else if (t_kind(a, t, o) == 1 && (N - 1 - k) + t_acc(a, t, bg) > 0) ++cnt;
            }
        }
        int64_t tot;
        int64_t out = block_exclusive_sum<int64_t>(cnt, sm, &tot) + base_off;
        if (valid && r0 < r1) {
            for (int64_t e = r0; e < r1; ++e) {
                while (e >= nxt && own + 1 < T) { ++own; beg = nxt; nxt = t_ptr(a, t, own + 1); }
                if (e == beg) a.tensor_pptr[own] = out;
                const int64_t k = t_acc(a, t, e);
                if (e != nxt - 1) {
                    const int64_t k2 = t_acc(a, t, e + 1);
                    if (k2 - k > 1) {
                        a.p_tensor[out] = own; a.p_start[out] = (int32_t)(k + 1);
                        a.p_end[out] = (int32_t)(k2 - 1); a.p_wraps[out] = 0; ++out;
                    }
                } else if (t_kind(a, t, own) == 1) {
                    const int64_t first = t_acc(a, t, beg);
                    if ((N - 1 - k) + first > 0) {
                        a.p_tensor[out] = own; a.p_start[out] = (int32_t)((k + 1) % N);
                        a.p_end[out] = (int32_t)(((first - 1) % N + N) % N);
                        a.p_wraps[out] = 1; ++out;
                    }
                }
            }
        }
    }
    if (b == 0 && threadIdx.x == 0) {
        a.tensor_pptr[T] = total_periods;
        a.scalars[SC_NUM_PERIODS] = total_periods;
    }
    // kernel start times for this block's chunk
    {
        int64_t v = 0;
        for (int j = threadIdx.x; j < b; j += blockDim.x)
            v += __ldcg(reinterpret_cast<const long long *>(&a.blk_dur[j]));
        int64_t run = block_sum<int64_t>(v, sm);
        for (int64_t base = k0; base < k1; base += blockDim.x) {
            const int64_t k = base + threadIdx.x;
            const int64_t d = k < k1 ? a.dur[k] : 0;
            int64_t tot;
            const int64_t ex = block_exclusive_sum<int64_t>(d, sm, &tot);
            if (k < k1) a.starts[k] = run + ex;
            run += tot;
        }
        if (b == G - 1 && threadIdx.x == 0) a.starts[N] = run;
    }
    // diff chunk sums (the atomics of phase A are complete)
    {
        int64_t v = 0;
        for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x)
            v += __ldcg(reinterpret_cast<const long long *>(&a.diff[k]));
        const int64_t tot = block_sum<int64_t>(v, sm);
        if (threadIdx.x == 0) a.blk_diff[b] = tot;
    }
    grid.sync();

    // ------------------------------------------------------------ phase C
    {
        int64_t v = 0;
        for (int j = threadIdx.x; j < b; j += blockDim.x)
            v += __ldcg(reinterpret_cast<const long long *>(&a.blk_diff[j]));
        const int64_t pv = block_sum<int64_t>(v, sm);
        int64_t run = pv + __ldcg(reinterpret_cast<const long long *>(&a.scalars[SC_GLOBAL_BYTES]));
        for (int64_t base = k0; base < k1; base += blockDim.x) {
            const int64_t k = base + threadIdx.x;
            const int64_t d = k < k1 ? __ldcg(reinterpret_cast<const long long *>(&a.diff[k])) : 0;
            int64_t tot;
            const int64_t ex = block_exclusive_sum<int64_t>(d, sm, &tot);
            if (k < k1) {
                a.timeline[k] = run + ex + d;
                a.diff[k] = 0;                        // ready for the next call
            }
            run += tot;
        }
        if (b == G - 1 && threadIdx.x == 0) a.diff[N] = 0;
    }
}

int lifetime_grid(int *blocks) {
    static int cached = 0;
    if (!cached) {
        int dev = 0, sms = 0, per_sm = 0;
        TIO_CUDA(cudaGetDevice(&dev));
        TIO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        TIO_CUDA(cudaFuncSetAttribute(lifetime_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)sizeof(TileSmem)));
        TIO_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, lifetime_kernel, LIFETIME_THREADS,
                                                               sizeof(TileSmem)));
        if (per_sm < 1) return fail(TIO_ERR_CUDA, "lifetime kernel cannot be resident");
        cached = sms * (per_sm < 4 ? per_sm : 4);
        if (cached > 1024) cached = 1024;
    }
    *blocks = cached;
    return TIO_OK;
}

int64_t lifetime_tiles(int64_t E) { return (E + TILE_E - 1) / TILE_E; }

int launch_lifetime(const LifetimeArgs &args, int blocks, cudaStream_t stream) {
    void *params[] = {const_cast<LifetimeArgs *>(&args)};
    TIO_CUDA(cudaLaunchCooperativeKernel((const void *)lifetime_kernel, dim3(blocks),
                                         dim3(LIFETIME_THREADS), params, sizeof(TileSmem), stream));
    count_launch();
    return TIO_OK;
}

}  // namespace tio
