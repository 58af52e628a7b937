// lifetime.cu — the lifetime stage on sm_100a (reference analysis.py:58-117,
// trace.py:97-107) as three streaming kernels, each a single pass over its
// input with decoupled look-back scans between tiles (no grid barrier, no
// second read of the events):
//
//   k_tile_owners  owner tensor of every event-tile boundary (32-ary warp
//                  searches over the CSR offsets).
//   k_events       one tile of LT_EPT consecutive events per thread (LT_TILE
//                  per block, tiles claimed in order from an atomic counter):
//                    active[k] += size                (per_kernel_active_bytes, :111-117)
//                    diff[first] += size, diff[last+1] -= size for intermediates
//                                                     (compute_memory_timeline, :97-108)
//                    inactive periods: gaps b-a>1, and the wrap of a global
//                    when (n-1-last)+first > 0, written at their scanned
//                    offsets in reference order (compute_inactive_periods, :58-83)
//                    with the per-tensor period offsets;
//                  plus a slice of the tensor table: CSR / size / kind / id
//                  order checks and the bytes of the globals.
//   k_kernels      per kernel tile: start times = exclusive scan of the
//                  durations, timeline = global bytes + inclusive scan of diff
//                  (diff re-zeroed behind the scan for the next call).
//
// Invalid input never faults (every index is range-checked); it raises a flag
// the host turns into TIO_ERR_INVALID.
// Roofline: HBM-bound integer work, algorithmic bytes per trace
//   B_L = 8E + 16T + 8N + 24P + 24N; DESIGN.md §4.
#include "common.cuh"
#include "block_scan.cuh"
#include "lifetime.cuh"
#include "warp_search.cuh"

namespace tio {

enum : unsigned long long {
    LF_BAD_DURATION = 1, LF_BAD_SIZE = 2, LF_BAD_PTR = 4, LF_ACCESS_RANGE = 8,
    LF_NOT_INCREASING = 16, LF_BAD_KIND = 32
};

constexpr int LT_EPT = 8;                           // events per thread
constexpr int LT_TILE = LIFETIME_THREADS * LT_EPT;  // events per tile
constexpr int LT_MAXO = LT_TILE + 2;                // staged tensors per tile
#ifndef KT_THREADS
#define KT_THREADS 256
#endif
#ifndef KT_EPT_
#define KT_EPT_ 8
#endif
#ifndef KT_MINB
#define KT_MINB (1024 / KT_THREADS)
#endif
constexpr int KT_EPT = KT_EPT_;                     // kernels per thread
constexpr int KT_TILE = KT_THREADS * KT_EPT;

__host__ __device__ int64_t lifetime_event_tiles(int64_t E) { return (E + LT_TILE - 1) / LT_TILE; }
__host__ __device__ int64_t lifetime_kernel_tiles(int64_t N) { return (N + KT_TILE - 1) / KT_TILE; }

// Tile prefixes without a look-back chain: every tile publishes its
// aggregate {value, flag} and adds it into its group of LB_GROUP tiles
// ({sum, count}); a tile's exclusive prefix is the sum of the complete groups
// before its own plus the aggregates of the earlier tiles of its group, all
// loaded in parallel by one warp.  Tiles are claimed in order from an atomic
// ticket, so every earlier tile is resident or finished and publishes without
// waiting on anything: the wait is for the slowest predecessor's publish, not
// for a chain of inclusive prefixes (a decoupled look-back's inclusive
// frontier advances ~64 tiles per L2 round trip — at C3's 4,851 event tiles
// that chain was the k_events time).
constexpr int LB_GROUP = 32;
__host__ __device__ __forceinline__ int64_t lb_groups(int64_t ntiles) { return (ntiles + LB_GROUP - 1) / LB_GROUP; }

// workspace layout (int64 words): [0,2) tile counters | owners [NTe+1],
// padded to an even length | event tile status [2 NTe] | dur / diff tile
// status [2 NTk] each | event groups [2 NGe] | dur / diff groups [2 NGk]
// each (16-byte words, 16-byte aligned; everything after the owners is
// zeroed by k_tile_owners)
__host__ __device__ __forceinline__ int64_t owners_len(int64_t nte) { return (nte + 3) & ~(int64_t)1; }
int64_t lifetime_workspace_elems(int64_t N, int64_t E) {
    const int64_t nte = lifetime_event_tiles(E), ntk = lifetime_kernel_tiles(N);
    return 2 + owners_len(nte) + 2 * nte + 4 * ntk + 2 * lb_groups(nte) + 4 * lb_groups(ntk) + 8;
}
struct LtWork {
    int64_t *owner;          // [NTe + 1]
    int64_t *est, *kst;      // event tile status [2 NTe]; dur / diff tile status [2 NTk] each
    int64_t *egrp, *kgrp;    // event groups [2 NGe]; dur / diff groups [2 NGk] each
    int64_t nzero;           // words from est to the end of the groups
};
__host__ __device__ __forceinline__ LtWork lt_work(int64_t *work, int64_t N, int64_t E) {
    const int64_t nte = lifetime_event_tiles(E), ntk = lifetime_kernel_tiles(N);
    LtWork w;
    w.owner = work + 2;
    w.est = w.owner + owners_len(nte);
    w.kst = w.est + 2 * nte;
    w.egrp = w.kst + 4 * ntk;
    w.kgrp = w.egrp + 2 * lb_groups(nte);
    w.nzero = 2 * nte + 4 * ntk + 2 * lb_groups(nte) + 4 * lb_groups(ntk);
    return w;
}

// ---------------------------------------------------------------- look-back
// Tile status {value, flag} as one 16-byte word: flag 1 = the tile's own
// aggregate, 2 = its inclusive prefix.  Published with a single vector store,
// polled with relaxed gpu-scope vector loads.
__device__ __forceinline__ void status_store(int64_t *st, int64_t tile, int64_t value, int64_t flag) {
    int64_t *p = st + 2 * tile;
    asm volatile("st.relaxed.gpu.global.v2.s64 [%0], {%1, %2};" ::"l"(p), "l"(value), "l"(flag) : "memory");
}

__device__ __forceinline__ void status_load(const int64_t *st, int64_t tile, int64_t *value, int64_t *flag) {
    const int64_t *p = st + 2 * tile;
    long long v, f;
    asm volatile("ld.relaxed.gpu.global.v2.s64 {%0, %1}, [%2];" : "=l"(v), "=l"(f) : "l"(p) : "memory");
    *value = v;
    *flag = f;
}

// Publish a tile's aggregate (lane 0 of the calling warp): the tile status,
// then the group sum and, with release semantics, the group count.
__device__ __forceinline__ void agg_publish(int64_t *st, int64_t *grp, int64_t tile, int64_t agg) {
    if ((threadIdx.x & 31) == 0) {
        status_store(st, tile, agg, 1);
        int64_t *g = grp + 2 * (tile / LB_GROUP);
        if (agg) atomic_add_i64(g, agg);
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(g + 1) : "memory");
    }
}

// Exclusive prefix of tile `tile` (one warp, all lanes; the result in every
// lane) over NCH independent chains (status / group arrays at strides sst /
// sgrp words).  Complete groups first, then the own group's earlier tiles.
template <int NCH>
__device__ void agg_prefix(const int64_t *st, int64_t sst, const int64_t *grp, int64_t sgrp, int64_t tile,
                           int64_t *prefix) {
    const int lane = threadIdx.x & 31;
    const int64_t g = tile / LB_GROUP;
    int64_t acc[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc[c] = 0;
    for (int64_t q = lane; q < g; q += 32) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int64_t *gp = grp + c * sgrp + 2 * q;
            long long n;
            do {
                asm volatile("ld.acquire.gpu.global.s64 %0, [%1];" : "=l"(n) : "l"(gp + 1) : "memory");
            } while (n < LB_GROUP);
            long long v;
            asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(gp) : "memory");
            acc[c] += v;
        }
    }
    const int64_t j = g * LB_GROUP + lane;
    if (j < tile) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            int64_t v, f;
            do { status_load(st + c * sst, j, &v, &f); } while (f == 0);
            acc[c] += v;
        }
    }
#pragma unroll
    for (int c = 0; c < NCH; ++c) prefix[c] = warp_sum<int64_t>(acc[c]);
}

// ---------------------------------------------------------------- owners
// owner[t] = largest i in [0, T) with ptr[i] <= e_t, e_t = min(t * LT_TILE, E - 1)
// Also zeroes the tile counters and the look-back status words for the two
// kernels that follow (work[0, 2) and zero[0, nzero)).
__global__ void k_tile_owners(const int64_t *ptr, int64_t T, int64_t E, int64_t ntiles, int64_t *owner,
                              int64_t *work, int64_t *zero, int64_t nzero) {
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gtid < 2) work[gtid] = 0;
    for (int64_t i = gtid; i < nzero; i += (int64_t)gridDim.x * blockDim.x) zero[i] = 0;
    const int64_t warp = gtid >> 5;
    if (warp > ntiles) return;
    int64_t e = warp * LT_TILE;
    if (e > E - 1) e = E - 1;
    int64_t o = warp_lower_bound(0, T, [&](int64_t j) { return __ldg(ptr + j) > e; }) - 1;
    if (o < 0) o = 0;
    if ((threadIdx.x & 31) == 0) owner[warp] = o;
}

// ---------------------------------------------------------------- events
struct EvSmem {
    alignas(16) int32_t acc[LT_TILE + 4];   // the tile's accesses (+ the next tile's first); first: 16-byte aligned
    int32_t ptr[LT_MAXO + 1];   // staged CSR offsets relative to the tile's first event
    int16_t own[LT_TILE];       // staged owner index of every event of the tile
    union {
        uint64_t sk[LT_MAXO];   // during the walks: size | kind << 63 of the staged tensors
        int16_t rec[LT_TILE];   // afterwards: the event opening each period, tile-local order
    };
    int32_t scan32[40];
    int64_t scan[40];
    int64_t prefix;
    int64_t tile;
};

// exclusive block max-scan of int32 (-1 identity), all threads
__device__ __forceinline__ int32_t block_exclusive_max(int32_t v, int32_t *sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t n = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o && n > inc) inc = n;
    }
    if (lane == 31) sm[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        int32_t w = lane < nw ? sm[lane] : -1;
        int32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t n = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o && n > wi) wi = n;
        }
        const int32_t ex = __shfl_up_sync(0xffffffffu, wi, 1);
        if (lane < nw) sm[lane] = lane == 0 ? -1 : ex;
    }
    __syncthreads();
    int32_t ex = __shfl_up_sync(0xffffffffu, inc, 1);
    if (lane == 0) ex = -1;
    const int32_t r = sm[warp] > ex ? sm[warp] : ex;
    __syncthreads();
    return r;
}

// One event tile.  Staging: the tile's tensors (CSR offsets, sizes, kinds)
// and accesses in shared memory, and an owner map (tensor heads, then a
// block max-scan).  Walks over each thread's LT_EPT consecutive events:
// (1) validation, period count, masks; (2) the atomics; (3) period records
// in shared memory at tile-local offsets.  The tile prefix comes from a
// decoupled look-back; records are then stored coalesced.
__device__ __forceinline__ unsigned long long event_tile(const LifetimeArgs &a, EvSmem &sm, int64_t tile,
                                                         int64_t NTe, int64_t *est, int64_t *egrp,
                                                         const int64_t *owner) {
    const int64_t T = a.T, E = a.E;
    const int32_t N = (int32_t)a.N;
    unsigned long long flags = 0;
    const int64_t e0 = tile * LT_TILE, e1 = (e0 + LT_TILE < E) ? e0 + LT_TILE : E;
    const int32_t ne = (int32_t)(e1 - e0);
    const int64_t o0 = __ldcg(reinterpret_cast<const long long *>(owner + tile));
    int64_t o1 = __ldcg(reinterpret_cast<const long long *>(owner + tile + 1));
    if (o1 < o0) o1 = o0;
    const int64_t no = o1 - o0 + 1;
    // more staged tensors than events can only come from empty tensors (an
    // invalid trace, flagged by the tensor-table checks): skip the tile
    const bool staged = no <= LT_MAXO;
    for (int i = threadIdx.x; i < LT_TILE; i += blockDim.x) sm.own[i] = i == 0 ? 0 : -1;   // o0 starts at or before the tile
    if (staged) {
        for (int64_t i = threadIdx.x; i <= no; i += blockDim.x) {
            const int64_t p = (o0 + i <= T) ? __ldg(a.ptr + o0 + i) : E;
            sm.ptr[i] = (int32_t)(p - e0 < INT32_MIN ? INT32_MIN : (p - e0 > INT32_MAX ? INT32_MAX : p - e0));
        }
        for (int64_t i = threadIdx.x; i < no; i += blockDim.x) {
            sm.sk[i] = (uint64_t)__ldg(a.size + o0 + i) | ((uint64_t)(__ldg(a.kind + o0 + i) == 1) << 63);
        }
    }
    if (((uintptr_t)a.acc & 15) == 0 && ne == LT_TILE) {
        const int4 *q = reinterpret_cast<const int4 *>(a.acc + e0);
        for (int i = threadIdx.x; i < LT_TILE / 4; i += blockDim.x)
            reinterpret_cast<int4 *>(sm.acc)[i] = __ldg(q + i);
    } else {
        for (int i = threadIdx.x; i < ne; i += blockDim.x) sm.acc[i] = __ldg(a.acc + e0 + i);
    }
    if (threadIdx.x == 0) sm.acc[ne] = e1 < E ? __ldg(a.acc + e1) : 0;
    __syncthreads();
    // owner map: tensor heads inside the tile, then a running max
    if (staged)
        for (int64_t i = threadIdx.x; i < no; i += blockDim.x) {
            const int32_t r = sm.ptr[i];
            if (r >= 0 && r < ne) sm.own[r] = (int16_t)i;
        }
    __syncthreads();
    const int32_t frel = (int32_t)threadIdx.x * LT_EPT;           // tile-relative first event
    const int nv = (!staged || frel >= ne) ? 0 : (ne - frel < LT_EPT ? ne - frel : LT_EPT);
    int32_t own[LT_EPT];
    {
        int32_t run = -1;
#pragma unroll
        for (int j = 0; j < LT_EPT; ++j) {
            const int32_t v = frel + j < LT_TILE ? sm.own[frel + j] : -1;
            run = v > run ? v : run;
            own[j] = run;
        }
        const int32_t ex = block_exclusive_max(run, sm.scan32);
#pragma unroll
        for (int j = 0; j < LT_EPT; ++j) {
            own[j] = own[j] > ex ? own[j] : ex;
            if (frel + j < LT_TILE) sm.own[frel + j] = (int16_t)own[j];   // resolved, for the record pass
        }
    }
    int32_t k[LT_EPT + 1];
#pragma unroll
    for (int j = 0; j <= LT_EPT; ++j) k[j] = frel + j <= ne ? sm.acc[frel + j] : 0;

    // ---- walk 1: validation, period count, masks
    int64_t cnt = 0;
    uint32_t pmask = 0;                      // bit j: event j opens a period
    uint32_t fmask = 0;                      // bit j: event j is its tensor's first access
#pragma unroll
    for (int j = 0; j < LT_EPT; ++j) {
        if (j >= nv) break;
        const int32_t e = frel + j, o = own[j];
        const int32_t beg = sm.ptr[o], nxt = sm.ptr[o + 1];
        const int32_t kk = k[j];
        if (e == beg) fmask |= 1u << j;
        if (e < beg || e >= nxt) { flags |= LF_BAD_PTR; continue; }
        if ((uint32_t)kk >= (uint32_t)N) { flags |= LF_ACCESS_RANGE; continue; }
        if (e != nxt - 1) {
            const int32_t k2 = k[j + 1];
            if (k2 <= kk) flags |= LF_NOT_INCREASING;
            else if (k2 - kk > 1) { pmask |= 1u << j; ++cnt; }
        } else if (sm.sk[o] >> 63) {
            const int32_t fk = beg >= 0 ? sm.acc[beg] : __ldg(a.acc + e0 + beg);
            if ((N - 1 - kk) + fk > 0) { pmask |= 1u << j; ++cnt; }
        }
    }
    // tile-local offsets; the aggregate goes out before the atomics so the
    // successors' look-backs only wait for this counting walk
    int64_t tot;
    const int64_t loc = block_exclusive_sum<int64_t>(cnt, sm.scan, &tot);
    if (threadIdx.x < 32) agg_publish(est, egrp, tile, tot);

    // ---- walk 2: per-kernel active bytes and the timeline difference array
#ifndef LT_NO_REDS          // (timing experiments only: tools/build_variant.sh -DLT_NO_REDS)
    if (!(flags & (LF_ACCESS_RANGE | LF_BAD_PTR))) {
#else
    if (false) {
#endif
#pragma unroll
        for (int j = 0; j < LT_EPT; ++j) {
            if (j >= nv) break;
            const int32_t e = frel + j, o = own[j];
            const int32_t kk = k[j];
            const int64_t sz = (int64_t)(sm.sk[o] & ~(1ull << 63));
            atomic_add_i64(&a.active[kk], sz);                     // per_kernel_active_bytes (:111-117)
            if (!(sm.sk[o] >> 63)) {                               // compute_memory_timeline (:97-108)
                if (e == sm.ptr[o]) atomic_add_i64(&a.diff[kk], sz);
                if (e == sm.ptr[o + 1] - 1) atomic_add_i64(&a.diff[kk + 1], -sz);
            }
        }
    }
    __syncthreads();                         // sizes / kinds no longer needed: records reuse them

    // ---- walk 3: period records in reference order (analysis.py:68-82:
    // tensor order, gaps ascending, wrap last) at tile-local offsets
    if (pmask && flags == 0) {
        int32_t q = (int32_t)loc;
#pragma unroll
        for (int j = 0; j < LT_EPT; ++j)
            if (pmask & (1u << j)) sm.rec[q++] = (int16_t)(frel + j);
    }

    // ---- tile prefix
    if (threadIdx.x < 32) {
        int64_t pre;
        agg_prefix<1>(est, 0, egrp, 0, tile, &pre);
        if (threadIdx.x == 0) sm.prefix = pre;
    }
    __syncthreads();
    const int64_t prefix = sm.prefix;
    if (tile == NTe - 1 && threadIdx.x == 0) {
        a.tensor_pptr[T] = prefix + tot;
        a.scalars[SC_NUM_PERIODS] = prefix + tot;
    }
    const bool ok = __syncthreads_or(flags != 0) == 0;
    if (!ok) return flags;
    // per-tensor period offsets
    if (fmask) {
        int64_t q = prefix + loc;
#pragma unroll
        for (int j = 0; j < LT_EPT; ++j) {
            if (fmask & (1u << j)) a.tensor_pptr[o0 + own[j]] = q;
            if (pmask & (1u << j)) ++q;
        }
    }
    // period records, stored coalesced: the staged event and the staged
    // accesses / owner map give the record back
#ifdef LT_NO_RECORDS
    return flags;
#endif
    for (int64_t i = threadIdx.x; i < tot; i += blockDim.x) {
        const int32_t e = sm.rec[i], o = sm.own[e], kk = sm.acc[e];
        const int64_t g = prefix + i;
        a.p_tensor[g] = o0 + o;
        if (e != sm.ptr[o + 1] - 1) {
            a.p_start[g] = kk + 1; a.p_end[g] = sm.acc[e + 1] - 1; a.p_wraps[g] = 0;
        } else {
            const int32_t beg = sm.ptr[o];
            const int32_t fk = beg >= 0 ? sm.acc[beg] : __ldg(a.acc + e0 + beg);
            a.p_start[g] = (kk + 1) % N; a.p_end[g] = ((fk - 1) % N + N) % N; a.p_wraps[g] = 1;
        }
    }
    return flags;
}

#ifndef LT_MINB
#define LT_MINB 6            // 40 registers: 5 blocks (shared memory bound) per SM; measured 211 vs 226 us at C3
#endif
__global__ void __launch_bounds__(LIFETIME_THREADS, LT_MINB)
k_events(LifetimeArgs a) {
    asm volatile("griddepcontrol.wait;" ::: "memory");      // owners + zeroed status (programmatic launch)
    extern __shared__ __align__(16) unsigned char smraw[];
    EvSmem &sm = *reinterpret_cast<EvSmem *>(smraw);
    const int64_t T = a.T, E = a.E;
    const int64_t NTe = lifetime_event_tiles(E);
    if (threadIdx.x == 0) sm.tile = (int64_t)atomicAdd(reinterpret_cast<unsigned long long *>(a.work), 1ull);
    __syncthreads();
    const int64_t tile = sm.tile;
    unsigned long long flags = 0;
    const LtWork w = lt_work(a.work, a.N, E);
    if (tile < NTe) flags = event_tile(a, sm, tile, NTe, w.est, w.egrp, w.owner);

    // ---- a slice of the tensor table: CSR / size / kind / id order, global bytes
    {
        const int64_t per = (T + gridDim.x - 1) / gridDim.x;
        const int64_t i0 = tile * per, i1 = i0 + per < T ? i0 + per : T;
        int64_t glob = 0;
        for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
            if (__ldg(a.ptr + i + 1) <= __ldg(a.ptr + i)) flags |= LF_BAD_PTR;
            const int64_t sz = __ldg(a.size + i);
            if (sz <= 0) flags |= LF_BAD_SIZE;
            const int8_t kd = __ldg(a.kind + i);
            if (kd != 0 && kd != 1) flags |= LF_BAD_KIND;
            if (kd == 1) glob += sz;
            if (i + 1 < T && !(__ldg(a.tid + i) < __ldg(a.tid + i + 1))) a.scalars[SC_IDS_UNSORTED] = 1;
        }
        if (tile == 0 && threadIdx.x == 0 && (__ldg(a.ptr) != 0 || __ldg(a.ptr + T) != E)) flags |= LF_BAD_PTR;
        const int64_t g = block_sum<int64_t>(glob, sm.scan);
        if (threadIdx.x == 0 && g) atomic_add_i64(&a.scalars[SC_GLOBAL_BYTES], g);
    }
    if (flags) atomicOr(reinterpret_cast<unsigned long long *>(&a.scalars[SC_FLAGS]), flags);
}

// ---------------------------------------------------------------- kernels
__global__ void __launch_bounds__(KT_THREADS, KT_MINB)
k_kernels(LifetimeArgs a) {
    asm volatile("griddepcontrol.wait;" ::: "memory");      // k_events complete (programmatic launch)
    __shared__ int64_t scan[40];
    __shared__ int64_t s_pre[2];
    __shared__ int64_t s_tile;
    const int64_t N = a.N, E = a.E;
    const int64_t NTe = lifetime_event_tiles(E), NTk = lifetime_kernel_tiles(N);
    const LtWork w = lt_work(a.work, N, E);                     // dur chain, then diff chain
    if (threadIdx.x == 0) s_tile = (int64_t)atomicAdd(reinterpret_cast<unsigned long long *>(a.work + 1), 1ull);
    // the globals' bytes (k_events' sum) load early, beside the tile's loads
    const int64_t gbytes = __ldcg(reinterpret_cast<const long long *>(&a.scalars[SC_GLOBAL_BYTES]));
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= NTk) return;
    const int64_t k0 = tile * KT_TILE + (int64_t)threadIdx.x * KT_EPT;
    const bool vec = (((uintptr_t)a.dur | (uintptr_t)a.diff | (uintptr_t)a.starts | (uintptr_t)a.timeline) & 15) == 0;
    int64_t d[KT_EPT], df[KT_EPT];
    if (k0 + KT_EPT <= N && vec) {
        const longlong2 *qd = reinterpret_cast<const longlong2 *>(a.dur + k0);
        const longlong2 *qf = reinterpret_cast<const longlong2 *>(a.diff + k0);
#pragma unroll
        for (int j = 0; j < KT_EPT / 2; ++j) {
            const longlong2 x = __ldg(qd + j), y = __ldcg(qf + j);
            d[2 * j] = x.x; d[2 * j + 1] = x.y; df[2 * j] = y.x; df[2 * j + 1] = y.y;
        }
    } else {
#pragma unroll
        for (int j = 0; j < KT_EPT; ++j) {
            d[j] = k0 + j < N ? __ldg(a.dur + k0 + j) : 0;
            df[j] = k0 + j < N ? __ldcg(reinterpret_cast<const long long *>(a.diff + k0 + j)) : 0;
        }
    }
    unsigned long long flags = 0;
    int64_t sd = 0, sf = 0;
#pragma unroll
    for (int j = 0; j < KT_EPT; ++j) {
        if (k0 + j < N && d[j] <= 0) flags |= LF_BAD_DURATION;
        sd += d[j];
        sf += df[j];
    }
    if (flags) atomicOr(reinterpret_cast<unsigned long long *>(&a.scalars[SC_FLAGS]), flags);
    int64_t agg[2];
    int64_t xd = block_exclusive_sum<int64_t>(sd, scan, &agg[0]);
    int64_t xf = block_exclusive_sum<int64_t>(sf, scan, &agg[1]);
    if (threadIdx.x < 32) {
        agg_publish(w.kst, w.kgrp, tile, agg[0]);
        agg_publish(w.kst + 2 * NTk, w.kgrp + 2 * lb_groups(NTk), tile, agg[1]);
        int64_t pre[2];
        agg_prefix<2>(w.kst, 2 * NTk, w.kgrp, 2 * lb_groups(NTk), tile, pre);
        if (threadIdx.x == 0) { s_pre[0] = pre[0]; s_pre[1] = pre[1]; }
    }
    __syncthreads();
    xd += s_pre[0];
    xf += s_pre[1] + gbytes;
    if (k0 + KT_EPT <= N && vec) {
        longlong2 *ps = reinterpret_cast<longlong2 *>(a.starts + k0);
        longlong2 *pt = reinterpret_cast<longlong2 *>(a.timeline + k0);
        longlong2 *pz = reinterpret_cast<longlong2 *>(a.diff + k0);
#pragma unroll
        for (int j = 0; j < KT_EPT / 2; ++j) {
            const int64_t s0 = xd, s1 = xd + d[2 * j];
            xd = s1 + d[2 * j + 1];
            const int64_t t0 = xf + df[2 * j], t1 = t0 + df[2 * j + 1];
            xf = t1;
            ps[j] = make_longlong2(s0, s1);
            pt[j] = make_longlong2(t0, t1);
            pz[j] = make_longlong2(0, 0);                      // ready for the next call
        }
    } else {
#pragma unroll
        for (int j = 0; j < KT_EPT; ++j)
            if (k0 + j < N) {
                a.starts[k0 + j] = xd; xd += d[j];
                xf += df[j]; a.timeline[k0 + j] = xf;
                a.diff[k0 + j] = 0;
            }
    }
    if (tile == NTk - 1 && threadIdx.x == blockDim.x - 1) {
        a.starts[N] = s_pre[0] + agg[0];
        a.diff[N] = 0;
    }
}

int launch_lifetime(const LifetimeArgs &args, cudaStream_t stream) {
    static bool attr = false;
    if (!attr) {
        TIO_CUDA(cudaFuncSetAttribute(k_events, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(EvSmem)));
        attr = true;
    }
    const int64_t NTe = lifetime_event_tiles(args.E), NTk = lifetime_kernel_tiles(args.N);
    // counters + tile status + group sums: zeroed by k_tile_owners
    const LtWork w = lt_work(args.work, args.N, args.E);
    int64_t *status = w.est;
    const int64_t nstatus = w.nzero;
    if (NTe > 0) {
        const int64_t thr = 32 * (NTe + 1);
        k_tile_owners<<<(unsigned)((thr + 255) / 256), 256, 0, stream>>>(args.ptr, args.T, args.E, NTe, args.work + 2,
                                                                          args.work, status, nstatus);
        count_launch();
    } else {
        TIO_CUDA(cudaMemsetAsync(args.work, 0, sizeof(int64_t) * 2, stream));
        TIO_CUDA(cudaMemsetAsync(status, 0, sizeof(int64_t) * nstatus, stream));
    }
    // the next two kernels launch programmatically (PDL): their blocks become
    // resident while the previous grid drains and wait in griddepcontrol.wait
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.stream = stream;
    cfg.attrs = pdl;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3((unsigned)(NTe > 0 ? NTe : 1));     // >= 1 block: the tensor-table checks
    cfg.blockDim = dim3(LIFETIME_THREADS);
    cfg.dynamicSmemBytes = sizeof(EvSmem);
    TIO_CUDA(cudaLaunchKernelEx(&cfg, k_events, args));
    count_launch();
#ifdef LT_NO_KERNELS
    if (false) {
#else
    if (NTk > 0) {
#endif
        cfg.gridDim = dim3((unsigned)NTk);
        cfg.blockDim = dim3(KT_THREADS);
        cfg.dynamicSmemBytes = 0;
        TIO_CUDA(cudaLaunchKernelEx(&cfg, k_kernels, args));
        count_launch();
    }
    TIO_CUDA(cudaGetLastError());
    return TIO_OK;
}

}  // namespace tio
