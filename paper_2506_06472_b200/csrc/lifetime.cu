// lifetime.cu — the lifetime stage on sm_100a (reference analysis.py:58-117,
// trace.py:97-107) as three streaming kernels, each a single pass over its
// input with chain-free tile prefixes (agg_prefix: no grid barrier, no second
// read of the events):
//
//   k_tile_owners  owner tensor of every event-tile boundary (32-ary warp
//                  searches over the CSR offsets).
//   k_events       one tile of LT_TILE events per block (tile = blockIdx),
//                  walked warp-contiguously (periods and checks; the atomics
//                  go out after the tile's period count is published)
//                  (lane = event) with owners from a tensor-head bitmask:
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

#ifndef TIO_LT_EPT
#define TIO_LT_EPT 8
#endif
constexpr int LT_EPT = TIO_LT_EPT;                         // events per thread
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
// loaded in parallel by one warp.  A block's tile is its blockIdx: blocks of
// a 1-D grid are dispatched in index order (the premise of CUB's single-pass
// scan, which also takes its tile from blockIdx), so every earlier tile is
// resident or finished and publishes without waiting on anything (an atomic
// ticket per block measured 4% slower at C3: one more L2 round trip ahead of
// every tile's loads): the wait is for the slowest predecessor's publish, not
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

// The event chain's group words pack {count, sum} into one 64-bit word
// (count << 40 | sum: a tile has at most LT_TILE periods, so a group's sum
// stays below 2^17): a relaxed RED publishes both, a relaxed load reads both —
// no release on the publishing side, no fence and no second load on the
// reading side.
constexpr int GP_SHIFT = 40;
static_assert((int64_t)LB_GROUP * LT_TILE < (1ll << GP_SHIFT) && LB_GROUP < (1 << (63 - GP_SHIFT)),
              "a group's period count and tile count fit the packed word");
__device__ __forceinline__ void agg_publish_packed(int64_t *st, int64_t *grp, int64_t tile, int64_t agg) {
    if ((threadIdx.x & 31) == 0) {
        status_store(st, tile, agg, 1);
        const unsigned long long w = (1ull << GP_SHIFT) + (unsigned long long)agg;
        asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(grp + 2 * (tile / LB_GROUP)), "l"(w) : "memory");
    }
}
__device__ int64_t agg_prefix_packed(const int64_t *st, const int64_t *grp, int64_t tile) {
    constexpr int U = 4;
    const int lane = threadIdx.x & 31;
    const int64_t g = tile / LB_GROUP;
    const int64_t j = g * LB_GROUP + lane;
    int64_t tv = 0, tf = 1, acc = 0;
    if (j < tile) status_load(st, j, &tv, &tf);
    for (int64_t q0 = lane; q0 < g; q0 += 32 * U) {
        long long n[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            n[u] = (long long)LB_GROUP << GP_SHIFT;
            if (q0 + 32 * u < g)
                asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(n[u]) : "l"(grp + 2 * (q0 + 32 * u)) : "memory");
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            while ((n[u] >> GP_SHIFT) < LB_GROUP)
                asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(n[u]) : "l"(grp + 2 * (q0 + 32 * u)) : "memory");
            if (q0 + 32 * u < g) acc += n[u] & ((1ll << GP_SHIFT) - 1);
        }
    }
    if (j < tile) {
        while (tf == 0) status_load(st, j, &tv, &tf);
        acc += tv;
    }
    return warp_sum<int64_t>(acc);
}

// ---------------------------------------------------------------- owners
// owner[t] = largest i in [0, T) with ptr[i] <= e_t, e_t = min(t * LT_TILE, E - 1)
// Also zeroes the look-back status words for the two kernels that follow
// (zero[0, nzero); work[0, 2) are spare counters).
// It also zeroes the stage's accumulators (active bytes, scalars): one
// launch instead of three memsets ahead of the stage.
__global__ void k_tile_owners(const int64_t *ptr, int64_t T, int64_t E, int64_t ntiles, int64_t *owner,
                              int64_t *work, int64_t *zero, int64_t nzero, int64_t *active, int64_t N,
                              int64_t *scalars) {
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
    if (gtid < 2) work[gtid] = 0;
    if (gtid < SC_COUNT) scalars[gtid] = 0;
    for (int64_t i = gtid; i < nzero; i += nthr) zero[i] = 0;
    if (((uintptr_t)active & 15) == 0) {
        longlong2 *a2 = reinterpret_cast<longlong2 *>(active);
        for (int64_t i = gtid; i < (N >> 1); i += nthr) a2[i] = make_longlong2(0, 0);
        if ((N & 1) && gtid == 0) active[N - 1] = 0;
    } else {
        for (int64_t i = gtid; i < N; i += nthr) active[i] = 0;
    }
    const int64_t warp = gtid >> 5;
    if (warp > ntiles) return;
    int64_t e = warp * LT_TILE;
    if (e > E - 1) e = E - 1;
    int64_t o = warp_lower_bound(0, T, [&](int64_t j) { return __ldg(ptr + j) > e; }) - 1;
    if (o < 0) o = 0;
    if ((threadIdx.x & 31) == 0) owner[warp] = o;
}

// ---------------------------------------------------------------- events
// Warp-contiguous form: warp w of a tile walks events [256 w, 256 w + 256) in
// 8 steps of 32 (lane = event).  A tensor-head bitmask over the tile (one bit
// per event where a staged tensor starts) gives every event its owner with
// one broadcast load and a popcount; a step's periods are a ballot, so the
// tile-local record offsets need one block exchange (warp totals) and the
// records are stored straight to their final positions.
struct EvSmem {
    alignas(16) int32_t acc[LT_TILE + 4];
    int32_t ptr[LT_MAXO + 1];
    uint64_t sk[LT_MAXO];
    uint32_t head[LT_TILE / 32];
    int32_t wcnt[LIFETIME_THREADS / 32];
    int64_t wglob[LIFETIME_THREADS / 32];
    unsigned long long wflags[LIFETIME_THREADS / 32];
    int64_t prefix;
};

__device__ __forceinline__ unsigned long long event_tile(const LifetimeArgs &a, EvSmem &sm, int64_t tile,
                                                          int64_t NTe, int64_t *est, int64_t *egrp,
                                                          const int64_t *owner) {
    constexpr int STEPS = LT_TILE / LIFETIME_THREADS;        // 8 steps of 32 events per warp
    const int64_t T = a.T, E = a.E;
    const int32_t N = (int32_t)a.N;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long flags = 0;
    const int64_t e0 = tile * LT_TILE, e1 = (e0 + LT_TILE < E) ? e0 + LT_TILE : E;
    const int32_t ne = (int32_t)(e1 - e0);
    const int64_t o0 = __ldcg(reinterpret_cast<const long long *>(owner + tile));
    int64_t o1 = __ldcg(reinterpret_cast<const long long *>(owner + tile + 1));
    if (o1 < o0) o1 = o0;
    const int32_t no = (int32_t)(o1 - o0 + 1);
    const bool staged = no <= LT_MAXO;

    // ---- staging
    if (((uintptr_t)a.acc & 15) == 0 && ne == LT_TILE) {
        const int4 *q = reinterpret_cast<const int4 *>(a.acc + e0);
        // asynchronous copies: the thread goes on to issue the CSR-slice and
        // tensor-table loads while the access column lands in shared memory
        for (int i = threadIdx.x; i < LT_TILE / 4; i += LIFETIME_THREADS) {
            const unsigned dst = (unsigned)__cvta_generic_to_shared(reinterpret_cast<int4 *>(sm.acc) + i);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(q + i) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    } else {
        for (int i = threadIdx.x; i < ne; i += LIFETIME_THREADS) sm.acc[i] = __ldg(a.acc + e0 + i);
    }
    // the head mask is zeroed here, with the owner loads and the access-column
    // copies already in flight (the barrier orders it before the atomicOr below)
    for (int i = threadIdx.x; i < LT_TILE / 32; i += LIFETIME_THREADS) sm.head[i] = 0;
    __syncthreads();
    if (threadIdx.x == 0) sm.acc[ne] = e1 < E ? __ldg(a.acc + e1) : 0;
    if (staged) {
#pragma unroll 2                       // two tensors' loads in flight per thread
        for (int32_t i = threadIdx.x; i <= no; i += LIFETIME_THREADS) {
            const int64_t p = (o0 + i <= T) ? __ldg(a.ptr + o0 + i) : E;
            const int64_t r = p - e0;
            sm.ptr[i] = (int32_t)(r < INT32_MIN ? INT32_MIN : (r > INT32_MAX ? INT32_MAX : r));
            if (i < no) {
                sm.sk[i] = (uint64_t)__ldg(a.size + o0 + i) | ((uint64_t)(__ldg(a.kind + o0 + i) == 1) << 63);
                if (i > 0 && r >= 0 && r < LT_TILE) atomicOr(&sm.head[r >> 5], 1u << (r & 31));
            }
        }
    }
    // tensor-table slice (validation, globals' bytes)
    int64_t glob = 0;
    {
#ifdef LT_NO_TABLE
        const int64_t per = 0;
#else
        const int64_t per = (T + NTe - 1) / NTe;
#endif
        const int64_t i0 = tile * per, i1 = i0 + per < T ? i0 + per : T;
#pragma unroll 2                       // two tensors' loads in flight per thread
        for (int64_t i = i0 + threadIdx.x; i < i1; i += LIFETIME_THREADS) {
            if (__ldg(a.ptr + i + 1) <= __ldg(a.ptr + i)) flags |= LF_BAD_PTR;
            const int64_t sz = __ldg(a.size + i);
            if (sz <= 0) flags |= LF_BAD_SIZE;
            const int8_t kd = __ldg(a.kind + i);
            if (kd != 0 && kd != 1) flags |= LF_BAD_KIND;
            if (kd == 1) glob += sz;
            if (i + 1 < T && !(__ldg(a.tid + i) < __ldg(a.tid + i + 1))) a.scalars[SC_IDS_UNSORTED] = 1;
        }
        if (tile == 0 && threadIdx.x == 0 && (__ldg(a.ptr) != 0 || __ldg(a.ptr + T) != E)) flags |= LF_BAD_PTR;
    }
    if (!staged) flags |= LF_BAD_PTR;
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();

    // ---- walk: this warp's events, one per lane per step
    const int32_t wbase = warp * (STEPS * 32);
    // heads before this warp's first word (each lane sums its share, then the warp)
    int32_t hb = 0;
    for (int j = lane; j < (wbase >> 5); j += 32) hb += __popc(sm.head[j]);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) hb += __shfl_xor_sync(0xffffffffu, hb, d);
    const uint32_t le = (lane == 31) ? 0xffffffffu : ((2u << lane) - 1u);   // lanes <= this one
    const uint32_t lt = (1u << lane) - 1u;                                  // lanes < this one
    uint32_t pb[STEPS];                       // period ballot per step
    int32_t wcnt = 0;
    const bool live = staged && flags == 0;
#pragma unroll
    for (int st = 0; st < STEPS; ++st) {
        const int32_t e = wbase + st * 32 + lane;
        const uint32_t hw = sm.head[(wbase >> 5) + st];
        const int32_t o = hb + __popc(hw & le);
        hb += __popc(hw);
        const bool in = live && e < ne && o < no;
        bool per = false;
        if (in) {
            const int32_t beg = sm.ptr[o], nxt = sm.ptr[o + 1];
            const int32_t kk = sm.acc[e];
            const uint64_t sk = sm.sk[o];
            const bool glob_t = sk >> 63;
            if (e < beg || e >= nxt) {
                flags |= LF_BAD_PTR;
            } else if ((uint32_t)kk >= (uint32_t)N) {
                flags |= LF_ACCESS_RANGE;
            } else {
                if (e != nxt - 1) {
                    const int32_t k2 = sm.acc[e + 1];
                    if (k2 <= kk) flags |= LF_NOT_INCREASING;
                    else per = k2 - kk > 1;
                } else if (glob_t) {
                    const int32_t fk = beg >= 0 ? sm.acc[beg] : __ldg(a.acc + e0 + beg);
                    per = (N - 1 - kk) + fk > 0;
                }
            }
        }
        pb[st] = __ballot_sync(0xffffffffu, per);
        wcnt += __popc(pb[st]);
    }

    // ---- one block exchange: warp totals, globals' bytes, flags
    const int64_t wg = warp_sum<int64_t>(glob);
    unsigned long long wf = flags;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) wf |= __shfl_xor_sync(0xffffffffu, wf, d);
    if (lane == 0) { sm.wcnt[warp] = wcnt; sm.wglob[warp] = wg; sm.wflags[warp] = wf; }
    __syncthreads();
    int32_t woff = 0, tot = 0;
    int64_t gsum = 0;
    unsigned long long fall = 0;
#pragma unroll
    for (int w = 0; w < LIFETIME_THREADS / 32; ++w) {
        const int32_t c = sm.wcnt[w];
        if (w < warp) woff += c;
        tot += c;
        gsum += sm.wglob[w];
        fall |= sm.wflags[w];
    }
    // ---- the tile's atomics: per_kernel_active_bytes (:111-117) and the
    // timeline difference array of the intermediates (compute_memory_timeline,
    // :97-108).  They go out after the tile's period count is published
    // (warp 0: publish, atomics, then its predecessors' counts; warps 1-7
    // straight away), overlapping the wait for the predecessors instead of
    // delaying this tile's publish, which its successors wait on (issued
    // inside the walk they cost C3 182 -> 164 us).  Only for a tile whose
    // events all passed the walk's checks (indices in range).
    auto tile_reds = [&]() {
#ifndef LT_NO_REDS
        if (fall) return;
        int32_t h2 = 0;
        for (int j = lane; j < (wbase >> 5); j += 32) h2 += __popc(sm.head[j]);
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) h2 += __shfl_xor_sync(0xffffffffu, h2, d);
#pragma unroll
        for (int st = 0; st < STEPS; ++st) {
            const int32_t e = wbase + st * 32 + lane;
            const uint32_t hw = sm.head[(wbase >> 5) + st];
            const int32_t o = h2 + __popc(hw & le);
            h2 += __popc(hw);
            if (e < ne && o < no) {
                const int32_t beg = sm.ptr[o], nxt = sm.ptr[o + 1];
                const int32_t kk = sm.acc[e];
                const uint64_t sk = sm.sk[o];
                const int64_t sz = (int64_t)(sk & ~(1ull << 63));
                atomicAdd(reinterpret_cast<unsigned long long *>(&a.active[kk]), (unsigned long long)sz);
                if (!(sk >> 63)) {
                    if (e == beg) atomic_add_i64(&a.diff[kk], sz);
                    if (e == nxt - 1) atomic_add_i64(&a.diff[kk + 1], -sz);
                }
            }
        }
#endif
    };
    if (warp != 0) tile_reds();

    if (warp == 0) {
        agg_publish_packed(est, egrp, tile, tot);
        tile_reds();
        const int64_t pre = agg_prefix_packed(est, egrp, tile);
        if (lane == 0) {
            sm.prefix = pre;
            if (gsum) atomic_add_i64(&a.scalars[SC_GLOBAL_BYTES], gsum);
            if (tile == NTe - 1) {
                a.tensor_pptr[T] = pre + tot;
                a.scalars[SC_NUM_PERIODS] = pre + tot;
            }
        }
    }
    __syncthreads();
    if (fall) return flags;
#ifdef LT_NO_RECORDS
    return flags;
#endif
    // ---- records and per-tensor period offsets, at their final positions
    int64_t q = sm.prefix + woff;             // periods before this warp's current step
    hb = 0;
    for (int j = lane; j < (wbase >> 5); j += 32) hb += __popc(sm.head[j]);
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) hb += __shfl_xor_sync(0xffffffffu, hb, d);
#pragma unroll
    for (int st = 0; st < STEPS; ++st) {
        const int32_t e = wbase + st * 32 + lane;
        const uint32_t hw = sm.head[(wbase >> 5) + st];
        const int32_t o = hb + __popc(hw & le);
        hb += __popc(hw);
        if (e < ne && o < no) {
            const int32_t beg = sm.ptr[o];
            const int64_t my = q + __popc(pb[st] & lt);
            if (e == beg) a.tensor_pptr[o0 + o] = my;
            if (pb[st] & (1u << lane)) {
                const int32_t nxt = sm.ptr[o + 1], kk = sm.acc[e];
                a.p_tensor[my] = o0 + o;
                if (e != nxt - 1) {
                    a.p_start[my] = kk + 1; a.p_end[my] = sm.acc[e + 1] - 1; a.p_wraps[my] = 0;
                } else {
                    const int32_t fk = beg >= 0 ? sm.acc[beg] : __ldg(a.acc + e0 + beg);
                    a.p_start[my] = (kk + 1) % N; a.p_end[my] = ((fk - 1) % N + N) % N; a.p_wraps[my] = 1;
                }
            }
        }
        q += __popc(pb[st]);
    }
    return flags;
}

#ifndef LT_MINB
#define LT_MINB 6            // 40 registers; 5 blocks per SM by shared memory
#endif
__global__ void __launch_bounds__(LIFETIME_THREADS, LT_MINB)
k_events(LifetimeArgs a) {
    asm volatile("griddepcontrol.wait;" ::: "memory");      // owners + zeroed status (programmatic launch)
    extern __shared__ __align__(16) unsigned char smraw[];
    EvSmem &sm = *reinterpret_cast<EvSmem *>(smraw);
    const int64_t NTe = lifetime_event_tiles(a.E);
    const int64_t tile = blockIdx.x;
    const LtWork w = lt_work(a.work, a.N, a.E);
    unsigned long long flags = 0;
    if (tile < NTe) flags = event_tile(a, sm, tile, NTe, w.est, w.egrp, w.owner);
    else if (a.T > 0) {
        flags = LF_BAD_PTR;                  // tensors but no events: every tensor is empty
    }
    if (flags) atomicOr(reinterpret_cast<unsigned long long *>(&a.scalars[SC_FLAGS]), flags);
}

// ---------------------------------------------------------------- kernels
__global__ void __launch_bounds__(KT_THREADS, KT_MINB)
k_kernels(LifetimeArgs a) {
    asm volatile("griddepcontrol.wait;" ::: "memory");      // k_events complete (programmatic launch)
    static_assert(KT_THREADS <= 512, "scan[] holds 16 warp totals per chain");
    __shared__ int64_t scan[40];
    __shared__ int64_t s_pre[2];
    __shared__ int64_t s_tile;
    const int64_t N = a.N, E = a.E;
    const int64_t NTe = lifetime_event_tiles(E), NTk = lifetime_kernel_tiles(N);
    const LtWork w = lt_work(a.work, N, E);                     // dur chain, then diff chain
    if (threadIdx.x == 0) s_tile = blockIdx.x;
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
    // both chains in one exchange: warp-level inclusive scans, the warp totals
    // through shared memory, one barrier; warp 0 then publishes the tile's
    // aggregates and resolves its prefix (one more barrier)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t id = warp_inclusive_sum<int64_t>(sd), iff = warp_inclusive_sum<int64_t>(sf);
    if (lane == 31) { scan[warp] = id; scan[16 + warp] = iff; }
    __syncthreads();
    int64_t xd = id - sd, xf = iff - sf, agg[2] = {0, 0};
#pragma unroll
    for (int q = 0; q < KT_THREADS / 32; ++q) {
        const int64_t vd = scan[q], vf = scan[16 + q];
        if (q < warp) { xd += vd; xf += vf; }
        agg[0] += vd; agg[1] += vf;
    }
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
                                                                          args.work, status, nstatus, args.active,
                                                                          args.N, args.scalars);
        count_launch();
    } else {
        TIO_CUDA(cudaMemsetAsync(args.work, 0, sizeof(int64_t) * 2, stream));
        TIO_CUDA(cudaMemsetAsync(status, 0, sizeof(int64_t) * nstatus, stream));
        TIO_CUDA(cudaMemsetAsync(args.active, 0, sizeof(int64_t) * (args.N > 0 ? args.N : 1), stream));
        TIO_CUDA(cudaMemsetAsync(args.scalars, 0, sizeof(int64_t) * SC_COUNT, stream));
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
