// planner.cu — Algorithm 1 (reference planner.py:267-370) as one persistent
// cooperative kernel: every round re-derives, in parallel, exactly the
// candidates the last commit can have changed, reduces the exact argmax of
// benefit/cost, and commits it, with two grid barriers per round.
//
// Exactness — how each reference rule is kept:
//   * channel searches (bandwidth.py:88-120) run on sorted, pairwise disjoint
//     interval arrays (committed bookings and their +-iteration shadows,
//     :139-151); the walk starts at a binary-searched position, which cannot
//     change the result for disjoint intervals (the merge step flags any
//     overlap as an invariant failure);
//   * a candidate's cached placement is re-derived only when the last commit's
//     bookings overlap it (booking more intervals can only push an earliest
//     fit later and a latest fit earlier, so a non-overlapped placement is still
//     the optimum); SSD infeasibility is permanent for the same reason;
//   * benefit = size x sum of durations of covered kernels with residual >
//     capacity (planner.py:253-262); covered kernels form <= 2 contiguous
//     ranges (:232-250) and the sum comes from a chunked prefix array that is
//     rebuilt where kernels flipped to non-critical;
//   * the winner is the max of benefit/cost by 192-bit cross products, ties to
//     the lowest candidate index = first in (tensor_id, start_kernel) order
//     (:295-310);
//   * commit: bookings + shadows, residual -= size on every covered kernel,
//     host occupancy (:314-348).
// Candidates that can never win again are dropped (st GONE): infeasible on
// both paths, or zero benefit on a path whose window can only shrink (SSD
// without a host path, or host).
#include "common.cuh"
#include "block_scan.cuh"
#include "planner.cuh"
#ifdef TIO_PLAN_PROFILE
// warp fit-walk iterations (32 bookings each) of the refits: total and max
__device__ unsigned long long g_wwalk_total, g_wwalk_max, g_wwalk_n;
#define WWALK_COUNT(n) do { if ((threadIdx.x & 31) == 0) { atomicAdd(&g_wwalk_total, (unsigned long long)(n)); \
    atomicAdd(&g_wwalk_n, 1ull); atomicMax(&g_wwalk_max, (unsigned long long)(n)); } } while (0)
#endif
#include "warp_search.cuh"

namespace cg = cooperative_groups;

namespace tio {

constexpr int MAXG = 1024;
// longest wait for the other ranks' round message before a sharded planning
// call gives up (status 3, TIO_ERR_CUDA "rank exchange timed out")
#ifndef TIO_EXCHANGE_TIMEOUT_NS
#define TIO_EXCHANGE_TIMEOUT_NS 30000000000ll
#endif
constexpr int64_t EXCHANGE_TIMEOUT_NS = TIO_EXCHANGE_TIMEOUT_NS;

struct LastCommit {
    int64_t dest;                 // 0 none (first round), 1 SSD, 2 CPU
    int64_t off_s[3], off_e[3];   // new bookings on the offload channel
    int64_t pre_s[3], pre_e[3];   // new bookings on the prefetch channel
    int64_t nb;                   // bookings per channel (3 with shadows, 1 without)
    int64_t occ_s, occ_e;         // new host occupancy (CPU commits)
};

// A channel as the searches see it: the sorted interval arrays in global
// memory, optionally with a window [w0, w1) of them staged in shared memory
// (a dirty tile's time span); indices outside the window read global memory.
struct ChanView {
    const int64_t *s, *e;
    int64_t n;
    const int64_t *ws = nullptr, *we = nullptr;
    int64_t w0 = 0, w1 = 0;
    // search bounds valid for every placement inside the staged tile span
    // [t_lo, t_hi): the first booking ending after t_lo .. the first starting
    // at or after t_hi (a fit's searched index lies between them)
    int64_t lb = 0, ub = INT64_MAX;
    __device__ __forceinline__ int64_t S(int64_t i) const { return (i >= w0 && i < w1) ? ws[i - w0] : ld_cg(s + i); }
    __device__ __forceinline__ int64_t E(int64_t i) const { return (i >= w0 && i < w1) ? we[i - w0] : ld_cg(e + i); }
};

// kernel start times, optionally with a shared-memory window [w0, w1)
struct StartsView {
    const int64_t *g;
    const int64_t *w = nullptr;
    int64_t w0 = 0, w1 = 0;
    __device__ __forceinline__ int64_t operator()(int64_t k) const { return (k >= w0 && k < w1) ? w[k - w0] : __ldg(g + k); }
};

// ---------------------------------------------------------------- searches
// first k in [lo, hi) with pred(k) (monotone false..true), hi if none;
// exponential probing upward from lo, then bisection.
template <typename Pred>
__device__ __forceinline__ int64_t gallop_up(int64_t lo, int64_t hi, Pred pred) {
    if (lo >= hi || pred(lo)) return lo;
    int64_t f = lo, step = 1;          // pred(f) false
    int64_t t = hi;                    // pred(t) true (hi by convention)
    while (true) {
        const int64_t x = f + step;
        if (x >= hi) break;
        if (pred(x)) { t = x; break; }
        f = x;
        step <<= 1;
    }
    while (t - f > 1) {
        const int64_t m = f + ((t - f) >> 1);
        if (pred(m)) t = m; else f = m;
    }
    return t;
}

// same, probing downward from hi - 1 (the answer is expected near hi)
template <typename Pred>
__device__ __forceinline__ int64_t gallop_down(int64_t lo, int64_t hi, Pred pred) {
    if (lo >= hi || !pred(hi - 1)) return hi;
    int64_t t = hi - 1, step = 1;      // pred(t) true
    int64_t f = lo - 1;                // pred(f) false (lo - 1 by convention)
    while (true) {
        const int64_t x = t - step;
        if (x < lo) break;
        if (!pred(x)) { f = x; break; }
        t = x;
        step <<= 1;
    }
    while (t - f > 1) {
        const int64_t m = f + ((t - f) >> 1);
        if (pred(m)) t = m; else f = m;
    }
    return t;
}

// bisection for a cold search, galloping from lo for a hinted one
template <typename Pred>
__device__ __forceinline__ int64_t first_true(int64_t lo, int64_t hi, bool cold, Pred pred) {
    if (!cold) return gallop_up(lo, hi, pred);
    while (lo < hi) {
        const int64_t m = (lo + hi) >> 1;
        if (pred(m)) hi = m; else lo = m + 1;
    }
    return lo;
}

// ---------------------------------------------------------------- channels
// bandwidth.py:88-100 reserve_earliest.  The first booking that can matter
// (end > ready) lies in [lo_idx, hi_idx] (0..n for a cold search; a window
// from the candidate's last fit for a refit).  *p = index where the walk
// stopped: every booking before it ends at or before the fit.
#ifdef TIO_PLAN_PROFILE
__device__ unsigned long long g_walk_total, g_walk_max;
#define WALK_COUNT(n) do { atomicAdd(&g_walk_total, (unsigned long long)(n)); atomicMax(&g_walk_max, (unsigned long long)(n)); } while (0)
#else
#define WALK_COUNT(n) do { } while (0)
#endif

__device__ int64_t ch_earliest(const ChanView &c, int64_t ready, int64_t d, int64_t lo_idx, int64_t hi_idx,
                               bool cold, int64_t *p) {
    if (lo_idx < c.lb) lo_idx = c.lb;
    if (hi_idx > c.ub) hi_idx = c.ub;
    if (hi_idx < lo_idx) hi_idx = lo_idx;
    int64_t i = first_true(lo_idx, hi_idx, cold && hi_idx - lo_idx > 64, [&](int64_t j) { return c.E(j) > ready; });
    int64_t t = ready;
    const int64_t i0 = i;
    for (; i < c.n; ++i) {
        int64_t s = c.S(i);
        if (s >= t + d) break;
        int64_t e = c.E(i);
        if (e > t) t = e;
    }
    WALK_COUNT(i - i0);
    *p = i;
    return t;
}

// bandwidth.py:102-120 reserve_latest; false = None.  The first booking at or
// after the deadline lies in [lo_idx, hi_idx]; *q = first booking after the fit.
__device__ bool ch_latest(const ChanView &c, int64_t deadline, int64_t not_before, int64_t d,
                          int64_t lo_idx, int64_t hi_idx, bool cold, int64_t *out, int64_t *q) {
    int64_t start = deadline - d;
    if (lo_idx < c.lb) lo_idx = c.lb;
    if (hi_idx > c.ub) hi_idx = c.ub;
    if (hi_idx < lo_idx) hi_idx = lo_idx;
    const int64_t lo = first_true(lo_idx, hi_idx, cold && hi_idx - lo_idx > 64, [&](int64_t j) { return c.S(j) >= deadline; });
    int64_t i = lo - 1;
    for (; i >= 0; --i) {
        if (start < not_before) { WALK_COUNT(lo - 1 - i); return false; }
        int64_t s = c.S(i);
        if (s >= start + d) continue;
        int64_t e = c.E(i);
        if (e <= start) break;
        start = s - d;
    }
    WALK_COUNT(lo - 1 - i);
    if (start < not_before) return false;
    *out = start;
    *q = i + 1;
    return true;
}

// candidate_window (planner.py:147-176) on one channel pair.
// Incremental refit: channels only gain bookings, so the new earliest offload
// is >= the cached one and the new latest prefetch <= the cached one; the
// searches restart from the cached placement (hint_off / hint_pre_end) instead
// of from ready / deadline, which gives the same optimum without re-walking
// the packed prefix.  First fits pass hint_off = ready, hint_pre_end = deadline.
// Index hints: (hp, hq) from the last fit at channel size hn; since then at
// most n - hn bookings were inserted, so the searched indices lie in
// [hp, hp + n - hn] and [hq, hq + n - hn].  hn < 0: cold search.
__device__ bool fit_pair(const ChanView &off, const ChanView &pre, int64_t d_off, int64_t d_pre,
                         int64_t iteration, int64_t hint_off, int64_t hint_pre_end,
                         int64_t *off_s, int64_t *pre_s, int64_t hp = 0, int64_t hq = 0, int64_t hn = -1,
                         int64_t *np_ = nullptr, int64_t *nq_ = nullptr) {
    if (d_off > iteration || d_pre > iteration) return false;
    int64_t plo = 0, phi = off.n, qlo = 0, qhi = pre.n;
    if (hn >= 0) {
        const int64_t delta = off.n - hn;
        plo = hp; phi = hp + delta < off.n ? hp + delta : off.n;
        qlo = hq; qhi = hq + delta < pre.n ? hq + delta : pre.n;
    }
    int64_t p, q;
    int64_t o = ch_earliest(off, hint_off, d_off, plo, phi, hn < 0, &p);
    int64_t t_off = o + d_off;
    int64_t f;
    if (!ch_latest(pre, hint_pre_end, t_off, d_pre, qlo, qhi, hn < 0, &f, &q)) return false;
    if (!(t_off < f)) return false;
    *off_s = o;
    *pre_s = f;
    if (np_) { *np_ = p; *nq_ = q; }
    return true;
}

// _host_peak_occupancy (planner.py:179-186)
__device__ int64_t host_peak(const int64_t *os, const int64_t *oe, const int64_t *oz, int64_t h,
                             int64_t lo, int64_t hi) {
    int64_t peak = 0;
    for (int64_t pi = -1; pi < h; ++pi) {
        int64_t p;
        if (pi < 0) p = lo;
        else {
            p = ld_cg(os + pi);
            if (!(lo <= p && p <= hi)) continue;
        }
        int64_t sum = 0;
        for (int64_t j = 0; j < h; ++j)
            if (ld_cg(os + j) <= p && p < ld_cg(oe + j)) sum += ld_cg(oz + j);
        if (sum > peak) peak = sum;
    }
    return peak;
}

// ---- host-occupancy index (see PlanArgs): the same maximum as host_peak in
// O(log h): occ(p) = (sizes of starts <= p) - (sizes of ends <= p); the points
// are lo and the starts in [lo, hi].
__device__ __forceinline__ int64_t hx_ub(const int64_t *v, int64_t n, int64_t x) {   // first i: v[i] > x
    int64_t lo = 0, hi = n;
    while (lo < hi) { const int64_t m = (lo + hi) >> 1; if (ld_cg(v + m) <= x) lo = m + 1; else hi = m; }
    return lo;
}
__device__ __forceinline__ int64_t hx_lb(const int64_t *v, int64_t n, int64_t x) {   // first i: v[i] >= x
    int64_t lo = 0, hi = n;
    while (lo < hi) { const int64_t m = (lo + hi) >> 1; if (ld_cg(v + m) < x) lo = m + 1; else hi = m; }
    return lo;
}
__device__ int64_t host_peak_ix(const PlanArgs &a, int64_t h, int64_t lo, int64_t hi) {
    if (h <= 0) return 0;
    const int buf = (int)(h & 1);
    const int64_t *S = a.hx_s[buf], *E = a.hx_e[buf], *A = a.hx_a[buf];
    const int64_t us = hx_ub(S, h, lo), ue = hx_ub(E, h, lo);
    int64_t peak = (us ? ld_cg(a.hx_ps[buf] + us) : 0) - (ue ? ld_cg(a.hx_pe[buf] + ue) : 0);
    if (peak < 0) peak = 0;
    const int64_t i0 = hx_lb(S, us, lo), i1 = hx_ub(S, h, hi);      // starts in [lo, hi]: [i0, i1)
    if (i0 >= i1) return peak;
    const int64_t b0 = i0 >> 5, b1 = (i1 - 1) >> 5;
    int64_t m = INT64_MIN;
    const int64_t e0 = b0 == b1 ? i1 : (b0 + 1) << 5;
    for (int64_t i = i0; i < e0; ++i) { const int64_t v = ld_cg(A + i); m = v > m ? v : m; }
    if (b1 > b0) {
        for (int64_t i = b1 << 5; i < i1; ++i) { const int64_t v = ld_cg(A + i); m = v > m ? v : m; }
        if (b1 - b0 >= 2) {                       // whole blocks b0+1 .. b1-1 from the table
            const int64_t L = b0 + 1, R = b1;     // [L, R)
            int l = 0;
            while (((int64_t)2 << l) <= R - L) ++l;
            const int64_t x = ld_cg(a.hx_tab + (int64_t)l * a.hx_nbmax + L);
            const int64_t y = ld_cg(a.hx_tab + (int64_t)l * a.hx_nbmax + R - ((int64_t)1 << l));
            m = x > m ? x : m;
            m = y > m ? y : m;
        }
    }
    return m > peak ? m : peak;
}

// Block 0, after a CPU commit of [s_new, e_new) x z: the index of h + 1
// intervals into buffer (h + 1) & 1 from buffer h & 1 (one sorted insertion
// per array; prefix sums and occupancies shift and add, no scan), then the
// 32-start block maxima and the range-max table.  The three insertion
// searches run as 32-ary warp searches on warps 0-2; the shift loop keeps
// four elements' loads in flight per thread.
__device__ void hx_insert(const PlanArgs &a, int64_t h, int64_t s_new, int64_t e_new, int64_t z,
                          int64_t *sm_i) {
    const int ob = (int)(h & 1), nbuf = (int)((h + 1) & 1);
    const int64_t *__restrict__ S0 = a.hx_s[ob];
    const int64_t *__restrict__ Z0 = a.hx_sz[ob];
    const int64_t *__restrict__ E0 = a.hx_e[ob];
    const int64_t *__restrict__ EZ0 = a.hx_ez[ob];
    const int64_t *__restrict__ PS0 = a.hx_ps[ob];
    const int64_t *__restrict__ PE0 = a.hx_pe[ob];
    const int64_t *__restrict__ A0 = a.hx_a[ob];
    int64_t *__restrict__ S1 = a.hx_s[nbuf];
    int64_t *__restrict__ Z1 = a.hx_sz[nbuf];
    int64_t *__restrict__ E1 = a.hx_e[nbuf];
    int64_t *__restrict__ EZ1 = a.hx_ez[nbuf];
    int64_t *__restrict__ PS1 = a.hx_ps[nbuf];
    int64_t *__restrict__ PE1 = a.hx_pe[nbuf];
    int64_t *__restrict__ A1 = a.hx_a[nbuf];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (warp < 3) {
        // ks = first start > s_new, ke = first end > e_new, ue = first end > s_new
        const int64_t *v = warp == 0 ? S0 : E0;
        const int64_t x = warp == 1 ? e_new : s_new;
        const int64_t r = warp_lower_bound(0, h, [&](int64_t j) { return ld_cg(v + j) > x; });
        if (lane == 0) sm_i[warp] = r;
    }
    __syncthreads();
    const int64_t ks = sm_i[0], ke = sm_i[1], ue = sm_i[2], n = h + 1;
    const int64_t bd = blockDim.x;
    for (int64_t i0 = threadIdx.x; i0 <= n; i0 += 4 * bd) {
        int64_t sv[4], zv[4], av[4], ev[4], ezv[4], ps[4], pe[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + u * bd;
            sv[u] = zv[u] = av[u] = ev[u] = ezv[u] = ps[u] = pe[u] = 0;
            if (i > n) continue;
            if (i < n) {
                if (i != ks) {
                    const int64_t si = i < ks ? i : i - 1;
                    sv[u] = ld_cg(S0 + si); zv[u] = ld_cg(Z0 + si); av[u] = ld_cg(A0 + si);
                } else {
                    // occupancy at the new start: the old intervals over s_new, plus itself
                    av[u] = (ks ? ld_cg(PS0 + ks) : 0) - (ue ? ld_cg(PE0 + ue) : 0);
                }
                if (i != ke) {
                    const int64_t ei = i < ke ? i : i - 1;
                    ev[u] = ld_cg(E0 + ei); ezv[u] = ld_cg(EZ0 + ei);
                }
            }
            // prefix sums (n + 1 entries; entry 0 is 0 and never read)
            const int64_t pi = i <= ks ? i : i - 1, qi = i <= ke ? i : i - 1;
            ps[u] = pi ? ld_cg(PS0 + pi) : 0;
            pe[u] = qi ? ld_cg(PE0 + qi) : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + u * bd;
            if (i > n) continue;
            if (i < n) {
                if (i == ks) { sv[u] = s_new; zv[u] = z; av[u] += z; }
                else if (sv[u] >= s_new && sv[u] < e_new) av[u] += z;      // the new interval holds this start
                if (i == ke) { ev[u] = e_new; ezv[u] = z; }
                S1[i] = sv[u]; Z1[i] = zv[u]; A1[i] = av[u];
                E1[i] = ev[u]; EZ1[i] = ezv[u];
            }
            PS1[i] = ps[u] + (i > ks ? z : 0);
            PE1[i] = pe[u] + (i > ke ? z : 0);
        }
    }
    __syncthreads();
    // 32-start block maxima = table level 0 (one warp per block of starts)
    const int64_t nb = (n + 31) >> 5;
    for (int64_t j = warp; j < nb; j += nw) {
        const int64_t i = (j << 5) + lane;
        int64_t v = i < n ? ld_cg(A1 + i) : INT64_MIN;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) { const int64_t w = __shfl_xor_sync(0xffffffffu, v, o); v = w > v ? w : v; }
        if (lane == 0) a.hx_tab[j] = v;
    }
    __syncthreads();
    for (int l = 1; l < HX_LEVELS && ((int64_t)1 << l) <= nb; ++l) {
        const int64_t half = (int64_t)1 << (l - 1);
        const int64_t *src = a.hx_tab + (int64_t)(l - 1) * a.hx_nbmax;
        int64_t *dst = a.hx_tab + (int64_t)l * a.hx_nbmax;
        for (int64_t j = threadIdx.x; j + 2 * half <= nb; j += blockDim.x) {
            const int64_t x = ld_cg(src + j), y = ld_cg(src + j + half);
            dst[j] = x > y ? x : y;
        }
        __syncthreads();
    }
}

// _covered_kernels (planner.py:232-250) as <= 2 kernel ranges
__device__ void covered_ranges(const StartsView &starts, int64_t N, int64_t iteration,
                               int wraps, int32_t sk, int32_t ek, int32_t first, int32_t last,
                               int64_t lo_t, int64_t hi_t, int32_t r[4]) {
    r[0] = 1; r[1] = 0; r[2] = 1; r[3] = 0;
    auto range = [&](int64_t a, int64_t b, int64_t sh, int32_t &olo, int32_t &ohi) {
        int64_t L = a, H = b + 1;
        while (L < H) {
            int64_t M = (L + H) >> 1;
            if (starts(M) + sh >= lo_t) H = M; else L = M + 1;
        }
        int64_t klo = L;
        L = klo; H = b + 1;
        while (L < H) {
            int64_t M = (L + H) >> 1;
            if (starts(M + 1) + sh <= hi_t) L = M + 1; else H = M;
        }
        olo = (int32_t)klo;
        ohi = (int32_t)(L - 1);
    };
    if (!wraps) {
        if (sk <= ek) range(sk, ek, 0, r[0], r[1]);
    } else {
        if (last + 1 <= N - 1) range(last + 1, N - 1, 0, r[0], r[1]);
        if (first - 1 >= 0) range(0, first - 1, iteration, r[2], r[3]);
    }
}

// Refit version: the new window [lo_t, hi_t] lies inside the old one, so each
// new range lies inside the old range r_old (planner.py:232-250 restated);
// gallop inward from the old endpoints.
__device__ void covered_ranges_shrunk(const StartsView &starts, int64_t iteration, int wraps,
                                      int64_t lo_t, int64_t hi_t, const int32_t r_old[4], int32_t r[4]) {
    for (int q = 0; q < 4; q += 2) {
        const int64_t a = r_old[q], bnd = r_old[q + 1];
        if (a > bnd) { r[q] = r_old[q]; r[q + 1] = r_old[q + 1]; continue; }
        const int64_t sh = (wraps && q == 2) ? iteration : 0;
        const int64_t klo = gallop_up(a, bnd + 1, [&](int64_t k) { return starts(k) + sh >= lo_t; });
        const int64_t kend = gallop_down(klo, bnd + 1, [&](int64_t k) { return starts(k + 1) + sh > hi_t; });
        r[q] = (int32_t)klo;
        r[q + 1] = (int32_t)(kend - 1);
    }
}

__device__ __forceinline__ bool overlaps(int64_t x, int64_t d, const int64_t *s, const int64_t *e, int64_t nb) {
    for (int q = 0; q < nb; ++q)
        if (x < e[q] && s[q] < x + d) return true;
    return false;
}

// ---------------------------------------------------------------- argmax keys
// The round's argmax carries 4 words: the exact benefit (u128), the cost and
// meta = candidate index << 33 | column position << 2 | destination (both
// < 2^31), compared unsigned: the tie-break is the candidate index.  The rest
// of the winner is re-read from its column once it is known.
__device__ __forceinline__ int64_t key_meta(int64_t cid, int64_t c, int dest) {
    return (int64_t)(((uint64_t)cid << 33) | ((uint64_t)c << 2) | (uint64_t)dest);
}

__device__ __forceinline__ bool kbetter(const Key &a, const Key &b) {
    const bool az = (a.blo | a.bhi) == 0, bz = (b.blo | b.bhi) == 0;
    if (az) return false;
    if (bz) return true;
    const u128 ab = ((u128)a.bhi << 64) | a.blo, bb = ((u128)b.bhi << 64) | b.blo;
    if (ratio_gt(ab, a.cost, bb, b.cost)) return true;
    if (ratio_gt(bb, b.cost, ab, a.cost)) return false;
    return (uint64_t)a.meta < (uint64_t)b.meta;   // tie: lowest candidate index = first in (tensor_id, start_kernel) order
}

__device__ __forceinline__ Key none_key() { return Key{0, 0, 1, 0}; }

__device__ __forceinline__ Key kshfl(const Key &k, int src) {
    Key o;
    o.blo = __shfl_sync(0xffffffffu, k.blo, src);
    o.bhi = __shfl_sync(0xffffffffu, k.bhi, src);
    o.cost = __shfl_sync(0xffffffffu, k.cost, src);
    o.meta = __shfl_sync(0xffffffffu, k.meta, src);
    return o;
}

__device__ __forceinline__ Key warp_best(Key mine) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        Key other = kshfl(mine, (threadIdx.x + o) & 31);
        if (((threadIdx.x & 31) + o) < 32 && kbetter(other, mine)) mine = other;
    }
    return mine;   // valid in lane 0
}

// block-wide argmax; the result is returned to every thread
__device__ Key block_best(Key mine, Key *sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    mine = warp_best(mine);
    if (lane == 0) sm[warp] = mine;
    __syncthreads();
    if (warp == 0) {
        Key k = lane < nw ? sm[lane] : Key{0, 0, 1, 0};
        k = warp_best(k);
        if (lane == 0) sm[32] = k;
    }
    __syncthreads();
    Key r = sm[32];
    __syncthreads();
    return r;
}

__device__ __forceinline__ Key kload(const Key *p) {
    const ulonglong2 *q = reinterpret_cast<const ulonglong2 *>(p);
    const ulonglong2 x = __ldcg(q), y = __ldcg(q + 1);
    return Key{x.x, x.y, (int64_t)y.x, (int64_t)y.y};
}

__device__ __forceinline__ void kstore(Key *p, const Key &k) {
    ulonglong2 *q = reinterpret_cast<ulonglong2 *>(p);
    q[0] = make_ulonglong2(k.blo, k.bhi);
    q[1] = make_ulonglong2((unsigned long long)k.cost, (unsigned long long)k.meta);
}

__device__ __forceinline__ void l2_prefetch(const void *p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// ---------------------------------------------------------------- the kernel
//
// Tiles.  Candidates are grouped into tiles of TILE (= 32, one warp)
// consecutive candidates in ready-time order (a permutation built by the
// setup; the candidate index, i.e. the (tensor_id, start_kernel) rank, stays
// the tie-break key).  Every tile has a static time span [min ready, max
// deadline) that contains every placement its candidates can ever have, two
// kernel hulls that contain every kernel they can ever cover, and a superset
// hull of its current SSD placements.  Round r:
//   phase R + E (no barrier between them)
//     * every warp of the grid takes SSD refits the last commit queued
//       (candidates whose cached placement its bookings overlap): warp
//       searches from the cached placement, then lane 0 re-derives the key
//       and folds it into its block's best;
//     * each block re-derives its own tiles that can have changed: refits were
//       queued there (those candidates are left out this round, taken back
//       the next), it held the last winner, kernels flipped from critical to
//       non-critical inside one of its kernel hulls, or a CPU commit's
//       bookings / host occupancy meet its span.  Unchanged candidates reuse
//       their cached key; a clean tile keeps its tile best, a block with no
//       change keeps its block best.
//   grid barrier
//   phase C (every block, redundantly): exact global argmax, then the commit:
//     channel merge (all blocks), residual update + flip detection + critical
//     prefix rebuild (chunk owners), refit queueing for the next round (tile
//     owners, against the placement hulls), commit record (block 0).
//   grid barrier
__device__ __forceinline__ int64_t gtime() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return (int64_t)t;
}

__device__ __forceinline__ bool spans_hit(int64_t lo, int64_t hi, const int64_t *s, const int64_t *e, int64_t nb) {
    for (int q = 0; q < nb; ++q)
        if (lo < e[q] && s[q] < hi) return true;
    return false;
}


struct WinInfo {
    int64_t idx, dest, size, cost;
    int64_t off_s, off_e, pre_s, pre_e;
    int32_t r[4];
    uint64_t blo, bhi;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// WinMsg copies through 16-byte volatile accesses (peer / IPC memory, never
// cached in L1)
__device__ __forceinline__ void msg_store(WinMsg *dst, const WinMsg &m) {
    const ulonglong2 *s = reinterpret_cast<const ulonglong2 *>(&m);
    ulonglong2 *d = reinterpret_cast<ulonglong2 *>(dst);
#pragma unroll
    for (int i = 0; i < (int)(sizeof(WinMsg) / 16); ++i)
        asm volatile("st.volatile.global.v2.u64 [%0], {%1, %2};" ::"l"(d + i), "l"(s[i].x), "l"(s[i].y) : "memory");
}
__device__ __forceinline__ WinMsg msg_load(const WinMsg *src) {
    WinMsg m;
    ulonglong2 *d = reinterpret_cast<ulonglong2 *>(&m);
    const ulonglong2 *s = reinterpret_cast<const ulonglong2 *>(src);
#pragma unroll
    for (int i = 0; i < (int)(sizeof(WinMsg) / 16); ++i) {
        unsigned long long x, y;
        asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(x), "=l"(y) : "l"(s + i) : "memory");
        d[i] = make_ulonglong2(x, y);
    }
    return m;
}

// The round's winner (replaces a grid barrier + a redundant per-block
// argmax): every block arrives on the grid's arrival counter after writing
// its block best; the last arrival's block reduces the G block bests, thread
// 0 reads the winner's column into a WinMsg, and with R > 1 ranks puts it
// into slot [round & 1][rank] of every rank's mailbox, raises its flag there
// (release, system scope), waits for all R flags of its own mailbox, and
// takes the best of the R messages (kbetter: ratio, then lowest candidate
// index — the same winner on every rank).  It publishes the winner and bumps
// win_gen; every block waits for win_gen and reads the winner.
__device__ void round_winner(const PlanArgs &a, int64_t round, int G, Key *sm_key, WinMsg *out) {
    __shared__ int s_last;
    __shared__ WinMsg s_msg;
    __shared__ int s_pick, s_lost;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long *ctr = reinterpret_cast<unsigned long long *>(a.bar);
        unsigned long long v;
        asm volatile("atom.add.acq_rel.gpu.u64 %0, [%1], 1;" : "=l"(v) : "l"(ctr) : "memory");
        s_last = ((v + 1) % (unsigned long long)G) == 0;
    }
    __syncthreads();
    if (s_last) {
        Key w{0, 0, 1, 0};
        for (int j = threadIdx.x; j < G; j += blockDim.x) {
            const Key o = kload(&a.blk_best[j]);
            if (kbetter(o, w)) w = o;
        }
        w = block_best(w, sm_key);
        if (threadIdx.x == 0) {
            WinMsg m;
            memset(&m, 0, sizeof(m));
            m.k = w;
            if ((w.blo | w.bhi) != 0) {
                const int64_t c = (int64_t)(((uint64_t)w.meta >> 2) & 0x7fffffffu);
                const int q0 = (w.meta & 3) == TIO_DEST_SSD ? 0 : 2;
                m.size = __ldg(&a.c_size[c]);
                m.off_s = ld_cg(&a.place[4 * c + q0]);
                m.off_e = m.off_s + __ldg(&a.c_d[4 * c + q0]);
                m.pre_s = ld_cg(&a.place[4 * c + q0 + 1]);
                m.pre_e = m.pre_s + __ldg(&a.c_d[4 * c + q0 + 1]);
                for (int q = 0; q < 4; ++q) m.r[q] = ld_cg(&a.rng[4 * c + q]);
            }
            s_msg = m;
            s_pick = 0;
            s_lost = 0;
        }
        __syncthreads();
        if (a.nranks > 1 && threadIdx.x < 32) {
            // the exchange, one lane per rank p (in parallel): lane p puts
            // this rank's message into rank p's mailbox and raises its flag
            // there (release, system scope), then waits for rank p's flag in
            // this rank's mailbox (acquire).  The slot parity follows the tag,
            // so it keeps alternating across consecutive planning calls
            // (epoch += rounds + 2 between calls).
            const int lane = threadIdx.x;
            const unsigned long long tag = a.epoch + (unsigned long long)round + 1;
            const int slot = (int)(tag & 1);
            const int R = a.nranks;
            if (lane < R) {
                Mailbox *mb = a.mb_peer[lane];
                msg_store(&mb->msg[slot][a.rank], s_msg);
                st_release_sys(&mb->flag[a.rank], tag);
            }
            // bounded wait: a rank that never arrives (died, or was never
            // launched) ends this planning call with status 3 instead of
            // hanging the GPU; the round then has no winner on this rank
            bool lost = false;
            if (lane < R) {
                const int64_t t0 = gtime();
                unsigned spins = 0;
                while (ld_acquire_sys(&a.mb_self->flag[lane]) < tag)
                    if ((++spins & 1023u) == 0 && gtime() - t0 > EXCHANGE_TIMEOUT_NS) { lost = true; break; }
            }
            lost = __any_sync(0xffffffffu, lost);
            // best of the R messages: ratio, then lowest candidate index
            // (the same winner on every rank)
            Key k = none_key();
            if (!lost && lane < R) k = msg_load(&a.mb_self->msg[slot][lane]).k;
            int who = lane;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const Key ok = kshfl(k, (lane + o) & 31);
                const int ow = __shfl_sync(0xffffffffu, who, (lane + o) & 31);
                if (lane + o < 32 && kbetter(ok, k)) { k = ok; who = ow; }
            }
            if (lane == 0) {
                if (lost) { s_lost = 1; a.scalars[PS_STATUS] = 3; }
                s_pick = who;
            }
            __syncwarp();
            if (lane == 0) {
                WinMsg m;
                if (s_lost) memset(&m, 0, sizeof(m));
                else m = msg_load(&a.mb_self->msg[slot][s_pick]);
                s_msg = m;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const WinMsg m = s_msg;
#ifdef TIO_VDEBUG
            printf("[vdbg] rank %d/%d round %lld blk %d: winner meta %llx blo %llx\n", a.rank, a.nranks,
                   (long long)round, (int)blockIdx.x, (unsigned long long)m.k.meta, (unsigned long long)m.k.blo);
#endif
            msg_store(a.win, m);
            st_release_gpu(a.win_gen, (unsigned long long)round + 1);
        }
    }
    if (threadIdx.x == 0) {
        while (ld_acquire_gpu(a.win_gen) < (unsigned long long)round + 1) {
        }
        *out = msg_load(a.win);
    }
    __syncthreads();
}

constexpr int DIRTY_MAX = 2048;  // own tiles tested / listed per pass
constexpr size_t PLAN_DYN_SMEM = 0;

// The round loop of one planner instance on G blocks; b = this block's index
// among them.  plan_loop_kernel runs one instance on the whole grid;
// plan_loop_kernel_multi runs one instance per virtual rank on its share.
__device__ __forceinline__ void plan_loop_body(const PlanArgs &a, const int G, const int b) {
    __shared__ int64_t cp_prefix[MAXG + 1];
    __shared__ Key sm_key[33];
    __shared__ WinMsg s_win;
    __shared__ LastCommit last;
    __shared__ int64_t sm_scan[40];
    __shared__ int64_t ch_n[4];
    __shared__ int32_t ch_par[4];
    __shared__ int64_t s_nocc;
    __shared__ int64_t s_crit;
    __shared__ int64_t s_flip[3];          // previous round: flipped count, lo, hi
    __shared__ int64_t s_win_tile;
    __shared__ int32_t s_dirty[DIRTY_MAX];
    __shared__ Key s_rbest[32];            // best key per warp among this round's refits here
    __shared__ bool s_prev_refit;          // refits ran here last round (their keys are in blk_best)
    __shared__ Key s_tmax;                 // best key over the own tiles (as of their last change)
    __shared__ int32_t s_ndirty;
    __shared__ int64_t s_fmin, s_fmax;     // this round's flipped kernels in the block's chunk

    const int64_t N = a.N, I = a.iteration, cap = a.capacity;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int64_t KC = a.chunk;
    const int64_t x0 = (int64_t)b * KC;                       // chunk over x in [0, N]
    const int64_t x1 = (x0 + KC < N + 1) ? x0 + KC : N + 1;
    const int64_t period = I > 0 ? I : 0;
    const int64_t nb = period > 0 ? 3 : 1;
    const int64_t NT = a.ntiles;
    // tile ownership: rank `rank` of R owns tiles t = rank + R u; its block b
    // owns u = b, b + G, ... (R = 1: tiles b, b + G, ...)
    const int64_t R = a.nranks > 1 ? a.nranks : 1, rk = a.nranks > 1 ? a.rank : 0;
    const int64_t NTr = NT > rk ? (NT - rk + R - 1) / R : 0;
    const int64_t my_tiles = NTr > b ? (NTr - 1 - b) / G + 1 : 0;
    auto own_tile = [&](int64_t j) -> int64_t { return rk + R * (b + j * G); };
    int64_t *flip = &a.scalars[PS_FLIP];                       // [3 slots][cnt, lo, hi]
    const Key none{0, 0, 1, 0};

    if (ld_cg(&a.scalars[PS_STATUS]) != 0) return;  // unsatisfiable (set by setup)

    // ---- setup: chunk prefix of critical durations
    // prefix of duration x [residual > capacity] over this block's chunk,
    // four kernels per thread per block scan
    // from: the first position whose prefix can have changed (the prefix up
    // to it, local_cp[from], is unchanged and seeds the running sum)
    // software-pipelined: the next step's residual / duration loads are in
    // flight across this step's block scan
    auto rebuild_chunk = [&](int64_t from) {
        int64_t run = from > x0 ? ld_cg(&a.local_cp[from]) : 0;
        const int64_t step = 4 * (int64_t)blockDim.x;
        int64_t rc[4], dc[4];
        auto load4 = [&](int64_t x, int64_t *r, int64_t *d) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const bool ok = x + u < x1 && x + u < N;
                r[u] = ok ? ld_cg(&a.resid[x + u]) : 0;
                d[u] = ok ? __ldg(&a.dur[x + u]) : 0;
            }
        };
        load4(from + 4 * (int64_t)threadIdx.x, rc, dc);
        for (int64_t base = from; base < x1; base += step) {
            const int64_t x = base + 4 * (int64_t)threadIdx.x;
            int64_t rn[4], dn[4];
            if (base + step < x1) load4(x + step, rn, dn);
            int64_t wv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) wv[u] = rc[u] > cap ? dc[u] : 0;
#pragma unroll
            for (int u = 0; u < 4; ++u) { rc[u] = rn[u]; dc[u] = dn[u]; }
            int64_t tot;
            int64_t ex = run + block_exclusive_sum<int64_t>(wv[0] + wv[1] + wv[2] + wv[3], sm_scan, &tot);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (x + u < x1) a.local_cp[x + u] = ex;
                ex += wv[u];
            }
            run += tot;
        }
        if (threadIdx.x == 0) a.chunk_sum[b] = run;
    };
    {
        int64_t crit = 0;
        for (int64_t x = x0 + threadIdx.x; x < x1 && x < N; x += blockDim.x)
            crit += ld_cg(&a.resid[x]) > cap;
        __syncthreads();
        rebuild_chunk(x0);
        int64_t tot = block_sum<int64_t>(crit, sm_scan);
        if (threadIdx.x == 0 && tot) atomic_add_i64(&a.scalars[PS_CRIT], tot);
        if (threadIdx.x == 0) {
            last.dest = 0;
            last.nb = nb;
            s_nocc = 0;
            s_win_tile = -1;
            s_prev_refit = false;
            s_tmax = Key{0, 0, 1, 0};
            for (int q = 0; q < 4; ++q) { ch_n[q] = 0; ch_par[q] = 0; }
            if (b == 0)
                for (int q = 0; q < 3; ++q) { flip[3 * q] = 0; flip[3 * q + 1] = INT64_MAX; flip[3 * q + 2] = -1; }
#ifdef TIO_PLAN_PROFILE
            if (b == 0) { g_walk_total = 0; g_walk_max = 0; g_wwalk_total = 0; g_wwalk_max = 0; g_wwalk_n = 0; }
#endif
        }
    }
    grid_barrier(a.bar, G);

#ifdef TIO_PLAN_PROFILE
    // phase profile (block 0, %globaltimer): a debug build only, the timer
    // read is a long-latency operation
    int64_t dbg[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int64_t tprev = gtime();
    const bool tb = (b == 0 && threadIdx.x == 0);
#define TICK(slot) do { if (tb) { int64_t _t = gtime(); dbg[slot] += _t - tprev; tprev = _t; } } while (0)
#define PROF(stmt) stmt
    // per-block phase-E split (thread 0 of every block): dirty test, pass 1,
    // window staging, pass 2, tile reduce, block reduce
    int64_t sub[6] = {0, 0, 0, 0, 0, 0};      // this round
    int64_t slow[7] = {0, 0, 0, 0, 0, 0, 0};  // summed over rounds whose phase E took > 15 us; [6] = count
    int64_t tsub = 0;
#define SUB(slot) do { if (threadIdx.x == 0) { int64_t _t = gtime(); sub[slot] += _t - tsub; tsub = _t; } } while (0)
#else
#define TICK(slot) do { } while (0)
#define PROF(stmt)
#define SUB(slot) do { } while (0)
#endif
    for (int64_t round = 0;; ++round) {
        // ---- round prologue: crit count, last round's flips, chunk prefix
        if (threadIdx.x == 0) {
            s_fmin = INT64_MAX;            // this round's flips in the chunk (phase C)
            s_fmax = -1;
            s_crit = ld_cg(&a.scalars[PS_CRIT]);
            if (round > 0) {
                const int64_t *f = flip + 3 * ((round - 1) % 3);
                s_flip[0] = ld_cg(f); s_flip[1] = ld_cg(f + 1); s_flip[2] = ld_cg(f + 2);
            }
            // slot of the next round's commit; nobody reads it this round
            if (b == 0) {
                int64_t *f = flip + 3 * ((round + 1) % 3);
                f[0] = 0; f[1] = INT64_MAX; f[2] = -1;
            }
        }
        __syncthreads();
        if (round == 0 || s_flip[0] > 0) {
            int64_t v = 0;
            int nchunks = (int)((N + 1 + KC - 1) / KC);
            // exclusive prefix of chunk sums into cp_prefix[0..nchunks]
            for (int base = 0; base < nchunks; base += blockDim.x) {
                int j = base + threadIdx.x;
                int64_t w = j < nchunks ? ld_cg(&a.chunk_sum[j]) : 0;
                int64_t tot;
                int64_t ex = block_exclusive_sum<int64_t>(w, sm_scan, &tot);
                if (j < nchunks) cp_prefix[j] = v + ex;
                v += tot;
            }
            if (threadIdx.x == 0) cp_prefix[nchunks] = v;
        }
        __syncthreads();
#ifdef TIO_VDEBUG
        if (threadIdx.x == 0 && (b == 0 || b == G - 1))
            printf("[vdbg] rank %d blk %d round %lld start: crit %lld\n", a.rank, b, (long long)round, (long long)s_crit);
#endif
        if (s_crit <= 0 || N == 0) break;   // planner.py:293 peak <= capacity
        if (a.max_rounds > 0 && round >= a.max_rounds) break;
        TICK(0);
        PROF(const int64_t te0 = gtime());
        PROF(if (threadIdx.x == 0) { tsub = te0; for (int q = 0; q < 6; ++q) sub[q] = 0; });

        // ---- phase E: re-evaluate the dirty tiles of this block
        ChanView cv[4];
        for (int q = 0; q < 4; ++q) {
            cv[q].s = a.ch_s[q][ch_par[q]];
            cv[q].e = a.ch_e[q][ch_par[q]];
            cv[q].n = ch_n[q];
        }
        // Re-derive candidate c's key against the current state (planner.py:147-262):
        // first fit (round 0), refit flags from phase R, host path, benefit
        // from the critical prefix or the cached key; writes st / vkey.
        auto eval_lane = [&](int64_t c, int32_t cid, int8_t st, const Key &ck, const int4 &rr, bool rr_fresh) -> Key {
            Key mine = none;
            if (!(st & ST_GONE)) {
                int ssd = st & 3, host = (st >> 2) & 3;
                // round 0: first fits here; later rounds phase R refitted the
                // SSD placements the last commit overlapped and flagged them
                const bool need = ssd == S_UNK || (st & ST_REFIT);
                bool moved = false;
                if (ssd == S_UNK) {
                    const int64_t d0 = __ldg(&a.c_d[4 * c]), d1 = __ldg(&a.c_d[4 * c + 1]);
                    int64_t os, ps, np, nq;
                    if (fit_pair(cv[0], cv[1], d0, d1, I, __ldg(&a.c_ready[c]), __ldg(&a.c_deadline[c]),
                                 &os, &ps, 0, 0, -1, &np, &nq)) {
                        int32_t r[4];
                        covered_ranges(StartsView{a.starts}, N, I, __ldg(&a.c_wraps[c]), __ldg(&a.c_sk[c]),
                                       __ldg(&a.c_ek[c]), __ldg(&a.c_first[c]), __ldg(&a.c_last[c]),
                                       os + d0, ps, r);
                        *reinterpret_cast<int4 *>(&a.rng[4 * c]) = make_int4(r[0], r[1], r[2], r[3]);
                        ssd = S_OK;
                        a.place[4 * c] = os;
                        a.place[4 * c + 1] = ps;
                        a.hidx[2 * c] = (int32_t)np;
                        a.hidx[2 * c + 1] = (int32_t)nq;
                        a.hver[c] = (int32_t)cv[0].n;
                    } else {
                        ssd = S_DEAD;
                        moved = true;
                    }
                } else if ((st & ST_REFIT) && ssd == S_DEAD) {
                    moved = true;
                }
                // host path (only consulted once the SSD path is dead: planner.py:211-227)
                if (ssd == S_DEAD && a.has_host && host != H_DEAD) {
                    const int64_t d2 = __ldg(&a.c_d[4 * c + 2]), d3 = __ldg(&a.c_d[4 * c + 3]);
                    bool refit = host == H_UNK;
                    bool recap = false;
                    if (!refit && last.dest == TIO_DEST_CPU) {
                        refit = overlaps(ld_cg(&a.place[4 * c + 2]), d2, last.off_s, last.off_e, last.nb) ||
                                overlaps(ld_cg(&a.place[4 * c + 3]), d3, last.pre_s, last.pre_e, last.nb);
                        if (!refit && host == H_OK) {
                            int64_t lo = ld_cg(&a.place[4 * c + 2]) + d2, hi = ld_cg(&a.place[4 * c + 3]);
                            recap = last.occ_s <= hi && last.occ_e > lo;
                        }
                    }
                    if (refit) {
                        int64_t os, ps;
                        int64_t g_off = __ldg(&a.c_ready[c]), g_pre = __ldg(&a.c_deadline[c]);
                        if (host != H_UNK) { g_off = ld_cg(&a.place[4 * c + 2]); g_pre = ld_cg(&a.place[4 * c + 3]) + d3; }
                        if (fit_pair(cv[2], cv[3], d2, d3, I, g_off, g_pre, &os, &ps)) {
                            a.place[4 * c + 2] = os;
                            a.place[4 * c + 3] = ps;
                            recap = true;
                            moved = true;
                        } else {
                            host = H_DEAD;
                            moved = true;
                        }
                    }
                    if (recap) {
                        int64_t lo = ld_cg(&a.place[4 * c + 2]) + d2, hi = ld_cg(&a.place[4 * c + 3]);
                        int64_t occ = host_peak_ix(a, s_nocc, lo, hi);
                        host = (occ + __ldg(&a.c_size[c]) > a.host_cap) ? H_CAPFAIL : H_OK;
                    }
                }
                int dest = ssd == S_OK ? TIO_DEST_SSD : (ssd == S_DEAD && host == H_OK ? TIO_DEST_CPU : 0);
                int8_t nst = (int8_t)(ssd | (host << 2));
                if (ssd == S_DEAD && (!a.has_host || host == H_DEAD)) {
                    nst |= ST_GONE;
                } else if (dest) {
                    const int q0 = dest == TIO_DEST_SSD ? 0 : 2;
                    // unchanged since its last evaluation: same window on the same
                    // path and no kernel of its covered ranges flipped -> same key
                    bool cached = false;
                    if (round > 0 && !moved && !need) {
                        if ((ck.meta & 3) == dest && ((uint64_t)ck.meta >> 33) == (uint64_t)cid) {
                            cached = true;
                            if (s_flip[0] > 0) {
                                const int64_t fl = s_flip[1], fh = s_flip[2];
                                cached = !((rr.x <= rr.y && rr.x <= fh && fl <= rr.y) ||
                                           (rr.z <= rr.w && rr.z <= fh && fl <= rr.w));
                            }
                            if (cached) mine = ck;
                        }
                    }
                    if (!cached) {
                        const int64_t doff = __ldg(&a.c_d[4 * c + q0]), dpre = __ldg(&a.c_d[4 * c + q0 + 1]);
                        const int64_t size = __ldg(&a.c_size[c]);
                        int32_t r[4];
                        if (moved) {
                            const int64_t os = ld_cg(&a.place[4 * c + q0]);
                            const int64_t ps = ld_cg(&a.place[4 * c + q0 + 1]);
                            covered_ranges(StartsView{a.starts}, N, I, __ldg(&a.c_wraps[c]), __ldg(&a.c_sk[c]),
                                           __ldg(&a.c_ek[c]), __ldg(&a.c_first[c]), __ldg(&a.c_last[c]),
                                           os + doff, ps, r);
                            *reinterpret_cast<int4 *>(&a.rng[4 * c]) = make_int4(r[0], r[1], r[2], r[3]);
                        } else if (need && !rr_fresh) {
                            // first fit above: the ranges were just written
                            const int4 r2 = __ldcg(reinterpret_cast<const int4 *>(&a.rng[4 * c]));
                            r[0] = r2.x; r[1] = r2.y; r[2] = r2.z; r[3] = r2.w;
                        } else {
                            // cached ranges, or phase R's refit passing the ranges it
                            // just derived (no reload of what this thread stored)
                            r[0] = rr.x; r[1] = rr.y; r[2] = rr.z; r[3] = rr.w;
                        }
                        // sum of critical durations over the <= 2 covered ranges: the
                        // four prefix loads issued together, 32-bit chunk division
                        const bool v0 = r[0] <= r[1], v1 = r[2] <= r[3];
                        const int32_t xa0 = v0 ? r[0] : 0, xb0 = v0 ? r[1] + 1 : 0;
                        const int32_t xa1 = v1 ? r[2] : 0, xb1 = v1 ? r[3] + 1 : 0;
                        const int64_t la0 = ld_cg(&a.local_cp[xa0]), lb0 = ld_cg(&a.local_cp[xb0]);
                        const int64_t la1 = ld_cg(&a.local_cp[xa1]), lb1 = ld_cg(&a.local_cp[xb1]);
                        const int32_t kc = (int32_t)KC;
                        int64_t ct = 0;
                        if (v0) ct += (cp_prefix[xb0 / kc] + lb0) - (cp_prefix[xa0 / kc] + la0);
                        if (v1) ct += (cp_prefix[xb1 / kc] + lb1) - (cp_prefix[xa1 / kc] + la1);
                        if (ct == 0) {
                            // benefit only ever shrinks on a host window or on an SSD
                            // window without a host path to fall back to
                            if (dest == TIO_DEST_CPU || !a.has_host) nst |= ST_GONE;
                        } else {
                            const u128 bf = (u128)(uint64_t)size * (uint64_t)ct;
                            mine.blo = (uint64_t)bf;
                            mine.bhi = (uint64_t)(bf >> 64);
                            mine.cost = doff + dpre;
                            mine.meta = key_meta(cid, c, dest);
                        }
                        // the key (zero benefit included) for later rounds
                        kstore(&a.vkey[c], Key{mine.blo, mine.bhi, doff + dpre, key_meta(cid, c, dest)});
                    }
                }
                if (nst != st) a.st[c] = nst;
            }
            return mine;
        };
        // ---- phase R: the SSD refits the last commit queued (candidates whose
        // cached placement its bookings overlap), spread over every warp of
        // the grid: 32-ary searches and 32-wide fit walks (bandwidth.py:88-120);
        // lane 0 then re-derives the key; the block's best refit key joins its
        // block best.  No barrier: the owners' tile summaries below leave these
        // candidates out this round (they take them back next round).
        if (threadIdx.x < 32) s_rbest[threadIdx.x] = none;
        __syncthreads();
        if (round > 0) {
            const int q = (int)((round - 1) & 1);
            const int64_t nq = ld_cg(&a.scalars[PS_RQ + q]);
            const int64_t gw = ((int64_t)b * blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)G * blockDim.x) >> 5;
            for (int64_t k = gw; k < nq; k += nw) {
                const int64_t cc = ld_cg(&a.rq[q][k]);
                const int8_t sc = ld_cg(&a.st[cc]);
                const longlong2 dd = __ldg(reinterpret_cast<const longlong2 *>(&a.c_d[4 * cc]));
                const longlong2 pl = __ldcg(reinterpret_cast<const longlong2 *>(&a.place[4 * cc]));
                const int2 hx = __ldcg(reinterpret_cast<const int2 *>(&a.hidx[2 * cc]));
                const int32_t hv = ld_cg(&a.hver[cc]);
                const int4 rr = __ldcg(reinterpret_cast<const int4 *>(&a.rng[4 * cc]));
                const int32_t ccid = (int32_t)__ldg(&a.tcand[cc]);     // loaded with the rest, used after the fit
                const int64_t d0 = dd.x, d1 = dd.y;
                const int64_t h_off = pl.x, h_pre = pl.y + d1;
                const int64_t delta = cv[0].n - hv;
                const int64_t plo = hx.x, qlo = hx.y;
                const int64_t phi = plo + delta < cv[0].n ? plo + delta : cv[0].n;
                const int64_t qhi = qlo + delta < cv[1].n ? qlo + delta : cv[1].n;
                const int32_t ro[4] = {rr.x, rr.y, rr.z, rr.w};
                int64_t os = 0, ps = 0, np = 0, nq2 = 0;
                const bool ok = warp_fit_pair(cv[0].s, cv[0].e, cv[0].n, cv[1].s, cv[1].e, cv[1].n, d0, d1, I,
                                              h_off, h_pre, plo, phi, qlo, qhi, &os, &ps, &np, &nq2);
                int32_t r[4] = {1, 0, 1, 0};
                if (ok) warp_covered_ranges_shrunk(a.starts, I, __ldg(&a.c_wraps[cc]), os + d0, ps, ro, r);
                if (lane == 0) {
                    if (ok) {
                        a.place[4 * cc] = os;
                        a.place[4 * cc + 1] = ps;
                        *reinterpret_cast<int4 *>(&a.rng[4 * cc]) = make_int4(r[0], r[1], r[2], r[3]);
                        // keep the tile's placement hulls supersets: an offload only
                        // moves later, a prefetch only earlier
                        long long *h = reinterpret_cast<long long *>(a.t_hull + 4 * (cc / TILE));
                        atomicMax(h + 1, (long long)(os + d0));
                        atomicMin(h + 2, (long long)ps);
                        a.hidx[2 * cc] = (int32_t)np;
                        a.hidx[2 * cc + 1] = (int32_t)nq2;
                        a.hver[cc] = (int32_t)cv[0].n;
                    }
                    const int8_t st2 = (int8_t)((sc & ~3) | (ok ? S_OK : S_DEAD) | ST_REFIT);
                    const Key kk = eval_lane(cc, ccid, st2, none, make_int4(r[0], r[1], r[2], r[3]), ok);
                    if (kbetter(kk, s_rbest[warp])) s_rbest[warp] = kk;
                }
                __syncwarp();
            }
            PROF(if (b == 0 && threadIdx.x == 0) atomic_add_i64(&a.scalars[PS_DBG + 9], nq));
        }
        bool any_dirty = false;
        for (int64_t j0 = 0; j0 < my_tiles; j0 += DIRTY_MAX) {
            // dirty test of up to DIRTY_MAX own tiles, compacted into s_dirty
            if (threadIdx.x == 0) s_ndirty = 0;
            __syncthreads();
            for (int64_t j = j0 + threadIdx.x; j < my_tiles && j < j0 + DIRTY_MAX; j += blockDim.x) {
                const int64_t t = own_tile(j);
                // tiles whose candidates phase R handled last round take them back
                bool d = round == 0 || t == s_win_tile || (round > 1 && ld_cg(&a.t_refit[t]) == (int32_t)(round - 2));
                if (!d && last.dest == TIO_DEST_SSD) {
                    // an SSD commit changes this tile only through the refits it queued
                    d = ld_cg(&a.t_refit[t]) == (int32_t)(round - 1);
                } else if (!d && last.dest) {
                    const int64_t lo = __ldg(&a.t_lo[t]), hi = __ldg(&a.t_hi[t]);
                    d = spans_hit(lo, hi, last.off_s, last.off_e, last.nb) ||
                        spans_hit(lo, hi, last.pre_s, last.pre_e, last.nb) ||
                        (last.dest == TIO_DEST_CPU && last.occ_s <= hi && last.occ_e > lo);
                }
                if (!d && round > 0 && s_flip[0] > 0) {
                    const int64_t fl = s_flip[1], fh = s_flip[2];
                    const int32_t alo = __ldg(&a.t_ka_lo[t]), ahi = __ldg(&a.t_ka_hi[t]);
                    const int32_t blo = __ldg(&a.t_kb_lo[t]), bhi = __ldg(&a.t_kb_hi[t]);
                    d = (alo <= ahi && alo <= fh && fl <= ahi) || (blo <= bhi && blo <= fh && fl <= bhi);
                }
                if (d) s_dirty[atomicAdd(&s_ndirty, 1)] = (int32_t)t;
            }
            __syncthreads();
            const int nd = s_ndirty;
            if (nd) any_dirty = true;
            PROF(if (nd && threadIdx.x == 0) atomic_add_i64(&a.scalars[PS_DBG + 8], nd));
            PROF(if (nd && threadIdx.x == 0)       // the most dirty tiles any block had this round
                     atomicMax(reinterpret_cast<long long *>(&a.scalars[PS_DBG + 14]), (long long)nd));
            // one warp per dirty tile, one lane per candidate
            for (int di = warp; di < nd; di += nwarps) {
                if (di + nwarps < nd) {
                    // pull the warp's next tile toward L2 while this one is evaluated
                    const int64_t pn = (int64_t)s_dirty[di + nwarps] * TILE + lane;
                    if (pn < a.P) {
                        l2_prefetch(&a.vkey[pn]);
                        l2_prefetch(&a.rng[4 * pn]);
                        if (lane == 0) { l2_prefetch(&a.st[pn]); l2_prefetch(&a.tcand[pn]); }
                    }
                }
                const int64_t t = s_dirty[di];
                const int64_t pos = t * TILE + lane;
                const int64_t c = pos < a.P ? pos : -1;                 // column position
                const int32_t cid = pos < a.P ? (int32_t)__ldg(&a.tcand[pos]) : -1;   // tie-break index
                const int8_t st = c >= 0 ? ld_cg(&a.st[c]) : ST_GONE;
                // issue the loads of the common (unchanged-candidate) path together
                const Key ck = c >= 0 ? kload(&a.vkey[c]) : none;
                const int4 rr = c >= 0 ? __ldcg(reinterpret_cast<const int4 *>(&a.rng[4 * c])) : make_int4(1, 0, 1, 0);
                // queued for a refit by the last commit: phase R owns it this round
                const bool tile_queued = round > 0 && ld_cg(&a.t_refit[t]) == (int32_t)(round - 1);
                const bool qround_skip = tile_queued && c >= 0 && ld_cg(&a.qround[c]) == (int32_t)(round - 1);
                const Key mine = qround_skip ? none : eval_lane(c, cid, st, ck, rr, false);
                if (round == 0) {
                    // hulls of the tile's SSD placements (offload, prefetch); the
                    // refit queueing tests a commit's bookings against them
                    int64_t h0 = INT64_MAX, h1 = INT64_MIN, h2 = INT64_MAX, h3 = INT64_MIN;
                    if (c >= 0) {
                        const int8_t s2 = ld_cg(&a.st[c]);
                        if (!(s2 & ST_GONE) && (s2 & 3) == S_OK) {
                            h0 = ld_cg(&a.place[4 * c]); h1 = h0 + __ldg(&a.c_d[4 * c]);
                            h2 = ld_cg(&a.place[4 * c + 1]); h3 = h2 + __ldg(&a.c_d[4 * c + 1]);
                        }
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        h0 = min(h0, (int64_t)__shfl_xor_sync(0xffffffffu, h0, o));
                        h1 = max(h1, (int64_t)__shfl_xor_sync(0xffffffffu, h1, o));
                        h2 = min(h2, (int64_t)__shfl_xor_sync(0xffffffffu, h2, o));
                        h3 = max(h3, (int64_t)__shfl_xor_sync(0xffffffffu, h3, o));
                    }
                    if (lane == 0) {
                        a.t_hull[4 * t] = h0; a.t_hull[4 * t + 1] = h1;
                        a.t_hull[4 * t + 2] = h2; a.t_hull[4 * t + 3] = h3;
                    }
                }
                const Key tk = warp_best(mine);
                if (lane == 0) a.tile_best[t] = tk;
                __syncwarp();
            }
            __syncthreads();
        }
        SUB(0);
        TICK(1);
        // block best over this block's tiles and its refit keys (unchanged when
        // no tile was dirty and no refit ran here this round or the last)
        __syncthreads();
        bool refits_here = false;
        for (int q = 0; q < nwarps; ++q) refits_here |= (s_rbest[q].blo | s_rbest[q].bhi) != 0;
        if (any_dirty) {
            // best over the own tiles, kept for the rounds where only refit
            // keys change the block best
            Key mine = none;
            for (int64_t j = threadIdx.x; j < my_tiles; j += blockDim.x) {
                const Key o = a.tile_best[own_tile(j)];
                if (kbetter(o, mine)) mine = o;
            }
            const Key tm = block_best(mine, sm_key);
            if (threadIdx.x == 0) s_tmax = tm;
            __syncthreads();
        }
        if (any_dirty || refits_here || s_prev_refit || round == 0) {
            if (warp == 0) {
                Key k = lane < nwarps ? s_rbest[lane] : (lane == nwarps ? s_tmax : none);
                k = warp_best(k);
                if (lane == 0) a.blk_best[b] = k;
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) s_prev_refit = refits_here;
        SUB(5);
        PROF(if (threadIdx.x == 0 && gtime() - te0 > 15000) {
            for (int q = 0; q < 6; ++q) slow[q] += sub[q];
            slow[6] += 1;
        });
        PROF(if (threadIdx.x == 0) atomicMax(reinterpret_cast<long long *>(&a.scalars[PS_DBG + 15]),
                                             (long long)(gtime() - te0)));
        TICK(2);
        // ---- the round's winner: the last block to arrive reduces the block
        // bests (one block instead of every block re-reading all of them),
        // exchanges its rank's best with the other ranks' (sharded planning),
        // and publishes the winner; the others wait for it.  This replaces
        // the first grid barrier.
        round_winner(a, round, G, sm_key, &s_win);
        TICK(3);
        PROF(if (tb) {
            a.scalars[PS_DBG + 10] += ld_cg(&a.scalars[PS_DBG + 15]);
            a.scalars[PS_DBG + 15] = 0;
            a.scalars[PS_DBG + 13] += ld_cg(&a.scalars[PS_DBG + 14]);
            a.scalars[PS_DBG + 14] = 0;
        })
        if (b == 0 && threadIdx.x == 0) a.scalars[PS_ROUNDS] = round + 1;
        WinInfo w;
        {
            const WinMsg wm = s_win;
            w.blo = wm.k.blo; w.bhi = wm.k.bhi; w.cost = wm.k.cost;
            w.idx = (w.blo | w.bhi) != 0 ? (int64_t)(((uint64_t)wm.k.meta >> 2) & 0x7fffffffu) : 0;   // column
            w.dest = wm.k.meta & 3;
            w.size = wm.size;
            w.off_s = wm.off_s; w.off_e = wm.off_e; w.pre_s = wm.pre_s; w.pre_e = wm.pre_e;
            for (int q = 0; q < 4; ++q) w.r[q] = wm.r[q];
        }
        TICK(4);
        if ((w.blo | w.bhi) == 0) break;  // planner.py:311-312 no viable candidate
        const int q0 = w.dest == TIO_DEST_SSD ? 0 : 2;
        // new bookings, sorted: (-period, 0, +period)
        int64_t ns[2][3], ne[2][3];
        {
            int64_t sh[3] = {-period, 0, period};
            int k = 0;
            for (int j = 0; j < 3; ++j) {
                if (nb == 1 && j != 1) continue;
                ns[0][k] = w.off_s + sh[j]; ne[0][k] = w.off_e + sh[j];
                ns[1][k] = w.pre_s + sh[j]; ne[1][k] = w.pre_e + sh[j];
                ++k;
            }
        }
        // queue the SSD refits this commit causes: own tiles whose span meets
        // the new bookings, candidates whose cached placement overlaps them
        if (w.dest == TIO_DEST_SSD) {
            const int qn = (int)(round & 1);
            for (int64_t j0 = 0; j0 < my_tiles; j0 += DIRTY_MAX) {
                if (threadIdx.x == 0) s_ndirty = 0;
                __syncthreads();
                for (int64_t j = j0 + threadIdx.x; j < my_tiles && j < j0 + DIRTY_MAX; j += blockDim.x) {
                    const int64_t t = own_tile(j);
                    const longlong2 h01 = __ldcg(reinterpret_cast<const longlong2 *>(a.t_hull + 4 * t));
                    const longlong2 h23 = __ldcg(reinterpret_cast<const longlong2 *>(a.t_hull + 4 * t + 2));
                    if (spans_hit(h01.x, h01.y, ns[0], ne[0], nb) || spans_hit(h23.x, h23.y, ns[1], ne[1], nb))
                        s_dirty[atomicAdd(&s_ndirty, 1)] = (int32_t)t;
                }
                __syncthreads();
                const int nd = s_ndirty;
                for (int64_t i = threadIdx.x; i < (int64_t)nd * TILE; i += blockDim.x) {
                    const int64_t t = s_dirty[i / TILE];
                    const int64_t c = t * TILE + (i % TILE);
                    if (c >= a.P || c == w.idx) continue;
                    const int8_t sc = ld_cg(&a.st[c]);
                    const longlong2 pl = __ldcg(reinterpret_cast<const longlong2 *>(&a.place[4 * c]));
                    const longlong2 dd = __ldg(reinterpret_cast<const longlong2 *>(&a.c_d[4 * c]));
                    if ((sc & ST_GONE) || (sc & 3) != S_OK) continue;
                    if (overlaps(pl.x, dd.x, ns[0], ne[0], nb) || overlaps(pl.y, dd.y, ns[1], ne[1], nb)) {
                        const unsigned long long k =
                            atomicAdd(reinterpret_cast<unsigned long long *>(&a.scalars[PS_RQ + qn]), 1ull);
                        a.rq[qn][k] = c;
                        a.qround[c] = (int32_t)round;
                        a.t_refit[t] = (int32_t)round;
                    }
                }
                __syncthreads();
            }
        }
        // the queue phase R consumed this round is free again
        if (b == 0 && threadIdx.x == 0 && round > 0) a.scalars[PS_RQ + (int)((round - 1) & 1)] = 0;
        // merge the bookings into the other buffer of both channels (all blocks)
        for (int side = 0; side < 2; ++side) {
            const int q = q0 + side;
            const int64_t n = ch_n[q];
            const int64_t *os = a.ch_s[q][ch_par[q]], *oe = a.ch_e[q][ch_par[q]];
            int64_t *ds = a.ch_s[q][ch_par[q] ^ 1], *de = a.ch_e[q][ch_par[q] ^ 1];
            for (int64_t i = (int64_t)b * blockDim.x + threadIdx.x; i <= n; i += (int64_t)G * blockDim.x) {
                int64_t si = i < n ? ld_cg(os + i) : 0, ei = i < n ? ld_cg(oe + i) : 0;
                int64_t sprev = i > 0 ? ld_cg(os + i - 1) : 0, eprev = i > 0 ? ld_cg(oe + i - 1) : 0;
                int64_t cnt = 0;
                for (int j = 0; j < nb; ++j) {
                    const int64_t js = ns[side][j], je = ne[side][j];
                    bool after_prev = i == 0 || sprev < js;
                    bool before_cur = i == n || js < si;
                    if (after_prev && before_cur) {
                        ds[i + j] = js; de[i + j] = je;
                        if ((i > 0 && eprev > js) || (i < n && je > si))
                            a.scalars[PS_INVARIANT] = 1;   // App. A-9 disjointness violated
                    }
                    if (i < n && js < si) ++cnt;
                }
                if (i < n) { ds[i + cnt] = si; de[i + cnt] = ei; }
            }
        }
        TICK(5);
        // residual update on this block's kernel chunk (planner.py:322-324)
        {
            int32_t flips = 0;
            int64_t kmin = INT64_MAX, kmax = -1;     // this thread's flipped kernels
            int64_t *fs = flip + 3 * (round % 3);
            for (int rq = 0; rq < 4; rq += 2) {
                int64_t lo = w.r[rq], hi = w.r[rq + 1];
                if (lo > hi) continue;
                if (lo < x0) lo = x0;
                if (hi > x1 - 1) hi = x1 - 1;
                if (hi > N - 1) hi = N - 1;
                // 4 kernels per thread per step, loads issued together, the
                // next step's loads in flight before this step's stores
                const int64_t stp = 4 * (int64_t)blockDim.x;
                int64_t ovn[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int64_t k = lo + threadIdx.x + (int64_t)u * blockDim.x;
                    ovn[u] = k <= hi ? ld_cg(&a.resid[k]) : 0;
                }
                for (int64_t k0 = lo + threadIdx.x; k0 <= hi; k0 += stp) {
                    int64_t ov[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) ov[u] = ovn[u];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int64_t k = k0 + stp + (int64_t)u * blockDim.x;
                        ovn[u] = k <= hi ? ld_cg(&a.resid[k]) : 0;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int64_t k = k0 + (int64_t)u * blockDim.x;
                        if (k > hi) break;
                        const int64_t nw = ov[u] - w.size;
                        a.resid[k] = nw;
                        if (ov[u] > cap && nw <= cap) {
                            ++flips;
                            kmin = k < kmin ? k : kmin;
                            kmax = k > kmax ? k : kmax;
                        }
                    }
                }
            }
            if (flips) {
                atomicMin(reinterpret_cast<unsigned long long *>(&s_fmin), (unsigned long long)kmin);
                atomicMax(reinterpret_cast<long long *>(&s_fmax), (long long)kmax);
            }
            int32_t tf = block_sum<int32_t>(flips, reinterpret_cast<int32_t *>(sm_scan));
            __syncthreads();
            if (tf) {
                const int64_t fmin = s_fmin;
                rebuild_chunk(fmin);             // only the prefix from the first flip changes
                if (threadIdx.x == 0) {
                    atomic_add_i64(&a.scalars[PS_CRIT], -(int64_t)tf);
                    atomic_add_i64(fs, (int64_t)tf);
                    atomicMin(reinterpret_cast<unsigned long long *>(fs + 1), (unsigned long long)fmin);
                    atomicMax(reinterpret_cast<long long *>(fs + 2), (long long)s_fmax);
                }
            }
        }
        TICK(6);
        // block 0: commit record, host occupancy, mark the winner gone
        if (b == 0 && threadIdx.x == 0) {
            int64_t j = a.scalars[PS_COMMITS];
            tio_commit cm;
            cm.tensor_id = a.c_tid[w.idx];
            cm.tensor_pos = a.c_tpos[w.idx];
            cm.start_kernel = a.c_sk[w.idx];
            cm.end_kernel = a.c_ek[w.idx];
            cm.wraps = a.c_wraps[w.idx];
            cm.destination = w.dest;
            cm.off_start = w.off_s; cm.off_end = w.off_e;
            cm.pre_start = w.pre_s; cm.pre_end = w.pre_e;
            cm.benefit_lo = w.blo;
            cm.benefit_hi = w.bhi;
            cm.cost = w.cost;
            cm.rel0_lo = w.r[0]; cm.rel0_hi = w.r[1]; cm.rel1_lo = w.r[2]; cm.rel1_hi = w.r[3];
            a.commits[j] = cm;
            a.scalars[PS_COMMITS] = j + 1;
            a.st[w.idx] = (int8_t)(ld_cg(&a.st[w.idx]) | ST_GONE);
            if (w.dest == TIO_DEST_CPU) {
                int64_t h = s_nocc;
                a.occ_s[h] = w.off_e; a.occ_e[h] = w.pre_s; a.occ_size[h] = w.size;
                a.scalars[PS_OCC] = h + 1;
            }
        }
        __syncthreads();
        if (b == 0 && w.dest == TIO_DEST_CPU) {
            hx_insert(a, s_nocc, w.off_e, w.pre_s, w.size, reinterpret_cast<int64_t *>(sm_scan));
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            last.dest = w.dest;
            for (int j = 0; j < nb; ++j) {
                last.off_s[j] = ns[0][j]; last.off_e[j] = ne[0][j];
                last.pre_s[j] = ns[1][j]; last.pre_e[j] = ne[1][j];
            }
            last.occ_s = w.off_e; last.occ_e = w.pre_s;
            if (w.dest == TIO_DEST_CPU) s_nocc += 1;
            ch_n[q0] += nb; ch_n[q0 + 1] += nb;
            ch_par[q0] ^= 1; ch_par[q0 + 1] ^= 1;
            s_win_tile = w.idx / TILE;
        }
        grid_barrier(a.bar, G);
        TICK(7);
    }
    PROF(if (tb) for (int q = 0; q < 8; ++q) a.scalars[PS_DBG + q] = dbg[q]);
    PROF(if (tb) { a.scalars[PS_DBG + 11] = (int64_t)g_walk_total; a.scalars[PS_DBG + 12] = (int64_t)g_walk_max; });
    PROF(if (tb) printf("[plan-profile] warp fit walks: %llu walks, %llu iterations (32 bookings each), longest %llu\n",
                        g_wwalk_n, g_wwalk_total, g_wwalk_max));
    PROF(if (threadIdx.x == 0 && a.prof) for (int q = 0; q < 7; ++q) a.prof[8 * b + q] = slow[q]);
#undef TICK
#undef PROF
#undef SUB
}

#ifndef TIO_PLAN_MINB
#define TIO_PLAN_MINB 2       // blocks per SM the register allocation must allow (build knob)
#endif
#ifndef TIO_PLAN_MAX_PER_SM
#define TIO_PLAN_MAX_PER_SM 2 // resident planner blocks per SM used (build knob)
#endif
__global__ void __launch_bounds__(PLAN_THREADS, TIO_PLAN_MINB)
plan_loop_kernel(PlanArgs a) {
    plan_loop_body(a, (int)gridDim.x, (int)blockIdx.x);
}

// The wide form: registers capped for 3 resident blocks per SM (80 registers,
// a small spill to L1) — 1.5x the warps for the dirty-tile and refit phases.
// Measured (tools/micro/plvar.sh): C3 (150K tiles) 59.2 -> 55.9 us/round,
// C2 (15K tiles) 22.6 -> 23.9 (more blocks in every barrier and reduction
// for little phase-E work), so it is chosen by tile count.
__global__ void __launch_bounds__(PLAN_THREADS, 3)
plan_loop_kernel_wide(PlanArgs a) {
    plan_loop_body(a, (int)gridDim.x, (int)blockIdx.x);
}

// Virtual ranks on one GPU (the sharded protocol's check): R planner
// instances in ONE cooperative grid, blocks [r Gr, (r + 1) Gr) run rank r
// with its own arguments (staged in shared memory).  Separate cooperative
// launches are not co-scheduled by the driver — a rank's grid would wait for
// the other's to finish while that one waits for its messages.
__global__ void __launch_bounds__(PLAN_THREADS, TIO_PLAN_MINB)
plan_loop_kernel_multi(const PlanArgs *args, int Gr) {
    __shared__ __align__(16) PlanArgs sa;
    const int r = (int)blockIdx.x / Gr;
    {
        const uint32_t *src = reinterpret_cast<const uint32_t *>(args + r);
        uint32_t *dst = reinterpret_cast<uint32_t *>(&sa);
        for (int i = threadIdx.x; i < (int)(sizeof(PlanArgs) / 4); i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    plan_loop_body(sa, Gr, (int)blockIdx.x % Gr);
}

bool plan_loop_wide(int64_t ntiles) {
    static int64_t thresh = -1;
    if (thresh < 0) {
        const char *e = getenv("TIO_PLAN_WIDE_TILES");
        thresh = e ? atoll(e) : 60000;
    }
    return thresh > 0 && ntiles >= thresh;
}

int plan_loop_grid(int *blocks, bool wide) {
    static int cached[2] = {0, 0};
    int &c = cached[wide ? 1 : 0];
    if (!c) {
        int dev = 0, sms = 0, per_sm = 0;
        const void *fn = wide ? (const void *)plan_loop_kernel_wide : (const void *)plan_loop_kernel;
        TIO_CUDA(cudaGetDevice(&dev));
        TIO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        TIO_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PLAN_DYN_SMEM));
        TIO_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, PLAN_THREADS, PLAN_DYN_SMEM));
        if (per_sm < 1) return fail(TIO_ERR_CUDA, "planner kernel cannot be resident");
        const int cap = wide ? 3 : TIO_PLAN_MAX_PER_SM;
        c = sms * (per_sm < cap ? per_sm : cap);
        if (c > MAXG) c = MAXG;
    }
    *blocks = c;
    return TIO_OK;
}

int plan_loop_multi_grid(int *blocks) {
    static int cached = 0;
    if (!cached) {
        int dev = 0, sms = 0, per_sm = 0;
        TIO_CUDA(cudaGetDevice(&dev));
        TIO_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        TIO_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, plan_loop_kernel_multi, PLAN_THREADS,
                                                               PLAN_DYN_SMEM));
        if (per_sm < 1) return fail(TIO_ERR_CUDA, "multi-rank planner kernel cannot be resident");
        cached = sms * (per_sm < TIO_PLAN_MAX_PER_SM ? per_sm : TIO_PLAN_MAX_PER_SM);
        if (cached > MAXG) cached = MAXG;
    }
    *blocks = cached;
    return TIO_OK;
}

int launch_plan_loop_multi(const PlanArgs *dev_args, int nranks, int blocks_per_rank, cudaStream_t stream) {
    int Gr = blocks_per_rank;
    void *params[] = {const_cast<PlanArgs **>(&dev_args), &Gr};
    TIO_CUDA(cudaLaunchCooperativeKernel((const void *)plan_loop_kernel_multi, dim3(nranks * blocks_per_rank),
                                         dim3(PLAN_THREADS), params, PLAN_DYN_SMEM, stream));
    count_launch();
    return TIO_OK;
}

int launch_plan_loop(const PlanArgs &args, int blocks, cudaStream_t stream, bool wide) {
    void *params[] = {const_cast<PlanArgs *>(&args)};
    TIO_CUDA(cudaLaunchCooperativeKernel(wide ? (const void *)plan_loop_kernel_wide : (const void *)plan_loop_kernel,
                                         dim3(blocks), dim3(PLAN_THREADS),
                                         params, PLAN_DYN_SMEM, stream));
    count_launch();
    return TIO_OK;
}

}  // namespace tio
