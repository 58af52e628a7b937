// warp_search.cuh — warp-cooperative searches for the planner's refits.
//
// A refit (a candidate whose cached placement was hit by the last commit) is
// a chain of dependent global loads when one thread does it alone: two
// binary searches over a channel (~17 steps each at 1e5 bookings), the fit
// walks, and two binary searches over the kernel start times (~18 steps each
// at 2.5e5 kernels).  Here a whole warp serves one refit: 32-ary searches
// (ceil(log32 n) dependent steps) and 32-wide fit walks with a ballot.
// Results are identical to the scalar versions in planner.cu
// (bandwidth.py:88-120 reserve_earliest / reserve_latest, planner.py:232-250
// _covered_kernels); all lanes return the same value.
#pragma once
#include <cstdint>
#include "common.cuh"

// walk-length statistics hook (the planner's debug build defines it)
#ifndef WWALK_COUNT
#define WWALK_COUNT(n) do { } while (0)
#endif

namespace tio {

// first index i in [lo, hi) with pred(i) true, for a monotone (false..true)
// predicate; hi if none.  All lanes must call with the same arguments.
template <typename Pred>
__device__ __forceinline__ int64_t warp_lower_bound(int64_t lo, int64_t hi, Pred pred) {
    const int lane = threadIdx.x & 31;
    while (hi - lo > 32) {
        const int64_t step = (hi - lo + 31) / 32;           // 32 chunks of `step`
        const int64_t probe = lo + (int64_t)(lane + 1) * step - 1;   // last index of chunk lane
        const bool t = probe < hi ? pred(probe) : true;
        const unsigned m = __ballot_sync(0xffffffffu, t);
        if (!m) return hi;                                   // predicate false on all of [lo, hi)
        const int c = __ffs(m) - 1;                          // first chunk whose last element is true
        const int64_t nlo = lo + (int64_t)c * step;
        const int64_t nhi = lo + (int64_t)(c + 1) * step;
        lo = nlo;
        hi = nhi < hi ? nhi : hi;
    }
    const int64_t i = lo + lane;
    const bool t = i < hi ? pred(i) : true;
    const unsigned m = __ballot_sync(0xffffffffu, t);
    return m ? lo + (__ffs(m) - 1) : hi;
}

// reserve_earliest (bandwidth.py:88-100) on sorted disjoint [s, e) arrays.
// The first booking that can matter lies in [lo_idx, hi_idx]; *p = index
// where the walk stopped (every booking before it ends at or before the fit).
__device__ __forceinline__ int64_t warp_earliest(const int64_t *cs, const int64_t *ce, int64_t n,
                                                 int64_t ready, int64_t d, int64_t lo_idx, int64_t hi_idx,
                                                 int64_t *p) {
    const int lane = threadIdx.x & 31;
    int64_t i = warp_lower_bound(lo_idx, hi_idx, [&](int64_t j) { return ld_cg(ce + j) > ready; });
    int64_t t = ready;
    int64_t iters = 0;
    while (i < n) {
        ++iters;
        const int64_t j = i + lane;
        const bool in = j < n;
        const int64_t s = in ? ld_cg(cs + j) : INT64_MAX;
        const int64_t e = in ? ld_cg(ce + j) : INT64_MAX;
        // running max of ends before lane j (ends increase: it is the previous end)
        int64_t pe = __shfl_up_sync(0xffffffffu, e, 1);
        int64_t tj = lane == 0 ? t : (pe > t ? pe : t);
        const bool gap = !in || s >= tj + d;
        const unsigned m = __ballot_sync(0xffffffffu, gap);
        if (m) {
            const int f = __ffs(m) - 1;
            *p = i + f;
            WWALK_COUNT(iters);
            return __shfl_sync(0xffffffffu, tj, f);
        }
        const int64_t last_e = __shfl_sync(0xffffffffu, e, 31);
        t = last_e > t ? last_e : t;
        i += 32;
    }
    *p = n;
    return t;
}

// reserve_latest (bandwidth.py:102-120); false = None.
// The first booking at or after the deadline lies in [lo_idx, hi_idx];
// *q = first booking after the fit.
__device__ __forceinline__ bool warp_latest(const int64_t *cs, const int64_t *ce, int64_t n, int64_t deadline,
                                            int64_t not_before, int64_t d, int64_t lo_idx, int64_t hi_idx,
                                            int64_t *out, int64_t *q) {
    const int lane = threadIdx.x & 31;
    // last index with s < deadline = (first index with s >= deadline) - 1
    int64_t i = warp_lower_bound(lo_idx, hi_idx, [&](int64_t j) { return ld_cg(cs + j) >= deadline; }) - 1;
    int64_t start = deadline - d;
    int64_t iters = 0;
    // Walking down from i: every visited booking starts before start + d
    // (sorted, disjoint), so the reference's `continue` branch never fires;
    // a booking either ends at or before `start` (fit) or pushes start to s - d.
    while (i >= 0) {
        ++iters;
        const int64_t j = i - lane;
        const bool in = j >= 0;
        const int64_t s = in ? ld_cg(cs + j) : INT64_MIN;
        const int64_t e = in ? ld_cg(ce + j) : INT64_MIN;
        const int64_t sprev = __shfl_up_sync(0xffffffffu, s, 1);   // booking j+1 (processed before j)
        const int64_t sj = lane == 0 ? start : sprev - d;
        const bool stop = !in || sj < not_before || e <= sj;
        const unsigned m = __ballot_sync(0xffffffffu, stop);
        if (m) {
            const int f = __ffs(m) - 1;
            WWALK_COUNT(iters);
            const int64_t st = __shfl_sync(0xffffffffu, sj, f);
            if (st < not_before) return false;
            *out = st;
            *q = i - f + 1;
            return true;
        }
        start = __shfl_sync(0xffffffffu, s, 31) - d;
        i -= 32;
    }
    if (start < not_before) return false;
    *out = start;
    *q = 0;
    return true;
}

// candidate_window (planner.py:147-176) on one channel pair, warp version of
// fit_pair() in planner.cu (same hints: restart from the cached placement).
__device__ __forceinline__ bool warp_fit_pair(const int64_t *os_, const int64_t *oe_, int64_t on,
                                              const int64_t *ps_, const int64_t *pe_, int64_t pn,
                                              int64_t d_off, int64_t d_pre, int64_t iteration, int64_t hint_off,
                                              int64_t hint_pre_end, int64_t plo, int64_t phi, int64_t qlo,
                                              int64_t qhi, int64_t *off_s, int64_t *pre_s, int64_t *np,
                                              int64_t *nq) {
    if (d_off > iteration || d_pre > iteration) return false;
    const int64_t o = warp_earliest(os_, oe_, on, hint_off, d_off, plo, phi, np);
    const int64_t t_off = o + d_off;
    int64_t f;
    if (!warp_latest(ps_, pe_, pn, hint_pre_end, t_off, d_pre, qlo, qhi, &f, nq)) return false;
    if (!(t_off < f)) return false;
    *off_s = o;
    *pre_s = f;
    return true;
}

// _covered_kernels (planner.py:232-250) as <= 2 kernel ranges, warp version.
__device__ __forceinline__ void warp_covered_ranges(const int64_t *__restrict__ starts, int64_t N, int64_t iteration,
                                                    int wraps, int32_t sk, int32_t ek, int32_t first, int32_t last,
                                                    int64_t lo_t, int64_t hi_t, int32_t r[4]) {
    r[0] = 1; r[1] = 0; r[2] = 1; r[3] = 0;
    auto range = [&](int64_t a, int64_t b, int64_t sh, int32_t &olo, int32_t &ohi) {
        // first k in [a, b] with starts[k] + sh >= lo_t
        const int64_t klo = warp_lower_bound(a, b + 1, [&](int64_t k) { return __ldg(starts + k) + sh >= lo_t; });
        // first k in [klo, b] with starts[k+1] + sh > hi_t  (kernels before it end inside the window)
        const int64_t kend = warp_lower_bound(klo, b + 1, [&](int64_t k) { return __ldg(starts + k + 1) + sh > hi_t; });
        olo = (int32_t)klo;
        ohi = (int32_t)(kend - 1);
    };
    if (!wraps) {
        if (sk <= ek) range(sk, ek, 0, r[0], r[1]);
    } else {
        if (last + 1 <= N - 1) range(last + 1, N - 1, 0, r[0], r[1]);
        if (first - 1 >= 0) range(0, first - 1, iteration, r[2], r[3]);
    }
}

// Refit version of warp_covered_ranges: the window only shrank, so each new
// range lies inside the old one.
__device__ __forceinline__ void warp_covered_ranges_shrunk(const int64_t *__restrict__ starts, int64_t iteration,
                                                           int wraps, int64_t lo_t, int64_t hi_t,
                                                           const int32_t r_old[4], int32_t r[4]) {
    for (int q = 0; q < 4; q += 2) {
        const int64_t a = r_old[q], b = r_old[q + 1];
        if (a > b) { r[q] = r_old[q]; r[q + 1] = r_old[q + 1]; continue; }
        const int64_t sh = (wraps && q == 2) ? iteration : 0;
        const int64_t klo = warp_lower_bound(a, b + 1, [&](int64_t k) { return __ldg(starts + k) + sh >= lo_t; });
        const int64_t kend = warp_lower_bound(klo, b + 1, [&](int64_t k) { return __ldg(starts + k + 1) + sh > hi_t; });
        r[q] = (int32_t)klo;
        r[q + 1] = (int32_t)(kend - 1);
    }
}

}  // namespace tio
