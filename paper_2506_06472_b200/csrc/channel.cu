// channel.cu — host-side serial migration channels and the per-candidate
// planning helpers over them: the objects behind the Python API's
// BandwidthChannel (reference bandwidth.py:47-164), candidate_window
// (planner.py:147-176), _host_peak_occupancy (:179-186) and
// candidate_benefit (:232-262).  These serve callers that inspect one
// candidate at a time (the reference's public helpers and its tests); the
// planner itself keeps its channels on the device (planner.cu, sorted
// interval arrays with index hints).  Host code only: no device memory.
//
// A channel is a vector of bookings kept sorted by start; bookings with equal
// starts stay in insertion order (the reference inserts with
// bisect.insort_right).  A booking made with a period also books its two
// images one period earlier and later (shadows), released with it.  The walks
// are the exact first-fit / last-fit of the reference over the whole vector:
// records (`tio_channel_record`) may overlap other bookings, so no prefix may
// be skipped by a search on end times.
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"

using namespace tio;

struct tio_channel {
    struct Res {
        int64_t start, end, tensor, id, owner;
        int8_t shadow;
    };
    RateCode rc{};
    int64_t period = 0;           // 0: no periodic images
    std::vector<Res> v;
    int64_t next_id = 1;

    void insert(const Res &r) {
        auto it = std::upper_bound(v.begin(), v.end(), r.start,
                                   [](int64_t s, const Res &x) { return s < x.start; });
        v.insert(it, r);
    }
    int64_t book(int64_t s, int64_t e, int64_t tensor) {
        const int64_t id = next_id++;
        insert({s, e, tensor, id, id, 0});
        if (period > 0) {
            insert({s - period, e - period, tensor, next_id++, id, 1});
            insert({s + period, e + period, tensor, next_id++, id, 1});
        }
        return id;
    }
    int duration(int64_t nbytes, int64_t *d) const {
        if (nbytes < 0) return fail(TIO_ERR_INVALID, "negative transfer size");
        *d = duration_of(rc, nbytes);
        if (*d <= 0) return fail(TIO_ERR_INVALID, "reserve requires a non-empty transfer");
        return TIO_OK;
    }
    // first fit at or after `ready`
    int64_t earliest(int64_t ready, int64_t d) const {
        int64_t t = ready;
        for (const Res &r : v) {
            if (r.start >= t + d) break;
            if (r.end > t) t = r.end;
        }
        return t;
    }
    // last fit ending at or before `deadline`, starting at or after
    // `not_before`; false when there is none
    bool latest(int64_t deadline, int64_t not_before, int64_t d, int64_t *out) const {
        int64_t s = deadline - d;
        for (auto it = v.rbegin(); it != v.rend(); ++it) {
            if (s < not_before) return false;
            if (it->start >= s + d) continue;
            if (it->end <= s) break;
            s = it->start - d;
        }
        if (s < not_before) return false;
        *out = s;
        return true;
    }
    void release(int64_t id) {
        v.erase(std::remove_if(v.begin(), v.end(), [id](const Res &r) { return r.owner == id; }), v.end());
    }
};

extern "C" {

int tio_channel_create(double rate, int64_t period, tio_channel **out) {
    if (!out) return fail(TIO_ERR_INVALID, "null argument");
    *out = nullptr;
    RateCode rc;
    TIO_TRY(decode_rate(rate, &rc));
    tio_channel *c = new tio_channel();
    c->rc = rc;
    c->period = period > 0 ? period : 0;
    *out = c;
    return TIO_OK;
}

int tio_channel_destroy(tio_channel *c) {
    delete c;
    return TIO_OK;
}

int tio_channel_reserve_earliest(tio_channel *c, int64_t ready, int64_t nbytes, int64_t tensor_id, int64_t *id,
                                 int64_t *start, int64_t *end) {
    if (!c || !id || !start || !end) return fail(TIO_ERR_INVALID, "null argument");
    int64_t d = 0;
    TIO_TRY(c->duration(nbytes, &d));
    const int64_t t = c->earliest(ready, d);
    *id = c->book(t, t + d, tensor_id);
    *start = t;
    *end = t + d;
    return TIO_OK;
}

int tio_channel_reserve_latest(tio_channel *c, int64_t deadline, int64_t not_before, int64_t nbytes,
                               int64_t tensor_id, int32_t *found, int64_t *id, int64_t *start, int64_t *end) {
    if (!c || !found || !id || !start || !end) return fail(TIO_ERR_INVALID, "null argument");
    int64_t d = 0;
    TIO_TRY(c->duration(nbytes, &d));
    int64_t s = 0;
    *found = c->latest(deadline, not_before, d, &s) ? 1 : 0;
    if (*found) {
        *id = c->book(s, s + d, tensor_id);
        *start = s;
        *end = s + d;
    }
    return TIO_OK;
}

int tio_channel_record(tio_channel *c, int64_t start, int64_t end, int64_t tensor_id, int32_t shadow,
                       int64_t *id) {
    if (!c || !id) return fail(TIO_ERR_INVALID, "null argument");
    const int64_t k = c->next_id++;
    c->insert({start, end, tensor_id, k, k, (int8_t)(shadow ? 1 : 0)});
    *id = k;
    return TIO_OK;
}

int tio_channel_release(tio_channel *c, int64_t id) {
    if (!c) return fail(TIO_ERR_INVALID, "null argument");
    c->release(id);
    return TIO_OK;
}

int tio_channel_size(const tio_channel *c, int64_t *n) {
    if (!c || !n) return fail(TIO_ERR_INVALID, "null argument");
    *n = (int64_t)c->v.size();
    return TIO_OK;
}

int tio_channel_copy(const tio_channel *c, int64_t *start, int64_t *end, int64_t *tensor, int64_t *id,
                     int64_t *owner, int8_t *shadow) {
    if (!c) return fail(TIO_ERR_INVALID, "null argument");
    for (size_t i = 0; i < c->v.size(); ++i) {
        const auto &r = c->v[i];
        if (start) start[i] = r.start;
        if (end) end[i] = r.end;
        if (tensor) tensor[i] = r.tensor;
        if (id) id[i] = r.id;
        if (owner) owner[i] = r.owner;
        if (shadow) shadow[i] = r.shadow;
    }
    return TIO_OK;
}

int tio_channel_busy(const tio_channel *c, int64_t w0, int64_t w1, int64_t *busy) {
    if (!c || !busy) return fail(TIO_ERR_INVALID, "null argument");
    if (w0 >= w1) return fail(TIO_ERR_INVALID, "window must be non-empty");
    int64_t b = 0;
    for (const auto &r : c->v) {
        if (r.shadow) continue;
        const int64_t lo = r.start > w0 ? r.start : w0, hi = r.end < w1 ? r.end : w1;
        if (hi > lo) b += hi - lo;
    }
    *busy = b;
    return TIO_OK;
}

// candidate_window (planner.py:147-176) on one channel pair: reject when a
// direction alone takes longer than the iteration; earliest offload from
// `ready`, latest prefetch before `deadline` not before the offload's end;
// feasible iff the offload ends strictly before the prefetch starts, else
// both bookings are rolled back.  On success both stay booked.
int tio_candidate_window(tio_channel *off, tio_channel *pre, int64_t ready, int64_t deadline, int64_t nbytes,
                         int64_t iteration, int64_t tensor_id, int32_t *ok, int64_t *off_id, int64_t *off_end,
                         int64_t *pre_id, int64_t *pre_start) {
    if (!off || !pre || !ok || !off_id || !off_end || !pre_id || !pre_start) return fail(TIO_ERR_INVALID, "null argument");
    *ok = 0;
    if (nbytes < 0) return fail(TIO_ERR_INVALID, "negative transfer size");
    if (duration_of(off->rc, nbytes) > iteration || duration_of(pre->rc, nbytes) > iteration) return TIO_OK;
    int64_t oid, os, oe;
    TIO_TRY(tio_channel_reserve_earliest(off, ready, nbytes, tensor_id, &oid, &os, &oe));
    int32_t found = 0;
    int64_t pid = 0, ps = 0, pe = 0;
    TIO_TRY(tio_channel_reserve_latest(pre, deadline, oe, nbytes, tensor_id, &found, &pid, &ps, &pe));
    if (!found || !(oe < ps)) {
        if (found) pre->release(pid);
        off->release(oid);
        return TIO_OK;
    }
    *ok = 1;
    *off_id = oid;
    *off_end = oe;
    *pre_id = pid;
    *pre_start = ps;
    return TIO_OK;
}

// _host_peak_occupancy (planner.py:179-186): the largest total size of
// occupancy intervals [s, e) live at a point of {lo} u {starts in [lo, hi]}
int tio_host_peak_occupancy(const int64_t *s, const int64_t *e, const int64_t *sz, int64_t n, int64_t lo,
                            int64_t hi, int64_t *out) {
    if (!out || (n > 0 && (!s || !e || !sz))) return fail(TIO_ERR_INVALID, "null argument");
    int64_t peak = 0;
    for (int64_t pi = -1; pi < n; ++pi) {
        const int64_t p = pi < 0 ? lo : s[pi];
        if (pi >= 0 && !(lo <= p && p <= hi)) continue;
        int64_t sum = 0;
        for (int64_t j = 0; j < n; ++j)
            if (s[j] <= p && p < e[j]) sum += sz[j];
        if (sum > peak) peak = sum;
    }
    *out = peak;
    return TIO_OK;
}

// candidate_benefit (planner.py:232-262): kernels of the period's range(s)
// fully inside [lo, hi] (wrap periods: last+1..N-1, then 0..first-1 shifted
// by the iteration), the over-capacity ones among them (residual > capacity),
// and size x the sum of their durations as a 128-bit value.  critical: [N]
// output mask (may be NULL).
int tio_candidate_benefit(const int64_t *starts, const int64_t *dur, const int64_t *residual, int64_t N,
                          int64_t capacity, int32_t wraps, int64_t start_kernel, int64_t end_kernel, int64_t first,
                          int64_t last, int64_t lo, int64_t hi, int64_t size, uint64_t *benefit_lo,
                          uint64_t *benefit_hi, int8_t *critical) {
    if (!starts || !dur || !residual || !benefit_lo || !benefit_hi) return fail(TIO_ERR_INVALID, "null argument");
    if (critical) memset(critical, 0, (size_t)(N > 0 ? N : 0));
    const int64_t iteration = N > 0 ? starts[N] : 0;
    struct Span { int64_t a, b, sh; } spans[2];
    int ns = 0;
    if (!wraps) spans[ns++] = {start_kernel, end_kernel + 1, 0};
    else {
        spans[ns++] = {last + 1, N, 0};
        spans[ns++] = {0, first, iteration};
    }
    unsigned __int128 total = 0;
    for (int q = 0; q < ns; ++q)
        for (int64_t k = spans[q].a < 0 ? 0 : spans[q].a; k < spans[q].b && k < N; ++k) {
            if (!(starts[k] + spans[q].sh >= lo && starts[k + 1] + spans[q].sh <= hi)) continue;
            if (residual[k] > capacity) {
                total += (unsigned __int128)dur[k];
                if (critical) critical[k] = 1;
            }
        }
    const unsigned __int128 b = total * (unsigned __int128)(uint64_t)size;
    *benefit_lo = (uint64_t)b;
    *benefit_hi = (uint64_t)(b >> 64);
    return TIO_OK;
}

}  // extern "C"
