// roofline.cu — the bandwidth sweep of the reference's roofline study
// (roofline.py:39-125), host C++ over the host trace columns.
//
// Policy (roofline.py:1-12): under memory pressure every inactive period is
// migrated; offloads leave on one serial channel in (ready kernel, tensor id,
// end kernel) order, prefetches ride the serial return channel in (need
// kernel, tensor id, start kernel) order once their offload has landed, and a
// kernel waits for its own prefetches.  The two processing orders do not
// depend on the bandwidth, so they are built once and every bandwidth of the
// sweep is one max/+ pass over them (the passes run on separate threads).
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "common.cuh"

namespace tio {
namespace {

struct RPeriod {
    int64_t tid, size;
    int64_t start, end;     // period kernels (compute_inactive_periods, analysis.py:58-83)
    int64_t ready, need;    // roofline.py:50-59
};

}  // namespace
}  // namespace tio

extern "C" int tio_roofline(const tio_trace_desc *d, int64_t capacity, const double *bandwidth, int64_t num_bandwidths,
                            int64_t *total_us, tio_roofline_info *info) {
    using namespace tio;
    if (!d || !info || (num_bandwidths > 0 && (!bandwidth || !total_us))) return fail(TIO_ERR_INVALID, "null argument");
    const int64_t N = d->num_kernels, T = d->num_tensors;
    for (int64_t t = 0; t < T; ++t) {
        if (d->access_ptr[t + 1] <= d->access_ptr[t]) return fail(TIO_ERR_INVALID, "tensor without accesses");
        for (int64_t j = d->access_ptr[t]; j < d->access_ptr[t + 1]; ++j)
            if (d->accesses[j] < 0 || d->accesses[j] >= N) return fail(TIO_ERR_INVALID, "access out of range");
    }
    // iteration length and memory-timeline peak (trace.py:103-107, analysis.py:97-108)
    int64_t ideal = 0;
    for (int64_t k = 0; k < N; ++k) ideal += d->duration_us[k];
    std::vector<int64_t> diff(N + 1, 0);
    int64_t glob = 0;
    for (int64_t t = 0; t < T; ++t) {
        const int32_t *a = d->accesses + d->access_ptr[t];
        const int64_t n = d->access_ptr[t + 1] - d->access_ptr[t];
        if (d->kind[t] == 1) { glob += d->size_bytes[t]; continue; }
        diff[a[0]] += d->size_bytes[t];
        diff[a[n - 1] + 1] -= d->size_bytes[t];
    }
    int64_t run = 0, peak = 0;
    for (int64_t k = 0; k < N; ++k) {
        run += diff[k];
        peak = std::max(peak, glob + run);
    }
    // periods, with their ready / need kernels
    std::vector<RPeriod> ps;
    int64_t num_periods = 0, max_size = 0;
    for (int64_t t = 0; t < T; ++t) {
        const int32_t *a = d->accesses + d->access_ptr[t];
        const int64_t n = d->access_ptr[t + 1] - d->access_ptr[t];
        const int64_t sz = d->size_bytes[t];
        auto add = [&](int64_t s, int64_t e, bool wraps) {
            ++num_periods;
            max_size = std::max(max_size, sz);
            const int64_t ready = wraps ? a[n - 1] + 1 : s;
            const int64_t need = wraps ? N + a[0] : e + 1;
            if (ready < N) ps.push_back(RPeriod{d->tensor_id[t], sz, s, e, ready, need});
        };
        for (int64_t j = 0; j + 1 < n; ++j)
            if (a[j + 1] - a[j] > 1) add(a[j] + 1, a[j + 1] - 1, false);
        if (d->kind[t] == 1 && (N - 1 - a[n - 1]) + a[0] > 0)
            add((a[n - 1] + 1) % N, ((a[0] - 1) % N + N) % N, true);
    }
    memset(info, 0, sizeof(*info));
    info->ideal_us = ideal;
    info->peak_bytes = peak;
    info->pressured = peak > capacity ? 1 : 0;
    info->num_periods = num_periods;
    info->max_period_bytes = num_periods ? max_size : 1;
    if (num_bandwidths <= 0) return TIO_OK;

    std::vector<RateCode> rc((size_t)num_bandwidths);
    for (int64_t i = 0; i < num_bandwidths; ++i) TIO_TRY(decode_rate(bandwidth[i], &rc[i]));
    if (!info->pressured || ideal == 0) {
        for (int64_t i = 0; i < num_bandwidths; ++i) total_us[i] = ideal;
        return TIO_OK;
    }
    const int64_t P = (int64_t)ps.size();
    std::vector<int64_t> off(P), pre(P);
    for (int64_t i = 0; i < P; ++i) off[i] = pre[i] = i;
    std::sort(off.begin(), off.end(), [&](int64_t x, int64_t y) {
        const RPeriod &a = ps[x], &b = ps[y];
        if (a.ready != b.ready) return a.ready < b.ready;
        if (a.tid != b.tid) return a.tid < b.tid;
        return a.end < b.end;
    });
    std::sort(pre.begin(), pre.end(), [&](int64_t x, int64_t y) {
        const RPeriod &a = ps[x], &b = ps[y];
        if (a.need != b.need) return a.need < b.need;
        if (a.tid != b.tid) return a.tid < b.tid;
        return a.start < b.start;
    });
    // roofline.py:39-87, one bandwidth
    auto one = [&](int64_t i) {
        std::vector<int64_t> done(P, 0);
        int64_t off_free = 0, pre_free = 0, now = 0;
        int64_t oi = 0, pi = 0;
        for (int64_t k = 0; k < N; ++k) {
            for (; oi < P && ps[off[oi]].ready == k; ++oi) {
                const RPeriod &p = ps[off[oi]];
                off_free = std::max(now, off_free) + duration_of(rc[i], p.size);
                done[off[oi]] = off_free;
            }
            for (; pi < P && ps[pre[pi]].need == k; ++pi) {
                const RPeriod &p = ps[pre[pi]];
                pre_free = std::max(done[pre[pi]], pre_free) + duration_of(rc[i], p.size);
                now = std::max(now, pre_free);
            }
            now += d->duration_us[k];
        }
        total_us[i] = now;
    };
    const int64_t nth = std::min<int64_t>(num_bandwidths, std::max(1u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (int64_t w = 0; w < nth; ++w)
        pool.emplace_back([&, w] {
            for (int64_t i = w; i < num_bandwidths; i += nth) one(i);
        });
    for (auto &th : pool) th.join();
    return TIO_OK;
}
