// capi.cu — the C ABI of libtio (include/tio.h): handle management and the
// orchestration of the lifetime / planner kernels on a caller stream.
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstring>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "lifetime.cuh"
#include "planner.cuh"
#include "plan_setup.cuh"
#include "radix_sort.cuh"
#include "scan.cuh"
#include "engine_sched.cuh"

namespace tio {

static thread_local char g_err[1024];
static std::atomic<long long> g_launches{0};

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int fail(int code, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

// Stream-ordered device allocations owned by a handle.
struct Arena {
    std::vector<void *> ptrs;
    cudaStream_t stream = nullptr;
    template <typename T>
    int alloc(T **out, int64_t n) {
        void *p = nullptr;
        size_t bytes = sizeof(T) * (size_t)(n > 0 ? n : 1);
        cudaError_t e = cudaMallocAsync(&p, bytes, stream);
        if (e != cudaSuccess) return fail(TIO_ERR_NOMEM, "cudaMallocAsync(%zu) failed: %s", bytes, cudaGetErrorString(e));
        ptrs.push_back(p);
        *out = static_cast<T *>(p);
        return TIO_OK;
    }
    void release() {
        for (void *p : ptrs) cudaFreeAsync(p, stream);
        ptrs.clear();
    }
};

static int ensure_pool() {
    static bool done = false;
    if (done) return TIO_OK;
    int dev = 0;
    TIO_CUDA(cudaGetDevice(&dev));
    cudaMemPool_t pool;
    TIO_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thresh = UINT64_MAX;  // keep freed blocks for reuse across plans
    TIO_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thresh));
    done = true;
    return TIO_OK;
}

// Decode a rate into the exact integer form used by duration_of.
int decode_rate(double rate, RateCode *rc) {
    memset(rc, 0, sizeof(*rc));
    if (!(rate > 0) || std::isnan(rate) || std::isinf(rate))
        return fail(TIO_ERR_CHANNEL_CONFIG, "rate must be > 0");
    if (rate == std::floor(rate)) {
        if (rate >= 9223372036854775808.0) { rc->huge = 1; rc->num = 1; return TIO_OK; }
        rc->num = (int64_t)rate;
        return TIO_OK;
    }
    int ex = 0;
    double mant = std::frexp(rate, &ex);
    uint64_t m = (uint64_t)std::ldexp(mant, 53);
    int k = 53 - ex;
    while (k > 0 && (m & 1u) == 0) { m >>= 1; --k; }
    // any k is exact: duration_of takes a long-division path past 64 bits
    rc->num = (int64_t)m;
    rc->shift = k;
    return TIO_OK;
}

// period_interior_duration (analysis.py:86-94) of every period: durations
// strictly inside it, from the start times — non-wrap: starts[end + 1] -
// starts[start]; wrap: the tail after the last access plus the head before
// the first (start = (last + 1) mod N, end = (first - 1) mod N, so a start of
// 0 means an empty tail and an end of N - 1 an empty head).
__global__ void k_period_interior(const int64_t *starts, const int32_t *p_start, const int32_t *p_end,
                                  const int8_t *p_wraps, int64_t P, int64_t N, int64_t *out) {
    const int64_t I = starts[N];
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t a = p_start[p], b = p_end[p];
        if (!p_wraps[p]) {
            out[p] = starts[b + 1] - starts[a];
        } else {
            const int64_t tail = a == 0 ? 0 : I - starts[a];
            const int64_t first = b == N - 1 ? 0 : b + 1;
            out[p] = tail + starts[first];
        }
    }
}

}  // namespace tio

using namespace tio;

// Virtual ranks (tio_plan_create_virtual): every rank thread prepares its
// planner instance with tio_plan_create2 up to the round loop, then hands its
// PlanArgs to this rendezvous; the last to arrive launches ONE cooperative
// grid running every instance (launch_plan_loop_multi) after the other ranks'
// setup work (their streams' ready events), and every rank's stream waits
// for that grid before its epilogue.
#include <condition_variable>
#include <mutex>
struct VGroup {
    int nranks = 0, blocks_per_rank = 0;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    bool launched = false;
    bool failed = false;                 // a rank failed before its launch point: nobody launches
    std::vector<char> here;              // rank r reached the rendezvous (or gave up)
    int rc = TIO_OK;
    std::vector<PlanArgs> args;
    std::vector<cudaEvent_t> ready;
    cudaEvent_t done = nullptr;
    PlanArgs *dev_args = nullptr;
};
static thread_local VGroup *t_vgroup = nullptr;
static thread_local int t_vrank = 0;

// a rank that ends (error) without reaching the launch still counts as
// arrived, so the others are released instead of waiting forever
static void vgroup_leave(VGroup *g, int rank) {
    std::unique_lock<std::mutex> lk(g->m);
    if (g->here[rank]) return;
    g->here[rank] = 1;
    g->failed = true;
    if (++g->arrived == g->nranks) {
        g->rc = fail(TIO_ERR_INTERNAL, "virtual ranks: a rank failed before the round loop");
        g->launched = true;
        g->cv.notify_all();
    }
}

static int vgroup_launch(VGroup *g, int rank, const PlanArgs &a, cudaStream_t s) {
    std::unique_lock<std::mutex> lk(g->m);
    g->here[rank] = 1;
    g->args[rank] = a;
    cudaEventRecord(g->ready[rank], s);
    if (++g->arrived == g->nranks && g->failed) {
        g->rc = fail(TIO_ERR_INTERNAL, "virtual ranks: a rank failed before the round loop");
        g->launched = true;
        g->cv.notify_all();
    } else if (g->arrived == g->nranks) {
        int rc = TIO_OK;
        for (int r = 0; r < g->nranks && rc == TIO_OK; ++r)
            if (cudaStreamWaitEvent(s, g->ready[r], 0) != cudaSuccess) rc = fail(TIO_ERR_CUDA, "virtual ranks: wait");
        if (rc == TIO_OK &&
            cudaMemcpyAsync(g->dev_args, g->args.data(), sizeof(PlanArgs) * g->nranks, cudaMemcpyHostToDevice, s) !=
                cudaSuccess)
            rc = fail(TIO_ERR_CUDA, "virtual ranks: argument upload");
        if (rc == TIO_OK) rc = launch_plan_loop_multi(g->dev_args, g->nranks, g->blocks_per_rank, s);
        if (rc == TIO_OK && cudaEventRecord(g->done, s) != cudaSuccess) rc = fail(TIO_ERR_CUDA, "virtual ranks: record");
        // the upload reads g->args (pageable): done before the host may reuse it
        cudaStreamSynchronize(s);
        g->rc = rc;
        g->launched = true;
        g->cv.notify_all();
    } else {
        g->cv.wait(lk, [g] { return g->launched; });
    }
    if (g->rc != TIO_OK) return g->rc;
    TIO_CUDA(cudaStreamWaitEvent(s, g->done, 0));
    return TIO_OK;
}

struct tio_trace {
    int64_t N = 0, T = 0, E = 0;
    const int64_t *dur = nullptr, *tid = nullptr, *size = nullptr, *ptr = nullptr;
    const int8_t *kind = nullptr;
    const int32_t *acc = nullptr;
    Arena arena;          // owned input columns (host input) + lifetime products
    bool lifetime_enqueued = false;
    bool synced = false;
    int64_t *starts = nullptr, *timeline = nullptr, *active = nullptr, *diff = nullptr;
    int64_t *p_tensor = nullptr, *tpp = nullptr, *blk = nullptr, *scalars = nullptr;
    int32_t *p_start = nullptr, *p_end = nullptr;
    int8_t *p_wraps = nullptr;
    // host copies after sync
    int64_t num_periods = 0, iteration = 0, flags = 0, ids_unsorted = 0;
};

struct tio_plan {
    Arena arena;
    tio_plan_info info{};
    int64_t N = 0;
    tio_commit *commits = nullptr;
    tio_entry *entries = nullptr;
    int64_t *resid = nullptr;
    int64_t *over = nullptr;
};

extern "C" {

int tio_abi_version(void) { return TIO_ABI_VERSION; }

int tio_kernel_launches(int64_t *out) {
    if (!out) return fail(TIO_ERR_INVALID, "null out");
    *out = g_launches.load(std::memory_order_relaxed);
    return TIO_OK;
}

int tio_last_error(char *buf, size_t len) {
    if (!buf || !len) return TIO_ERR_INVALID;
    strncpy(buf, g_err, len - 1);
    buf[len - 1] = 0;
    return TIO_OK;
}

int tio_device_info(char *buf, size_t len) {
    int dev = 0;
    cudaDeviceProp prop;
    TIO_CUDA(cudaGetDevice(&dev));
    TIO_CUDA(cudaGetDeviceProperties(&prop, dev));
    snprintf(buf, len, "%s sm_%d%d %d SMs, built for sm_100a", prop.name, prop.major, prop.minor,
             prop.multiProcessorCount);
    return TIO_OK;
}

int tio_transfer_duration(double rate, int64_t nbytes, int64_t *out) {
    if (!out) return fail(TIO_ERR_INVALID, "null out");
    if (nbytes < 0) return fail(TIO_ERR_INVALID, "negative transfer size");
    RateCode rc;
    TIO_TRY(decode_rate(rate, &rc));
    *out = duration_of(rc, nbytes);
    return TIO_OK;
}

int tio_trace_create(const tio_trace_desc *d, int mem_kind, void *stream, tio_trace **out) {
    if (!d || !out) return fail(TIO_ERR_INVALID, "null argument");
    if (d->num_kernels < 0 || d->num_tensors < 0 || d->num_events < 0)
        return fail(TIO_ERR_INVALID, "negative size");
    if (d->num_kernels >= INT32_MAX || d->num_events >= INT32_MAX || d->num_tensors >= INT32_MAX)
        return fail(TIO_ERR_OVERFLOW, "trace too large for 32-bit kernel/tensor indices");
    TIO_TRY(ensure_pool());
    cudaStream_t s = (cudaStream_t)stream;
    tio_trace *t = new tio_trace();
    t->arena.stream = s;
    t->N = d->num_kernels;
    t->T = d->num_tensors;
    t->E = d->num_events;
    if (mem_kind == TIO_MEM_DEVICE) {
        t->dur = d->duration_us; t->tid = d->tensor_id; t->size = d->size_bytes;
        t->kind = d->kind; t->ptr = d->access_ptr; t->acc = d->accesses;
    } else if (mem_kind == TIO_MEM_HOST) {
        int64_t *dur, *tid, *size, *ptr;
        int8_t *kind;
        int32_t *acc;
        int rc = TIO_OK;
        if ((rc = t->arena.alloc(&dur, t->N)) || (rc = t->arena.alloc(&tid, t->T)) ||
            (rc = t->arena.alloc(&size, t->T)) || (rc = t->arena.alloc(&kind, t->T)) ||
            (rc = t->arena.alloc(&ptr, t->T + 1)) || (rc = t->arena.alloc(&acc, t->E))) {
            t->arena.release();
            delete t;
            return rc;
        }
        cudaError_t e = cudaSuccess;
        if (t->N) e = cudaMemcpyAsync(dur, d->duration_us, 8 * t->N, cudaMemcpyHostToDevice, s);
        if (!e && t->T) e = cudaMemcpyAsync(tid, d->tensor_id, 8 * t->T, cudaMemcpyHostToDevice, s);
        if (!e && t->T) e = cudaMemcpyAsync(size, d->size_bytes, 8 * t->T, cudaMemcpyHostToDevice, s);
        if (!e && t->T) e = cudaMemcpyAsync(kind, d->kind, t->T, cudaMemcpyHostToDevice, s);
        if (!e) e = cudaMemcpyAsync(ptr, d->access_ptr, 8 * (t->T + 1), cudaMemcpyHostToDevice, s);
        if (!e && t->E) e = cudaMemcpyAsync(acc, d->accesses, 4 * t->E, cudaMemcpyHostToDevice, s);
        if (e) {
            t->arena.release();
            delete t;
            return fail(TIO_ERR_CUDA, "trace upload failed: %s", cudaGetErrorString(e));
        }
        t->dur = dur; t->tid = tid; t->size = size; t->kind = kind; t->ptr = ptr; t->acc = acc;
    } else {
        delete t;
        return fail(TIO_ERR_INVALID, "unknown mem_kind %d", mem_kind);
    }
    *out = t;
    return TIO_OK;
}

int tio_trace_destroy(tio_trace *t) {
    if (!t) return TIO_OK;
    t->arena.release();
    cudaStreamSynchronize(t->arena.stream);
    delete t;
    return TIO_OK;
}

int tio_lifetime(tio_trace *t, void *stream) {
    if (!t) return fail(TIO_ERR_INVALID, "null trace");
    cudaStream_t s = (cudaStream_t)stream;
    t->arena.stream = s;
    if (!t->starts) {
        TIO_TRY(t->arena.alloc(&t->starts, t->N + 1));
        TIO_TRY(t->arena.alloc(&t->timeline, t->N));
        TIO_TRY(t->arena.alloc(&t->active, t->N));
        TIO_TRY(t->arena.alloc(&t->diff, t->N + 1));
        TIO_TRY(t->arena.alloc(&t->p_tensor, t->E));
        TIO_TRY(t->arena.alloc(&t->p_start, t->E));
        TIO_TRY(t->arena.alloc(&t->p_end, t->E));
        TIO_TRY(t->arena.alloc(&t->p_wraps, t->E));
        TIO_TRY(t->arena.alloc(&t->tpp, t->T + 1));
        TIO_TRY(t->arena.alloc(&t->blk, lifetime_workspace_elems(t->N, t->E)));
        TIO_CUDA(cudaMemsetAsync(t->diff, 0, 8 * (t->N + 1), s));   // the kernel re-zeroes it behind its scan
        TIO_TRY(t->arena.alloc(&t->scalars, SC_COUNT));
    }
    // active bytes and the scalars are zeroed by the stage's first kernel
    // (k_tile_owners) — or here when it has no kernels
    if (t->N == 0) {
        TIO_CUDA(cudaMemsetAsync(t->active, 0, 8, s));
        TIO_CUDA(cudaMemsetAsync(t->scalars, 0, 8 * SC_COUNT, s));
    }
    if (t->T == 0) TIO_CUDA(cudaMemsetAsync(t->tpp, 0, 8, s));
    LifetimeArgs a;
    a.N = t->N; a.T = t->T; a.E = t->E;
    a.dur = t->dur; a.tid = t->tid; a.size = t->size; a.kind = t->kind; a.ptr = t->ptr; a.acc = t->acc;
    a.starts = t->starts; a.timeline = t->timeline; a.active = t->active; a.diff = t->diff;
    a.p_tensor = t->p_tensor; a.p_start = t->p_start; a.p_end = t->p_end; a.p_wraps = t->p_wraps;
    a.tensor_pptr = t->tpp;
    a.work = t->blk;
    a.scalars = t->scalars;
    if (t->N == 0) {
        // no kernels: every trace with tensors is invalid (accesses out of range)
        TIO_CUDA(cudaMemsetAsync(t->starts, 0, 8, s));
        if (t->T > 0) {
            int64_t bad = 8;
            TIO_CUDA(cudaMemcpyAsync(t->scalars + SC_FLAGS, &bad, 8, cudaMemcpyHostToDevice, s));
            TIO_CUDA(cudaStreamSynchronize(s));
        }
    } else {
        TIO_TRY(launch_lifetime(a, s));
    }
    t->lifetime_enqueued = true;
    t->synced = false;
    return TIO_OK;
}

static int lifetime_sync(tio_trace *t, cudaStream_t s) {
    if (!t->lifetime_enqueued) TIO_TRY(tio_lifetime(t, s));
    if (t->synced) return TIO_OK;
    int64_t sc[SC_COUNT];
    TIO_CUDA(cudaMemcpyAsync(sc, t->scalars, sizeof(sc), cudaMemcpyDeviceToHost, s));
    int64_t it = 0;
    TIO_CUDA(cudaMemcpyAsync(&it, t->starts + t->N, 8, cudaMemcpyDeviceToHost, s));
    TIO_CUDA(cudaStreamSynchronize(s));
    t->num_periods = t->T > 0 ? sc[SC_NUM_PERIODS] : 0;
    t->flags = sc[SC_FLAGS];
    t->ids_unsorted = sc[SC_IDS_UNSORTED];
    t->iteration = it;
    t->synced = true;
    if (t->flags) return fail(TIO_ERR_INVALID, "trace violates model invariants (flags 0x%llx)",
                              (unsigned long long)t->flags);
    return TIO_OK;
}

int tio_lifetime_view_get(tio_trace *t, void *stream, tio_lifetime_view *v) {
    if (!t || !v) return fail(TIO_ERR_INVALID, "null argument");
    TIO_TRY(lifetime_sync(t, (cudaStream_t)stream));
    v->num_kernels = t->N; v->num_tensors = t->T; v->num_periods = t->num_periods;
    v->iteration_us = t->iteration;
    v->starts = t->starts; v->timeline = t->timeline; v->active = t->active;
    v->period_tensor = t->p_tensor; v->period_start = t->p_start; v->period_end = t->p_end;
    v->period_wraps = t->p_wraps; v->tensor_period_ptr = t->tpp;
    return TIO_OK;
}

int tio_period_interior(tio_trace *t, void *stream, int64_t *out) {
    if (!t || !out) return fail(TIO_ERR_INVALID, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    TIO_TRY(lifetime_sync(t, s));
    const int64_t P = t->num_periods;
    if (P == 0) return TIO_OK;
    int64_t *d = nullptr;
    TIO_CUDA(cudaMallocAsync(&d, 8 * P, s));
    int64_t b = (P + 255) / 256;
    if (b > 148 * 16) b = 148 * 16;
    k_period_interior<<<(unsigned)b, 256, 0, s>>>(t->starts, t->p_start, t->p_end, t->p_wraps, P, t->N, d);
    count_launch();
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, d, 8 * P, cudaMemcpyDeviceToHost, s);
    cudaFreeAsync(d, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return fail(TIO_ERR_CUDA, "period interior: %s", cudaGetErrorString(e));
    return TIO_OK;
}

int tio_lifetime_copy_out(tio_trace *t, void *stream, int64_t *starts, int64_t *timeline, int64_t *active,
                          int64_t *period_tensor, int32_t *period_start, int32_t *period_end,
                          int8_t *period_wraps) {
    if (!t) return fail(TIO_ERR_INVALID, "null trace");
    cudaStream_t s = (cudaStream_t)stream;
    TIO_TRY(lifetime_sync(t, s));
    const int64_t N = t->N, P = t->num_periods;
    if (starts) TIO_CUDA(cudaMemcpyAsync(starts, t->starts, 8 * (N + 1), cudaMemcpyDeviceToHost, s));
    if (timeline && N) TIO_CUDA(cudaMemcpyAsync(timeline, t->timeline, 8 * N, cudaMemcpyDeviceToHost, s));
    if (active && N) TIO_CUDA(cudaMemcpyAsync(active, t->active, 8 * N, cudaMemcpyDeviceToHost, s));
    if (P) {
        if (period_tensor) TIO_CUDA(cudaMemcpyAsync(period_tensor, t->p_tensor, 8 * P, cudaMemcpyDeviceToHost, s));
        if (period_start) TIO_CUDA(cudaMemcpyAsync(period_start, t->p_start, 4 * P, cudaMemcpyDeviceToHost, s));
        if (period_end) TIO_CUDA(cudaMemcpyAsync(period_end, t->p_end, 4 * P, cudaMemcpyDeviceToHost, s));
        if (period_wraps) TIO_CUDA(cudaMemcpyAsync(period_wraps, t->p_wraps, P, cudaMemcpyDeviceToHost, s));
    }
    TIO_CUDA(cudaStreamSynchronize(s));
    return TIO_OK;
}

static int bitlen(uint64_t v) {
    int b = 0;
    while (v) { ++b; v >>= 1; }
    return b;
}

static unsigned grid_for(int64_t n, int threads = 256) {
    int64_t b = (n + threads - 1) / threads;
    if (b < 1) b = 1;
    if (b > 148 * 16) b = 148 * 16;
    return (unsigned)b;
}

int tio_plan_create(tio_trace *t, int64_t capacity, const tio_rates *rates, int64_t host_cap, void *stream,
                    tio_plan **out, tio_plan_info *info) {
    return tio_plan_create2(t, capacity, rates, host_cap, nullptr, stream, out, info);
}

int tio_plan_create2(tio_trace *t, int64_t capacity, const tio_rates *rates, int64_t host_cap,
                     const tio_plan_opts *opts, void *stream, tio_plan **out, tio_plan_info *info) {
    if (!t || !rates || !out) return fail(TIO_ERR_INVALID, "null argument");
    *out = nullptr;
    cudaStream_t s = (cudaStream_t)stream;
    TIO_TRY(lifetime_sync(t, s));
    const int64_t N = t->N, T = t->T, P = t->num_periods, I = t->iteration;
    tio_plan *p = new tio_plan();
    p->arena.stream = s;
    p->N = N;
    tio_plan_info &pi = p->info;
    memset(&pi, 0, sizeof(pi));
    pi.capacity_bytes = capacity;
    pi.num_candidates = P;
    Arena &A = p->arena;
    auto bail = [&](int rc) { A.release(); cudaStreamSynchronize(s); if (info) *info = pi; delete p; return rc; };
#define PTRY(expr) do { int _r = (expr); if (_r != TIO_OK) return bail(_r); } while (0)
#define PCUDA(expr) do { cudaError_t _e = (expr); if (_e != cudaSuccess) return bail(fail(TIO_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(_e))); } while (0)

    int64_t *ps;
    PTRY(A.alloc(&ps, PS_COUNT));
    PCUDA(cudaMemsetAsync(ps, 0, 8 * PS_COUNT, s));
    // unsatisfiable check first (planner.py:275-278), before any channel is built
    {
        unsigned long long *first;
        PTRY(A.alloc(&first, 1));
        PCUDA(cudaMemsetAsync(first, 0xff, 8, s));
        if (N) k_unsat<<<grid_for(N), 256, 0, s>>>(t->active, N, capacity, first); ::tio::count_launch();
        k_unsat_finish<<<1, 1, 0, s>>>(t->active, first, N, ps, t->scalars + SC_FLAGS); ::tio::count_launch();
        PCUDA(cudaGetLastError());
    }
    RateCode rc[4];
    int rate_err = decode_rate(rates->ssd_offload, &rc[0]);
    if (!rate_err) rate_err = decode_rate(rates->ssd_prefetch, &rc[1]);
    if (!rate_err && rates->has_host) rate_err = decode_rate(rates->host_offload, &rc[2]);
    if (!rate_err && rates->has_host) rate_err = decode_rate(rates->host_prefetch, &rc[3]);
    if (!rates->has_host) { rc[2] = rc[0]; rc[3] = rc[1]; }
    if (rate_err) {
        int64_t hs[PS_COUNT];
        PCUDA(cudaMemcpyAsync(hs, ps, sizeof(hs), cudaMemcpyDeviceToHost, s));
        PCUDA(cudaStreamSynchronize(s));
        if (hs[PS_STATUS] == 1) {
            pi.unsat_kernel = hs[PS_UNSAT_K]; pi.unsat_bytes = hs[PS_UNSAT_B];
            return bail(fail(TIO_ERR_UNSATISFIABLE, "kernel %lld uses %lld bytes actively, more than capacity %lld; "
                             "no offloading plan can help", (long long)pi.unsat_kernel,
                             (long long)pi.unsat_bytes, (long long)capacity));
        }
        return bail(rate_err);
    }
    const bool has_host = rates->has_host != 0;

    // ---- candidate order: tensors by id, then start kernel
    int32_t *rank;
    int64_t *cnt_by_rank, *cand_ptr, *scan_tmp;
    PTRY(A.alloc(&rank, T));
    PTRY(A.alloc(&cnt_by_rank, T + 1));
    PTRY(A.alloc(&cand_ptr, T + 1));
    PTRY(A.alloc(&scan_tmp, scan_tmp_elems(T + 1) + 2));
    int64_t *dupflag;
    PTRY(A.alloc(&dupflag, 1));
    PCUDA(cudaMemsetAsync(dupflag, 0, 8, s));
    if (T > 0) {
        if (t->ids_unsorted) {
            uint64_t *k0, *k1;
            uint32_t *v0, *v1;
        int64_t *hist;
            PTRY(A.alloc(&k0, T)); PTRY(A.alloc(&k1, T));
            PTRY(A.alloc(&v0, T)); PTRY(A.alloc(&v1, T));
            PTRY(A.alloc(&hist, radix_hist_elems(T)));
            k_id_keys<<<grid_for(T), 256, 0, s>>>(t->tid, T, k0, v0); ::tio::count_launch();
            bool in_tmp = false;
            PTRY(radix_sort_pairs(k0, v0, k1, v1, hist, T, 64, s, &in_tmp));
            k_rank<<<grid_for(T), 256, 0, s>>>(in_tmp ? k1 : k0, in_tmp ? v1 : v0, T, t->tpp, rank,
                                              cnt_by_rank, dupflag); ::tio::count_launch();
        } else {
            k_rank<<<grid_for(T), 256, 0, s>>>(nullptr, nullptr, T, t->tpp, rank, cnt_by_rank, dupflag); ::tio::count_launch();
        }
        PCUDA(cudaGetLastError());
        PTRY(exclusive_scan(cnt_by_rank, cand_ptr, T, scan_tmp, cand_ptr + T, s));
    }

    // ---- candidates + planner state
    PlanArgs a;
    memset(&a, 0, sizeof(a));
    int64_t *c_size, *c_ready, *c_deadline, *c_d, *c_tid, *place;
    int32_t *c_sk, *c_ek, *c_first, *c_last, *c_tpos, *rng;
    int8_t *c_wraps, *st;
    PTRY(A.alloc(&c_size, P)); PTRY(A.alloc(&c_ready, P)); PTRY(A.alloc(&c_deadline, P));
    PTRY(A.alloc(&c_d, 4 * P)); PTRY(A.alloc(&c_tid, P)); PTRY(A.alloc(&place, 4 * P));
    PTRY(A.alloc(&c_sk, P)); PTRY(A.alloc(&c_ek, P)); PTRY(A.alloc(&c_first, P)); PTRY(A.alloc(&c_last, P));
    PTRY(A.alloc(&c_tpos, P)); PTRY(A.alloc(&rng, 4 * P));
    int32_t *hidx, *hver;
    PTRY(A.alloc(&hidx, 2 * P)); PTRY(A.alloc(&hver, P));
    PTRY(A.alloc(&c_wraps, P)); PTRY(A.alloc(&st, P));
    if (P > 0) {
        CandBuild cb;
        cb.num_periods = t->scalars + SC_NUM_PERIODS;
        cb.p_tensor = t->p_tensor; cb.p_start = t->p_start; cb.p_end = t->p_end; cb.p_wraps = t->p_wraps;
        cb.tpp = t->tpp; cb.rank = rank; cb.cand_ptr = cand_ptr;
        cb.size = t->size; cb.tid = t->tid; cb.ptr = t->ptr; cb.starts = t->starts; cb.dur = t->dur; cb.acc = t->acc;
        cb.iteration = I; cb.has_host = has_host;
        for (int q = 0; q < 4; ++q) cb.rates[q] = rc[q];
        cb.c_size = c_size; cb.c_sk = c_sk; cb.c_ek = c_ek; cb.c_first = c_first; cb.c_last = c_last;
        cb.c_wraps = c_wraps; cb.c_ready = c_ready; cb.c_deadline = c_deadline; cb.c_d = c_d; cb.c_tid = c_tid;
        cb.c_tpos = c_tpos; cb.st = st;
        k_build_candidates<<<grid_for(P), 256, 0, s>>>(cb); ::tio::count_launch();
        PCUDA(cudaGetLastError());
    }
    // ---- tiles: candidates in ready-time order (planner.cu).  The planner's
    // candidate columns are stored in tile order (position p) so a tile's
    // data is contiguous; tcand[p] = candidate index (the tie-break key; the
    // argmax key carries both).
    const int64_t ntiles = (P + TILE - 1) / TILE;
    uint32_t *tcand;
    int32_t *t_ka_lo, *t_ka_hi, *t_kb_lo, *t_kb_hi;
    int64_t *t_lo, *t_hi;
    Key *tile_best;
    PTRY(A.alloc(&t_lo, ntiles)); PTRY(A.alloc(&t_hi, ntiles));
    PTRY(A.alloc(&t_ka_lo, ntiles)); PTRY(A.alloc(&t_ka_hi, ntiles));
    PTRY(A.alloc(&t_kb_lo, ntiles)); PTRY(A.alloc(&t_kb_hi, ntiles));
    PTRY(A.alloc(&tile_best, ntiles));
    PTRY(A.alloc(&a.vkey, P));
    PTRY(A.alloc(&a.rq[0], P)); PTRY(A.alloc(&a.rq[1], P));
    PTRY(A.alloc(&a.t_refit, ntiles));
    PTRY(A.alloc(&a.t_hull, 4 * ntiles));
    PTRY(A.alloc(&a.qround, P));
    PCUDA(cudaMemsetAsync(a.qround, 0xff, 4 * (size_t)(P > 0 ? P : 1), s));
    PCUDA(cudaMemsetAsync(a.t_refit, 0xff, 4 * (size_t)(ntiles > 0 ? ntiles : 1), s));
    CandCols src{c_size, c_ready, c_deadline, c_d, c_tid, c_sk, c_ek, c_first, c_last, c_tpos, c_wraps, st};
    CandCols dst;
    PTRY(A.alloc(&dst.size, P)); PTRY(A.alloc(&dst.ready, P)); PTRY(A.alloc(&dst.deadline, P));
    PTRY(A.alloc(&dst.d, 4 * P)); PTRY(A.alloc(&dst.tid, P));
    PTRY(A.alloc(&dst.sk, P)); PTRY(A.alloc(&dst.ek, P)); PTRY(A.alloc(&dst.first, P)); PTRY(A.alloc(&dst.last, P));
    PTRY(A.alloc(&dst.tpos, P)); PTRY(A.alloc(&dst.wraps, P)); PTRY(A.alloc(&dst.st, P));
    {
        uint64_t *k0, *k1;
        uint32_t *v0, *v1;
        int64_t *hist;
        PTRY(A.alloc(&k0, P)); PTRY(A.alloc(&k1, P)); PTRY(A.alloc(&v0, P)); PTRY(A.alloc(&v1, P));
        PTRY(A.alloc(&hist, radix_hist_elems(P)));
        bool in_tmp = false;
        if (P > 0) {
            k_ready_keys<<<grid_for(P), 256, 0, s>>>(c_ready, P, k0, v0); ::tio::count_launch();
            PTRY(radix_sort_pairs(k0, v0, k1, v1, hist, P, bitlen((uint64_t)(I > 0 ? I : 1)), s, &in_tmp));
        }
        tcand = in_tmp ? v1 : v0;
        if (P > 0) {
            k_permute_candidates<<<grid_for(P), 256, 0, s>>>(tcand, P, src, dst); ::tio::count_launch();
            k_tile_spans<<<grid_for(ntiles * 32), 256, 0, s>>>(nullptr, P, ntiles, TILE, N, dst.ready, dst.deadline,
                                                              dst.wraps, dst.sk, dst.ek, dst.first, dst.last, nullptr, t_lo,
                                                              t_hi, t_ka_lo, t_ka_hi, t_kb_lo, t_kb_hi); ::tio::count_launch();
        }
        PCUDA(cudaGetLastError());
    }
    c_size = dst.size; c_ready = dst.ready; c_deadline = dst.deadline; c_d = dst.d; c_tid = dst.tid;
    c_sk = dst.sk; c_ek = dst.ek; c_first = dst.first; c_last = dst.last; c_tpos = dst.tpos;
    c_wraps = dst.wraps; st = dst.st;
    a.ntiles = ntiles; a.tcand = tcand; a.t_lo = t_lo; a.t_hi = t_hi;
    a.t_ka_lo = t_ka_lo; a.t_ka_hi = t_ka_hi; a.t_kb_lo = t_kb_lo; a.t_kb_hi = t_kb_hi; a.tile_best = tile_best;
    int G = 0;
    const int nranks = opts && opts->nranks > 1 ? opts->nranks : 1;
    // the wide form pays off with many tiles per rank (sharded: this rank's share)
    const bool wide = !t_vgroup && plan_loop_wide(ntiles / nranks);
    PTRY(plan_loop_grid(&G, wide));
    if (opts && opts->blocks > 0 && opts->blocks < G) G = opts->blocks;
    if (nranks > MAX_RANKS) return bail(fail(TIO_ERR_INVALID, "at most %d ranks", MAX_RANKS));
    if (nranks > 1) {
        if (!opts->mailbox || !opts->peer_mailboxes || opts->rank < 0 || opts->rank >= nranks)
            return bail(fail(TIO_ERR_INVALID, "sharded planning needs rank, mailbox and peer mailboxes"));
        a.nranks = nranks;
        a.rank = opts->rank;
        a.epoch = opts->epoch;
        a.mb_self = static_cast<Mailbox *>(opts->mailbox);
        for (int r = 0; r < nranks; ++r) a.mb_peer[r] = static_cast<Mailbox *>(opts->peer_mailboxes[r]);
    }
    PTRY(A.alloc(&a.win, 1));
    PTRY(A.alloc(&a.win_gen, 1));
    PCUDA(cudaMemsetAsync(a.win_gen, 0, 8, s));
    int64_t *resid, *local_cp, *chunk_sum;
    PTRY(A.alloc(&resid, N)); PTRY(A.alloc(&local_cp, N + 1)); PTRY(A.alloc(&chunk_sum, G));
    if (N) PCUDA(cudaMemcpyAsync(resid, t->timeline, 8 * N, cudaMemcpyDeviceToDevice, s));
    const int nch = has_host ? 4 : 2;
    const int64_t ch_cap = 3 * P + 3;
    for (int q = 0; q < 4; ++q)
        for (int bb = 0; bb < 2; ++bb) {
            if (q < nch) {
                PTRY(A.alloc(&a.ch_s[q][bb], ch_cap));
                PTRY(A.alloc(&a.ch_e[q][bb], ch_cap));
            } else {
                a.ch_s[q][bb] = a.ch_s[0][bb];
                a.ch_e[q][bb] = a.ch_e[0][bb];
            }
        }
    int64_t *occ_s, *occ_e, *occ_z;
    PTRY(A.alloc(&occ_s, has_host ? P : 1)); PTRY(A.alloc(&occ_e, has_host ? P : 1)); PTRY(A.alloc(&occ_z, has_host ? P : 1));
    Key *blk_best;
    PTRY(A.alloc(&blk_best, G));
    int64_t *prof;
    PTRY(A.alloc(&prof, 8 * (int64_t)G));
    PCUDA(cudaMemsetAsync(prof, 0, 64 * (size_t)G, s));
    a.prof = prof;
    unsigned *bar;
    PTRY(A.alloc(&bar, 2));
    PCUDA(cudaMemsetAsync(bar, 0, 8, s));
    a.bar = bar;
    PTRY(A.alloc(&p->commits, P));
    a.N = N; a.P = P; a.iteration = I; a.capacity = capacity; a.host_cap = host_cap;
    a.has_host = has_host;
    a.chunk = (int32_t)((N + 1 + G - 1) / G);
    a.max_rounds = opts ? opts->max_rounds : 0;
    a.starts = t->starts; a.dur = t->dur; a.resid = resid; a.local_cp = local_cp; a.chunk_sum = chunk_sum;
    a.c_size = c_size; a.c_sk = c_sk; a.c_ek = c_ek; a.c_first = c_first; a.c_last = c_last; a.c_wraps = c_wraps;
    a.c_ready = c_ready; a.c_deadline = c_deadline; a.c_d = c_d;
    a.st = st; a.place = place; a.rng = rng; a.hidx = hidx; a.hver = hver;
    a.ch_cap = ch_cap;
    a.occ_s = occ_s; a.occ_e = occ_e; a.occ_size = occ_z;
    if (has_host) {                    // host-occupancy index (planner.cuh PlanArgs)
        const int64_t nx = P + 1;
        for (int bb = 0; bb < 2; ++bb) {
            PTRY(A.alloc(&a.hx_s[bb], nx)); PTRY(A.alloc(&a.hx_sz[bb], nx));
            PTRY(A.alloc(&a.hx_e[bb], nx)); PTRY(A.alloc(&a.hx_ez[bb], nx));
            PTRY(A.alloc(&a.hx_ps[bb], nx)); PTRY(A.alloc(&a.hx_pe[bb], nx));
            PTRY(A.alloc(&a.hx_a[bb], nx));
        }
        a.hx_nbmax = (P + 31) / 32 + 1;
        PTRY(A.alloc(&a.hx_tab, HX_LEVELS * a.hx_nbmax));
    }
    a.blk_best = blk_best; a.commits = p->commits; a.scalars = ps; a.c_tid = c_tid; a.c_tpos = c_tpos;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    PCUDA(cudaEventCreate(&ev0));
    PCUDA(cudaEventCreate(&ev1));
    PCUDA(cudaEventRecord(ev0, s));
    int loop_rc = t_vgroup ? vgroup_launch(t_vgroup, t_vrank, a, s) : launch_plan_loop(a, G, s, wide);
    PCUDA(cudaEventRecord(ev1, s));
    if (loop_rc != TIO_OK) { cudaEventDestroy(ev0); cudaEventDestroy(ev1); return bail(loop_rc); }

    int64_t hs[PS_COUNT];
    int64_t dup = 0;
    PCUDA(cudaMemcpyAsync(hs, ps, sizeof(hs), cudaMemcpyDeviceToHost, s));
    PCUDA(cudaMemcpyAsync(&dup, dupflag, 8, cudaMemcpyDeviceToHost, s));
    PCUDA(cudaStreamSynchronize(s));
    {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev0, ev1);
        pi.loop_ns = (int64_t)((double)ms * 1e6);
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
    }
    if (dup) return bail(fail(TIO_ERR_INVALID, "duplicate tensor id"));
    if (hs[PS_STATUS] == 1) {
        pi.unsat_kernel = hs[PS_UNSAT_K]; pi.unsat_bytes = hs[PS_UNSAT_B];
        return bail(fail(TIO_ERR_UNSATISFIABLE, "kernel %lld uses %lld bytes actively, more than capacity %lld; "
                         "no offloading plan can help", (long long)pi.unsat_kernel,
                         (long long)pi.unsat_bytes, (long long)capacity));
    }
    if (hs[PS_STATUS] == 2) return bail(fail(TIO_ERR_INVALID, "trace violates model invariants"));
    if (hs[PS_STATUS] == 3)
        return bail(fail(TIO_ERR_CUDA, "sharded planning: rank exchange timed out in round %lld (a peer rank never "
                         "published its round message)", (long long)hs[PS_ROUNDS]));
    if (hs[PS_INVARIANT]) return bail(fail(TIO_ERR_INTERNAL, "channel bookings overlapped (disjointness invariant)"));
    const int64_t nc = hs[PS_COMMITS];
    pi.num_commits = nc;
    pi.num_entries = 2 * nc;
    pi.rounds = hs[PS_ROUNDS];
    for (int q = 0; q < 14; ++q) pi.dbg[q] = hs[PS_DBG + q];
    if (getenv("TIO_PLAN_PROFILE_DUMP")) {
        std::vector<int64_t> hp(8 * (size_t)G);
        cudaMemcpy(hp.data(), prof, 64 * (size_t)G, cudaMemcpyDeviceToHost);
        int64_t tot[7] = {0, 0, 0, 0, 0, 0, 0};
        for (int bb = 0; bb < G; ++bb)
            for (int q = 0; q < 7; ++q) tot[q] += hp[8 * bb + q];
        fprintf(stderr, "fit walks: %lld steps total, longest %lld\n", (long long)hs[PS_DBG + 11],
                (long long)hs[PS_DBG + 12]);
        fprintf(stderr, "slow phase-E rounds (>15us): %lld block-rounds; mean us: dirty %.2f pass1 %.2f window %.2f "
                "pass2 %.2f tile-reduce %.2f block-reduce %.2f\n", (long long)tot[6],
                tot[0] / 1e3 / (tot[6] ? tot[6] : 1), tot[1] / 1e3 / (tot[6] ? tot[6] : 1),
                tot[2] / 1e3 / (tot[6] ? tot[6] : 1), tot[3] / 1e3 / (tot[6] ? tot[6] : 1),
                tot[4] / 1e3 / (tot[6] ? tot[6] : 1), tot[5] / 1e3 / (tot[6] ? tot[6] : 1));
    }

    // ---- epilogue: over list, peak, planned host, sorted + urgent entries
    p->resid = resid;
    int64_t *flag, *pos, *ovt, *peakp, *hostp;
    PTRY(A.alloc(&flag, N)); PTRY(A.alloc(&pos, N + 1)); PTRY(A.alloc(&p->over, N));
    PTRY(A.alloc(&ovt, scan_tmp_elems(N) + 2)); PTRY(A.alloc(&peakp, 2)); PTRY(A.alloc(&hostp, 1));
    PCUDA(cudaMemsetAsync(peakp, 0, 16, s));
    {
        int64_t lmin = LLONG_MIN;
        PCUDA(cudaMemcpyAsync(peakp, &lmin, 8, cudaMemcpyHostToDevice, s));
    }
    if (N) {
        k_over_flags<<<grid_for(N), 256, 0, s>>>(resid, N, capacity, flag, (long long *)peakp); ::tio::count_launch();
        PTRY(exclusive_scan(flag, pos, N, ovt, pos + N, s));
        k_over_write<<<grid_for(N), 256, 0, s>>>(flag, pos, N, p->over); ::tio::count_launch();
    }
    PCUDA(cudaMemsetAsync(hostp, 0, 8, s));
    k_planned_host<<<grid_for(hs[PS_OCC] > 0 ? hs[PS_OCC] : 1), 256, 0, s>>>(occ_s, occ_e, occ_z, hs[PS_OCC], hostp);
    ::tio::count_launch();
    PTRY(A.alloc(&p->entries, 2 * nc));
    if (nc > 0) {
        const int64_t ne = 2 * nc;
        uint64_t *k0, *k1;
        uint32_t *v0, *v1;
        int64_t *hist;
        PTRY(A.alloc(&k0, ne)); PTRY(A.alloc(&k1, ne)); PTRY(A.alloc(&v0, ne)); PTRY(A.alloc(&v1, ne));
        PTRY(A.alloc(&hist, radix_hist_elems(ne)));
        const int rbits = bitlen((uint64_t)(T > 0 ? T - 1 : 0));
        const int tbits = bitlen((uint64_t)(2 * I > 0 ? 2 * I : 1));
        bool in_tmp = false;
        uint32_t *order;
        if (tbits + rbits + 1 <= 64) {
            k_entry_keys<<<grid_for(ne), 256, 0, s>>>(p->commits, nc, rank, rbits, 0, k0, v0); ::tio::count_launch();
            PTRY(radix_sort_pairs(k0, v0, k1, v1, hist, ne, tbits + rbits + 1, s, &in_tmp));
            order = in_tmp ? v1 : v0;
        } else {
            k_entry_keys<<<grid_for(ne), 256, 0, s>>>(p->commits, nc, rank, rbits, 1, k0, v0); ::tio::count_launch();
            PTRY(radix_sort_pairs(k0, v0, k1, v1, hist, ne, rbits + 1, s, &in_tmp));
            uint64_t *kk = in_tmp ? k1 : k0, *kt = in_tmp ? k0 : k1;
            uint32_t *vv = in_tmp ? v1 : v0, *vt = in_tmp ? v0 : v1;
            k_regather_keys<<<grid_for(ne), 256, 0, s>>>(p->commits, vv, ne, kk); ::tio::count_launch();
            bool in2 = false;
            PTRY(radix_sort_pairs(kk, vv, kt, vt, hist, ne, tbits, s, &in2));
            order = in2 ? vt : vv;
        }
        k_emit_entries<<<grid_for(ne), 256, 0, s>>>(p->commits, order, ne, t->starts, t->ptr, t->acc, t->kind, I,
                                                     p->entries); ::tio::count_launch();
        PCUDA(cudaGetLastError());
    }
    int64_t tail[3] = {0, 0, 0};
    PCUDA(cudaMemcpyAsync(&tail[0], peakp, 8, cudaMemcpyDeviceToHost, s));
    PCUDA(cudaMemcpyAsync(&tail[1], hostp, 8, cudaMemcpyDeviceToHost, s));
    if (N) PCUDA(cudaMemcpyAsync(&tail[2], pos + N, 8, cudaMemcpyDeviceToHost, s));
    PCUDA(cudaStreamSynchronize(s));
    pi.residual_peak_bytes = N ? tail[0] : 0;
    pi.planned_host_bytes = tail[1];
    pi.num_over = N ? tail[2] : 0;
    if (info) *info = pi;
    *out = p;
    return TIO_OK;
#undef PTRY
#undef PCUDA
}

int tio_plan_info_get(tio_plan *p, tio_plan_info *out) {
    if (!p || !out) return fail(TIO_ERR_INVALID, "null argument");
    *out = p->info;
    return TIO_OK;
}

int tio_plan_copy_out(tio_plan *p, void *stream, tio_commit *commits, tio_entry *entries, int64_t *residual,
                      int64_t *over) {
    if (!p) return fail(TIO_ERR_INVALID, "null plan");
    cudaStream_t s = (cudaStream_t)stream;
    const tio_plan_info &i = p->info;
    if (commits && i.num_commits)
        TIO_CUDA(cudaMemcpyAsync(commits, p->commits, sizeof(tio_commit) * i.num_commits, cudaMemcpyDeviceToHost, s));
    if (entries && i.num_entries)
        TIO_CUDA(cudaMemcpyAsync(entries, p->entries, sizeof(tio_entry) * i.num_entries, cudaMemcpyDeviceToHost, s));
    if (residual && p->N) TIO_CUDA(cudaMemcpyAsync(residual, p->resid, 8 * p->N, cudaMemcpyDeviceToHost, s));
    if (over && i.num_over) TIO_CUDA(cudaMemcpyAsync(over, p->over, 8 * i.num_over, cudaMemcpyDeviceToHost, s));
    TIO_CUDA(cudaStreamSynchronize(s));
    return TIO_OK;
}

// write_plan (planner.py:402-420): json.dumps default separators
int tio_plan_write(tio_plan *p, void *stream, char *buf, size_t *len) {
    if (!p || !len) return fail(TIO_ERR_INVALID, "null argument");
    const tio_plan_info &i = p->info;
    std::vector<tio_entry> ents((size_t)i.num_entries);
    std::vector<int64_t> over((size_t)i.num_over);
    TIO_TRY(tio_plan_copy_out(p, stream, nullptr, ents.data(), nullptr, over.data()));
    std::string out;
    out.reserve(160 + 24 * over.size() + 110 * ents.size());
    char tmp[256];
    snprintf(tmp, sizeof(tmp),
             "{\"version\": 1, \"capacity_bytes\": %lld, \"residual_peak_bytes\": %lld, "
             "\"planned_host_bytes\": %lld, \"over_capacity_kernels\": [",
             (long long)i.capacity_bytes, (long long)i.residual_peak_bytes, (long long)i.planned_host_bytes);
    out += tmp;
    for (size_t k = 0; k < over.size(); ++k) {
        snprintf(tmp, sizeof(tmp), k ? ", %lld" : "%lld", (long long)over[k]);
        out += tmp;
    }
    out += "]}";
    static const char *targets[] = {"GPU", "SSD", "CPU"};
    for (const tio_entry &e : ents) {
        snprintf(tmp, sizeof(tmp),
                 "\n{\"tensor\": %lld, \"action\": \"%s\", \"trigger_us\": %lld, \"deadline_us\": %lld, "
                 "\"target\": \"%s\", \"urgent\": %s}",
                 (long long)e.tensor_id, e.action ? "prefetch" : "offload", (long long)e.trigger_us,
                 (long long)e.deadline_us, targets[e.target < 0 || e.target > 2 ? 0 : e.target],
                 e.urgent ? "true" : "false");
        out += tmp;
    }
    out += "\n";
    if (!buf) { *len = out.size(); return TIO_OK; }
    if (*len < out.size()) { *len = out.size(); return fail(TIO_ERR_INVALID, "buffer too small"); }
    memcpy(buf, out.data(), out.size());
    *len = out.size();
    return TIO_OK;
}

int tio_plan_destroy(tio_plan *p) {
    if (!p) return TIO_OK;
    p->arena.release();
    cudaStreamSynchronize(p->arena.stream);
    delete p;
    return TIO_OK;
}

size_t tio_mailbox_bytes(void) { return sizeof(Mailbox); }

static_assert(sizeof(cudaIpcMemHandle_t) == TIO_IPC_HANDLE_BYTES, "IPC handle size");

int tio_mailbox_create(void **mailbox, unsigned char *ipc_handle) {
    if (!mailbox || !ipc_handle) return fail(TIO_ERR_INVALID, "null argument");
    *mailbox = nullptr;
    void *p = nullptr;
    TIO_CUDA(cudaMalloc(&p, sizeof(Mailbox)));
    cudaIpcMemHandle_t h;
    // zeroed (legacy stream, then waited for) before any planner stream can use it
    if (cudaMemset(p, 0, sizeof(Mailbox)) != cudaSuccess || cudaStreamSynchronize(nullptr) != cudaSuccess ||
        cudaIpcGetMemHandle(&h, p) != cudaSuccess) {
        cudaFree(p);
        return fail(TIO_ERR_CUDA, "mailbox: %s", cudaGetErrorString(cudaGetLastError()));
    }
    memcpy(ipc_handle, &h, sizeof(h));
    *mailbox = p;
    return TIO_OK;
}

int tio_mailbox_destroy(void *mailbox) {
    if (mailbox) TIO_CUDA(cudaFree(mailbox));
    return TIO_OK;
}

int tio_mailbox_open(const unsigned char *ipc_handle, void **mapped) {
    if (!ipc_handle || !mapped) return fail(TIO_ERR_INVALID, "null argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc_handle, sizeof(h));
    *mapped = nullptr;
    TIO_CUDA(cudaIpcOpenMemHandle(mapped, h, cudaIpcMemLazyEnablePeerAccess));
    return TIO_OK;
}

int tio_mailbox_close(void *mapped) {
    if (mapped) TIO_CUDA(cudaIpcCloseMemHandle(mapped));
    return TIO_OK;
}

int tio_plan_create_virtual(tio_trace *t, int64_t capacity, const tio_rates *rates, int64_t host_cap,
                            const tio_plan_opts *opts, int32_t nranks, tio_plan **out, tio_plan_info *info) {
    if (!t || !rates || !out || !info) return fail(TIO_ERR_INVALID, "null argument");
    if (nranks < 1 || nranks > MAX_RANKS) return fail(TIO_ERR_INVALID, "nranks must be in [1, %d]", MAX_RANKS);
    TIO_TRY(lifetime_sync(t, nullptr));        // shared trace products, before the rank threads start
    int G = 0;
    TIO_TRY(plan_loop_multi_grid(&G));
    int dev = 0;
    TIO_CUDA(cudaGetDevice(&dev));
    Mailbox *mb = nullptr;
    TIO_CUDA(cudaMalloc((void **)&mb, sizeof(Mailbox) * nranks));
    TIO_CUDA(cudaMemset(mb, 0, sizeof(Mailbox) * nranks));
    TIO_CUDA(cudaDeviceSynchronize());          // zeroed before any rank's stream (non-blocking) runs
    VGroup grp;
    grp.nranks = nranks;
    grp.blocks_per_rank = G / nranks;
    grp.args.resize(nranks);
    grp.ready.resize(nranks);
    grp.here.assign(nranks, 0);
    for (int r = 0; r < nranks; ++r) TIO_CUDA(cudaEventCreateWithFlags(&grp.ready[r], cudaEventDisableTiming));
    TIO_CUDA(cudaEventCreateWithFlags(&grp.done, cudaEventDisableTiming));
    TIO_CUDA(cudaMalloc((void **)&grp.dev_args, sizeof(PlanArgs) * nranks));
    std::vector<void *> peers(nranks);
    for (int r = 0; r < nranks; ++r) peers[r] = mb + r;
    std::vector<int> rcs(nranks, TIO_OK);
    std::vector<std::string> errs(nranks);
    std::vector<std::thread> th;
    for (int r = 0; r < nranks; ++r) {
        out[r] = nullptr;
        th.emplace_back([&, r]() {
            cudaSetDevice(dev);
            t_vgroup = &grp;
            t_vrank = r;
            cudaStream_t s = nullptr;
            if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) {
                rcs[r] = fail(TIO_ERR_CUDA, "stream creation failed");
                errs[r] = "stream creation failed";
                vgroup_leave(&grp, r);
                return;
            }
            tio_plan_opts o;
            memset(&o, 0, sizeof(o));
            if (opts) o.max_rounds = opts->max_rounds;
            o.nranks = nranks;
            o.rank = r;
            o.blocks = grp.blocks_per_rank;
            o.epoch = 0;
            o.mailbox = mb + r;
            o.peer_mailboxes = peers.data();
            rcs[r] = tio_plan_create2(t, capacity, rates, host_cap, &o, s, &out[r], &info[r]);
            vgroup_leave(&grp, r);           // no-op when the rank reached the launch
            if (rcs[r] != TIO_OK) {
                char b[1024];
                tio_last_error(b, sizeof(b));
                errs[r] = b;
            }
            cudaStreamSynchronize(s);
            if (out[r]) out[r]->arena.stream = nullptr;   // later frees on the legacy stream
            cudaStreamDestroy(s);
        });
    }
    for (auto &x : th) x.join();
    cudaFree(mb);
    cudaFree(grp.dev_args);
    for (auto e : grp.ready) cudaEventDestroy(e);
    cudaEventDestroy(grp.done);
    for (int r = 0; r < nranks; ++r)
        if (rcs[r] != TIO_OK) {
            for (int q = 0; q < nranks; ++q) { tio_plan_destroy(out[q]); out[q] = nullptr; }
            return fail(rcs[r], "virtual rank %d: %s", r, errs[r].c_str());
        }
    return TIO_OK;
}

int tio_plan_host(const tio_trace_desc *desc, int64_t capacity, const tio_rates *rates, int64_t host_cap,
                  void *stream, tio_plan_info *info, tio_entry *entries, int64_t entries_cap) {
    tio_trace *t = nullptr;
    TIO_TRY(tio_trace_create(desc, TIO_MEM_HOST, stream, &t));
    tio_plan *p = nullptr;
    int rc = tio_plan_create(t, capacity, rates, host_cap, stream, &p, info);
    if (rc == TIO_OK) {
        if (entries && info->num_entries > entries_cap) rc = fail(TIO_ERR_INVALID, "entries buffer too small");
        else rc = tio_plan_copy_out(p, stream, nullptr, entries, nullptr, nullptr);
        tio_plan_destroy(p);
    }
    tio_trace_destroy(t);
    return rc;
}

}  // extern "C"

// ---- engine scheduler (simulator.py:178-560) ----------------------------------
static int simulate_impl(const tio_trace_desc *d, const tio_entry *entries, int64_t num_entries, int64_t capacity,
                         const tio_rates *rates, const int64_t *k_layer, const int64_t *t_layer,
                         tio_sim_report *report, int64_t *per_kernel_start, int64_t *stall_per_kernel,
                         int64_t *per_kernel_resident) {
    if (!d || !rates || !report || (num_entries > 0 && !entries)) return fail(TIO_ERR_INVALID, "null argument");
    SchedInput in;
    in.N = d->num_kernels; in.T = d->num_tensors;
    in.dur = d->duration_us; in.tid = d->tensor_id; in.size = d->size_bytes; in.kind = d->kind;
    in.ptr = d->access_ptr; in.acc = d->accesses;
    std::vector<int64_t> e_tid(num_entries), e_trig(num_entries), e_dl(num_entries);
    std::vector<int32_t> e_act(num_entries), e_tgt(num_entries), e_urg(num_entries);
    for (int64_t i = 0; i < num_entries; ++i) {
        e_tid[i] = entries[i].tensor_id; e_trig[i] = entries[i].trigger_us; e_dl[i] = entries[i].deadline_us;
        e_act[i] = entries[i].action; e_tgt[i] = entries[i].target; e_urg[i] = entries[i].urgent;
    }
    in.num_entries = num_entries;
    in.e_tid = e_tid.data(); in.e_trigger = e_trig.data(); in.e_deadline = e_dl.data();
    in.e_action = e_act.data(); in.e_target = e_tgt.data(); in.e_urgent = e_urg.data();
    in.capacity = capacity;
    in.rate[0] = rates->ssd_offload; in.rate[1] = rates->ssd_prefetch;
    in.rate[2] = rates->host_offload; in.rate[3] = rates->host_prefetch;
    in.has_host = rates->has_host;
    in.layer_policy = k_layer != nullptr;
    in.k_layer = k_layer; in.t_layer = t_layer;
    for (int64_t t = 0; t < in.T; ++t)
        for (int64_t j = in.ptr[t]; j < in.ptr[t + 1]; ++j)
            if (in.acc[j] < 0 || in.acc[j] >= in.N) return fail(TIO_ERR_INVALID, "access out of range");
    SchedOutput out;
    std::string err;
    int rc = engine_schedule(in, &out, &err);
    if (rc != TIO_OK) return fail(rc, "%s", err.c_str());
    memset(report, 0, sizeof(*report));
    report->total_time = out.total_time;
    report->ideal_time = out.ideal_time;
    report->stall_time_total = out.stall_total;
    report->peak_resident_bytes = out.peak_resident;
    report->emergency_offloads = out.emergency;
    for (int c = 0; c < 4; ++c) report->channel_busy[c] = out.busy[c];
    report->num_transfers = (int64_t)out.transfers.size();
    const size_t nb = sizeof(int64_t) * (size_t)in.N;
    if (in.N) {
        if (per_kernel_start) memcpy(per_kernel_start, out.start.data(), nb);
        if (stall_per_kernel) memcpy(stall_per_kernel, out.stall.data(), nb);
        if (per_kernel_resident) memcpy(per_kernel_resident, out.resident.data(), nb);
    }
    return TIO_OK;
}

extern "C" int tio_simulate(const tio_trace_desc *d, const tio_entry *entries, int64_t num_entries, int64_t capacity,
                            const tio_rates *rates, tio_sim_report *report, int64_t *per_kernel_start,
                            int64_t *stall_per_kernel, int64_t *per_kernel_resident) {
    return simulate_impl(d, entries, num_entries, capacity, rates, nullptr, nullptr, report, per_kernel_start,
                         stall_per_kernel, per_kernel_resident);
}

extern "C" int tio_simulate_layers(const tio_trace_desc *d, const int64_t *kernel_layer, const int64_t *tensor_layer,
                                   int64_t capacity, const tio_rates *rates, tio_sim_report *report,
                                   int64_t *per_kernel_start, int64_t *stall_per_kernel,
                                   int64_t *per_kernel_resident) {
    if (!d || (d->num_kernels > 0 && !kernel_layer) || (d->num_tensors > 0 && !tensor_layer))
        return fail(TIO_ERR_INVALID, "null argument");
    static const int64_t none = INT64_MIN;
    return simulate_impl(d, nullptr, 0, capacity, rates, kernel_layer ? kernel_layer : &none,
                         tensor_layer ? tensor_layer : &none, report, per_kernel_start, stall_per_kernel,
                         per_kernel_resident);
}

// The engine program: the scheduler's transfers (start order per run) and
// kernel start times, as the executor consumes them.
extern "C" int tio_schedule(const tio_trace_desc *d, const tio_entry *entries, int64_t num_entries, int64_t capacity,
                            const tio_rates *rates, tio_transfer_rec *transfers, int64_t transfers_cap,
                            int64_t *num_transfers, int64_t *kernel_start, int64_t *kernel_seq,
                            int8_t *initial_loc) {
    if (!d || !rates || !num_transfers) return fail(TIO_ERR_INVALID, "null argument");
    SchedInput in;
    in.N = d->num_kernels; in.T = d->num_tensors;
    in.dur = d->duration_us; in.tid = d->tensor_id; in.size = d->size_bytes; in.kind = d->kind;
    in.ptr = d->access_ptr; in.acc = d->accesses;
    std::vector<int64_t> e_tid(num_entries), e_trig(num_entries), e_dl(num_entries);
    std::vector<int32_t> e_act(num_entries), e_tgt(num_entries), e_urg(num_entries);
    for (int64_t i = 0; i < num_entries; ++i) {
        e_tid[i] = entries[i].tensor_id; e_trig[i] = entries[i].trigger_us; e_dl[i] = entries[i].deadline_us;
        e_act[i] = entries[i].action; e_tgt[i] = entries[i].target; e_urg[i] = entries[i].urgent;
    }
    in.num_entries = num_entries;
    in.e_tid = e_tid.data(); in.e_trigger = e_trig.data(); in.e_deadline = e_dl.data();
    in.e_action = e_act.data(); in.e_target = e_tgt.data(); in.e_urgent = e_urg.data();
    in.capacity = capacity;
    in.rate[0] = rates->ssd_offload; in.rate[1] = rates->ssd_prefetch;
    in.rate[2] = rates->host_offload; in.rate[3] = rates->host_prefetch;
    in.has_host = rates->has_host;
    SchedOutput out;
    std::string err;
    int rc = engine_schedule(in, &out, &err);
    if (rc != TIO_OK) return fail(rc, "%s", err.c_str());
    *num_transfers = (int64_t)out.transfers.size();
    if (transfers) {
        if (transfers_cap < *num_transfers) return fail(TIO_ERR_INVALID, "transfers buffer too small");
        for (size_t i = 0; i < out.transfers.size(); ++i) {
            const SchedTransfer &s = out.transfers[i];
            tio_transfer_rec &r = transfers[i];
            r.tensor_pos = s.tensor; r.tensor_id = in.tid[s.tensor]; r.action = s.action;
            r.device = s.device == LOC_SSD ? TIO_DEST_SSD : TIO_DEST_CPU;
            r.urgent = s.urgent; r.emergency = s.emergency; r.start_us = s.start; r.end_us = s.end;
            r.after_kernel = s.issue_kernel; r.tail = s.tail; r.seq = s.seq;
        }
    }
    if (kernel_start && in.N) memcpy(kernel_start, out.start.data(), sizeof(int64_t) * in.N);
    if (kernel_seq && in.N) memcpy(kernel_seq, out.kseq.data(), sizeof(int64_t) * in.N);
    if (initial_loc && in.T) memcpy(initial_loc, out.initial_loc.data(), (size_t)in.T);
    return TIO_OK;
}
