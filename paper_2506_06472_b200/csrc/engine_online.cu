// engine_online.cu — the migration engine driving a REAL training step.
//
// tio_engine_replay (engine.cu) executes a whole iteration against
// placeholder kernels.  This file is the online form a framework hook calls
// around every operator of the real step (reference semantics:
// simulator.py:178-528 `_Engine`; runtime design PAPER.md:429-444, a
// location table plus GPU<->storage transfers gated on kernel progress):
//
//   tio_engine_create        schedule the plan once (engine_sched.cu: the
//                            reference engine's exact decisions over the
//                            profiled durations) and build the program: the
//                            transfers and kernel launches in the model's
//                            processing order;
//   tio_engine_before_kernel issue every transfer the program places before
//                            kernel k on its channel stream, then make the
//                            compute stream wait for what kernel k needs
//                            (simulator.py:430-469 `_try_launch`: its tensors'
//                            prefetches; memory the model frees first);
//   tio_engine_after_kernel  record kernel k's completion event, bind the
//                            device addresses of tensors k created;
//   tio_engine_step_end      issue the transfers placed after the last kernel.
//
// Device memory stays the framework's: an offload copies the tensor to its
// 4 KB-aligned pinned host extent on the channel stream and calls
// free_cb(tensor, channel stream) (the host frees the storage once the copy is
// done — e.g. PyTorch record_stream + storage resize to 0); a prefetch calls
// alloc_cb(tensor, bytes) on the host thread (the framework allocates on the
// compute stream), makes the channel wait for the compute stream's current
// position (the allocation is safe from there on) and copies back.
//
// Steady state across steps: the plan is folded to one periodic iteration
// (simulator.py:243-293), so the program of every step is the same.  A
// boundary-straddling transfer the scheduler pre-installs as running at t=0
// (`tail`) IS the previous step's late transfer of the same tensor: in step 1
// the engine issues it at the start (after moving every tensor whose
// steady-state location at t=0 is off the GPU there), in later steps it only
// points the tensor's dependency at that previous transfer's event.
//
// Verification (cfg.verify): a position-dependent 64-bit checksum of every
// offloaded tensor is taken on the channel stream before the D2H copy and
// re-taken after every prefetch; mismatches are counted on the device.

#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "engine_sched.cuh"

namespace tio {

__device__ __forceinline__ uint64_t cs_mix(uint64_t x) {
    x ^= x >> 31; x *= 0x7fb5d329728ea185ull;
    x ^= x >> 27; x *= 0x81dadef4bc2dd44dull;
    x ^= x >> 33;
    return x;
}

// sum over 8-byte words of mix(word + index * golden) (+ tail bytes): order
// independent, so blocks add their partial sums atomically
__global__ void k_checksum(const uint8_t *p, int64_t bytes, unsigned long long *out) {
    const int64_t words = bytes >> 3;
    const uint64_t *w = reinterpret_cast<const uint64_t *>(p);
    uint64_t acc = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 2;
    int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 2;
    const bool al16 = (reinterpret_cast<uintptr_t>(p) & 15) == 0;
    for (; i + 1 < words; i += stride) {
        uint64_t a, b;
        if (al16) {
            const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2 *>(w + i));
            a = v.x; b = v.y;
        } else {
            a = w[i]; b = w[i + 1];
        }
        acc += cs_mix(a + (uint64_t)i * 0x9e3779b97f4a7c15ull) + cs_mix(b + (uint64_t)(i + 1) * 0x9e3779b97f4a7c15ull);
    }
    if (i < words) acc += cs_mix(w[i] + (uint64_t)i * 0x9e3779b97f4a7c15ull);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        uint64_t t = 0;
        for (int64_t b = words << 3; b < bytes; ++b) t = (t << 8) | p[b];
        acc += cs_mix(t ^ 0xabcdefull ^ (uint64_t)bytes);
    }
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(out, (unsigned long long)acc);
}

// after a prefetch: compare the re-taken checksum with the offload's
__global__ void k_checksum_compare(const unsigned long long *a, const unsigned long long *b,
                                   unsigned long long *bad) {
    if (*a != *b) atomicAdd(bad, 1ull);
}

static int launch_checksum(const void *p, int64_t bytes, unsigned long long *out, cudaStream_t s) {
    TIO_CUDA(cudaMemsetAsync(out, 0, sizeof(unsigned long long), s));
    int64_t blocks = (bytes / 16 + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    k_checksum<<<(unsigned)blocks, 256, 0, s>>>(static_cast<const uint8_t *>(p), bytes, out);
    count_launch();
    TIO_CUDA(cudaGetLastError());
    return TIO_OK;
}

}  // namespace tio

using namespace tio;

// CUDA calls of the engine are skipped in a dry (program-check) engine
#define GPU(expr) do { if (!dry) TIO_CUDA(expr); } while (0)
#define EGPU(expr) do { if (!E->dry) TIO_CUDA(expr); } while (0)

struct tio_engine {
    // owned trace columns + plan (the caller's arrays need not outlive create)
    std::vector<int64_t> dur, tid, size, ptr;
    std::vector<int8_t> kind;
    std::vector<int32_t> acc;
    std::vector<int64_t> e_tid, e_trig, e_dl;
    std::vector<int32_t> e_act, e_tgt, e_urg;
    SchedInput in;
    SchedOutput sc;
    tio_engine_config cfg{};
    int64_t N = 0, T = 0, X = 0;

    struct Op { int64_t seq; int kind; int64_t idx; };   // kind 0 transfer, 1 kernel
    std::vector<Op> ops;
    std::vector<int64_t> kop;                // op position of kernel k
    std::vector<int64_t> straddler;          // tail transfer -> the late transfer it continues (-1: none)
    std::vector<int64_t> act_ptr, act;       // tensors of each kernel
    std::vector<int64_t> first_k, last_acc;  // per tensor: first / last access
    std::vector<uint8_t> movable;            // tensor ever transferred / starts off the GPU

    cudaStream_t comp = nullptr, ch[4] = {nullptr, nullptr, nullptr, nullptr};
    std::vector<cudaEvent_t> kdone, xdone, xt0, xt1;
    std::vector<cudaEvent_t> pool;
    cudaEvent_t alloc_ev = nullptr;
    std::vector<void *> dptr;
    std::vector<int64_t> hoff;
    uint8_t *host = nullptr;
    int64_t host_bytes = 0;
    std::vector<int64_t> last_x, last_k;
    std::vector<std::pair<int64_t, int64_t>> offs_done[2];
    unsigned long long *dcs = nullptr;       // [T] offload checksums, [T] prefetch checksums, [1] bad

    tio_alloc_cb alloc_cb = nullptr;
    tio_free_cb free_cb = nullptr;
    void *user = nullptr;

    int64_t step = 0, cursor = 0, next_kernel = 0;
    bool in_step = false;
    bool dry = false;                        // program walk only: no CUDA calls, internal callbacks
    int64_t bytes_dir[2] = {0, 0}, count_dir[2] = {0, 0};
    std::vector<uint8_t> issued_this_step;
    std::vector<int8_t> xact_rec;            // action of each reconciliation slot
    std::vector<uint8_t> end_resident;       // per global: resident when the next step begins (program view)
    std::vector<uint8_t> reconciled;         // per tensor: moved by the last step_end's reconciliation
    int64_t n_reconcile = 0, bytes_reconcile = 0;

    ~tio_engine() {
        if (dry) return;
        if (comp) cudaStreamSynchronize(comp);
        for (int c = 0; c < 4; ++c) if (ch[c]) { cudaStreamSynchronize(ch[c]); cudaStreamDestroy(ch[c]); }
        for (auto e : pool) cudaEventDestroy(e);
        if (alloc_ev) cudaEventDestroy(alloc_ev);
        if (host) cudaFreeHost(host);
        if (dcs) cudaFree(dcs);
    }
    int mk_event(cudaEvent_t *e, bool timing) {
        GPU(cudaEventCreateWithFlags(e, timing ? cudaEventDefault : cudaEventDisableTiming));
        pool.push_back(*e);
        return TIO_OK;
    }
    int64_t latest_off_before(int dv, int64_t t) const {
        const auto &v = offs_done[dv];
        int64_t lo = 0, hi = (int64_t)v.size();
        while (lo < hi) {
            const int64_t m = (lo + hi) >> 1;
            if (v[m].first <= t) lo = m + 1; else hi = m;
        }
        return lo > 0 ? v[lo - 1].second : -1;
    }
    int channel_of(const SchedTransfer &x) const { return (x.device == LOC_SSD ? 0 : 2) + x.action; }

    // transfer slots: [0, X) the program's transfers, [X, X + T) one
    // reconciliation slot per tensor (step_end)
    int64_t slot_action(int64_t slot) const {
        return slot < X ? sc.transfers[slot].action : xact_rec[slot - X];
    }
    int offload(int64_t t, int c, int64_t slot, int64_t wait_kernel) {
        const int64_t nb = size[t];
        cudaStream_t s = ch[c];
        if (wait_kernel >= 0) GPU(cudaStreamWaitEvent(s, kdone[wait_kernel], 0));
        if (last_x[t] >= 0) GPU(cudaStreamWaitEvent(s, xdone[last_x[t]], 0));
        if (last_k[t] >= 0) GPU(cudaStreamWaitEvent(s, kdone[last_k[t]], 0));
        if (!dptr[t])
            return fail(TIO_ERR_INTERNAL, "step %lld: offload of tensor %lld that is not resident / not bound",
                        (long long)step, (long long)tid[t]);
        if (cfg.verify && !dry) TIO_TRY(launch_checksum(dptr[t], nb, dcs + t, s));
        GPU(cudaEventRecord(xt0[slot], s));
        GPU(cudaMemcpyAsync(host + hoff[t], dptr[t], (size_t)nb, cudaMemcpyDeviceToHost, s));
        GPU(cudaEventRecord(xt1[slot], s));
        if (free_cb(user, t, (void *)s) != 0)
            return fail(TIO_ERR_INVALID, "free callback failed for tensor %lld", (long long)tid[t]);
        dptr[t] = nullptr;
        GPU(cudaEventRecord(xdone[slot], s));
        last_x[t] = slot;
        return TIO_OK;
    }
    int prefetch(int64_t t, int c, int64_t slot, int64_t mem_time) {
        const int64_t nb = size[t];
        cudaStream_t s = ch[c];
        // the model reserves memory at prefetch start once the offloads it
        // counted as complete have freed theirs (simulator.py:353-354)
        if (mem_time >= 0)
            for (int dv = 0; dv < 2; ++dv) {
                const int64_t lo = latest_off_before(dv, mem_time);
                if (lo >= 0) GPU(cudaStreamWaitEvent(s, xdone[lo], 0));
            }
        if (last_x[t] >= 0) GPU(cudaStreamWaitEvent(s, xdone[last_x[t]], 0));
        if (dptr[t])
            return fail(TIO_ERR_INTERNAL, "step %lld: prefetch of resident tensor %lld", (long long)step,
                        (long long)tid[t]);
        void *p = nullptr;
        if (alloc_cb(user, t, nb, &p) != 0 || !p)
            return fail(TIO_ERR_NOMEM, "alloc callback failed for tensor %lld (%lld bytes)", (long long)tid[t],
                        (long long)nb);
        // the framework allocated in compute-stream order: the block is free
        // for the channel only once the compute stream reaches this point
        GPU(cudaEventRecord(alloc_ev, comp));
        GPU(cudaStreamWaitEvent(s, alloc_ev, 0));
        dptr[t] = p;
        GPU(cudaEventRecord(xt0[slot], s));
        GPU(cudaMemcpyAsync(p, host + hoff[t], (size_t)nb, cudaMemcpyHostToDevice, s));
        GPU(cudaEventRecord(xt1[slot], s));
        if (cfg.verify && !dry) {
            TIO_TRY(launch_checksum(p, nb, dcs + T + t, s));
            k_checksum_compare<<<1, 1, 0, s>>>(dcs + t, dcs + T + t, dcs + 2 * T);
            count_launch();
        }
        GPU(cudaEventRecord(xdone[slot], s));
        last_x[t] = slot;
        return TIO_OK;
    }
    int transfer(int64_t xi) {
        const SchedTransfer &x = sc.transfers[xi];
        const int64_t t = x.tensor;
        const int dv = x.device == LOC_SSD ? 0 : 1;
        if (x.tail && step > 0) {
            // already running: the previous step's late transfer of this
            // tensor (unless step_end had to reconcile the tensor instead)
            const int64_t y = straddler[xi];
            if (!reconciled[t] && y >= 0) last_x[t] = y;
            if (x.action == 0) offs_done[dv].push_back({x.end, last_x[t]});
            return TIO_OK;
        }
        if (x.action == 0) TIO_TRY(offload(t, channel_of(x), xi, x.tail ? -1 : x.issue_kernel));
        else TIO_TRY(prefetch(t, channel_of(x), xi, x.start));
        if (x.action == 0) offs_done[dv].push_back({x.end, xi});
        bytes_dir[x.action] += size[t];
        count_dir[x.action] += 1;
        issued_this_step[xi] = 1;
        return TIO_OK;
    }
    // after the step's program: every movable global must be where the next
    // step's program expects it (the one-iteration model does not carry state
    // across iterations: e.g. a Belady emergency eviction of a global whose
    // next use is in the next iteration, simulator.py:414-469)
    int reconcile() {
        std::fill(reconciled.begin(), reconciled.end(), 0);
        for (int64_t t = 0; t < T; ++t) {
            if (!movable[t] || kind[t] != TIO_KIND_GLOBAL) continue;
            const bool res = dptr[t] != nullptr;
            if (res == (bool)end_resident[t]) continue;
            const int64_t slot = X + t;
            if (end_resident[t]) {
                xact_rec[t] = 1;
                TIO_TRY(prefetch(t, 1, slot, -1));
            } else {
                xact_rec[t] = 0;
                TIO_TRY(offload(t, 0, slot, -1));
            }
            reconciled[t] = 1;
            n_reconcile += 1;
            bytes_reconcile += size[t];
        }
        return TIO_OK;
    }
    // process program ops up to (excluding) position `until`
    int advance(int64_t until) {
        for (; cursor < until; ++cursor) {
            const Op &op = ops[cursor];
            if (op.kind == 0) TIO_TRY(transfer(op.idx));
        }
        return TIO_OK;
    }
};

static inline int64_t align4k(int64_t x) { return (x + 4095) & ~(int64_t)4095; }

static int engine_create(const tio_trace_desc *d, const tio_entry *entries, int64_t num_entries,
                         const tio_engine_config *cfg, void *compute_stream, tio_alloc_cb alloc_cb,
                         tio_free_cb free_cb, void *user, bool dry, tio_engine **out) {
    if (!d || !cfg || !out || (!dry && (!alloc_cb || !free_cb)) || (num_entries > 0 && !entries))
        return fail(TIO_ERR_INVALID, "null argument");
    *out = nullptr;
    tio_engine *E = new tio_engine();
    std::unique_ptr<tio_engine> guard(E);
    E->dry = dry;
    const int64_t N = d->num_kernels, T = d->num_tensors;
    E->N = N; E->T = T;
    E->dur.assign(d->duration_us, d->duration_us + N);
    E->tid.assign(d->tensor_id, d->tensor_id + T);
    E->size.assign(d->size_bytes, d->size_bytes + T);
    E->kind.assign(d->kind, d->kind + T);
    E->ptr.assign(d->access_ptr, d->access_ptr + T + 1);
    E->acc.assign(d->accesses, d->accesses + d->num_events);
    for (int64_t i = 0; i < num_entries; ++i) {
        E->e_tid.push_back(entries[i].tensor_id); E->e_trig.push_back(entries[i].trigger_us);
        E->e_dl.push_back(entries[i].deadline_us); E->e_act.push_back(entries[i].action);
        E->e_tgt.push_back(entries[i].target); E->e_urg.push_back(entries[i].urgent);
    }
    E->cfg = *cfg;
    SchedInput &in = E->in;
    in.N = N; in.T = T;
    in.dur = E->dur.data(); in.tid = E->tid.data(); in.size = E->size.data(); in.kind = E->kind.data();
    in.ptr = E->ptr.data(); in.acc = E->acc.data();
    in.num_entries = num_entries;
    in.e_tid = E->e_tid.data(); in.e_trigger = E->e_trig.data(); in.e_deadline = E->e_dl.data();
    in.e_action = E->e_act.data(); in.e_target = E->e_tgt.data(); in.e_urgent = E->e_urg.data();
    in.capacity = cfg->capacity;
    in.rate[0] = cfg->rates.ssd_offload; in.rate[1] = cfg->rates.ssd_prefetch;
    in.rate[2] = cfg->rates.host_offload; in.rate[3] = cfg->rates.host_prefetch;
    in.has_host = cfg->rates.has_host;
    {
        std::string err;
        const int rc = engine_schedule(in, &E->sc, &err);
        if (rc != TIO_OK) return fail(rc, "%s", err.c_str());
    }
    const SchedOutput &sc = E->sc;
    const int64_t X = (int64_t)sc.transfers.size();
    E->X = X;
    // program: transfers and kernel launches in the model's processing order
    E->ops.reserve(X + N);
    for (int64_t i = 0; i < X; ++i) E->ops.push_back({sc.transfers[i].seq, 0, i});
    for (int64_t k = 0; k < N; ++k) E->ops.push_back({sc.kseq[k], 1, k});
    std::sort(E->ops.begin(), E->ops.end(), [](const tio_engine::Op &a, const tio_engine::Op &b) { return a.seq < b.seq; });
    E->kop.assign(N, -1);
    for (int64_t i = 0; i < (int64_t)E->ops.size(); ++i)
        if (E->ops[i].kind == 1) E->kop[E->ops[i].idx] = i;
    // tails continue the last non-tail transfer of the same tensor and action
    E->straddler.assign(X, -1);
    for (int64_t i = 0; i < X; ++i) {
        const SchedTransfer &x = sc.transfers[i];
        if (!x.tail) continue;
        int64_t best = -1;
        for (int64_t j = 0; j < X; ++j) {
            const SchedTransfer &y = sc.transfers[j];
            if (y.tail || y.tensor != x.tensor || y.action != x.action || y.emergency) continue;
            if (best < 0 || y.seq > sc.transfers[best].seq) best = j;
        }
        // none: the step never issues it (skipped / cancelled in the model);
        // step_end's reconciliation then performs the boundary move
        E->straddler[i] = best;
    }
    // kernel -> tensors; per-tensor first / last access
    E->act_ptr.assign(N + 1, 0);
    for (int64_t t = 0; t < T; ++t)
        for (int64_t j = E->ptr[t]; j < E->ptr[t + 1]; ++j) E->act_ptr[E->acc[j] + 1]++;
    for (int64_t k = 0; k < N; ++k) E->act_ptr[k + 1] += E->act_ptr[k];
    E->act.assign(E->act_ptr[N], 0);
    {
        std::vector<int64_t> fill(E->act_ptr.begin(), E->act_ptr.end() - 1);
        for (int64_t t = 0; t < T; ++t)
            for (int64_t j = E->ptr[t]; j < E->ptr[t + 1]; ++j) E->act[fill[E->acc[j]]++] = t;
    }
    E->first_k.assign(T, -1);
    E->last_acc.assign(T, -1);
    for (int64_t t = 0; t < T; ++t)
        if (E->ptr[t + 1] > E->ptr[t]) { E->first_k[t] = E->acc[E->ptr[t]]; E->last_acc[t] = E->acc[E->ptr[t + 1] - 1]; }
    E->movable.assign(T, 0);
    E->hoff.assign(T, -1);
    for (int64_t i = 0; i < X; ++i) E->movable[sc.transfers[i].tensor] = 1;
    for (int64_t t = 0; t < T; ++t)
        if (sc.initial_loc[t] == LOC_SSD || sc.initial_loc[t] == LOC_HOST) E->movable[t] = 1;
    for (int64_t t = 0; t < T; ++t)
        if (E->movable[t]) { E->hoff[t] = E->host_bytes; E->host_bytes += align4k(E->size[t]); }
    E->dptr.assign(T, nullptr);
    E->last_x.assign(T, -1);
    E->last_k.assign(T, -1);
    E->issued_this_step.assign(X, 0);
    E->xact_rec.assign(T, 0);
    E->reconciled.assign(T, 0);
    // residency of each global when a step begins, as the program leaves it:
    // a boundary transfer's direction decides, else the folded t = 0 location
    E->end_resident.assign(T, 0);
    for (int64_t t = 0; t < T; ++t) E->end_resident[t] = sc.initial_loc[t] == LOC_GPU;
    for (int64_t i = 0; i < X; ++i)
        if (sc.transfers[i].tail) E->end_resident[sc.transfers[i].tensor] = sc.transfers[i].action == 1;
    E->alloc_cb = alloc_cb; E->free_cb = free_cb; E->user = user;
    if (dry) {
        *out = guard.release();
        return TIO_OK;
    }
    // resources
    E->comp = (cudaStream_t)compute_stream;
    for (int c = 0; c < 4; ++c) TIO_CUDA(cudaStreamCreateWithFlags(&E->ch[c], cudaStreamNonBlocking));
    if (E->host_bytes) TIO_CUDA(cudaHostAlloc((void **)&E->host, (size_t)E->host_bytes, cudaHostAllocPortable));
    TIO_CUDA(cudaMalloc((void **)&E->dcs, sizeof(unsigned long long) * (2 * T + 2)));
    TIO_CUDA(cudaMemset(E->dcs, 0, sizeof(unsigned long long) * (2 * T + 2)));
    E->kdone.resize(N); E->xdone.resize(X + T); E->xt0.resize(X + T); E->xt1.resize(X + T);
    for (int64_t k = 0; k < N; ++k) TIO_TRY(E->mk_event(&E->kdone[k], false));
    for (int64_t i = 0; i < X + T; ++i) {
        if (i >= X && !(E->movable[i - X] && E->kind[i - X] == TIO_KIND_GLOBAL)) continue;
        TIO_TRY(E->mk_event(&E->xdone[i], false));
        TIO_TRY(E->mk_event(&E->xt0[i], true));
        TIO_TRY(E->mk_event(&E->xt1[i], true));
    }
    TIO_CUDA(cudaEventCreateWithFlags(&E->alloc_ev, cudaEventDisableTiming));
    *out = guard.release();
    return TIO_OK;
}

extern "C" int tio_engine_create(const tio_trace_desc *d, const tio_entry *entries, int64_t num_entries,
                                 const tio_engine_config *cfg, void *compute_stream, tio_alloc_cb alloc_cb,
                                 tio_free_cb free_cb, void *user, tio_engine **out) {
    return engine_create(d, entries, num_entries, cfg, compute_stream, alloc_cb, free_cb, user, false, out);
}

// dry engine callbacks: a fake, non-null address per tensor; frees are no-ops
static int dry_alloc(void *, int64_t t, int64_t, void **p) {
    *p = reinterpret_cast<void *>((uintptr_t)(0x10000 + 16 * t));
    return 0;
}
static int dry_free(void *, int64_t, void *) { return 0; }

extern "C" int tio_engine_check_program(const tio_trace_desc *d, const tio_entry *entries, int64_t num_entries,
                                        const tio_engine_config *cfg, int64_t steps, tio_engine_info_t *info) {
    tio_engine *E = nullptr;
    TIO_TRY(engine_create(d, entries, num_entries, cfg, nullptr, dry_alloc, dry_free, nullptr, true, &E));
    std::unique_ptr<tio_engine> guard(E);
    if (info) TIO_TRY(tio_engine_info(E, info, nullptr));
    // globals exist before the step (bound); intermediates when created
    for (int64_t t = 0; t < E->T; ++t)
        if (E->kind[t] == TIO_KIND_GLOBAL && E->movable[t]) dry_alloc(nullptr, t, 0, &E->dptr[t]);
    std::vector<int64_t> npos;
    std::vector<void *> nptr;
    for (int64_t st = 0; st < steps; ++st) {
        TIO_TRY(tio_engine_step_begin(E));
        for (int64_t k = 0; k < E->N; ++k) {
            TIO_TRY(tio_engine_before_kernel(E, k));
            npos.clear(); nptr.clear();
            for (int64_t j = E->act_ptr[k]; j < E->act_ptr[k + 1]; ++j) {
                const int64_t t = E->act[j];
                if (E->kind[t] != TIO_KIND_GLOBAL && E->first_k[t] == k && E->movable[t]) {
                    npos.push_back(t);
                    void *p;
                    dry_alloc(nullptr, t, 0, &p);
                    nptr.push_back(p);
                }
            }
            TIO_TRY(tio_engine_after_kernel(E, k, (int64_t)npos.size(), npos.data(), nptr.data()));
        }
        TIO_TRY(tio_engine_step_end(E, nullptr));
    }
    return TIO_OK;
}

extern "C" int tio_engine_info(const tio_engine *E, tio_engine_info_t *info, uint8_t *movable);
extern "C" int tio_engine_info(const tio_engine *E, tio_engine_info_t *info, uint8_t *movable) {
    if (!E || !info) return fail(TIO_ERR_INVALID, "null argument");
    memset(info, 0, sizeof(*info));
    const SchedOutput &sc = E->sc;
    info->num_kernels = E->N; info->num_tensors = E->T; info->num_transfers = E->X;
    info->host_bytes = E->host_bytes;
    info->model_total_us = sc.total_time; info->model_ideal_us = sc.ideal_time;
    info->model_stall_us = sc.stall_total; info->model_peak_resident = sc.peak_resident;
    info->emergency_offloads = sc.emergency;
    for (const auto &x : sc.transfers) {
        if (x.action == 0) { info->model_offload_bytes += E->size[x.tensor]; info->model_offloads++; }
        else { info->model_prefetch_bytes += E->size[x.tensor]; info->model_prefetches++; }
    }
    if (movable) memcpy(movable, E->movable.data(), (size_t)E->T);
    return TIO_OK;
}

extern "C" int tio_engine_bind(tio_engine *E, int64_t n, const int64_t *tensor_pos, void *const *dev_ptr) {
    if (!E || (n > 0 && (!tensor_pos || !dev_ptr))) return fail(TIO_ERR_INVALID, "null argument");
    for (int64_t i = 0; i < n; ++i) {
        const int64_t t = tensor_pos[i];
        if (t < 0 || t >= E->T) return fail(TIO_ERR_INVALID, "tensor position %lld out of range", (long long)t);
        E->dptr[t] = dev_ptr[i];
    }
    return TIO_OK;
}

extern "C" int tio_engine_step_begin(tio_engine *E) {
    if (!E) return fail(TIO_ERR_INVALID, "null engine");
    if (E->in_step) return fail(TIO_ERR_INVALID, "step already begun");
    if (E->step == 0) {
        // move every tensor whose steady-state location at t = 0 is off the
        // GPU (incl. those a boundary prefetch is bringing back) to its extent
        for (int64_t t = 0; t < E->T; ++t) {
            const int8_t l = E->sc.initial_loc[t];
            if (l != LOC_SSD && l != LOC_HOST) continue;
            if (!E->dptr[t])
                return fail(TIO_ERR_INVALID, "tensor %lld starts the step off the GPU but was never bound",
                            (long long)E->tid[t]);
            if (E->cfg.verify && !E->dry) TIO_TRY(launch_checksum(E->dptr[t], E->size[t], E->dcs + t, E->comp));
            EGPU(cudaMemcpyAsync(E->host + E->hoff[t], E->dptr[t], (size_t)E->size[t], cudaMemcpyDeviceToHost,
                                     E->comp));
            EGPU(cudaStreamSynchronize(E->comp));
            if (E->free_cb(E->user, t, (void *)E->comp) != 0)
                return fail(TIO_ERR_INVALID, "free callback failed for tensor %lld", (long long)E->tid[t]);
            E->dptr[t] = nullptr;
        }
    }
    for (int dv = 0; dv < 2; ++dv) E->offs_done[dv].clear();
    std::fill(E->issued_this_step.begin(), E->issued_this_step.end(), 0);
    E->cursor = 0;
    E->next_kernel = 0;
    E->in_step = true;
    return TIO_OK;
}

extern "C" int tio_engine_before_kernel(tio_engine *E, int64_t k) {
    if (!E || !E->in_step) return fail(TIO_ERR_INVALID, "no step in progress");
    if (k != E->next_kernel)
        return fail(TIO_ERR_INVALID, "kernel %lld launched out of order (expected %lld): the step diverges from the "
                    "profiled trace", (long long)k, (long long)E->next_kernel);
    TIO_TRY(E->advance(E->kop[k]));
    // gate kernel k on its tensors' prefetches and on the memory the model
    // frees before it starts (simulator.py:430-469)
    bool creates = false;
    for (int64_t j = E->act_ptr[k]; j < E->act_ptr[k + 1]; ++j) {
        const int64_t t = E->act[j], xi = E->last_x[t];
        if (xi >= 0 && E->slot_action(xi) == 1) EGPU(cudaStreamWaitEvent(E->comp, E->xdone[xi], 0));
        if (E->first_k[t] == k && E->kind[t] != TIO_KIND_GLOBAL) creates = true;
        else if (E->movable[t] && !E->dptr[t])
            return fail(TIO_ERR_INTERNAL, "kernel %lld needs tensor %lld that is off the GPU", (long long)k,
                        (long long)E->tid[t]);
    }
    if (creates)
        for (int dv = 0; dv < 2; ++dv) {
            const int64_t lo = E->latest_off_before(dv, E->sc.start[k]);
            if (lo >= 0) EGPU(cudaStreamWaitEvent(E->comp, E->xdone[lo], 0));
        }
    E->cursor = E->kop[k] + 1;
    return TIO_OK;
}

extern "C" int tio_engine_after_kernel(tio_engine *E, int64_t k, int64_t n_new, const int64_t *new_pos,
                                       void *const *new_ptr) {
    if (!E || !E->in_step) return fail(TIO_ERR_INVALID, "no step in progress");
    if (k != E->next_kernel) return fail(TIO_ERR_INVALID, "after_kernel(%lld) without before_kernel", (long long)k);
    EGPU(cudaEventRecord(E->kdone[k], E->comp));
    for (int64_t j = E->act_ptr[k]; j < E->act_ptr[k + 1]; ++j) E->last_k[E->act[j]] = k;
    TIO_TRY(tio_engine_bind(E, n_new, new_pos, new_ptr));
    // an intermediate's storage is the framework's to free after its last use
    for (int64_t j = E->act_ptr[k]; j < E->act_ptr[k + 1]; ++j) {
        const int64_t t = E->act[j];
        if (E->kind[t] != TIO_KIND_GLOBAL && E->last_acc[t] == k) E->dptr[t] = nullptr;
    }
    E->next_kernel = k + 1;
    return TIO_OK;
}

extern "C" int tio_engine_step_end(tio_engine *E, void *done_stream) {
    if (!E || !E->in_step) return fail(TIO_ERR_INVALID, "no step in progress");
    if (E->next_kernel != E->N)
        return fail(TIO_ERR_INVALID, "step ended after %lld of %lld kernels: the step diverges from the profiled "
                    "trace", (long long)E->next_kernel, (long long)E->N);
    TIO_TRY(E->advance((int64_t)E->ops.size()));
    TIO_TRY(E->reconcile());
    if (done_stream) {
        // make `done_stream` wait for every transfer of the step (end-of-step
        // fence for timing; the steady state does not need it)
        for (int c = 0; c < 4; ++c) {
            EGPU(cudaEventRecord(E->alloc_ev, E->ch[c]));
            EGPU(cudaStreamWaitEvent((cudaStream_t)done_stream, E->alloc_ev, 0));
        }
    }
    E->in_step = false;
    E->step += 1;
    return TIO_OK;
}

extern "C" int tio_engine_step_abort(tio_engine *E) {
    if (!E) return fail(TIO_ERR_INVALID, "null engine");
    if (!E->dry) {
        for (int c = 0; c < 4; ++c) TIO_CUDA(cudaStreamSynchronize(E->ch[c]));
        TIO_CUDA(cudaStreamSynchronize(E->comp));
    }
    E->in_step = false;
    // tensors the aborted step created are gone; globals keep their state
    for (int64_t t = 0; t < E->T; ++t)
        if (E->kind[t] != TIO_KIND_GLOBAL) E->dptr[t] = nullptr;
    return TIO_OK;
}

extern "C" int tio_engine_stats_get(tio_engine *E, tio_engine_online_stats *st) {
    if (!E || !st) return fail(TIO_ERR_INVALID, "null argument");
    memset(st, 0, sizeof(*st));
    for (int c = 0; c < 4; ++c) EGPU(cudaStreamSynchronize(E->ch[c]));
    EGPU(cudaStreamSynchronize(E->comp));
    st->steps = E->step;
    st->offload_bytes = E->bytes_dir[0]; st->prefetch_bytes = E->bytes_dir[1];
    st->n_offloads = E->count_dir[0]; st->n_prefetches = E->count_dir[1];
    // per-copy device time of the last step's transfers
    for (int64_t i = 0; i < E->X; ++i) {
        if (!E->issued_this_step[i]) continue;
        float m = 0.f;
        if (cudaEventElapsedTime(&m, E->xt0[i], E->xt1[i]) != cudaSuccess) { cudaGetLastError(); continue; }
        const SchedTransfer &x = E->sc.transfers[i];
        if (x.action == 0) { st->last_offload_busy_ms += m; st->last_offload_bytes += E->size[x.tensor]; }
        else { st->last_prefetch_busy_ms += m; st->last_prefetch_bytes += E->size[x.tensor]; }
    }
    unsigned long long bad = 0;
    EGPU(cudaMemcpy(&bad, E->dcs + 2 * E->T, sizeof(bad), cudaMemcpyDeviceToHost));
    st->verify_mismatches = (int64_t)bad;
    st->verify = E->cfg.verify;
    st->reconcile_transfers = E->n_reconcile;
    st->reconcile_bytes = E->bytes_reconcile;
    return TIO_OK;
}

extern "C" int tio_engine_restore(tio_engine *E) {
    if (!E) return fail(TIO_ERR_INVALID, "null engine");
    if (E->in_step) return fail(TIO_ERR_INVALID, "restore inside a step");
    for (int c = 0; c < 4; ++c) EGPU(cudaStreamSynchronize(E->ch[c]));
    EGPU(cudaStreamSynchronize(E->comp));
    // every global whose latest copy is its host extent comes back
    for (int64_t t = 0; t < E->T; ++t) {
        if (!E->movable[t] || E->kind[t] != TIO_KIND_GLOBAL || E->dptr[t]) continue;
        void *p = nullptr;
        if (E->alloc_cb(E->user, t, E->size[t], &p) != 0 || !p)
            return fail(TIO_ERR_NOMEM, "alloc callback failed for tensor %lld", (long long)E->tid[t]);
        EGPU(cudaStreamSynchronize(E->comp));
        EGPU(cudaMemcpy(p, E->host + E->hoff[t], (size_t)E->size[t], cudaMemcpyHostToDevice));
        E->dptr[t] = p;
    }
    std::fill(E->last_x.begin(), E->last_x.end(), -1);
    std::fill(E->last_k.begin(), E->last_k.end(), -1);
    E->step = 0;              // the next step sets the steady state up again
    return TIO_OK;
}

extern "C" int tio_engine_set_verify(tio_engine *E, int verify) {
    if (!E) return fail(TIO_ERR_INVALID, "null engine");
    E->cfg.verify = verify ? 1 : 0;
    return TIO_OK;
}

extern "C" int tio_checksum(const void *dev_ptr, int64_t bytes, unsigned long long *dev_out, void *stream) {
    if ((!dev_ptr && bytes > 0) || !dev_out || bytes < 0) return fail(TIO_ERR_INVALID, "bad argument");
    return launch_checksum(dev_ptr, bytes, dev_out, (cudaStream_t)stream);
}

extern "C" int tio_engine_destroy(tio_engine *E) {
    delete E;
    return TIO_OK;
}
