// engine_sched.cu — the migration engine's scheduler (host C++), a
// restatement of the reference runtime engine semantics (simulator.py:178-528)
// as an exact integer discrete-event model.  See engine_sched.cuh.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <queue>
#include <unordered_map>

#include "common.cuh"
#include "engine_sched.cuh"

namespace tio {

namespace {

enum { A_OFF = 0, A_PRE = 1 };
enum { K_COMPLETE = 0, K_ISSUE = 1 };

struct Tr {                 // simulator.py:78-87 _Transfer
    int64_t t, nbytes;
    int action, device;     // device: LOC_SSD / LOC_HOST
    bool urgent, emergency, started;
    int64_t end;
};

struct Issue {              // a (possibly folded) plan entry
    int64_t t, trigger, deadline;
    int action, target, urgent;
};

struct Ev {                 // heap key (time, prio, tensor_id, seq), simulator.py:295-297
    int64_t time;
    int prio;
    int64_t tid;
    int64_t seq;
    int kind;
    int64_t payload;
};

struct EvLess {             // min-heap via std::priority_queue
    bool operator()(const Ev &a, const Ev &b) const {
        if (a.time != b.time) return a.time > b.time;
        if (a.prio != b.prio) return a.prio > b.prio;
        if (a.tid != b.tid) return a.tid > b.tid;
        return a.seq > b.seq;
    }
};

struct Engine {
    const SchedInput &in;
    SchedOutput &out;
    std::string &err;
    int64_t N, T, cap, iteration = 0;
    std::vector<int64_t> act_ptr, act;          // active_at[k], sorted by tensor id
    std::vector<int8_t> loc;
    std::vector<int> engaged;                   // transfer index or -1
    int n_emergency_engaged = 0;
    std::vector<Tr> trs;
    std::vector<Issue> issues;
    std::vector<int> queue[4];
    int running[4] = {-1, -1, -1, -1};
    bool chan_exists[4] = {true, true, false, false};
    RateCode rc[4];
    std::vector<std::pair<int64_t, int64_t>> booked[4];
    std::vector<int64_t> tr_sched;              // transfer -> index in out.transfers
    std::priority_queue<Ev, std::vector<Ev>, EvLess> events;
    int64_t seq = 0, resident = 0, peak = 0;
    int64_t order = 0;                          // processing order of transfer starts and kernel launches
    // layer policy (simulator.py:95-177): blocks of consecutive kernels with
    // one layer id; tensors of each layer in id order; in-flight batch prefetches
    bool pol = false;
    std::vector<int64_t> blk_layer, blk_first, blk_last;
    std::vector<int64_t> block_of;
    std::unordered_map<int64_t, std::vector<int64_t>> layer_tensors;
    std::vector<char> outstanding;              // per transfer: an in-flight batch prefetch
    int64_t n_out = 0, exec_block = 0, next_batch = 0;

    Engine(const SchedInput &i, SchedOutput &o, std::string &e)
        : in(i), out(o), err(e), N(i.N), T(i.T), cap(i.capacity) {}

    int chan(int device, int action) const { return (device == LOC_SSD ? 0 : 2) + (action == A_OFF ? 0 : 1); }
    bool is_global(int64_t t) const { return in.kind[t] == 1; }

    void push(int64_t time, int prio, int64_t t, int kind, int64_t payload) {
        events.push(Ev{time, prio, in.tid[t], ++seq, kind, payload});
    }
    void grow(int64_t b) {
        resident += b;
        if (resident > peak) peak = resident;
    }
    void engage(int64_t t, int x) {
        engaged[t] = x;
        if (trs[x].emergency) ++n_emergency_engaged;
    }
    void disengage(int64_t t) {
        const int x = engaged[t];
        if (x >= 0 && trs[x].emergency) --n_emergency_engaged;
        engaged[t] = -1;
    }
    int64_t duration(int c, int64_t nbytes) const { return duration_of(rc[c], nbytes); }

    // simulator.py:309-313: first access after k; globals wrap to the next iteration
    bool next_use(int64_t t, int64_t k, int64_t *use) const {
        const int32_t *a = in.acc + in.ptr[t];
        const int64_t n = in.ptr[t + 1] - in.ptr[t];
        const int64_t i = std::upper_bound(a, a + n, (int32_t)k) - a;
        if (i < n) { *use = a[i]; return true; }
        if (is_global(t)) { *use = N + a[0]; return true; }
        return false;
    }

    void record_start(int x, int c, int64_t now, bool tail) {
        const Tr &tr = trs[x];
        booked[c].push_back({now, tr.end});
        SchedTransfer s;
        s.tensor = tr.t; s.action = tr.action; s.device = tr.device;
        s.urgent = tr.urgent; s.emergency = tr.emergency;
        s.start = now; s.end = tr.end; s.issue_kernel = -1; s.tail = tail ? 1 : 0; s.pad = 0;
        s.seq = order++;
        tr_sched[x] = (int64_t)out.transfers.size();
        out.transfers.push_back(s);
    }

    // simulator.py:349-363
    void pump(int c, int64_t now) {
        if (running[c] >= 0 || queue[c].empty()) return;
        const int x = queue[c].front();
        Tr &h = trs[x];
        if (h.action == A_PRE && resident + h.nbytes > cap) return;   // no room to land it yet
        queue[c].erase(queue[c].begin());
        h.started = true;
        h.end = now + duration(c, h.nbytes);
        running[c] = x;
        record_start(x, c, now, false);
        if (h.action == A_PRE) grow(h.nbytes);
        push(h.end, 0, h.t, K_COMPLETE, x);
    }
    void pump_all(int64_t now) {
        for (int c = 0; c < 4; ++c)
            if (chan_exists[c]) pump(c, now);
    }

    // simulator.py:315-327
    void enqueue(int x, int64_t now, bool front = false) {
        const Tr &tr = trs[x];
        const int c = chan(tr.device, tr.action);
        std::vector<int> &q = queue[c];
        if (front) {
            q.insert(q.begin(), x);
        } else if (tr.urgent) {
            size_t pos = 0;
            while (pos < q.size() && trs[q[pos]].urgent) ++pos;
            q.insert(q.begin() + pos, x);
        } else {
            q.push_back(x);
        }
        engage(tr.t, x);
        pump(c, now);
    }

    int new_tr(int64_t t, int action, int device, bool urgent, bool emergency) {
        Tr tr;
        tr.t = t; tr.nbytes = in.size[t]; tr.action = action; tr.device = device;
        tr.urgent = urgent; tr.emergency = emergency; tr.started = false; tr.end = 0;
        trs.push_back(tr);
        tr_sched.push_back(-1);
        outstanding.push_back(0);
        return (int)trs.size() - 1;
    }

    // simulator.py:329-335
    void cancel(int x) {
        for (int c = 0; c < 4; ++c) {
            auto it = std::find(queue[c].begin(), queue[c].end(), x);
            if (it != queue[c].end()) { queue[c].erase(it); break; }
        }
        disengage(trs[x].t);
    }

    // simulator.py:337-347
    void promote_front(int x, int64_t now) {
        for (int c = 0; c < 4; ++c) {
            auto it = std::find(queue[c].begin(), queue[c].end(), x);
            if (it != queue[c].end()) {
                queue[c].erase(it);
                trs[x].urgent = true;
                queue[c].insert(queue[c].begin(), x);
                pump(c, now);
                return;
            }
        }
    }

    // simulator.py:369-382
    void complete(int x, int64_t now) {
        Tr &tr = trs[x];
        const int c = chan(tr.device, tr.action);
        running[c] = -1;
        disengage(tr.t);
        if (tr.action == A_OFF) {
            resident -= tr.nbytes;
            loc[tr.t] = (int8_t)tr.device;
        } else {
            loc[tr.t] = LOC_GPU;
        }
        pump_all(now);
        if (pol) on_transfer_complete(x, now);
    }

    // ---- layer policy hooks (simulator.py:137-177)
    void maybe_issue(int64_t now) {
        const int64_t nblocks = (int64_t)blk_layer.size();
        while (n_out == 0 && next_batch < nblocks && next_batch <= exec_block + 1) {
            const int64_t batch = next_batch++;
            // the block's active tensors, in id order (_block_tensors)
            std::vector<int64_t> ts;
            for (int64_t k = blk_first[batch]; k <= blk_last[batch]; ++k)
                ts.insert(ts.end(), act.begin() + act_ptr[k], act.begin() + act_ptr[k + 1]);
            std::sort(ts.begin(), ts.end(), [&](int64_t x, int64_t y) { return in.tid[x] < in.tid[y]; });
            ts.erase(std::unique(ts.begin(), ts.end()), ts.end());
            for (int64_t t : ts) {
                if ((loc[t] == LOC_SSD || loc[t] == LOC_HOST) && engaged[t] < 0) {
                    const int x = new_tr(t, A_PRE, loc[t], false, false);
                    enqueue(x, now);
                    outstanding[x] = 1;
                    ++n_out;
                }
            }
        }
    }
    void on_transfer_complete(int x, int64_t now) {
        if (outstanding[x]) { outstanding[x] = 0; --n_out; }
        if (n_out == 0) maybe_issue(now);
    }
    void on_kernel_launched(int64_t k, int64_t now) {
        exec_block = block_of[k];
        maybe_issue(now);
    }
    void on_kernel_end(int64_t k, int64_t now) {
        const int64_t b = block_of[k];
        if (k != blk_last[b]) return;
        // the layer's still-needed GPU tensors go out as one batch, id order
        auto it = layer_tensors.find(blk_layer[b]);
        if (it != layer_tensors.end())
            for (int64_t t : it->second) {
                int64_t use;
                if (loc[t] == LOC_GPU && engaged[t] < 0 && next_use(t, k, &use))
                    enqueue(new_tr(t, A_OFF, LOC_SSD, false, false), now);
            }
        maybe_issue(now);
    }
    int setup_layer_policy() {
        // simulator.py:549-560: engaged only when the timeline peak exceeds capacity
        std::vector<int64_t> diff(N + 1, 0);
        int64_t glob = 0;
        for (int64_t t = 0; t < T; ++t) {
            if (in.ptr[t + 1] == in.ptr[t]) continue;
            if (is_global(t)) { glob += in.size[t]; continue; }
            diff[in.acc[in.ptr[t]]] += in.size[t];
            diff[in.acc[in.ptr[t + 1] - 1] + 1] -= in.size[t];
        }
        int64_t run = 0, pk = 0;
        for (int64_t k = 0; k < N; ++k) {
            run += diff[k];
            if (glob + run > pk) pk = glob + run;
        }
        if (pk <= cap) return TIO_OK;
        const int64_t NONE = INT64_MIN;
        for (int64_t k = 0; k < N; ++k)
            if (in.k_layer[k] == NONE) {
                char b[96];
                snprintf(b, sizeof(b), "kernel %lld has no layer id", (long long)k);
                err = b;
                return TIO_ERR_CONFIG;
            }
        for (int64_t t = 0; t < T; ++t)
            if (in.t_layer[t] == NONE) {
                char b[96];
                snprintf(b, sizeof(b), "tensor %lld has no layer id", (long long)in.tid[t]);
                err = b;
                return TIO_ERR_CONFIG;
            }
        block_of.assign(N, 0);
        for (int64_t k = 0; k < N; ++k) {
            if (!blk_layer.empty() && blk_layer.back() == in.k_layer[k]) {
                blk_last.back() = k;
            } else {
                blk_layer.push_back(in.k_layer[k]);
                blk_first.push_back(k);
                blk_last.push_back(k);
            }
            block_of[k] = (int64_t)blk_layer.size() - 1;
        }
        std::vector<int64_t> by_id(T);
        for (int64_t t = 0; t < T; ++t) by_id[t] = t;
        std::sort(by_id.begin(), by_id.end(), [&](int64_t x, int64_t y) { return in.tid[x] < in.tid[y]; });
        for (int64_t t : by_id) layer_tensors[in.t_layer[t]].push_back(t);
        pol = true;
        return TIO_OK;
    }

    // simulator.py:384-397
    void issue_entry(const Issue &e, int64_t now) {
        const int64_t t = e.t;
        if (engaged[t] >= 0) return;                         // superseded by an urgent/emergency transfer
        if (e.action == A_OFF) {
            if (loc[t] != LOC_GPU) return;                   // already evicted at runtime
            enqueue(new_tr(t, A_OFF, e.target == TIO_DEST_CPU ? LOC_HOST : LOC_SSD, e.urgent != 0, false), now);
        } else {
            if (loc[t] != LOC_SSD && loc[t] != LOC_HOST) return;   // already back (or never left)
            enqueue(new_tr(t, A_PRE, loc[t], e.urgent != 0, false), now);
        }
    }

    // simulator.py:399-410
    void drain(int64_t upto, bool issues_at_upto) {
        while (!events.empty()) {
            const Ev ev = events.top();
            if (ev.time > upto) break;
            if (ev.time == upto && ev.prio != 0 && !issues_at_upto) break;
            events.pop();
            if (ev.kind == K_COMPLETE) complete((int)ev.payload, ev.time);
            else issue_entry(issues[ev.payload], ev.time);
        }
    }

    // simulator.py:417-428: farthest next use, ties to the smallest id
    int64_t pick_victim(int64_t k) {
        int64_t best = -1, best_use = 0;
        const int64_t a0 = act_ptr[k], a1 = act_ptr[k + 1];
        for (int64_t t = 0; t < T; ++t) {
            if (loc[t] != LOC_GPU || engaged[t] >= 0) continue;
            bool needed = false;
            for (int64_t j = a0; j < a1; ++j)
                if (act[j] == t) { needed = true; break; }
            if (needed) continue;
            int64_t use;
            if (!next_use(t, k, &use)) continue;
            if (best < 0 || use > best_use || (use == best_use && in.tid[t] < in.tid[best])) {
                best = t;
                best_use = use;
            }
        }
        return best;
    }

    // simulator.py:430-469
    bool try_launch(int64_t k, int64_t now) {
        bool waiting = false, mem_blocked = false;
        for (int64_t j = act_ptr[k]; j < act_ptr[k + 1]; ++j) {
            const int64_t t = act[j];
            const int x = engaged[t];
            if (x >= 0) {
                Tr &tr = trs[x];
                if (tr.action == A_OFF && !tr.started) { cancel(x); continue; }   // still on GPU; keep it
                if (tr.action == A_PRE) {
                    if (!tr.started) {
                        promote_front(x, now);
                        if (!trs[x].started && resident + trs[x].nbytes > cap) mem_blocked = true;
                    }
                    waiting = true;
                } else {
                    waiting = true;                          // a running offload cannot be aborted
                }
            } else if (loc[t] == LOC_SSD || loc[t] == LOC_HOST) {
                const int y = new_tr(t, A_PRE, loc[t], true, false);
                enqueue(y, now, true);
                if (!trs[engaged[t]].started && resident + in.size[t] > cap) mem_blocked = true;
                waiting = true;
            }
        }
        if (!waiting) {
            int64_t new_alloc = 0;
            for (int64_t j = act_ptr[k]; j < act_ptr[k + 1]; ++j)
                if (loc[act[j]] == LOC_NONE) new_alloc += in.size[act[j]];
            if (resident + new_alloc > cap) mem_blocked = true;
        }
        if (mem_blocked && n_emergency_engaged == 0) {
            const int64_t v = pick_victim(k);
            if (v >= 0) {
                const int y = new_tr(v, A_OFF, LOC_SSD, true, true);
                out.emergency += 1;
                enqueue(y, now);
            }
        }
        return !waiting && !mem_blocked;
    }

    // simulator.py:275-293
    int install_tail(const Issue &e, int source, int64_t end) {
        int device, action;
        if (e.action == A_OFF) { device = e.target == TIO_DEST_CPU ? LOC_HOST : LOC_SSD; action = A_OFF; }
        else { device = source; action = A_PRE; }
        if (device != LOC_SSD && device != LOC_HOST) {
            err = "plan prefetch crosses the iteration boundary from the GPU";
            return TIO_ERR_SIMULATION;
        }
        const int c = chan(device, action);
        if (!chan_exists[c]) { err = "plan targets the host tier but no host rates were given"; return TIO_ERR_INVALID; }
        if (running[c] >= 0) {
            err = "two boundary-straddling transfers on one channel";
            return TIO_ERR_SIMULATION;
        }
        const int x = new_tr(e.t, action, device, e.urgent != 0, false);
        trs[x].started = true;
        trs[x].end = end;
        running[c] = x;
        record_start(x, c, 0, true);
        engage(e.t, x);
        push(end, 0, e.t, K_COMPLETE, x);
        loc[e.t] = (int8_t)(action == A_OFF ? LOC_GPU : source);
        return TIO_OK;
    }

    // simulator.py:243-273: steady-state folding of the plan
    int install_plan() {
        // entries grouped by tensor id (ascending), each group by trigger (stable)
        std::vector<int64_t> order(in.num_entries);
        for (int64_t i = 0; i < in.num_entries; ++i) order[i] = i;
        std::unordered_map<int64_t, int64_t> pos_of;
        pos_of.reserve((size_t)T * 2 + 1);
        for (int64_t t = 0; t < T; ++t) pos_of[in.tid[t]] = t;
        for (int64_t i = 0; i < in.num_entries; ++i)
            if (!pos_of.count(in.e_tid[i])) {
                char b[128];
                snprintf(b, sizeof(b), "plan entry for unknown tensor %lld", (long long)in.e_tid[i]);
                err = b;
                return TIO_ERR_INVALID;
            }
        std::stable_sort(order.begin(), order.end(), [&](int64_t x, int64_t y) {
            if (in.e_tid[x] != in.e_tid[y]) return in.e_tid[x] < in.e_tid[y];
            return in.e_trigger[x] < in.e_trigger[y];
        });
        for (size_t g = 0; g < order.size();) {
            size_t h = g;
            while (h < order.size() && in.e_tid[order[h]] == in.e_tid[order[g]]) ++h;
            const int64_t t = pos_of[in.e_tid[order[g]]];
            int l = LOC_GPU;
            bool have_tail = false;
            Issue tail{};
            int tail_src = LOC_GPU;
            for (size_t j = g; j < h; ++j) {
                const int64_t i = order[j];
                Issue e{t, in.e_trigger[i], in.e_deadline[i], in.e_action[i], in.e_target[i], in.e_urgent[i]};
                if (iteration > 0 && e.trigger >= iteration) {
                    e.trigger -= iteration;
                    e.deadline -= iteration;
                    issues.push_back(e);
                    push(e.trigger, 2, t, K_ISSUE, (int64_t)issues.size() - 1);
                    continue;
                }
                issues.push_back(e);
                push(e.trigger, 2, t, K_ISSUE, (int64_t)issues.size() - 1);
                const int nl = e.action == A_PRE ? LOC_GPU : (e.target == TIO_DEST_CPU ? LOC_HOST : LOC_SSD);
                if (e.deadline > iteration) {
                    tail_src = l;
                    tail = e;
                    have_tail = true;
                }
                l = nl;
            }
            if (have_tail && tail.deadline > iteration) {
                const int rc = install_tail(tail, tail_src, tail.deadline - iteration);
                if (rc != TIO_OK) return rc;
            } else if (l != LOC_GPU) {
                loc[t] = (int8_t)l;
            }
            g = h;
        }
        return TIO_OK;
    }

    int run() {
        for (int64_t t = 0; t < T; ++t)
            for (int64_t j = in.ptr[t]; j < in.ptr[t + 1]; ++j)
                if (in.acc[j] < 0 || in.acc[j] >= N) {
                    err = "tensor " + std::to_string(in.tid[t]) + ": access " + std::to_string(in.acc[j]) +
                          " out of range";
                    return TIO_ERR_INVALID;
                }
        for (int64_t k = 0; k < N; ++k) iteration += in.dur[k];
        // active_at[k] sorted by tensor id (simulator.py:187-198)
        act_ptr.assign(N + 1, 0);
        for (int64_t t = 0; t < T; ++t)
            for (int64_t j = in.ptr[t]; j < in.ptr[t + 1]; ++j) act_ptr[in.acc[j] + 1]++;
        for (int64_t k = 0; k < N; ++k) act_ptr[k + 1] += act_ptr[k];
        act.assign(act_ptr[N], 0);
        {
            std::vector<int64_t> fill(act_ptr.begin(), act_ptr.end() - 1);
            for (int64_t t = 0; t < T; ++t)
                for (int64_t j = in.ptr[t]; j < in.ptr[t + 1]; ++j) act[fill[in.acc[j]]++] = t;
        }
        for (int64_t k = 0; k < N; ++k)
            std::sort(act.begin() + act_ptr[k], act.begin() + act_ptr[k + 1],
                      [&](int64_t x, int64_t y) { return in.tid[x] < in.tid[y]; });
        // simulator.py:200-204
        for (int64_t k = 0; k < N; ++k) {
            int64_t b = 0;
            for (int64_t j = act_ptr[k]; j < act_ptr[k + 1]; ++j) b += in.size[act[j]];
            if (b > cap) {
                char buf[160];
                snprintf(buf, sizeof(buf), "kernel %lld actively uses %lld bytes, above capacity %lld",
                         (long long)k, (long long)b, (long long)cap);
                err = buf;
                return TIO_ERR_SIMULATION;
            }
        }
        // simulator.py:206-216: the channels are built after the active-bytes
        // check, so a bad rate surfaces only on a satisfiable trace
        static const char *names[4] = {"ssd.offload", "ssd.prefetch", "host.offload", "host.prefetch"};
        for (int c = 0; c < 4; ++c) {
            if (c >= 2 && !in.has_host) { chan_exists[c] = false; continue; }
            chan_exists[c] = true;
            const int r = decode_rate(in.rate[c], &rc[c]);
            if (r != TIO_OK) { err = std::string("channel ") + names[c] + ": rate must be > 0"; return r; }
        }
        loc.assign(T, LOC_NONE);
        for (int64_t t = 0; t < T; ++t) loc[t] = is_global(t) ? LOC_GPU : LOC_NONE;
        engaged.assign(T, -1);
        int rc0 = install_plan();
        if (rc0 != TIO_OK) return rc0;
        if (in.layer_policy) {
            rc0 = setup_layer_policy();
            if (rc0 != TIO_OK) return rc0;
        }
        out.initial_loc = loc;
        // initial residency (simulator.py:234-239)
        for (int64_t t = 0; t < T; ++t)
            if (loc[t] == LOC_GPU) grow(in.size[t]);
        for (int c = 0; c < 4; ++c)
            if (running[c] >= 0 && trs[running[c]].action == A_PRE) grow(trs[running[c]].nbytes);

        out.start.assign(N, 0);
        out.stall.assign(N, 0);
        out.resident.assign(N, 0);
        out.kseq.assign(N, 0);
        int64_t now = 0;
        if (pol) maybe_issue(now);                  // on_start (simulator.py:477-478)
        for (int64_t k = 0; k < N; ++k) {
            const int64_t ready = now;
            while (true) {
                drain(now, false);
                if (try_launch(k, now)) break;
                drain(now, true);
                if (events.empty()) {
                    char buf[160];
                    snprintf(buf, sizeof(buf),
                             "simulation stuck before kernel %lld: no transfer can free enough memory", (long long)k);
                    err = buf;
                    return TIO_ERR_SIMULATION;
                }
                if (events.top().time > now) now = events.top().time;
            }
            out.stall[k] = now - ready;
            out.start[k] = now;
            out.kseq[k] = order++;
            for (int64_t j = act_ptr[k]; j < act_ptr[k + 1]; ++j) {
                const int64_t t = act[j];
                if (loc[t] == LOC_NONE) { loc[t] = LOC_GPU; grow(in.size[t]); }
            }
            out.resident[k] = resident;
            if (pol) on_kernel_launched(k, now);
            now += in.dur[k];
            for (int64_t j = act_ptr[k]; j < act_ptr[k + 1]; ++j) {
                const int64_t t = act[j];
                if (!is_global(t) && in.acc[in.ptr[t + 1] - 1] == k) {
                    loc[t] = LOC_NONE;
                    resident -= in.size[t];
                }
            }
            pump_all(now);
            if (pol) on_kernel_end(k, now);
        }
        out.total_time = now;
        out.ideal_time = iteration;
        for (int64_t k = 0; k < N; ++k) out.stall_total += out.stall[k];
        out.peak_resident = peak;
        for (int c = 0; c < 4; ++c) {
            int64_t busy = 0;
            for (auto &iv : booked[c]) {
                const int64_t lo = iv.first > 0 ? iv.first : 0, hi = iv.second < now ? iv.second : now;
                if (hi > lo) busy += hi - lo;
            }
            out.busy[c] = busy;
        }
        // issue_kernel: last kernel that has finished (model time) when the transfer starts
        for (auto &s : out.transfers) {
            int64_t lo = 0, hi = N;   // first k with start[k] + dur[k] > s.start
            while (lo < hi) {
                const int64_t m = (lo + hi) >> 1;
                if (out.start[m] + in.dur[m] > s.start) hi = m; else lo = m + 1;
            }
            s.issue_kernel = lo - 1;
        }
        return TIO_OK;
    }
};

}  // namespace

int engine_schedule(const SchedInput &in, SchedOutput *out, std::string *err) {
    Engine e(in, *out, *err);
    return e.run();
}

}  // namespace tio
