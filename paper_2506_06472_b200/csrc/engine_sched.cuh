// engine_sched.cuh — the migration engine's scheduler (host C++).
//
// A discrete-event model of the runtime engine with the reference engine's
// exact semantics (simulator.py:178-528 `_Engine`): location table, four
// serial channels with urgent / front queueing, capacity-gated prefetch
// admission, memory released at offload completion and reserved at prefetch
// start, kernel gating with cancel / promote / fetch-on-demand, Belady
// emergency eviction to the SSD channel (one in flight), steady-state plan
// folding.  Its output is (a) the SimReport of the reference (parity-tested
// against simulate()) and (b) the transfer schedule that the GPU executor
// (engine.cu) turns into stream operations.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace tio {

enum Loc : int8_t { LOC_NONE = 0, LOC_GPU = 1, LOC_SSD = 2, LOC_HOST = 3 };

struct SchedTransfer {
    int64_t tensor;        // tensor position in the trace
    int32_t action;        // 0 offload, 1 prefetch
    int32_t device;        // LOC_SSD / LOC_HOST
    int32_t urgent, emergency;
    int64_t start, end;    // model time (us)
    int64_t issue_kernel;  // kernel index whose start the transfer may not precede (-1: before kernel 0)
    int32_t tail;          // 1 = installed running at t=0 (boundary-straddling, plan folding)
    int32_t pad;
    int64_t seq;           // position in the model's processing order (shared with kernel launches)
};

struct SchedInput {
    int64_t N, T;
    const int64_t *dur;
    const int64_t *tid, *size;
    const int8_t *kind;
    const int64_t *ptr;
    const int32_t *acc;
    int64_t num_entries;
    const int64_t *e_tid;       // per entry: tensor id
    const int64_t *e_trigger, *e_deadline;
    const int32_t *e_action;    // 0 offload, 1 prefetch
    const int32_t *e_target;    // 1 SSD, 2 CPU (offloads)
    const int32_t *e_urgent;
    int64_t capacity;
    double rate[4];             // ssd.off, ssd.pre, host.off, host.pre
    int has_host;
    // layer-granularity baseline policy (simulator.py:95-177, :549-560):
    // engaged when the memory-timeline peak exceeds capacity; layers per
    // kernel and per tensor, INT64_MIN = none
    int layer_policy = 0;
    const int64_t *k_layer = nullptr, *t_layer = nullptr;
};

struct SchedOutput {
    int64_t total_time = 0, ideal_time = 0, stall_total = 0, peak_resident = 0, emergency = 0;
    int64_t busy[4] = {0, 0, 0, 0};   // per channel: booked time inside [0, total]
    std::vector<int64_t> start, stall, resident;     // per kernel
    std::vector<int64_t> kseq;                      // per kernel: launch position in the processing order
    std::vector<SchedTransfer> transfers;           // in start order per channel
    std::vector<int8_t> initial_loc;                // location at t = 0 (after plan folding)
};

// Returns 0, or TIO_ERR_SIMULATION / TIO_ERR_INVALID / TIO_ERR_CONFIG with *err set.
int engine_schedule(const SchedInput &in, SchedOutput *out, std::string *err);

}  // namespace tio
