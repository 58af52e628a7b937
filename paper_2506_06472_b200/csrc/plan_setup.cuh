// plan_setup.cuh — planner prologue/epilogue kernels.
#pragma once
#include <cstdint>
#include <climits>
#include <cuda_runtime.h>
#include "common.cuh"

namespace tio {

struct CandBuild {
    const int64_t *num_periods;    // device scalar
    const int64_t *p_tensor;
    const int32_t *p_start, *p_end;
    const int8_t *p_wraps;
    const int64_t *tpp;
    const int32_t *rank;
    const int64_t *cand_ptr;       // [T+1] by rank
    const int64_t *size, *tid, *ptr, *starts, *dur;
    const int32_t *acc;
    int64_t iteration;
    int32_t has_host;
    RateCode rates[4];
    // outputs
    int64_t *c_size;
    int32_t *c_sk, *c_ek, *c_first, *c_last;
    int8_t *c_wraps;
    int64_t *c_ready, *c_deadline, *c_d, *c_tid;
    int32_t *c_tpos;
    int8_t *st;
};

__global__ void k_fill_i64(int64_t *p, int64_t n, int64_t v);
__global__ void k_unsat(const int64_t *active, int64_t N, int64_t cap, unsigned long long *first);
__global__ void k_unsat_finish(const int64_t *active, const unsigned long long *first, int64_t N,
                               int64_t *ps, const int64_t *lifetime_flags);
__global__ void k_id_keys(const int64_t *tid, int64_t T, uint64_t *keys, uint32_t *vals);
__global__ void k_rank(const uint64_t *skeys, const uint32_t *order, int64_t T, const int64_t *tpp,
                       int32_t *rank, int64_t *cnt_by_rank, int64_t *flags);
__global__ void k_build_candidates(CandBuild a);
struct CandCols {
    int64_t *size, *ready, *deadline, *d, *tid;
    int32_t *sk, *ek, *first, *last, *tpos;
    int8_t *wraps, *st;
};
__global__ void k_permute_candidates(const uint32_t *tcand, int64_t P, CandCols src, CandCols dst);
__global__ void k_ready_keys(const int64_t *ready, int64_t P, uint64_t *keys, uint32_t *vals);
__global__ void k_tile_spans(const uint32_t *tcand, int64_t P, int64_t ntiles, int tile, int64_t N,
                             const int64_t *ready, const int64_t *deadline, const int8_t *wraps,
                             const int32_t *sk, const int32_t *ek, const int32_t *first, const int32_t *last,
                             int32_t *ctile, int64_t *t_lo, int64_t *t_hi, int32_t *ka_lo, int32_t *ka_hi,
                             int32_t *kb_lo, int32_t *kb_hi);
__global__ void k_over_flags(const int64_t *resid, int64_t N, int64_t cap, int64_t *flag, long long *peak);
__global__ void k_over_write(const int64_t *flag, const int64_t *pos, int64_t N, int64_t *over);
__global__ void k_planned_host(const int64_t *os, const int64_t *oe, const int64_t *oz, int64_t h, int64_t *out);
__global__ void k_entry_keys(const tio_commit *cm, int64_t nc, const int32_t *rank, int rbits, int part,
                             uint64_t *keys, uint32_t *vals);
__global__ void k_regather_keys(const tio_commit *cm, const uint32_t *vals, int64_t n, uint64_t *keys);
__global__ void k_emit_entries(const tio_commit *cm, const uint32_t *order, int64_t n, const int64_t *starts,
                               const int64_t *ptr, const int32_t *acc, const int8_t *kind, int64_t iteration,
                               tio_entry *out);

}  // namespace tio
