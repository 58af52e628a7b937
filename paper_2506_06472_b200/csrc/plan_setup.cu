// plan_setup.cu — planner prologue/epilogue kernels.
//
//   unsat check          planner.py:275-278 (first kernel with active > capacity)
//   candidate build      planner.py:283-284 periods sorted by (tensor_id, start_kernel),
//                        _period_times :130-144, transfer durations bandwidth.py:75-84,
//                        the duration > iteration rejection :161-164
//   over list / peak     planner.py:353, MemoryTimeline.peak
//   planned host bytes   planner.py:354-358
//   entries              planner.py:328-335 + sort :360-361 + mark_urgent :373-397
#include <climits>
#include "common.cuh"
#include "block_scan.cuh"
#include "planner.cuh"
#include "plan_setup.cuh"

namespace tio {

__global__ void k_fill_i64(int64_t *p, int64_t n, int64_t v) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = v;
}

// first kernel whose active bytes exceed capacity
__global__ void k_unsat(const int64_t *active, int64_t N, int64_t cap, unsigned long long *first) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < N; k += (int64_t)gridDim.x * blockDim.x)
        if (active[k] > cap) atomicMin(first, (unsigned long long)k);
}

__global__ void k_unsat_finish(const int64_t *active, const unsigned long long *first, int64_t N,
                               int64_t *ps, const int64_t *lifetime_flags) {
    if (*lifetime_flags != 0) { ps[PS_STATUS] = 2; return; }  // invalid trace
    unsigned long long k = *first;
    if (k < (unsigned long long)N) {
        ps[PS_STATUS] = 1;
        ps[PS_UNSAT_K] = (int64_t)k;
        ps[PS_UNSAT_B] = active[k];
    }
}

// id-order keys: signed id with the sign bit flipped sorts as unsigned
__global__ void k_id_keys(const int64_t *tid, int64_t T, uint64_t *keys, uint32_t *vals) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < T; i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = (uint64_t)tid[i] ^ (1ull << 63);
        vals[i] = (uint32_t)i;
    }
}

// rank[pos] = position in id order; per-rank period counts; duplicate-id flag
__global__ void k_rank(const uint64_t *skeys, const uint32_t *order, int64_t T, const int64_t *tpp,
                       int32_t *rank, int64_t *cnt_by_rank, int64_t *flags) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < T; j += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = order ? order[j] : j;
        rank[i] = (int32_t)j;
        cnt_by_rank[j] = tpp[i + 1] - tpp[i];
        if (order && j > 0 && skeys[j] == skeys[j - 1]) *flags = 1;  // duplicate tensor id
    }
}

__global__ void k_build_candidates(CandBuild a) {
    const int64_t P = *a.num_periods;
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < P; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = a.p_tensor[q];
        const int64_t p0 = a.tpp[i], p1 = a.tpp[i + 1];
        const int64_t l = q - p0, cnt = p1 - p0;
        // a wrap period starting at kernel 0 sorts first within its tensor
        const bool rot = a.p_wraps[p1 - 1] && a.p_start[p1 - 1] == 0;
        const int64_t l2 = rot ? (l == cnt - 1 ? 0 : l + 1) : l;
        const int64_t c = a.cand_ptr[a.rank[i]] + l2;
        const int64_t size = a.size[i];
        const int32_t first = a.acc[a.ptr[i]], last = a.acc[a.ptr[i + 1] - 1];
        const int8_t wraps = a.p_wraps[q];
        int64_t ready, deadline;
        if (!wraps) {
            ready = a.starts[a.p_start[q]];
            deadline = a.starts[a.p_end[q] + 1];
        } else {
            ready = a.starts[last] + a.dur[last];
            deadline = a.iteration + a.starts[first];
        }
        int64_t d[4];
        for (int ch = 0; ch < 4; ++ch) d[ch] = (ch < 2 || a.has_host) ? duration_of(a.rates[ch], size) : 0;
        a.c_size[c] = size;
        a.c_sk[c] = a.p_start[q];
        a.c_ek[c] = a.p_end[q];
        a.c_wraps[c] = wraps;
        a.c_first[c] = first;
        a.c_last[c] = last;
        a.c_ready[c] = ready;
        a.c_deadline[c] = deadline;
        for (int ch = 0; ch < 4; ++ch) a.c_d[4 * c + ch] = d[ch];
        a.c_tid[c] = a.tid[i];
        a.c_tpos[c] = (int32_t)i;
        int ssd = (d[0] > a.iteration || d[1] > a.iteration) ? S_DEAD : S_UNK;
        int host = (!a.has_host || d[2] > a.iteration || d[3] > a.iteration) ? H_DEAD : H_UNK;
        int8_t st = (int8_t)(ssd | (host << 2));
        if (ssd == S_DEAD && host == H_DEAD) st |= ST_GONE;
        a.st[c] = st;
    }
}

// ---- tiles (planner.cu): ready-time order keys, then per-tile spans/hulls ----
__global__ void k_ready_keys(const int64_t *ready, int64_t P, uint64_t *keys, uint32_t *vals) {
    for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < P; c += (int64_t)gridDim.x * blockDim.x) {
        keys[c] = (uint64_t)ready[c];
        vals[c] = (uint32_t)c;
    }
}

// one warp per tile
__global__ void k_tile_spans(const uint32_t *tcand, int64_t P, int64_t ntiles, int tile, int64_t N,
                             const int64_t *ready, const int64_t *deadline, const int8_t *wraps,
                             const int32_t *sk, const int32_t *ek, const int32_t *first, const int32_t *last,
                             int32_t *ctile, int64_t *t_lo, int64_t *t_hi, int32_t *ka_lo, int32_t *ka_hi,
                             int32_t *kb_lo, int32_t *kb_hi) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t t = warp; t < ntiles; t += nwarps) {
        long long lo = LLONG_MAX, hi = LLONG_MIN;
        int alo = INT_MAX, ahi = INT_MIN, blo = INT_MAX, bhi = INT_MIN;
        for (int64_t p = t * tile + lane; p < (t + 1) * tile && p < P; p += 32) {
            const int64_t c = tcand ? (int64_t)tcand[p] : p;      // arrays in tile order: identity
            if (ctile) ctile[c] = (int32_t)t;
            lo = min(lo, (long long)ready[c]);
            hi = max(hi, (long long)deadline[c]);
            int a0, a1, b0 = 1, b1 = 0;
            if (!wraps[c]) { a0 = sk[c]; a1 = ek[c]; }
            else { a0 = last[c] + 1; a1 = (int)N - 1; b0 = 0; b1 = first[c] - 1; }
            if (a0 <= a1) { alo = min(alo, a0); ahi = max(ahi, a1); }
            if (b0 <= b1) { blo = min(blo, b0); bhi = max(bhi, b1); }
        }
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
            alo = min(alo, __shfl_xor_sync(0xffffffffu, alo, o));
            ahi = max(ahi, __shfl_xor_sync(0xffffffffu, ahi, o));
            blo = min(blo, __shfl_xor_sync(0xffffffffu, blo, o));
            bhi = max(bhi, __shfl_xor_sync(0xffffffffu, bhi, o));
        }
        if (lane == 0) {
            t_lo[t] = lo; t_hi[t] = hi;
            ka_lo[t] = alo <= ahi ? alo : 1; ka_hi[t] = alo <= ahi ? ahi : 0;
            kb_lo[t] = blo <= bhi ? blo : 1; kb_hi[t] = blo <= bhi ? bhi : 0;
        }
    }
}

// candidate columns from planner order (index c) into tile order (position p)
__global__ void k_permute_candidates(const uint32_t *tcand, int64_t P, CandCols src, CandCols dst) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = tcand[p];
        dst.size[p] = src.size[c]; dst.ready[p] = src.ready[c]; dst.deadline[p] = src.deadline[c];
        for (int q = 0; q < 4; ++q) dst.d[4 * p + q] = src.d[4 * c + q];
        dst.tid[p] = src.tid[c];
        dst.sk[p] = src.sk[c]; dst.ek[p] = src.ek[c]; dst.first[p] = src.first[c]; dst.last[p] = src.last[c];
        dst.tpos[p] = src.tpos[c];
        dst.wraps[p] = src.wraps[c]; dst.st[p] = src.st[c];
    }
}

// ---- epilogue ------------------------------------------------------------------
__global__ void k_over_flags(const int64_t *resid, int64_t N, int64_t cap, int64_t *flag, long long *peak) {
    long long m = LLONG_MIN;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < N; k += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = resid[k];
        flag[k] = r > cap;
        if (r > m) m = r;
    }
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0 && m != LLONG_MIN) atomicMax(peak, m);   // one atomic per warp
}

__global__ void k_over_write(const int64_t *flag, const int64_t *pos, int64_t N, int64_t *over) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < N; k += (int64_t)gridDim.x * blockDim.x)
        if (flag[k]) over[pos[k]] = k;
}

__global__ void k_planned_host(const int64_t *os, const int64_t *oe, const int64_t *oz, int64_t h, int64_t *out) {
    // _host_peak_occupancy over [min start, max end] (planner.py:354-358); all
    // starts qualify, so it is the largest occupancy at any start: one start
    // per thread over the grid, block maxima, atomicMax into *out (zeroed)
    __shared__ int64_t sm[40];
    int64_t best = 0;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < h; p += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = os[p];
        int64_t sum = 0;
        for (int64_t j = 0; j < h; ++j)
            if (os[j] <= t && t < oe[j]) sum += oz[j];
        if (sum > best) best = sum;
    }
    for (int o = 16; o > 0; o >>= 1) {
        const int64_t x = __shfl_xor_sync(0xffffffffu, best, o);
        if (x > best) best = x;
    }
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        int64_t m = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) if (sm[w] > m) m = sm[w];
        if (m > 0) atomicMax(reinterpret_cast<long long *>(out), (long long)m);
    }
}

// sort key: (trigger, tensor rank, action) packed; value = entry index (commit order)
__global__ void k_entry_keys(const tio_commit *cm, int64_t nc, const int32_t *rank, int rbits,
                             int part, uint64_t *keys, uint32_t *vals) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < 2 * nc; j += (int64_t)gridDim.x * blockDim.x) {
        const tio_commit &c = cm[j >> 1];
        const int action = (int)(j & 1);
        const uint64_t trig = (uint64_t)(action ? c.pre_start : c.off_start);
        const uint64_t r = (uint64_t)rank[c.tensor_pos];
        uint64_t key;
        if (part == 0) key = (trig << (rbits + 1)) | (r << 1) | (uint64_t)action;  // single pass
        else if (part == 1) key = (r << 1) | (uint64_t)action;                       // two-stage: low
        else key = trig;                                                           // two-stage: high
        keys[j] = key;
        vals[j] = (uint32_t)j;
    }
}

__global__ void k_regather_keys(const tio_commit *cm, const uint32_t *vals, int64_t n, uint64_t *keys) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        uint32_t v = vals[j];
        const tio_commit &c = cm[v >> 1];
        keys[j] = (uint64_t)((v & 1) ? c.pre_start : c.off_start);
    }
}

__global__ void k_emit_entries(const tio_commit *cm, const uint32_t *order, int64_t n, const int64_t *starts,
                               const int64_t *ptr, const int32_t *acc, const int8_t *kind, int64_t iteration,
                               tio_entry *out) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t v = order[j];
        const tio_commit &c = cm[v >> 1];
        tio_entry e;
        e.tensor_id = c.tensor_id;
        e.tensor_pos = c.tensor_pos;
        e.pad = 0;
        if ((v & 1) == 0) {
            e.action = 0;
            e.trigger_us = c.off_start;
            e.deadline_us = c.off_end;
            e.target = (int32_t)c.destination;
            e.urgent = 0;
        } else {
            e.action = 1;
            e.trigger_us = c.pre_start;
            e.deadline_us = c.pre_end;
            e.target = 0;
            // mark_urgent: deadline == earliest need time at or after it
            const int64_t D = c.pre_end;
            const int64_t t = c.tensor_pos;
            int64_t lo = ptr[t], hi = ptr[t + 1];
            const int64_t first_start = starts[acc[lo]];
            while (lo < hi) {
                int64_t mid = (lo + hi) >> 1;
                if (starts[acc[mid]] >= D) hi = mid; else lo = mid + 1;
            }
            bool have = lo < ptr[t + 1];
            int64_t need = have ? starts[acc[lo]] : 0;
            if (kind[t] == 1) {
                int64_t wrap = iteration + first_start;
                if (wrap >= D && (!have || wrap < need)) { need = wrap; have = true; }
            }
            e.urgent = have && need == D;
        }
        out[j] = e;
    }
}

}  // namespace tio
