// planner.cuh — on-device Algorithm 1 (reference planner.py:267-370).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "common.cuh"

namespace tio {

#ifndef TIO_PLAN_THREADS
#define TIO_PLAN_THREADS 256
#endif
constexpr int PLAN_THREADS = TIO_PLAN_THREADS;   // per block; 2 blocks per SM at 256
constexpr int TILE = 32;             // candidates per tile (one warp)

// candidate SSD/host evaluation state (2 bits each in st[c])
enum : int { S_UNK = 0, S_OK = 1, S_DEAD = 2 };                   // SSD path
enum : int { H_UNK = 0, H_OK = 1, H_CAPFAIL = 2, H_DEAD = 3 };    // host path
constexpr int8_t ST_GONE = (int8_t)0x40;  // committed or permanently useless
constexpr int8_t ST_REFIT = (int8_t)0x20; // placement refitted by phase R this round

// planner scalars[] slots
enum {
    PS_COMMITS = 0, PS_ROUNDS = 1, PS_CRIT = 2, PS_STATUS = 3, PS_OCC = 4,
    PS_UNSAT_K = 5, PS_UNSAT_B = 6, PS_INVARIANT = 7, PS_FLIP = 8 /* 3 slots x (cnt, lo, hi) */,
    PS_DBG = 17 /* 16 debug counters */, PS_RQ = 33 /* 2 refit-queue counts */, PS_COUNT = 35
};

// argmax key of a candidate (benefit 0 = none); meta = index << 33 | column << 2 | destination
struct Key {
    uint64_t blo, bhi;     // benefit = size x critical duration (u128)
    int64_t cost;          // offload + prefetch duration
    int64_t meta;
};

// A round's winner as one rank publishes it: the key plus everything the
// commit needs from the winner's column (a rank only evaluates the
// candidates of its own tiles, so the others do not have it).
struct WinMsg {
    Key k;
    int64_t size, off_s, off_e, pre_s, pre_e;
    int32_t r[4];
    int64_t pad[3];
};
static_assert(sizeof(WinMsg) == 112, "WinMsg layout");

// Sharded planner (candidate tiles split over ranks, state replicated):
// every rank's mailbox in device memory (its own; peers reach it through
// P2P / IPC mappings, or it is another instance's on the same GPU):
//   flag[r]          = epoch + round + 1 once rank r's round-`round` message is in
//   msg[round & 1][r] the message
constexpr int MAX_RANKS = 8;
struct Mailbox {
    unsigned long long flag[MAX_RANKS];
    WinMsg msg[2][MAX_RANKS];
};

constexpr int HX_LEVELS = 26;      // range-max table levels (2^26 blocks of 32 starts)

struct PlanArgs {
    int64_t N, P, iteration, capacity, host_cap;
    int32_t has_host;
    int32_t chunk;                 // kernels per chunk (crit prefix / residual ownership)
    int32_t pad0;
    int64_t max_rounds;            // > 0: stop after that many commits
    // immutable per-kernel data
    const int64_t *starts;         // [N+1]
    const int64_t *dur;            // [N]
    // residual pressure
    int64_t *resid;                // [N]
    int64_t *local_cp;             // [N+1] prefix of dur*[resid>cap] within each chunk
    int64_t *chunk_sum;            // [grid]
    // candidates (immutable), all per-candidate columns in tile order (position)
    const int64_t *c_size;
    const int32_t *c_sk, *c_ek, *c_first, *c_last;
    const int8_t *c_wraps;
    const int64_t *c_ready, *c_deadline;
    const int64_t *c_d;            // [4P] ssd_off, ssd_pre, host_off, host_pre
    // candidate state
    int8_t *st;                    // [P]
    int64_t *place;                // [4P] ssd_off_s, ssd_pre_s, host_off_s, host_pre_s
    int32_t *rng;                  // [4P]
    int32_t *hidx;                 // [2P] SSD channel index hints of the last fit (p, q)
    int32_t *hver;                 // [P]  SSD channel size at the last fit
    // tiles: candidates in ready-time order, TILE per tile
    int64_t ntiles;
    const uint32_t *tcand;         // [P] candidate index (planner order) at tile position
    const int64_t *t_lo, *t_hi;    // [ntiles] span [min ready, max deadline)
    const int32_t *t_ka_lo, *t_ka_hi, *t_kb_lo, *t_kb_hi;  // [ntiles] kernel hulls (lo > hi: empty)
    Key *tile_best;                // [ntiles]
    int64_t *rq[2];                // [P] each: queued SSD refits (positions), alternating by round
    int32_t *t_refit;              // [ntiles] last round whose commit queued a refit in the tile
    int64_t *t_hull;               // [4 ntiles] supersets of the SSD placements: off lo/hi, pre lo/hi
    int32_t *qround;               // [P] round whose commit queued the candidate's refit (-1 none)
    Key *vkey;                     // [P] key at the last evaluation (reused while unchanged)
    // channels: 4 channels (ssd.off, ssd.pre, host.off, host.pre) x 2 buffers
    int64_t *ch_s[4][2];
    int64_t *ch_e[4][2];
    int64_t ch_cap;
    // host occupancy intervals (CPU commits)
    int64_t *occ_s, *occ_e, *occ_size;
    // host-occupancy index (planner.py:179-186 as O(log h) queries), rebuilt
    // by block 0 after every CPU commit; buffer (h & 1) holds the index of h
    // intervals: starts / ends sorted with their sizes, prefix sums of the
    // sizes (h + 1), occupancy at every sorted start, and a range-max table
    // over 32-start blocks (single buffer: read only in phase E)
    int64_t *hx_s[2], *hx_sz[2], *hx_e[2], *hx_ez[2], *hx_ps[2], *hx_pe[2], *hx_a[2];
    int64_t *hx_tab;               // [HX_LEVELS x hx_nbmax]
    int64_t hx_nbmax;
    // reduction + outputs
    Key *blk_best;                 // [grid]
    int64_t *prof;                 // [grid * 8] phase-E split per block (debug build)
    unsigned *bar;                 // [2] grid barrier (count, generation), zeroed
    tio_commit *commits;           // [P]
    int64_t *scalars;              // [PS_COUNT]
    const int64_t *c_tid;          // [P] tensor id per candidate (for commit records)
    const int32_t *c_tpos;         // [P]
    // the round's winner (the last block to arrive reduces the block bests,
    // exchanges with the other ranks, publishes it here and bumps win_gen)
    WinMsg *win;                   // [1]
    unsigned long long *win_gen;   // [1] zeroed
    // sharding: rank `rank` of `nranks` owns tiles t with t % nranks == rank
    int32_t nranks, rank;
    unsigned long long epoch;      // added to every mailbox flag (one per planning call)
    Mailbox *mb_self;              // this rank's mailbox
    Mailbox *mb_peer[MAX_RANKS];   // every rank's mailbox as mapped here (mb_peer[rank] == mb_self)
};

// the wide form (3 blocks per SM) for large candidate sets (env
// TIO_PLAN_WIDE_TILES: tile threshold, default 60000; 0 = never)
bool plan_loop_wide(int64_t ntiles);
int plan_loop_grid(int *blocks, bool wide = false);
int launch_plan_loop(const PlanArgs &args, int blocks, cudaStream_t stream, bool wide = false);
// one cooperative grid of nranks x blocks_per_rank blocks, rank r running the
// planner on dev_args[r] (device memory)
int plan_loop_multi_grid(int *blocks);
int launch_plan_loop_multi(const PlanArgs *dev_args, int nranks, int blocks_per_rank, cudaStream_t stream);

}  // namespace tio
