/*
 * lazy_probe.c — experiment: the reference greedy (planner.py:267-370) run as
 * a lazy greedy (stale upper bounds in a max-heap, re-evaluated on pop).
 * Exact when every candidate's value is non-increasing over rounds, which
 * holds on the SSD path (bookings only added, residual only decreases);
 * with a host path the bound is max(ssd value, host value).
 * Counts pops / re-evaluations per commit; the result is compared with the
 * oracle's commit list by tools/lazy_probe.py.  Not product code.
 */
#include "../oracle/tio_oracle.c"

typedef struct { u128 b; int64_t c; int64_t idx; } hkey_t;

static int hk_gt(const hkey_t *x, const hkey_t *y) {   /* x ranks before y */
    if (ratio_gt(x->b, x->c, y->b, y->c)) return 1;
    if (ratio_gt(y->b, y->c, x->b, x->c)) return 0;
    return x->idx < y->idx;
}

typedef struct { hkey_t *v; int64_t n; } heap_t;
static void h_push(heap_t *h, hkey_t k) {
    int64_t i = h->n++;
    while (i > 0) { int64_t p = (i - 1) / 2; if (!hk_gt(&k, &h->v[p])) break; h->v[i] = h->v[p]; i = p; }
    h->v[i] = k;
}
static hkey_t h_pop(heap_t *h) {
    hkey_t top = h->v[0], last = h->v[--h->n];
    int64_t i = 0;
    for (;;) {
        int64_t l = 2 * i + 1, r = l + 1, m = i;
        const hkey_t *mk = &last;
        if (l < h->n && hk_gt(&h->v[l], mk)) { m = l; mk = &h->v[l]; }
        if (r < h->n && hk_gt(&h->v[r], mk)) { m = r; mk = &h->v[r]; }
        if (m == i) break;
        h->v[i] = h->v[m]; i = m;
    }
    if (h->n) h->v[i] = last;
    return top;
}

/* Fenwick tree over dur*[resid > cap] */
static void bit_add(int64_t *t, int64_t n, int64_t i, int64_t v) { for (++i; i <= n; i += i & -i) t[i] += v; }
static int64_t bit_pre(const int64_t *t, int64_t i) { int64_t s = 0; for (; i > 0; i -= i & -i) s += t[i]; return s; }

int64_t g_pops, g_evals, g_host_evals;

int64_t g_stats[3];
int64_t *tio_lazy_stats(void) { return g_stats; }
/* same signature as tio_oracle_plan (the unsat check is left to the oracle) */
int tio_lazy_plan(int64_t n, const int64_t *dur, const int64_t *active, const int64_t *timeline_in,
                  int64_t capacity, double ssd_off, double ssd_pre, int has_host, double host_off,
                  double host_pre, int64_t host_cap, int64_t P, const int64_t *p_size, const int64_t *p_start,
                  const int64_t *p_end, const int8_t *p_wraps, const int64_t *p_first, const int64_t *p_last,
                  int64_t *resid, plan_result_t *res, int verbose, int64_t max_rounds) {
    int64_t *stats = g_stats;
    (void)active; (void)verbose; (void)max_rounds;
    memset(res, 0, sizeof(*res));
    int64_t *starts = malloc(sizeof(int64_t) * (size_t)(n + 1));
    tio_oracle_starts(n, dur, starts);
    int64_t iteration = starts[n], period = iteration > 0 ? iteration : 0;
    memcpy(resid, timeline_in, sizeof(int64_t) * (size_t)n);
    int64_t *bit = calloc((size_t)n + 1, sizeof(int64_t));
    int64_t crit = 0;
    for (int64_t k = 0; k < n; ++k) if (resid[k] > capacity) { bit_add(bit, n, k, dur[k]); ++crit; }
    int64_t (*dd)[4] = malloc(sizeof(int64_t[4]) * (size_t)(P > 0 ? P : 1));
    int64_t *ready = malloc(sizeof(int64_t) * (size_t)(P > 0 ? P : 1));
    int64_t *deadl = malloc(sizeof(int64_t) * (size_t)(P > 0 ? P : 1));
    int64_t *stamp = malloc(sizeof(int64_t) * (size_t)(P > 0 ? P : 1));
    for (int64_t i = 0; i < P; ++i) {
        dur_of(ssd_off, p_size[i], &dd[i][0]); dur_of(ssd_pre, p_size[i], &dd[i][1]);
        if (has_host) { dur_of(host_off, p_size[i], &dd[i][2]); dur_of(host_pre, p_size[i], &dd[i][3]); }
        if (!p_wraps[i]) { ready[i] = starts[p_start[i]]; deadl[i] = starts[p_end[i] + 1]; }
        else { ready[i] = starts[p_last[i]] + dur[p_last[i]]; deadl[i] = iteration + starts[p_first[i]]; }
    }
    chan_t ch[4]; memset(ch, 0, sizeof(ch));
    occ_t *occ = NULL; int64_t n_occ = 0, cap_occ = 0, cap_commits = 0;
    heap_t h = {malloc(sizeof(hkey_t) * (size_t)(P > 0 ? P : 1)), 0};
    hkey_t *park = malloc(sizeof(hkey_t) * (size_t)(P > 0 ? P : 1));
    int64_t npark = 0;
    window_t *wv = malloc(sizeof(window_t) * (size_t)(P > 0 ? P : 1));
    int *wdest = malloc(sizeof(int) * (size_t)(P > 0 ? P : 1));

    /* exact value now (reference rule) + upper bound valid until the next re-evaluation */
    #define EVAL(i, V, U) do {                                                                   \
        window_t w; int dest = 0; u128 vb = 0, ub = 0; int64_t vc = 1, uc = 1;                  \
        int64_t r[4], ct;                                                                        \
        ++g_evals;                                                                               \
        if (try_pair(&ch[0], &ch[1], dd[i][0], dd[i][1], iteration, ready[i], deadl[i], &w)) {  \
            dest = 1;                                                                            \
            covered(n, starts, iteration, p_wraps[i], p_start[i], p_end[i], p_first[i], p_last[i], w.off_e, w.pre_s, r); \
            ct = 0;                                                                              \
            if (r[0] <= r[1]) ct += bit_pre(bit, r[1] + 1) - bit_pre(bit, r[0]);                 \
            if (r[2] <= r[3]) ct += bit_pre(bit, r[3] + 1) - bit_pre(bit, r[2]);                 \
            vb = (u128)(uint64_t)p_size[i] * (uint64_t)ct; vc = w.cost; ub = vb; uc = vc;        \
            wv[i] = w;                                                                           \
        }                                                                                        \
        if (has_host) {                                                                          \
            window_t w2;                                                                         \
            ++g_host_evals;                                                                      \
            if (try_pair(&ch[2], &ch[3], dd[i][2], dd[i][3], iteration, ready[i], deadl[i], &w2) && \
                host_peak(occ, n_occ, w2.off_e, w2.pre_s) + p_size[i] <= host_cap) {             \
                covered(n, starts, iteration, p_wraps[i], p_start[i], p_end[i], p_first[i], p_last[i], w2.off_e, w2.pre_s, r); \
                ct = 0;                                                                          \
                if (r[0] <= r[1]) ct += bit_pre(bit, r[1] + 1) - bit_pre(bit, r[0]);             \
                if (r[2] <= r[3]) ct += bit_pre(bit, r[3] + 1) - bit_pre(bit, r[2]);             \
                u128 hb = (u128)(uint64_t)p_size[i] * (uint64_t)ct;                              \
                if (!dest) { dest = 2; vb = hb; vc = w2.cost; wv[i] = w2; ub = hb; uc = vc; }    \
                else if (hb && (ub == 0 || ratio_gt(hb, w2.cost, ub, uc))) { ub = hb; uc = w2.cost; } \
            }                                                                                    \
        }                                                                                        \
        wdest[i] = dest;                                                                         \
        V.b = vb; V.c = vc; V.idx = i; U.b = ub; U.c = uc; U.idx = i;                            \
    } while (0)

    for (int64_t i = 0; i < P; ++i) {
        hkey_t V, U;
        EVAL(i, V, U);
        stamp[i] = 0;
        if (U.b) h_push(&h, U);
    }
    int64_t commits = 0;
    int rc = 0;
    while (crit > 0) {
        /* best exact value among candidates resolved this round */
        hkey_t best = {0, 1, -1};
        npark = 0;
        for (;;) {
            if (best.idx >= 0 && (h.n == 0 || hk_gt(&best, &h.v[0]))) break;
            if (h.n == 0) break;
            hkey_t k = h_pop(&h);
            ++g_pops;
            int64_t i = k.idx;
            hkey_t V = {0, 1, i}, U = {0, 1, i};
            if (stamp[i] == commits) {
                /* fresh: the cached bound is exact only if it equals the value */
                EVAL(i, V, U);   /* cheap enough for a probe; keeps the code simple */
                --g_evals;
            } else {
                EVAL(i, V, U);
                stamp[i] = commits;
            }
            if (U.b == 0) continue;                   /* dead for good */
            if (V.b && (best.idx < 0 || hk_gt(&V, &best))) best = V;
            park[npark++] = U;                        /* back into the heap after the commit */
        }
        if (best.idx < 0) break;
        int64_t i = best.idx;
        for (int64_t q = 0; q < npark; ++q) if (park[q].idx != i) h_push(&h, park[q]);
        window_t w = wv[i];
        int dest = wdest[i];
        int c0 = dest == 1 ? 0 : 2;
        if ((rc = chan_book(&ch[c0], w.off_s, w.off_e, period))) break;
        if ((rc = chan_book(&ch[c0 + 1], w.pre_s, w.pre_e, period))) break;
        int64_t r[4];
        covered(n, starts, iteration, p_wraps[i], p_start[i], p_end[i], p_first[i], p_last[i], w.off_e, w.pre_s, r);
        for (int q = 0; q < 4; q += 2)
            for (int64_t k = r[q]; k <= r[q + 1]; ++k) {
                int64_t old = resid[k];
                resid[k] -= p_size[i];
                if (old > capacity && resid[k] <= capacity) { bit_add(bit, n, k, -dur[k]); --crit; }
            }
        if (dest == 2) {
            if (n_occ == cap_occ) { cap_occ = cap_occ ? 2 * cap_occ : 64; occ = realloc(occ, sizeof(occ_t) * (size_t)cap_occ); }
            occ[n_occ].s = w.off_e; occ[n_occ].e = w.pre_s; occ[n_occ].size = p_size[i]; ++n_occ;
        }
        if (res->n_commits == cap_commits) {
            cap_commits = cap_commits ? 2 * cap_commits : 256;
            res->commits = realloc(res->commits, sizeof(commit_t) * (size_t)cap_commits);
        }
        commit_t *cm = &res->commits[res->n_commits++];
        cm->cand = i; cm->dest = dest;
        cm->off_s = w.off_s; cm->off_e = w.off_e; cm->pre_s = w.pre_s; cm->pre_e = w.pre_e;
        cm->benefit = best.b; cm->cost = best.c;
        cm->r0_lo = r[0]; cm->r0_hi = r[1]; cm->r1_lo = r[2]; cm->r1_hi = r[3];
        ++commits;
        res->rounds++;
    }
    if (n_occ > 0) {
        int64_t lo = INT64_MAX, hi = INT64_MIN;
        for (int64_t j = 0; j < n_occ; ++j) { if (occ[j].s < lo) lo = occ[j].s; if (occ[j].e > hi) hi = occ[j].e; }
        res->planned_host = host_peak(occ, n_occ, lo, hi);
    }
    stats[0] = g_pops; stats[1] = g_evals; stats[2] = g_host_evals;
    return rc;
}
