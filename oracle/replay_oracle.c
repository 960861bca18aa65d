/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference CPU algorithms on the RecMG hot path.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library, and only as the checker or as the
 * timed CPU baseline.  The product path (paper_2511_08568_b200) never calls it.
 *
 * Pinned against the reference: tests/golden/ fixtures were produced by running
 * the reference package (/root/reference/pkg/src/embcache) in the build
 * container (tests/golden/make_golden.py); tests/test_oracle.py checks this
 * file against every one of them.
 *
 * Reference citations are relative to /root/reference/pkg/src/embcache/.
 *
 *   oracle_replay       runtime.py:220-283  (replay) with
 *                       runtime.py:41-112   (PriorityBuffer),
 *                       runtime.py:115-137  (load_embeddings, Alg. 1),
 *                       runtime.py:100-112  (populate / gpu_buffer_populate, Alg. 2)
 *                       and trace.py:226-250 (chunk).  ways > 0 composes one
 *                       reference PriorityBuffer per set (set = gid % S, the
 *                       cache_sim.py:33-35 convention).
 *   oracle_lru          cache_sim.py:92-106 (_simulate_lru) via simulate(),
 *                       cache_sim.py:223-260.
 *   oracle_lru_prefetch runtime.py:304-349 (replay_policy_only with a
 *                       prefetcher: fully associative LRU + prefetch tags).
 *   oracle_coverage_sum runtime.py:276,282 (sequential float64 coverage sum).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum {
    C_CACHE_HITS = 0, C_PREFETCH_HITS, C_ON_DEMAND, C_PREFETCH_ISSUED,
    C_PREFETCH_USEFUL, C_EVICTIONS, C_PREFETCH_INSERTS, C_MAX_OCCUPANCY,
    C_NUM
};

/* ------------------------------------------------------------------------ */
/* Buffer: either "dense" (the reference's layout: flat arrays over every id,
 * argmin by ascending gid scan, runtime.py:53-55,105-108) or "compact"
 * (per-set slot arrays; victim = min (priority, gid), which is the same
 * element np.argmin picks because ties resolve to the lowest index = gid).  */
typedef struct {
    int dense;
    int64_t V, S, W;            /* ids, sets, ways per set                     */
    int64_t es;                 /* eviction_speed                              */
    /* dense layout */
    int64_t *prio;              /* [V]                                         */
    uint8_t *resident, *tag;    /* [V]                                         */
    /* compact layout */
    int64_t *slot_gid, *slot_prio;  /* [S*W]                                   */
    uint8_t *slot_tag;
    int32_t *slot_of;           /* [V] -> slot index or -1                     */
    int64_t *count;             /* [S]                                         */
    int64_t evictions, inserts_pf, occupancy, max_occupancy;
} buf_t;

static int buf_init(buf_t *b, int dense, int64_t V, int64_t S, int64_t W, int64_t es)
{
    memset(b, 0, sizeof(*b));
    b->dense = dense; b->V = V; b->S = S; b->W = W; b->es = es;
    b->count = (int64_t *)calloc((size_t)S, sizeof(int64_t));
    if (!b->count) return -1;
    if (dense) {
        b->prio = (int64_t *)calloc((size_t)V, sizeof(int64_t));
        b->resident = (uint8_t *)calloc((size_t)V, 1);
        b->tag = (uint8_t *)calloc((size_t)V, 1);
        if (!b->prio || !b->resident || !b->tag) return -1;
    } else {
        b->slot_gid = (int64_t *)malloc((size_t)(S * W) * sizeof(int64_t));
        b->slot_prio = (int64_t *)calloc((size_t)(S * W), sizeof(int64_t));
        b->slot_tag = (uint8_t *)calloc((size_t)(S * W), 1);
        b->slot_of = (int32_t *)malloc((size_t)V * sizeof(int32_t));
        if (!b->slot_gid || !b->slot_prio || !b->slot_tag || !b->slot_of) return -1;
        for (int64_t i = 0; i < S * W; i++) b->slot_gid[i] = -1;
        for (int64_t i = 0; i < V; i++) b->slot_of[i] = -1;
    }
    return 0;
}

static void buf_free(buf_t *b)
{
    free(b->count); free(b->prio); free(b->resident); free(b->tag);
    free(b->slot_gid); free(b->slot_prio); free(b->slot_tag); free(b->slot_of);
}

/* __contains__  runtime.py:61-62 */
static int buf_contains(const buf_t *b, int64_t g)
{
    return b->dense ? b->resident[g] : (b->slot_of[g] >= 0);
}

/* full  runtime.py:64-66 (per set buffer) */
static int buf_full(const buf_t *b, int64_t g)
{
    return b->count[g % b->S] >= b->W;
}

/* set_priority  runtime.py:78-81 (caller checked residency) */
static void buf_set_priority(buf_t *b, int64_t g, int64_t p)
{
    if (b->dense) b->prio[g] = p; else b->slot_prio[b->slot_of[g]] = p;
}

/* reference  runtime.py:93-98 */
static int buf_reference(buf_t *b, int64_t g)
{
    uint8_t *t = b->dense ? &b->tag[g] : &b->slot_tag[b->slot_of[g]];
    if (*t) { *t = 0; return 1; }
    return 0;
}

/* add  runtime.py:83-91 (caller guarantees not resident and not full) */
static void buf_add(buf_t *b, int64_t g, int64_t p, int prefetched)
{
    int64_t s = g % b->S;
    if (b->dense) {
        b->resident[g] = 1; b->prio[g] = p; b->tag[g] = (uint8_t)prefetched;
    } else {
        int64_t base = s * b->W, slot = -1;
        for (int64_t w = 0; w < b->W; w++)
            if (b->slot_gid[base + w] < 0) { slot = base + w; break; }
        b->slot_gid[slot] = g; b->slot_prio[slot] = p;
        b->slot_tag[slot] = (uint8_t)prefetched; b->slot_of[g] = (int32_t)slot;
    }
    b->count[s]++;
    b->occupancy++;
    if (b->occupancy > b->max_occupancy) b->max_occupancy = b->occupancy;
}

/* populate  runtime.py:100-112: evict argmin priority (ties -> smallest gid,
 * which is np.argmin's first-index rule over the gid-indexed array), then
 * age every resident priority > 0 by one. Operates on the set of g.        */
static int64_t buf_populate(buf_t *b, int64_t set)
{
    int64_t victim = -1;
    if (b->dense) {
        int64_t best = INT64_MAX;
        for (int64_t g = set; g < b->V; g += b->S)             /* :105-106 */
            if (b->resident[g] && b->prio[g] < best) { best = b->prio[g]; victim = g; }
        for (int64_t g = set; g < b->V; g += b->S)             /* :107-108 */
            if (b->resident[g] && b->prio[g] > 0) b->prio[g]--;
        b->resident[victim] = 0; b->tag[victim] = 0;            /* :109-110 */
    } else {
        int64_t base = set * b->W, vs = -1, bp = INT64_MAX, bg = INT64_MAX;
        for (int64_t w = 0; w < b->W; w++) {
            int64_t g = b->slot_gid[base + w];
            if (g < 0) continue;
            int64_t p = b->slot_prio[base + w];
            if (p < bp || (p == bp && g < bg)) { bp = p; bg = g; vs = base + w; }
        }
        for (int64_t w = 0; w < b->W; w++)
            if (b->slot_gid[base + w] >= 0 && b->slot_prio[base + w] > 0) b->slot_prio[base + w]--;
        victim = bg;
        b->slot_of[victim] = -1; b->slot_gid[vs] = -1; b->slot_tag[vs] = 0;
    }
    b->count[set]--;
    b->occupancy--;
    b->evictions++;
    return victim;
}

/* serve closure  runtime.py:254-264 */
static void serve(buf_t *b, int64_t g, int64_t *ctr, uint8_t *cls)
{
    if (buf_contains(b, g)) {
        if (buf_reference(b, g)) { ctr[C_PREFETCH_HITS]++; if (cls) *cls = 1; }
        else { ctr[C_CACHE_HITS]++; if (cls) *cls = 0; }
    } else {
        ctr[C_ON_DEMAND]++; if (cls) *cls = 2;
        if (buf_full(b, g)) buf_populate(b, g % b->S);
        buf_add(b, g, b->es, 0);
    }
}

/* load_embeddings  runtime.py:115-137 (Alg. 1); inputs already validated */
static void load_embeddings(buf_t *b, const int64_t *chunk, const uint8_t *bits, int32_t l_in,
                            const int64_t *pf, int32_t npf)
{
    for (int32_t i = 0; i < l_in; i++) {                       /* :126-130 */
        int64_t g = chunk[i];
        if (buf_contains(b, g)) buf_set_priority(b, g, (int64_t)bits[i] + b->es);
    }
    for (int32_t j = 0; j < npf; j++) {                        /* :131-137 */
        int64_t g = pf[j];
        if (buf_contains(b, g)) { buf_set_priority(b, g, b->es); continue; }
        if (buf_full(b, g)) buf_populate(b, g % b->S);
        buf_add(b, g, b->es, 1);
        b->inserts_pf++;
    }
}

/* number of chunks emitted by chunk()  trace.py:238-250 */
int64_t oracle_num_chunks(int64_t n, int32_t l_in, int32_t l_out, int32_t window_ratio)
{
    int64_t l_win = (int64_t)window_ratio * l_out, k = 0;
    for (int64_t origin = 0; origin + l_in + l_win <= n; origin += l_in) k++;
    return k;
}

/* per-chunk prefetch statistics  runtime.py:272-276 */
static void chunk_stats(const int64_t *win, int64_t l_win, const int64_t *pf, int32_t npf,
                        int64_t *useful, int64_t *num, int64_t *den)
{
    int64_t d = 0, u = 0, c = 0;
    for (int64_t i = 0; i < l_win; i++) {          /* |set(window)| */
        int dup = 0;
        for (int64_t j = 0; j < i; j++) if (win[j] == win[i]) { dup = 1; break; }
        if (!dup) d++;
    }
    for (int32_t j = 0; j < npf; j++) {            /* sum(p in wset)  :275 */
        for (int64_t i = 0; i < l_win; i++) if (win[i] == pf[j]) { u++; break; }
    }
    for (int32_t j = 0; j < npf; j++) {            /* |set(P) & wset|  :276 */
        int dup = 0;
        for (int32_t k = 0; k < j; k++) if (pf[k] == pf[j]) { dup = 1; break; }
        if (dup) continue;
        for (int64_t i = 0; i < l_win; i++) if (win[i] == pf[j]) { c++; break; }
    }
    *useful = u; *num = c; *den = d;
}

/*
 * replay  runtime.py:220-283.
 *   gids[n]                  trace.gid_array
 *   capacity, ways           ways == 0: one fully associative buffer (the
 *                            reference exactly); ways > 0: capacity/ways sets
 *   bits[K*l_in] or NULL     cache bits (NULL = caching_params None: zeros,
 *                            runtime.py:184-185)
 *   pf[K*pf_stride] or NULL  prefetch gids, -1 padded (NULL = no prefetcher)
 *   counters[C_NUM]          out
 *   coverage                 out, runtime.py:282
 *   access_class[n] or NULL  out: 0 cache hit, 1 prefetch hit, 2 on-demand
 * Returns 0, or -1 (allocation) / -2 (invalid config).
 */
int oracle_replay(const int64_t *gids, int64_t n, int64_t total_ids,
                  int64_t capacity, int64_t ways, int64_t eviction_speed,
                  int32_t l_in, int32_t l_out, int32_t window_ratio,
                  const uint8_t *bits, const int64_t *pf, int32_t pf_stride,
                  int dense, int64_t *counters, double *coverage,
                  uint8_t *access_class)
{
    if (capacity < 1 || eviction_speed < 1 || l_in < 1 || l_out < 1 || window_ratio < 1)
        return -2;
    if (ways < 0 || (ways > 0 && capacity % ways != 0)) return -2;
    int64_t S = ways > 0 ? capacity / ways : 1;
    int64_t W = ways > 0 ? ways : capacity;
    buf_t b;
    if (buf_init(&b, dense, total_ids, S, W, eviction_speed) != 0) { buf_free(&b); return -1; }
    for (int i = 0; i < C_NUM; i++) counters[i] = 0;

    int64_t K = oracle_num_chunks(n, l_in, l_out, window_ratio);
    int64_t l_win = (int64_t)window_ratio * l_out;
    static const uint8_t zero_bits[4096];
    double coverage_sum = 0.0;
    for (int64_t k = 0; k < K; k++) {                          /* :266-276 */
        int64_t origin = k * l_in;
        for (int32_t i = 0; i < l_in; i++)
            serve(&b, gids[origin + i], counters, access_class ? &access_class[origin + i] : NULL);
        const int64_t *pk = pf ? pf + k * pf_stride : NULL;
        int32_t npf = 0;
        if (pk) while (npf < pf_stride && pk[npf] >= 0) npf++;
        load_embeddings(&b, gids + origin, bits ? bits + k * l_in : zero_bits, l_in, pk, npf);
        int64_t u, num, den;
        chunk_stats(gids + origin + l_in, l_win, pk, npf, &u, &num, &den);
        counters[C_PREFETCH_ISSUED] += npf;
        counters[C_PREFETCH_USEFUL] += u;
        coverage_sum += (double)num / (double)den;
    }
    for (int64_t i = K * l_in; i < n; i++)                     /* :278-280 */
        serve(&b, gids[i], counters, access_class ? &access_class[i] : NULL);
    *coverage = K ? coverage_sum / (double)K : 0.0;           /* :282 */
    counters[C_EVICTIONS] = b.evictions;
    counters[C_PREFETCH_INSERTS] = b.inserts_pf;
    counters[C_MAX_OCCUPANCY] = b.max_occupancy;
    buf_free(&b);
    return 0;
}

/*
 * Set-associative LRU  cache_sim.py:92-106 (set = gid % set_count, one
 * OrderedDict per set: move_to_end on hit, popitem(last=False) when full).
 * ways == 0 means fully associative (cache_sim.py:52-58).
 */
int oracle_lru(const int64_t *gids, int64_t n, int64_t total_ids, int64_t capacity,
               int64_t ways, uint8_t *per_access_hit, int64_t *hits_out)
{
    if (capacity < 1 || ways < 0 || (ways > 0 && capacity % ways != 0)) return -2;
    int64_t S = ways > 0 ? capacity / ways : 1;
    int64_t W = ways > 0 ? ways : capacity;
    int64_t *slot_gid = (int64_t *)malloc((size_t)(S * W) * sizeof(int64_t));
    int64_t *slot_ts = (int64_t *)malloc((size_t)(S * W) * sizeof(int64_t));
    int32_t *slot_of = (int32_t *)malloc((size_t)total_ids * sizeof(int32_t));
    int64_t *count = (int64_t *)calloc((size_t)S, sizeof(int64_t));
    if (!slot_gid || !slot_ts || !slot_of || !count) {
        free(slot_gid); free(slot_ts); free(slot_of); free(count); return -1;
    }
    for (int64_t i = 0; i < S * W; i++) slot_gid[i] = -1;
    for (int64_t i = 0; i < total_ids; i++) slot_of[i] = -1;
    int64_t hits = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t g = gids[i], s = g % S, base = s * W;
        if (slot_of[g] >= 0) {                                 /* :98-100 */
            slot_ts[slot_of[g]] = i; hits++;
            if (per_access_hit) per_access_hit[i] = 1;
            continue;
        }
        if (per_access_hit) per_access_hit[i] = 0;
        int64_t slot = -1;
        if (count[s] == W) {                                   /* :103-104 */
            int64_t best = INT64_MAX;
            for (int64_t w = 0; w < W; w++)
                if (slot_ts[base + w] < best) { best = slot_ts[base + w]; slot = base + w; }
            slot_of[slot_gid[slot]] = -1;
            count[s]--;
        } else {
            for (int64_t w = 0; w < W; w++) if (slot_gid[base + w] < 0) { slot = base + w; break; }
        }
        slot_gid[slot] = g; slot_ts[slot] = i; slot_of[g] = (int32_t)slot;   /* :105 */
        count[s]++;
    }
    *hits_out = hits;
    free(slot_gid); free(slot_ts); free(slot_of); free(count);
    return 0;
}

/*
 * replay_policy_only with a prefetcher  runtime.py:304-349: fully associative
 * LRU where predicted rows are inserted at MRU with a prefetch tag.
 * counters as oracle_replay (evictions / inserts / occupancy left 0).
 */
int oracle_lru_prefetch(const int64_t *gids, int64_t n, int64_t total_ids, int64_t capacity,
                        int32_t l_in, int32_t l_out, int32_t window_ratio,
                        const int64_t *pf, int32_t pf_stride, int64_t *counters,
                        double *coverage)
{
    if (capacity < 1) return -2;
    int64_t *slot_gid = (int64_t *)malloc((size_t)capacity * sizeof(int64_t));
    int64_t *slot_ts = (int64_t *)malloc((size_t)capacity * sizeof(int64_t));
    uint8_t *slot_tag = (uint8_t *)calloc((size_t)capacity, 1);
    int32_t *slot_of = (int32_t *)malloc((size_t)total_ids * sizeof(int32_t));
    if (!slot_gid || !slot_ts || !slot_tag || !slot_of) {
        free(slot_gid); free(slot_ts); free(slot_tag); free(slot_of); return -1;
    }
    for (int64_t i = 0; i < capacity; i++) slot_gid[i] = -1;
    for (int64_t i = 0; i < total_ids; i++) slot_of[i] = -1;
    for (int i = 0; i < C_NUM; i++) counters[i] = 0;
    int64_t count = 0, clock = 0;

#define LRU_EVICT_IF_FULL()                                                     \
    do {                                                                        \
        if (count == capacity) {                                                \
            int64_t best = INT64_MAX, vs = -1;                                  \
            for (int64_t w = 0; w < capacity; w++)                              \
                if (slot_gid[w] >= 0 && slot_ts[w] < best) { best = slot_ts[w]; vs = w; } \
            slot_of[slot_gid[vs]] = -1; slot_gid[vs] = -1; slot_tag[vs] = 0; count--; \
        }                                                                       \
    } while (0)
#define LRU_INSERT(g, t)                                                        \
    do {                                                                        \
        int64_t fs = -1;                                                        \
        for (int64_t w = 0; w < capacity; w++) if (slot_gid[w] < 0) { fs = w; break; } \
        slot_gid[fs] = (g); slot_ts[fs] = clock++; slot_tag[fs] = (uint8_t)(t); \
        slot_of[(g)] = (int32_t)fs; count++;                                    \
    } while (0)

    int64_t K = oracle_num_chunks(n, l_in, l_out, window_ratio);
    int64_t l_win = (int64_t)window_ratio * l_out;
    double coverage_sum = 0.0;
    for (int64_t i = 0, k = 0; i < n; ) {
        /* serve  runtime.py:318-330 */
        int64_t end = (k < K) ? (k + 1) * l_in : n;
        for (; i < end; i++) {
            int64_t g = gids[i];
            if (slot_of[g] >= 0) {
                int32_t s = slot_of[g];
                if (slot_tag[s]) { slot_tag[s] = 0; counters[C_PREFETCH_HITS]++; }
                else counters[C_CACHE_HITS]++;
                slot_ts[s] = clock++;
            } else {
                counters[C_ON_DEMAND]++;
                LRU_EVICT_IF_FULL();
                LRU_INSERT(g, 0);
            }
        }
        if (k >= K) break;
        const int64_t *pk = pf ? pf + k * pf_stride : NULL;
        int32_t npf = 0;
        if (pk) while (npf < pf_stride && pk[npf] >= 0) npf++;
        for (int32_t j = 0; j < npf; j++) {                    /* :335-339 */
            int64_t p = pk[j];
            if (slot_of[p] < 0) { LRU_EVICT_IF_FULL(); LRU_INSERT(p, 1); }
        }
        int64_t u, num, den;
        chunk_stats(gids + k * l_in + l_in, l_win, pk, npf, &u, &num, &den);
        counters[C_PREFETCH_ISSUED] += npf;
        counters[C_PREFETCH_USEFUL] += u;
        coverage_sum += (double)num / (double)den;
        k++;
    }
#undef LRU_EVICT_IF_FULL
#undef LRU_INSERT
    *coverage = K ? coverage_sum / (double)K : 0.0;
    free(slot_gid); free(slot_ts); free(slot_tag); free(slot_of);
    return 0;
}

/* Sequential float64 coverage accumulation  runtime.py:276,282 */
double oracle_coverage_sum(const uint8_t *num, const uint8_t *den, int64_t K)
{
    double s = 0.0;
    for (int64_t k = 0; k < K; k++) s += (double)num[k] / (double)den[k];
    return K ? s / (double)K : 0.0;
}

/* generate_trace's sequential pass  trace.py:144-160.  With probability
 * `stickiness` the access reuses pool[floor(pool_coin * len)] (the pool holds
 * the last `pool_size` distinct ids, most recent first), otherwise it takes
 * the Zipf draw; the id then moves to the pool front (no-op when already
 * there), the pool keeping at most pool_size entries.  `pool` / `len` carry
 * the pool across consecutive blocks of one trace (start with *len = 0). */
int oracle_pool_pass(const int64_t *zipf_gids, const double *sticky_coin,
                     const double *pool_coin, int64_t n, double stickiness,
                     int32_t pool_size, int64_t *pool, int32_t *len_io, int64_t *out)
{
    if (n < 0 || pool_size < 1 || !pool || !len_io) return -1;
    int32_t len = *len_io;
    for (int64_t i = 0; i < n; i++) {
        int64_t g = (len > 0 && sticky_coin[i] < stickiness)
                        ? pool[(int64_t)(pool_coin[i] * (double)len)]
                        : zipf_gids[i];
        out[i] = g;
        if (len > 0 && pool[0] == g) continue;
        int32_t j = 0;
        while (j < len && pool[j] != g) j++;
        if (j == len && len < pool_size) len++;      /* new id: the pool grows   */
        if (j == len) j = len - 1;                   /* full: the oldest drops   */
        for (; j > 0; j--) pool[j] = pool[j - 1];    /* shift the front down     */
        pool[0] = g;
    }
    *len_io = len;
    return 0;
}
