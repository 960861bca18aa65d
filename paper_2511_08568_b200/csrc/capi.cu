// extern "C" entry points declared in include/recmg.h.
#include <chrono>
#include <cstdio>
#include <string.h>

#include "lstm.cuh"
#include "lstm_tc.cuh"
#include "model_layout.cuh"
#include "partition.cuh"
#include "replay.cuh"

using namespace recmg;

#include <atomic>
namespace recmg {
static std::atomic<unsigned long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace recmg

namespace {

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

struct ReplayPlan {
    Geometry g;
    int64_t K = 0, Ec = 0, E = 0;   // E: events of this call's chunk range (+ tail)
    int64_t k0 = 0, nk = 0;
    bool tail = true;
    bool vals = false;
    uint32_t *ev = nullptr, *vv = nullptr;
    PartitionBuffers pb;
};

bool plan_replay(const recmg_buffer_cfg *cfg, int64_t n, int32_t l_in, int32_t l_out,
                 int32_t window_ratio, int32_t pf_stride, bool with_class, int64_t k_begin,
                 int64_t k_end, bool with_tail, Arena &a, ReplayPlan &p) {
    if (!geometry_of(cfg, &p.g)) return false;
    if (cfg->policy != RECMG_POLICY_PRIORITY && cfg->policy != RECMG_POLICY_LRU_PF) return false;
    if (cfg->policy == RECMG_POLICY_PRIORITY && cfg->eviction_speed < 1) return false;
    if (n < 0 || l_in < 1 || l_out < 1 || window_ratio < 1 || pf_stride < 0) return false;
    if ((int64_t)window_ratio * l_out > 65535) return false;  // uint16 coverage counts
    p.K = recmg_num_chunks(n, l_in, l_out, window_ratio);
    if (k_begin < 0) k_begin = 0;
    if (k_end < 0 || k_end > p.K) k_end = p.K;
    if (k_begin > k_end) return false;
    if (with_tail && k_end != p.K) return false;   // the tail follows the last chunk
    p.k0 = k_begin;
    p.nk = k_end - k_begin;
    p.tail = with_tail;
    p.Ec = 2 * (int64_t)l_in + pf_stride;
    p.E = p.nk * p.Ec + (with_tail ? (n - p.K * l_in) : 0);
    if (p.K * p.Ec + n >= ((int64_t)1 << 32)) return false;
    p.vals = with_class && p.g.S > 1;
    p.ev = a.take<uint32_t>((size_t)p.E);
    p.vv = p.vals ? a.take<uint32_t>((size_t)p.E) : nullptr;
    if (p.g.S > 1) partition_plan(a, p.pb, p.E, p.g.S, p.vals);
    return true;
}

#ifdef RECMG_CHAIN_TIMING
// diagnostic builds only: host wall time of each stage of the replay chain
struct ChainTimer {
    cudaStream_t s;
    std::chrono::steady_clock::time_point t;
    explicit ChainTimer(cudaStream_t st) : s(st) {
        cudaStreamSynchronize(s);
        t = std::chrono::steady_clock::now();
    }
    void lap(const char *what) {
        cudaStreamSynchronize(s);
        const auto u = std::chrono::steady_clock::now();
        fprintf(stderr, "chain %-10s %8.3f ms\n", what,
                std::chrono::duration<double, std::milli>(u - t).count());
        t = u;
    }
};
#define RECMG_LAP(x) tm.lap(x)
#else
struct ChainTimer {
    explicit ChainTimer(cudaStream_t) {}
};
#define RECMG_LAP(x) ((void)0)
#endif

int replay_range(const recmg_buffer_cfg *cfg, void *state, const int32_t *gids, int64_t n,
                 int32_t l_in, int32_t l_out, int32_t window_ratio, int64_t k_begin,
                 int64_t k_end, int with_tail, const uint8_t *bits, const int32_t *pf,
                 int32_t pf_stride, recmg_counters *counters, uint16_t *cov_num,
                 uint16_t *cov_den, uint8_t *access_class, void *ws, size_t ws_bytes,
                 cudaStream_t s, int32_t flags = 0, const recmg_buffer_cfg *lru_cfg = nullptr,
                 void *lru_state = nullptr, int64_t *lru_hm = nullptr) {
    if (!pf) pf_stride = 0;
    ChainTimer tm(s);
    (void)tm;
    Arena a{(char *)ws, ws_bytes, 0};
    ReplayPlan p;
    if (!state || !counters || (n > 0 && !gids)) return RECMG_E_INVALID_CONFIG;
    if (!plan_replay(cfg, n, l_in, l_out, window_ratio, pf_stride, access_class != nullptr,
                     k_begin, k_end, with_tail != 0, a, p))
        return RECMG_E_INVALID_CONFIG;
    if (p.nk > 0 && !(flags & RECMG_REPLAY_SKIP_STATS)) {
        prefetch_stats_kernel<<<(unsigned)((p.nk + 255) / 256), 256, 0, s>>>(
            gids, p.k0, p.nk, l_in, window_ratio * l_out, pf, pf_stride, cov_num, cov_den,
            counters);
        RECMG_LAUNCH_CHECK();
        RECMG_LAP("stats");
    }
    if (p.E == 0) return RECMG_OK;
    if (!a.ok() || !ws) return RECMG_E_WORKSPACE;
    StateView st = state_view(state, cfg, p.g);
    const uint32_t magic = set_magic((uint32_t)p.g.S);
    int64_t i_begin = 0;
    if (l_in <= 16 && p.nk > 0) {   // thread per chunk, then the tail below
        build_chunk_events_kernel<16><<<(unsigned)imin64((p.nk + 127) / 128, 16 * kSmCount), 128,
                                        0, s>>>(gids, l_in, bits, pf, pf_stride, p.K, p.k0, p.nk,
                                                (uint32_t)p.g.S, magic, p.ev, p.vv, counters,
                                                access_class);
        RECMG_LAUNCH_CHECK();
        RECMG_LAP("events");
        i_begin = p.nk * p.Ec;
    }
    if (p.E > i_begin) {
        build_events_kernel<<<(unsigned)imin64((p.E - i_begin + 255) / 256, 16 * kSmCount), 256, 0,
                              s>>>(gids, n, l_in, bits, pf, pf_stride, p.K, p.k0, p.nk,
                                   p.tail ? 1 : 0, (uint32_t)p.g.S, magic, i_begin, p.ev, p.vv,
                                   counters, access_class);
        RECMG_LAUNCH_CHECK();
    }
    uint32_t *ev = p.ev, *vv = p.vv;
    ReplayArgs ra;
    memset(&ra, 0, sizeof(ra));
    if (p.g.S > 1) {
        int rc = partition_run(p.pb, ev, vv, s);
        if (rc) return rc;
        RECMG_LAP("partition");
        ra.seg_start = p.pb.seg_start;
        ra.seg_end = p.pb.seg_end;
        ra.heavy = p.g.wide ? nullptr : p.pb.heavy;
        ra.work = p.g.wide ? nullptr : p.pb.work;
    }
    ra.ev = ev;
    ra.vals = vv;
    ra.E = p.E;
    ra.S = p.g.S;
    ra.W = p.g.W;
    ra.es = cfg->eviction_speed;
    ra.gid_bits = gid_bits_of(cfg->total_ids);
    ra.total_ids = cfg->total_ids;
    ra.l_in = l_in;
    ra.Ec = p.Ec;
    ra.K = p.K;
    ra.ev_base = p.k0 * p.Ec;
    ra.st = st;
    ra.ctr = counters;
    ra.access_class = access_class;
    // the LRU comparator fused in (recmg_replay_chunks_lru): the same sets, its
    // own state, the serves of these events; hits = accesses - misses
    ReplayArgs rl;
    const ReplayArgs *lru2 = nullptr;
    if (lru_cfg) {
        Geometry gl;
        if (!geometry_of(lru_cfg, &gl) || lru_cfg->policy != RECMG_POLICY_LRU || !lru_state ||
            !lru_hm || gl.S != p.g.S || gl.W != p.g.W || p.g.wide || p.g.W > 32 || p.g.S < 2 ||
            cfg->policy != RECMG_POLICY_PRIORITY || lru_cfg->total_ids != cfg->total_ids)
            return RECMG_E_INVALID_CONFIG;
        rl = ra;
        rl.st = state_view(lru_state, lru_cfg, gl);
        rl.ctr = nullptr;
        rl.access_class = nullptr;
        rl.per_access_hit = nullptr;
        rl.next_use = nullptr;
        rl.hits_misses = lru_hm;
        rl.es = lru_cfg->eviction_speed;
        rl.serve_only = 1;
        lru2 = &rl;
        const int64_t n_acc = p.nk * l_in + (p.tail ? n - p.K * l_in : 0);
        add_i64_kernel<<<1, 1, 0, s>>>(lru_hm, n_acc);
        RECMG_LAUNCH_CHECK();
    }
    int rc = launch_replay(cfg->policy, !p.g.wide, access_class != nullptr, ra, p.g.S, s, lru2);
    if (rc) return rc;
    RECMG_LAP("replay");
    if (lru2) {
        // the comparator's clocks are event positions of this call: keep them
        // monotonic across calls
        clock_bump_kernel<<<1, 1, 0, s>>>(rl.st.header, p.E);
        RECMG_LAUNCH_CHECK();
    }
    if (cfg->policy == RECMG_POLICY_LRU_PF) {
        // clocks are event positions of this call: keep them monotonic across calls
        clock_bump_kernel<<<1, 1, 0, s>>>(st.header, p.E);
        RECMG_LAUNCH_CHECK();
    }
    return RECMG_OK;
}

}  // namespace

extern "C" {

const char *recmg_status_string(int status) {
    switch (status) {
        case RECMG_OK: return "ok";
        case RECMG_E_INVALID_CONFIG: return "invalid configuration";
        case RECMG_E_VOCAB_MISMATCH: return "model vocabulary does not match trace";
        case RECMG_E_OUT_OF_VOCAB: return "embedding index outside the vocabulary";
        case RECMG_E_BUFFER_STATE: return "buffer operation not valid in this state";
        case RECMG_E_NON_FINITE: return "non-finite value";
        case RECMG_E_CUDA: return "CUDA error";
        case RECMG_E_WORKSPACE: return "workspace too small";
        default: return "unknown status";
    }
}

const char *recmg_status_category(int status) {
    switch (status) {
        case RECMG_OK: return "ok";
        case RECMG_E_INVALID_CONFIG: return "invalid-config";
        case RECMG_E_VOCAB_MISMATCH: return "vocabulary-mismatch";
        case RECMG_E_OUT_OF_VOCAB: return "out-of-vocabulary";
        case RECMG_E_BUFFER_STATE: return "buffer-state";
        case RECMG_E_NON_FINITE: return "non-finite";
        default: return "error";
    }
}

uint64_t recmg_launch_count(void) { return g_launches.load(); }

int64_t recmg_num_chunks(int64_t n, int32_t l_in, int32_t l_out, int32_t window_ratio) {
    // trace.py:238-250: origins 0, l_in, ... while origin + l_in + l_win <= n
    const int64_t l_win = (int64_t)window_ratio * l_out;
    if (l_in < 1 || n < l_in + l_win) return 0;
    return (n - l_in - l_win) / l_in + 1;
}

size_t recmg_buffer_state_bytes(const recmg_buffer_cfg *cfg) {
    Geometry g;
    if (!geometry_of(cfg, &g)) return 0;
    return state_bytes(cfg, g);
}

int recmg_buffer_reset(const recmg_buffer_cfg *cfg, void *state, void *stream) {
    Geometry g;
    if (!geometry_of(cfg, &g) || !state) return RECMG_E_INVALID_CONFIG;
    if (cfg->policy == RECMG_POLICY_PRIORITY && cfg->eviction_speed < 1) return RECMG_E_INVALID_CONFIG;
    StateView v = state_view(state, cfg, g);
    const int64_t SW = g.S * g.W;
    const int64_t work = SW > cfg->total_ids ? SW : cfg->total_ids;
    unsigned grid = (unsigned)((work + 255) / 256);
    if (grid > 8 * kSmCount) grid = 8 * kSmCount;
    if (grid < 1) grid = 1;
    state_reset_kernel<<<grid, 256, 0, as_stream(stream)>>>(v, SW, g.S, cfg->total_ids);
    RECMG_LAUNCH_CHECK();
    return RECMG_OK;
}

int recmg_replay_workspace_bytes(const recmg_buffer_cfg *cfg, int64_t n, int32_t l_in,
                                 int32_t l_out, int32_t window_ratio, int32_t pf_stride,
                                 size_t *bytes) {
    Arena a{nullptr, 0, 0};
    ReplayPlan p;
    if (!plan_replay(cfg, n, l_in, l_out, window_ratio, pf_stride, true, 0, -1, true, a, p))
        return RECMG_E_INVALID_CONFIG;
    *bytes = a.used + 256;
    return RECMG_OK;
}

int recmg_replay(const recmg_buffer_cfg *cfg, void *state, const int32_t *gids, int64_t n,
                 int32_t l_in, int32_t l_out, int32_t window_ratio, const uint8_t *bits,
                 const int32_t *pf, int32_t pf_stride, recmg_counters *counters,
                 uint16_t *cov_num, uint16_t *cov_den, uint8_t *access_class, void *ws,
                 size_t ws_bytes, void *stream) {
    return replay_range(cfg, state, gids, n, l_in, l_out, window_ratio, 0, -1, 1, bits, pf,
                        pf_stride, counters, cov_num, cov_den, access_class, ws, ws_bytes,
                        as_stream(stream));
}

int recmg_replay_chunks_ex(const recmg_buffer_cfg *cfg, void *state, const int32_t *gids,
                           int64_t n, int32_t l_in, int32_t l_out, int32_t window_ratio,
                           int64_t k_begin, int64_t k_end, int32_t with_tail, const uint8_t *bits,
                           const int32_t *pf, int32_t pf_stride, recmg_counters *counters,
                           uint16_t *cov_num, uint16_t *cov_den, uint8_t *access_class,
                           void *ws, size_t ws_bytes, int32_t flags, void *stream) {
    if (flags & ~RECMG_REPLAY_SKIP_STATS) return RECMG_E_INVALID_CONFIG;
    return replay_range(cfg, state, gids, n, l_in, l_out, window_ratio, k_begin, k_end,
                        with_tail, bits, pf, pf_stride, counters, cov_num, cov_den,
                        access_class, ws, ws_bytes, as_stream(stream), flags);
}

int recmg_replay_chunks_lru(const recmg_buffer_cfg *cfg, void *state, const int32_t *gids,
                            int64_t n, int32_t l_in, int32_t l_out, int32_t window_ratio,
                            int64_t k_begin, int64_t k_end, int32_t with_tail,
                            const uint8_t *bits, const int32_t *pf, int32_t pf_stride,
                            recmg_counters *counters, uint16_t *cov_num, uint16_t *cov_den,
                            const recmg_buffer_cfg *lru_cfg, void *lru_state,
                            int64_t *lru_hits_misses, void *ws, size_t ws_bytes, int32_t flags,
                            void *stream) {
    if (flags & ~RECMG_REPLAY_SKIP_STATS) return RECMG_E_INVALID_CONFIG;
    if (!lru_cfg) return RECMG_E_INVALID_CONFIG;
    return replay_range(cfg, state, gids, n, l_in, l_out, window_ratio, k_begin, k_end,
                        with_tail, bits, pf, pf_stride, counters, cov_num, cov_den, nullptr, ws,
                        ws_bytes, as_stream(stream), flags, lru_cfg, lru_state, lru_hits_misses);
}

int recmg_prefetch_stats(const int32_t *gids, int64_t n, int32_t l_in, int32_t l_out,
                         int32_t window_ratio, int64_t k_begin, int64_t k_end, const int32_t *pf,
                         int32_t pf_stride, recmg_counters *counters, uint16_t *cov_num,
                         uint16_t *cov_den, void *stream) {
    if (n < 0 || l_in < 1 || l_out < 1 || window_ratio < 1 || pf_stride < 0 || !counters ||
        (int64_t)window_ratio * l_out > 65535)
        return RECMG_E_INVALID_CONFIG;
    const int64_t K = recmg_num_chunks(n, l_in, l_out, window_ratio);
    if (k_begin < 0) k_begin = 0;
    if (k_end < 0 || k_end > K) k_end = K;
    if (k_begin > k_end || (k_end > k_begin && !gids)) return RECMG_E_INVALID_CONFIG;
    if (!pf) pf_stride = 0;
    const int64_t nk = k_end - k_begin;
    if (nk == 0) return RECMG_OK;
    cudaStream_t s = as_stream(stream);
    prefetch_stats_kernel<<<(unsigned)((nk + 255) / 256), 256, 0, s>>>(
        gids, k_begin, nk, l_in, window_ratio * l_out, pf, pf_stride, cov_num, cov_den, counters);
    RECMG_LAUNCH_CHECK();
    return RECMG_OK;
}

int recmg_replay_chunks(const recmg_buffer_cfg *cfg, void *state, const int32_t *gids, int64_t n,
                        int32_t l_in, int32_t l_out, int32_t window_ratio, int64_t k_begin,
                        int64_t k_end, int32_t with_tail, const uint8_t *bits, const int32_t *pf,
                        int32_t pf_stride, recmg_counters *counters, uint16_t *cov_num,
                        uint16_t *cov_den, uint8_t *access_class, void *ws, size_t ws_bytes,
                        void *stream) {
    return replay_range(cfg, state, gids, n, l_in, l_out, window_ratio, k_begin, k_end,
                        with_tail, bits, pf, pf_stride, counters, cov_num, cov_den,
                        access_class, ws, ws_bytes, as_stream(stream));
}

double recmg_coverage_mean(const uint16_t *num, const uint16_t *den, int64_t K) {
    // runtime.py:276 accumulates len(P & W)/len(W) left to right in float64,
    // runtime.py:282 divides by the chunk count.
    double acc = 0.0;
    for (int64_t k = 0; k < K; k++) acc += (double)num[k] / (double)den[k];
    return K ? acc / (double)K : 0.0;
}

double recmg_coverage_accumulate(const uint16_t *num, const uint16_t *den, int64_t count,
                                 double acc) {
    for (int64_t k = 0; k < count; k++) acc += (double)num[k] / (double)den[k];
    return acc;
}

static bool sim_policy_ok(const recmg_buffer_cfg *cfg, const Geometry &g) {
    switch (cfg->policy) {
        case RECMG_POLICY_LRU:
        case RECMG_POLICY_LFU:
        case RECMG_POLICY_OPTGEN: return true;
        case RECMG_POLICY_SRRIP: return cfg->eviction_speed >= 0;
        default: return false;
    }
}

struct SimPlan {
    uint32_t *keys = nullptr, *vals = nullptr;
    PartitionBuffers pb, pb_id;        // by set; by id (OPTGEN next use)
    int32_t *next_use = nullptr;
    uint8_t *hit = nullptr;            // OPTGEN keep bits need the hits
    uint32_t *ids = nullptr, *pos = nullptr;
};

static void plan_sim(const recmg_buffer_cfg *cfg, const Geometry &g, int64_t n, bool keep,
                     bool have_hits, Arena &a, SimPlan &p) {
    p.keys = a.take<uint32_t>((size_t)n);
    p.vals = a.take<uint32_t>((size_t)n);
    if (g.S > 1) partition_plan(a, p.pb, n, g.S, true);
    if (cfg->policy == RECMG_POLICY_OPTGEN) {
        p.next_use = a.take<int32_t>((size_t)n);
        p.ids = a.take<uint32_t>((size_t)n);
        p.pos = a.take<uint32_t>((size_t)n);
        partition_plan(a, p.pb_id, n, cfg->total_ids, true);
        if (keep && !have_hits) p.hit = a.take<uint8_t>((size_t)n);
    }
}

int recmg_simulate_workspace_bytes(const recmg_buffer_cfg *cfg, int64_t n, size_t *bytes) {
    Geometry g;
    if (!geometry_of(cfg, &g) || !sim_policy_ok(cfg, g) || n < 0) return RECMG_E_INVALID_CONFIG;
    Arena a{nullptr, 0, 0};
    SimPlan p;
    plan_sim(cfg, g, n, true, false, a, p);
    *bytes = a.used + 256;
    return RECMG_OK;
}

__global__ void iota_copy_kernel(const int32_t *in, uint32_t *keys, uint32_t *vals, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = (uint32_t)in[i];  // EV_SERVE == 0: the gid is the event word
        if (vals) vals[i] = (uint32_t)i;
    }
}

// LRU serve stream with collapsed repeats: an access whose previous same-set
// access (within the last kLookback accesses) names the same id is an LRU hit
// that leaves its way most recent -- no way of the set can pass it in
// between -- so it is counted as a hit here and emitted as an empty event
// (cache_sim.py:92-106; the same argument as build_events_kernel's).
constexpr int kLookback = 8;
__global__ void lru_events_kernel(const int32_t *in, uint32_t *keys, uint32_t *vals, int64_t n,
                                  uint32_t S, uint8_t *per_access_hit, int64_t *hits_misses) {
    unsigned collapsed = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t g = (uint32_t)in[i];
        int64_t q = i - 1;
        const int64_t lo = i - kLookback > 0 ? i - kLookback : 0;
        while (q >= lo && (uint32_t)in[q] != g) q--;
        bool dup = q >= lo;
        if (dup) {
            const uint32_t set = g % S;
            for (int64_t p = q + 1; p < i && dup; p++) dup = (uint32_t)in[p] % S != set;
        }
        keys[i] = dup ? kGidMask : g;   // EV_SERVE == 0: the gid is the event word
        if (vals) vals[i] = (uint32_t)i;
        if (dup) {
            collapsed++;
        }
    }
    collapsed = __reduce_add_sync(0xFFFFFFFFu, collapsed);
    if ((threadIdx.x & 31) == 0 && collapsed)
        atomicAdd((unsigned long long *)&hits_misses[0], (unsigned long long)collapsed);
}

int recmg_simulate_ex(const recmg_buffer_cfg *cfg, void *state, const int32_t *gids, int64_t n,
                      uint8_t *per_access_hit, uint8_t *keep_decisions, int64_t *hits_misses,
                      void *ws, size_t ws_bytes, void *stream) {
    cudaStream_t s = as_stream(stream);
    Geometry g;
    if (!geometry_of(cfg, &g) || !sim_policy_ok(cfg, g) || !state || n < 0)
        return RECMG_E_INVALID_CONFIG;
    if (keep_decisions && cfg->policy != RECMG_POLICY_OPTGEN) return RECMG_E_INVALID_CONFIG;
    if (n == 0) return RECMG_OK;
    Arena a{(char *)ws, ws_bytes, 0};
    SimPlan p;
    plan_sim(cfg, g, n, keep_decisions != nullptr, per_access_hit != nullptr, a, p);
    if (!a.ok() || !ws) return RECMG_E_WORKSPACE;
    const unsigned grid = (unsigned)imin64((n + 255) / 256, 16 * kSmCount);
    uint8_t *hit = per_access_hit ? per_access_hit : p.hit;
    // every access a hit until a kernel writes its miss: hit runs (most of a
    // skewed trace) then cost no scattered byte stores
    if (hit) RECMG_CUDA_TRY(cudaMemsetAsync(hit, 1, (size_t)n, s));
    if (cfg->policy == RECMG_POLICY_OPTGEN) {
        // next use of every access: stable sort by id, neighbours (cache_sim.py:80-89)
        iota_copy_kernel<<<grid, 256, 0, s>>>(gids, p.ids, p.pos, n);
        RECMG_LAUNCH_CHECK();
        uint32_t *ki = p.ids, *vi = p.pos;
        int rc = partition_run(p.pb_id, ki, vi, s);
        if (rc) return rc;
        next_use_kernel<<<grid, 256, 0, s>>>(ki, vi, n, p.next_use);
        RECMG_LAUNCH_CHECK();
    }
    if (cfg->policy == RECMG_POLICY_LRU && hits_misses)
        lru_events_kernel<<<grid, 256, 0, s>>>(gids, p.keys, p.vals, n, (uint32_t)g.S, hit,
                                               hits_misses);
    else
        iota_copy_kernel<<<grid, 256, 0, s>>>(gids, p.keys, p.vals, n);
    RECMG_LAUNCH_CHECK();
    ReplayArgs ra;
    memset(&ra, 0, sizeof(ra));
    uint32_t *k = p.keys, *v = p.vals;
    if (g.S > 1) {
        int rc = partition_run(p.pb, k, v, s);
        if (rc) return rc;
        ra.seg_start = p.pb.seg_start;
        ra.seg_end = p.pb.seg_end;
        ra.heavy = g.wide ? nullptr : p.pb.heavy;
        ra.work = g.wide ? nullptr : p.pb.work;
    }
    ra.ev = k;
    ra.vals = v;
    ra.E = n;
    ra.S = g.S;
    ra.W = g.W;
    ra.es = cfg->eviction_speed;            // SRRIP: max rrpv
    ra.gid_bits = gid_bits_of(cfg->total_ids);
    ra.total_ids = cfg->total_ids;
    ra.st = state_view(state, cfg, g);
    ra.hits_misses = hits_misses;
    ra.per_access_hit = hit;
    ra.next_use = p.next_use;
    int rc = launch_replay(cfg->policy, !g.wide, false, ra, g.S, s);
    if (rc) return rc;
    clock_bump_kernel<<<1, 1, 0, s>>>(ra.st.header, n);
    RECMG_LAUNCH_CHECK();
    if (keep_decisions) {
        keep_kernel<<<grid, 256, 0, s>>>(p.next_use, hit, n, keep_decisions);
        RECMG_LAUNCH_CHECK();
    }
    return RECMG_OK;
}

int recmg_simulate(const recmg_buffer_cfg *cfg, void *state, const int32_t *gids, int64_t n,
                   uint8_t *per_access_hit, int64_t *hits_misses, void *ws, size_t ws_bytes,
                   void *stream) {
    return recmg_simulate_ex(cfg, state, gids, n, per_access_hit, nullptr, hits_misses, ws,
                             ws_bytes, stream);
}

int recmg_buffer_op(const recmg_buffer_cfg *cfg, void *state, int32_t op, int64_t gid,
                    int64_t arg, int32_t flag, int64_t *result, void *stream) {
    Geometry g;
    if (!geometry_of(cfg, &g) || !state || !result) return RECMG_E_INVALID_CONFIG;
    if (op < RECMG_OP_ADD || op > RECMG_OP_QUERY) return RECMG_E_INVALID_CONFIG;
    if (op != RECMG_OP_POPULATE && (gid < 0 || gid >= cfg->total_ids)) return RECMG_E_OUT_OF_VOCAB;
    if (op == RECMG_OP_POPULATE && (arg < 0 || arg >= g.S)) return RECMG_E_INVALID_CONFIG;
    buffer_op_kernel<<<1, 32, 0, as_stream(stream)>>>(state_view(state, cfg, g), g.S, g.W, op, gid,
                                                      arg, flag, result);
    RECMG_LAUNCH_CHECK();
    return RECMG_OK;
}

// ---- models -----------------------------------------------------------------
int64_t recmg_model_dense_floats(const recmg_model_shape *shape) {
    if (!shape_ok(shape)) return -1;
    return raw_layout(shape).total;
}

static size_t dense_bytes_aligned(const recmg_model_shape *shape) {
    return align_up((size_t)packed_layout(shape).total * sizeof(float), 256);
}

size_t recmg_model_packed_bytes(const recmg_model_shape *shape, int32_t precision) {
    if (!shape_ok(shape)) return 0;
    if (precision == RECMG_PREC_FP32) return (size_t)packed_layout(shape).total * sizeof(float);
    if ((precision == RECMG_PREC_TC32 || precision == RECMG_PREC_TC16) && tc_supported(shape))
        return dense_bytes_aligned(shape) + (size_t)tc_layout(shape).total;
    return 0;
}

int recmg_model_pack(const recmg_model_shape *shape, const float *dense_raw, void *packed,
                     int32_t precision, void *stream) {
    if (!shape_ok(shape) || precision != RECMG_PREC_FP32 || !dense_raw || !packed)
        return RECMG_E_INVALID_CONFIG;
    return model_pack(shape, dense_raw, packed, as_stream(stream));
}

int recmg_model_pack_tc(const recmg_model_shape *shape, const float *dense_raw,
                        const float *embed_id, const int64_t *table_offsets, void *packed,
                        void *stream) {
    if (!tc_supported(shape) || !dense_raw || !embed_id || !table_offsets || !packed)
        return RECMG_E_INVALID_CONFIG;
    return model_pack_tc(shape, dense_raw, embed_id, table_offsets, packed,
                         (char *)packed + dense_bytes_aligned(shape), as_stream(stream));
}

size_t recmg_model_workspace_bytes(const recmg_model_shape *shape, int32_t precision,
                                   int64_t batch) {
    if ((precision == RECMG_PREC_TC32 || precision == RECMG_PREC_TC16) && tc_supported(shape)) return tc_workspace_bytes(shape, batch);
    return 0;
}

int recmg_model_forward_signal(const recmg_model_shape *shape, int32_t precision,
                               const float *embed_id, const void *packed, const int32_t *gid,
                               const int32_t *tid, int64_t batch, int64_t decode_ids,
                               float *logits, uint8_t *bits, int32_t *pf_gid, void *ws,
                               size_t ws_bytes, int32_t *progress, int64_t piece_chunks,
                               void *stream) {
    if (!shape_ok(shape) || batch < 0 || !logits || decode_ids < 0 ||
        decode_ids >= (int64_t)kGidMask || !progress)
        return RECMG_E_INVALID_CONFIG;
    if (batch > 0 && (!packed || !gid || !tid)) return RECMG_E_INVALID_CONFIG;
    if (!((precision == RECMG_PREC_TC32 || precision == RECMG_PREC_TC16) && tc_supported(shape)))
        return RECMG_E_INVALID_CONFIG;
    return model_forward_tc(shape, packed, (const char *)packed + dense_bytes_aligned(shape), gid,
                            tid, batch, logits, bits, pf_gid, ws, ws_bytes, as_stream(stream),
                            nullptr, decode_ids, precision == RECMG_PREC_TC16, progress,
                            piece_chunks);
}

int recmg_wait_progress(const int32_t *progress, int64_t piece, int32_t target, void *stream) {
    if (!progress || piece < 0 || target < 0) return RECMG_E_INVALID_CONFIG;
    return wait_progress(progress + piece, target, as_stream(stream));
}

int recmg_model_forward_ex(const recmg_model_shape *shape, int32_t precision,
                           const float *embed_id, const void *packed, const int32_t *gid,
                           const int32_t *tid, int64_t batch, int64_t decode_ids, float *logits,
                           uint8_t *bits, int32_t *pf_gid, void *ws, size_t ws_bytes,
                           void *stream) {
    if (!shape_ok(shape) || batch < 0 || !logits || decode_ids < 0 ||
        decode_ids >= (int64_t)kGidMask)
        return RECMG_E_INVALID_CONFIG;
    if (batch > 0 && (!packed || !gid || !tid)) return RECMG_E_INVALID_CONFIG;
    if (precision == RECMG_PREC_TC32 || precision == RECMG_PREC_TC16) {
        if (!tc_supported(shape)) return RECMG_E_INVALID_CONFIG;
        return model_forward_tc(shape, packed, (const char *)packed + dense_bytes_aligned(shape),
                                gid, tid, batch, logits, bits, pf_gid, ws, ws_bytes,
                                as_stream(stream), nullptr, decode_ids,
                                precision == RECMG_PREC_TC16);
    }
    if (precision != RECMG_PREC_FP32) return RECMG_E_INVALID_CONFIG;
    if (batch > 0 && !embed_id) return RECMG_E_INVALID_CONFIG;
    return model_forward_fp32(shape, embed_id, packed, gid, tid, batch, logits, bits, pf_gid,
                              as_stream(stream), decode_ids);
}

int recmg_model_forward(const recmg_model_shape *shape, int32_t precision,
                        const float *embed_id, const void *packed, const int32_t *gid,
                        const int32_t *tid, int64_t batch, float *logits, uint8_t *bits,
                        int32_t *pf_gid, void *ws, size_t ws_bytes, void *stream) {
    return recmg_model_forward_ex(shape, precision, embed_id, packed, gid, tid, batch, 0, logits,
                                  bits, pf_gid, ws, ws_bytes, stream);
}

int recmg_set_model_sm_budget(int n) { return set_model_sm_budget(n); }

int recmg_model_forward_profile(const recmg_model_shape *shape, const void *packed,
                                const int32_t *gid, const int32_t *tid, int64_t batch,
                                float *logits, void *ws, size_t ws_bytes, long long *prof,
                                void *stream) {
    if (!tc_supported(shape) || !prof) return RECMG_E_INVALID_CONFIG;
    return model_forward_tc(shape, packed, (const char *)packed + dense_bytes_aligned(shape), gid,
                            tid, batch, logits, nullptr, nullptr, ws, ws_bytes,
                            as_stream(stream), prof);
}

// ---- trace helpers -----------------------------------------------------------
__global__ void table_ids_kernel(const int32_t *gids, int64_t n, const int64_t *offsets,
                                 int32_t n_tables, int32_t *tid) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = gids[i];
        // searchsorted(offsets, g, side="right") - 1  (trace.py:86)
        int lo = 0, hi = n_tables;  // offsets[lo] <= g < offsets[hi]
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(offsets + mid) <= g) lo = mid; else hi = mid;
        }
        tid[i] = lo;
    }
}

int recmg_table_ids(const int32_t *gids, int64_t n, const int64_t *offsets, int32_t n_tables,
                    int32_t *tid, void *stream) {
    if (n < 0 || n_tables < 1) return RECMG_E_INVALID_CONFIG;
    if (n == 0) return RECMG_OK;
    table_ids_kernel<<<(unsigned)imin64((n + 255) / 256, 16 * kSmCount), 256, 0,
                       as_stream(stream)>>>(gids, n, offsets, n_tables, tid);
    RECMG_LAUNCH_CHECK();
    return RECMG_OK;
}

// global gid -> (shard-local row, shard-local table) for a table shard
__global__ void shard_local_ids_kernel(const int32_t *gids, int64_t n, const int64_t *offsets,
                                       int32_t n_tables, const int32_t *table_local,
                                       const int64_t *local_offsets, int32_t *lgid,
                                       int32_t *ltid) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = gids[i];
        int lo = 0, hi = n_tables;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (__ldg(offsets + mid) <= g) lo = mid; else hi = mid;
        }
        const int32_t lt = __ldg(table_local + lo);
        ltid[i] = lt;
        lgid[i] = lt < 0 ? -1 : (int32_t)(g - __ldg(offsets + lo) + __ldg(local_offsets + lt));
    }
}

int recmg_shard_local_ids(const int32_t *gids, int64_t n, const int64_t *offsets,
                          int32_t n_tables, const int32_t *table_local,
                          const int64_t *local_offsets, int32_t *local_gids,
                          int32_t *local_tids, void *stream) {
    if (n < 0 || n_tables < 1) return RECMG_E_INVALID_CONFIG;
    if (n == 0) return RECMG_OK;
    shard_local_ids_kernel<<<(unsigned)imin64((n + 255) / 256, 16 * kSmCount), 256, 0,
                             as_stream(stream)>>>(gids, n, offsets, n_tables, table_local,
                                                  local_offsets, local_gids, local_tids);
    RECMG_LAUNCH_CHECK();
    return RECMG_OK;
}

}  // extern "C"
