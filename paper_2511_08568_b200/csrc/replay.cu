// K3 (priority-decay buffer replay) and K4 (LRU comparator) kernels plus the
// event builder and the prefetch-statistics kernel (R1).
//
// Semantics (reference citations relative to
// /root/reference/pkg/src/embcache/):
//   chunk k, origin o = k*l_in:  l_in x S(gid)   serve          runtime.py:254-264
//                                l_in x U(gid,b) keep-bit update runtime.py:126-130
//                                pf   x P(gid)   prefetch        runtime.py:131-137
//   then S(gid) for the tail accesses                            runtime.py:278-280
//   EVICT = victim argmin (priority, gid); every resident p>0 ages by one
//           (populate, runtime.py:100-112), applied per set.
//
// Sets of up to kSmemMaxWays (4096) ways: one warp per set, the set's ways
// and a gid -> way hash index in shared memory (replay_smem_kernel).  The warp
// consumes its event segment 64 events at a time: membership of every event,
// then every event before the first residency-changing miss is applied in
// bulk (hits never change residency, so this is exactly the sequential
// order), then that one miss is resolved.  Wider sets (the reference's fully
// associative buffer at a realistic capacity): one CTA per set, ways in
// global memory, an id -> slot map, the same batching by warp 0 and the
// victim scan by the whole CTA (replay_wide_kernel).
#include "replay.cuh"
#include "lstm_tc.cuh"
#include <cstdlib>

namespace recmg {

// ---------------------------------------------------------------------------
// event builder: one thread per event slot
//
// Collapsed serves: a serve S(g) whose previous same-set access in its chunk
// (or in the tail) is also g is a guaranteed hit on an untagged entry -- no
// event of its set lies between the two, so nothing can have evicted g, and
// the first one cleared any prefetch tag (runtime.py:93-98, 254-258).  Its
// only effect is cache_hits += 1 (and, for the LRU+prefetch policy, an LRU
// position that no other way of the set can pass in between), so it is
// counted here and emitted as an empty event.  Under Zipf skew with a sticky
// pool this removes most of the hottest set's events.
//
// set = gid % S with one multiply-high: q = umulhi(g, M), M = ceil(2^32 / S),
// is floor(g / S) or one more for every g < 2^30 (g*M/2^32 - g/S < 1/4), so
// r = g - q*S needs at most one correction (M = ceil(2^32/S) needs S >= 2).
__device__ __forceinline__ uint32_t set_of(uint32_t g, uint32_t S, uint32_t M) {
    if (S == 1) return 0;
    const uint32_t q = __umulhi(g, M);
    const int64_t r = (int64_t)g - (int64_t)q * S;
    return (uint32_t)(r < 0 ? r + S : r);
}

__global__ void build_events_kernel(const int32_t *__restrict__ gids, int64_t n, int32_t l_in,
                                    const uint8_t *__restrict__ bits,
                                    const int32_t *__restrict__ pf, int32_t pf_stride, int64_t K,
                                    int64_t k0, int64_t nk, int with_tail, uint32_t S,
                                    uint32_t M, int64_t i_begin,
                                    uint32_t *__restrict__ ev, uint32_t *__restrict__ vals,
                                    recmg_counters *__restrict__ ctr,
                                    uint8_t *__restrict__ access_class) {
    // events of chunks [k0, k0+nk) (+ the tail when with_tail, i.e. k0+nk == K);
    // local event i has global position k0*Ec + i; this launch builds events
    // [i_begin, E) (the thread-per-chunk kernel below builds the chunks' ones
    // when l_in <= 16, this one the tail)
    const int64_t Ec = 2 * (int64_t)l_in + pf_stride;
    const int64_t chunk_ev = nk * Ec;
    const int64_t E = chunk_ev + (with_tail ? (n - K * l_in) : 0);
    unsigned collapsed = 0;
    // serve of access a: collapsed iff its previous same-set access in
    // [block_start, a) exists and names the same id
    // (the latest earlier access of the same id first; sets -- one modulo
    // each -- only for the accesses between it and this one)
    auto dup_serve = [&](int64_t block_start, int64_t acc) {
        const uint32_t g = (uint32_t)gids[acc];
        int64_t q = acc - 1;
        while (q >= block_start && (uint32_t)gids[q] != g) q--;
        if (q < block_start) return false;
        const uint32_t set = set_of(g, S, M);
        for (int64_t p = q + 1; p < acc; p++)
            if (set_of((uint32_t)gids[p], S, M) == set) return false;
        return true;
    };
    // Across chunks (Zipf skew puts one id's accesses in nearly every chunk):
    // the serve at `acc`, the first access to its set in block [bs, ...), is
    // a guaranteed untagged hit when the previous chunk's last access to the
    // set names the same id and none of that chunk's prefetches into the set
    // names another id -- between the two, the set only sees that chunk's
    // updates (no residency change) and prefetches of the id itself (resident:
    // priority only, tag unchanged), runtime.py:83-137.
    auto cross_serve = [&](int64_t bs, int64_t acc) {
        const int64_t kp = bs / l_in - 1;        // the previous chunk
        if (kp < 0) return false;
        const uint32_t g = (uint32_t)gids[acc];
        const uint32_t set = set_of(g, S, M);
        for (int64_t p = bs; p < acc; p++)
            if (set_of((uint32_t)gids[p], S, M) == set) return false;
        int64_t q = bs - 1;
        while (q >= kp * l_in && set_of((uint32_t)gids[q], S, M) != set) q--;
        if (q < kp * l_in || (uint32_t)gids[q] != g) return false;
        if (pf) {
            const int32_t *row = pf + kp * pf_stride;
            for (int j = 0; j < pf_stride && row[j] >= 0; j++)
                if (set_of((uint32_t)row[j], S, M) == set && (uint32_t)row[j] != g) return false;
        }
        return true;
    };
    // The (last) keep-bit update of id g in chunk k is dead -- overwritten
    // before any eviction in its set reads priorities -- when the first event
    // of the set after it is a prefetch of g (priority = es if resident), or,
    // with no prefetch into the set, when chunk k+1 touches the set and only
    // with g: those serves are hits (no eviction) and chunk k+1's last update
    // of g overwrites the priority (runtime.py:100-112, 126-137).  If g is not
    // resident the update is a no-op either way.
    auto dead_update = [&](int64_t k, uint32_t g) {
        const uint32_t set = set_of(g, S, M);
        if (pf) {
            const int32_t *row = pf + k * pf_stride;
            for (int j = 0; j < pf_stride && row[j] >= 0; j++)
                if (set_of((uint32_t)row[j], S, M) == set) return (uint32_t)row[j] == g;
        }
        if (k + 1 >= K) return false;
        bool touched = false;
        for (int64_t p = (k + 1) * l_in; p < (k + 2) * l_in; p++) {
            const uint32_t x = (uint32_t)gids[p];
            if (set_of(x, S, M) != set) continue;
            if (x != g) return false;
            touched = true;
        }
        return touched;
    };
    for (int64_t i = i_begin + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t e;
        if (i < chunk_ev) {
            int64_t kk = i / Ec, r = i - kk * Ec;
            const int64_t k = k0 + kk;
            if (r < l_in) {
                const int64_t acc = k * l_in + r;
                if (dup_serve(k * l_in, acc) || cross_serve(k * l_in, acc)) {
                    e = ev_make(EV_SERVE, kGidMask);
                    collapsed++;
                    if (access_class) access_class[acc] = 0;
                } else {
                    e = ev_make(EV_SERVE, (uint32_t)gids[acc]);
                }
            } else if (r < 2 * l_in) {
                // keep-bit update; inside one chunk's update block nothing changes
                // residency, so only the LAST update of an id can matter
                // (runtime.py:126-130): earlier duplicates become empty events
                int64_t j = r - l_in;
                const int32_t gj = gids[k * l_in + j];
                bool later = false;
                for (int64_t q = j + 1; q < l_in; q++) later |= (gids[k * l_in + q] == gj);
                uint32_t b = bits ? (uint32_t)bits[k * l_in + j] : 0u;
                e = (later || dead_update(k, (uint32_t)gj))
                        ? ev_make(EV_UPD0, kGidMask)
                        : ev_make(b ? EV_UPD1 : EV_UPD0, (uint32_t)gj);
            } else {
                // -1 pads a row: that entry and everything after it is empty
                const int32_t *row = pf + k * pf_stride;
                const int64_t j = r - 2 * l_in;
                bool pad = false;
                for (int64_t q = 0; q <= j; q++) pad |= (row[q] < 0);
                e = ev_make(EV_PREFETCH, pad ? kGidMask : (uint32_t)row[j]);
            }
        } else {
            const int64_t acc = K * l_in + (i - chunk_ev);
            if (dup_serve(K * l_in, acc) || cross_serve(K * l_in, acc)) {
                e = ev_make(EV_SERVE, kGidMask);
                collapsed++;
                if (access_class) access_class[acc] = 0;
            } else {
                e = ev_make(EV_SERVE, (uint32_t)gids[acc]);
            }
        }
        ev[i] = e;
        if (vals) vals[i] = (uint32_t)(k0 * Ec + i);
    }
    collapsed = __reduce_add_sync(0xFFFFFFFFu, collapsed);
    if ((threadIdx.x & 31) == 0 && collapsed)
        atomicAdd((unsigned long long *)&ctr->cache_hits, (unsigned long long)collapsed);
}

// The same events, one thread per chunk (l_in <= LM): the chunk's ids and
// sets, and those of its neighbours, are held in registers, so the
// within-chunk / cross-chunk collapsing rules above cost register compares
// instead of per-event scans through global memory.
template <int LM>
__global__ void __launch_bounds__(128)
build_chunk_events_kernel(const int32_t *__restrict__ gids, int32_t l_in,
                          const uint8_t *__restrict__ bits, const int32_t *__restrict__ pf,
                          int32_t pf_stride, int64_t K, int64_t k0, int64_t nk, uint32_t S,
                          uint32_t M, uint32_t *__restrict__ ev, uint32_t *__restrict__ vals,
                          recmg_counters *__restrict__ ctr, uint8_t *__restrict__ access_class) {
    const int64_t Ec = 2 * (int64_t)l_in + pf_stride;
    unsigned collapsed = 0;
    for (int64_t kk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; kk < nk;
         kk += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = k0 + kk;
        uint32_t g[LM], st[LM], pg[LM], ps[LM], ng[LM], ns[LM];
#pragma unroll
        for (int r = 0; r < LM; r++) {
            st[r] = ps[r] = ns[r] = 0xFFFFFFFFu;   // no set
            g[r] = pg[r] = ng[r] = 0;
            if (r < l_in) {
                g[r] = (uint32_t)__ldg(gids + k * l_in + r);
                st[r] = set_of(g[r], S, M);
                if (k > 0) {
                    pg[r] = (uint32_t)__ldg(gids + (k - 1) * l_in + r);
                    ps[r] = set_of(pg[r], S, M);
                }
                if (k + 1 < K) {
                    ng[r] = (uint32_t)__ldg(gids + (k + 1) * l_in + r);
                    ns[r] = set_of(ng[r], S, M);
                }
            }
        }
        const int32_t *prow = (pf && k > 0) ? pf + (k - 1) * pf_stride : nullptr;
        const int32_t *crow = pf ? pf + k * pf_stride : nullptr;
        uint32_t *out = ev + kk * Ec;
        // serves (runtime.py:254-264) with the within- and cross-chunk hit rules
#pragma unroll
        for (int r = 0; r < LM; r++) {
            if (r >= l_in) continue;
            bool found = false, dup = false;
#pragma unroll
            for (int q = LM - 1; q >= 0; q--)
                if (q < r && !found && st[q] == st[r]) { found = true; dup = g[q] == g[r]; }
            bool coll = dup;
            if (!found && k > 0) {
                bool f2 = false;
                uint32_t last = 0;
#pragma unroll
                for (int q = LM - 1; q >= 0; q--)
                    if (!f2 && ps[q] == st[r]) { f2 = true; last = pg[q]; }
                coll = f2 && last == g[r];
                if (coll && prow)
                    for (int j = 0; j < pf_stride && prow[j] >= 0; j++)
                        if (set_of((uint32_t)prow[j], S, M) == st[r] && (uint32_t)prow[j] != g[r]) {
                            coll = false;
                            break;
                        }
            }
            if (coll) {
                collapsed++;
                if (access_class) access_class[k * l_in + r] = 0;
            }
            out[r] = ev_make(EV_SERVE, coll ? kGidMask : g[r]);
        }
        // keep-bit updates (runtime.py:126-130): the last of an id in the
        // chunk, unless dead (overwritten before any eviction in its set)
#pragma unroll
        for (int j = 0; j < LM; j++) {
            if (j >= l_in) continue;
            bool later = false;
#pragma unroll
            for (int q = 0; q < LM; q++) later |= (q > j && q < l_in && g[q] == g[j]);
            bool dead = later;
            if (!dead) {
                bool decided = false;
                if (crow)
                    for (int q = 0; q < pf_stride && crow[q] >= 0; q++)
                        if (set_of((uint32_t)crow[q], S, M) == st[j]) {
                            decided = true;
                            dead = (uint32_t)crow[q] == g[j];
                            break;
                        }
                if (!decided && k + 1 < K) {
                    bool touched = false, only = true;
#pragma unroll
                    for (int q = 0; q < LM; q++)
                        if (ns[q] == st[j]) { touched = true; only = only && ng[q] == g[j]; }
                    dead = touched && only;
                }
            }
            const uint32_t b = bits ? (uint32_t)bits[k * l_in + j] : 0u;
            out[l_in + j] = dead ? ev_make(EV_UPD0, kGidMask) : ev_make(b ? EV_UPD1 : EV_UPD0, g[j]);
        }
        // prefetches (runtime.py:131-137); -1 ends a row
        bool pad = false;
        for (int j = 0; j < pf_stride; j++) {
            const int32_t x = crow[j];
            pad |= x < 0;
            out[2 * l_in + j] = ev_make(EV_PREFETCH, pad ? kGidMask : (uint32_t)x);
        }
        if (vals)
            for (int64_t i = 0; i < Ec; i++) vals[kk * Ec + i] = (uint32_t)(k * Ec + i);
    }
    collapsed = __reduce_add_sync(0xFFFFFFFFu, collapsed);
    if ((threadIdx.x & 31) == 0 && collapsed)
        atomicAdd((unsigned long long *)&ctr->cache_hits, (unsigned long long)collapsed);
}

template __global__ void build_chunk_events_kernel<16>(const int32_t *, int32_t, const uint8_t *,
                                                       const int32_t *, int32_t, int64_t, int64_t,
                                                       int64_t, uint32_t, uint32_t, uint32_t *,
                                                       uint32_t *, recmg_counters *, uint8_t *);

// event position -> access index (only meaningful for serve events)
__device__ __forceinline__ int64_t access_of_event(int64_t pos, int64_t Ec, int64_t K,
                                                   int32_t l_in) {
    int64_t chunk_ev = K * Ec;
    if (pos < chunk_ev) {
        int64_t k = pos / Ec;
        return k * l_in + (pos - k * Ec);
    }
    return K * l_in + (pos - chunk_ev);
}

// ---------------------------------------------------------------------------
// prefetch statistics, one thread per chunk  (runtime.py:272-276)
__global__ void prefetch_stats_kernel(const int32_t *__restrict__ gids, int64_t k0, int64_t nk,
                                      int32_t l_in, int32_t l_win, const int32_t *__restrict__ pf,
                                      int32_t pf_stride, uint16_t *__restrict__ cov_num,
                                      uint16_t *__restrict__ cov_den,
                                      recmg_counters *__restrict__ ctr) {
    const int64_t k = k0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t K = k0 + nk;
    int64_t issued = 0, useful = 0;
    if (k < K) {
        const int32_t *w = gids + k * l_in + l_in;
        int den = 0;
        for (int i = 0; i < l_win; i++) {
            int32_t g = w[i];
            bool dup = false;
            for (int j = 0; j < i; j++) dup |= (w[j] == g);
            den += !dup;
        }
        int num = 0;
        if (pf) {
            const int32_t *p = pf + k * pf_stride;
            for (int j = 0; j < pf_stride; j++) {
                int32_t g = p[j];
                if (g < 0) break;
                issued++;
                bool in = false;
                for (int i = 0; i < l_win; i++) in |= (w[i] == g);
                useful += in;
                bool dup = false;
                for (int q = 0; q < j; q++) dup |= (p[q] == g);
                num += (in && !dup);
            }
        }
        if (cov_num) cov_num[k] = (uint16_t)num;
        if (cov_den) cov_den[k] = (uint16_t)den;
    }
    issued = __reduce_add_sync(0xFFFFFFFFu, (unsigned)issued);
    useful = __reduce_add_sync(0xFFFFFFFFu, (unsigned)useful);
    if ((threadIdx.x & 31) == 0 && (issued | useful)) {
        atomicAdd((unsigned long long *)&ctr->prefetch_issued, (unsigned long long)issued);
        atomicAdd((unsigned long long *)&ctr->prefetch_useful, (unsigned long long)useful);
    }
}

// ---------------------------------------------------------------------------
// ReplayArgs is declared in replay.cuh

__device__ __forceinline__ void seg_range(const ReplayArgs &a, int64_t set, int64_t &lo,
                                          int64_t &hi) {
    if (a.seg_start) {
        lo = a.seg_start[set];
        hi = a.seg_end[set];
    } else {
        lo = 0;
        hi = a.E;
    }
}

__device__ __forceinline__ void write_class(const ReplayArgs &a, int64_t pos, uint8_t c) {
    int64_t orig = a.vals ? (int64_t)a.vals[pos] : a.ev_base + pos;
    a.access_class[access_of_event(orig, a.Ec, a.K, a.l_in)] = c;
}

// LRU counts: hits and misses; in serve_only mode (the comparator fused into
// the priority replay's launch, on its events) the caller pre-added the
// call's accesses to the hits and each miss moves one over, because the
// event builder drops serves that are guaranteed hits (collapsed repeats)
__device__ __forceinline__ void flush_lru(const ReplayArgs &a, unsigned long long hits,
                                          unsigned long long misses) {
    if (!a.hits_misses) return;
    if (a.serve_only) {
        if (misses) {
            atomicAdd((unsigned long long *)&a.hits_misses[0], (unsigned long long)(-(long long)misses));
            atomicAdd((unsigned long long *)&a.hits_misses[1], misses);
        }
        return;
    }
    if (hits) atomicAdd((unsigned long long *)&a.hits_misses[0], hits);
    if (misses) atomicAdd((unsigned long long *)&a.hits_misses[1], misses);
}

// the event as the LRU comparator sees it: in serve_only mode every
// non-serve event is no event
template <int POLICY>
__device__ __forceinline__ uint32_t lru_view(const ReplayArgs &a, uint32_t e) {
    if (POLICY != RECMG_POLICY_LRU) return e;
    return (a.serve_only && ev_type(e) != EV_SERVE) ? kGidMask : e;
}

__device__ __forceinline__ void flush_counters(recmg_counters *ctr, unsigned long long ch,
                                               unsigned long long ph, unsigned long long od,
                                               unsigned long long ev, unsigned long long ins,
                                               unsigned long long occ) {
    if (ch) atomicAdd((unsigned long long *)&ctr->cache_hits, ch);
    if (ph) atomicAdd((unsigned long long *)&ctr->prefetch_hits, ph);
    if (od) atomicAdd((unsigned long long *)&ctr->on_demand, od);
    if (ev) atomicAdd((unsigned long long *)&ctr->evictions, ev);
    if (ins) atomicAdd((unsigned long long *)&ctr->prefetch_inserts, ins);
    if (occ) atomicAdd((unsigned long long *)&ctr->occupancy, occ);
}

// ---------------------------------------------------------------------------
// Per-warp shared-memory ring over one set's event segment, filled with
// cp.async: 4 slots x 256 events, up to 4 blocks in flight, so the serial
// consumer reads every window from shared memory instead of paying an L2/DRAM
// round trip per 32-event batch (the replay of the hottest set is a single
// dependency chain).
constexpr int kRingBlk = 256;
#ifndef RECMG_RING_SLOTS
#define RECMG_RING_SLOTS 4
#endif
constexpr int kRingSlots = RECMG_RING_SLOTS;       // power of two
constexpr int kRingMask = kRingBlk * kRingSlots - 1;
constexpr int kL2Ahead = 32;   // blocks prefetched into L2 beyond the ring (long segments)

struct EventRing {
    uint32_t *buf;       // [kRingSlots * kRingBlk] shared, 16 B aligned
    const uint32_t *src; // segment base rounded down to 16 B
    int64_t n;           // words from src to the segment end
    int64_t nblk, issued;
    int shift;           // words between src and the segment start
    int lane;

    // block k = words [k*256, k*256+256) from src into slot k % kRingSlots:
    // full blocks as 16 B cp.async (2 per lane), the last one word by word
    __device__ __forceinline__ void issue_next() {
        const int64_t k = issued;
        const uint32_t *s = src + k * kRingBlk;
        uint32_t *d = buf + (k & (kRingSlots - 1)) * kRingBlk;
        const int64_t cnt = n - k * kRingBlk;
        // the hottest set's segment is one long serial stream: keep L2 ahead of
        // the ring so every ring block is an L2 hit (one 128 B line per lane)
        if (k + kL2Ahead < nblk && lane < kRingBlk * 4 / 128)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(s + kL2Ahead * kRingBlk + lane * 32));
        if (cnt >= kRingBlk) {
#pragma unroll
            for (int t = 0; t < 2; t++) {
                const int c = (lane + 32 * t) * 4;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                                 (uint32_t)__cvta_generic_to_shared(d + c)),
                             "l"(s + c) : "memory");
            }
        } else {
            for (int i = lane; i < cnt; i += 32) {
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                                 (uint32_t)__cvta_generic_to_shared(d + i)),
                             "l"(s + i) : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        issued++;
    }
    __device__ __forceinline__ void init(uint32_t *b, const uint32_t *e, int64_t len, int l) {
        shift = (int)((reinterpret_cast<uintptr_t>(e) >> 2) & 3);
        buf = b; src = e - shift; n = len + shift; lane = l; issued = 0;
        nblk = len > 0 ? (n + kRingBlk - 1) / kRingBlk : 0;
        while (issued < nblk && issued < kRingSlots) issue_next();
    }
    // make segment events [r, r + cnt) readable; refill freed slots
    __device__ __forceinline__ void ensure(int64_t r, int cnt) {
        const int64_t k0 = (r + shift) / kRingBlk;
        while (issued < nblk && issued < k0 + kRingSlots) issue_next();
        const int64_t k1 = (r + shift + cnt - 1) / kRingBlk;
        const int64_t pending = issued - 1 - k1;   // groups allowed to stay in flight
        if (pending <= 0) asm volatile("cp.async.wait_group 0;" ::: "memory");
        else if (pending == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
        else if (pending == 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
        else if (pending == 3) asm volatile("cp.async.wait_group 3;" ::: "memory");
        else if (pending == 4) asm volatile("cp.async.wait_group 4;" ::: "memory");
        else if (pending == 5) asm volatile("cp.async.wait_group 5;" ::: "memory");
        else asm volatile("cp.async.wait_group 6;" ::: "memory");
        __syncwarp();
    }
    __device__ __forceinline__ uint32_t at(int64_t r) const {
        return buf[(uint32_t)(r + shift) & kRingMask];
    }
};

// ---------------------------------------------------------------------------
// Sets of up to kSmemMaxWays ways: one warp per set, the set's ways and an
// open-addressing gid -> way hash index live in shared memory.  Per batch of
// 32 events: one hash probe per lane (membership), one ballot for the first
// residency-changing miss, __match_any_sync groups the hit-run by way and the
// group leader applies the run's effect on its way (S: tag clear / hit
// class, U/P: last write wins), then the miss is resolved serially.
// LFU way metadata: the reference count (saturating at 2^27 - 1 -- only a
// block hit that often in ONE residency could tie wrongly) above the clock of
// the last use (36 bits, 6.9e10 events); victim = min (count, clock), i.e.
// least recently used among the least frequently used (cache_sim.py:109-137).
constexpr int kLfuShift = 36;
constexpr int64_t kLfuCountMax = (int64_t(1) << 27) - 1;
__device__ __forceinline__ int64_t lfu_meta(int64_t m, int64_t add, int64_t clk) {
    int64_t c = (m >> kLfuShift) + add;
    c = c > kLfuCountMax ? kLfuCountMax : c;
    return (c << kLfuShift) | (clk & ((int64_t(1) << kLfuShift) - 1));
}

constexpr uint64_t kHtEmpty = ~0ull;

struct SetView {
    uint32_t *ring;
    int32_t *tags;
    int64_t *meta;
    uint64_t *ht;
    uint32_t hmask;
    int hbits;
};

__device__ __forceinline__ uint32_t ht_home(uint32_t g, int bits) {
    return (g * 0x9E3779B1u) >> (32 - bits);
}

__device__ __forceinline__ int ht_find(const SetView &v, uint32_t g) {
    uint32_t p = ht_home(g, v.hbits);
    while (true) {
        const uint64_t x = v.ht[p];
        if (x == kHtEmpty) return -1;
        if ((uint32_t)(x >> 32) == g) return (int)(uint32_t)x;
        p = (p + 1) & v.hmask;
    }
}

__device__ __forceinline__ void ht_insert(const SetView &v, uint32_t g, uint32_t way) {
    uint32_t p = ht_home(g, v.hbits);
    while (v.ht[p] != kHtEmpty) p = (p + 1) & v.hmask;
    v.ht[p] = ((uint64_t)g << 32) | way;
}

// linear-probing delete with backward shift (no tombstones)
__device__ __forceinline__ void ht_erase(const SetView &v, uint32_t g) {
    uint32_t i = ht_home(g, v.hbits);
    while ((uint32_t)(v.ht[i] >> 32) != g) i = (i + 1) & v.hmask;
    uint32_t j = i;
    while (true) {
        j = (j + 1) & v.hmask;
        const uint64_t x = v.ht[j];
        if (x == kHtEmpty) break;
        const uint32_t k = ht_home((uint32_t)(x >> 32), v.hbits);
        const bool stay = (i <= j) ? (i < k && k <= j) : (i < k || k <= j);
        if (!stay) {
            v.ht[i] = x;
            i = j;
        }
    }
    v.ht[i] = kHtEmpty;
}

// ---------------------------------------------------------------------------
// Register-resident replay of one set of W <= 32 ways (PRIORITY and LRU, the
// two policies of the hot path): lane w IS way w -- its gid, its priority
// (lazy decay, see replay_smem_kernel) and prefetch tag, or its LRU clock
// live in registers, so membership needs no hash index and a miss no
// shared-memory bookkeeping.  Per batch of 32 events (lane j holds event j):
//   membership   32 x (SHFL of event j's gid, compare with my tag, set bit j):
//                `mine` = the batch's events that name my way; hit = OR of
//                every way's `mine` (one REDUX.OR)
//   hit run      the events before the first residency-changing miss, applied
//                per way from `mine` (first S takes the tag, last U/P sets the
//                priority; LRU: clock of the last hit), which equals the
//                sequential order because hits never change residency
//   miss         victim = argmin (priority, gid) [LRU: min clock] as two
//                REDUX.MIN over the lanes, the victim lane takes the new gid,
//                its `mine` becomes the remaining events naming that gid
// The result (counters, per-access class, per-access hit, the state written
// back) is identical to replay_smem_kernel's.  Used for every set that is
// not on the heavy list: sets whose events are mostly misses and short hit
// runs, where the shared-memory kernel's hash probing, run grouping
// (MATCH.ANY) and per-miss hash updates cost ~150 warp instructions per event.
template <int POLICY, bool CLASS>
__device__ __forceinline__ unsigned long long replay_set_regs(const ReplayArgs &a, int64_t set, int64_t lo,
                                                int64_t hi, EventRing &ring, int lane) {
    constexpr bool PRIO = (POLICY == RECMG_POLICY_PRIORITY);
    const unsigned FULL = 0xFFFFFFFFu;
    const int W = (int)a.W;
    const int64_t sbase = set * a.W;
    const bool is_way = lane < W;
    int32_t tag = is_way ? a.st.tags[sbase + lane] : -2;   // -2: no such way
    const int64_t m0 = is_way ? a.st.meta[sbase + lane] : 0;
    // PRIORITY: pr = stored priority (+ decay), mhi = the meta's high word
    // (bit 0 = prefetch tag); LRU: clk = clock of the last use
    int32_t pr = (int32_t)(m0 & 0xFFFFFFFF);
    uint32_t mhi = (uint32_t)((uint64_t)m0 >> 32);
    int64_t clk = m0;
    int count = __popc(__ballot_sync(FULL, tag >= 0));
    const int64_t clock_base = a.st.header[0];
    int32_t decay = 0;
    unsigned long long ch = 0, ph = 0, od = 0, nev = 0, ins = 0, lhits = 0;
    // one 32-bit victim key (a single REDUX.MIN) when it orders the ways
    // exactly: PRIORITY (priority << gid_bits) | gid while every priority fits
    // (events only ever set es or es + 1; the decay only lowers them); LRU the
    // clock relative to clock_base - 2^31 while every clock of the launch fits
    const int gb = a.gid_bits;
    const int64_t kbase = clock_base - 0x80000000ll;
    bool key32;
    if (PRIO) {
        const int32_t lim = gb > 0 && gb <= 28 ? (1 << (32 - gb)) - 1 : 0;
        key32 = a.es + 1 < lim && __all_sync(FULL, tag < 0 || pr < lim);
    } else {
        key32 = hi - lo < 0x7FFFFFFFll && clock_base + hi - kbase < 0xFFFFFFFFll &&
                __all_sync(FULL, tag < 0 || clk >= kbase);
    }

    // Wide step: 128 events (4 per lane) at once while the previous steps saw
    // no residency-changing miss -- the long sets (Zipf's hot ids: one set can
    // carry 3% of the events with a miss per ~800) are hit runs, so their cost
    // is the per-step overhead, which this spreads over 4x the events.  A
    // window with a miss falls back to the 32-event step below.
    constexpr int kWide = 4;
    bool try_wide = true;
    for (int64_t pos = lo; pos < hi;) {
        if (try_wide && hi - pos >= 32 * kWide) {
            ring.ensure(pos - lo, 32 * kWide);
            uint32_t gq[kWide];
            unsigned mq[kWide], Sq[kWide], UPq[kWide], U1q[kWide];
            unsigned missing = 0;
#pragma unroll
            for (int q = 0; q < kWide; q++) {
                const uint32_t e = lru_view<POLICY>(a, ring.at(pos - lo + 32 * q + lane));
                gq[q] = ev_gid(e);
                const uint32_t ty = ev_type(e);
                const bool real = gq[q] != kGidMask;
                Sq[q] = __ballot_sync(FULL, real && ty == EV_SERVE);
                if (PRIO) {
                    UPq[q] = __ballot_sync(FULL, real && ty != EV_SERVE);
                    U1q[q] = __ballot_sync(FULL, real && ty == EV_UPD1);
                }
                unsigned m = 0;
#pragma unroll
                for (int j = 0; j < 32; j++) {
                    const uint32_t gj = __shfl_sync(FULL, gq[q], j);
                    if ((uint32_t)tag == gj) m |= 1u << j;
                }
                mq[q] = m;
                const unsigned cand = PRIO ? (Sq[q] | __ballot_sync(FULL, real && ty == EV_PREFETCH))
                                           : __ballot_sync(FULL, real);
                missing |= cand & ~__reduce_or_sync(FULL, m);
            }
            if (missing == 0) {
                // the whole window is one hit run: per way, the S count (the
                // first S takes the prefetch tag) and the last U/P write
                if (PRIO) {
                    unsigned nS = 0;
                    int fS = -1, lU = -1;
#pragma unroll
                    for (int q = 0; q < kWide; q++) {
                        const unsigned sp = mq[q] & Sq[q], up = mq[q] & UPq[q];
                        nS += __popc(sp);
                        if (fS < 0 && sp) fS = 32 * q + __ffs(sp) - 1;
                        if (up) lU = 32 * q + 31 - __clz(up);
                    }
                    const bool tagged = (mhi & 1u) && nS;
                    if (nS) {
                        if (mhi & 1u) { ph += 1; ch += nS - 1; mhi &= ~1u; }
                        else ch += nS;
                    }
                    if (lU >= 0) {
                        unsigned u1 = U1q[0];
#pragma unroll
                        for (int q = 1; q < kWide; q++) u1 = (lU >> 5) == q ? U1q[q] : u1;
                        pr = a.es + (int32_t)((u1 >> (lU & 31)) & 1u) + decay;
                    }
                    if (CLASS) {
#pragma unroll
                        for (int q = 0; q < kWide; q++) {
                            const unsigned pf = __reduce_or_sync(
                                FULL, (tagged && (fS >> 5) == q) ? 1u << (fS & 31) : 0u);
                            if ((Sq[q] >> lane) & 1u)
                                write_class(a, pos + 32 * q + lane, ((pf >> lane) & 1u) ? 1 : 0);
                        }
                    }
                } else {
                    int last = -1;
#pragma unroll
                    for (int q = 0; q < kWide; q++) {
                        lhits += __popc(mq[q]);
                        if (mq[q]) last = 32 * q + 31 - __clz(mq[q]);
                    }
                    if (last >= 0) clk = clock_base + pos + last;
                }
                pos += 32 * kWide;
                continue;
            }
            try_wide = false;
        }
        const int nb = (int)imin64(32, hi - pos);
        ring.ensure(pos - lo, nb);
        const uint32_t e = lane < nb ? lru_view<POLICY>(a, ring.at(pos - lo + lane)) : kGidMask;
        const uint32_t g = ev_gid(e), ty = ev_type(e);
        const bool real = g != kGidMask;
        unsigned mine = 0;
#pragma unroll
        for (int j = 0; j < 32; j++) {
            const uint32_t gj = __shfl_sync(FULL, g, j);
            if ((uint32_t)tag == gj) mine |= 1u << j;
        }
        unsigned hit = __reduce_or_sync(FULL, mine);
        const unsigned Sm = __ballot_sync(FULL, real && ty == EV_SERVE);
        unsigned cand, UPm = 0, U1m = 0;
        if (PRIO) {
            UPm = __ballot_sync(FULL, real && ty != EV_SERVE);
            U1m = __ballot_sync(FULL, real && ty == EV_UPD1);
            cand = Sm | __ballot_sync(FULL, real && ty == EV_PREFETCH);
        } else {
            cand = __ballot_sync(FULL, real);   // simulate(): every event is a serve
        }
        int start = 0;
        for (;;) {
            const unsigned from = ~0u << start;
            const unsigned miss = cand & ~hit & from;
            const int cut = miss ? __ffs(miss) - 1 : nb;
            const unsigned R = (cut >= 32 ? ~0u : ((1u << cut) - 1u)) & from;
            const unsigned rk = mine & R;
            if (PRIO) {
                const unsigned sp = rk & Sm, up = rk & UPm;
                unsigned pfirst = 0;
                if (sp) {
                    const unsigned c = __popc(sp);
                    if (mhi & 1u) { ph += 1; ch += c - 1; mhi &= ~1u; pfirst = sp & (0u - sp); }
                    else ch += c;
                }
                if (up) {
                    const int last = 31 - __clz(up);
                    pr = a.es + (int32_t)((U1m >> last) & 1u) + decay;
                }
                if (CLASS) {
                    const unsigned pf = __reduce_or_sync(FULL, pfirst);
                    if ((R & Sm) >> lane & 1u) write_class(a, pos + lane, (pf >> lane & 1u) ? 1 : 0);
                }
            } else if (rk) {
                lhits += __popc(rk);
                clk = clock_base + pos + (31 - __clz(rk));
            }
            if (cut >= nb) break;
            // the miss at `cut`
            const uint32_t gc = __shfl_sync(FULL, g, cut);
            const bool isS = (Sm >> cut) & 1u;
            if (PRIO) {
                if (isS) {
                    od++;
                    if (CLASS && lane == 0) write_class(a, pos + cut, 2);
                } else {
                    ins++;
                }
            } else {
                od++;
                if (a.per_access_hit && lane == 0)
                    a.per_access_hit[a.vals ? a.vals[pos + cut] : pos + cut] = 0;
            }
            int target;
            if (count >= W && key32) {
                unsigned key;
                if (PRIO) {
                    const int32_t pe = pr - decay;
                    key = tag >= 0 ? ((unsigned)(pe > 0 ? pe : 0) << gb) | (unsigned)tag : ~0u;
                } else {
                    key = tag >= 0 ? (unsigned)(clk - kbase) : ~0u;
                }
                const unsigned kmin = __reduce_min_sync(FULL, key);
                target = __ffs(__ballot_sync(FULL, key == kmin)) - 1;
                if (PRIO) decay++;
                nev++;
                count--;
            } else if (count >= W) {
                // populate(): victim = argmin (priority, gid)  [LRU: min clock]
                unsigned khi, klo;
                if (PRIO) {
                    const int32_t pe = pr - decay;
                    khi = tag >= 0 ? (unsigned)(pe > 0 ? pe : 0) : ~0u;
                    klo = (unsigned)tag;
                } else {
                    khi = tag >= 0 ? (unsigned)((uint64_t)clk >> 32) : ~0u;
                    klo = (unsigned)clk;
                }
                const unsigned hmin = __reduce_min_sync(FULL, khi);
                const unsigned lmin = __reduce_min_sync(FULL, khi == hmin ? klo : ~0u);
                target = __ffs(__ballot_sync(FULL, khi == hmin && klo == lmin)) - 1;
                if (PRIO) decay++;
                nev++;
                count--;
            } else {
                // the first free way (the shared-memory kernel's choice)
                target = __ffs(__ballot_sync(FULL, tag == -1)) - 1;
            }
            const unsigned named = __ballot_sync(FULL, g == gc);
            if (lane == target) {
                tag = (int32_t)gc;
                if (PRIO) {
                    pr = a.es + decay;
                    mhi = isS ? 0u : 1u;
                } else {
                    clk = clock_base + pos + cut;
                }
                mine = named;   // the evicted gid's events now miss
            }
            count++;
            hit = __reduce_or_sync(FULL, mine);
            start = cut + 1;
            if (start >= nb) break;
        }
        try_wide = start == 0;   // this step had no miss: try the wide step again
        pos += nb;
    }

    if (is_way) {
        a.st.tags[sbase + lane] = tag;
        int64_t m;
        if (PRIO) {
            const int32_t pe = pr - decay;
            m = (int64_t)((uint64_t)mhi << 32) | (int64_t)(uint32_t)(pe > 0 ? pe : 0);
        } else {
            m = clk;
        }
        a.st.meta[sbase + lane] = m;
    }
    if (lane == 0) a.st.count[set] = count;
    if (PRIO) {
        ch = __reduce_add_sync(FULL, (unsigned)ch);
        ph = __reduce_add_sync(FULL, (unsigned)ph);
        if (lane == 0) flush_counters(a.ctr, ch, ph, od, nev, ins, (unsigned long long)count);
    } else {
        lhits = __reduce_add_sync(FULL, (unsigned)lhits);
        if (lane == 0) flush_lru(a, lhits, od);
    }
    return od + ins;
}

// ---------------------------------------------------------------------------
// Long sets (>= kTableMinEvents events; the hot sets of a Zipf trace are hit
// runs with one residency-changing miss per ~800 events): the same register
// ways, but membership from a direct-mapped way map in shared memory --
// every gid of set s is q * S + s, so wmap[q] (q = gid / S, one byte per id
// of the set: ceil(total_ids / S) bytes) holds its way or 0xFF -- one LDS per
// event instead of a 32-step shuffle scan; the hit run is applied per
// distinct way (a ballot per way the run touches: a handful), 128 events per
// step while the steps see no miss.
constexpr int64_t kTableMinEvents = 8192;
constexpr int kTableMaxBytes = 4096;

__device__ __forceinline__ uint32_t div_set(uint32_t g, uint32_t S, uint32_t M) {
    uint32_t q = __umulhi(g, M);   // M = ceil(2^32 / S): q is floor(g / S) or one more
    return q * S > g ? q - 1 : q;
}

template <int POLICY, bool CLASS>
__device__ __forceinline__ unsigned long long replay_set_table(const ReplayArgs &a, int64_t set,
                                                               int64_t lo, int64_t hi,
                                                               uint8_t *wmap, int lane) {
    constexpr bool PRIO = (POLICY == RECMG_POLICY_PRIORITY);
    constexpr int kNone = 0xFF;
    const unsigned FULL = 0xFFFFFFFFu;
    const int W = (int)a.W;
    const uint32_t S = (uint32_t)a.S, M = a.smagic;
    const int64_t sbase = set * a.W;
    const bool is_way = lane < W;
    int32_t tag = is_way ? a.st.tags[sbase + lane] : -2;
    const int64_t m0 = is_way ? a.st.meta[sbase + lane] : 0;
    int32_t pr = (int32_t)(m0 & 0xFFFFFFFF);
    uint32_t mhi = (uint32_t)((uint64_t)m0 >> 32);
    int64_t clk = m0;
    int count = __popc(__ballot_sync(FULL, tag >= 0));
    const int64_t clock_base = a.st.header[0];
    int32_t decay = 0;
    unsigned long long ch = 0, ph = 0, od = 0, nev = 0, ins = 0, lhits = 0;
    const int gb = a.gid_bits;
    const int64_t kbase = clock_base - 0x80000000ll;
    bool key32;
    if (PRIO) {
        const int32_t lim = gb > 0 && gb <= 28 ? (1 << (32 - gb)) - 1 : 0;
        key32 = a.es + 1 < lim && __all_sync(FULL, tag < 0 || pr < lim);
    } else {
        key32 = hi - lo < 0x7FFFFFFFll && clock_base + hi - kbase < 0xFFFFFFFFll &&
                __all_sync(FULL, tag < 0 || clk >= kbase);
    }
    for (int i = lane * 16; i < a.qn; i += 32 * 16)
        *reinterpret_cast<uint4 *>(wmap + i) = make_uint4(~0u, ~0u, ~0u, ~0u);
    __syncwarp();
    if (tag >= 0) wmap[div_set((uint32_t)tag, S, M)] = (uint8_t)lane;
    __syncwarp();

    // applies one way's share of a hit run (the events in m) -- called by the
    // way's lane; returns the event (bit) whose S took the prefetch tag
    auto apply_way = [&](unsigned m, unsigned Sm, unsigned UPm, unsigned U1m, int64_t base)
        -> unsigned {
        unsigned took = 0;
        if (PRIO) {
            const unsigned sp = m & Sm, up = m & UPm;
            if (sp) {
                const unsigned c = __popc(sp);
                if (mhi & 1u) { ph += 1; ch += c - 1; mhi &= ~1u; took = sp & (0u - sp); }
                else ch += c;
            }
            if (up) {
                const int last = 31 - __clz(up);
                pr = a.es + (int32_t)((U1m >> last) & 1u) + decay;
            }
        } else if (m) {
            lhits += __popc(m);
            clk = clock_base + base + (31 - __clz(m));
        }
        return took;
    };

    // 128-event windows, 4 events per lane in registers (lane j of part q holds
    // event 32 q + j), loaded one window ahead straight from the partitioned
    // segment (coalesced; L2 prefetch 8 windows ahead); past the segment end
    // the slots hold kGidMask, an event that is no event
#ifndef RECMG_TABLE_WIDE
#define RECMG_TABLE_WIDE 4
#endif
    constexpr int kWide = RECMG_TABLE_WIDE, kWin = 32 * kWide;
    const uint32_t *seg = a.ev + lo;
    const int64_t len = hi - lo;
    uint32_t nxt[kWide];
#pragma unroll
    for (int q = 0; q < kWide; q++) {
        const int64_t i = 32 * q + lane;
        nxt[q] = i < len ? __ldcs(seg + i) : kGidMask;
    }
    for (int64_t wp = 0; wp < len; wp += kWin) {
        uint32_t cur[kWide];
#pragma unroll
        for (int q = 0; q < kWide; q++) {
            cur[q] = lru_view<POLICY>(a, nxt[q]);   // (not at the load: it would wait)
            const int64_t i = wp + kWin + 32 * q + lane;
            nxt[q] = i < len ? __ldcs(seg + i) : kGidMask;
        }
        if (lane < 4 && wp + 8 * kWin + 32 * lane < len)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(seg + wp + 8 * kWin + 32 * lane));
        const int64_t pos = lo + wp;
        int wq[kWide];
        unsigned Sq[kWide], UPq[kWide], U1q[kWide], Hq[kWide], Cq[kWide];
#pragma unroll
        for (int q = 0; q < kWide; q++) {
            const uint32_t g = ev_gid(cur[q]), ty = ev_type(cur[q]);
            const bool real = g != kGidMask;
            wq[q] = real ? wmap[div_set(g, S, M)] : kNone;
            Sq[q] = __ballot_sync(FULL, real && ty == EV_SERVE);
            if (PRIO) {
                UPq[q] = __ballot_sync(FULL, real && ty != EV_SERVE);
                U1q[q] = __ballot_sync(FULL, real && ty == EV_UPD1);
            }
            Hq[q] = __ballot_sync(FULL, wq[q] != kNone);
            Cq[q] = PRIO ? (Sq[q] | __ballot_sync(FULL, real && ty == EV_PREFETCH))
                         : __ballot_sync(FULL, real);
        }
        // The window as hit runs and misses: the run before the first miss is
        // applied per distinct way it touches (a ballot per way: a handful;
        // the first S takes the tag, the last U/P writes the priority [LRU: the
        // last hit sets the clock]), the miss is resolved, the window's way
        // numbers are patched for the two gids it changed, and the next run
        // starts after it.  A window without a miss is one run.
        uint32_t gw[kWide];
#pragma unroll
        for (int q = 0; q < kWide; q++) gw[q] = ev_gid(cur[q]);
        int start = 0;
        for (;;) {
            unsigned Rq[kWide], mq[kWide];
            int m = kWin;
#pragma unroll
            for (int q = kWide - 1; q >= 0; q--) {
                const int lo32 = start - 32 * q;
                const unsigned from = lo32 <= 0 ? ~0u : (lo32 >= 32 ? 0u : ~0u << lo32);
                mq[q] = Cq[q] & ~Hq[q] & from;
                if (mq[q]) m = 32 * q + __ffs(mq[q]) - 1;
                Rq[q] = from;
            }
#pragma unroll
            for (int q = 0; q < kWide; q++) {
                const int hi32 = m - 32 * q;
                Rq[q] &= hi32 >= 32 ? ~0u : (hi32 <= 0 ? 0u : (1u << hi32) - 1u);
            }
            // each way's events of the run: one ballot per part for every way
            // the window names -- independent ballots, no per-way round trip
            unsigned mine[kWide], took[kWide];
            unsigned named_l = 0;
#pragma unroll
            for (int q = 0; q < kWide; q++) {
                mine[q] = 0;
                took[q] = 0;
                if (wq[q] != kNone) named_l |= 1u << wq[q];
            }
            for (unsigned named = __reduce_or_sync(FULL, named_l); named; named &= named - 1) {
                const int wv = __ffs(named) - 1;
#pragma unroll
                for (int q = 0; q < kWide; q++) {
                    const unsigned b = __ballot_sync(FULL, wq[q] == wv);
                    if (lane == wv) mine[q] = b & Rq[q];
                }
            }
            unsigned any_mine = 0;
#pragma unroll
            for (int q = 0; q < kWide; q++) any_mine |= mine[q];
            if (any_mine) {
                if (PRIO) {
                    unsigned nS = 0, u1 = 0;
                    int fS = -1, lU = -1;
#pragma unroll
                    for (int q = 0; q < kWide; q++) {
                        const unsigned sp = mine[q] & Sq[q], up = mine[q] & UPq[q];
                        nS += __popc(sp);
                        if (fS < 0 && sp) fS = 32 * q + __ffs(sp) - 1;
                        if (up) { lU = 32 * q + 31 - __clz(up); u1 = U1q[q]; }
                    }
                    if (nS) {
                        if (mhi & 1u) {
                            ph += 1; ch += nS - 1; mhi &= ~1u;
#pragma unroll
                            for (int q = 0; q < kWide; q++)
                                if ((fS >> 5) == q) took[q] = 1u << (fS & 31);
                        } else {
                            ch += nS;
                        }
                    }
                    if (lU >= 0) pr = a.es + (int32_t)((u1 >> (lU & 31)) & 1u) + decay;
                } else {
                    int last = -1;
#pragma unroll
                    for (int q = 0; q < kWide; q++) {
                        lhits += __popc(mine[q]);
                        if (mine[q]) last = 32 * q + 31 - __clz(mine[q]);
                    }
                    clk = clock_base + pos + last;
                }
            }
            if (PRIO && CLASS) {
#pragma unroll
                for (int q = 0; q < kWide; q++) {
                    const unsigned pf = __reduce_or_sync(FULL, took[q]);
                    if ((Sq[q] & Rq[q]) >> lane & 1u)
                        write_class(a, pos + 32 * q + lane, ((pf >> lane) & 1u) ? 1 : 0);
                }
            }
            if (m >= kWin) break;
            // the miss at window position m
            const int qm = m >> 5, lm = m & 31;
            uint32_t gsel = gw[0];
            unsigned Ssel = Sq[0];
#pragma unroll
            for (int q = 1; q < kWide; q++)
                if (qm == q) { gsel = gw[q]; Ssel = Sq[q]; }
            const uint32_t gc = __shfl_sync(FULL, gsel, lm);
            const bool isS = (Ssel >> lm) & 1u;
            const int64_t at_m = pos + m;
            if (PRIO) {
                if (isS) {
                    od++;
                    if (CLASS && lane == 0) write_class(a, at_m, 2);
                } else {
                    ins++;
                }
            } else {
                od++;
                if (a.per_access_hit && lane == 0)
                    a.per_access_hit[a.vals ? a.vals[at_m] : at_m] = 0;
            }
            int target;
            const bool full = count >= W;
            if (full && key32) {
                unsigned key;
                if (PRIO) {
                    const int32_t pe = pr - decay;
                    key = tag >= 0 ? ((unsigned)(pe > 0 ? pe : 0) << gb) | (unsigned)tag : ~0u;
                } else {
                    key = tag >= 0 ? (unsigned)(clk - kbase) : ~0u;
                }
                const unsigned kmin = __reduce_min_sync(FULL, key);
                target = __ffs(__ballot_sync(FULL, key == kmin)) - 1;
            } else if (full) {
                unsigned khi, klo;
                if (PRIO) {
                    const int32_t pe = pr - decay;
                    khi = tag >= 0 ? (unsigned)(pe > 0 ? pe : 0) : ~0u;
                    klo = (unsigned)tag;
                } else {
                    khi = tag >= 0 ? (unsigned)((uint64_t)clk >> 32) : ~0u;
                    klo = (unsigned)clk;
                }
                const unsigned hmin = __reduce_min_sync(FULL, khi);
                const unsigned lmin = __reduce_min_sync(FULL, khi == hmin ? klo : ~0u);
                target = __ffs(__ballot_sync(FULL, khi == hmin && klo == lmin)) - 1;
            } else {
                target = __ffs(__ballot_sync(FULL, tag == -1)) - 1;
            }
            const int32_t evicted = __shfl_sync(FULL, tag, target);   // -1: a free way
            if (full) {
                if (PRIO) decay++;
                nev++;
                count--;
            }
            if (lane == target) {
                tag = (int32_t)gc;
                if (PRIO) {
                    pr = a.es + decay;
                    mhi = isS ? 0u : 1u;
                } else {
                    clk = clock_base + at_m;
                }
            }
            if (lane == 0) {
                if (evicted >= 0) wmap[div_set((uint32_t)evicted, S, M)] = (uint8_t)kNone;
                wmap[div_set(gc, S, M)] = (uint8_t)target;
            }
            count++;
#pragma unroll
            for (int q = 0; q < kWide; q++) {
                if (wq[q] == target) wq[q] = kNone;        // the evicted gid's events now miss
                if (gw[q] == gc) wq[q] = target;           // the inserted gid's events hit
                Hq[q] = __ballot_sync(FULL, wq[q] != kNone);
            }
            __syncwarp();
            start = m + 1;
        }
    }

    if (is_way) {
        a.st.tags[sbase + lane] = tag;
        int64_t m;
        if (PRIO) {
            const int32_t pe = pr - decay;
            m = (int64_t)((uint64_t)mhi << 32) | (int64_t)(uint32_t)(pe > 0 ? pe : 0);
        } else {
            m = clk;
        }
        a.st.meta[sbase + lane] = m;
    }
    if (lane == 0) a.st.count[set] = count;
    if (PRIO) {
        ch = __reduce_add_sync(FULL, (unsigned)ch);
        ph = __reduce_add_sync(FULL, (unsigned)ph);
        if (lane == 0) flush_counters(a.ctr, ch, ph, od, nev, ins, (unsigned long long)count);
    } else {
        lhits = __reduce_add_sync(FULL, (unsigned)lhits);
        if (lane == 0) flush_lru(a, lhits, od);
    }
    return od + ins;
}

// Diagnostic (scripts/replay_set_timeline.py): when set, every replay_smem_kernel
// warp records [set, start ns, end ns, smid, path] of its set.
__device__ int64_t *g_set_timing = nullptr;

#ifndef RECMG_REPLAY_MINB
#define RECMG_REPLAY_MINB 24
#endif
template <int POLICY, bool CLASS>
__device__ __forceinline__ void replay_one_set(const ReplayArgs &a, int64_t set, uint8_t *base,
                                               int Wp, int hbits, int regs, int tables,
                                               bool heavy_item) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    if (set >= a.S) return;
    const int W = (int)a.W;
    const int64_t sbase = set * a.W;
    SetView v;
    v.ring = reinterpret_cast<uint32_t *>(base);
    v.tags = reinterpret_cast<int32_t *>(base + kRingSlots * kRingBlk * 4);
    v.meta = reinterpret_cast<int64_t *>(base + kRingSlots * kRingBlk * 4 + 4 * Wp);
    v.ht = reinterpret_cast<uint64_t *>(base + kRingSlots * kRingBlk * 4 + 12 * Wp);
    v.hbits = hbits;
    v.hmask = (1u << hbits) - 1u;

    int64_t lo, hi;
    seg_range(a, set, lo, hi);
    int64_t *const timing = g_set_timing;
    uint64_t t_start = 0;
    if (timing) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    auto note_time = [&](int path, unsigned long long misses) {
        if (timing && lane == 0) {
            uint64_t t_end;
            uint32_t sm;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            int64_t *r = timing + 4 * (set + (a.serve_only ? a.S : 0));
            r[0] = (int64_t)t_start;
            r[1] = (int64_t)t_end;
            r[2] = (int64_t)sm | ((int64_t)path << 32);
            r[3] = (hi - lo) | ((int64_t)misses << 32);
        }
    };
    EventRing ring;
    ring.init(v.ring, a.ev + lo, hi - lo, lane);
    if constexpr (POLICY == RECMG_POLICY_PRIORITY || POLICY == RECMG_POLICY_LRU) {
        // every set but the listed heavy ones (their long uniform runs take the
        // fast path below) replays with its ways in registers
        if (W <= 32 && (!heavy_item || regs < 0) && hi - lo < (int64_t)(regs < 0 ? 0x7FFFFFFF : regs)) {
            if (a.qn > 0 && hi - lo >= kTableMinEvents && tables) {
                const unsigned long long m = replay_set_table<POLICY, CLASS>(
                    a, set, lo, hi, base + kRingSlots * kRingBlk * 4, lane);
                note_time(2, m);
                return;
            }
            const unsigned long long m = replay_set_regs<POLICY, CLASS>(a, set, lo, hi, ring, lane);
            note_time(1, m);
            return;
        }
    }

    for (uint32_t i = lane; i <= v.hmask; i += 32) v.ht[i] = kHtEmpty;
    int cnt = 0;
    for (int w = lane; w < Wp; w += 32) {
        const int32_t t = w < W ? a.st.tags[sbase + w] : -2;
        v.tags[w] = t;
        v.meta[w] = w < W ? a.st.meta[sbase + w] : 0;
        cnt += t >= 0;
    }
    __syncwarp();
    for (int w = lane; w < W; w += 32) {
        const int32_t t = v.tags[w];
        if (t < 0) continue;
        uint32_t p = ht_home((uint32_t)t, hbits);
        const unsigned long long entry = ((unsigned long long)(uint32_t)t << 32) | (uint32_t)w;
        while (atomicCAS((unsigned long long *)&v.ht[p], kHtEmpty, entry) != kHtEmpty)
            p = (p + 1) & v.hmask;
    }
    int count = (int)__reduce_add_sync(FULL, (unsigned)cnt);
    __syncwarp();
    const int64_t clock_base = a.st.header[0];
    unsigned long long ch = 0, ph = 0, od = 0, nev = 0, ins = 0, lhits = 0;
    const unsigned lt = (1u << lane) - 1u;
    // PRIORITY: populate()'s decay (every positive priority -1 on each
    // eviction, runtime.py:100-112) is applied lazily -- priorities are stored
    // as p + decay (decay = evictions so far in this launch) and read as
    // max(0, stored - decay), which orders the ways exactly as the eager
    // decrement does, so an eviction costs no pass over the set's ways
    int32_t decay = 0;
    int64_t free_hint = 0;
    // LRU_PF (replay_policy_only with a prefetcher, runtime.py:318-339):
    // meta = clock | prefetch tag << 62; keep-bit updates do not exist there
    constexpr bool PRIO = (POLICY == RECMG_POLICY_PRIORITY);
    constexpr bool LRUPF = (POLICY == RECMG_POLICY_LRU_PF);
    constexpr int64_t kClockMask = (int64_t(1) << 62) - 1;
    // simulate() policies (cache_sim.py:92-249), serve events only:
    //   LRU    meta = clock of the last use                victim min clock
    //   LFU    meta = lfu_meta(count, clock of the last use)  victim min (count, clock)
    //   SRRIP  meta = rrpv                                 victim first way with
    //          rrpv >= max after aging (max_rrpv in a.es)
    //   OPTGEN meta = next use of the last access          victim max next use,
    //          ties (never used again) -> smallest gid
    constexpr bool LFU = (POLICY == RECMG_POLICY_LFU);
    constexpr bool SRRIP = (POLICY == RECMG_POLICY_SRRIP);
    constexpr bool OPT = (POLICY == RECMG_POLICY_OPTGEN);

    // Apply the hit-run part held by one 32-event half (events base+lane,
    // lane < n_run): group by way, the group leader updates its way.
    auto apply_run = [&](int64_t base, uint32_t e, int way, int r0, int n_run) {
        const uint32_t ty = ev_type(e);
        const bool inrun = way >= 0 && lane >= r0 && lane < n_run;
        const unsigned peers = __match_any_sync(FULL, inrun ? (unsigned)way : (0x80000000u | lane));
        const int leader = 31 - __clz(peers);
        if (PRIO) {
            const unsigned Smask = __ballot_sync(FULL, inrun && ty == EV_SERVE);
            const unsigned UPmask = __ballot_sync(FULL, inrun && ty != EV_SERVE);
            const unsigned U1mask = __ballot_sync(FULL, inrun && ty == EV_UPD1);
            bool flag0 = false;
            if (inrun && lane == leader) {
                const int64_t m0 = v.meta[way];
                flag0 = (m0 >> 32) & 1;
                const unsigned sp = peers & Smask, up = peers & UPmask;
                int32_t pr = (int32_t)(m0 & 0xFFFFFFFF);
                bool f = flag0;
                if (sp) {
                    const unsigned c = __popc(sp);
                    if (f) { ph += 1; ch += c - 1; f = false; }
                    else ch += c;
                }
                if (up) {
                    const int last = 31 - __clz(up);
                    pr = a.es + (((U1mask >> last) & 1u) ? 1 : 0) + decay;
                }
                if (sp || up) v.meta[way] = (int64_t)(uint32_t)pr | ((int64_t)f << 32);
            }
            if (CLASS) {
                const bool f0 = __shfl_sync(FULL, flag0, leader);
                if (inrun && ty == EV_SERVE) {
                    const bool first = ((peers & Smask) & lt) == 0;
                    write_class(a, base + lane, (f0 && first) ? 1 : 0);
                }
            }
        } else if (LRUPF) {
            // S hits: first S on a tagged way is the prefetch hit, the way moves
            // to MRU at its last S; P hits change nothing (runtime.py:318-325,336)
            const unsigned Smask = __ballot_sync(FULL, inrun && ty == EV_SERVE);
            bool flag0 = false;
            if (inrun && lane == leader) {
                const unsigned sp = peers & Smask;
                if (sp) {
                    const int64_t m0 = v.meta[way];
                    flag0 = (m0 >> 62) & 1;
                    const unsigned c = __popc(sp);
                    if (flag0) { ph += 1; ch += c - 1; }
                    else ch += c;
                    v.meta[way] = clock_base + base + (31 - __clz(sp));
                }
            }
            if (CLASS) {
                const bool f0 = __shfl_sync(FULL, flag0, leader);
                if (inrun && ty == EV_SERVE) {
                    const bool first = ((peers & Smask) & lt) == 0;
                    write_class(a, base + lane, (f0 && first) ? 1 : 0);
                }
            }
        } else {
            int64_t nu = 0;
            if (OPT && inrun && lane == leader)
                nu = a.next_use[a.vals ? a.vals[base + lane] : base + lane];
            if (inrun && lane == leader) {
                const int64_t clk = clock_base + base + leader;
                if (LFU) v.meta[way] = lfu_meta(v.meta[way], __popc(peers), clk);
                else if (SRRIP) v.meta[way] = 0;
                else if (OPT) v.meta[way] = nu;
                else v.meta[way] = clk;
                lhits += __popc(peers);
            }
        }
        __syncwarp();
    };

    // Uniform-run fast path.  Under Zipf skew the hottest set's segment is
    // mostly long runs of events on ONE resident gid (at
    // config 3 one id is half of a shard's accesses).  Hits never change
    // residency, so a window whose real events all name one resident gid is
    // applied in O(1): S count (the first S takes the prefetch tag), last
    // U/P write, last-use clock.  Tried only after a 64-event step that was
    // itself one such run, so other sets pay nothing.
    constexpr int kFast = 512;          // events per fast step (16 per lane)
    bool try_fast = false;
    for (int64_t pos = lo; pos < hi;) {
        if (try_fast && hi - pos >= 64) {
            const int nf = (int)imin64(kFast, hi - pos);
            const int64_t r0 = pos - lo;
            ring.ensure(r0, nf);
            const uint32_t ef = ring.at(r0);
            const uint32_t G = ev_gid(ef);
            // the window's events all name G (in any event type): its effect
            // is the first/last S, the last U/P and the counts.  Per event: one
            // LDS, an xor-and into the uniformity word and (replays only) two
            // ballots; positions i = j*32 + lane are in event order.
            uint32_t diff = 0, lastUe = 0;
            unsigned sm[kFast / 32], um[kFast / 32];
            constexpr bool TRACK = PRIO || LRUPF;
#pragma unroll
            for (int j = 0; j < kFast / 32; j++) {
                const int i = j * 32 + lane;
                const uint32_t e = i < nf ? ring.at(r0 + i) : ef;
                diff |= (e ^ G) & kGidMask;
                if (TRACK) {
                    const bool isS = i < nf && e == G;            // EV_SERVE == 0
                    const bool isU = i < nf && e != G && (!LRUPF || ev_type(e) == EV_PREFETCH);
                    sm[j] = __ballot_sync(FULL, isS);
                    um[j] = __ballot_sync(FULL, isU);
                    lastUe = isU ? e : lastUe;
                }
            }
            const int way = (G != kGidMask) ? ht_find(v, G) : -1;
            if (__all_sync(FULL, diff == 0) && way >= 0) {
                unsigned nS = 0;
                int fS = -1, lS = -1, lU = -1;
                if (TRACK) {
#pragma unroll
                    for (int j = 0; j < kFast / 32; j++) {
                        nS += __popc(sm[j]);
                        if (fS < 0 && sm[j]) fS = j * 32 + __ffs(sm[j]) - 1;
                        if (sm[j]) lS = j * 32 + 31 - __clz(sm[j]);
                        if (um[j]) lU = j * 32 + 31 - __clz(um[j]);
                    }
                }
                const uint32_t lUty = ev_type(__shfl_sync(FULL, lastUe, lU >= 0 ? (lU & 31) : 0));
                if (PRIO) {
                    const int64_t m0 = v.meta[way];
                    const bool f0 = (m0 >> 32) & 1;
                    if (lane == 0) {
                        int32_t pr = (int32_t)(m0 & 0xFFFFFFFF);
                        bool f = f0;
                        if (nS) {
                            if (f) { ph += 1; ch += nS - 1; f = false; }
                            else ch += nS;
                        }
                        if (lU >= 0) pr = a.es + (lUty == EV_UPD1 ? 1 : 0) + decay;
                        if (nS || lU >= 0) v.meta[way] = (int64_t)(uint32_t)pr | ((int64_t)f << 32);
                    }
                    if (CLASS) {
#pragma unroll
                        for (int j = 0; j < kFast / 32; j++) {
                            const int i = j * 32 + lane;
                            if (i < nf && ev_type(ring.at(r0 + i)) == EV_SERVE)
                                write_class(a, pos + i, (f0 && i == fS) ? 1 : 0);
                        }
                    }
                } else if (LRUPF) {
                    const int64_t m0 = v.meta[way];
                    const bool f0 = (m0 >> 62) & 1;
                    if (lane == 0 && nS) {
                        if (f0) { ph += 1; ch += nS - 1; }
                        else ch += nS;
                        v.meta[way] = clock_base + pos + lS;
                    }
                    if (CLASS) {
#pragma unroll
                        for (int j = 0; j < kFast / 32; j++) {
                            const int i = j * 32 + lane;
                            if (i < nf && ev_type(ring.at(r0 + i)) == EV_SERVE)
                                write_class(a, pos + i, (f0 && i == fS) ? 1 : 0);
                        }
                    }
                } else {
                    // simulate(): every event is a serve hit
                    if (lane == 0) {
                        const int last = nf - 1;
                        const int64_t clk = clock_base + pos + last;
                        if (LFU) v.meta[way] = lfu_meta(v.meta[way], nf, clk);
                        else if (SRRIP) v.meta[way] = 0;
                        else if (OPT) v.meta[way] = a.next_use[a.vals ? a.vals[pos + last] : pos + last];
                        else v.meta[way] = clk;
                        lhits += nf;
                    }
                }
                __syncwarp();
                pos += nf;
                continue;
            }
            try_fast = false;
        }
        // 64 events per step (two per lane): membership of both halves against
        // the same tag set, cut at the first residency-changing miss, the run
        // before it applied half by half, the miss resolved -- and then the
        // rest of the SAME window continues from the miss: a miss changes the
        // membership of at most two gids (the inserted one, now at `target`,
        // and the evicted one), so the window's ways are patched instead of
        // re-read and re-probed (miss-dense sets resolved several misses per
        // 64 probes instead of one)
        const int nb = (int)imin64(64, hi - pos);
        ring.ensure(pos - lo, nb);
        const bool v0 = lane < nb, v1 = lane + 32 < nb;
        const uint32_t e0 = v0 ? ring.at(pos - lo + lane) : 0u;
        const uint32_t e1 = v1 ? ring.at(pos - lo + 32 + lane) : 0u;
        const uint32_t g0 = ev_gid(e0), g1 = ev_gid(e1);
        bool real0 = v0 && g0 != kGidMask, real1 = v1 && g1 != kGidMask;
        if (LRUPF) {
            real0 = real0 && (ev_type(e0) == EV_SERVE || ev_type(e0) == EV_PREFETCH);
            real1 = real1 && (ev_type(e1) == EV_SERVE || ev_type(e1) == EV_PREFETCH);
        }
        int way0 = real0 ? ht_find(v, g0) : -1;
        int way1 = real1 ? ht_find(v, g1) : -1;
        bool cand0, cand1;   // events that miss when not resident
        if (PRIO || LRUPF) {
            const uint32_t t0 = ev_type(e0), t1 = ev_type(e1);
            cand0 = real0 && (t0 == EV_SERVE || t0 == EV_PREFETCH);
            cand1 = real1 && (t1 == EV_SERVE || t1 == EV_PREFETCH);
        } else {
            cand0 = real0;
            cand1 = real1;
        }
        int start = 0;
        for (;;) {
            const unsigned miss0 = __ballot_sync(FULL, cand0 && way0 < 0 && lane >= start);
            const unsigned miss1 = __ballot_sync(FULL, cand1 && way1 < 0 && lane + 32 >= start);
            const int cut = miss0 ? (__ffs(miss0) - 1) : (miss1 ? 32 + __ffs(miss1) - 1 : nb);
            if (start == 0) {
                // a whole 64-window of hits on one gid: the next window may be a long run
                const uint32_t gref = __shfl_sync(FULL, g0, 0);
                const bool same = (!real0 || g0 == gref) && (!real1 || g1 == gref);
                try_fast = cut == nb && nb == 64 && __all_sync(FULL, same);
#ifdef RECMG_NO_FASTRUN
                try_fast = false;
#endif
            }
            if (start < 32) apply_run(pos, e0, way0, start, cut < 32 ? cut : 32);
            if (cut > 32) apply_run(pos + 32, e1, way1, start > 32 ? start - 32 : 0, cut - 32);
            if (cut >= nb) break;
            const uint32_t e = cut < 32 ? e0 : e1;
            int32_t evicted = -1;
                const uint32_t ec = __shfl_sync(FULL, e, cut & 31);
                const uint32_t gc = ev_gid(ec);
                const uint32_t tc = ev_type(ec);
                if (PRIO || LRUPF) {
                    if (tc == EV_SERVE) {
                        od++;
                        if (CLASS && lane == 0) write_class(a, pos + cut, 2);
                    } else {
                        ins++;
                    }
                } else {
                    od++;
                    if (a.per_access_hit && lane == 0)
                        a.per_access_hit[a.vals ? a.vals[pos + cut] : pos + cut] = 0;
                }
                int target;
                if (count >= W) {
                    // populate(): victim = argmin (priority, gid) [LRU: min clock]
                    unsigned long long best = ~0ull;
                    int bslot = -1;
                    for (int w = lane; w < W; w += 32) {
                        const int32_t t = v.tags[w];
                        if (t < 0) continue;
                        const int64_t m = v.meta[w];
                        unsigned long long key;
                        if (PRIO) {
                            const int32_t pe = (int32_t)(m & 0xFFFFFFFF) - decay;
                            key = ((unsigned long long)(uint32_t)(pe > 0 ? pe : 0) << 32) | (uint32_t)t;
                        }
                        else if (OPT) key = ((unsigned long long)((int64_t(1) << 31) - m) << 32) | (uint32_t)t;
                        else if (SRRIP) key = (unsigned long long)w;   // chosen below
                        else if (LFU) key = (unsigned long long)m;
                        else key = (unsigned long long)(m & kClockMask);
                        if (key < best) { best = key; bslot = w; }
                    }
                    if (SRRIP) {
                        // age until some way reaches max (cache_sim.py:158-165), then
                        // take the first such way in slot order
                        int64_t mx = 0;
                        for (int w = lane; w < W; w += 32)
                            if (v.tags[w] >= 0) mx = v.meta[w] > mx ? v.meta[w] : mx;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) {
                            const int64_t om = __shfl_xor_sync(FULL, mx, o);
                            mx = om > mx ? om : mx;
                        }
                        const int64_t dlt = (int64_t)a.es - mx;
                        best = ~0ull;
                        bslot = -1;
                        for (int w = lane; w < W; w += 32) {
                            if (v.tags[w] < 0) continue;
                            const int64_t r = v.meta[w] + (dlt > 0 ? dlt : 0);
                            if (dlt > 0) v.meta[w] = r;
                            if (r >= a.es && (unsigned long long)w < best) { best = (unsigned long long)w; bslot = w; }
                        }
                    }
                    {
                        // warp min of the 64-bit keys (unique per way) with two
                        // REDUX.MIN: the high words, then the low words of the
                        // lanes holding the high minimum; the winner's slot
                        const unsigned hi = (unsigned)(best >> 32);
                        const unsigned hmin = __reduce_min_sync(FULL, hi);
                        const unsigned lmin = __reduce_min_sync(FULL, hi == hmin ? (unsigned)best
                                                                                 : 0xFFFFFFFFu);
                        const unsigned win = __ballot_sync(FULL, hi == hmin && (unsigned)best == lmin);
                        bslot = __shfl_sync(FULL, bslot, __ffs(win) - 1);
                    }
                    if (PRIO) decay++;   // the lazy decay (see `decay`)
                    __syncwarp();
                    evicted = v.tags[bslot];
                    __syncwarp();
                    if (lane == 0) {
                        ht_erase(v, (uint32_t)evicted);
                        v.tags[bslot] = -1;
                    }
                    count--;
                    nev++;
                    target = bslot;
                } else {
                    // first free way at or after the hint (ways below it are occupied:
                    // inside a launch a way is only freed by an eviction, refilled at once)
                    int found = -1;
                    for (int64_t b = free_hint; b < Wp && found < 0; b += 32) {
                        const int w = (int)b + lane;
                        const unsigned fm = __ballot_sync(FULL, w < W && v.tags[w] == -1);
                        if (fm) found = (int)b + __ffs(fm) - 1;
                    }
                    target = found;
                    free_hint = found + 1;
                }
                __syncwarp();
                if (lane == 0) {
                    v.tags[target] = (int32_t)gc;
                    int64_t m;
                    if (PRIO) m = (int64_t)(uint32_t)(a.es + decay) | ((int64_t)(tc == EV_PREFETCH) << 32);
                    else if (LFU) m = lfu_meta(0, 1, clock_base + pos + cut);
                    else if (SRRIP) m = a.es > 1 ? a.es - 1 : 0;
                    else if (OPT) m = a.next_use[a.vals ? a.vals[pos + cut] : pos + cut];
                    else m = (clock_base + pos + cut) | (LRUPF ? ((int64_t)(tc == EV_PREFETCH) << 62) : 0);
                    v.meta[target] = m;
                    ht_insert(v, gc, (uint32_t)target);
                }
                count++;
                __syncwarp();
            // patch the window's membership: the inserted gid now lives at
            // `target`, the evicted one nowhere
            if (evicted >= 0) {
                if (g0 == (uint32_t)evicted) way0 = -1;
                if (g1 == (uint32_t)evicted) way1 = -1;
            }
            if (real0 && g0 == gc) way0 = target;
            if (real1 && g1 == gc) way1 = target;
            start = cut + 1;
            if (start >= nb) break;
        }
        pos += nb;
    }

    // write back the set (PRIORITY: the effective priorities, decay applied)
    for (int w = lane; w < W; w += 32) {
        a.st.tags[sbase + w] = v.tags[w];
        int64_t m = v.meta[w];
        if (PRIO) {
            const int32_t pe = (int32_t)(m & 0xFFFFFFFF) - decay;
            m = (m & ~int64_t(0xFFFFFFFF)) | (int64_t)(uint32_t)(pe > 0 ? pe : 0);
        }
        a.st.meta[sbase + w] = m;
    }
    if (lane == 0) a.st.count[set] = count;
    if (PRIO || LRUPF) {
        ch = __reduce_add_sync(FULL, (unsigned)ch);
        ph = __reduce_add_sync(FULL, (unsigned)ph);
        if (lane == 0) flush_counters(a.ctr, ch, ph, od, nev, ins, (unsigned long long)count);
    } else {
        lhits = __reduce_add_sync(FULL, (unsigned)lhits);
        if (lane == 0) flush_lru(a, lhits, od);
    }
    note_time(0, od + ins);
}

// One warp per CTA.  With a work queue (a.work, the hot path's replays): the
// CTAs of one resident wave pull set items from a global counter -- the
// listed heavy sets first, then every other set in order -- and a warp that
// replays a heavy set marks its SM, so the other warps on that SM stop taking
// new sets once their current one is done: the longest dependency chains
// (which bound the launch: one set can carry 3% of the events) keep an SM's
// issue slots to themselves instead of sharing them with ~20 warps of short
// sets.  Without a queue: one set per CTA, heavy sets in the first CTAs.
// LRU2 (the priority replay with the LRU comparator fused in, on the same
// partitioned events): b holds the comparator's state; items are the heavy
// sets of both (priority first), then every set of the priority buffer, then
// every set of the comparator.
template <int POLICY, bool CLASS, bool LRU2>
__global__ void __launch_bounds__(32, RECMG_REPLAY_MINB)
replay_smem_kernel(ReplayArgs a, ReplayArgs b, int Wp, int hbits, int regs, int tables,
                   int64_t items) {
    extern __shared__ __align__(16) uint8_t dsm[];
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const int nh = a.heavy ? min(__ldg(a.heavy), kHeavySets) : 0;
    const int32_t my_heavy = lane < nh ? __ldg(a.heavy + 1 + lane) : -1;
    uint32_t *const work = a.work;
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    // with a queue, the heavy items go to the first CTAs directly -- one per SM
    // in the launch's first wave -- so no two long chains share an SM; every
    // other item is pulled from the queue
    const int64_t hv = (work && a.heavy) ? (LRU2 ? 2 * kHeavySets : kHeavySets) : 0;
    for (int64_t next = blockIdx.x, round = 0;; round++) {
        int64_t item = next;
        if (work && !(round == 0 && (int64_t)blockIdx.x < hv)) {
            if (*(volatile uint32_t *)(work + 1 + smid) != 0) return;
            uint32_t it = 0;
            if (lane == 0) it = atomicAdd(work, 1u);
            item = hv + (int64_t)__shfl_sync(FULL, it, 0);
        }
        if (item >= items) return;
        next = item + gridDim.x;   // no queue: one item per CTA (grid == items)
        bool second = false;       // LRU2: an item of the comparator
        if (LRU2) {
            if (item < 2 * kHeavySets) {
                second = item >= kHeavySets;
                if (second) item -= kHeavySets;
            } else {
                int64_t r = item - 2 * kHeavySets;
                second = r >= a.S;
                if (second) r -= a.S;
                item = kHeavySets + r;
            }
        }
        int64_t set = item;
        bool heavy_item = false;
        if (a.heavy) {
            if (item < kHeavySets) {
                if (item >= nh) { if (work) continue; return; }
                set = __shfl_sync(FULL, my_heavy, (int)item);
                heavy_item = true;
            } else {
                set = item - kHeavySets;
                if (__any_sync(FULL, my_heavy == (int32_t)set)) { if (work) continue; return; }
            }
        }
        if (heavy_item && work && lane == 0) atomicAdd(work + 1 + smid, 1u);
        if (LRU2 && second)
            replay_one_set<RECMG_POLICY_LRU, false>(b, set, dsm, Wp, hbits, -1, tables, heavy_item);
        else
            replay_one_set<POLICY, CLASS>(a, set, dsm, Wp, hbits, regs, tables, heavy_item);
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        if (heavy_item && work && lane == 0) atomicSub(work + 1 + smid, 1u);
        if (!work) return;
    }
}

// ---------------------------------------------------------------------------
// Wide sets (W > kSmemMaxWays, e.g. the reference's fully associative buffer
// at a realistic capacity): one CTA per set, ways in global memory and an
// id -> slot map for membership.  Warp 0 consumes the event segment 32 events
// at a time exactly as the shared-memory kernel does (membership, cut at the
// first residency-changing miss, the hit-run grouped by slot and applied by
// the group's last lane, the miss resolved); a miss into a full set hands
// the victim search -- an O(W) scan of the set's ways, plus the decay of
// populate() / the SRRIP ageing -- to the whole CTA, then warp 0 inserts.
// Every policy of the engine: PRIORITY (runtime.py:100-112), LRU_PF
// (runtime.py:318-339), LRU / LFU / SRRIP / OPTGEN (cache_sim.py:92-249).
constexpr int kWideThreads = 512;

template <int POLICY, bool CLASS>
__global__ void __launch_bounds__(kWideThreads)
replay_wide_kernel(ReplayArgs a) {
    constexpr bool PRIO = (POLICY == RECMG_POLICY_PRIORITY);
    constexpr bool LRUPF = (POLICY == RECMG_POLICY_LRU_PF);
    constexpr bool LFU = (POLICY == RECMG_POLICY_LFU);
    constexpr bool SRRIP = (POLICY == RECMG_POLICY_SRRIP);
    constexpr bool OPT = (POLICY == RECMG_POLICY_OPTGEN);
    constexpr int64_t kClockMask = (int64_t(1) << 62) - 1;
    constexpr int kWarps = kWideThreads / 32;
    const unsigned FULL = 0xFFFFFFFFu;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t set = blockIdx.x;
    const int64_t W = a.W;
    int32_t *tags = a.st.tags + set * W;
    int64_t *meta = a.st.meta + set * W;
    int32_t *slot_of = a.st.slot_of;
    const int64_t clock_base = a.st.header[0];
    int64_t lo, hi;
    seg_range(a, set, lo, hi);

    __shared__ __align__(16) uint32_t ring_buf[kRingSlots * kRingBlk];
    __shared__ unsigned long long s_key[kWarps];
    __shared__ int64_t s_slot[kWarps];
    __shared__ int64_t s_victim, s_dlt;
    __shared__ int s_cmd;

    // warp 0's replay state
    int32_t count = a.st.count[set];
    unsigned long long ch = 0, ph = 0, od = 0, nev = 0, ins = 0, lhits = 0;
    const unsigned lt = (1u << lane) - 1u;
    int64_t free_hint = 0;
    int64_t pos = lo;
    uint32_t pend_e = 0;     // the miss waiting for a victim, at event pos + pend_cut
    int pend_cut = 0;
    EventRing ring;
    if (warp == 0) ring.init(ring_buf, a.ev + lo, hi - lo, lane);

    auto access_at = [&](int64_t p) -> int64_t { return a.vals ? (int64_t)a.vals[p] : p; };
    auto insert_meta = [&](uint32_t tc, int64_t p) -> int64_t {
        if (PRIO) return (int64_t)(uint32_t)a.es | ((int64_t)(tc == EV_PREFETCH) << 32);
        if (LFU) return lfu_meta(0, 1, clock_base + p);
        if (SRRIP) return a.es > 1 ? a.es - 1 : 0;
        if (OPT) return a.next_use[access_at(p)];
        return (clock_base + p) | (LRUPF ? ((int64_t)(tc == EV_PREFETCH) << 62) : 0);
    };

    while (true) {
        if (warp == 0) {
            int cmd = 0;
            while (pos < hi) {
                const int nb = (int)imin64(32, hi - pos);
                const bool valid = lane < nb;
                ring.ensure(pos - lo, nb);
                const uint32_t e = valid ? ring.at(pos - lo + lane) : 0u;
                const int32_t g = (int32_t)ev_gid(e);
                const uint32_t ty = ev_type(e);
                bool real = valid && (uint32_t)g != kGidMask;
                if (LRUPF) real = real && (ty == EV_SERVE || ty == EV_PREFETCH);
                const int32_t slot = real ? slot_of[g] : -1;
                const bool member = slot >= 0;
                unsigned missmask;
                if (PRIO || LRUPF)
                    missmask = __ballot_sync(FULL, real && !member && (ty == EV_SERVE || ty == EV_PREFETCH));
                else
                    missmask = __ballot_sync(FULL, real && !member);
                const int cut = missmask ? (__ffs(missmask) - 1) : nb;
                const bool inrun = member && lane < cut;
                const unsigned peers = __match_any_sync(FULL, inrun ? (unsigned)slot : (0x80000000u | lane));
                const int owner = 31 - __clz(peers);
                if (PRIO) {
                    const unsigned Smask = __ballot_sync(FULL, inrun && ty == EV_SERVE);
                    const unsigned UPmask = __ballot_sync(FULL, inrun && ty != EV_SERVE);
                    const unsigned U1mask = __ballot_sync(FULL, inrun && ty == EV_UPD1);
                    bool flag0 = false;
                    if (inrun && lane == owner) {
                        const int64_t m0 = meta[slot];
                        flag0 = (m0 >> 32) & 1;
                        const unsigned sp = peers & Smask, up = peers & UPmask;
                        int32_t p = (int32_t)(m0 & 0xFFFFFFFF);
                        bool f = flag0;
                        if (sp) {
                            const unsigned c = __popc(sp);
                            if (f) { ph += 1; ch += c - 1; f = false; }
                            else ch += c;
                        }
                        if (up) {
                            const int last = 31 - __clz(up);
                            p = a.es + (((U1mask >> last) & 1u) ? 1 : 0);
                        }
                        if (sp || up) meta[slot] = (int64_t)(uint32_t)p | ((int64_t)f << 32);
                    }
                    if (CLASS) {
                        const bool f0 = __shfl_sync(FULL, flag0, owner);
                        if (inrun && ty == EV_SERVE) {
                            const bool first = ((peers & Smask) & lt) == 0;
                            write_class(a, pos + lane, (f0 && first) ? 1 : 0);
                        }
                    }
                } else if (LRUPF) {
                    const unsigned Smask = __ballot_sync(FULL, inrun && ty == EV_SERVE);
                    bool flag0 = false;
                    if (inrun && lane == owner) {
                        const unsigned sp = peers & Smask;
                        if (sp) {
                            const int64_t m0 = meta[slot];
                            flag0 = (m0 >> 62) & 1;
                            const unsigned c = __popc(sp);
                            if (flag0) { ph += 1; ch += c - 1; }
                            else ch += c;
                            meta[slot] = clock_base + pos + (31 - __clz(sp));
                        }
                    }
                    if (CLASS) {
                        const bool f0 = __shfl_sync(FULL, flag0, owner);
                        if (inrun && ty == EV_SERVE) {
                            const bool first = ((peers & Smask) & lt) == 0;
                            write_class(a, pos + lane, (f0 && first) ? 1 : 0);
                        }
                    }
                } else {
                    if (inrun && lane == owner) {
                        const int64_t clk = clock_base + pos + owner;
                        if (LFU) meta[slot] = lfu_meta(meta[slot], __popc(peers), clk);
                        else if (SRRIP) meta[slot] = 0;
                        else if (OPT) meta[slot] = a.next_use[access_at(pos + owner)];
                        else meta[slot] = clk;
                        lhits += __popc(peers);
                    }
                }
                __syncwarp();
                if (cut == nb) {
                    pos += nb;
                    continue;
                }
                const uint32_t ec = __shfl_sync(FULL, e, cut);
                const int32_t gc = (int32_t)ev_gid(ec);
                const uint32_t tc = ev_type(ec);
                if (PRIO || LRUPF) {
                    if (tc == EV_SERVE) {
                        od++;
                        if (CLASS && lane == 0) write_class(a, pos + cut, 2);
                    } else {
                        ins++;
                    }
                } else {
                    od++;
                    if (a.per_access_hit && lane == 0) a.per_access_hit[access_at(pos + cut)] = 0;
                }
                if (count >= W) {          // the CTA finds the victim
                    pend_e = ec;
                    pend_cut = cut;
                    cmd = 1;
                    break;
                }
                // first free slot at or after the hint (slots below it are
                // occupied: inside a launch a slot is only freed by an
                // eviction, which the same miss refills at once)
                int64_t found = -1;
                for (int64_t b = free_hint; b < W && found < 0; b += 32) {
                    const int64_t w = b + lane;
                    const unsigned fm = __ballot_sync(FULL, w < W && tags[w] < 0);
                    if (fm) found = b + __ffs(fm) - 1;
                }
                free_hint = found + 1;
                if (lane == 0) {
                    tags[found] = gc;
                    meta[found] = insert_meta(tc, pos + cut);
                    slot_of[gc] = (int32_t)found;
                }
                count++;
                __syncwarp();
                pos += cut + 1;
            }
            if (lane == 0) s_cmd = cmd;
        }
        __syncthreads();
        if (s_cmd == 0) break;

        // ---- victim search over the W ways, the whole CTA ------------------
        int64_t dlt = 0;
        if (SRRIP) {
            // age until some way reaches max (cache_sim.py:158-165): by max - top
            int64_t mx = 0;
            for (int64_t w = tid; w < W; w += kWideThreads)
                if (tags[w] >= 0) mx = meta[w] > mx ? meta[w] : mx;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const int64_t om = __shfl_xor_sync(FULL, mx, o);
                mx = om > mx ? om : mx;
            }
            if (lane == 0) s_slot[warp] = mx;
            __syncthreads();
            if (tid == 0) {
                int64_t m = 0;
                for (int i = 0; i < kWarps; i++) m = s_slot[i] > m ? s_slot[i] : m;
                s_dlt = (int64_t)a.es - m;
            }
            __syncthreads();
            dlt = s_dlt;
        }
        unsigned long long best = ~0ull;
        int64_t bslot = -1;
        for (int64_t w = tid; w < W; w += kWideThreads) {
            const int32_t t = tags[w];
            if (t < 0) continue;
            const int64_t m = meta[w];
            unsigned long long key;
            if (PRIO) key = ((unsigned long long)(uint32_t)m << 32) | (uint32_t)t;
            else if (OPT) key = ((unsigned long long)((int64_t(1) << 31) - m) << 32) | (uint32_t)t;
            else if (SRRIP) {
                const int64_t r = m + (dlt > 0 ? dlt : 0);
                if (dlt > 0) meta[w] = r;
                key = r >= a.es ? (unsigned long long)w : ~0ull;   // first such way
            } else if (LFU) key = (unsigned long long)m;
            else key = (unsigned long long)(m & kClockMask);
            if (key < best) { best = key; bslot = w; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ob = __shfl_xor_sync(FULL, best, o);
            const int64_t os = __shfl_xor_sync(FULL, bslot, o);
            if (ob < best) { best = ob; bslot = os; }
        }
        if (lane == 0) { s_key[warp] = best; s_slot[warp] = bslot; }
        __syncthreads();
        if (tid == 0) {
            unsigned long long b = s_key[0];
            int64_t bs = s_slot[0];
            for (int i = 1; i < kWarps; i++)
                if (s_key[i] < b) { b = s_key[i]; bs = s_slot[i]; }
            s_victim = bs;
        }
        if (PRIO) {
            // populate(): every resident with p > 0 ages by one (runtime.py:107-108)
            for (int64_t w = tid; w < W; w += kWideThreads) {
                if (tags[w] < 0) continue;
                const int64_t m = meta[w];
                if ((int32_t)(m & 0xFFFFFFFF) > 0) meta[w] = m - 1;
            }
        }
        __syncthreads();
        if (warp == 0) {
            const int64_t v = s_victim;
            if (lane == 0) {
                const int32_t gc = (int32_t)ev_gid(pend_e);
                slot_of[tags[v]] = -1;
                tags[v] = gc;
                meta[v] = insert_meta(ev_type(pend_e), pos + pend_cut);
                slot_of[gc] = (int32_t)v;
            }
            nev++;
            __syncwarp();
            pos += pend_cut + 1;
        }
    }
    if (warp != 0) return;
    if (lane == 0) a.st.count[set] = count;
    if (PRIO || LRUPF) {
        ch = __reduce_add_sync(FULL, (unsigned)ch);
        ph = __reduce_add_sync(FULL, (unsigned)ph);
        if (lane == 0) flush_counters(a.ctr, ch, ph, od, nev, ins, (unsigned long long)count);
    } else {
        lhits = __reduce_add_sync(FULL, (unsigned)lhits);
        if (lane == 0) flush_lru(a, lhits, od);
    }
}

// ---------------------------------------------------------------------------
__global__ void state_reset_kernel(StateView st, int64_t SW, int64_t S, int64_t V) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = i; j < SW; j += stride) {
        st.tags[j] = -1;
        st.meta[j] = 0;
    }
    for (int64_t j = i; j < S; j += stride) st.count[j] = 0;
    if (st.slot_of)
        for (int64_t j = i; j < V; j += stride) st.slot_of[j] = -1;
    if (i < 8) st.header[i] = 0;
}

__global__ void clock_bump_kernel(int64_t *header, int64_t by) { header[0] += by; }
__global__ void add_i64_kernel(int64_t *x, int64_t by) { x[0] += by; }

// next_use[i] = index of the next access to gids[i] (n if none), from the
// accesses stably sorted by id (cache_sim.py:80-89)
__global__ void next_use_kernel(const uint32_t *__restrict__ sorted_ids,
                                const uint32_t *__restrict__ sorted_pos, int64_t n,
                                int32_t *__restrict__ next_use) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const bool more = i + 1 < n && sorted_ids[i + 1] == sorted_ids[i];
        next_use[sorted_pos[i]] = more ? (int32_t)sorted_pos[i + 1] : (int32_t)n;
    }
}

// keep[i] = 1 exactly when the next reference to the block hits
// (simulate_optgen keep_decisions, cache_sim.py:214-218)
__global__ void keep_kernel(const int32_t *__restrict__ next_use, const uint8_t *__restrict__ hit,
                            int64_t n, uint8_t *__restrict__ keep) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = next_use[i];
        keep[i] = (j < n && hit[j]) ? 1 : 0;
    }
}

// Single PriorityBuffer operation on set (gid % S); one warp.
__global__ void buffer_op_kernel(StateView st, int64_t S, int64_t W, int32_t op, int64_t gid,
                                 int64_t arg, int32_t flag, int64_t *result) {
    const int lane = threadIdx.x;
    const unsigned FULL = 0xFFFFFFFFu;
    const int64_t set = (op == RECMG_OP_POPULATE) ? arg : gid % S;
    int32_t *tags = st.tags + set * W;
    int64_t *meta = st.meta + set * W;
    // locate gid
    int64_t found = -1;
    if (op != RECMG_OP_POPULATE) {
        for (int64_t base = 0; base < W && found < 0; base += 32) {
            const int64_t w = base + lane;
            const unsigned fm = __ballot_sync(FULL, w < W && tags[w] == (int32_t)gid);
            if (fm) found = base + __ffs(fm) - 1;
        }
    }
    int64_t status = 0, value = 0;
    if (op == RECMG_OP_ADD) {
        if (found >= 0) status = RECMG_E_BUFFER_STATE;            // runtime.py:84-85
        else if (st.count[set] >= W) status = RECMG_E_BUFFER_STATE;  // :86-87
        else {
            int64_t fs = -1;
            for (int64_t base = 0; base < W && fs < 0; base += 32) {
                const int64_t w = base + lane;
                const unsigned fm = __ballot_sync(FULL, w < W && tags[w] < 0);
                if (fm) fs = base + __ffs(fm) - 1;
            }
            if (lane == 0) {
                tags[fs] = (int32_t)gid;
                meta[fs] = (int64_t)(uint32_t)arg | ((int64_t)(flag != 0) << 32);
                st.count[set]++;
                if (st.slot_of) st.slot_of[gid] = (int32_t)fs;
            }
        }
    } else if (op == RECMG_OP_POPULATE) {
        if (st.count[set] == 0) status = RECMG_E_BUFFER_STATE;    // runtime.py:103-104
        else {
            unsigned long long best = ~0ull;
            int64_t bslot = -1;
            for (int64_t w = lane; w < W; w += 32) {
                if (tags[w] < 0) continue;
                unsigned long long key = ((unsigned long long)(uint32_t)meta[w] << 32) | (uint32_t)tags[w];
                if (key < best) { best = key; bslot = w; }
            }
            for (int o = 16; o > 0; o >>= 1) {
                unsigned long long ob = __shfl_xor_sync(FULL, best, o);
                int64_t os = __shfl_xor_sync(FULL, bslot, o);
                if (ob < best) { best = ob; bslot = os; }
            }
            for (int64_t w = lane; w < W; w += 32)
                if (tags[w] >= 0 && (int32_t)(meta[w] & 0xFFFFFFFF) > 0) meta[w] -= 1;
            __syncwarp();
            value = tags[bslot];
            __syncwarp();
            if (lane == 0) {
                if (st.slot_of) st.slot_of[value] = -1;
                tags[bslot] = -1;
                meta[bslot] = 0;
                st.count[set]--;
            }
        }
    } else if (op == RECMG_OP_REFERENCE) {
        if (found >= 0) {
            int64_t m = meta[found];
            value = (m >> 32) & 1;
            __syncwarp();
            if (lane == 0 && value) meta[found] = m & 0xFFFFFFFFll;
        }
    } else if (op == RECMG_OP_SET_PRIORITY) {
        if (found < 0) status = RECMG_E_BUFFER_STATE;             // KeyError :79-80
        else if (lane == 0) meta[found] = (meta[found] & ~0xFFFFFFFFll) | (uint32_t)arg;
    } else if (op == RECMG_OP_QUERY) {
        value = found >= 0 ? (int64_t)(uint32_t)(meta[found] & 0xFFFFFFFF) : -1;
        if (found >= 0) status = (meta[found] >> 32) & 1;  // tag bit reported in status slot
    }
    if (lane == 0) {
        result[0] = status;
        result[1] = value;
    }
}

// ---------------------------------------------------------------------------
int launch_replay(int policy, bool narrow, bool cls, const ReplayArgs &a, int64_t nsets,
                  cudaStream_t s, const ReplayArgs *lru2) {
    (void)narrow;
    if (nsets <= 0) return RECMG_OK;
    // RECMG_REPLAY_REGS=0: every set through the shared-memory path (A/B, tests)
    // sets of <= 32 ways replay in registers (replay_set_regs / _table).  A/B
    // and tests: RECMG_REPLAY_REGS=0: none; =1: all but the heavy list; =N > 1:
    // sets shorter than N events, heavy ones excluded; -1: all.  Default: all
    // for the priority buffer; the LRU's heavy sets stay on the shared-memory
    // path, whose uniform-run step takes their long single-id runs in O(1)
    // (config 2 hot set: 3.3 vs 4.4 ns/event)
    const char *regs_env = getenv("RECMG_REPLAY_REGS");
    int regs = policy == RECMG_POLICY_PRIORITY ? -1 : 0x7FFFFFFF;
    if (regs_env && regs_env[0]) {
        const long v = strtol(regs_env, nullptr, 10);
        regs = v == 1 ? 0x7FFFFFFF : (int)(v < -1 ? 0 : (v > 0x7FFFFFFF ? 0x7FFFFFFF : v));
    }
    if (a.W <= kSmemMaxWays) {
        const int Wp = (int)((a.W + 31) / 32 * 32);
        int hbits = 6;
        while ((1 << hbits) < (Wp <= 256 ? 4 * Wp : 2 * Wp)) hbits++;
        int bytes = kRingSlots * kRingBlk * 4 + 12 * Wp + 8 * (1 << hbits);
        // long sets of <= 32 ways: a direct-mapped way map after the ring
        // (replay_set_table); RECMG_REPLAY_TABLES=0 disables it
        const char *t_env = getenv("RECMG_REPLAY_TABLES");
        const int tables = (t_env && t_env[0] == '0') ? 0 : 1;
        ReplayArgs at = a;
        at.qn = 0;
        if (a.W <= 32 && a.S > 1 && a.total_ids > 0) {
            const int64_t qn = (a.total_ids + a.S - 1) / a.S;
            if (qn <= kTableMaxBytes) {
                at.qn = (int32_t)((qn + 15) / 16 * 16);
                at.smagic = set_magic((uint32_t)a.S);
                const int need = kRingSlots * kRingBlk * 4 + at.qn;
                bytes = bytes > need ? bytes : need;
            }
        }
        // one warp (one set) per CTA: a few KB of shared memory, so replay
        // CTAs co-reside with other kernels' CTAs (pipelined with the forwards)
        const size_t smem = (size_t)bytes;
        int64_t items = nsets + (a.heavy ? kHeavySets : 0);
        const bool fused = lru2 && policy == RECMG_POLICY_PRIORITY && a.heavy && a.W <= 32 && !cls;
        ReplayArgs bq;
        if (fused) {
            bq = *lru2;
            bq.qn = at.qn;
            bq.smagic = at.smagic;
            bq.heavy = a.heavy;
            bq.work = a.work;
            items *= 2;
        } else {
            memset(&bq, 0, sizeof(bq));
        }
        // diagnostic: RECMG_REPLAY_ONLY_HEAVY=1 replays the heavy list alone
        const char *h_env = getenv("RECMG_REPLAY_ONLY_HEAVY");
        if (h_env && h_env[0] == '1' && a.heavy) items = fused ? 2 * kHeavySets : kHeavySets;
        // RECMG_REPLAY_QUEUE=0: one set per CTA, no SM reservation (A/B)
        // The queue (and its SM reservation for the heavy chains) only when the
        // replay has the GPU to itself: beside the forwards of a pipelined
        // schedule (a model SM budget below the SM count) the few free SMs
        // must all take sets (config 3 shard 0: 372 vs 431 M acc/s)
        const char *q_env = getenv("RECMG_REPLAY_QUEUE");
        ReplayArgs aq = at;
        if ((q_env && q_env[0] == '0') || (!(q_env && q_env[0] == '1') &&
                                           model_sm_budget() < kSmCount))
            aq.work = nullptr;
        if (aq.work) RECMG_CUDA_TRY(cudaMemsetAsync(aq.work, 0, sizeof(uint32_t) * kWorkWords, s));
#define RECMG_SMEM_LAUNCH2(P, C, L2)                                                       \
    do {                                                                                    \
        RECMG_CUDA_TRY(cudaFuncSetAttribute(replay_smem_kernel<P, C, L2>,                   \
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                                            (int)smem));                                    \
        unsigned grid = (unsigned)items;                                                    \
        if (aq.work) {                                                                      \
            int per_sm = 0;                                                                 \
            RECMG_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(                   \
                &per_sm, replay_smem_kernel<P, C, L2>, 32, smem));                          \
            const int64_t wave = (int64_t)kSmCount * (per_sm > 0 ? per_sm : 1);             \
            grid = (unsigned)(items < wave ? items : wave);                                 \
        }                                                                                   \
        replay_smem_kernel<P, C, L2><<<grid, 32, smem, s>>>(aq, bq, Wp, hbits, regs,        \
                                                           tables, items);                  \
    } while (0)
#define RECMG_SMEM_LAUNCH(P, C) RECMG_SMEM_LAUNCH2(P, C, false)
        if (fused) {
            RECMG_SMEM_LAUNCH2(RECMG_POLICY_PRIORITY, false, true);
        } else if (policy == RECMG_POLICY_PRIORITY) {
            if (cls) RECMG_SMEM_LAUNCH(RECMG_POLICY_PRIORITY, true);
            else RECMG_SMEM_LAUNCH(RECMG_POLICY_PRIORITY, false);
        } else if (policy == RECMG_POLICY_LRU_PF) {
            if (cls) RECMG_SMEM_LAUNCH(RECMG_POLICY_LRU_PF, true);
            else RECMG_SMEM_LAUNCH(RECMG_POLICY_LRU_PF, false);
        } else if (policy == RECMG_POLICY_LFU) {
            RECMG_SMEM_LAUNCH(RECMG_POLICY_LFU, false);
        } else if (policy == RECMG_POLICY_SRRIP) {
            RECMG_SMEM_LAUNCH(RECMG_POLICY_SRRIP, false);
        } else if (policy == RECMG_POLICY_OPTGEN) {
            RECMG_SMEM_LAUNCH(RECMG_POLICY_OPTGEN, false);
        } else {
            RECMG_SMEM_LAUNCH(RECMG_POLICY_LRU, false);
        }
#undef RECMG_SMEM_LAUNCH
#undef RECMG_SMEM_LAUNCH2
    } else {
#define RECMG_WIDE_LAUNCH(P, C) \
    replay_wide_kernel<P, C><<<(unsigned)nsets, kWideThreads, 0, s>>>(a)
        if (policy == RECMG_POLICY_PRIORITY) {
            if (cls) RECMG_WIDE_LAUNCH(RECMG_POLICY_PRIORITY, true);
            else RECMG_WIDE_LAUNCH(RECMG_POLICY_PRIORITY, false);
        } else if (policy == RECMG_POLICY_LRU_PF) {
            if (cls) RECMG_WIDE_LAUNCH(RECMG_POLICY_LRU_PF, true);
            else RECMG_WIDE_LAUNCH(RECMG_POLICY_LRU_PF, false);
        } else if (policy == RECMG_POLICY_LFU) {
            RECMG_WIDE_LAUNCH(RECMG_POLICY_LFU, false);
        } else if (policy == RECMG_POLICY_SRRIP) {
            RECMG_WIDE_LAUNCH(RECMG_POLICY_SRRIP, false);
        } else if (policy == RECMG_POLICY_OPTGEN) {
            RECMG_WIDE_LAUNCH(RECMG_POLICY_OPTGEN, false);
        } else {
            RECMG_WIDE_LAUNCH(RECMG_POLICY_LRU, false);
        }
#undef RECMG_WIDE_LAUNCH
    }
    RECMG_LAUNCH_CHECK();
    return RECMG_OK;
}

}  // namespace recmg

// diagnostic: per-set timing records of the following replay launches
// ([4 * S] int64 on the device, or null to stop)
extern "C" int recmg_diag_set_timing(int64_t *dev_buf) {
    return cudaMemcpyToSymbol(recmg::g_set_timing, &dev_buf, sizeof(dev_buf)) == cudaSuccess
               ? RECMG_OK
               : RECMG_E_CUDA;
}
