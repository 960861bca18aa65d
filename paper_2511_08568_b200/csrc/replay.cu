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
// Narrow sets (W <= 32): one warp per set, way w in lane w (registers).  The
// warp consumes its event segment 32 events at a time: membership of all 32
// events against the 32 tags in one pass, then every event before the first
// residency-changing miss is applied in bulk (hits never change residency,
// so this is exactly the sequential order), then that one miss is resolved.
// Wide sets (W > 32, incl. the reference's fully associative buffer): one
// warp per set, ways in global memory (L1/L2 resident), an id->slot map for
// lookups, and the same 32-event batching with __match_any_sync grouping.
#include "replay.cuh"

namespace recmg {

// ---------------------------------------------------------------------------
// event builder: one thread per event slot
__global__ void build_events_kernel(const int32_t *__restrict__ gids, int64_t n, int32_t l_in,
                                    const uint8_t *__restrict__ bits,
                                    const int32_t *__restrict__ pf, int32_t pf_stride, int64_t K,
                                    uint32_t *__restrict__ ev, uint32_t *__restrict__ vals) {
    const int64_t Ec = 2 * (int64_t)l_in + pf_stride;
    const int64_t chunk_ev = K * Ec;
    const int64_t E = chunk_ev + (n - K * l_in);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t e;
        if (i < chunk_ev) {
            int64_t k = i / Ec, r = i - k * Ec;
            if (r < l_in) {
                e = ev_make(EV_SERVE, (uint32_t)gids[k * l_in + r]);
            } else if (r < 2 * l_in) {
                int64_t j = r - l_in;
                uint32_t b = bits ? (uint32_t)bits[k * l_in + j] : 0u;
                e = ev_make(b ? EV_UPD1 : EV_UPD0, (uint32_t)gids[k * l_in + j]);
            } else {
                // -1 pads a row: that entry and everything after it is empty
                const int32_t *row = pf + k * pf_stride;
                const int64_t j = r - 2 * l_in;
                bool pad = false;
                for (int64_t q = 0; q <= j; q++) pad |= (row[q] < 0);
                e = ev_make(EV_PREFETCH, pad ? kGidMask : (uint32_t)row[j]);
            }
        } else {
            e = ev_make(EV_SERVE, (uint32_t)gids[K * l_in + (i - chunk_ev)]);
        }
        ev[i] = e;
        if (vals) vals[i] = (uint32_t)i;
    }
}

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
__global__ void prefetch_stats_kernel(const int32_t *__restrict__ gids, int64_t K, int32_t l_in,
                                      int32_t l_win, const int32_t *__restrict__ pf,
                                      int32_t pf_stride, uint8_t *__restrict__ cov_num,
                                      uint8_t *__restrict__ cov_den,
                                      recmg_counters *__restrict__ ctr) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
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
        if (cov_num) cov_num[k] = (uint8_t)num;
        if (cov_den) cov_den[k] = (uint8_t)den;
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
    int64_t orig = a.vals ? (int64_t)a.vals[pos] : pos;
    a.access_class[access_of_event(orig, a.Ec, a.K, a.l_in)] = c;
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
constexpr int kRingSlots = 4;

struct EventRing {
    uint32_t *buf;       // [kRingSlots * kRingBlk] shared
    const uint32_t *ev;  // global segment base (= ev + lo)
    int64_t n;           // segment length
    int64_t nblk, issued;
    int lane;

    __device__ __forceinline__ void issue_next() {
        const int64_t k = issued;
        const uint32_t *src = ev + k * kRingBlk;
        uint32_t *dst = buf + (k % kRingSlots) * kRingBlk;
        const int cnt = (int)imin64(kRingBlk, n - k * kRingBlk);
        for (int i = lane; i < cnt; i += 32) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                             (uint32_t)__cvta_generic_to_shared(dst + i)),
                         "l"(src + i) : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        issued++;
    }
    __device__ __forceinline__ void init(uint32_t *b, const uint32_t *e, int64_t len, int l) {
        buf = b; ev = e; n = len; lane = l; issued = 0;
        nblk = (len + kRingBlk - 1) / kRingBlk;
        while (issued < nblk && issued < kRingSlots) issue_next();
    }
    // make events [r, r + cnt) (relative) readable; refill freed slots
    __device__ __forceinline__ void ensure(int64_t r, int cnt) {
        const int64_t k0 = r / kRingBlk;
        while (issued < nblk && issued < k0 + kRingSlots) issue_next();
        const int64_t k1 = (r + cnt - 1) / kRingBlk;
        const int64_t pending = issued - 1 - k1;   // groups allowed to stay in flight
        if (pending <= 0) asm volatile("cp.async.wait_group 0;" ::: "memory");
        else if (pending == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
        else if (pending == 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
        else asm volatile("cp.async.wait_group 3;" ::: "memory");
        __syncwarp();
    }
    __device__ __forceinline__ uint32_t at(int64_t r) const {
        return buf[((r / kRingBlk) % kRingSlots) * kRingBlk + (r % kRingBlk)];
    }
};

// ---------------------------------------------------------------------------
// Narrow sets: warp per set, W <= 32 ways in lanes.
template <int POLICY, bool CLASS>
__global__ void __launch_bounds__(kNarrowWarps * 32)
replay_narrow_kernel(ReplayArgs a) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x & 31;
    const int64_t set = (int64_t)blockIdx.x * kNarrowWarps + (threadIdx.x >> 5);
    if (set >= a.S) return;
    const int W = (int)a.W;
    const unsigned wayMask = (W == 32) ? FULL : ((1u << W) - 1u);
    const int64_t sbase = set * a.W;

    // way state in registers; lanes >= W hold -2 (never resident, never free)
    int32_t tag = -2;
    int64_t meta = 0;
    if (lane < W) {
        tag = a.st.tags[sbase + lane];
        meta = a.st.meta[sbase + lane];
    }
    int32_t prio = (int32_t)(meta & 0xFFFFFFFF);
    bool flag = (meta >> 32) & 1;
    const int64_t clock_base = a.st.header[0];

    int64_t lo, hi;
    seg_range(a, set, lo, hi);
    unsigned long long ch = 0, ph = 0, od = 0, nev = 0, ins = 0, lhits = 0;

    __shared__ uint32_t ring_buf[kNarrowWarps][kRingSlots * kRingBlk];
    EventRing ring;
    ring.init(ring_buf[threadIdx.x >> 5], a.ev + lo, hi - lo, lane);
    for (int64_t pos = lo; pos < hi;) {
        const int nb = (int)imin64(32, hi - pos);
        const bool valid = lane < nb;
        ring.ensure(pos - lo, nb);
        const uint32_t e = valid ? ring.at(pos - lo + lane) : 0u;
        const int32_t g = (int32_t)ev_gid(e);
        const uint32_t ty = ev_type(e);

        // membership: event lanes learn their way; way lanes learn their events
        int myway = -1;
        unsigned myev = 0;
#pragma unroll
        for (int w = 0; w < 32; w++) {
            const int32_t tw = __shfl_sync(FULL, tag, w);
            const bool hit = valid && (g == tw);
            const unsigned b = __ballot_sync(FULL, hit);
            if (hit) myway = w;
            if (lane == w) myev = b;
        }
        const bool member = myway >= 0;
        unsigned missmask;
        const bool real = valid && (uint32_t)g != kGidMask;  // kGidMask = empty prefetch slot
        if (POLICY == RECMG_POLICY_PRIORITY)
            missmask = __ballot_sync(FULL, real && !member && (ty == EV_SERVE || ty == EV_PREFETCH));
        else
            missmask = __ballot_sync(FULL, real && !member);
        const int cut = missmask ? (__ffs(missmask) - 1) : nb;
        const unsigned below = (cut >= 32) ? FULL : ((1u << cut) - 1u);

        if (POLICY == RECMG_POLICY_PRIORITY) {
            const unsigned Smask = __ballot_sync(FULL, valid && ty == EV_SERVE);
            const unsigned UPmask = __ballot_sync(FULL, valid && ty != EV_SERVE);
            const unsigned U1mask = __ballot_sync(FULL, valid && ty == EV_UPD1);
            const unsigned m = myev & below;
            const unsigned sm = m & Smask;
            const bool pf_first = (sm != 0) && flag;
            if (sm) {
                const unsigned c = __popc(sm);
                if (flag) { ph += 1; ch += c - 1; flag = false; }
                else ch += c;
            }
            const unsigned upm = m & UPmask;
            if (upm) {
                const int last = 31 - __clz(upm);
                prio = a.es + (((U1mask >> last) & 1u) ? 1 : 0);
            }
            if (CLASS) {
                const int first_s = sm ? (__ffs(sm) - 1) : -1;
                const int fs = __shfl_sync(FULL, first_s, member ? myway : 0);
                const bool pff = __shfl_sync(FULL, pf_first, member ? myway : 0);
                if (lane < cut && member && ty == EV_SERVE)
                    write_class(a, pos + lane, (pff && fs == lane) ? 1 : 0);
            }
        } else {
            const unsigned m = myev & below;
            if (m) {
                lhits += __popc(m);
                meta = clock_base + pos + (31 - __clz(m));
            }
            if (a.per_access_hit && lane < cut)
                a.per_access_hit[a.vals ? a.vals[pos + lane] : pos + lane] = 1;
        }

        if (cut < nb) {
            // the first residency-changing event: resolve it serially
            const uint32_t ec = __shfl_sync(FULL, e, cut);
            const int32_t gc = (int32_t)ev_gid(ec);
            const uint32_t tc = ev_type(ec);
            const unsigned resident = __ballot_sync(FULL, tag >= 0);
            if (POLICY == RECMG_POLICY_PRIORITY) {
                if (tc == EV_SERVE) {
                    od++;
                    if (CLASS && lane == 0) write_class(a, pos + cut, 2);
                } else {
                    ins++;
                }
                if (__popc(resident) == W) {
                    // populate(): argmin (priority, gid), age all p>0
                    const unsigned key = (tag >= 0) ? (unsigned)prio : 0xFFFFFFFFu;
                    const unsigned minp = __reduce_min_sync(FULL, key);
                    const unsigned gk = (tag >= 0 && (unsigned)prio == minp) ? (unsigned)tag : 0xFFFFFFFFu;
                    const unsigned ming = __reduce_min_sync(FULL, gk);
                    if (tag >= 0 && prio > 0) prio--;
                    if (tag >= 0 && (unsigned)tag == ming) { tag = -1; flag = false; }
                    nev++;
                }
                const unsigned freem = __ballot_sync(FULL, tag == -1) & wayMask;
                if (lane == __ffs(freem) - 1) {
                    tag = gc;
                    prio = a.es;
                    flag = (tc == EV_PREFETCH);
                }
            } else {
                od++;
                if (a.per_access_hit && lane == 0)
                    a.per_access_hit[a.vals ? a.vals[pos + cut] : pos + cut] = 0;
                if (__popc(resident) == W) {
                    // evict the least recently used way (unique clocks)
                    const long long key = (tag >= 0) ? (long long)meta : LLONG_MAX;
                    long long mn = key;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) mn = min(mn, __shfl_xor_sync(FULL, mn, o));
                    if (tag >= 0 && key == mn) tag = -1;
                    nev++;
                }
                const unsigned freem = __ballot_sync(FULL, tag == -1) & wayMask;
                if (lane == __ffs(freem) - 1) {
                    tag = gc;
                    meta = clock_base + pos + cut;
                }
            }
            pos += cut + 1;
        } else {
            pos += nb;
        }
    }

    // write back
    if (lane < W) {
        a.st.tags[sbase + lane] = tag;
        if (POLICY == RECMG_POLICY_PRIORITY)
            a.st.meta[sbase + lane] = (int64_t)(uint32_t)prio | ((int64_t)flag << 32);
        else
            a.st.meta[sbase + lane] = meta;
    }
    const unsigned occ = __popc(__ballot_sync(FULL, tag >= 0));
    if (lane == 0) a.st.count[set] = (int32_t)occ;
    if (POLICY == RECMG_POLICY_PRIORITY) {
        ch = __reduce_add_sync(FULL, (unsigned)ch);
        ph = __reduce_add_sync(FULL, (unsigned)ph);
        if (lane == 0) flush_counters(a.ctr, ch, ph, od, nev, ins, occ);
    } else {
        lhits = __reduce_add_sync(FULL, (unsigned)lhits);
        if (lane == 0 && a.hits_misses) {
            if (lhits) atomicAdd((unsigned long long *)&a.hits_misses[0], lhits);
            if (od) atomicAdd((unsigned long long *)&a.hits_misses[1], od);
        }
    }
}

// ---------------------------------------------------------------------------
// Wide sets: one warp per set, W > 32 ways in global memory.
template <int POLICY, bool CLASS>
__global__ void __launch_bounds__(32)
replay_wide_kernel(ReplayArgs a) {
    const unsigned FULL = 0xFFFFFFFFu;
    const int lane = threadIdx.x;
    const int64_t set = blockIdx.x;
    const int64_t W = a.W;
    int32_t *tags = a.st.tags + set * W;
    int64_t *meta = a.st.meta + set * W;
    int32_t *slot_of = a.st.slot_of;
    int32_t count = a.st.count[set];
    const int64_t clock_base = a.st.header[0];
    int64_t lo, hi;
    seg_range(a, set, lo, hi);
    unsigned long long ch = 0, ph = 0, od = 0, nev = 0, ins = 0, lhits = 0;
    const unsigned lt = (1u << lane) - 1u;
    int64_t free_hint = 0;

    __shared__ uint32_t ring_buf[kRingSlots * kRingBlk];
    EventRing ring;
    ring.init(ring_buf, a.ev + lo, hi - lo, lane);
    for (int64_t pos = lo; pos < hi;) {
        const int nb = (int)imin64(32, hi - pos);
        const bool valid = lane < nb;
        ring.ensure(pos - lo, nb);
        const uint32_t e = valid ? ring.at(pos - lo + lane) : 0u;
        const int32_t g = (int32_t)ev_gid(e);
        const uint32_t ty = ev_type(e);
        const bool real = valid && (uint32_t)g != kGidMask;
        const int32_t slot = real ? slot_of[g] : -1;
        const bool member = slot >= 0;
        unsigned missmask;
        if (POLICY == RECMG_POLICY_PRIORITY)
            missmask = __ballot_sync(FULL, real && !member && (ty == EV_SERVE || ty == EV_PREFETCH));
        else
            missmask = __ballot_sync(FULL, real && !member);
        const int cut = missmask ? (__ffs(missmask) - 1) : nb;
        const bool inrun = member && lane < cut;
        // group the run's events by slot
        const unsigned peers = __match_any_sync(FULL, inrun ? (unsigned)slot : (0x80000000u | lane));
        const int owner = 31 - __clz(peers);
        if (POLICY == RECMG_POLICY_PRIORITY) {
            const unsigned Smask = __ballot_sync(FULL, inrun && ty == EV_SERVE);
            const unsigned UPmask = __ballot_sync(FULL, inrun && ty != EV_SERVE);
            const unsigned U1mask = __ballot_sync(FULL, inrun && ty == EV_UPD1);
            int64_t m0 = 0;
            bool flag0 = false;
            if (inrun && lane == owner) {
                m0 = meta[slot];
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
        } else {
            if (inrun && lane == owner) {
                meta[slot] = clock_base + pos + owner;
                lhits += __popc(peers);
            }
            if (a.per_access_hit && lane < cut)
                a.per_access_hit[a.vals ? a.vals[pos + lane] : pos + lane] = 1;
        }
        __syncwarp();

        if (cut < nb) {
            const uint32_t ec = __shfl_sync(FULL, e, cut);
            const int32_t gc = (int32_t)ev_gid(ec);
            const uint32_t tc = ev_type(ec);
            if (POLICY == RECMG_POLICY_PRIORITY) {
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
            int64_t target = -1;
            if (count >= W) {
                // victim: min (priority, gid) [priority policy] or min clock [LRU]
                unsigned long long best = ~0ull;
                int64_t bslot = -1;
                for (int64_t w = lane; w < W; w += 32) {
                    const int32_t t = tags[w];
                    if (t < 0) continue;
                    const int64_t m = meta[w];
                    unsigned long long key;
                    if (POLICY == RECMG_POLICY_PRIORITY)
                        key = ((unsigned long long)(uint32_t)m << 32) | (uint32_t)t;
                    else
                        key = (unsigned long long)m;
                    if (key < best) { best = key; bslot = w; }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const unsigned long long ob = __shfl_xor_sync(FULL, best, o);
                    const int64_t os = __shfl_xor_sync(FULL, bslot, o);
                    if (ob < best) { best = ob; bslot = os; }
                }
                if (POLICY == RECMG_POLICY_PRIORITY) {
                    for (int64_t w = lane; w < W; w += 32) {
                        if (tags[w] < 0) continue;
                        const int64_t m = meta[w];
                        if ((int32_t)(m & 0xFFFFFFFF) > 0) meta[w] = m - 1;
                    }
                }
                __syncwarp();
                if (lane == 0) {
                    slot_of[tags[bslot]] = -1;
                    tags[bslot] = -1;
                }
                count--;
                nev++;
                target = bslot;
            } else {
                // first free slot at or after the hint (slots below it are
                // occupied: inside a launch a slot is only freed by an
                // eviction, which the same miss refills immediately)
                int64_t found = -1;
                for (int64_t base = free_hint; base < W && found < 0; base += 32) {
                    const int64_t w = base + lane;
                    const unsigned fm = __ballot_sync(FULL, w < W && tags[w] < 0);
                    if (fm) found = base + __ffs(fm) - 1;
                }
                target = found;
                free_hint = found + 1;
            }
            __syncwarp();
            if (lane == 0) {
                tags[target] = gc;
                if (POLICY == RECMG_POLICY_PRIORITY)
                    meta[target] = (int64_t)(uint32_t)a.es | ((int64_t)(tc == EV_PREFETCH) << 32);
                else
                    meta[target] = clock_base + pos + cut;
                slot_of[gc] = (int32_t)target;
            }
            count++;
            __syncwarp();
            pos += cut + 1;
        } else {
            pos += nb;
        }
    }
    if (lane == 0) a.st.count[set] = count;
    if (POLICY == RECMG_POLICY_PRIORITY) {
        ch = __reduce_add_sync(FULL, (unsigned)ch);
        ph = __reduce_add_sync(FULL, (unsigned)ph);
        if (lane == 0) flush_counters(a.ctr, ch, ph, od, nev, ins, (unsigned long long)count);
    } else {
        lhits = __reduce_add_sync(FULL, (unsigned)lhits);
        if (lane == 0 && a.hits_misses) {
            if (lhits) atomicAdd((unsigned long long *)&a.hits_misses[0], lhits);
            if (od) atomicAdd((unsigned long long *)&a.hits_misses[1], od);
        }
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
                  cudaStream_t s) {
    if (nsets <= 0) return RECMG_OK;
    if (narrow) {
        unsigned grid = (unsigned)((nsets + kNarrowWarps - 1) / kNarrowWarps);
        if (policy == RECMG_POLICY_PRIORITY) {
            if (cls) replay_narrow_kernel<RECMG_POLICY_PRIORITY, true><<<grid, kNarrowWarps * 32, 0, s>>>(a);
            else replay_narrow_kernel<RECMG_POLICY_PRIORITY, false><<<grid, kNarrowWarps * 32, 0, s>>>(a);
        } else {
            replay_narrow_kernel<RECMG_POLICY_LRU, false><<<grid, kNarrowWarps * 32, 0, s>>>(a);
        }
    } else {
        if (policy == RECMG_POLICY_PRIORITY) {
            if (cls) replay_wide_kernel<RECMG_POLICY_PRIORITY, true><<<(unsigned)nsets, 32, 0, s>>>(a);
            else replay_wide_kernel<RECMG_POLICY_PRIORITY, false><<<(unsigned)nsets, 32, 0, s>>>(a);
        } else {
            replay_wide_kernel<RECMG_POLICY_LRU, false><<<(unsigned)nsets, 32, 0, s>>>(a);
        }
    }
    RECMG_LAUNCH_CHECK();
    return RECMG_OK;
}

}  // namespace recmg
