// Streamed, bit-exact restatement of the reference trace generator
// (generate_trace, trace.py:124-161) for traces too large to materialise
// through numpy (config 3: 500 M accesses over 85.6 M ids).
//
// generate_trace draws, from one numpy default_rng (PCG64):
//   rank_to_gid = permutation(V)                 (left to numpy: the caller)
//   zipf_ranks  = choice(V, n, p)  == cdf.searchsorted(random(n), 'right')
//   sticky_coin = random(n)
//   pool_coin   = random(n)
// then runs the sequential sticky-pool pass.  random() consumes exactly one
// PCG64 output per double, so the three streams start at outputs 0, n and 2n
// after the permutation; any block [i0, i0+count) of any stream is reached
// with the PCG64 jump-ahead (numpy's PCG64.advance).  The searchsorted uses a
// guide table over u in [0,1) so each lookup binary-searches only the cdf
// entries inside its 2^-g bucket; the result is defined by the cdf
// comparisons alone, so it is the numpy result exactly.
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <thread>
#include <vector>

#include "recmg.h"

namespace {

typedef unsigned __int128 u128;

// numpy/random/src/pcg64/pcg64.h: PCG_DEFAULT_MULTIPLIER_{HIGH,LOW}
const u128 kMult = ((u128)2549297995355413924ULL << 64) | (u128)4865540595714422341ULL;

struct Pcg64 {
    u128 state, inc;
    // pcg_setseq_128_xsl_rr_64_random_r: step, then output
    inline uint64_t next() {
        state = state * kMult + inc;
        const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
        const unsigned rot = (unsigned)(state >> 122);
        const uint64_t x = hi ^ lo;
        return (x >> rot) | (x << ((64u - rot) & 63u));
    }
    // pcg_advance_lcg_128 (Brown's jump-ahead)
    void advance(u128 delta) {
        u128 acc_mult = 1, acc_plus = 0, cur_mult = kMult, cur_plus = inc;
        while (delta > 0) {
            if (delta & 1) {
                acc_mult *= cur_mult;
                acc_plus = acc_plus * cur_mult + cur_plus;
            }
            cur_plus = (cur_mult + 1) * cur_plus;
            cur_mult *= cur_mult;
            delta >>= 1;
        }
        state = acc_mult * state + acc_plus;
    }
};

inline double to_double(uint64_t x) {   // numpy next_double
    return (double)(x >> 11) * (1.0 / 9007199254740992.0);
}

Pcg64 make(const uint64_t pcg[4]) {
    Pcg64 g;
    g.state = ((u128)pcg[0] << 64) | (u128)pcg[1];
    g.inc = ((u128)pcg[2] << 64) | (u128)pcg[3];
    return g;
}

template <class F>
void parallel_for(int64_t n, int threads, F f) {
    if (threads < 1) threads = 1;
    const int64_t per = std::max<int64_t>((n + threads - 1) / threads, 1 << 16);
    std::vector<std::thread> ts;
    for (int64_t b = 0; b < n; b += per) ts.emplace_back(f, b, std::min(n, b + per));
    for (auto &t : ts) t.join();
}

}  // namespace

extern "C" int recmg_pcg64_uniforms(const uint64_t pcg[4], int64_t skip, int64_t count,
                                    double *host_out, int32_t threads) {
    if (skip < 0 || count < 0) return RECMG_E_INVALID_CONFIG;
    parallel_for(count, threads, [&](int64_t b, int64_t e) {
        Pcg64 g = make(pcg);
        g.advance((u128)(skip + b));
        for (int64_t i = b; i < e; i++) host_out[i] = to_double(g.next());
    });
    return RECMG_OK;
}

extern "C" int recmg_trace_guide(const double *host_cdf, int64_t V, int32_t guide_log2,
                                 int64_t *host_guide) {
    // guide[b] = #{ j : cdf[j] <= b / 2^g }, b = 0 .. 2^g
    if (V <= 0 || guide_log2 < 1 || guide_log2 > 30) return RECMG_E_INVALID_CONFIG;
    const int64_t M = (int64_t)1 << guide_log2;
    int64_t j = 0;
    for (int64_t b = 0; b <= M; b++) {
        const double edge = (double)b / (double)M;
        while (j < V && host_cdf[j] <= edge) j++;
        host_guide[b] = j;
    }
    return RECMG_OK;
}

extern "C" int recmg_trace_generate_block(const uint64_t pcg[4], int64_t n_total, int64_t i0,
                                          int64_t count, const double *host_cdf, int64_t V,
                                          const int64_t *host_guide, int32_t guide_log2,
                                          const int64_t *host_rank_to_gid, double stickiness,
                                          int32_t pool_size, int64_t *host_pool,
                                          int32_t *host_pool_len, int32_t *host_out,
                                          int32_t threads) {
    if (n_total < 0 || i0 < 0 || count < 0 || i0 + count > n_total || pool_size < 1 ||
        V <= 0 || V > INT32_MAX || *host_pool_len < 0 || *host_pool_len > pool_size)
        return RECMG_E_INVALID_CONFIG;
    const int64_t M = (int64_t)1 << guide_log2;
    std::vector<int32_t> zipf((size_t)count);
    std::vector<double> sticky((size_t)count), coin((size_t)count);
    parallel_for(count, threads, [&](int64_t b, int64_t e) {
        Pcg64 gz = make(pcg), gs = make(pcg), gp = make(pcg);
        gz.advance((u128)(i0 + b));
        gs.advance((u128)(n_total + i0 + b));
        gp.advance((u128)(2 * n_total + i0 + b));
        for (int64_t i = b; i < e; i++) {
            const double u = to_double(gz.next());
            const int64_t k = (int64_t)(u * (double)M);            // exact: M = 2^g
            const double *lo = host_cdf + host_guide[k];
            const double *hi = host_cdf + host_guide[k + 1];
            const int64_t r = std::upper_bound(lo, hi, u) - host_cdf;  // side='right'
            zipf[i] = (int32_t)host_rank_to_gid[r];
            sticky[i] = to_double(gs.next());
            coin[i] = to_double(gp.next());
        }
    });
    // sequential sticky-pool pass (trace.py:144-160), state carried across blocks
    int64_t *pool = host_pool;
    int32_t len = *host_pool_len;
    for (int64_t i = 0; i < count; i++) {
        int64_t gid;
        if (len > 0 && sticky[i] < stickiness)
            gid = pool[(int64_t)(coin[i] * (double)len)];
        else
            gid = zipf[i];
        host_out[i] = (int32_t)gid;
        if (len > 0 && pool[0] == gid) continue;
        int32_t at = -1;
        for (int32_t j = 0; j < len; j++)
            if (pool[j] == gid) { at = j; break; }
        if (at >= 0) {
            memmove(pool + 1, pool, sizeof(int64_t) * (size_t)at);
        } else {
            memmove(pool + 1, pool, sizeof(int64_t) * (size_t)(len < pool_size ? len : pool_size - 1));
            if (len < pool_size) len++;
        }
        pool[0] = gid;
    }
    *host_pool_len = len;
    return RECMG_OK;
}

// Text trace body (trace.py:172-204): lines "table_id,row_id".  Parses from
// byte `pos` while lines have the plain form [ws][+-]digits[ws],[ws][+-]digits[ws]
// and lie in range; stops at the first other line (the caller re-reads that
// line with the reference's own rules, which raise or accept it) or at the
// end.  Blank / whitespace-only lines are skipped, as the reference does.
extern "C" int recmg_trace_parse_text(const char *host_buf, int64_t len, int64_t pos,
                                      const int64_t *host_offsets, int32_t n_tables,
                                      int32_t *host_out, int64_t cap, int64_t *n_out,
                                      int64_t *stop_pos, int64_t *lines_done) {
    int64_t n = *n_out, lines = 0;
    auto ws = [](char ch) { return ch == ' ' || ch == '\t'; };
    while (pos < len) {
        const int64_t line_start = pos;
        int64_t e = pos;
        while (e < len && host_buf[e] != '\n') e++;
        int64_t p = pos, q = e;
        while (p < q && ws(host_buf[p])) p++;
        while (q > p && ws(host_buf[q - 1])) q--;
        if (p == q) {                       // blank line
            pos = e + 1;
            lines++;
            continue;
        }
        int64_t v[2];
        bool ok = true;
        for (int f = 0; f < 2 && ok; f++) {
            while (p < q && ws(host_buf[p])) p++;
            bool neg = false;
            if (p < q && (host_buf[p] == '+' || host_buf[p] == '-')) neg = host_buf[p++] == '-';
            int64_t x = 0;
            int digits = 0;
            while (p < q && host_buf[p] >= '0' && host_buf[p] <= '9' && digits < 18) {
                x = x * 10 + (host_buf[p++] - '0');
                digits++;
            }
            while (p < q && ws(host_buf[p])) p++;
            ok = digits > 0 && (f == 0 ? (p < q && host_buf[p] == ',') : p == q);
            if (f == 0) p++;
            v[f] = neg ? -x : x;
        }
        if (!ok || n >= cap || v[0] < 0 || v[0] >= n_tables || v[1] < 0 ||
            v[1] >= host_offsets[v[0] + 1] - host_offsets[v[0]]) {
            pos = line_start;
            break;
        }
        host_out[n++] = (int32_t)(host_offsets[v[0]] + v[1]);
        pos = e + 1;
        lines++;
    }
    *n_out = n;
    *stop_pos = pos < len ? pos : len;
    *lines_done = lines;
    return RECMG_OK;
}
