// Host-side helpers exported through the C ABI (include/recmg.h).
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "recmg.h"

extern "C" int recmg_trace_pool_pass(const int64_t *zipf_gids, const double *sticky_coin,
                                     const double *pool_coin, int64_t n, double stickiness,
                                     int32_t pool_size, int64_t *out) {
    // generate_trace's sequential pass (trace.py:144-160): with probability
    // `stickiness` reuse one of the last `pool_size` distinct ids (most
    // recent first), otherwise take the Zipf draw; then move the id to the
    // pool front, dropping the oldest beyond pool_size.
    if (n < 0 || pool_size < 1) return RECMG_E_INVALID_CONFIG;
    int64_t *pool = (int64_t *)malloc(sizeof(int64_t) * ((size_t)pool_size + 1));
    if (!pool) return RECMG_E_INVALID_CONFIG;
    int32_t len = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t gid;
        if (len > 0 && sticky_coin[i] < stickiness)
            gid = pool[(int64_t)(pool_coin[i] * (double)len)];   // :147-148
        else
            gid = zipf_gids[i];                                  // :149-150
        out[i] = gid;
        if (len > 0 && pool[0] == gid) continue;                  // :152-153
        int32_t at = -1;
        for (int32_t j = 0; j < len; j++)
            if (pool[j] == gid) { at = j; break; }
        if (at >= 0) {                                            // pool.remove(gid)
            memmove(pool + 1, pool, sizeof(int64_t) * (size_t)at);
        } else {
            memmove(pool + 1, pool, sizeof(int64_t) * (size_t)len);
            if (len < pool_size) len++;                           // del pool[size:]
        }
        pool[0] = gid;                                            // pool.insert(0, gid)
    }
    free(pool);
    return RECMG_OK;
}
