// Shared helpers for the sm_100a kernels of the RecMG hot path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "recmg.h"

#define RECMG_CUDA_TRY(expr)                                        \
    do {                                                            \
        cudaError_t _e = (expr);                                    \
        if (_e != cudaSuccess) return RECMG_E_CUDA;                 \
    } while (0)

// Every kernel launch is followed by exactly one RECMG_LAUNCH_CHECK, which
// also counts it (recmg_launch_count, the bench's gpu_launches evidence).
namespace recmg { void note_launch(); }
#define RECMG_LAUNCH_CHECK()            \
    do {                                \
        recmg::note_launch();           \
        RECMG_CUDA_TRY(cudaGetLastError()); \
    } while (0)

namespace recmg {

constexpr int kSmCount = 148;  // B200: 2 dies x 74 SMs
constexpr int64_t kSmemMaxWays = 4096;  // sets up to this many ways replay in shared memory
// sets whose event segment is far above the mean are replayed by the first
// CTAs of the launch (so the longest dependency chains start first)
constexpr int kHeavySets = 32;
constexpr int kHeavyCand = 1024;  // candidates ranked for the heavy list
// replay work queue words: the next item, then one heavy-chain count per SM id
constexpr int kWorkWords = 1 + 256;

// Event word: [type:2][gid:30]
enum : uint32_t { EV_SERVE = 0u, EV_UPD0 = 1u, EV_UPD1 = 2u, EV_PREFETCH = 3u };
constexpr uint32_t kGidMask = (1u << 30) - 1u;
__host__ __device__ __forceinline__ uint32_t ev_make(uint32_t type, uint32_t gid) {
    return (type << 30) | gid;
}
__host__ __device__ __forceinline__ uint32_t ev_type(uint32_t e) { return e >> 30; }
__host__ __device__ __forceinline__ uint32_t ev_gid(uint32_t e) { return e & kGidMask; }

// Buffer state layout inside the caller's state allocation.
struct StateView {
    int64_t *header;   // [8]: 0 = LRU clock base
    int32_t *tags;     // [S*W] gid or -1
    int64_t *meta;     // [S*W] priority | (prefetch tag << 32)   or LRU clock
    int32_t *count;    // [S]
    int32_t *slot_of;  // [V] (wide sets only), slot within set or -1
};

__host__ __device__ __forceinline__ size_t align_up(size_t x, size_t a) {
    return (x + a - 1) / a * a;
}

struct Geometry {
    int64_t S, W;  // sets, ways per set
    bool wide;     // W > kSmemMaxWays: global-memory ways + id->slot map
};

inline bool geometry_of(const recmg_buffer_cfg *cfg, Geometry *g) {
    if (!cfg || cfg->capacity < 1 || cfg->total_ids < 1 || cfg->total_ids > (int64_t)kGidMask)
        return false;
    if (cfg->ways < 0) return false;
    if (cfg->ways > 0 && cfg->capacity % cfg->ways != 0) return false;
    g->S = cfg->ways > 0 ? cfg->capacity / cfg->ways : 1;
    g->W = cfg->ways > 0 ? cfg->ways : cfg->capacity;
    g->wide = g->W > kSmemMaxWays;
    return true;
}

inline size_t state_bytes(const recmg_buffer_cfg *cfg, const Geometry &g) {
    size_t b = 64;
    b += align_up((size_t)(g.S * g.W) * 4, 256);
    b += align_up((size_t)(g.S * g.W) * 8, 256);
    b += align_up((size_t)g.S * 4, 256);
    if (g.wide) b += align_up((size_t)cfg->total_ids * 4, 256);
    return b;
}

inline StateView state_view(void *state, const recmg_buffer_cfg *cfg, const Geometry &g) {
    char *p = (char *)state;
    StateView v;
    v.header = (int64_t *)p;
    p += 64;
    v.tags = (int32_t *)p;
    p += align_up((size_t)(g.S * g.W) * 4, 256);
    v.meta = (int64_t *)p;
    p += align_up((size_t)(g.S * g.W) * 8, 256);
    v.count = (int32_t *)p;
    p += align_up((size_t)g.S * 4, 256);
    v.slot_of = g.wide ? (int32_t *)p : nullptr;
    return v;
}

// Bump allocator over the caller's workspace.
struct Arena {
    char *base;
    size_t size, used;
    template <typename T>
    T *take(size_t count) {
        size_t off = align_up(used, 256);
        used = off + count * sizeof(T);
        return base ? (T *)(base + off) : nullptr;
    }
    bool ok() const { return used <= size; }
};

// bits needed for the largest gid (total_ids - 1), at least 1
inline int gid_bits_of(int64_t total_ids) {
    int b = 1;
    while (b < 62 && (int64_t(1) << b) < total_ids) b++;
    return b;
}

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

__device__ __forceinline__ unsigned lane_id() {
    unsigned r;
    asm volatile("mov.u32 %0, %%laneid;" : "=r"(r));
    return r;
}

}  // namespace recmg
