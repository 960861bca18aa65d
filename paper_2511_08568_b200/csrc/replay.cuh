// Replay engine internals (see replay.cu).
#pragma once
#include "common.cuh"

namespace recmg {


struct ReplayArgs;

__global__ void build_events_kernel(const int32_t *__restrict__ gids, int64_t n, int32_t l_in,
                                    const uint8_t *__restrict__ bits,
                                    const int32_t *__restrict__ pf, int32_t pf_stride, int64_t K,
                                    int64_t k0, int64_t nk, int with_tail, uint32_t S,
                                    uint32_t M, int64_t i_begin,
                                    uint32_t *__restrict__ ev, uint32_t *__restrict__ vals,
                                    recmg_counters *__restrict__ ctr,
                                    uint8_t *__restrict__ access_class);
template <int LM>
__global__ void build_chunk_events_kernel(const int32_t *__restrict__ gids, int32_t l_in,
                                          const uint8_t *__restrict__ bits,
                                          const int32_t *__restrict__ pf, int32_t pf_stride,
                                          int64_t K, int64_t k0, int64_t nk, uint32_t S,
                                          uint32_t M, uint32_t *__restrict__ ev,
                                          uint32_t *__restrict__ vals,
                                          recmg_counters *__restrict__ ctr,
                                          uint8_t *__restrict__ access_class);
// M = ceil(2^32 / S) for set_of (0 for S = 1)
inline uint32_t set_magic(uint32_t S) {
    return S <= 1 ? 0u : (uint32_t)((((uint64_t)1 << 32) + S - 1) / S);
}
__global__ void prefetch_stats_kernel(const int32_t *__restrict__ gids, int64_t k0, int64_t nk,
                                      int32_t l_in, int32_t l_win, const int32_t *__restrict__ pf,
                                      int32_t pf_stride, uint16_t *__restrict__ cov_num,
                                      uint16_t *__restrict__ cov_den,
                                      recmg_counters *__restrict__ ctr);
__global__ void state_reset_kernel(StateView st, int64_t SW, int64_t S, int64_t V);
__global__ void clock_bump_kernel(int64_t *header, int64_t by);
__global__ void add_i64_kernel(int64_t *x, int64_t by);
__global__ void next_use_kernel(const uint32_t *__restrict__ sorted_ids,
                                const uint32_t *__restrict__ sorted_pos, int64_t n,
                                int32_t *__restrict__ next_use);
__global__ void keep_kernel(const int32_t *__restrict__ next_use, const uint8_t *__restrict__ hit,
                            int64_t n, uint8_t *__restrict__ keep);
__global__ void buffer_op_kernel(StateView st, int64_t S, int64_t W, int32_t op, int64_t gid,
                                 int64_t arg, int32_t flag, int64_t *result);

struct ReplayArgs {
    const uint32_t *ev;
    const uint32_t *vals;
    const uint32_t *seg_start, *seg_end;
    const int32_t *heavy;      // [1 + kHeavySets] or null: sets started first
    int64_t E;
    int64_t S, W;
    int32_t es;
    int32_t l_in;
    int64_t Ec, K;
    int64_t ev_base;           // global position of local event 0 (chunk-range replays)
    StateView st;
    recmg_counters *ctr;
    uint8_t *access_class;
    int64_t *hits_misses;
    uint8_t *per_access_hit;   // pre-filled with 1 by the caller: kernels write the misses
    const int32_t *next_use;   // OPTGEN: next reference of each access (n if none)
    int32_t gid_bits;          // bits of the largest gid (0: unknown)
    int64_t total_ids;         // ids of the trace (0: unknown)
    int32_t qn;                // way-map bytes per set (0: no way map), set by launch_replay
    uint32_t smagic;           // ceil(2^32 / S)
    int32_t serve_only;        // LRU on the priority replay's events: serves only
    uint32_t *work = nullptr;  // [kWorkWords] or null: replay work queue (see replay_smem_kernel)
};

// lru2: the LRU comparator fused into a priority replay of sets <= 32 ways on
// the same partitioned events (its own state, serve_only) -- or null
int launch_replay(int policy, bool narrow, bool cls, const ReplayArgs &a, int64_t nsets,
                  cudaStream_t s, const ReplayArgs *lru2 = nullptr);

}  // namespace recmg
