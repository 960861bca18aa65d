// Stable radix partition of event words by buffer set (see partition.cu).
#pragma once
#include "common.cuh"

namespace recmg {

struct PartitionBuffers {
    int64_t N = 0, S = 0;
    int ntiles = 0;
    uint32_t *alt_keys = nullptr, *alt_vals = nullptr;
    uint32_t *hist = nullptr, *offs = nullptr, *partial = nullptr;
    uint32_t *seg_start = nullptr, *seg_end = nullptr;  // [S+1]
    int32_t *heavy = nullptr;  // [1 + kHeavySets]: count, then the heaviest sets
    uint32_t *work = nullptr;  // [kWorkWords]: the replay launch's work queue
    int32_t *heavy_cand = nullptr;  // [1 + kHeavyCand]: count, then sets above the threshold
    uint32_t *n_real = nullptr;     // [1]: events kept (no-events, set S, are dropped)
};

int partition_passes(int64_t S);
void partition_plan(Arena &a, PartitionBuffers &pb, int64_t N, int64_t S, bool vals);
// Sorts keys (and vals) stably by set, dropping the no-events (gid kGidMask,
// set S: collapsed serves, dead updates, padding); on return keys/vals point
// at the sorted arrays (which may be the workspace copies), *n_real of them
// valid, and seg_start/seg_end hold each set's [start, end) range (empty
// sets: 0,0).
int partition_run(PartitionBuffers &pb, uint32_t *&keys, uint32_t *&vals, cudaStream_t s);

size_t scan_workspace_elems(int64_t M);
int exclusive_scan_u32(const uint32_t *in, uint32_t *out, int64_t M, uint32_t *partial,
                       cudaStream_t s);

}  // namespace recmg
