// K5: host-row gathers into the HBM embedding buffer and K6: EmbeddingBag
// sum pooling (the DLRM embedding stage the buffer serves; absent from the
// reference, SPEC.md:14,100 — parity is torch.nn.functional.embedding_bag).
//
// Rows live in pinned host memory (cudaHostAlloc, mapped: the kernels read
// them through the UVA pointer, zero-copy over PCIe).  The HBM row buffer
// has one row per buffer slot (set * W + way).  After a replay,
// rows_refresh copies the row of every slot whose occupant changed
// (loaded[slot] != tags[slot]); pooling then reads each access's row from
// its slot when resident, from host memory otherwise (a row evicted again
// inside the same batch), so the pooled sums never depend on buffer state.
#include <string.h>

#include "common.cuh"

namespace recmg {

// one warp: 32 slots per iteration, then warp-wide 16 B/lane copies of the changed rows
__global__ void rows_refresh_kernel(const int32_t *__restrict__ tags, int32_t *__restrict__ loaded,
                                    int64_t nslots, const float4 *__restrict__ host,
                                    float4 *__restrict__ buf, int row_f4,
                                    unsigned long long *copied) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long n = 0;
    for (int64_t base = warp * 32; base < nslots; base += nwarps * 32) {
        const int64_t slot = base + lane;
        int32_t t = -1, l = -1;
        if (slot < nslots) {
            t = tags[slot];
            l = loaded[slot];
        }
        unsigned todo = __ballot_sync(0xFFFFFFFFu, slot < nslots && t >= 0 && t != l);
        while (todo) {
            const int src_lane = __ffs(todo) - 1;
            todo &= todo - 1;
            const int64_t s = base + src_lane;
            const int32_t g = __shfl_sync(0xFFFFFFFFu, t, src_lane);
            for (int i = lane; i < row_f4; i += 32)
                buf[s * row_f4 + i] = host[(int64_t)g * row_f4 + i];   // PCIe zero-copy read
            if (lane == 0) n++;
        }
        if (slot < nslots && t >= 0 && t != l) loaded[slot] = t;
    }
    if (lane == 0 && n) atomicAdd(copied, n);
}

// one warp per bag: for every id, look its set up (32 tags, one per lane),
// read the row from HBM (resident) or host memory (not resident), accumulate.
template <int F4_PER_LANE>
__global__ void embedding_bag_kernel(const int32_t *__restrict__ gids,
                                     const int64_t *__restrict__ offsets, int64_t n_bags,
                                     const int32_t *__restrict__ tags, int64_t S, int W,
                                     const float4 *__restrict__ buf,
                                     const float4 *__restrict__ host, int row_f4,
                                     float4 *__restrict__ out, unsigned long long *src_counts) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long from_hbm = 0, from_host = 0;
    for (int64_t b = warp; b < n_bags; b += nwarps) {
        float4 acc[F4_PER_LANE];
#pragma unroll
        for (int k = 0; k < F4_PER_LANE; k++) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        const int64_t lo = offsets[b], hi = offsets[b + 1];
        for (int64_t i = lo; i < hi; i++) {
            const int32_t g = gids[i];
            const int64_t set = g % S;
            const int32_t t = lane < W ? tags[set * W + lane] : -2;
            const unsigned hit = __ballot_sync(0xFFFFFFFFu, t == g);
            const float4 *row = hit ? buf + (set * W + (__ffs(hit) - 1)) * row_f4
                                    : host + (int64_t)g * row_f4;
            if (hit) from_hbm++; else from_host++;
#pragma unroll
            for (int k = 0; k < F4_PER_LANE; k++) {
                const int c = lane + 32 * k;
                if (c < row_f4) {
                    const float4 v = row[c];
                    acc[k].x += v.x; acc[k].y += v.y; acc[k].z += v.z; acc[k].w += v.w;
                }
            }
        }
#pragma unroll
        for (int k = 0; k < F4_PER_LANE; k++) {
            const int c = lane + 32 * k;
            if (c < row_f4) out[b * row_f4 + c] = acc[k];
        }
    }
    if (lane == 0 && src_counts) {
        if (from_hbm) atomicAdd(&src_counts[0], from_hbm);
        if (from_host) atomicAdd(&src_counts[1], from_host);
    }
}

// K7 fused (DLRM mode): EmbeddingBag(sum) whose epilogue stores every pooled
// row straight into the receiving rank's output over NVLink (P2P stores
// through CUDA-IPC-mapped pointers) -- the all-to-all of pooled embeddings
// is the pooling kernel's own store, no pack kernel and no NCCL call.  Bag
// (b, j) = sample b of the batch, local table j; sample b belongs to rank
// b / (B/G) and lands at [b % (B/G), table_global[j], :] of its output.
template <int F4_PER_LANE>
__global__ void embedding_bag_a2a_kernel(const int32_t *__restrict__ gids,
                                         const int64_t *__restrict__ offsets, int64_t n_bags,
                                         const int32_t *__restrict__ tags, int64_t S, int W,
                                         const float4 *__restrict__ buf,
                                         const float4 *__restrict__ host, int row_f4, int Tg,
                                         int per_rank, int T, const int32_t *__restrict__ tglob,
                                         float4 *const *__restrict__ peer_out,
                                         unsigned long long *src_counts,
                                         unsigned long long *const *peer_flags, int world,
                                         int rank, unsigned long long epoch,
                                         unsigned int *done_blocks) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long from_hbm = 0, from_host = 0;
    for (int64_t bag = warp; bag < n_bags; bag += nwarps) {
        float4 acc[F4_PER_LANE];
#pragma unroll
        for (int k = 0; k < F4_PER_LANE; k++) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        const int64_t lo = offsets[bag], hi = offsets[bag + 1];
        for (int64_t i = lo; i < hi; i++) {
            const int32_t g = gids[i];
            const int64_t set = g % S;
            const int32_t t = lane < W ? tags[set * W + lane] : -2;
            const unsigned hit = __ballot_sync(0xFFFFFFFFu, t == g);
            const float4 *row = hit ? buf + (set * W + (__ffs(hit) - 1)) * row_f4
                                    : host + (int64_t)g * row_f4;
            if (hit) from_hbm++; else from_host++;
#pragma unroll
            for (int k = 0; k < F4_PER_LANE; k++) {
                const int c = lane + 32 * k;
                if (c < row_f4) {
                    const float4 v = row[c];
                    acc[k].x += v.x; acc[k].y += v.y; acc[k].z += v.z; acc[k].w += v.w;
                }
            }
        }
        const int64_t b = bag / Tg;
        const int j = (int)(bag - b * Tg);
        const int dst = (int)(b / per_rank);
        float4 *o = peer_out[dst] + ((b - (int64_t)dst * per_rank) * T + tglob[j]) * row_f4;
#pragma unroll
        for (int k = 0; k < F4_PER_LANE; k++) {
            const int c = lane + 32 * k;
            if (c < row_f4) o[c] = acc[k];
        }
    }
    if (lane == 0 && src_counts) {
        if (from_hbm) atomicAdd(&src_counts[0], from_hbm);
        if (from_host) atomicAdd(&src_counts[1], from_host);
    }
    // completion: every thread fences its peer stores at system scope; the
    // last block to finish publishes `epoch` into every receiver's flag slot
    // [rank] (one-sided release; receivers wait in a2a_wait_kernel)
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(done_blocks, 1u);
        if (prev == gridDim.x - 1) {
            __threadfence_system();
            for (int g = 0; g < world; g++) atomicMax_system(peer_flags[g] + rank, epoch);
            *done_blocks = 0u;   // reusable by the next exchange on this stream
        }
    }
}

__global__ void a2a_wait_kernel(volatile unsigned long long *flags, int world,
                                unsigned long long epoch) {
    for (int g = threadIdx.x; g < world; g += blockDim.x)
        while (flags[g] < epoch) __nanosleep(64);
    __threadfence_system();
}

}  // namespace recmg

using namespace recmg;

extern "C" int recmg_embedding_bag_a2a(const recmg_buffer_cfg *cfg, const void *state,
                                       const int32_t *gids, const int64_t *bag_offsets,
                                       int64_t n_bags, const float *buf_rows,
                                       const float *host_rows, int32_t dim, int32_t batch,
                                       int32_t world, int32_t rank, int32_t n_tables,
                                       const int32_t *table_global, float *const *peer_out,
                                       unsigned long long *const *peer_flags,
                                       unsigned long long *flags, uint64_t epoch,
                                       int64_t *src_counts, void *stream) {
    Geometry g;
    if (!geometry_of(cfg, &g) || g.W > 32 || !state || !host_rows || !buf_rows || dim < 4 ||
        dim % 4 || dim > 512 || world < 1 || rank < 0 || rank >= world || batch % world ||
        n_tables < 1 || !table_global || !peer_out || !peer_flags || !flags || epoch == 0)
        return RECMG_E_INVALID_CONFIG;
    const int Tg = batch > 0 ? (int)(n_bags / batch) : 0;
    if ((int64_t)Tg * batch != n_bags || (n_bags > 0 && (!gids || !bag_offsets)))
        return RECMG_E_INVALID_CONFIG;
    cudaStream_t s = (cudaStream_t)stream;
    // the done-block counter lives in the word after this rank's `world` flags
    unsigned int *done_blocks = reinterpret_cast<unsigned int *>(flags + world);
    {
        StateView st = state_view(const_cast<void *>(state), cfg, g);
        const unsigned grid = (unsigned)imin64(n_bags > 0 ? (n_bags + 7) / 8 : 1, 64 * kSmCount);
        const int f4 = dim / 4;
#define RECMG_BAG_A2A(N)                                                                      \
    embedding_bag_a2a_kernel<N><<<grid, 256, 0, s>>>(                                         \
        gids, bag_offsets, n_bags, st.tags, g.S, (int)g.W, (const float4 *)buf_rows,          \
        (const float4 *)host_rows, f4, Tg, batch / world, n_tables, table_global,            \
        (float4 *const *)peer_out, (unsigned long long *)src_counts, peer_flags, world, rank, \
        epoch, done_blocks)
        if (f4 <= 32) RECMG_BAG_A2A(1);
        else if (f4 <= 64) RECMG_BAG_A2A(2);
        else RECMG_BAG_A2A(4);
#undef RECMG_BAG_A2A
        RECMG_LAUNCH_CHECK();
    }
    a2a_wait_kernel<<<1, 32, 0, s>>>(flags, world, epoch);
    RECMG_LAUNCH_CHECK();
    return RECMG_OK;
}

// ---- peer memory: a dedicated allocation per exchange buffer, mapped into
// the other ranks' processes with CUDA IPC (NVLink P2P on one B200 node) ---
extern "C" int recmg_peer_alloc(size_t bytes, void **dev_ptr) {
    if (!dev_ptr || !bytes) return RECMG_E_INVALID_CONFIG;
    RECMG_CUDA_TRY(cudaMalloc(dev_ptr, bytes));
    RECMG_CUDA_TRY(cudaMemset(*dev_ptr, 0, bytes));
    return RECMG_OK;
}

extern "C" int recmg_peer_free(void *dev_ptr) {
    RECMG_CUDA_TRY(cudaFree(dev_ptr));
    return RECMG_OK;
}

extern "C" int recmg_peer_handle(void *dev_ptr, uint8_t *host_handle64) {
    cudaIpcMemHandle_t h;
    RECMG_CUDA_TRY(cudaIpcGetMemHandle(&h, dev_ptr));
    memcpy(host_handle64, &h, sizeof(h));
    return RECMG_OK;
}

extern "C" int recmg_peer_open(const uint8_t *host_handle64, void **dev_ptr) {
    cudaIpcMemHandle_t h;
    memcpy(&h, host_handle64, sizeof(h));
    RECMG_CUDA_TRY(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return RECMG_OK;
}

extern "C" int recmg_peer_close(void *dev_ptr) {
    RECMG_CUDA_TRY(cudaIpcCloseMemHandle(dev_ptr));
    return RECMG_OK;
}

extern "C" int recmg_rows_refresh(const recmg_buffer_cfg *cfg, const void *state, int32_t *loaded,
                                  const float *host_rows, int32_t dim, float *buf_rows,
                                  int64_t *copied, void *stream) {
    Geometry g;
    if (!geometry_of(cfg, &g) || g.W > 32 || !state || !loaded || !host_rows || !buf_rows ||
        dim < 4 || dim % 4 || !copied)
        return RECMG_E_INVALID_CONFIG;
    StateView st = state_view(const_cast<void *>(state), cfg, g);
    const int64_t nslots = g.S * g.W;
    const unsigned grid = (unsigned)imin64((nslots + 255) / 256 + 1, 8 * kSmCount);
    rows_refresh_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
        st.tags, loaded, nslots, (const float4 *)host_rows, (float4 *)buf_rows, dim / 4,
        (unsigned long long *)copied);
    RECMG_LAUNCH_CHECK();
    return RECMG_OK;
}

extern "C" int recmg_embedding_bag(const recmg_buffer_cfg *cfg, const void *state,
                                   const int32_t *gids, const int64_t *bag_offsets,
                                   int64_t n_bags, const float *buf_rows, const float *host_rows,
                                   int32_t dim, float *out, int64_t *src_counts, void *stream) {
    Geometry g;
    if (!geometry_of(cfg, &g) || g.W > 32 || !state || !gids || !bag_offsets || !host_rows ||
        !buf_rows || !out || dim < 4 || dim % 4 || dim > 512 || n_bags < 0)
        return RECMG_E_INVALID_CONFIG;
    if (n_bags == 0) return RECMG_OK;
    StateView st = state_view(const_cast<void *>(state), cfg, g);
    const unsigned grid = (unsigned)imin64((n_bags + 7) / 8, 64 * kSmCount);
    const int f4 = dim / 4;
    cudaStream_t s = (cudaStream_t)stream;
#define RECMG_BAG(N)                                                                            \
    embedding_bag_kernel<N><<<grid, 256, 0, s>>>(gids, bag_offsets, n_bags, st.tags, g.S,     \
                                                 (int)g.W, (const float4 *)buf_rows,           \
                                                 (const float4 *)host_rows, f4, (float4 *)out, \
                                                 (unsigned long long *)src_counts)
    if (f4 <= 32) RECMG_BAG(1);
    else if (f4 <= 64) RECMG_BAG(2);
    else RECMG_BAG(4);
#undef RECMG_BAG
    RECMG_LAUNCH_CHECK();
    return RECMG_OK;
}
