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

}  // namespace recmg

using namespace recmg;

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
