// Stable partition of event words by buffer set (set = gid % S; the null
// prefetch sentinel goes to bucket S).  LSD radix with 8-bit digits:
//   hist    : per-tile digit histogram (warp-aggregated smem atomics)
//   scan    : exclusive scan over the digit-major [256][tiles] histogram
//   scatter : stable in-tile ranks via __match_any_sync, coalesced-as-possible
//             scatter of keys (+ optional 32-bit values)
// Every pass reads the tile twice and writes it once: ~12 B/event/pass
// (+8 with values), i.e. HBM-bound; the per-set order of events is the
// original stream order (required: each set replays its events in order).
#include "partition.cuh"

namespace recmg {

constexpr int kPartThreads = 256;
constexpr int kPartItems = 16;
constexpr int kPartTile = kPartThreads * kPartItems;  // 4096
constexpr int kPartWarps = kPartThreads / 32;

__device__ __forceinline__ uint32_t set_of_event(uint32_t e, uint32_t S) {
    uint32_t g = ev_gid(e);
    return g == kGidMask ? S : g % S;
}

__global__ void __launch_bounds__(kPartThreads)
part_hist_kernel(const uint32_t *__restrict__ keys, int64_t N, uint32_t S, int shift,
                 uint32_t *__restrict__ hist, int ntiles, const uint32_t *__restrict__ n_lim) {
    __shared__ uint32_t h[256];
    const int tile = blockIdx.x;
    if (n_lim) N = imin64(N, (int64_t)*n_lim);
    for (int i = threadIdx.x; i < 256; i += kPartThreads) h[i] = 0;
    __syncthreads();
    const int64_t base = (int64_t)tile * kPartTile;
#pragma unroll 4
    for (int r = 0; r < kPartItems; r++) {
        int64_t i = base + (int64_t)r * kPartThreads + threadIdx.x;
        uint32_t d = 0xFFFFFFFFu;
        if (i < N) {
            const uint32_t st = set_of_event(__ldg(keys + i), S);
            if (st < S) d = (st >> shift) & 255u;   // no-events (set S) are dropped
        }
        unsigned peers = __match_any_sync(0xFFFFFFFFu, d);
        if (d != 0xFFFFFFFFu && (threadIdx.x & 31) == (unsigned)(__ffs(peers) - 1))
            atomicAdd(&h[d], (uint32_t)__popc(peers));
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 256; i += kPartThreads) hist[(int64_t)i * ntiles + tile] = h[i];
}

template <bool VALS>
__global__ void __launch_bounds__(kPartThreads)
part_scatter_kernel(const uint32_t *__restrict__ kin, const uint32_t *__restrict__ vin,
                    uint32_t *__restrict__ kout, uint32_t *__restrict__ vout, int64_t N,
                    uint32_t S, int shift, const uint32_t *__restrict__ offs, int ntiles,
                    const uint32_t *__restrict__ n_lim) {
    __shared__ uint32_t wcnt[kPartWarps][256];
    if (n_lim) N = imin64(N, (int64_t)*n_lim);
    __shared__ uint32_t toff[256];
    const int tile = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < kPartWarps * 256; i += kPartThreads) (&wcnt[0][0])[i] = 0;
    for (int i = threadIdx.x; i < 256; i += kPartThreads) toff[i] = offs[(int64_t)i * ntiles + tile];
    __syncthreads();

    const int64_t wbase = (int64_t)tile * kPartTile + (int64_t)warp * (32 * kPartItems);
    uint32_t k[kPartItems], v[kPartItems], rank[kPartItems];
    uint32_t d[kPartItems];
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < kPartItems; r++) {
        int64_t i = wbase + r * 32 + lane;
        d[r] = 0xFFFFFFFFu;
        if (i < N) {
            k[r] = __ldg(kin + i);
            if (VALS) v[r] = __ldg(vin + i);
            const uint32_t st = set_of_event(k[r], S);
            if (st < S) d[r] = (st >> shift) & 255u;
        }
    }
#pragma unroll
    for (int r = 0; r < kPartItems; r++) {
        unsigned peers = __match_any_sync(0xFFFFFFFFu, d[r]);
        uint32_t before = 0;
        if (d[r] != 0xFFFFFFFFu) before = wcnt[warp][d[r]];
        rank[r] = before + __popc(peers & lt);
        __syncwarp();
        if (d[r] != 0xFFFFFFFFu && lane == __ffs(peers) - 1) wcnt[warp][d[r]] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // exclusive scan across warps, per digit
    for (int dg = threadIdx.x; dg < 256; dg += kPartThreads) {
        uint32_t run = toff[dg];
#pragma unroll
        for (int w = 0; w < kPartWarps; w++) {
            uint32_t c = wcnt[w][dg];
            wcnt[w][dg] = run;
            run += c;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kPartItems; r++) {
        if (d[r] == 0xFFFFFFFFu) continue;
        uint32_t pos = wcnt[warp][d[r]] + rank[r];
        kout[pos] = k[r];
        if (VALS) vout[pos] = v[r];
    }
}

// --- generic exclusive scan of uint32 (3 phase) ----------------------------
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t x, uint32_t *total) {
    __shared__ uint32_t warp_sums[32];
    __shared__ uint32_t s_total;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        uint32_t s = (lane < (int)(blockDim.x >> 5)) ? warp_sums[lane] : 0;
        uint32_t si = s;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(0xFFFFFFFFu, si, o);
            if (lane >= o) si += y;
        }
        warp_sums[lane] = si - s;
        if (lane == 31) s_total = si;
    }
    __syncthreads();
    uint32_t res = warp_sums[warp] + incl - x;
    if (total) *total = s_total;
    __syncthreads();
    return res;
}

__global__ void __launch_bounds__(kScanThreads)
scan_reduce_kernel(const uint32_t *__restrict__ in, int64_t M, uint32_t *__restrict__ partial) {
    int64_t base = (int64_t)blockIdx.x * kScanTile;
    uint32_t s = 0;
#pragma unroll
    for (int r = 0; r < kScanItems; r++) {
        int64_t i = base + (int64_t)r * kScanThreads + threadIdx.x;
        if (i < M) s += in[i];
    }
    s = __reduce_add_sync(0xFFFFFFFFu, s);
    __shared__ uint32_t ws[32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        uint32_t t = ws[threadIdx.x];
        t = __reduce_add_sync(0xFFFFFFFFu, t);
        if (threadIdx.x == 0) partial[blockIdx.x] = t;
    }
}

// Single-CTA exclusive scan of `partial` (nblocks entries, loops in tiles).
__global__ void __launch_bounds__(kScanThreads)
scan_partials_kernel(uint32_t *partial, int64_t nblocks) {
    uint32_t carry = 0;
    for (int64_t base = 0; base < nblocks; base += kScanThreads) {
        int64_t i = base + threadIdx.x;
        uint32_t x = i < nblocks ? partial[i] : 0;
        uint32_t tot;
        uint32_t ex = block_exclusive_scan(x, &tot);
        if (i < nblocks) partial[i] = carry + ex;
        carry += tot;
    }
}

__global__ void __launch_bounds__(kScanThreads)
scan_downsweep_kernel(const uint32_t *__restrict__ in, uint32_t *__restrict__ out, int64_t M,
                      const uint32_t *__restrict__ partial) {
    int64_t base = (int64_t)blockIdx.x * kScanTile + (int64_t)threadIdx.x * kScanItems;
    uint32_t x[kScanItems], s = 0;
#pragma unroll
    for (int r = 0; r < kScanItems; r++) {
        x[r] = (base + r < M) ? in[base + r] : 0;
        s += x[r];
    }
    uint32_t tot;
    uint32_t ex = block_exclusive_scan(s, &tot) + partial[blockIdx.x];
#pragma unroll
    for (int r = 0; r < kScanItems; r++) {
        if (base + r < M) out[base + r] = ex;
        ex += x[r];
    }
}

size_t scan_workspace_elems(int64_t M) { return (size_t)((M + kScanTile - 1) / kScanTile) + 1; }

int exclusive_scan_u32(const uint32_t *in, uint32_t *out, int64_t M, uint32_t *partial,
                       cudaStream_t s) {
    if (M <= 0) return RECMG_OK;
    int64_t nb = (M + kScanTile - 1) / kScanTile;
    scan_reduce_kernel<<<(unsigned)nb, kScanThreads, 0, s>>>(in, M, partial);
    RECMG_LAUNCH_CHECK();
    scan_partials_kernel<<<1, kScanThreads, 0, s>>>(partial, nb);
    RECMG_LAUNCH_CHECK();
    scan_downsweep_kernel<<<(unsigned)nb, kScanThreads, 0, s>>>(in, out, M, partial);
    RECMG_LAUNCH_CHECK();
    return RECMG_OK;
}

// --- segment bounds after the sort -----------------------------------------
__global__ void seg_bounds_kernel(const uint32_t *__restrict__ k, int64_t N, uint32_t S,
                                  uint32_t *__restrict__ start, uint32_t *__restrict__ end,
                                  const uint32_t *__restrict__ n_lim) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    N = imin64(N, (int64_t)*n_lim);
    if (i >= N) return;
    uint32_t s = set_of_event(k[i], S);
    if (s >= S) return;
    if (i == 0 || set_of_event(k[i - 1], S) != s) start[s] = (uint32_t)i;
    if (i == N - 1 || set_of_event(k[i + 1], S) != s) end[s] = (uint32_t)(i + 1);
}

// events kept by the first pass (every no-event, set S, is dropped there):
// the exclusive scan's last offset plus the last count
__global__ void n_real_kernel(const uint32_t *__restrict__ hist,
                              const uint32_t *__restrict__ offs, int64_t M,
                              uint32_t *__restrict__ n_real) {
    n_real[0] = offs[M - 1] + hist[M - 1];
}

// Sets whose segment is much longer than the mean (Zipf skew: one set can
// hold half of a shard's events): listed so the replay launch starts them
// first instead of in set order behind thousands of short sets.
__global__ void heavy_sets_kernel(const uint32_t *__restrict__ start,
                                  const uint32_t *__restrict__ end, int64_t S, uint32_t thr,
                                  int32_t *__restrict__ cand) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= S) return;
    if (end[s] > start[s] && end[s] - start[s] >= thr) {
        const int i = atomicAdd(cand, 1);
        if (i < kHeavyCand) cand[1 + i] = (int32_t)s;
    }
}

// The kHeavySets longest of the candidates, longest first (ties: lower set),
// so the longest chains are the first items of the replay launch.
__global__ void __launch_bounds__(kHeavyCand)
heavy_rank_kernel(const uint32_t *__restrict__ start, const uint32_t *__restrict__ end,
                  const int32_t *__restrict__ cand, int32_t *__restrict__ heavy) {
    __shared__ uint32_t len[kHeavyCand];
    __shared__ int32_t id[kHeavyCand];
    const int n = min(cand[0], kHeavyCand);
    const int i = threadIdx.x;
    if (i < n) {
        id[i] = cand[1 + i];
        len[i] = end[id[i]] - start[id[i]];
    }
    __syncthreads();
    if (i == 0) heavy[0] = min(n, kHeavySets);
    if (i >= n) return;
    int rank = 0;
    for (int j = 0; j < n; j++)
        rank += (len[j] > len[i]) || (len[j] == len[i] && id[j] < id[i]);
    if (rank < kHeavySets) heavy[1 + rank] = id[i];
}

int partition_passes(int64_t S) {
    int bits = 0;
    while ((int64_t(1) << bits) < S + 1) bits++;  // buckets 0..S
    return bits == 0 ? 1 : (bits + 7) / 8;
}

void partition_plan(Arena &a, PartitionBuffers &pb, int64_t N, int64_t S, bool vals) {
    pb.N = N;
    pb.S = S;
    pb.ntiles = (int)((N + kPartTile - 1) / kPartTile);
    pb.alt_keys = a.take<uint32_t>((size_t)N);
    pb.alt_vals = vals ? a.take<uint32_t>((size_t)N) : nullptr;
    int64_t M = (int64_t)256 * pb.ntiles;
    pb.hist = a.take<uint32_t>((size_t)M);
    pb.offs = a.take<uint32_t>((size_t)M);
    pb.partial = a.take<uint32_t>(scan_workspace_elems(M));
    pb.seg_start = a.take<uint32_t>((size_t)S + 1);
    pb.seg_end = a.take<uint32_t>((size_t)S + 1);
    pb.heavy = a.take<int32_t>(1 + kHeavySets);
    pb.heavy_cand = a.take<int32_t>(1 + kHeavyCand);
    pb.n_real = a.take<uint32_t>(1);
    pb.work = a.take<uint32_t>(kWorkWords);
}

int partition_run(PartitionBuffers &pb, uint32_t *&keys, uint32_t *&vals, cudaStream_t s) {
    const int64_t N = pb.N, S = pb.S;
    RECMG_CUDA_TRY(cudaMemsetAsync(pb.seg_start, 0, sizeof(uint32_t) * (S + 1), s));
    RECMG_CUDA_TRY(cudaMemsetAsync(pb.seg_end, 0, sizeof(uint32_t) * (S + 1), s));
    if (N == 0) return RECMG_OK;
    const int passes = partition_passes(S);
    uint32_t *kin = keys, *vin = vals, *kout = pb.alt_keys, *vout = pb.alt_vals;
    const int64_t M = (int64_t)256 * pb.ntiles;
    for (int p = 0; p < passes; p++) {
        int shift = 8 * p;
        // pass 0 reads all N events and keeps the real ones (n_real of them);
        // later passes read those
        const uint32_t *lim = p == 0 ? nullptr : pb.n_real;
        part_hist_kernel<<<pb.ntiles, kPartThreads, 0, s>>>(kin, N, (uint32_t)S, shift, pb.hist,
                                                           pb.ntiles, lim);
        RECMG_LAUNCH_CHECK();
        int rc = exclusive_scan_u32(pb.hist, pb.offs, M, pb.partial, s);
        if (rc) return rc;
        if (p == 0) {
            n_real_kernel<<<1, 1, 0, s>>>(pb.hist, pb.offs, M, pb.n_real);
            RECMG_LAUNCH_CHECK();
        }
        if (vin)
            part_scatter_kernel<true><<<pb.ntiles, kPartThreads, 0, s>>>(
                kin, vin, kout, vout, N, (uint32_t)S, shift, pb.offs, pb.ntiles, lim);
        else
            part_scatter_kernel<false><<<pb.ntiles, kPartThreads, 0, s>>>(
                kin, nullptr, kout, nullptr, N, (uint32_t)S, shift, pb.offs, pb.ntiles, lim);
        RECMG_LAUNCH_CHECK();
        uint32_t *t = kin; kin = kout; kout = t;
        t = vin; vin = vout; vout = t;
    }
    // the sorted data is in kin/vin; hand back the other buffers as spares
    pb.alt_keys = kout;
    pb.alt_vals = vout;
    keys = kin;
    vals = vin;
    seg_bounds_kernel<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(keys, N, (uint32_t)S,
                                                                  pb.seg_start, pb.seg_end,
                                                                  pb.n_real);
    RECMG_LAUNCH_CHECK();
    RECMG_CUDA_TRY(cudaMemsetAsync(pb.heavy_cand, 0, sizeof(int32_t), s));
    const int64_t mean = N / (S > 0 ? S : 1);
    const uint32_t thr = (uint32_t)(mean * 8 > 4096 ? mean * 8 : 4096);
    heavy_sets_kernel<<<(unsigned)((S + 255) / 256), 256, 0, s>>>(pb.seg_start, pb.seg_end, S,
                                                                   thr, pb.heavy_cand);
    RECMG_LAUNCH_CHECK();
    heavy_rank_kernel<<<1, kHeavyCand, 0, s>>>(pb.seg_start, pb.seg_end, pb.heavy_cand,
                                               pb.heavy);
    RECMG_LAUNCH_CHECK();
    return RECMG_OK;
}

}  // namespace recmg
