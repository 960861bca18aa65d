// Diagnostic microbenchmark (not part of the product): tcgen05.mma kind::f16
// issue rate for the operand forms the LSTM kernels can use.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2511_08568_b200/csrc \
//        scripts/umma_rate.cu -o /tmp/umma_rate && /tmp/umma_rate
// Each CTA (one per SM) issues `rounds` x (`per` MMAs of 128xNx16 + commit +
// mbarrier wait) and reports cycles per MMA and per round.
#include <cstdio>
#include <vector>

#include "umma.cuh"

using namespace recmg;

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)1u << 16;                       // LBO (ignored for swizzled K-major)
    d |= (uint64_t)((1024u >> 4) & 0x3FFFu) << 32;  // SBO: 8 rows x 128 B
    d |= (uint64_t)1u << 46;
    d |= (uint64_t)2u << 61;                        // SWIZZLE_128B
    return d;
}

// mode: 0 ts/no-swizzle, 1 ss/no-swizzle, 2 ss/sw128, 3 ts/sw128
__global__ void rate_kernel(int mode, int N, int per, int rounds, long long *out, int rnd, int waitmode) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tbase_s;
    const int tid = threadIdx.x;
    for (int i = tid; i < 100 * 1024 / 16; i += blockDim.x)
    {
        uint32_t x = 2654435761u * (i + 1) ^ (blockIdx.x * 977u);
        uint32_t w[4];
        for (int q = 0; q < 4; q++) {
            x ^= x << 13; x ^= x >> 17; x ^= x << 5;
            // random fp16 pairs in +-[0.03, 1)
            const float a = ((x & 0xffff) / 65536.0f - 0.5f) * 0.2f, b = ((x >> 16) / 65536.0f - 0.5f) * 0.2f;
            w[q] = umma::pack_half2(a, b);
        }
        reinterpret_cast<int4 *>(smem)[i] = rnd ? make_int4(w[0], w[1], w[2], w[3])
                                                : make_int4(0x3c003c00, 0x3c003c00, 0, 0);
    }
    umma::fence_proxy_async();
    if (tid == 0) umma::mbar_init(&mbar, 1);
    if (tid < 32) umma::tmem_alloc<512>(&tbase_s);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tb = tbase_s;
    if (tid < 128) {
        uint32_t r[16];
        for (int k = 0; k < 16; k++) r[k] = rnd ? umma::pack_half2(0.01f * ((tid * 7 + k) % 13 - 6), 0.02f * ((tid + k) % 5 - 2)) : 0x3c003c00u;
        const uint32_t la = tb + ((uint32_t)(32 * (tid >> 5)) << 16);
        for (int c0 = 384; c0 < 512; c0 += 16) umma::tmem_st16(la + c0, r);
        umma::tmem_st_wait();
    }
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t sb = umma::smem_u32(smem);
    const uint32_t idesc = umma::idesc_f16(128, N);
    uint32_t phase = 0;
    long long t0 = clock64();
    for (int r = 0; r < rounds; r++) {
        if (tid == 0) {
            umma::fence_after();
            if (mode == 4) {
                for (int g = 0; g < 2; g++) {
                    const int NN = g ? 64 : 256;
                    const uint32_t id2 = umma::idesc_f16(128, NN);
                    const uint32_t bb = sb + (g ? 65536 : 0);
                    const uint32_t dd = tb + (g ? 256 : 0);
                    for (int ks = 0; ks < 4; ks++)
                        umma::mma_ts(dd, tb + 384 + 8 * ks, umma::make_desc(bb + 256 * ks, 128, 1024), id2, ks > 0 || g == 0);
                    for (int ks = 0; ks < 4; ks++)
                        umma::mma_ts(dd, tb + 384 + 8 * ks, umma::make_desc(bb + NN * 128 + 256 * ks, 128, 1024), id2, 1u);
                    for (int ks = 0; ks < 4; ks++)
                        umma::mma_ts(dd, tb + 416 + 8 * ks, umma::make_desc(bb + 256 * ks, 128, 1024), id2, 1u);
                }
            }
            for (int i = 0; i < (mode == 4 ? 0 : per); i++) {
                const int ks = i & 3;
                uint64_t bd, ad;
                if (mode == 2 || mode == 3) {
                    bd = desc_sw128(sb + 32768 + 32 * ks);
                    ad = desc_sw128(sb + 32 * ks);
                } else {
                    bd = umma::make_desc(sb + 32768 + 256 * ks, 128, 1024);
                    ad = umma::make_desc(sb + 256 * ks, 128, 1024);
                }
                if (mode == 0 || mode == 3)
                    umma::mma_ts(tb, tb + 384 + 8 * ks, bd, idesc, i > 0 ? 1u : 0u);
                else
                    umma::mma_ss(tb, ad, bd, idesc, i > 0 ? 1u : 0u);
            }
            umma::commit(&mbar);
        }
        if (waitmode == 0 || tid == 0) umma::mbar_wait(&mbar, phase);
        if (waitmode == 1) __syncthreads();
        phase ^= 1u;
        umma::fence_after();
    }
    long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = t1 - t0;
    umma::fence_before();
    __syncthreads();
    if (tid < 32) umma::tmem_free<512>(tb);
}

int main(int argc, char **argv) {
    long long *d;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    auto run = [&](int mode, int N, int per, int nt, int wm, const char *name) {
        const int rounds = 2000;
        rate_kernel<<<148, nt, 100 * 1024>>>(mode, N, per, rounds, d, 1, wm);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
        std::vector<long long> h(148);
        cudaMemcpy(h.data(), d, 148 * sizeof(long long), cudaMemcpyDeviceToHost);
        double m = 0;
        for (auto v : h) m += v;
        m /= 148.0 * rounds;
        printf("%-16s N=%3d per=%2d threads=%d: %8.1f cyc/round %7.1f cyc/MMA (peak-rate MMA %5.1f cyc)\n",
               name, N, per, nt, m, per ? m / per : 0.0, 128.0 * N * 16 / 4096.0);
    };
    const char *names[] = {"ts/no-swizzle", "ss/no-swizzle", "ss/sw128", "ts/sw128"};
    for (int mode = 0; mode < 4; mode++)
        for (int N : {64, 128, 256})
            for (int per : {1, 12, 48}) run(mode, N, per, 128, 0, names[mode]);
    for (int nt : {128, 512})
        for (int wm = 0; wm < 2; wm++) run(4, 256, 0, nt, wm, "mma3 Z256+Q64");
    return 0;
}
