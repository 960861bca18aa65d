// Diagnostic microbenchmark (not part of the product): tcgen05.mma issue cost
// with all descriptors precomputed (no per-MMA address math): `per` MMAs of
// 128xNx16 kind::f16 into one accumulator, fully unrolled, then commit + wait.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2511_08568_b200/csrc \
//        scripts/umma_issue.cu -o scripts/umma_issue.bin
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "umma.cuh"

using namespace recmg;

template <int PER, int N, bool TS>
__global__ void issue_kernel(int rounds, long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tbase_s;
    const int tid = threadIdx.x;
    for (int i = tid; i < 96 * 1024 / 16; i += blockDim.x)
        reinterpret_cast<int4 *>(smem)[i] = make_int4(0x3c003c00, 0x3c003c00, 0, 0);
    umma::fence_proxy_async();
    if (tid == 0) umma::mbar_init(&mbar, 1);
    if (tid < 32) umma::tmem_alloc<512>(&tbase_s);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tb = tbase_s;
    const uint32_t sb = umma::smem_u32(smem);
    constexpr uint32_t idesc = umma::idesc_f16(128, N);
    uint64_t ad[4], bd[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        ad[k] = umma::make_desc(sb + 256 * k, 128, 1024);
        bd[k] = umma::make_desc(sb + 32768 + 256 * k, 128, 1024);
    }
    uint32_t phase = 0;
    long long t0 = clock64();
    for (int r = 0; r < rounds; r++) {
        if (tid == 0) {
            umma::fence_after();
#pragma unroll
            for (int i = 0; i < PER; i++) {
                if (TS)
                    umma::mma_ts(tb, tb + 384 + 8 * (i & 3), bd[i & 3], idesc, i > 0 ? 1u : 0u);
                else
                    umma::mma_ss(tb, ad[i & 3], bd[i & 3], idesc, i > 0 ? 1u : 0u);
            }
            umma::commit(&mbar);
        }
        umma::mbar_wait(&mbar, phase);
        phase ^= 1u;
        umma::fence_after();
    }
    long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = t1 - t0;
    umma::fence_before();
    __syncthreads();
    if (tid < 32) umma::tmem_free<512>(tb);
}

long long *d;
template <int PER, int N, bool TS>
void run(int grid) {
    const int rounds = 1000;
    cudaFuncSetAttribute(issue_kernel<PER, N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    issue_kernel<PER, N, TS><<<grid, 128, 96 * 1024>>>(rounds, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
    std::vector<long long> h(grid);
    cudaMemcpy(h.data(), d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    double m = 0;
    for (auto v : h) m += v;
    m /= (double)grid * rounds;
    printf("%s N=%3d per=%2d grid=%3d: %8.1f cyc/round %7.1f cyc/MMA (floor %5.1f)\n", TS ? "ts" : "ss", N,
           PER, grid, m, m / PER, 128.0 * N / 256.0);
}

int main() {
    cudaMalloc(&d, 148 * sizeof(long long));
    run<1, 64, true>(148);
    run<12, 64, true>(148);
    run<48, 64, true>(148);
    run<12, 256, true>(148);
    run<48, 256, true>(148);
    run<12, 64, false>(148);
    run<48, 256, false>(148);
    run<48, 128, true>(148);
    return 0;
}
