// Diagnostic microbenchmark (not part of the product): does a tcgen05.mma
// chain into ONE accumulator serialize?  Each CTA (one per SM) issues
// `per` MMAs of 128xNx16 (kind::f16, A and B from smem, no swizzle),
// rotating the D address over `nacc` accumulators, then commit + wait.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2511_08568_b200/csrc \
//        scripts/umma_dep.cu -o scripts/umma_dep.bin
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "umma.cuh"

using namespace recmg;

__global__ void dep_kernel(int N, int M, int per, int nacc, int rounds, int kstep, long long *out) {
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
    const uint32_t idesc = umma::idesc_f16(M, N);
    uint32_t phase = 0;
    long long t0 = clock64();
    for (int r = 0; r < rounds; r++) {
        if (tid == 0) {
            umma::fence_after();
            for (int i = 0; i < per; i++) {
                const int ks = kstep ? (i & 3) : 0;
                const uint64_t ad = umma::make_desc(sb + 256 * ks, 128, 1024);
                const uint64_t bd = umma::make_desc(sb + 32768 + 256 * ks, 128, 1024);
                const uint32_t dcol = (uint32_t)((i % nacc) * N);
                umma::mma_ss(tb + dcol, ad, bd, idesc, i >= nacc ? 1u : 0u);
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

int main() {
    long long *d;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaFuncSetAttribute(dep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    auto run = [&](int N, int M, int per, int nacc, int kstep, int grid) {
        const int rounds = 1000;
        dep_kernel<<<grid, 128, 96 * 1024>>>(N, M, per, nacc, rounds, kstep, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); exit(1); }
        std::vector<long long> h(grid);
        cudaMemcpy(h.data(), d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
        double m = 0;
        for (auto v : h) m += v;
        m /= (double)grid * rounds;
        printf("M=%3d N=%3d per=%2d nacc=%d kstep=%d grid=%3d: %8.1f cyc/round %7.1f cyc/MMA (4096 MAC/clk: %5.1f)\n",
               M, N, per, nacc, kstep, grid, m, m / per, (double)M * N * 16 / 4096.0);
    };
    for (int grid : {1, 148})
        for (int N : {64, 256})
            for (int nacc : {1, 2, 4})
                if (nacc * N <= 512) run(N, 128, 48, nacc, 1, grid);
    run(256, 128, 48, 1, 0, 148);
    run(256, 64, 48, 1, 1, 148);
    run(128, 128, 48, 1, 1, 148);
    run(128, 128, 48, 4, 1, 148);
    return 0;
}
