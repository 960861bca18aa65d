// Diagnostic tcgen05 GEMM (recmg_selftest_umma): D[128 x N] = A[128 x K] * B[N x K]^T
// with fp16 operands and fp32 accumulation in TMEM, A from shared memory or
// from TMEM.  The tests pin the descriptor / TMEM layouts the LSTM kernels
// rely on against a host GEMM.
#include "common.cuh"
#include "umma.cuh"

namespace recmg {

__global__ void __launch_bounds__(128, 1)
umma_selftest_kernel(const __half *__restrict__ A, const __half *__restrict__ B,
                     float *__restrict__ D, int N, int K, int a_in_tmem) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base_s;
    const int tid = threadIdx.x, warp = tid >> 5;
    uint8_t *sA = smem;                      // 128 x K
    uint8_t *sB = smem + 128 * K * 2;        // N x K
    for (int i = tid; i < 128 * K; i += 128) {
        const int r = i / K, k = i % K;
        *reinterpret_cast<__half *>(sA + umma::kmajor_offset(r, k, K)) = A[i];
    }
    for (int i = tid; i < N * K; i += 128) {
        const int r = i / K, k = i % K;
        *reinterpret_cast<__half *>(sB + umma::kmajor_offset(r, k, K)) = B[i];
    }
    if (tid == 0) umma::mbar_init(&mbar, 1);
    if (warp == 0) umma::tmem_alloc<512>(&tmem_base_s);
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tbase = tmem_base_s;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const uint32_t a_col = 256;  // A-in-TMEM columns [256, 256 + K/2)
    if (a_in_tmem) {
        // row tid of A, two fp16 per 32-bit column
        for (int c0 = 0; c0 < K / 2; c0 += 16) {
            uint32_t r[16];
#pragma unroll
            for (int j = 0; j < 16; j++) {
                const int k = 2 * (c0 + j);
                r[j] = umma::pack_half2(__half2float(A[tid * K + k]), __half2float(A[tid * K + k + 1]));
            }
            umma::tmem_st16(tbase + lane_base + a_col + c0, r);
        }
        umma::tmem_st_wait();
        umma::fence_before();
    }
    __syncthreads();
    if (tid == 0) {
        umma::fence_after();
        const uint32_t idesc = umma::idesc_f16(128, N);
        const uint32_t aaddr = umma::smem_u32(sA), baddr = umma::smem_u32(sB);
        for (int ks = 0; ks < K / 16; ks++) {
            const uint64_t bd = umma::make_desc(baddr + ks * 256, 128, (K / 8) * 128);
            if (a_in_tmem) {
                umma::mma_ts(tbase, tbase + a_col + ks * 8, bd, idesc, ks > 0);
            } else {
                const uint64_t ad = umma::make_desc(aaddr + ks * 256, 128, (K / 8) * 128);
                umma::mma_ss(tbase, ad, bd, idesc, ks > 0);
            }
        }
        umma::commit(&mbar);
    }
    umma::mbar_wait(&mbar, 0);
    umma::fence_after();
    for (int c0 = 0; c0 < N; c0 += 16) {
        float v[16];
        umma::tmem_ld16(tbase + lane_base + c0, v);
        umma::tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; j++) D[tid * N + c0 + j] = v[j];
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_free<512>(tbase);
}

}  // namespace recmg

extern "C" int recmg_selftest_umma(const void *A, const void *B, float *D, int N, int K,
                                   int a_in_tmem, void *stream) {
    using namespace recmg;
    if (N < 16 || N > 256 || N % 16 || K < 16 || K > 256 || K % 16) return RECMG_E_INVALID_CONFIG;
    const size_t smem = (size_t)(128 + N) * K * 2;
    RECMG_CUDA_TRY(cudaFuncSetAttribute(umma_selftest_kernel,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    umma_selftest_kernel<<<1, 128, smem, (cudaStream_t)stream>>>(
        (const __half *)A, (const __half *)B, D, N, K, a_in_tmem);
    RECMG_LAUNCH_CHECK();
    return RECMG_OK;
}
