// Probe (diagnostic, not product code): where does a cta_group::1 M=64
// tcgen05.mma put its 64 accumulator rows in TMEM, and may the D address
// carry a lane offset (to place a second 64-row tile in the other lanes)?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -I../include -o umma_m64_probe.bin umma_m64_probe.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_fp16.h>

#include "../paper_2511_08568_b200/csrc/umma.cuh"

using namespace recmg;

// D = A[64 x 16] * B[64 x 16]^T ; dump all 128 lanes x 64 columns of TMEM
__global__ void probe(const __half *A, const __half *B, float *out, int lane_off, int a_tmem) {
    __shared__ __align__(1024) uint8_t sA[128 * 16 * 2];
    __shared__ __align__(1024) uint8_t sB[64 * 16 * 2];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tbase_s;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int i = tid; i < 64 * 16; i += 128) {
        const int r = i / 16, k = i % 16;
        *reinterpret_cast<__half *>(sA + umma::kmajor_offset(r, k, 16)) = A[i];
        *reinterpret_cast<__half *>(sB + umma::kmajor_offset(r, k, 16)) = B[i];
    }
    if (tid == 0) umma::mbar_init(&mbar, 1);
    if (warp == 0) umma::tmem_alloc<512>(&tbase_s);
    umma::fence_proxy_async();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tb = tbase_s;
    const uint32_t la = tb + ((uint32_t)(warp * 32) << 16);
    // zero 64 columns of every lane; with a_tmem, A row r (r < 64) goes to the
    // lane the D layout uses for row r under the probed mapping (lane = r
    // for r < 64 here: written at columns [256, 264))
    uint32_t z[16];
    for (int j = 0; j < 16; j++) z[j] = 0u;
    for (int c = 0; c < 64; c += 16) umma::tmem_st16(la + c, z);
    if (a_tmem) {
        const int row = warp * 32 + lane;   // lane of TMEM = row (probe: M=64 A rows 0..63 in lanes 0..63)
        uint32_t r[16];
        for (int j = 0; j < 8; j++)
            r[j] = row < 64 ? umma::pack_half2(__half2float(A[row * 16 + 2 * j]),
                                               __half2float(A[row * 16 + 2 * j + 1])) : 0u;
        for (int j = 8; j < 16; j++) r[j] = 0u;
        umma::tmem_st16(la + 256, r);
    }
    umma::tmem_st_wait();
    umma::fence_before();
    __syncthreads();
    if (tid == 0) {
        umma::fence_after();
        const uint32_t idesc = umma::idesc_f16(64, 64);
        const uint64_t bd = umma::make_desc(umma::smem_u32(sB), 128, 2 * 128);
        const uint32_t d = tb + ((uint32_t)lane_off << 16);
        if (a_tmem) {
            umma::mma_ts(d, tb + 256, bd, idesc, 0u);
        } else {
            const uint64_t ad = umma::make_desc(umma::smem_u32(sA), 128, 2 * 128);
            umma::mma_ss(d, ad, bd, idesc, 0u);
        }
        umma::commit(&mbar);
    }
    umma::mbar_wait(&mbar, 0);
    umma::fence_after();
    for (int c = 0; c < 64; c += 16) {
        float v[16];
        umma::tmem_ld16(la + c, v);
        umma::tmem_ld_wait();
        for (int j = 0; j < 16; j++) out[(warp * 32 + lane) * 64 + c + j] = v[j];
    }
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_free<512>(tb);
}

int main() {
    std::vector<__half> A(64 * 16), B(64 * 16);
    std::vector<float> Af(64 * 16), Bf(64 * 16);
    srand(1);
    for (int i = 0; i < 64 * 16; i++) {
        Af[i] = (float)((rand() % 17) - 8) / 8.0f;
        Bf[i] = (float)((rand() % 17) - 8) / 8.0f;
        A[i] = __float2half(Af[i]);
        B[i] = __float2half(Bf[i]);
    }
    std::vector<float> ref(64 * 64);
    for (int r = 0; r < 64; r++)
        for (int n = 0; n < 64; n++) {
            float s = 0;
            for (int k = 0; k < 16; k++) s += Af[r * 16 + k] * Bf[n * 16 + k];
            ref[r * 64 + n] = s;
        }
    __half *dA, *dB;
    float *dO;
    cudaMalloc(&dA, A.size() * 2);
    cudaMalloc(&dB, B.size() * 2);
    cudaMalloc(&dO, 128 * 64 * 4);
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    for (int a_tmem = 0; a_tmem < 2; a_tmem++) {
        for (int lane_off : {0, 16, 32, 64}) {
            cudaMemset(dO, 0xFF, 128 * 64 * 4);
            probe<<<1, 128>>>(dA, dB, dO, lane_off, a_tmem);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("a_tmem=%d lane_off=%d: %s\n", a_tmem, lane_off, cudaGetErrorString(e));
                return 1;
            }
            std::vector<float> o(128 * 64);
            cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
            // for every TMEM lane, which reference row (if any) it holds
            printf("a_tmem=%d lane_off=%d lane->row:", a_tmem, lane_off);
            for (int l = 0; l < 128; l++) {
                int found = -2;
                bool zero = true;
                for (int n = 0; n < 64; n++) zero = zero && o[l * 64 + n] == 0.0f;
                if (zero) found = -1;
                else
                    for (int r = 0; r < 64 && found < 0; r++) {
                        bool eq = true;
                        for (int n = 0; n < 64 && eq; n++) eq = o[l * 64 + n] == ref[r * 64 + n];
                        if (eq) found = r;
                    }
                printf(" %d", found);
            }
            printf("\n");
        }
    }
    return 0;
}
