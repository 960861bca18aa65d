// Probe (diagnostic, not product code): thread <-> (TMEM lane, column) map of
// tcgen05.ld .16x32bx2 (16 lanes, two column halves at an immediate offset),
// the access shape a two-tile (M = 64 per tile) LSTM kernel would use so that
// one warp serves the 16 lanes of one tile in its quadrant.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tmem_probe.bin tmem_16x32bx2_probe.cu
#include <cstdio>

#include "../paper_2511_08568_b200/csrc/umma.cuh"

using namespace recmg;

__global__ void probe(unsigned *out, int lane_base) {
    __shared__ uint32_t tbase_s;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) umma::tmem_alloc<512>(&tbase_s);
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    const uint32_t tb = tbase_s;
    const uint32_t la = tb + ((uint32_t)(warp * 32) << 16);
    // value = lane << 16 | column, written with the known .32x32b shape
    for (int c0 = 0; c0 < 256; c0 += 16) {
        uint32_t r[16];
        for (int j = 0; j < 16; j++) r[j] = ((uint32_t)(warp * 32 + lane) << 16) | (uint32_t)(c0 + j);
        umma::tmem_st16(la + c0, r);
    }
    umma::tmem_st_wait();
    umma::fence_before();
    __syncthreads();
    umma::fence_after();
    // .16x32bx2.x4: 16 lanes from (quadrant base + lane_base), columns [8, 8+4)
    // for the first half-warp and [8+64, 8+64+4) for the second (offset 64)
    uint32_t v[4];
    const uint32_t addr = tb + ((uint32_t)(warp * 32 + lane_base) << 16) + 8;
    asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x4.b32 {%0,%1,%2,%3}, [%4], 64;"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 4; j++) out[tid * 4 + j] = v[j];
    umma::fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_free<512>(tb);
}

int main() {
    unsigned *d;
    cudaMalloc(&d, 128 * 4 * 4);
    for (int lb : {0, 16}) {
        probe<<<1, 128>>>(d, lb);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("lane_base %d: %s\n", lb, cudaGetErrorString(e));
            return 1;
        }
        unsigned h[128 * 4];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("lane_base=%d (thread: lane/col of its 4 registers)\n", lb);
        for (int t = 0; t < 64; t++) {
            printf(" t%d:", t);
            for (int j = 0; j < 4; j++) printf(" %u/%u", h[t * 4 + j] >> 16, h[t * 4 + j] & 0xFFFF);
            printf(t % 4 == 3 ? "\n" : " |");
        }
    }
    return 0;
}
