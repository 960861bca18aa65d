// Diagnostic (not product code): occupy `ctas` SMs for `ms` milliseconds with
// one 1024-thread CTA per SM that holds the whole register file and only
// spins on the clock (no memory traffic), so a kernel on another stream runs
// on the remaining SMs without memory-system interference.
//   nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC \
//        scripts/sm_hog.cu -o scripts/libsmhog.so
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void __launch_bounds__(1024, 1) hog_kernel(long long cycles, int *sink) {
    const long long t0 = clock64();
    float acc = threadIdx.x;
    while (clock64() - t0 < cycles) {
#pragma unroll 8
        for (int i = 0; i < 64; i++) acc = acc * 0.999f + 1.0f;
    }
    if (acc == -1.0f) *sink = 1;   // never true: keeps the loop
}

// memory hog: every thread streams float4 loads over [buf, buf + n) for the
// same time (mode 1: n large = DRAM, mode 2: n = 64 MB = L2-resident)
__global__ void __launch_bounds__(1024, 1) mem_hog_kernel(long long cycles, const float4 *buf,
                                                          long long n, int *sink) {
    const long long t0 = clock64();
    float acc = 0.0f;
    long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long stride = (long long)gridDim.x * blockDim.x;
    while (clock64() - t0 < cycles) {
#pragma unroll 4
        for (int k = 0; k < 16; k++) {
            const float4 v = __ldcg(buf + i);
            acc += v.x;
            i += stride;
            if (i >= n) i -= n;
        }
    }
    if (acc == -1.0f) *sink = 1;
}

// random 32-byte sector gathers over the buffer (DRAM-unfriendly, like the
// forwards' folded-row gathers): LDG.256 at hashed addresses
__global__ void __launch_bounds__(1024, 1) gather_hog_kernel(long long cycles, const float4 *buf,
                                                             long long n32, int *sink) {
    const long long t0 = clock64();
    float acc = 0.0f;
    unsigned long long x = 0x9E3779B97F4A7C15ull * (blockIdx.x * 1024 + threadIdx.x + 1);
    while (clock64() - t0 < cycles) {
#pragma unroll 4
        for (int k = 0; k < 8; k++) {
            x ^= x << 13; x ^= x >> 7; x ^= x << 17;
            const float4 v = __ldcg(buf + 2 * (long long)(x % (unsigned long long)n32));
            acc += v.x;
        }
    }
    if (acc == -1.0f) *sink = 1;
}

extern "C" int gather_hog(int ctas, double ms, long long bytes, void *stream) {
    static int *sink = nullptr;
    static float4 *buf = nullptr;
    static long long have = 0;
    if (!sink) cudaMalloc(&sink, 4);
    if (have < bytes) {
        if (buf) cudaFree(buf);
        cudaMalloc(&buf, bytes);
        cudaMemset(buf, 0, bytes);
        have = bytes;
    }
    gather_hog_kernel<<<ctas, 1024, 200 * 1024, (cudaStream_t)stream>>>(
        (long long)(ms * 1.9e6), buf, bytes / 32, sink);
    return (int)cudaGetLastError();
}

extern "C" int mem_hog(int ctas, double ms, long long bytes, void *stream) {
    static int *sink = nullptr;
    static float4 *buf = nullptr;
    static long long have = 0;
    if (!sink) cudaMalloc(&sink, 4);
    if (have < bytes) {
        if (buf) cudaFree(buf);
        cudaMalloc(&buf, bytes);
        cudaMemset(buf, 0, bytes);
        have = bytes;
    }
    mem_hog_kernel<<<ctas, 1024, 200 * 1024, (cudaStream_t)stream>>>(
        (long long)(ms * 1.9e6), buf, bytes / 16, sink);
    return (int)cudaGetLastError();
}

// the forward's shape: 512 threads x 128 registers, 115 KB of shared memory,
// optionally with the 512 TMEM columns allocated (tmem = 1)
__global__ void __launch_bounds__(512, 1) shape_hog_kernel(long long cycles, int tmem, int *sink) {
    __shared__ uint32_t base;
    if (tmem && threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                     ::"r"((uint32_t)__cvta_generic_to_shared(&base)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    __syncthreads();
    const long long t0 = clock64();
    float acc[120];
#pragma unroll
    for (int i = 0; i < 120; i++) acc[i] = threadIdx.x + i;
    while (clock64() - t0 < cycles) {
#pragma unroll
        for (int i = 0; i < 120; i++) acc[i] = acc[i] * 0.999f + 1.0f;
    }
    float t = 0.0f;
#pragma unroll
    for (int i = 0; i < 120; i++) t += acc[i];
    if (t == -1.0f) *sink = 1;
    __syncthreads();
    if (tmem && threadIdx.x < 32)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base) : "memory");
}

extern "C" int shape_hog(int ctas, double ms, int tmem, void *stream) {
    static int *sink = nullptr;
    if (!sink) cudaMalloc(&sink, 4);
    cudaFuncSetAttribute(shape_hog_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 118 * 1024);
    shape_hog_kernel<<<ctas, 512, 115 * 1024, (cudaStream_t)stream>>>((long long)(ms * 1.9e6),
                                                                     tmem, sink);
    return (int)cudaGetLastError();
}

extern "C" int sm_hog(int ctas, double ms, void *stream) {
    static int *sink = nullptr;
    if (!sink) cudaMalloc(&sink, 4);
    const long long cycles = (long long)(ms * 1.9e6);
    // 64 registers x 1024 threads = the whole 64K register file of an SM
    hog_kernel<<<ctas, 1024, 200 * 1024, (cudaStream_t)stream>>>(cycles, sink);
    return (int)cudaGetLastError();
}
