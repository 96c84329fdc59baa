// Shared-memory atomic throughput on one B200 (all SMs): red.shared.add.u32
// with random addresses vs addresses whose 32 lanes hit 32 distinct banks.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_atoms tools/microbench_atoms.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <int MODE>
__global__ void __launch_bounds__(1024, 1) k(uint32_t words, int iters, uint32_t* out) {
    extern __shared__ uint32_t acc[];
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) acc[i] = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t base = __cvta_generic_to_shared(acc);
    const uint32_t rows = words / 32;
    uint32_t h = hash32(threadIdx.x * 7919u + blockIdx.x * 104729u);
    for (int it = 0; it < iters; ++it) {
#pragma unroll 8
        for (int u = 0; u < 8; ++u) {
            h = hash32(h + u);
            uint32_t w;
            if (MODE == 0) w = h % words;                       // random
            else if (MODE == 1) w = (h % rows) * 32 + lane;      // distinct banks
            else w = (h % rows) * 32 + ((lane * 5) & 31);        // distinct banks, permuted
            asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(base + w * 4), "r"(1u) : "memory");
        }
    }
    __syncthreads();
    uint32_t s = 0;
    for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) s += acc[i];
    atomicAdd(out, s);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const uint32_t words = 6784 * 8;  // the config-2 pending tile, both parities
    const size_t smem = words * 4;
    uint32_t* out;
    cudaMalloc(&out, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 2000;
    for (int mode = 0; mode < 3; ++mode) {
        void (*fn)(uint32_t, int, uint32_t*) = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            fn<<<sms, 1024, smem>>>(words, iters, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double ops = (double)sms * 1024 * iters * 8;
        printf("mode %d (%s): %.3f ms, %.3e lane-atomics/s chip, %.2f per SM-clock @1.965GHz\n", mode,
               mode == 0 ? "random" : mode == 1 ? "distinct banks" : "distinct banks permuted", ms,
               ops / (ms * 1e-3), ops / (ms * 1e-3) / sms / 1.965e9);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
