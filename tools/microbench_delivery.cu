// Delivery ceiling microbenchmark (B200): how fast can the scatter-add of
// synaptic events into per-neuron accumulators go, and what limits it?
//
//   load-only   stream tgt (u32) + w (u64) entries, no stores     -> HBM bound
//   red-only    reds to hashed random targets, no entry loads     -> atomic bound
//   deliver     stream entries + red.add.u64 per entry            -> the real thing
//   red32       same with two 32-bit reds packed... (1 red.u32)   -> width effect
//   smem        stream entries, atomics into shared memory tiles  -> smem-atomic bound
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench_delivery.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e = (x);                                                   \
        if (e != cudaSuccess) {                                                \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            return 1;                                                          \
        }                                                                      \
    } while (0)

__device__ __forceinline__ uint32_t hash32(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    return (uint32_t)x;
}

__global__ void k_load(const uint32_t* __restrict__ tgt, const uint64_t* __restrict__ w,
                       uint64_t n, unsigned long long* sink) {
    uint64_t acc = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        acc += __ldcs(tgt + i) + __ldcs((const unsigned long long*)w + i);
    if (acc == 42) *sink = acc;
}

__global__ void k_red(uint64_t n, uint32_t nt, unsigned long long* acc) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t t = hash32(i) % nt;
        asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(acc + 2 * (size_t)t),
                     "l"((uint64_t)1) : "memory");
    }
}

__global__ void k_deliver(const uint32_t* __restrict__ tgt, const uint64_t* __restrict__ w,
                          uint64_t n, unsigned long long* acc) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t t = __ldcs(tgt + i);
        const uint64_t v = __ldcs((const unsigned long long*)w + i);
        asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(acc + 2 * (size_t)(t & 0x7fffffffu) + (t >> 31)),
                     "l"(v) : "memory");
    }
}

__global__ void k_red32(uint64_t n, uint32_t nt, unsigned int* acc) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t t = hash32(i) % nt;
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(acc + 4 * (size_t)t),
                     "r"(1u) : "memory");
    }
}

// targets restricted to a tile of `tile` neurons per CTA (smem accumulators)
__global__ void k_smem(uint64_t n, uint32_t tile) {
    extern __shared__ unsigned long long s[];
    for (uint32_t i = threadIdx.x; i < 2 * tile; i += blockDim.x) s[i] = 0;
    __syncthreads();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t t = hash32(i) % tile;
        atomicAdd(s + 2 * t, 1ull);
    }
}

int main() {
    const uint32_t nt = 1u << 20;  // 1M targets -> 16 MB accumulators (config 2)
    const uint64_t n = 1ull << 28;  // 268M events
    uint32_t* tgt;
    uint64_t* w;
    unsigned long long *acc, *sink;
    CK(cudaMalloc(&tgt, n * 4));
    CK(cudaMalloc(&w, n * 8));
    CK(cudaMalloc(&acc, 2ull * nt * 8));
    CK(cudaMalloc(&sink, 8));
    std::vector<uint32_t> h(n);
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t x = i * 0x9e3779b97f4a7c15ull;
        x ^= x >> 31;
        h[i] = (uint32_t)(x % nt) | ((x >> 40) & 1 ? 0x80000000u : 0u);
    }
    CK(cudaMemcpy(tgt, h.data(), n * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(w, 1, n * 8));
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto time = [&](auto launch) {
        launch();
        cudaEventRecord(a);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        return ms / 5;
    };
    const int g = sms * 8, t = 256;
    float ms;
    ms = time([&] { k_load<<<g, t>>>(tgt, w, n, sink); });
    printf("load-only : %.3f ms  %.3g entries/s  %.1f GB/s\n", ms, n / ms * 1e3, n * 12.0 / ms / 1e6);
    ms = time([&] { k_red<<<g, t>>>(n, nt, acc); });
    printf("red-only  : %.3f ms  %.3g reds/s (u64, 1M targets)\n", ms, n / ms * 1e3);
    ms = time([&] { k_red32<<<g, t>>>(n, nt, (unsigned int*)acc); });
    printf("red32-only: %.3f ms  %.3g reds/s (u32, 1M targets)\n", ms, n / ms * 1e3);
    ms = time([&] { k_deliver<<<g, t>>>(tgt, w, n, acc); });
    printf("deliver   : %.3f ms  %.3g events/s  %.1f GB/s entries\n", ms, n / ms * 1e3, n * 12.0 / ms / 1e6);
    for (uint32_t tile : {2048u, 8192u}) {
        CK(cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * tile));
        ms = time([&] { k_smem<<<g, t, 16 * tile>>>(n, tile); });
        printf("smem tile %5u: %.3f ms  %.3g atoms/s\n", tile, ms, n / ms * 1e3);
    }
    // smaller target sets: L2 locality of the accumulators
    for (uint32_t m : {1u << 14, 1u << 17, 1u << 22}) {
        ms = time([&] { k_red<<<g, t>>>(n, m, acc); });
        printf("red-only %8u targets: %.3g reds/s\n", m, n / ms * 1e3);
        if (m == (1u << 17)) break;
    }
    CK(cudaGetLastError());
    return 0;
}
