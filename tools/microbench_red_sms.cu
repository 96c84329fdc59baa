// Where is the scattered-atomic ceiling of spike delivery: in the SMs
// (LSU issue per lane) or in L2 (atomic units per slice)?  Runs red-only
// scatter-adds from k SMs (one 1024-thread CTA per SM, pinned by shared
// memory) for growing k: if the rate grows linearly up to 148 SMs the SM
// side is the limit, if it flattens the L2 side is.  Also times TMA bulk
// reductions (cp.reduce.async.bulk .add.u64, 16 B per event) as the
// alternative issue path.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbred tools/microbench_red_sms.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e = (x);                                                          \
        if (e != cudaSuccess) {                                                       \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

__device__ __forceinline__ uint32_t hash32(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    return (uint32_t)x;
}

__global__ void __launch_bounds__(1024, 1) k_red(uint64_t per_cta, uint32_t nt, unsigned long long* acc) {
    extern __shared__ unsigned char pin[];
    for (uint64_t i = threadIdx.x; i < per_cta; i += blockDim.x) {
        const uint32_t t = hash32(i + per_cta * blockIdx.x) % nt;
        asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(acc + 2 * (size_t)t),
                     "l"((uint64_t)1) : "memory");
    }
    if (per_cta == 0) pin[0] = 0;
}

// TMA bulk reduction: each thread reduces a 16-B smem record into the
// target's 16-B pending record
__global__ void __launch_bounds__(1024, 1) k_bulkred(uint64_t per_cta, uint32_t nt, unsigned long long* acc) {
    extern __shared__ __align__(16) unsigned long long src[];
    src[2 * threadIdx.x] = 1;
    src[2 * threadIdx.x + 1] = 0;
    __syncthreads();
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(src + 2 * threadIdx.x);
    uint32_t n = 0;
    for (uint64_t i = threadIdx.x; i < per_cta; i += blockDim.x) {
        const uint32_t t = hash32(i + per_cta * blockIdx.x) % nt;
        asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], 16;"
                     ::"l"(acc + 2 * (size_t)t), "r"(sa) : "memory");
        if (++n == 8) {
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
            n = 0;
        }
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const uint32_t nt = 1u << 20;
    unsigned long long* acc;
    CK(cudaMalloc(&acc, 16ull * nt));
    CK(cudaMemset(acc, 0, 16ull * nt));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int smem = 160 * 1024;  // one CTA per SM
    CK(cudaFuncSetAttribute(k_red, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(k_bulkred, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const uint64_t per_cta = 1ull << 21;
    for (int pass = 0; pass < 2; ++pass)
        for (int k : {1, 8, 16, 37, 74, 111, 148}) {
            if (k > sms) continue;
            for (int warm = 0; warm < 2; ++warm) {
                CK(cudaEventRecord(e0));
                if (pass == 0)
                    k_red<<<k, 1024, smem>>>(per_cta, nt, acc);
                else
                    k_bulkred<<<k, 1024, smem>>>(per_cta / 4, nt, acc);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                CK(cudaGetLastError());
            }
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            const double ops = (double)k * (pass == 0 ? per_cta : per_cta / 4);
            printf("%-9s SMs=%3d  %.3g ops/s  %.3f ops/cycle/SM (at 1.965 GHz)\n",
                   pass == 0 ? "red.u64" : "bulk-red", k, ops / (ms * 1e-3),
                   ops / (ms * 1e-3) / k / 1.965e9);
        }
    return 0;
}
