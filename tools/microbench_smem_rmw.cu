// Shared-memory accumulation rates on B200 for spike delivery into
// SM-resident pending tiles: per-warp owned target ranges updated with plain
// LDS/STS read-modify-writes (duplicates inside a warp merged first with
// match.any), against shared atomics (2 x ATOMS.ADD.32 or the 64-bit CAS
// loop) on the same addresses.  Targets are hashed (no global loads): this
// isolates the shared-memory side of the delivery.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbrmw tools/microbench_smem_rmw.cu
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

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

// MODE 0: match.any merge + plain RMW (warp-owned range)
// MODE 1: 2 x atomicAdd u32 (warp-owned range)
// MODE 2: atomicAdd u64 (CAS loop) (warp-owned range)
// MODE 3: 2 x atomicAdd u32, targets over the whole tile
template <int MODE>
__global__ void __launch_bounds__(1024, 1) k_acc(uint32_t per_warp_events, uint32_t tile,
                                                 unsigned long long* out) {
    extern __shared__ unsigned long long acc[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (uint32_t k = threadIdx.x; k < 2 * tile; k += blockDim.x) acc[k] = 0;
    __syncthreads();
    const uint32_t R = tile / nw, lo = warp * R;
    unsigned long long expect = 0;
    uint32_t x = (blockIdx.x * 1024 + threadIdx.x) * 0x9e3779b9u;
    for (uint32_t e = 0; e < per_warp_events; e += 32) {
        x = hash32(x + e);
        const uint32_t t = MODE == 3 ? x % tile : lo + x % R;
        const uint32_t cls = (x >> 28) & 1u;
        const uint64_t v = (uint64_t)((x & 0xffffu) + 1u) | ((uint64_t)(((x >> 8) & 0xffu) + 1u) << 32);
        expect += v;
        unsigned long long* p = acc + 2 * t + cls;
        if constexpr (MODE == 0) {
            const unsigned peers = __match_any_sync(0xffffffffu, 2 * t + cls);
            const int leader = __ffs(peers) - 1;
            uint64_t s = v;
            for (unsigned m = peers & ~(1u << leader); m; m &= m - 1)  // rare
                s += __shfl_sync(peers, v, __ffs(m) - 1);
            if ((int)lane == leader) *p += s;
        } else if constexpr (MODE == 1 || MODE == 3) {
            unsigned* q = reinterpret_cast<unsigned*>(p);
            atomicAdd(q, (unsigned)v);
            atomicAdd(q + 1, (unsigned)(v >> 32));
        } else {
            atomicAdd(p, (unsigned long long)v);
        }
    }
    __syncthreads();
    unsigned long long sum = 0;
    for (uint32_t k = threadIdx.x; k < 2 * tile; k += blockDim.x) sum += acc[k];
    atomicAdd(out, sum);
    atomicAdd(out + 1, expect);
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    unsigned long long* out;
    CK(cudaMalloc(&out, 16));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const uint32_t tile = 6784, per_warp = 1u << 16;
    const int smem = tile * 16;
    auto run = [&](auto kern, const char* name, int threads) -> int {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        for (int w = 0; w < 2; ++w) {
            CK(cudaMemset(out, 0, 16));
            CK(cudaEventRecord(e0));
            kern<<<sms, threads, smem>>>(per_warp, tile, out);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            CK(cudaGetLastError());
        }
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        unsigned long long h[2] = {0, 0};
        CK(cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost));
        const double ev = (double)sms * (threads / 32) * per_warp;
        printf("%-22s %4d thr: %.3g events/s  %.3f events/cycle/SM  check %s\n", name, threads,
               ev / (ms * 1e-3), ev / (ms * 1e-3) / sms / 1.965e9,
               h[0] == h[1] ? "ok" : "BAD");
        return 0;
    };
    for (int th : {256, 512, 1024}) {
        run(k_acc<0>, "match.any + plain RMW", th);
        run(k_acc<1>, "2 x ATOMS.ADD.32", th);
        run(k_acc<2>, "ATOMS CAS u64", th);
        run(k_acc<3>, "2 x ATOMS.32 whole tile", th);
    }
    return 0;
}
