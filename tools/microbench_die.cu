// Does die locality matter for spike-delivery atomics on B200 (two dies)?
// 1. Latency probe: from one SM, the latency of an atomic to the first word
//    of every 64 KB page of a buffer (pages homed on the SM's own die should
//    answer faster), once from the lowest and once from the highest SM id.
// 2. Throughput: every SM issues red.add.u64 to hashed words of either the
//    pages classified "near" to its die or the "far" ones.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbdie tools/microbench_die.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e = (x);                                                          \
        if (e != cudaSuccess) {                                                       \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

__device__ __forceinline__ uint32_t smid() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

constexpr uint32_t kPage = 64 * 1024;

// one thread on the CTA that landed on SM `want`: dependent atomics per page
__global__ void probe(unsigned long long* buf, uint32_t pages, uint32_t want, uint32_t* lat,
                      int* found) {
    if (threadIdx.x != 0 || smid() != want) return;
    *found = 1;
    for (uint32_t p = 0; p < pages; ++p) {
        unsigned long long* a = buf + (size_t)p * (kPage / 8);
        unsigned long long v = atomicAdd(a, 1ull);  // warm the line
        long long t0 = clock64();
        for (int r = 0; r < 8; ++r) v = atomicAdd(a + (v >> 62), 1ull);
        long long t1 = clock64();
        lat[p] = (uint32_t)((t1 - t0) / 8) + (uint32_t)(v >> 62);
    }
}

// every CTA (one per SM): latency from this SM to page pa and to page pb
__global__ void probe_all(unsigned long long* buf, uint32_t pa, uint32_t pb, uint32_t* out) {
    if (threadIdx.x != 0) return;
    const uint32_t s = smid();
    uint32_t r[2];
    for (int k = 0; k < 2; ++k) {
        unsigned long long* a = buf + (size_t)(k ? pb : pa) * (kPage / 8) + 64 * (s + 1);
        unsigned long long v = atomicAdd(a, 1ull);
        long long t0 = clock64();
        for (int i = 0; i < 16; ++i) v = atomicAdd(a + (v >> 62), 1ull);
        r[k] = (uint32_t)((clock64() - t0) / 16) + (uint32_t)(v >> 62);
    }
    out[2 * s] = r[0];
    out[2 * s + 1] = r[1];
}

__device__ __forceinline__ uint32_t hash32(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    return (uint32_t)x;
}

// die of SM s = side[s]; CTA targets pages list[die ^ cross]
__global__ void __launch_bounds__(1024, 1) reds(unsigned long long* buf, const uint32_t* near0,
                                                uint32_t n0, const uint32_t* near1, uint32_t n1,
                                                const uint8_t* side, int cross, uint64_t per_cta) {
    extern __shared__ uint32_t spl[];
    const uint32_t d = side[smid()] ^ (uint32_t)cross;
    const uint32_t* pl = d ? near1 : near0;
    uint32_t np = min(d ? n1 : n0, 8192u);
    while (np & (np - 1)) np &= np - 1;  // power of two: mask instead of modulo
    for (uint32_t k = threadIdx.x; k < np; k += blockDim.x) spl[k] = pl[k];
    __syncthreads();
    for (uint64_t i = threadIdx.x; i < per_cta; i += blockDim.x) {
        const uint32_t h = hash32(i + per_cta * blockIdx.x);
        const uint32_t page = spl[h & (np - 1)];
        const uint32_t word = (h >> 13) & 255u;  // 4 KB of each page: the set stays L2-resident
        asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(buf + (size_t)page * (kPage / 8) + 2 * word),
                     "l"((uint64_t)1) : "memory");
    }
}

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint32_t pages = 4096;  // 256 MB
    unsigned long long* buf;
    uint32_t* lat;
    int* found;
    CK(cudaMalloc(&buf, (size_t)pages * kPage));
    CK(cudaMemset(buf, 0, (size_t)pages * kPage));
    CK(cudaMalloc(&lat, 4 * pages));
    CK(cudaMalloc(&found, 4));
    std::vector<uint32_t> l0(pages), l1(pages);
    for (int which = 0; which < 2; ++which) {
        const uint32_t want = which ? sms - 1 : 0;
        CK(cudaMemset(found, 0, 4));
        probe<<<sms * 2, 32>>>(buf, pages, want, lat, found);
        CK(cudaDeviceSynchronize());
        int f = 0;
        CK(cudaMemcpy(&f, found, 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(which ? l1.data() : l0.data(), lat, 4 * pages, cudaMemcpyDeviceToHost));
        std::vector<uint32_t> s(which ? l1 : l0);
        std::sort(s.begin(), s.end());
        printf("probe from SM %u (found %d): atomic latency cycles p10 %u p50 %u p90 %u\n", want, f,
               s[pages / 10], s[pages / 2], s[9 * pages / 10]);
    }
    {  // joint histogram of (latency from SM 0, latency from the last SM) in 100-cycle bins
        int hist[10][10] = {};
        for (uint32_t p = 0; p < pages; ++p)
            ++hist[std::min(9u, l0[p] / 100)][std::min(9u, l1[p] / 100)];
        printf("rows: latency from SM 0 (x100 cycles), cols: from the last SM\n");
        for (int a = 2; a < 10; ++a) {
            printf("%d:", a);
            for (int b = 2; b < 10; ++b) printf(" %5d", hist[a][b]);
            printf("\n");
        }
    }
    // classify: near to SM 0's die if faster from SM 0 than from the last SM
    std::vector<uint32_t> n0, n1;  // pages near / far from SM 0's die
    for (uint32_t p = 0; p < pages; ++p) (l0[p] < 450 ? n0 : n1).push_back(p);
    printf("pages nearer SM 0: %zu, nearer SM %d: %zu; first 16 classes:", n0.size(), sms - 1, n1.size());
    for (uint32_t p = 0; p < 16; ++p) printf(" %d", l0[p] < l1[p] ? 0 : 1);
    printf("\n");
    if (n0.empty() || n1.empty()) return 0;
    // die of each SM: probe one page of each class from every SM is costly; assume
    // SM ids split in halves and also test the alternative (even/odd)
    uint32_t *d0, *d1;
    uint8_t* side;
    CK(cudaMalloc(&d0, 4 * n0.size()));
    CK(cudaMalloc(&d1, 4 * n1.size()));
    CK(cudaMalloc(&side, 256));
    CK(cudaMemcpy(d0, n0.data(), 4 * n0.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(d1, n1.data(), 4 * n1.size(), cudaMemcpyHostToDevice));
    const int smem = 160 * 1024;
    CK(cudaFuncSetAttribute(reds, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(probe_all, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    const uint64_t per = 1ull << 21;
    std::vector<uint8_t> die(256, 0);
    {
        uint32_t* pr;
        CK(cudaMalloc(&pr, 8 * 256));
        CK(cudaMemset(pr, 0, 8 * 256));
        probe_all<<<sms, 32, 160 * 1024>>>(buf, n0[0], n1[0], pr);
        CK(cudaDeviceSynchronize());
        std::vector<uint32_t> h(512);
        CK(cudaMemcpy(h.data(), pr, 8 * 256, cudaMemcpyDeviceToHost));
        int c0 = 0;
        printf("die of SM (0 = SM 0's die):");
        for (int s = 0; s < sms; ++s) {
            die[s] = h[2 * s] < h[2 * s + 1] ? 0 : 1;
            c0 += die[s] == 0;
            printf("%s%d", s % 37 ? "" : "\n  ", die[s]);
        }
        printf("\n  %d SMs on die 0, %d on die 1\n", c0, sms - c0);
    }
    for (int layout = 0; layout < 3; ++layout) {
        std::vector<uint8_t> sd(256, 0);
        for (int s = 0; s < 256; ++s) sd[s] = layout == 0 ? (s >= sms / 2) : layout == 1 ? (s & 1) : die[s];
        CK(cudaMemcpy(side, sd.data(), 256, cudaMemcpyHostToDevice));
        for (int cross = 0; cross < 2; ++cross) {
            for (int w = 0; w < 2; ++w) {
                CK(cudaEventRecord(e0));
                reds<<<sms, 1024, smem>>>(buf, d0, (uint32_t)n0.size(), d1, (uint32_t)n1.size(), side,
                                          cross, per);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                CK(cudaGetLastError());
            }
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            printf("SM sides by %-8s targets %-5s: %.3g red/s\n", layout == 2 ? "probe" : layout ? "parity" : "id-half",
                   cross ? "far" : "near", (double)sms * per / (ms * 1e-3));
        }
    }
    return 0;
}
