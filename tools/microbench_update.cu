// Memory-pattern microbenchmark of the l2 path's neuron update on one B200:
// per neuron read v (4 B), i_ou (4), j (16), g (16), pending (16) and write
// v, i_ou, j and zero the pending (16): 96 B/neuron, 20M neurons (config 3,
// not L2-resident).  Variants: DEPTH chunks of 32 neurons in flight per warp
// (registers), and a TMA variant (cp.async.bulk of each chunk's five arrays
// into a per-warp shared-memory ring of DEPTH stages).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_upd tools/microbench_update.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct Arr { float* v; float* iou; float4* j; float4* g; ulonglong2* p; };

template <int DEPTH, int TPB>
__global__ void __launch_bounds__(TPB) upd_regs(Arr a, uint32_t n) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warps = gridDim.x * (TPB / 32);
    const uint32_t w = blockIdx.x * (TPB / 32) + (threadIdx.x >> 5);
    const uint32_t nch = n / 32;
    float v[DEPTH], io[DEPTH]; float4 j[DEPTH], g[DEPTH]; ulonglong2 p[DEPTH];
    uint32_t c = w;
#pragma unroll
    for (int d = 0; d < DEPTH; ++d) {
        const uint32_t cc = c + d * warps;
        if (cc < nch) { const uint32_t i = cc * 32 + lane; v[d] = a.v[i]; io[d] = a.iou[i]; j[d] = a.j[i]; g[d] = a.g[i]; p[d] = __ldcg(a.p + i); }
    }
    for (; c < nch; c += warps * DEPTH) {
#pragma unroll
        for (int d = 0; d < DEPTH; ++d) {
            const uint32_t cc = c + d * warps;
            if (cc >= nch) break;
            const uint32_t i = cc * 32 + lane;
            float4 jj = j[d];
            jj.x = jj.x * 0.9f + g[d].x * (float)(p[d].x & 0xffff);
            jj.y = jj.y * 0.9f + g[d].y * (float)(p[d].x >> 32);
            jj.z = jj.z * 0.9f + g[d].z * (float)(p[d].y & 0xffff);
            jj.w = jj.w * 0.9f + g[d].w * (float)(p[d].y >> 32);
            a.j[i] = jj; a.v[i] = v[d] + jj.x; a.iou[i] = io[d] * 0.99f; a.p[i] = make_ulonglong2(0, 0);
            const uint32_t cn = cc + DEPTH * warps;
            if (cn < nch) { const uint32_t k = cn * 32 + lane; v[d] = a.v[k]; io[d] = a.iou[k]; j[d] = a.j[k]; g[d] = a.g[k]; p[d] = __ldcg(a.p + k); }
        }
    }
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int DEPTH, int TPB>
__global__ void __launch_bounds__(TPB) upd_tma(Arr a, uint32_t n) {
    extern __shared__ __align__(128) unsigned char sm[];
    constexpr uint32_t CH = 32 * (4 + 4 + 16 + 16 + 16);  // 1792 B per chunk
    const uint32_t lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    unsigned char* ring = sm + wl * (DEPTH * CH + 8 * DEPTH);
    uint64_t* bar = reinterpret_cast<uint64_t*>(ring + DEPTH * CH);
    const uint32_t warps = gridDim.x * (TPB / 32);
    const uint32_t w = blockIdx.x * (TPB / 32) + wl;
    const uint32_t nch = n / 32;
    if (lane == 0) for (int d = 0; d < DEPTH; ++d) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(bar + d)));
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    auto issue = [&](uint32_t cc, int d) {
        if (lane == 0 && cc < nch) {
            unsigned char* st = ring + d * CH;
            const uint32_t b = su32(bar + d);
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(CH) : "memory");
            const size_t i0 = (size_t)cc * 32;
            asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(st)), "l"(a.v + i0), "r"(128u), "r"(b) : "memory");
            asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(st + 128)), "l"(a.iou + i0), "r"(128u), "r"(b) : "memory");
            asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(st + 256)), "l"(a.j + i0), "r"(512u), "r"(b) : "memory");
            asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(st + 768)), "l"(a.g + i0), "r"(512u), "r"(b) : "memory");
            asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(st + 1280)), "l"(a.p + i0), "r"(512u), "r"(b) : "memory");
        }
    };
    uint32_t c = w;
    for (int d = 0; d < DEPTH; ++d) issue(c + d * warps, d);
    uint32_t phase = 0;
    for (int d = 0; c < nch; c += warps) {
        const uint32_t b = su32(bar + d);
        asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(b), "r"((phase >> d) & 1u) : "memory");
        phase ^= 1u << d;
        unsigned char* st = ring + d * CH;
        const uint32_t i = c * 32 + lane;
        float v = reinterpret_cast<float*>(st)[lane], io = reinterpret_cast<float*>(st + 128)[lane];
        float4 jj = reinterpret_cast<float4*>(st + 256)[lane];
        const float4 g = reinterpret_cast<float4*>(st + 768)[lane];
        const ulonglong2 p = reinterpret_cast<ulonglong2*>(st + 1280)[lane];
        __syncwarp();
        issue(c + DEPTH * warps, d);
        jj.x = jj.x * 0.9f + g.x * (float)(p.x & 0xffff);
        jj.y = jj.y * 0.9f + g.y * (float)(p.x >> 32);
        jj.z = jj.z * 0.9f + g.z * (float)(p.y & 0xffff);
        jj.w = jj.w * 0.9f + g.w * (float)(p.y >> 32);
        a.j[i] = jj; a.v[i] = v + jj.x; a.iou[i] = io * 0.99f; a.p[i] = make_ulonglong2(0, 0);
        d = d + 1 == DEPTH ? 0 : d + 1;
    }
}

int main() {
    const uint32_t n = 20000000;
    Arr a;
    cudaMalloc(&a.v, 4ull * n); cudaMalloc(&a.iou, 4ull * n); cudaMalloc(&a.j, 16ull * n);
    cudaMalloc(&a.g, 16ull * n); cudaMalloc(&a.p, 16ull * n);
    cudaMemset(a.v, 0, 4ull * n); cudaMemset(a.iou, 0, 4ull * n); cudaMemset(a.j, 0, 16ull * n);
    cudaMemset(a.g, 0, 16ull * n); cudaMemset(a.p, 0, 16ull * n);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const double bytes = 96.0 * n;
    auto run = [&](const char* name, auto fn, int blocks, int tpb, size_t smem) {
        if (smem) cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int r = 0; r < 2; ++r) fn<<<blocks, tpb, smem>>>(a, n);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) fn<<<blocks, tpb, smem>>>(a, n);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
        printf("%-28s %7.1f us  %6.2f TB/s  (%s)\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    };
    run("regs depth1 24 warps/SM", upd_regs<1, 256>, sms * 3, 256, 0);
    run("regs depth2 24 warps/SM", upd_regs<2, 256>, sms * 3, 256, 0);
    run("regs depth3 24 warps/SM", upd_regs<3, 256>, sms * 3, 256, 0);
    run("regs depth1 48 warps/SM", upd_regs<1, 256>, sms * 6, 256, 0);
    run("regs depth2 48 warps/SM", upd_regs<2, 256>, sms * 6, 256, 0);
    run("tma depth2 24 warps/SM", upd_tma<2, 256>, sms * 3, 256, 8 * (2 * 1792 + 16));
    run("tma depth3 24 warps/SM", upd_tma<3, 256>, sms * 3, 256, 8 * (3 * 1792 + 24));
    run("tma depth4 24 warps/SM", upd_tma<4, 256>, sms * 3, 256, 8 * (4 * 1792 + 32));
    run("tma depth4 16 warps/SM", upd_tma<4, 256>, sms * 2, 256, 8 * (4 * 1792 + 32));
    return 0;
}
