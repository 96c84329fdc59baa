// Shared-memory-resident delivery microbenchmark (B200): every CTA owns a
// tile of targets whose pending accumulators live in its shared memory and
// delivers, for every spike of the step, the segment of the spike's
// target-sorted row that falls into its tile (per-source tile offsets),
// with shared-memory atomics.  Compared against the global red.add path.
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o mbsr tools/microbench_sr.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                           \
    do {                                                                                \
        cudaError_t e = (x);                                                            \
        if (e != cudaSuccess) {                                                         \
            printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);   \
            exit(1);                                                                    \
        }                                                                               \
    } while (0)

__host__ __device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

// stratified sorted targets: entry k of row s lies in [k*N/K, (k+1)*N/K)
__global__ void gen_rows(uint32_t n_src, uint32_t K, uint32_t N, uint32_t* tgt, uint64_t* w) {
    const uint64_t tot = (uint64_t)n_src * K;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < tot;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = (uint32_t)(i / K), k = (uint32_t)(i % K);
        const uint64_t lo = (uint64_t)k * N / K, hi = (uint64_t)(k + 1) * N / K;
        const uint64_t h = mix(i * 0x9e3779b97f4a7c15ull + 1);
        const uint32_t t = (uint32_t)(lo + h % (hi - lo));
        const uint32_t cls = (s % 5 == 0) ? 1u : 0u;
        tgt[i] = t | (cls << 31);
        w[i] = (uint64_t)(60000 + (h >> 40) % 10000) | ((uint64_t)(50000 + (h >> 20) % 10000) << 32);
    }
}

__global__ void tile_offsets(const uint32_t* tgt, uint32_t n_src, uint32_t K, uint32_t T,
                             uint32_t per, uint32_t* bo) {
    for (uint32_t s = blockIdx.x * blockDim.x + threadIdx.x; s < n_src; s += gridDim.x * blockDim.x) {
        const uint32_t* r = tgt + (uint64_t)s * K;
        uint32_t* o = bo + (uint64_t)s * (T + 1);
        uint32_t lo = 0;
        for (uint32_t b = 0; b <= T; ++b) {
            const uint64_t bound = (uint64_t)b * per;
            uint32_t hi = K;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if ((r[mid] & 0x7fffffffu) < bound) lo = mid + 1; else hi = mid;
            }
            o[b] = lo;
        }
    }
}

__global__ void ref_deliver(const uint32_t* spk, uint32_t S, const uint32_t* tgt, const uint64_t* w,
                            uint32_t K, unsigned long long* acc) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < (uint64_t)S * K;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t e = (uint64_t)spk[i / K] * K + i % K;
        const uint32_t t = tgt[e];
        atomicAdd(acc + 2 * (uint64_t)(t & 0x7fffffffu) + (t >> 31), (unsigned long long)w[e]);
    }
}

// packed (fast | slow << 32) add: one 64-bit shared atomic (a CAS loop in
// SASS) or two native 32-bit ATOMS.ADD (carry-free by construction)
template <bool W32>
__device__ __forceinline__ void sadd(unsigned long long* p, uint64_t v) {
    if constexpr (W32) {
        unsigned* q = reinterpret_cast<unsigned*>(p);
        atomicAdd(q, (unsigned)v);
        atomicAdd(q + 1, (unsigned)(v >> 32));
    } else {
        atomicAdd(p, (unsigned long long)v);
    }
}

// G lanes per segment, 32/G segments per round, R rounds unrolled
template <int G, bool W32>
__global__ void __launch_bounds__(1024, 1) sr_deliver(const uint32_t* __restrict__ spk, uint32_t S,
                                                      const uint32_t* __restrict__ tgt,
                                                      const uint64_t* __restrict__ w, uint32_t K,
                                                      const uint32_t* __restrict__ bo, uint32_t T,
                                                      uint32_t per, uint32_t N,
                                                      unsigned long long* out, int iters) {
    extern __shared__ unsigned long long sp[];
    constexpr int SPR = 32 / G;    // segments per round
    constexpr int R = 32 / SPR;    // rounds per 32 spikes
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t c = blockIdx.x, c_lo = c * per;
    for (uint32_t k = threadIdx.x; k < 2 * per; k += blockDim.x) sp[k] = 0;
    __syncthreads();
    for (int it = 0; it < iters; ++it) {
        const uint32_t* sl = spk + (size_t)it * S;
        for (uint32_t j0 = warp * 32; j0 < S; j0 += nw * 32) {
            uint64_t base = 0;
            uint32_t len = 0;
            if (j0 + lane < S) {
                const uint32_t s = __ldg(sl + j0 + lane);
                const uint32_t* o = bo + (uint64_t)s * (T + 1) + c;
                const uint32_t lo = __ldg(o), hi = __ldg(o + 1);
                base = (uint64_t)s * K + lo;
                len = hi - lo;
            }
            const uint32_t sub = lane % G, grp = lane / G;
            uint32_t tv[R];
            uint64_t wv[R];
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const uint32_t src = r * SPR + grp;
                const uint64_t b = __shfl_sync(0xffffffffu, base, src);
                const uint32_t l = __shfl_sync(0xffffffffu, len, src);
                tv[r] = 0xffffffffu;
                if (sub < l) {
                    tv[r] = __ldg(tgt + b + sub);
                    wv[r] = __ldg(reinterpret_cast<const unsigned long long*>(w) + b + sub);
                }
            }
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (tv[r] != 0xffffffffu)
                    sadd<W32>(sp + 2 * ((tv[r] & 0x7fffffffu) - c_lo) + (tv[r] >> 31), wv[r]);
            // tails longer than G: the whole warp, one segment at a time
            for (unsigned m = __ballot_sync(0xffffffffu, len > G); m; m &= m - 1) {
                const int l = __ffs(m) - 1;
                const uint64_t b = __shfl_sync(0xffffffffu, base, l);
                const uint32_t ln = __shfl_sync(0xffffffffu, len, l);
                for (uint32_t k = G + lane; k < ln; k += 32) {
                    const uint32_t t = __ldg(tgt + b + k);
                    const uint64_t v = __ldg(reinterpret_cast<const unsigned long long*>(w) + b + k);
                    sadd<W32>(sp + 2 * ((t & 0x7fffffffu) - c_lo) + (t >> 31), v);
                }
            }
        }
        __syncthreads();
    }
    for (uint32_t k = threadIdx.x; k < 2 * per; k += blockDim.x)
        if (c_lo * 2ull + k < 2ull * N) out[c_lo * 2ull + k] = sp[k];
}

// Flattened warp gather: a warp takes 32 spikes, compacts the non-empty
// segments to the low lanes, and walks their concatenation 32 entries at a
// time; the segment of entry q is found from the ends held in registers
// (ballot + redux.or + popc), so every lane loads a useful entry.
// MODE 0: loads + shared atomics, 1: loads only, 2: atomics only (hashed targets)
template <int MODE, bool W32, int U>
__global__ void __launch_bounds__(1024, 1) sr_flat(const uint32_t* __restrict__ spk, uint32_t S,
                                                   const uint32_t* __restrict__ tgt,
                                                   const uint64_t* __restrict__ w, uint32_t K,
                                                   const uint32_t* __restrict__ bo, uint32_t T,
                                                   uint32_t per, uint32_t N,
                                                   unsigned long long* out, int iters) {
    extern __shared__ unsigned long long sp[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t c = blockIdx.x, c_lo = c * per;
    const unsigned lt = (1u << lane) - 1u;
    for (uint32_t k = threadIdx.x; k < 2 * per; k += blockDim.x) sp[k] = 0;
    __syncthreads();
    uint64_t sink = 0;
    for (int it = 0; it < iters; ++it) {
        const uint32_t* sl = spk + (size_t)it * S;
        // bounds of the first batch
        auto bounds = [&](uint32_t j0, uint64_t& base, uint32_t& len) {
            base = 0;
            len = 0;
            if (j0 + lane < S) {
                const uint32_t s = __ldg(sl + j0 + lane);
                const uint32_t* o = bo + (uint64_t)s * (T + 1) + c;
                const uint32_t lo = __ldg(o), hi = __ldg(o + 1);
                base = (uint64_t)s * K + lo;
                len = hi - lo;
            }
        };
        uint64_t nbase;
        uint32_t nlen;
        bounds(warp * 32, nbase, nlen);
        for (uint32_t j0 = warp * 32; j0 < S; j0 += nw * 32) {
            uint64_t base = nbase;
            uint32_t len = nlen;
            bounds(j0 + nw * 32, nbase, nlen);  // next batch in flight
            // compact non-empty segments to lanes 0..m-1
            const unsigned nz = __ballot_sync(0xffffffffu, len != 0);
            const uint32_t m = __popc(nz);
            const uint32_t from = lane < m ? __fns(nz, 0, lane + 1) : 0u;
            base = __shfl_sync(0xffffffffu, base, from);
            len = __shfl_sync(0xffffffffu, len, from);
            if (lane >= m) len = 0;
            uint32_t end = len;  // inclusive scan
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, end, o);
                if (lane >= (uint32_t)o) end += y;
            }
            const uint32_t total = __shfl_sync(0xffffffffu, end, 31);
            if (lane >= m) end = 0xffffffffu;
            const uint64_t sbase = base - (end - len);  // entry index of concat position 0
            for (uint32_t e0 = 0; e0 < total; e0 += 32 * U) {
                uint32_t tv[U];
                uint64_t wv[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t c0 = e0 + 32 * u;
                    const uint32_t r0 = __popc(__ballot_sync(0xffffffffu, end <= c0));
                    const unsigned mk = __reduce_or_sync(
                        0xffffffffu, (end > c0 && end <= c0 + 32) ? 1u << (end - c0 - 1) : 0u);
                    const uint32_t src = min(r0 + __popc(mk & lt), 31u);
                    const uint64_t b = __shfl_sync(0xffffffffu, sbase, src);
                    const uint32_t q = c0 + lane;
                    tv[u] = 0xffffffffu;
                    if (q < total) {
                        if constexpr (MODE == 2) {
                            tv[u] = c_lo + (uint32_t)(mix(b + q) % per);
                            wv[u] = 1;
                        } else {
                            tv[u] = __ldg(tgt + b + q);
                            wv[u] = __ldg(reinterpret_cast<const unsigned long long*>(w) + b + q);
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (tv[u] != 0xffffffffu) {
                        if constexpr (MODE == 1)
                            sink += tv[u] + wv[u];
                        else
                            sadd<W32>(sp + 2 * ((tv[u] & 0x7fffffffu) - c_lo) + (tv[u] >> 31), wv[u]);
                    }
            }
        }
        __syncthreads();
    }
    if (sink == 42) sp[0] = 1;
    for (uint32_t k = threadIdx.x; k < 2 * per; k += blockDim.x)
        if (c_lo * 2ull + k < 2ull * N) out[c_lo * 2ull + k] = sp[k];
}

int main(int argc, char** argv) {
    const uint32_t N = 1000000, K = 1000, S = argc > 1 ? atoi(argv[1]) : 10000, ITERS = 20;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const uint32_t T = sms;
    const uint32_t per = (((N + T - 1) / T) + 31u) & ~31u;
    printf("N=%u K=%u S=%u spikes/step, tiles=%u x %u neurons (%u B smem)\n", N, K, S, T, per, per * 16);
    uint32_t *tgt, *bo, *spk;
    uint64_t* w;
    unsigned long long *acc, *out;
    CK(cudaMalloc(&tgt, 4ull * N * K));
    CK(cudaMalloc(&w, 8ull * N * K));
    CK(cudaMalloc(&bo, 4ull * N * (T + 1)));
    CK(cudaMalloc(&spk, 4ull * S * ITERS));
    CK(cudaMalloc(&acc, 16ull * N));
    CK(cudaMalloc(&out, 16ull * N));
    gen_rows<<<4096, 256>>>(N, K, N, tgt, w);
    tile_offsets<<<(N + 255) / 256, 256>>>(tgt, N, K, T, per, bo);
    std::vector<uint32_t> hs((size_t)S * ITERS);
    for (size_t i = 0; i < hs.size(); ++i) hs[i] = (uint32_t)(mix(i + 77) % N);
    CK(cudaMemcpy(spk, hs.data(), 4 * hs.size(), cudaMemcpyHostToDevice));
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    // reference: global atomics (also the timing of the current path's core)
    CK(cudaMemset(acc, 0, 16ull * N));
    ref_deliver<<<sms * 8, 256>>>(spk, S * ITERS, tgt, w, K, acc);
    CK(cudaMemset(acc, 0, 16ull * N));
    CK(cudaEventRecord(e0));
    ref_deliver<<<sms * 8, 256>>>(spk, S * ITERS, tgt, w, K, acc);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double ev = (double)S * K * ITERS;
    printf("global red : %.3f ms/step  %.3g events/s\n", ms / ITERS, ev / (ms * 1e-3));
    std::vector<unsigned long long> ha(2ull * N), hb(2ull * N);
    CK(cudaMemcpy(ha.data(), acc, 16ull * N, cudaMemcpyDeviceToHost));
    auto run = [&](auto kern, const char* name, int threads) {
        const int smem = per * 16;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        kern<<<T, threads, smem>>>(spk, S, tgt, w, K, bo, T, per, N, out, ITERS);  // warm
        CK(cudaEventRecord(e0));
        kern<<<T, threads, smem>>>(spk, S, tgt, w, K, bo, T, per, N, out, ITERS);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float m2 = 0;
        CK(cudaEventElapsedTime(&m2, e0, e1));
        CK(cudaMemcpy(hb.data(), out, 16ull * N, cudaMemcpyDeviceToHost));
        size_t bad = 0;
        for (size_t i = 0; i < ha.size(); ++i) bad += ha[i] != hb[i];
        printf("smem %-6s %4d thr: %.3f ms/step  %.3g events/s  %s\n", name, threads, m2 / ITERS,
               ev / (m2 * 1e-3), bad ? "MISMATCH" : "exact");
    };
    run(sr_deliver<8, true>, "G=8x32", 1024);
    for (int th : {512, 1024}) {
        run(sr_flat<0, true, 2>, "flat32u2", th);
        run(sr_flat<0, true, 4>, "flat32u4", th);
        run(sr_flat<0, false, 4>, "flat64u4", th);
        run(sr_flat<1, true, 4>, "loadonly", th);
        run(sr_flat<2, true, 4>, "atom32", th);
        run(sr_flat<2, false, 4>, "atom64", th);
    }
    return 0;
}
